"""The dcpsim C++ drop-in (include/dcpsim/*.hpp, device-backed) vs the oracle.

Two C++ programs written purely against the reference-shaped headers are
compiled with g++ and linked to libdcp_b200.so — as an existing caller of the
reference would relink:
  * dropin_examples: SPEC known-answer examples (water_fill, cp_degree, page
    table layout / lookup / free / LIFO reuse / InsufficientFrames,
    rebalance_active, routing invariants, bucket_shape, footprint, fp32
    sharded_attention_merge rel-L2 <= 1e-5, EmptyShard);
  * dropin_driver: replays seeded planner scripts through Scheduler::step /
    pt_free / append_token / build_binding_config / derive_routing_tables and
    prints results that must equal the oracle port's, byte for byte.
"""
import os
import subprocess

import numpy as np
import pytest

from tests import oracle_lib
from tests.oracle_lib import World
from tests.test_oracle import _random_world_script

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
LIBDIR = os.path.join(ROOT, "paper_2605_21100_b200", "_build")


def _compile(name):
    os.makedirs(BUILD, exist_ok=True)
    out = os.path.join(BUILD, name)
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT}/include", src, "-o", out, f"-L{LIBDIR}",
                    "-ldcp_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return out


@pytest.fixture(scope="module")
def driver():
    return _compile("dropin_driver")


def test_spec_examples_through_cpp_api():
    exe = _compile("dropin_examples")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ALL OK" in p.stdout, p.stdout + p.stderr


KIND = {"dcp": 0, "least_batch": 1, "least_cache": 2, "uniform": 3}


def _script_text(sc):
    lines = [f"cluster {sc['nodes']} {sc['ipn']} {sc['page']} {sc['capacity']}"]
    b = sc.get("bucket") or []
    lines.append(f"policy {KIND[sc['kind']]} {int(sc.get('hol_strict', True))} {sc.get('uniform_degree', 1)} {len(b)} "
                 + " ".join(f"{x[0]} {x[1]}" for x in b))
    for ev in sc["events"]:
        if ev[0] == "enqueue":
            lines.append(f"enqueue {ev[1]} {ev[2]}")
        elif ev[0] == "step":
            lines.append("step")
        elif ev[0] in ("finish", "finish?"):
            lines.append(f"finish {ev[1]}")
        elif ev[0] == "append":
            lines.append(f"append {ev[1]}")
    lines.append("end")
    return "\n".join(lines) + "\n"


def _j(v):
    return ",".join(str(x) for x in v)


def _oracle_text(sc):
    w = World(oracle_lib.port(), "dcpora_", sc["nodes"], sc["ipn"], sc["page"], sc["capacity"], sc["kind"],
              sc.get("bucket"), sc.get("uniform_degree", 1), sc.get("hol_strict", True))
    out, enq = [], []
    for ev in sc["events"]:
        if ev[0] == "enqueue":
            w.enqueue(ev[1], ev[2])
            enq.append(ev[1])
        elif ev[0] == "step":
            r = w.step()
            out.append(f"step c={_j(r['committed'])} d={_j(r['deferred'])} u={_j(r['unschedulable'])} "
                       f"hol={r['hol_events']}")
        elif ev[0] in ("finish", "finish?"):
            out.append(f"finish {w.finish(ev[1])}")
        elif ev[0] == "append":
            rc, inst = w.append_token(ev[1])
            out.append(f"append {rc} {inst if rc == 0 else 0}")
    st = w.instances()
    out.append(f"instances kv={_j(st['kv_load'])} b={_j(st['moe_batch'])} sc={_j(st['shard_count'])} "
               f"free={_j(st['free'])}")
    for i in enq:
        p = w.placement(i)
        out.append(f"placement {i} none" if p is None else f"placement {i} {_j(p['kv'])} {_j(p['split'])} {p['moe']}")
    return "\n".join(out) + "\n" + w.page_table_csv() + w.routing_csv()


def test_cpp_api_matches_oracle_on_random_scripts(driver):
    rng = np.random.default_rng(23)
    for trial in range(25):
        sc = _random_world_script(rng)
        p = subprocess.run([driver], input=_script_text(sc), capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
        assert p.stdout == _oracle_text(sc), f"trial {trial}"


def test_two_schedulers_share_a_cluster():
    """UniformCP round-robin state is per Scheduler (reference scheduler.hpp:88): two
    Schedulers (plus a LeastBatch one) interleaved on one cluster print exactly what the
    reference printed for the same program (tests/golden/two_schedulers.txt)."""
    exe = _compile("dropin_two_schedulers")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    with open(os.path.join(ROOT, "tests", "golden", "two_schedulers.txt")) as f:
        assert p.stdout == f.read()
