#!/usr/bin/env python3
"""Generate tests/golden/*.json from the reference itself.

Runs the reference dcpsim library compiled from /root/reference sources
(oracle/_ref/libdcpsim_ref.so, `make -C oracle`) on the SPEC known-answer
inputs (SPEC.md examples) and on seeded planner scenarios,
and records inputs + outputs as small JSON fixtures.  The fixtures travel with
the repo, so tests pin the oracle port and the device planner even where
/root/reference is absent.

    python tools/make_golden.py
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests import oracle_lib  # noqa: E402
from tests.oracle_lib import P, World  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
I64MAX = 2**63 - 1


def water_fill(L, K, ell):
    n = len(K)
    parts = np.arange(n, dtype=np.int32)
    loads = np.array(K, np.int64)
    split = np.zeros(n, np.int64)
    assert L.dcpref_water_fill(n, P(parts), ell, P(loads), P(split)) == 0
    return split.tolist()


def cp_degree(L, ell, node, bucket=None):
    if bucket:
        bl = np.array([b[0] for b in bucket], np.int64)
        bd = np.array([b[1] for b in bucket], np.int32)
        return L.dcpref_cp_degree(ell, P(bl), P(bd), len(bucket), node)
    return L.dcpref_cp_degree(ell, None, None, 0, node)


def run_scenario(L, sc):
    w = World(L, "dcpref_", sc["nodes"], sc["ipn"], sc["page"], sc["capacity"], sc["kind"],
              sc.get("bucket"), sc.get("uniform_degree", 1), sc.get("hol_strict", True))
    steps = []
    for ev in sc["events"]:
        if ev[0] == "enqueue":
            w.enqueue(ev[1], ev[2])
        elif ev[0] == "step":
            steps.append(w.step())
        elif ev[0] == "finish":
            assert w.finish(ev[1]) == 0
        elif ev[0] == "append":
            rc, inst = w.append_token(ev[1])
            steps.append({"append": ev[1], "instance": inst, "rc": rc})
    ids = sorted({e[1] for e in sc["events"] if e[0] == "enqueue"})
    out = {"steps": steps, "instances": w.instances(),
           "placements": {str(i): w.placement(i) for i in ids}}
    for key, text in (("page_table_csv", w.page_table_csv()), ("routing_csv", w.routing_csv())):
        out[key + "_sha256"] = hashlib.sha256(text.encode()).hexdigest()
        out[key + "_lines"] = text.count("\n")
        if len(text) <= 16384:
            out[key] = text
    return out


def scenarios(L):
    sc = []
    # SPEC.md:222 / SURVEY App. A: 1x2, K=(100K,100K), new 600K -> split {300K,300K}
    sc.append(dict(name="spec_dcp_600k", nodes=1, ipn=2, page=16, capacity=40000, kind="dcp",
                   events=[["enqueue", 0, 100000], ["enqueue", 1, 100000], ["step"],
                           ["enqueue", 2, 600000], ["step"]]))
    # page table l=40 split {A:30,B:10}
    sc.append(dict(name="spec_page_table_40", nodes=1, ipn=2, page=16, capacity=8, kind="dcp",
                   bucket=[[39, 1], [I64MAX, 2]],
                   events=[["enqueue", 0, 10], ["step"], ["enqueue", 1, 30], ["step"],
                           ["enqueue", 2, 40], ["step"], ["finish", 2], ["step"]]))
    # zero-token MoE binding; K=(1000,5), l=100 -> {0,100}, m_r=0
    sc.append(dict(name="zero_token_moe_binding", nodes=1, ipn=2, page=16, capacity=256, kind="dcp",
                   bucket=[[999, 1], [I64MAX, 2]],
                   events=[["enqueue", 0, 1000], ["step"], ["enqueue", 1, 5], ["step"],
                           ["enqueue", 2, 100], ["step"]]))
    # append_token fallback leaves a non-final partial page
    sc.append(dict(name="append_fallback", nodes=1, ipn=2, page=16, capacity=4, kind="dcp",
                   bucket=[[31, 1], [I64MAX, 2]],
                   events=[["enqueue", 9, 46], ["step"]] + [["append", 9]] * 20 +
                          [["enqueue", 10, 3], ["step"]] + [["append", 10]] * 30))
    # 2x4 cluster, 5%-long trace seed 42, 100 requests, one DCP step
    n = 400
    ids, sl, arr, ol = (np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(n), np.zeros(n, np.int64))
    cnt = L.dcpref_gen_trace(42, 0.05, 100.0, 1.0, 0, P(ids), P(sl), P(arr), P(ol), n)
    ev = [["enqueue", int(ids[i]), int(sl[i])] for i in range(min(cnt, 100))] + [["step"]]
    sc.append(dict(name="trace42_2x4_5pct", nodes=2, ipn=4, page=16, capacity=200000, kind="dcp",
                   hol_strict=True, events=ev))
    # baselines on the same trace
    for kind, extra in (("least_batch", {}), ("least_cache", {}), ("uniform", {"uniform_degree": 2}),
                        ("uniform", {"uniform_degree": 4})):
        d = dict(name=f"trace42_2x4_{kind}{extra.get('uniform_degree', '')}", nodes=2, ipn=4, page=16,
                 capacity=200000, kind=kind, events=ev)
        d.update(extra)
        sc.append(d)
    # HoL: tight capacity, strict and non-strict
    rng = np.random.default_rng(5)
    ev2 = []
    for i in range(60):
        ev2.append(["enqueue", i, int(rng.integers(1, 3000))])
    ev2 += [["step"], ["finish", 3], ["finish", 7], ["step"], ["finish", 11], ["step"]]
    for strict in (True, False):
        sc.append(dict(name=f"hol_tight_strict{int(strict)}", nodes=1, ipn=4, page=16, capacity=300,
                       kind="dcp", bucket=[[1000, 1], [2000, 2], [I64MAX, 4]], hol_strict=strict,
                       events=ev2))
    return sc


def two_schedulers():
    """tests/cpp/dropin_two_schedulers.cpp compiled against the reference headers and the
    reference library (-Ddcpsim=dcpsim_ref); its stdout is the drop-in's expected output."""
    import subprocess
    import tempfile
    ref = "/root/reference/proj"
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "two")
        lib = os.path.join(ROOT, "oracle", "_ref")
        subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-Ddcpsim=dcpsim_ref", f"-I{ref}/include",
                        os.path.join(ROOT, "tests", "cpp", "dropin_two_schedulers.cpp"), "-o", exe, f"-L{lib}",
                        "-ldcpsim_ref", f"-Wl,-rpath,{lib}", "-fopenmp"], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    with open(os.path.join(OUT, "two_schedulers.txt"), "w") as f:
        f.write(out)


def main():
    two_schedulers()
    L = oracle_lib.reference()
    if L is None:
        raise SystemExit("build oracle/_ref first: make -C oracle")
    os.makedirs(OUT, exist_ok=True)
    kat = {
        "water_fill": [dict(K=K, ell=ell, split=water_fill(L, K, ell)) for K, ell in
                       [([10, 30], 40), ([0, 0, 50], 60), ([5, 5, 5], 10), ([50, 0], 10),
                        ([100], 100), ([1000, 5], 100), ([100000, 100000], 600000),
                        ([7, 3, 9, 0, 0, 1, 2, 2], 1000), ([0] * 8, 524288)]],
        "cp_degree": [dict(ell=ell, node=node, k=cp_degree(L, ell, node)) for ell, node in
                      [(2048, 8), (32768, 8), (32769, 8), (131072, 8), (131073, 8), (393216, 8),
                       (393217, 8), (524288, 8), (524288, 4), (524288, 2), (1, 1)]],
        "bucket_shape": [],
        "footprint": [],
    }
    for m, n in [(5, 9), (17, 4), (200, 500), (8, 8), (1, 1), (256, 512), (0, 0), (65, 257)]:
        bm, bn = ctypes.c_int(), ctypes.c_int()
        rc = L.dcpref_bucket_shape_default(m, n, ctypes.byref(bm), ctypes.byref(bn))
        kat["bucket_shape"].append(dict(m=m, n=n, rc=rc, bm=bm.value, bn=bn.value))
    for m, n in [(257, 1), (1, 513)]:
        bm, bn = ctypes.c_int(), ctypes.c_int()
        kat["bucket_shape"].append(dict(m=m, n=n, rc=L.dcpref_bucket_shape_default(m, n, ctypes.byref(bm), ctypes.byref(bn))))
    for args in [(1, 128, 64, 7168, 1024, 2, 4), (8, 128, 64, 7168, 1024, 2, 4), (2, 32, 128, 2048, 2048, 2, 4)]:
        g, b = ctypes.c_int64(), ctypes.c_int64()
        assert L.dcpref_graph_footprint(*args, ctypes.byref(g), ctypes.byref(b)) == 0
        kat["footprint"].append(dict(args=list(args), graphs=g.value, bytes=b.value))
    lens = np.zeros(64, np.int64)
    L.dcpref_uniform_int(0, 1024, 32768, 64, P(lens))
    kat["cfg2_lengths"] = lens.tolist()
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(kat, f, indent=1)
    scen = scenarios(L)
    res = []
    for sc in scen:
        r = run_scenario(L, sc)
        res.append(dict(scenario=sc, result=r))
    with open(os.path.join(OUT, "planner_scenarios.json"), "w") as f:
        json.dump(res, f)
    print(f"wrote {OUT}/known_answers.json, planner_scenarios.json ({len(res)} scenarios)")


if __name__ == "__main__":
    main()
