"""Pin the CPU oracle port (oracle/dcp_oracle.c) before trusting it.

1. Against the committed golden fixtures (tests/golden/, generated from the
   reference itself by tools/make_golden.py) — works without /root/reference.
2. Against the reference compiled from its own sources (oracle/_ref) on seeded
   random inputs: bit-exact for all integer work, bit-exact fp64 attention.
3. The SPEC acceptance criteria AC1, AC2, AC3, AC11.
"""
import ctypes
import hashlib
import itertools
import json
import os

import numpy as np
import pytest

from tests import oracle_lib
from tests.oracle_lib import P, World

GOLD = os.path.join(os.path.dirname(__file__), "golden")
I64MAX = 2**63 - 1


@pytest.fixture(scope="module")
def port():
    return oracle_lib.port()


@pytest.fixture(scope="module")
def ref():
    L = oracle_lib.reference()
    if L is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return L


def _wf(L, prefix, K, ell):
    n = len(K)
    split = np.zeros(n, np.int64)
    rc = getattr(L, prefix + "water_fill")(n, P(np.arange(n, dtype=np.int32)), ell, P(np.array(K, np.int64)),
                                           P(split))
    assert rc == 0
    return split.tolist()


# ------------------------------------------------------------------ golden fixtures
def test_known_answers(port):
    kat = json.load(open(os.path.join(GOLD, "known_answers.json")))
    for c in kat["water_fill"]:
        assert _wf(port, "dcpora_", c["K"], c["ell"]) == c["split"], c
    for c in kat["cp_degree"]:
        assert port.dcpora_cp_degree(c["ell"], None, None, 0, c["node"]) == c["k"], c
    for c in kat["bucket_shape"]:
        bm, bn = ctypes.c_int(), ctypes.c_int()
        rc = port.dcpora_bucket_shape_default(c["m"], c["n"], ctypes.byref(bm), ctypes.byref(bn))
        assert rc == c["rc"]
        if rc == 0:
            assert (bm.value, bn.value) == (c["bm"], c["bn"])
    for c in kat["footprint"]:
        g, b = ctypes.c_int64(), ctypes.c_int64()
        port.dcpora_graph_footprint(*c["args"], ctypes.byref(g), ctypes.byref(b))
        assert (g.value, b.value) == (c["graphs"], c["bytes"])
    lens = np.zeros(64, np.int64)
    port.dcpora_uniform_int(0, 1024, 32768, 64, P(lens))
    assert lens.tolist() == kat["cfg2_lengths"] and int(lens.sum()) == 1068741


def test_spec_examples_pinned():
    kat = json.load(open(os.path.join(GOLD, "known_answers.json")))
    wf = {(tuple(c["K"]), c["ell"]): c["split"] for c in kat["water_fill"]}
    assert wf[((10, 30), 40)] == [30, 10]
    assert wf[((0, 0, 50), 60)] == [30, 30, 0]
    assert wf[((5, 5, 5), 10)] == [4, 3, 3]        # scheduler.cpp:94-100
    assert wf[((50, 0), 10)] == [0, 10]
    cp = {(c["ell"], c["node"]): c["k"] for c in kat["cp_degree"]}
    assert cp[(2048, 8)] == 1 and cp[(524288, 8)] == 8 and cp[(524288, 4)] == 4
    fp = kat["footprint"]
    assert fp[0]["graphs"] == 48 and fp[0]["bytes"] == 17368064 and fp[1]["bytes"] == 105907200


def _replay(L, prefix, sc):
    w = World(L, prefix, sc["nodes"], sc["ipn"], sc["page"], sc["capacity"], sc["kind"], sc.get("bucket"),
              sc.get("uniform_degree", 1), sc.get("hol_strict", True))
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
    return w, steps


def test_planner_scenarios_golden(port):
    for item in json.load(open(os.path.join(GOLD, "planner_scenarios.json"))):
        sc, res = item["scenario"], item["result"]
        w, steps = _replay(port, "dcpora_", sc)
        assert steps == res["steps"], sc["name"]
        assert w.instances() == res["instances"], sc["name"]
        ids = sorted({e[1] for e in sc["events"] if e[0] == "enqueue"})
        assert {str(i): w.placement(i) for i in ids} == res["placements"], sc["name"]
        pt, rt = w.page_table_csv(), w.routing_csv()
        assert hashlib.sha256(pt.encode()).hexdigest() == res["page_table_csv_sha256"], sc["name"]
        assert hashlib.sha256(rt.encode()).hexdigest() == res["routing_csv_sha256"], sc["name"]


def test_spec_600k_dcp_example():
    # "each hold 300K tokens of KV cache"
    item = next(x for x in json.load(open(os.path.join(GOLD, "planner_scenarios.json")))
                if x["scenario"]["name"] == "spec_dcp_600k")
    p = item["result"]["placements"]["2"]
    assert p == {"kv": [0, 1], "split": [300000, 300000], "moe": 0}
    assert item["result"]["instances"]["kv_load"] == [400000, 400000]


def test_spec_page_table_40():
    # l=40 split {A:30, B:10} -> A gets 2 pages, B 1 page
    item = next(x for x in json.load(open(os.path.join(GOLD, "planner_scenarios.json")))
                if x["scenario"]["name"] == "spec_page_table_40")
    assert item["result"]["placements"]["2"]["split"] == [30, 10]


def test_trace42_cp_histogram():
    # 2x4 cluster, 5%-long trace seed 42: CP {1:94, 2:2, 4:4}; ones = 114
    item = next(x for x in json.load(open(os.path.join(GOLD, "planner_scenarios.json")))
                if x["scenario"]["name"] == "trace42_2x4_5pct")
    ks = [len(p["kv"]) for p in item["result"]["placements"].values() if p]
    assert {k: ks.count(k) for k in set(ks)} == {1: 94, 2: 2, 4: 4}
    assert sum(ks) == 114


# ------------------------------------------------------------------ port vs reference
def test_water_fill_port_vs_ref_and_ac2(port, ref):
    # AC2: exhaustive optimality over 10,000 random instances
    rng = np.random.default_rng(2)
    for _ in range(10000):
        n = int(rng.integers(1, 5))
        K = rng.integers(0, 65, size=n).tolist()
        ell = int(rng.integers(1, 65))
        a = _wf(port, "dcpora_", K, ell)
        assert a == _wf(ref, "dcpref_", K, ell)
        assert sum(a) == ell and min(a) >= 0
        peak = max(k + s for k, s in zip(K, a))
        best = min(max(k + s for k, s in zip(K, comb))
                   for comb in itertools.product(range(ell + 1), repeat=n) if sum(comb) == ell) if n <= 3 else None
        if best is not None:
            assert peak == best


def test_water_fill_large(port, ref):
    rng = np.random.default_rng(3)
    for _ in range(2000):
        n = int(rng.integers(1, 9))
        K = rng.integers(0, 2_000_000, size=n).tolist()
        ell = int(rng.integers(1, 1_000_000))
        assert _wf(port, "dcpora_", K, ell) == _wf(ref, "dcpref_", K, ell)


def test_cp_degree_port_vs_ref(port, ref):
    rng = np.random.default_rng(4)
    bl = np.array([1000, 5000, 20000, I64MAX], np.int64)
    bd = np.array([1, 2, 4, 8], np.int32)
    for ell in rng.integers(1, 1_000_000, size=3000).tolist() + [32768, 32769, 131072, 131073, 393216, 393217]:
        for node in (1, 2, 4, 8):
            assert port.dcpora_cp_degree(ell, None, None, 0, node) == ref.dcpref_cp_degree(ell, None, None, 0, node)
            assert port.dcpora_cp_degree(ell, P(bl), P(bd), 4, node) == ref.dcpref_cp_degree(ell, P(bl), P(bd), 4, node)


def test_bucket_shape_ac11(port, ref):
    # AC11: monotonicity over 10,000 random pairs; port == ref
    rng = np.random.default_rng(5)
    def bs(L, pre, m, n):
        bm, bn = ctypes.c_int(), ctypes.c_int()
        rc = getattr(L, pre + "bucket_shape_default")(m, n, ctypes.byref(bm), ctypes.byref(bn))
        return rc, bm.value, bn.value
    for _ in range(10000):
        m, n = int(rng.integers(0, 300)), int(rng.integers(0, 600))
        a = bs(port, "dcpora_", m, n)
        b = bs(ref, "dcpref_", m, n)
        assert (a[0], a[1:] if a[0] == 0 else None) == (b[0], b[1:] if b[0] == 0 else None)
        m2, n2 = min(m + int(rng.integers(0, 20)), 256), min(n + int(rng.integers(0, 40)), 512)
        if a[0] == 0 and m <= 256 and n <= 512:
            c = bs(port, "dcpora_", m2, n2)
            assert c[1] >= a[1] and c[2] >= a[2] or (c[1], c[2]) >= (a[1], a[2])


def _random_world_script(rng):
    nodes = int(rng.integers(1, 3))
    ipn = int(rng.choice([1, 2, 4, 8]))
    kind = str(rng.choice(["dcp", "dcp", "least_batch", "least_cache", "uniform"]))
    udeg = int(rng.choice([d for d in (1, 2, 4, 8) if ipn % d == 0]))
    bucket = None
    if rng.random() < 0.5:
        b1 = int(rng.integers(16, 2000))
        bucket = [[b1, 1], [b1 * 3, 2], [b1 * 9, 4], [I64MAX, 8]]
    cap = int(rng.integers(8, 400))
    page = int(rng.choice([1, 3, 4, 12, 16, 16, 16]))  # non-powers of two take the division path
    ev = []
    nid = 0
    live = []
    for step in range(int(rng.integers(3, 12))):
        for _ in range(int(rng.integers(0, 12))):
            ell = int(rng.integers(1, cap * page * 2))
            ev.append(["enqueue", nid, ell])
            nid += 1
        ev.append(["step"])
        live = list(range(nid))
        for rid in rng.choice(live, size=min(len(live), int(rng.integers(0, 4))), replace=False).tolist():
            ev.append(["append", int(rid)])
        if rng.random() < 0.6 and live:
            ev.append(["finish?", int(rng.choice(live))])
    return dict(nodes=nodes, ipn=ipn, page=page, capacity=cap, kind=kind, bucket=bucket,
                uniform_degree=udeg, hol_strict=bool(rng.random() < 0.7), events=ev)


def _replay_safe(L, prefix, sc):
    w = World(L, prefix, sc["nodes"], sc["ipn"], sc["page"], sc["capacity"], sc["kind"], sc.get("bucket"),
              sc.get("uniform_degree", 1), sc.get("hol_strict", True))
    log = []
    for ev in sc["events"]:
        if ev[0] == "enqueue":
            w.enqueue(ev[1], ev[2])
        elif ev[0] == "step":
            log.append(w.step())
        elif ev[0] == "finish?":
            log.append(("finish", w.finish(ev[1])))
        elif ev[0] == "append":
            log.append(("append", w.append_token(ev[1])))
    return w, log


def test_planner_port_vs_ref_fuzz(port, ref):
    rng = np.random.default_rng(11)
    for trial in range(300):
        sc = _random_world_script(rng)
        wa, la = _replay_safe(port, "dcpora_", sc)
        wb, lb = _replay_safe(ref, "dcpref_", sc)
        assert la == lb, (trial, sc)
        assert wa.instances() == wb.instances(), trial
        assert wa.page_table_csv() == wb.page_table_csv(), trial
        assert wa.routing_csv() == wb.routing_csv(), trial


# ------------------------------------------------------------------ attention
def test_attention_ac1_and_port_vs_ref(port, ref):
    # AC1: 1,000 random instances, H_s in {8,16,64}, L <= 512,
    # shards in {1,2,4,8}: merged fp32 vs monolithic fp64 rel-L2 <= 1e-5.
    rng = np.random.default_rng(1)
    worst = 0.0
    for _ in range(1000):
        d = int(rng.choice([8, 16, 64]))
        L = int(rng.integers(1, 513))
        ns = int(rng.choice([1, 2, 4, 8]))
        q = rng.standard_normal(d)
        k = rng.standard_normal((L, d))
        v = rng.standard_normal((L, d))
        cuts = np.sort(rng.integers(0, L + 1, size=ns - 1))
        bounds = np.concatenate([cuts, [L]]).astype(np.int64)
        sc = 1.0 / np.sqrt(d)
        mono = np.zeros(d)
        assert ref.dcpref_reference_attention_f64(P(q), P(k), P(v), L, d, sc, P(mono)) == 0
        o32 = np.zeros(d, np.float32)
        q32, k32, v32 = q.astype(np.float32), k.astype(np.float32), v.astype(np.float32)
        assert port.dcpora_sharded_attention_merge_f32(P(q32), P(k32), P(v32), L, d, np.float32(sc),
                                                       P(bounds), ns, P(o32)) == 0
        r32 = np.zeros(d, np.float32)
        assert ref.dcpref_sharded_attention_merge_f32(P(q32), P(k32), P(v32), L, d, np.float32(sc),
                                                      P(bounds), ns, 0, P(r32)) == 0
        assert np.array_equal(o32, r32)            # port == reference, bit for bit
        o64, r64 = np.zeros(d), np.zeros(d)
        port.dcpora_sharded_attention_merge_f64(P(q), P(k), P(v), L, d, sc, P(bounds), ns, P(o64))
        ref.dcpref_sharded_attention_merge_f64(P(q), P(k), P(v), L, d, sc, P(bounds), ns, 0, P(r64))
        assert np.array_equal(o64, r64)
        worst = max(worst, np.linalg.norm(o32 - mono) / np.linalg.norm(mono))
    assert worst <= 1e-5, worst


def test_shard_attention_edge_cases(port, ref):
    d = 16
    q = np.ones(d)
    o, l = np.zeros(d), np.zeros(1)
    assert port.dcpora_shard_attention_f64(P(q), P(q), P(q), 0, d, 0.25, P(o), P(l)) == -6  # EmptyShard
    assert ref.dcpref_shard_attention_f64(P(q), P(q), P(q), 0, d, 0.25, P(o), P(l)) == -6
    # one key: partial_out = that value row, lse = scale * k.q (SPEC attn examples)
    rng = np.random.default_rng(0)
    k, v = rng.standard_normal(d), rng.standard_normal(d)
    assert port.dcpora_shard_attention_f64(P(q), P(k), P(v), 1, d, 0.25, P(o), P(l)) == 0
    assert np.allclose(o, v) and np.isclose(l[0], 0.25 * k @ q)
    # huge scores: max-shift keeps it finite (SPEC: magnitudes up to 1e3)
    kk = rng.standard_normal((64, d)) * 300
    vv = rng.standard_normal((64, d))
    assert port.dcpora_shard_attention_f64(P(q), P(kk), P(vv), 64, d, 1.0, P(o), P(l)) == 0
    assert np.all(np.isfinite(o)) and np.isfinite(l[0])


def test_paged_oracle_matches_reference_on_gathered_kv(port, ref):
    """The paged fp64 oracle (used to check K1) equals the reference's own
    shard_attention<double> on the same tokens gathered in page order."""
    from paper_2605_21100_b200 import workload
    rng = np.random.default_rng(8)
    lens = [1, 16, 17, 90, 0, 300]
    b = workload.paged_batch(lens, 8, 2, frame_order="shuffled", seed=3, spare_frames=9)
    q = rng.standard_normal((len(lens), 8, 128)).astype(np.float32)
    pool = rng.standard_normal((b.num_frames, 2, 2, 16, 128)).astype(np.float32)
    qb = (q.view(np.uint32) >> 16).astype(np.uint16)
    pb = (pool.view(np.uint32) >> 16).astype(np.uint16)
    out, lse = oracle_lib.paged_decode_f64(b, qb, pb)
    widen = lambda x: (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    for r, L in enumerate(lens):
        for h in range(8):
            j = h // 4
            if L == 0:
                assert np.isneginf(lse[r, h])
                continue
            frames = b.block_table[b.cu_pages[r]:b.cu_pages[r + 1]]
            kk = np.concatenate([widen(pb[f, 0, j]) for f in frames])[:L]
            vv = np.concatenate([widen(pb[f, 1, j]) for f in frames])[:L]
            qq = widen(qb[r, h])
            o, l = np.zeros(128), np.zeros(1)
            assert ref.dcpref_shard_attention_f64(P(np.ascontiguousarray(qq)), P(np.ascontiguousarray(kk)),
                                                  P(np.ascontiguousarray(vv)), L, 128, 1 / np.sqrt(128),
                                                  P(o), P(l)) == 0
            assert np.array_equal(o, out[r, h]) and l[0] == lse[r, h]


def test_paged_oracle_f32_pool_matches_reference(port, ref):
    """The fp32-pool paged oracle (used to check K1-f32, cfg1) equals the reference's
    shard_attention<double> on the same fp32 tokens gathered in page order, with page
    fills from append_token's fallback (partial non-final pages)."""
    from paper_2605_21100_b200 import workload
    rng = np.random.default_rng(11)
    lens = [3, 16, 40, 0, 129]
    b = workload.paged_batch(lens, 8, 8, frame_order="shuffled", seed=4, spare_frames=5)
    fill = np.zeros(int(b.cu_pages[-1]), np.uint8)
    lens2 = []
    for r, L in enumerate(lens):          # give every shard a partial page in the middle
        n = int(b.cu_pages[r + 1] - b.cu_pages[r])
        f = [16] * n
        if n:
            f[-1] = L - 16 * (n - 1)
        if n >= 2:
            f[0] = 9
        fill[b.cu_pages[r]:b.cu_pages[r + 1]] = f
        lens2.append(sum(f))
    b.shard_len[:] = lens2
    q = rng.standard_normal((len(lens), 8, 128)).astype(np.float32)
    pool = rng.standard_normal((b.num_frames, 2, 8, 16, 128)).astype(np.float32)
    out, lse = oracle_lib.paged_decode_f32in_f64(b, q, pool, page_fill=fill)
    for r, L in enumerate(lens2):
        frames = b.block_table[b.cu_pages[r]:b.cu_pages[r + 1]]
        fl = fill[b.cu_pages[r]:b.cu_pages[r + 1]]
        for h in range(8):
            if L == 0:
                assert np.isneginf(lse[r, h])
                continue
            kk = np.concatenate([pool[f, 0, h, :n] for f, n in zip(frames, fl)]).astype(np.float64)
            vv = np.concatenate([pool[f, 1, h, :n] for f, n in zip(frames, fl)]).astype(np.float64)
            o, l = np.zeros(128), np.zeros(1)
            assert ref.dcpref_shard_attention_f64(P(q[r, h].astype(np.float64)), P(np.ascontiguousarray(kk)),
                                                  P(np.ascontiguousarray(vv)), L, 128, 1 / np.sqrt(128),
                                                  P(o), P(l)) == 0
            assert np.array_equal(o, out[r, h]) and l[0] == lse[r, h]


def test_trace_generator_matches_reference(ref):
    """The bench trace source (paper_2605_21100_b200.workload.gen_trace) is the
    reference's gen_trace (workload.cpp:73-106), draw for draw."""
    from paper_2605_21100_b200 import workload
    n = 4000
    for seed, lr, rate, dur, pois in [(42, 0.05, 100.0, 1.0, 0), (7, 0.01, 37.5, 20.0, 1), (0, 0.0, 5.0, 3.0, 1)]:
        ids, sl, arr, ol = (np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(n), np.zeros(n, np.int64))
        cnt = ref.dcpref_gen_trace(seed, lr, rate, dur, pois, P(ids), P(sl), P(arr), P(ol), n)
        mine = workload.gen_trace(seed, lr, rate, dur, bool(pois))
        assert len(mine) == cnt
        assert [m[2] for m in mine] == sl[:cnt].tolist()
        assert [m[3] for m in mine] == ol[:cnt].tolist()
        assert np.allclose([m[1] for m in mine], arr[:cnt], rtol=0, atol=1e-9)


def test_mla_oracle_matches_reference_on_gathered_rows(port, ref):
    """The MLA fp64 oracle (used to check K10) equals the reference's own
    shard_attention<double> on the gathered 576-wide cache rows, with values =
    the rows' first 512 columns zero-padded to 576 (the reference needs equal
    key / value widths; the padding columns stay exactly 0)."""
    from paper_2605_21100_b200 import workload
    rng = np.random.default_rng(12)
    lens = [1, 20, 0, 77]
    heads = 128
    b = workload.paged_batch(lens, heads, 1, 576, 16, frame_order="shuffled", seed=4, spare_frames=5)
    q = rng.standard_normal((len(lens), heads, 576)).astype(np.float32)
    pool = rng.standard_normal((b.num_frames, 16, 576)).astype(np.float32)
    qb = (q.view(np.uint32) >> 16).astype(np.uint16)
    pb = (pool.view(np.uint32) >> 16).astype(np.uint16)
    sc = 1 / np.sqrt(192.0)
    out, lse = oracle_lib.mla_decode_f64(b, qb, pb, scale=sc)
    widen = lambda x: (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
    for r, L in enumerate(lens):
        if L == 0:
            assert np.all(np.isneginf(lse[r])) and np.all(out[r] == 0)
            continue
        frames = b.block_table[b.cu_pages[r]:b.cu_pages[r + 1]]
        kk = np.ascontiguousarray(np.concatenate([widen(pb[f]) for f in frames])[:L])
        vv = kk.copy()
        vv[:, 512:] = 0.0
        for h in range(0, heads, 9):
            qq = np.ascontiguousarray(widen(qb[r, h]))
            o, l = np.zeros(576), np.zeros(1)
            assert ref.dcpref_shard_attention_f64(P(qq), P(kk), P(vv), L, 576, sc, P(o), P(l)) == 0
            assert np.array_equal(o[:512], out[r, h]) and np.all(o[512:] == 0) and l[0] == lse[r, h]
