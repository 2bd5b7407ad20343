"""TEST INFRASTRUCTURE: ctypes loaders for the CPU oracle.

  port      oracle/_build/libdcp_oracle.so   our plain-C restatement (dcpora_*)
  reference oracle/_ref/libdcpsim_ref.so     the reference compiled from its own
                                             sources (dcpref_*), when built
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PORT_PATH = os.path.join(ROOT, "oracle", "_build", "libdcp_oracle.so")
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libdcpsim_ref.so")

_cache = {}


def _load(path, prefix):
    if path in _cache:
        return _cache[path]
    if not os.path.exists(path):
        return None
    L = ctypes.CDLL(path)
    vp = c_void_p
    sigs = {
        "world_create": (c_void_p, [c_int, c_int, c_int64, c_int64, c_int, vp, vp, c_int, c_int, c_int]),
        "world_destroy": (None, [c_void_p]),
        "world_enqueue": (c_int, [c_void_p, c_int64, c_int64]),
        "world_step": (c_int, [c_void_p, vp, vp, vp, vp, vp, vp, vp]),
        "world_finish": (c_int, [c_void_p, c_int64]),
        "world_append_token": (c_int, [c_void_p, c_int64, vp]),
        "world_placement": (c_int, [c_void_p, c_int64, vp, vp, vp, vp]),
        "world_instances": (c_int, [c_void_p, vp, vp, vp, vp]),
        "world_dump_page_table": (c_int, [c_void_p, c_char_p, c_int64]),
        "world_dump_routing": (c_int, [c_void_p, c_char_p, c_int64]),
        "water_fill": (c_int, [c_int, vp, c_int64, vp, vp]),
        "cp_degree": (c_int, [c_int64, vp, vp, c_int, c_int]),
        "bucket_shape_default": (c_int, [c_int, c_int, vp, vp]),
        "graph_footprint": (c_int, [c_int] * 7 + [vp, vp]),
        "uniform_int": (None, [c_uint64, c_int64, c_int64, c_int, vp]),
        "shard_attention_f64": (c_int, [vp, vp, vp, c_int64, c_int, c_double, vp, vp]),
        "shard_attention_f32": (c_int, [vp, vp, vp, c_int64, c_int, c_float, vp, vp]),
        "reference_attention_f64": (c_int, [vp, vp, vp, c_int64, c_int, c_double, vp]),
        "lse_merge_f64": (c_int, [c_int, vp, vp, c_int, vp]),
    }
    if prefix == "dcpora_":
        sigs["paged_decode_attn_f64"] = (c_int, [c_int, c_int, c_int, c_int, c_int, vp, vp, vp, vp, vp, vp,
                                                 c_double, vp, vp, c_int])
        sigs["paged_decode_attn_any_f64"] = (c_int, [c_int] * 6 + [vp] * 6 + [c_double, vp, vp, c_int])
        sigs["sharded_attention_merge_f64"] = (c_int, [vp, vp, vp, c_int64, c_int, c_double, vp, c_int, vp])
        sigs["sharded_attention_merge_f32"] = (c_int, [vp, vp, vp, c_int64, c_int, c_float, vp, c_int, vp])
        sigs["world_instance_shards"] = (c_int, [c_void_p, c_int, vp, vp, vp, vp, c_int, c_int])
        sigs["moe_layer_f64"] = (c_int, [c_int] * 5 + [vp] * 7 + [c_int])
        sigs["mla_paged_decode_f64"] = (c_int, [c_int] * 5 + [vp] * 6 + [c_double, vp, vp, c_int])
        sigs["shard_attention_kv_f64"] = (c_int, [vp, vp, vp, c_int64, c_int, c_int, c_int, c_double, vp, vp])
    else:
        sigs["sharded_attention_merge_f64"] = (c_int, [vp, vp, vp, c_int64, c_int, c_double, vp, c_int, c_int, vp])
        sigs["sharded_attention_merge_f32"] = (c_int, [vp, vp, vp, c_int64, c_int, c_float, vp, c_int, c_int, vp])
        sigs["batch_decode_attn_f32"] = (c_int, [c_int, c_int, c_int, c_int, c_float] + [vp] * 9 + [c_int])
        sigs["gen_trace"] = (c_int, [c_uint64, c_double, c_double, c_double, c_int, vp, vp, vp, vp, c_int])
        sigs["world_time_routing"] = (c_int, [c_void_p, c_int, vp])
    for name, (res, args) in sigs.items():
        f = getattr(L, prefix + name)
        f.restype = res
        f.argtypes = args
    _cache[path] = L
    return L


def port():
    L = _load(PORT_PATH, "dcpora_")
    if L is None:
        raise ImportError(f"{PORT_PATH} missing; run `make -C oracle`")
    return L


def reference():
    """The reference compiled from /root/reference sources, or None if not built."""
    return _load(REF_PATH, "dcpref_")


def P(a):
    """Pointer to a numpy array's data that keeps the array alive for the duration of the
    foreign call (P(x.cpu().numpy()) would otherwise hand C a pointer into a freed temporary)."""
    if a is None:
        return None
    p = ctypes.c_void_p(a.ctypes.data)
    p._keep = a
    return p


def paged_decode_f64(batch, q_bits: np.ndarray, pool_bits: np.ndarray, page_fill=None, scale=None,
                     threads: int = 0):
    """Oracle fp64 decode attention over a PagedBatch (numpy uint16 bf16 bits)."""
    L = port()
    R = len(batch.shard_len)
    out = np.zeros((R, batch.num_q_heads, batch.head_dim), np.float64)
    lse = np.zeros((R, batch.num_q_heads), np.float64)
    sc = scale if scale is not None else 1.0 / np.sqrt(batch.head_dim)
    th = threads or os.cpu_count() or 1
    rc = L.dcpora_paged_decode_attn_f64(
        R, batch.num_q_heads, batch.num_kv_heads, batch.head_dim, batch.page_size,
        P(np.ascontiguousarray(q_bits)), P(np.ascontiguousarray(pool_bits)),
        P(batch.block_table), P(batch.cu_pages), P(batch.shard_len),
        P(page_fill), sc, P(out), P(lse), th)
    assert rc == 0, rc
    return out, lse


def paged_decode_f32in_f64(batch, q: np.ndarray, pool: np.ndarray, page_fill=None, scale=None, threads: int = 0):
    """Oracle fp64 decode attention over a PagedBatch with fp32 q / pool (numpy float32)."""
    L = port()
    R = len(batch.shard_len)
    out = np.zeros((R, batch.num_q_heads, batch.head_dim), np.float64)
    lse = np.zeros((R, batch.num_q_heads), np.float64)
    sc = scale if scale is not None else 1.0 / np.sqrt(batch.head_dim)
    th = threads or os.cpu_count() or 1
    rc = L.dcpora_paged_decode_attn_any_f64(
        R, batch.num_q_heads, batch.num_kv_heads, batch.head_dim, batch.page_size, 4,
        P(np.ascontiguousarray(q, np.float32)), P(np.ascontiguousarray(pool, np.float32)),
        P(batch.block_table), P(batch.cu_pages), P(batch.shard_len),
        P(page_fill), sc, P(out), P(lse), th)
    assert rc == 0, rc
    return out, lse


def mla_decode_f64(batch, q_bits: np.ndarray, pool_bits: np.ndarray, page_fill=None, scale=None,
                   threads: int = 0):
    """Oracle fp64 MLA decode over a PagedBatch (pool [frames][page][576] bf16 bits)."""
    L = port()
    R = len(batch.shard_len)
    out = np.zeros((R, 128, 512), np.float64)
    lse = np.zeros((R, 128), np.float64)
    sc = scale if scale is not None else 1.0 / np.sqrt(192.0)
    th = threads or os.cpu_count() or 1
    rc = L.dcpora_mla_paged_decode_f64(
        R, 128, 576, 512, batch.page_size, P(np.ascontiguousarray(q_bits)), P(np.ascontiguousarray(pool_bits)),
        P(batch.block_table), P(batch.cu_pages), P(batch.shard_len), P(page_fill), sc, P(out), P(lse), th)
    assert rc == 0, rc
    return out, lse


class World:
    """Uniform Python view over dcpora_world_* / dcpref_world_*."""

    KINDS = {"dcp": 0, "least_batch": 1, "least_cache": 2, "uniform": 3}

    def __init__(self, L, prefix, nodes, ipn, page, capacity, kind="dcp", bucket=None,
                 uniform_degree=1, hol_strict=True):
        self.L, self.p = L, prefix
        bl = np.array([b[0] for b in bucket], np.int64) if bucket else np.zeros(1, np.int64)
        bd = np.array([b[1] for b in bucket], np.int32) if bucket else np.zeros(1, np.int32)
        self.W = nodes * ipn
        self.h = self._f("world_create")(nodes, ipn, page, capacity, self.KINDS[kind], P(bl), P(bd),
                                         len(bucket) if bucket else 0, uniform_degree, int(hol_strict))
        self.nreq = 0

    def _f(self, name):
        return getattr(self.L, self.p + name)

    def __del__(self):
        try:
            self._f("world_destroy")(self.h)
        except Exception:
            pass

    def enqueue(self, rid, seq_len):
        self.nreq += 1
        return self._f("world_enqueue")(self.h, rid, seq_len)

    def step(self):
        n = max(self.nreq, 1)
        c, d, u = (np.zeros(n, np.int64) for _ in range(3))
        nc, nd, nu = (np.zeros(1, np.int32) for _ in range(3))
        hol = np.zeros(1, np.int64)
        rc = self._f("world_step")(self.h, P(c), P(nc), P(d), P(nd), P(u), P(nu), P(hol))
        if rc:
            raise RuntimeError(f"step rc={rc}")
        return dict(committed=c[:nc[0]].tolist(), deferred=d[:nd[0]].tolist(),
                    unschedulable=u[:nu[0]].tolist(), hol_events=int(hol[0]))

    def finish(self, rid):
        return self._f("world_finish")(self.h, rid)

    def append_token(self, rid):
        inst = np.zeros(1, np.int32)
        rc = self._f("world_append_token")(self.h, rid, P(inst))
        return rc, int(inst[0])

    def placement(self, rid):
        kv = np.zeros(64, np.int32)
        sp = np.zeros(64, np.int64)
        moe = np.zeros(1, np.int32)
        k = np.zeros(1, np.int32)
        rc = self._f("world_placement")(self.h, rid, P(kv), P(sp), P(moe), P(k))
        if rc:
            return None
        return dict(kv=kv[:k[0]].tolist(), split=sp[:k[0]].tolist(), moe=int(moe[0]))

    def instances(self):
        kv, fr = np.zeros(self.W, np.int64), np.zeros(self.W, np.int64)
        b, sc = np.zeros(self.W, np.int32), np.zeros(self.W, np.int32)
        self._f("world_instances")(self.h, P(kv), P(b), P(sc), P(fr))
        return dict(kv_load=kv.tolist(), moe_batch=b.tolist(), shard_count=sc.tolist(), free=fr.tolist())

    def _dump(self, name):
        n = self._f(name)(self.h, None, 0)
        if n < 0:
            raise RuntimeError(f"{name} rc={n}")
        buf = ctypes.create_string_buffer(n + 1)
        self._f(name)(self.h, buf, n + 1)
        return buf.value.decode()

    def page_table_csv(self):
        return self._dump("world_dump_page_table")

    def routing_csv(self):
        return self._dump("world_dump_routing")

    def time_routing_ns(self, reps=5):
        """Reference only: best-of-reps ns of build_binding_config + derive_routing_tables."""
        t = np.zeros(1, np.int64)
        assert self.L.dcpref_world_time_routing(self.h, reps, P(t)) == 0
        return int(t[0])
