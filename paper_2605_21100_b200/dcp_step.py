"""One DCP decode-attention step across W instances (Fig. 7).

    planner (K6) -> routing / block tables (K7) -> per instance:
        Q-route puts (K2) -> split-KV attention with fused Res-route puts (K1)
        -> LSE merge at the MoE binding (K3)

An instance is one KV/MoE binding target (one GPU in production).  This
driver can host all W instances in one process — on distinct GPUs, or all on
one GPU for testing, where the "peer" stores are local stores through the
identical code path.  Multi-process deployments (one rank per GPU) use
DcpInstance with CUDA-IPC peer handles instead (see bench_dcp.py).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _capi
from .attention import DcpContext


class DcpInstance:
    """Exchange pools + KV pool + attention workspace of one instance.

    dtype "bf16": K1 (bf16 KV / Q, mma.sync GQA tiles); "f32": K1-f32 (fp32 KV / Q, the
    reference's production precision, cfg1).  Partials and merged outputs are fp32 either way.
    """

    def __init__(self, ctx: DcpContext, world: int, self_id: int, hq: int, hkv: int, capacity_pages: int,
                 head_dim: int = 128, page_size: int = 16, n_max: int = 512, m_max: int = 256,
                 kv_pool: torch.Tensor | None = None, dtype: str = "bf16", timeout_ms: int = 0):
        L = _capi.lib()
        if dtype not in ("bf16", "f32"):
            raise ValueError(f"dtype {dtype!r}")
        self.ctx, self.world, self.id = ctx, world, self_id
        self.hq, self.hkv, self.d, self.page = hq, hkv, head_dim, page_size
        self.n_max, self.m_max, self.dtype = n_max, m_max, dtype
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.tdtype = tdt
        cfg = _capi.XchgConfig(world, self_id, hq, head_dim, n_max, m_max, head_dim, head_dim,
                               2 if dtype == "bf16" else 4, timeout_ms)
        h = ctypes.c_void_p()
        _capi.check(L.dcp_xchg_create(ctx.handle, ctypes.byref(cfg), ctypes.byref(h)))
        self.x = h
        dev = torch.device("cuda", ctx.device)
        self.kv_pool = kv_pool if kv_pool is not None else torch.zeros(
            max(capacity_pages, 1), 2, hkv, page_size, head_dim, dtype=tdt, device=dev)
        if self.kv_pool.dtype != tdt:
            raise TypeError(f"kv_pool dtype {self.kv_pool.dtype} for a {dtype} instance")
        nbytes = L.dcp_attn_workspace_bytes(ctx.handle, n_max, hq, head_dim)
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        ql, qr, out, lse = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _capi.check(L.dcp_xchg_buffers(h, ctypes.byref(ql), ctypes.byref(qr), ctypes.byref(out),
                                       ctypes.byref(lse)))
        self.q_local_ptr, self.out_ptr, self.lse_ptr = ql.value, out.value, lse.value
        self.args = _capi.AttnArgs()
        a = self.args
        a.num_q_heads, a.num_kv_heads, a.head_dim, a.page_size = hq, hkv, head_dim, page_size
        a.num_frames = self.kv_pool.shape[0]
        a.kv_pool = self.kv_pool.data_ptr()
        a.scale = 1.0 / math.sqrt(head_dim)
        a.workspace, a.workspace_bytes = self.workspace.data_ptr(), self.workspace.numel()

    def status(self):
        """Raise ExchangeTimeout if a flag wait of this instance timed out (clears it)."""
        info = (ctypes.c_uint32 * 4)()
        _capi.check(_capi.lib().dcp_xchg_status(self.x, info))

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _capi.check(_capi.lib().dcp_xchg_ipc_handle(self.x, buf))
        return buf.raw

    def open_peer(self, peer: int, handle: bytes):
        _capi.check(_capi.lib().dcp_xchg_open_peer_ipc(self.x, peer, ctypes.create_string_buffer(handle, 64)))

    def set_peer_local(self, peer: int, other: "DcpInstance"):
        _capi.check(_capi.lib().dcp_xchg_set_peer_local(self.x, peer, other.x))

    def commit(self):
        _capi.check(_capi.lib().dcp_xchg_commit(self.x))

    # ---- per step ------------------------------------------------------------
    def write_queries(self, q_rows: torch.Tensor, stream=None):
        """q_rows: [M, hq, d] (bf16, or fp32 for an f32 instance) in this instance's M-row order."""
        s = (stream or torch.cuda.current_stream(self.ctx.device)).cuda_stream
        if q_rows.dtype != self.tdtype:
            raise TypeError(f"queries are {q_rows.dtype}, instance is {self.dtype}")
        q_rows = q_rows.contiguous()
        self._q_keep = q_rows
        _capi.check(_capi.lib().dcp_xchg_write_queries(self.x, ctypes.c_void_p(q_rows.data_ptr()),
                                                       q_rows.shape[0], ctypes.c_void_p(s)))

    def run(self, view: _capi.InstanceView, stream=None, phase: str = "all"):
        """phase "all" / "q" / "attn" / "merge": the four phased calls (or a subset); "fused": the
        whole step in one launch (dcp_decode_step_fused; bf16, one instance per GPU / process)."""
        L = _capi.lib()
        s = ctypes.c_void_p((stream or torch.cuda.current_stream(self.ctx.device)).cuda_stream)
        if phase == "fused":
            _capi.check(L.dcp_decode_step_fused(self.ctx.handle, self.x, ctypes.byref(view), ctypes.byref(self.args), s))
            return
        if phase in ("all", "q"):
            _capi.check(L.dcp_xchg_begin_step(self.x, s))
            _capi.check(L.dcp_route_q(self.x, ctypes.byref(view), s))
        if phase in ("all", "attn"):
            fn = L.dcp_decode_attn_routed if self.dtype == "bf16" else L.dcp_decode_attn_routed_f32
            _capi.check(fn(self.ctx.handle, self.x, ctypes.byref(view), ctypes.byref(self.args), s))
        if phase in ("all", "merge"):
            _capi.check(L.dcp_merge_partials(self.x, ctypes.byref(view), s))

    def results(self, m_rows: int):
        out = _capi.device_to_numpy(self.out_ptr, m_rows * self.hq * self.d, np.float32)
        lse = _capi.device_to_numpy(self.lse_ptr, m_rows * self.hq, np.float32)
        return out.reshape(m_rows, self.hq, self.d), lse.reshape(m_rows, self.hq)

    def close(self):
        if getattr(self, "x", None):
            _capi.lib().dcp_xchg_destroy(self.x)
            self.x = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MlaDcpInstance(DcpInstance):
    """One instance of a routed DCP step with MLA attention (cfg5, K10 on tcgen05 CTA pairs).

    The exchange pools are MLA-shaped: Q rows of 128 heads x 576 (absorbed q_nope | q_pe,
    bf16), partial O rows of 128 x 512 fp32 + LSE.  KV pool: bf16 [frames, page, 576]
    (c_kv | k_pe).  Steps are dcp_route_q -> dcp_mla_decode_attn_routed -> dcp_merge_partials.
    """

    HEADS, DK, DV = 128, 576, 512

    def __init__(self, ctx: DcpContext, world: int, self_id: int, capacity_pages: int, page_size: int = 16,
                 n_max: int = 256, m_max: int = 128, kv_pool: torch.Tensor | None = None, timeout_ms: int = 0,
                 scale: float | None = None):
        L = _capi.lib()
        self.ctx, self.world, self.id = ctx, world, self_id
        self.hq, self.hkv, self.d, self.page = self.HEADS, 1, self.DV, page_size
        self.n_max, self.m_max, self.dtype, self.tdtype = n_max, m_max, "bf16", torch.bfloat16
        cfg = _capi.XchgConfig(world, self_id, self.HEADS, self.DV, n_max, m_max, self.DK, self.DV, 2, timeout_ms)
        h = ctypes.c_void_p()
        _capi.check(L.dcp_xchg_create(ctx.handle, ctypes.byref(cfg), ctypes.byref(h)))
        self.x = h
        dev = torch.device("cuda", ctx.device)
        self.kv_pool = kv_pool if kv_pool is not None else torch.zeros(
            max(capacity_pages, 1), page_size, self.DK, dtype=torch.bfloat16, device=dev)
        nbytes = L.dcp_mla_workspace_bytes(ctx.handle, n_max)
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        ql, qr, out, lse = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _capi.check(L.dcp_xchg_buffers(h, ctypes.byref(ql), ctypes.byref(qr), ctypes.byref(out),
                                       ctypes.byref(lse)))
        self.q_local_ptr, self.out_ptr, self.lse_ptr = ql.value, out.value, lse.value
        a = self.margs = _capi.MlaArgs()
        a.num_q_heads, a.kv_lora_rank, a.rope_dim, a.page_size = self.HEADS, self.DV, self.DK - self.DV, page_size
        a.num_frames = self.kv_pool.shape[0]
        a.kv_pool = self.kv_pool.data_ptr()
        a.scale = scale if scale is not None else 1.0 / math.sqrt(192.0)
        a.workspace, a.workspace_bytes = self.workspace.data_ptr(), self.workspace.numel()

    def run(self, view: _capi.InstanceView, stream=None, phase: str = "all"):
        L = _capi.lib()
        s = ctypes.c_void_p((stream or torch.cuda.current_stream(self.ctx.device)).cuda_stream)
        if phase in ("all", "q"):
            _capi.check(L.dcp_xchg_begin_step(self.x, s))
            _capi.check(L.dcp_route_q(self.x, ctypes.byref(view), s))
        if phase in ("all", "attn"):
            _capi.check(L.dcp_mla_decode_attn_routed(self.ctx.handle, self.x, ctypes.byref(view),
                                                     ctypes.byref(self.margs), s))
        if phase in ("all", "merge"):
            _capi.check(L.dcp_merge_partials(self.x, ctypes.byref(view), s))


class StepGraph:
    """AOT step graphs of one instance (dcp_step_graph_*): one captured CUDA
    graph per M-bucket of the default ShapeSpace, replayed per decode step."""

    def __init__(self, inst: DcpInstance, view):
        L = _capi.lib()
        self.view = view  # device pointers captured by the graphs must stay alive
        h = ctypes.c_void_p()
        _capi.check(L.dcp_step_graph_create(inst.ctx.handle, inst.x, ctypes.byref(view), ctypes.byref(inst.args),
                                            ctypes.byref(h)))
        self.h, self.inst = h, inst
        b = ctypes.c_int32()
        self.graphs = L.dcp_step_graph_count(h, ctypes.byref(b))
        self.buckets = b.value

    def launch(self, m_rows: int, n_rows: int, stream=None):
        s = (stream or torch.cuda.current_stream(self.inst.ctx.device)).cuda_stream
        _capi.check(_capi.lib().dcp_step_graph_launch(self.h, m_rows, n_rows, ctypes.c_void_p(s)))

    def close(self):
        if getattr(self, "h", None):
            _capi.lib().dcp_step_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LayerGraph:
    """Whole-layer AOT decode graphs of one instance (dcp_layer_graph_*; Alg. 2).

    Captures [K7] -> begin -> K2 -> K1 -> K3 -> MoE begin -> K4 -> K5a -> expert -> K5b -> K5c
    once per (M-bucket, MoE parity) and replays it per decode step.  moe: a MoeInstance or None;
    moe_x bf16 [m_max, H], topk_idx int32 / topk_w fp32 [m_max, k] are the device buffers the
    graph reads every replay (write the step's values into them before launch).  expert: a
    ctypes EXPERT_FN (called at capture time to enqueue the expert stage) or None for the
    built-in gate-weighted identity expert.  planner: include K7 in the graph.
    """

    def __init__(self, inst: DcpInstance, view, moe=None, moe_x=None, topk_idx=None, topk_w=None,
                 planner=None, expert=None, fused=False):
        L = _capi.lib()
        self.inst, self.view, self.moe = inst, view, moe
        dev = torch.device("cuda", inst.ctx.device)
        d = _capi.LayerGraphDesc()
        d.planner = planner.h if planner is not None else None
        d.xchg = inst.x
        d.view = ctypes.pointer(view)
        d.attn = ctypes.pointer(inst.args)
        if moe is not None:
            self.y_region = torch.zeros(moe.world, moe.m_max, moe.H, dtype=torch.bfloat16, device=dev)
            d.moe, d.moe_x = moe.h, moe_x.data_ptr()
            d.topk_idx, d.topk_w = topk_idx.data_ptr(), topk_w.data_ptr()
            d.y_region, d.moe_out = self.y_region.data_ptr(), moe.out.data_ptr()
            self._keep = (moe_x, topk_idx, topk_w)
        if expert is not None:
            d.expert = expert
        self._expert = expert
        d.fused_step = int(fused)
        self.desc = d
        h = ctypes.c_void_p()
        _capi.check(L.dcp_layer_graph_create(inst.ctx.handle, ctypes.byref(d), ctypes.byref(h)))
        self.h = h

    def info(self):
        b, c = ctypes.c_int32(), ctypes.c_int32()
        n = _capi.lib().dcp_layer_graph_info(self.h, ctypes.byref(b), ctypes.byref(c))
        return dict(graphs=n, buckets=b.value, captures=c.value)

    def launch(self, m_rows: int, stream=None):
        s = (stream or torch.cuda.current_stream(self.inst.ctx.device)).cuda_stream
        _capi.check(_capi.lib().dcp_layer_graph_launch(self.h, m_rows, ctypes.c_void_p(s)))

    def close(self):
        if getattr(self, "h", None):
            _capi.lib().dcp_layer_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_local_step(planner, instances, q_of_request: dict, stream=None):
    """Run one routed step with all instances in this process.

    q_of_request: request id -> bf16 [hq, d] CUDA tensor (on instance m_r's device).
    Returns {request id: (O [hq, d] float32, LSE [hq])} read at each MoE binding.
    """
    planner.build_routing()
    W = len(instances)
    views = [planner.instance_view(s) for s in range(W)]
    m_ids = []
    for s, inst in enumerate(instances):
        v = views[s]
        ids = _capi.device_to_numpy(v.m_ids, v.m_rows, np.int64).tolist()
        m_ids.append(ids)
        if ids:
            q = torch.stack([q_of_request[i] for i in ids]).contiguous()
            inst.write_queries(q, stream)
    # phase order keeps a single GPU free of cross-kernel spin dependencies
    for s, inst in enumerate(instances):
        inst.run(views[s], stream, "q")
    for s, inst in enumerate(instances):
        inst.run(views[s], stream, "attn")
    for s, inst in enumerate(instances):
        inst.run(views[s], stream, "merge")
    torch.cuda.synchronize()
    for inst in instances:
        inst.status()
    res = {}
    for s, inst in enumerate(instances):
        o, l = inst.results(len(m_ids[s]))
        for j, rid in enumerate(m_ids[s]):
            res[rid] = (o[j], l[j])
    return res, views
