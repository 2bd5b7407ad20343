"""Multi-process plumbing for the DCP step: one rank per GPU (torch.distributed).

Used only for setup and timing reductions — the data path between GPUs is the
kernels' own NVLink stores into CUDA-IPC-mapped peer pools (dcp_xchg_*,
dcp_moe_*), not a collective.

* exchange_handles: all-gather each rank's 64-byte CUDA-IPC pool handle so
  every rank can map every peer's receive pools.
* check_replicas: the planner runs as an identical replica on every rank
  ("replicas only"); a digest all-gather proves the replicas
  produced the same routing tables before any rank stores into a peer.
* max_over_ranks: step latency is the slowest rank's device time.
"""
from __future__ import annotations

import hashlib

import torch
import torch.distributed as dist


def exchange_handles(handle: bytes) -> list[bytes]:
    if len(handle) != 64:
        raise ValueError("CUDA IPC handles are 64 bytes")
    out: list = [None] * dist.get_world_size()
    dist.all_gather_object(out, handle)
    return out


def digest(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def check_replicas(routing_csv: str) -> None:
    mine = digest(routing_csv)
    out: list = [None] * dist.get_world_size()
    dist.all_gather_object(out, mine)
    if any(d != mine for d in out):
        raise RuntimeError(f"planner replicas diverged on rank {dist.get_rank()}: {out}")


def max_over_ranks(x: float, device=None) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def connect_peers(inst, handles: list[bytes]) -> None:
    """Map every peer's pools into this rank's exchange object (self maps itself)."""
    me = dist.get_rank()
    for peer, h in enumerate(handles):
        if peer == me:
            inst.set_peer_local(me, inst)
        else:
            inst.open_peer(peer, h)
    inst.commit()


# ---------------------------------------------------------------------------------------------
class RankStep:
    """One rank of a multi-process DCP decode step: one DCP instance (one GPU in production).

    Every rank runs the identical planner replica (K6 admission + K7 routing; SURVEY §8(e)
    "replicas only"), checks the replicas agree, then maps every peer's exchange pools through
    CUDA IPC.  A step is this instance's
        begin_step -> K2 Q-route puts -> K1 (+ Res-route puts) -> K3 merge
    and optionally the MoE layer on its M list
        begin_step -> K4 dispatch -> K5a receive (region) -> experts -> K5b combine_put -> K5c reduce
    with no host synchronisation between ranks: every cross-rank dependency is a device flag.

    pool_fn(rank, capacity, hkv) -> KV pool tensor of this rank (bf16 [cap, 2, hkv, 16, 128]).
    moe: None or dict(hidden, experts, topk, m_max).
    """

    def __init__(self, ctx, world, rank, lens, hq, hkv, capacity, pool_fn, bucket=None, moe=None,
                 timeout_ms=30000, n_max=512, m_max=256, max_requests=None):
        from .dcp_step import DcpInstance
        from .moe import MoeInstance
        from .planner import DevicePlanner
        self.ctx, self.world, self.rank, self.hq, self.hkv = ctx, world, rank, hq, hkv
        self.ids = list(range(len(lens)))
        self.lens = list(lens)
        mr = max_requests or max(64, 2 * len(lens))
        self.planner = DevicePlanner(ctx, 1, world, 16, capacity, "dcp", bucket, max_requests=mr, reserve_pages=8)
        self.planner.enqueue_many(self.ids, self.lens)
        res = self.planner.step()
        if len(res["committed"]) != len(self.ids):
            raise RuntimeError(f"rank {rank}: only {len(res['committed'])} of {len(self.ids)} admitted")
        self.planner.build_routing()
        check_replicas(self.planner.routing_csv())
        self.view = self.planner.instance_view(rank)
        import numpy as np
        from ._capi import device_to_numpy
        self.m_ids = device_to_numpy(self.view.m_ids, self.view.m_rows, np.int64).tolist()
        self.n_ids = device_to_numpy(self.view.n_ids, self.view.n_rows, np.int64).tolist()
        self.inst = DcpInstance(ctx, world, rank, hq, hkv, capacity, kv_pool=pool_fn(rank, capacity, hkv),
                                n_max=n_max, m_max=m_max, timeout_ms=timeout_ms)
        connect_peers(self.inst, exchange_handles(self.inst.ipc_handle()))
        self.moe = None
        if moe:
            self.moe = MoeInstance(ctx, world, rank, moe["hidden"], moe["topk"], moe["experts"], moe["m_max"],
                                   timeout_ms=timeout_ms)
            connect_peers(self.moe, exchange_handles(self.moe.ipc_handle()))
            import torch
            self.y_region = torch.zeros(world, moe["m_max"], moe["hidden"], dtype=torch.bfloat16,
                                        device=torch.device("cuda", ctx.device))
        # K7's device M count of this instance feeds K4 (no host round trip)
        self.m_count_ptr = self.view.m_count_all + 4 * rank

    def attention(self, q_rows, stream=None):
        """q_rows bf16 [M, hq, 128] in this rank's M-row order."""
        if len(self.m_ids):
            self.inst.write_queries(q_rows, stream)
        self.inst.run(self.view, stream)

    def moe_layer(self, x, topk_idx, topk_w, expert_fn=None, stream=None, fused_combine=False, fused_receive=False):
        """x bf16 [M, H] in M-row order; expert_fn(x_region, meta_region, counts, y_region) fills
        self.y_region (None: the gate-weighted identity expert, dcp_moe_expert_identity, issued
        on the stream, no host sync).  fused_combine: K5b + K5c in one launch
        (dcp_moe_combine_fused); fused_receive: K4 + K5a in one launch (dcp_moe_step_dispatch_recv);
        both valid here, one instance per process."""
        m = self.moe
        m.dispatch(x, topk_idx, topk_w, m_count_ptr=self.m_count_ptr, stream=stream, with_receive=fused_receive)
        if not fused_receive:
            m.receive_regions(stream)
        xr, mr = m.regions()
        if expert_fn is None:
            m.expert_identity(self.y_region, stream)
        else:
            expert_fn(xr, mr, m.recv_counts(), self.y_region)
        if fused_combine:
            m.combine_fused(self.y_region, stream)
        else:
            m.combine_put_regions(self.y_region, stream)
            m.combine_reduce(stream)

    def results(self):
        return self.inst.results(len(self.m_ids))

    def status(self):
        self.inst.status()
        if self.moe is not None:
            self.moe.status()

    def close(self):
        self.inst.close()
        if self.moe is not None:
            self.moe.close()
        self.planner.close()
