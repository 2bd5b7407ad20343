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
