"""N>1 host-side logic on CPU: world_size-2 gloo process group.

Covers what the multi-GPU DCP step does before and around the kernels:
IPC-handle all-gather, peer wiring order, planner-replica digest check, and
the max-over-ranks latency reduction (paper_2605_21100_b200/multi.py).
"""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _FakeInst:
    def __init__(self):
        self.calls = []

    def set_peer_local(self, peer, other):
        self.calls.append(("local", peer))

    def open_peer(self, peer, handle):
        self.calls.append(("ipc", peer, handle))

    def commit(self):
        self.calls.append(("commit",))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2605_21100_b200 import multi
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        handles = multi.exchange_handles(bytes([rank]) * 64)
        inst = _FakeInst()
        multi.connect_peers(inst, handles)
        multi.check_replicas("instance,table,row,request_id,columns\n0,q_route,0,7,10\n")
        diverged = False
        try:
            multi.check_replicas(f"rank{rank}")
        except RuntimeError:
            diverged = True
        m = multi.max_over_ranks(0.5 + rank)
        q.put((rank, [h[0] for h in handles], inst.calls, diverged, m))
    finally:
        dist.destroy_process_group()


def test_two_rank_setup_logic():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, hs, calls, diverged, m in res:
        assert hs == [0, 1]                                   # every rank sees every handle, rank order
        assert calls[rank] == ("local", rank) and calls[-1] == ("commit",)
        other = 1 - rank
        assert calls[other] == ("ipc", other, bytes([other]) * 64)
        assert diverged                                       # divergent replicas are caught
        assert m == 1.5                                       # max over ranks
