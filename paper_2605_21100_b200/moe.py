"""Host mirror of the MoE dispatch/combine path (K4/K5, dcp_moe_* in dcp_capi.h).

One MoeInstance per DP-EP instance: the tokens are the instance's M list
(requests MoE-bound here, BindingConfig::moe_bound routing.hpp:18-19), each
routed to its top-k experts' ranks and combined back.  `expert_stage` is the
(out of scope) expert FFN between receive and combine, done with library
GEMMs (torch -> cuBLAS): y = sum over the row's local experts, ascending id,
of w * W_down(silu(W_gate x) * W_up x).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _capi


def _s(stream, dev):
    return ctypes.c_void_p((stream or torch.cuda.current_stream(dev)).cuda_stream)


def _view(ptr, shape, dtype, device):
    """A torch tensor aliasing device memory owned by the library (no copy, no ownership)."""
    n = int(np.prod(shape))
    itemsize = torch.empty((), dtype=dtype).element_size()

    class _Holder:
        __cuda_array_interface__ = {
            "shape": (n * itemsize,), "typestr": "|u1", "data": (ptr, False), "version": 3, "strides": None}

    raw = torch.as_tensor(_Holder(), device=torch.device("cuda", device))
    return raw.view(dtype).view(*shape)


class MoeInstance:
    def __init__(self, ctx, world, self_id, hidden, topk, num_experts, m_max, timeout_ms=0):
        L = _capi.lib()
        cfg = _capi.MoeConfig(world, self_id, hidden, topk, num_experts, m_max, timeout_ms)
        h = ctypes.c_void_p()
        _capi.check(L.dcp_moe_create(ctx.handle, ctypes.byref(cfg), ctypes.byref(h)))
        self.h, self.ctx = h, ctx
        self.world, self.id, self.H, self.k, self.E, self.m_max = world, self_id, hidden, topk, num_experts, m_max
        self.meta_w = L.dcp_moe_meta_width(h)
        dev = torch.device("cuda", ctx.device)
        self.x_rows = torch.empty(world * m_max, hidden, dtype=torch.bfloat16, device=dev)
        self.meta_rows = torch.zeros(world * m_max, self.meta_w, dtype=torch.int32, device=dev)
        self.y_rows = torch.zeros(world * m_max, hidden, dtype=torch.bfloat16, device=dev)
        self.out = torch.zeros(m_max, hidden, dtype=torch.float32, device=dev)
        self.m_count = torch.zeros(1, dtype=torch.int32, device=dev)

    def status(self):
        """Raise ExchangeTimeout if a flag wait of this instance timed out (clears it)."""
        info = (ctypes.c_uint32 * 4)()
        _capi.check(_capi.lib().dcp_moe_status(self.h, info))

    def ipc_handle(self):
        b = ctypes.create_string_buffer(64)
        _capi.check(_capi.lib().dcp_moe_ipc_handle(self.h, b))
        return b.raw

    def open_peer(self, peer, handle):
        _capi.check(_capi.lib().dcp_moe_open_peer_ipc(self.h, peer, ctypes.create_string_buffer(handle, 64)))

    def set_peer_local(self, peer, other):
        _capi.check(_capi.lib().dcp_moe_set_peer_local(self.h, peer, other.h))

    def commit(self):
        _capi.check(_capi.lib().dcp_moe_commit(self.h))

    def dispatch(self, x, topk_idx, topk_w, m_count_ptr=None, stream=None, fused=True, with_receive=False):
        """x bf16 [M, H], topk_idx int32 [M, k], topk_w fp32 [M, k] (device).  Starts the step:
        fused (default) = one launch (dcp_moe_step_dispatch), else begin_step + dispatch.
        with_receive: the region-mode receive in the same launch (dcp_moe_step_dispatch_recv; one
        instance per process / GPU only)."""
        L = _capi.lib()
        s = _s(stream, self.ctx.device)
        if m_count_ptr is None:
            self.m_count.fill_(x.shape[0])
            m_count_ptr = self.m_count.data_ptr()
        self._keep = (x, topk_idx, topk_w)
        args = (self.h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(topk_idx.data_ptr()),
                ctypes.c_void_p(topk_w.data_ptr()), ctypes.c_void_p(m_count_ptr), s)
        if with_receive:
            _capi.check(L.dcp_moe_step_dispatch_recv(*args))
        elif fused:
            _capi.check(L.dcp_moe_step_dispatch(*args))
        else:
            _capi.check(L.dcp_moe_begin_step(self.h, s))
            _capi.check(L.dcp_moe_dispatch(*args))

    def receive(self, stream=None):
        counts = np.zeros(self.world, np.int32)
        R = _capi.lib().dcp_moe_receive(self.h, ctypes.c_void_p(self.x_rows.data_ptr()),
                                        ctypes.c_void_p(self.meta_rows.data_ptr()),
                                        counts.ctypes.data_as(ctypes.c_void_p), _s(stream, self.ctx.device))
        if R < 0:
            _capi.check(R)
        return int(R), counts

    def receive_async(self, stream=None):
        """K5a without the host count read-back (counts stay on the device)."""
        _capi.check(_capi.lib().dcp_moe_receive_async(self.h, ctypes.c_void_p(self.x_rows.data_ptr()),
                                                      ctypes.c_void_p(self.meta_rows.data_ptr()),
                                                      _s(stream, self.ctx.device)))

    def receive_regions(self, stream=None):
        """K5a region mode: wait for every source; rows stay in the pool regions."""
        _capi.check(_capi.lib().dcp_moe_receive_regions(self.h, _s(stream, self.ctx.device)))

    def regions(self, parity=None):
        """(x_region bf16 [W, m_max, H], meta_region int32 [W, m_max, meta]) of a parity, as
        torch views of the pool (the current step's parity by default)."""
        L = _capi.lib()
        if parity is None:
            parity = L.dcp_moe_parity(self.h)
        xp, mp = ctypes.c_void_p(), ctypes.c_void_p()
        _capi.check(L.dcp_moe_regions(self.h, parity, ctypes.byref(xp), ctypes.byref(mp)))
        return (_view(xp.value, (self.world, self.m_max, self.H), torch.bfloat16, self.ctx.device),
                _view(mp.value, (self.world, self.m_max, self.meta_w), torch.int32, self.ctx.device))

    def recv_counts(self):
        """Per-source received row counts of the last receive (device -> host)."""
        p = _capi.lib().dcp_moe_recv_counts_dev(self.h)
        return _capi.device_to_numpy(p, self.world, np.int32)

    def combine_put_regions(self, y_region, stream=None):
        """K5b with y in region layout bf16 [W, m_max, H] (the expert stage's output in place)."""
        _capi.check(_capi.lib().dcp_moe_combine_put_regions(self.h, ctypes.c_void_p(y_region.data_ptr()),
                                                            _s(stream, self.ctx.device)))

    def expert_stage(self, R, w_gate, w_up, w_down):
        """Library-GEMM expert FFN over the R received rows (local experts
        w_*[e - first_local_expert]): the (row, expert, gate weight) pairs of the meta rows are
        grouped by expert on the device, then one gate / up / down GEMM triple per local expert
        in ascending expert order, y = sum_e w_e * W_down(silu(W_gate x) * W_up x)."""
        e0 = self.id * (self.E // self.world)
        y = torch.zeros(R, self.H, dtype=torch.float32, device=self.x_rows.device)
        if R > 0:
            meta = self.meta_rows[:R]
            k = (meta.shape[1] - 2) // 2
            n = meta[:, 1:2]
            ex = meta[:, 2:2 + 2 * k:2]
            wt = meta[:, 3:3 + 2 * k:2].contiguous().view(torch.float32)
            valid = torch.arange(k, device=meta.device)[None, :] < n
            rows = torch.arange(R, device=meta.device)[:, None].expand(R, k)[valid]
            ex, wt = ex[valid], wt[valid]
            order = torch.argsort(ex * R + rows)  # by expert, then row
            rows, ex, wt = rows[order], ex[order], wt[order]
            uniq, cnt = torch.unique_consecutive(ex, return_counts=True)
            x = self.x_rows[:R]
            start = 0
            for e, c in zip(uniq.tolist(), cnt.tolist()):
                rr, ww = rows[start:start + c], wt[start:start + c]
                start += c
                xe = x[rr]
                g = xe @ w_gate[e - e0].T
                u = xe @ w_up[e - e0].T
                a = (torch.nn.functional.silu(g.float()) * u.float()).to(torch.bfloat16)
                o = (a @ w_down[e - e0].T).float()
                y.index_add_(0, rr, o * ww[:, None])
        self.y_rows[:R] = y.to(torch.bfloat16)

    def expert_identity(self, y_region, stream=None):
        """Gate-weighted identity expert over this step's regions (dcp_moe_expert_identity)."""
        _capi.check(_capi.lib().dcp_moe_expert_identity(self.h, ctypes.c_void_p(y_region.data_ptr()),
                                                        _s(stream, self.ctx.device)))

    def combine_put(self, stream=None):
        _capi.check(_capi.lib().dcp_moe_combine_put(self.h, ctypes.c_void_p(self.y_rows.data_ptr()),
                                                    _s(stream, self.ctx.device)))

    def combine_reduce(self, stream=None):
        _capi.check(_capi.lib().dcp_moe_combine_reduce(self.h, ctypes.c_void_p(self.out.data_ptr()),
                                                       _s(stream, self.ctx.device)))

    def combine_fused(self, y_region, stream=None):
        """K5b + K5c in one launch (dcp_moe_combine_fused): one instance per process / GPU only."""
        _capi.check(_capi.lib().dcp_moe_combine_fused(self.h, ctypes.c_void_p(y_region.data_ptr()),
                                                      ctypes.c_void_p(self.out.data_ptr()),
                                                      _s(stream, self.ctx.device)))

    def close(self):
        if getattr(self, "h", None):
            _capi.lib().dcp_moe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
