"""Host mirror of the reference planner interface over the device planner (K6/K7).

The reference's control plane is `Scheduler::step` over a `ClusterState`
(scheduler.hpp:66-89, page_table.hpp:77-100) plus `build_binding_config` /
`derive_routing_tables` (routing.hpp:50-58).  Here the cluster state lives in
HBM and every operation is a device kernel behind dcp_planner_* (dcp_capi.h);
this class only marshals ids/lengths and reads results back.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _capi

POLICIES = {"dcp": 0, "least_batch": 1, "least_cache": 2, "uniform": 3}


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


class DevicePlanner:
    def __init__(self, ctx, nodes, instances_per_node, page_size, capacity_pages, policy="dcp",
                 bucket=None, uniform_degree=1, hol_strict=True, max_requests=4096, reserve_pages=4,
                 stream=None):
        L = _capi.lib()
        self.ctx = ctx
        self.W = nodes * instances_per_node
        self._bl = np.array([b[0] for b in bucket] if bucket else [0], np.int64)
        self._bd = np.array([b[1] for b in bucket] if bucket else [0], np.int32)
        cfg = _capi.PlannerConfig(nodes, instances_per_node, page_size, capacity_pages, POLICIES[policy],
                                  len(bucket) if bucket else 0, self._bl.ctypes.data, self._bd.ctypes.data,
                                  uniform_degree, int(hol_strict), max_requests, reserve_pages)
        h = ctypes.c_void_p()
        _capi.check(L.dcp_planner_create(ctx.handle, ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h
        self.stream = stream
        self.queued = 0

    def close(self):
        if getattr(self, "h", None):
            _capi.lib().dcp_planner_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _s(self):
        return ctypes.c_void_p(self.stream.cuda_stream) if self.stream is not None else None

    def enqueue(self, rid, seq_len):
        return self.enqueue_many([rid], [seq_len])

    def enqueue_many(self, ids, lens):
        ids = np.ascontiguousarray(ids, np.int64)
        lens = np.ascontiguousarray(lens, np.int64)
        _capi.check(_capi.lib().dcp_planner_enqueue(self.h, _p(ids), _p(lens), len(ids)))
        self.queued += len(ids)
        return 0

    def step_async(self):
        _capi.check(_capi.lib().dcp_planner_step(self.h, self._s()))

    def step_result(self):
        n = max(self.queued, 1)
        c, d, u = (np.zeros(n, np.int64) for _ in range(3))
        nc, nd, nu = (np.zeros(1, np.int32) for _ in range(3))
        hol = np.zeros(1, np.int64)
        _capi.check(_capi.lib().dcp_planner_step_result(self.h, _p(c), _p(nc), _p(d), _p(nd), _p(u), _p(nu),
                                                        _p(hol)))
        self.queued -= int(nc[0]) + int(nu[0])
        return dict(committed=c[:nc[0]].tolist(), deferred=d[:nd[0]].tolist(),
                    unschedulable=u[:nu[0]].tolist(), hol_events=int(hol[0]))

    def step(self):
        self.step_async()
        return self.step_result()

    def finish(self, rid):
        a = np.array([rid], np.int64)
        rc = _capi.lib().dcp_planner_finish(self.h, _p(a), 1, self._s())
        return rc

    def append_token(self, rid):
        a = np.array([rid], np.int64)
        out = np.zeros(1, np.int32)
        rc = _capi.lib().dcp_planner_append_token(self.h, _p(a), 1, _p(out))
        return rc, int(out[0])

    def append_many(self, ids):
        a = np.ascontiguousarray(ids, np.int64)
        out = np.zeros(len(a), np.int32)
        _capi.check(_capi.lib().dcp_planner_append_token(self.h, _p(a), len(a), _p(out)))
        return out

    def placement(self, rid):
        kv = np.zeros(64, np.int32)
        sp = np.zeros(64, np.int64)
        moe = np.zeros(1, np.int32)
        k = np.zeros(1, np.int32)
        rc = _capi.lib().dcp_planner_placement(self.h, rid, _p(kv), _p(sp), _p(moe), _p(k))
        if rc:
            return None
        return dict(kv=kv[:k[0]].tolist(), split=sp[:k[0]].tolist(), moe=int(moe[0]))

    def instances(self):
        kv, fr = np.zeros(self.W, np.int64), np.zeros(self.W, np.int64)
        b, sc = np.zeros(self.W, np.int32), np.zeros(self.W, np.int32)
        _capi.lib().dcp_planner_instances(self.h, _p(kv), _p(b), _p(sc), _p(fr))
        return dict(kv_load=kv.tolist(), moe_batch=b.tolist(), shard_count=sc.tolist(), free=fr.tolist())

    def _dump(self, fn):
        n = fn(self.h, None, 0)
        if n < 0:
            _capi.check(int(n))
        buf = ctypes.create_string_buffer(int(n) + 1)
        fn(self.h, buf, n + 1)
        return buf.value.decode()

    def page_table_csv(self):
        return self._dump(_capi.lib().dcp_planner_dump_page_table)

    def build_routing(self):
        _capi.check(_capi.lib().dcp_planner_build_routing(self.h, self._s()))

    def routing_csv(self):
        return self._dump(_capi.lib().dcp_planner_dump_routing)

    def instance_view(self, s):
        v = _capi.InstanceView()
        _capi.check(_capi.lib().dcp_planner_instance_view(self.h, s, ctypes.byref(v)))
        return v

    def kv_append(self, instance, kv_new, pools, stream=None):
        """K8: new-token K/V (bf16 [M, 2, hkv, d], M-row order of `instance`)
        into the frame/slot append_token chose, on whichever instance holds it."""
        arr = (ctypes.c_void_p * self.W)(*[p.data_ptr() for p in pools])
        s = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
        hkv, d = kv_new.shape[2], kv_new.shape[3]
        _capi.check(_capi.lib().dcp_kv_append(self.h, instance, ctypes.c_void_p(kv_new.data_ptr()), arr, hkv, d, s))

    def migrate_kv(self, ids, src_k, src_v, pools, stream=None):
        """Prefill -> decode KV migration (MIGRATE / TRANSFER; dcp_kv_migrate).

        src_k[i], src_v[i]: [seq_len, hkv, d] CUDA tensors (bf16 or fp32) of request ids[i];
        pools[s]: instance s's pool [frames, 2, hkv, page, d] (same dtype), as addressable
        from the launching device.  Each logical page of the request's page table receives
        its tokens, on whichever instance holds the frame."""
        n = len(ids)
        if not (len(src_k) == len(src_v) == n) or len(pools) != self.W:
            raise _capi.DcpInvalidArgument("migrate_kv: ids / sources / pools lengths")
        idv = np.ascontiguousarray(ids, np.int64)
        ks = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in src_k])
        vs = (ctypes.c_void_p * max(n, 1))(*[t.data_ptr() for t in src_v])
        arr = (ctypes.c_void_p * self.W)(*[p.data_ptr() for p in pools])
        hkv, d = pools[0].shape[2], pools[0].shape[4]
        for t in list(src_k) + list(src_v):
            if t.dtype != pools[0].dtype or not t.is_contiguous() or t.shape[1:] != (hkv, d):
                raise _capi.DcpInvalidArgument(f"migrate_kv: source {tuple(t.shape)} {t.dtype}")
        s = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
        _capi.check(_capi.lib().dcp_kv_migrate(self.h, _p(idv), n, ks, vs, arr, hkv, d,
                                               pools[0].element_size(), s))
