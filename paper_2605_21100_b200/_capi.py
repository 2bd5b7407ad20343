"""ctypes binding of include/dcp_capi.h (the product C ABI).

The product is libdcp_b200.so (sm_100a kernels + C ABI + dcpsim C++ drop-in).
This module only loads it and maps status codes onto the dcpsim exception
hierarchy (reference types.hpp:19-30).  There is no fallback: if the library
or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes
from ctypes import (POINTER, Structure, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t,
                    c_void_p)
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_build" / "libdcp_b200.so"


# ---- dcpsim exception hierarchy (types.hpp:19-30) -------------------------------
class SimError(RuntimeError):
    pass


class InsufficientFrames(SimError):
    pass


class UnknownRequest(SimError):
    pass


class UnknownPage(SimError):
    pass


class InconsistentPlacement(SimError):
    pass


class ShapeOverflow(SimError):
    pass


class EmptyShard(SimError):
    pass


class ConfigError(SimError):
    pass


class DcpInvalidArgument(ValueError):
    pass


class DcpUnsupported(NotImplementedError):
    pass


class DcpCudaError(RuntimeError):
    pass


class ExchangeTimeout(RuntimeError):
    """A peer flag wait of the exchange / MoE pools timed out (DCP_E_TIMEOUT)."""


_CODES = {
    -1: InsufficientFrames, -2: UnknownRequest, -3: UnknownPage, -4: InconsistentPlacement,
    -5: ShapeOverflow, -6: EmptyShard, -7: ConfigError, -8: DcpInvalidArgument,
    -9: DcpUnsupported, -10: DcpCudaError, -11: ExchangeTimeout,
}


class AttnArgs(Structure):
    _fields_ = [
        ("num_shards", c_int32), ("num_q_heads", c_int32), ("num_kv_heads", c_int32),
        ("head_dim", c_int32), ("page_size", c_int32), ("num_frames", c_int64),
        ("q", c_void_p), ("kv_pool", c_void_p), ("block_table", c_void_p),
        ("cu_pages", c_void_p), ("shard_len", c_void_p), ("page_fill", c_void_p),
        ("scale", c_float), ("out", c_void_p), ("lse", c_void_p),
        ("workspace", c_void_p), ("workspace_bytes", c_size_t),
    ]


class MlaArgs(Structure):
    _fields_ = [
        ("num_shards", c_int32), ("num_q_heads", c_int32), ("kv_lora_rank", c_int32),
        ("rope_dim", c_int32), ("page_size", c_int32), ("num_frames", c_int64),
        ("q", c_void_p), ("kv_pool", c_void_p), ("block_table", c_void_p),
        ("cu_pages", c_void_p), ("shard_len", c_void_p), ("page_fill", c_void_p),
        ("scale", c_float), ("out", c_void_p), ("lse", c_void_p),
        ("workspace", c_void_p), ("workspace_bytes", c_size_t),
    ]


class PlannerConfig(Structure):
    _fields_ = [
        ("nodes", c_int32), ("instances_per_node", c_int32), ("page_size", c_int64),
        ("capacity_pages", c_int64), ("policy", c_int32), ("n_bucket", c_int32),
        ("bucket_len", c_void_p), ("bucket_deg", c_void_p), ("uniform_degree", c_int32),
        ("hol_strict", c_int32), ("max_requests", c_int32), ("reserve_pages", c_int64),
    ]


class InstanceView(Structure):
    _fields_ = [
        ("n_rows", c_int32), ("m_rows", c_int32), ("bucket_m", c_int32), ("bucket_n", c_int32),
        ("n_ids", c_void_p), ("n_moe", c_void_p), ("q_route", c_void_p), ("m_ids", c_void_p),
        ("res_route", c_void_p), ("cu_pages", c_void_p), ("shard_len", c_void_p),
        ("block_table", c_void_p), ("page_fill", c_void_p),
        ("n_mrow", c_void_p), ("m_nrow", c_void_p), ("m_k", c_void_p), ("m_kv", c_void_p),
        ("m_count_all", c_void_p), ("n_count_dev", c_void_p), ("world", c_int32), ("instance", c_int32),
        ("total_pages_dev", c_void_p),
    ]


class MoeConfig(Structure):
    _fields_ = [("world", c_int32), ("self", c_int32), ("hidden", c_int32), ("topk", c_int32),
                ("num_experts", c_int32), ("m_max", c_int32), ("timeout_ms", c_int32)]


class XchgConfig(Structure):
    _fields_ = [("world", c_int32), ("self", c_int32), ("num_q_heads", c_int32), ("head_dim", c_int32),
                ("n_max", c_int32), ("m_max", c_int32), ("q_dim", c_int32), ("o_dim", c_int32),
                ("q_elem_bytes", c_int32), ("timeout_ms", c_int32)]


EXPERT_FN = ctypes.CFUNCTYPE(None, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p)


class LayerGraphDesc(Structure):
    _fields_ = [("planner", c_void_p), ("xchg", c_void_p), ("view", POINTER(InstanceView)),
                ("attn", POINTER(AttnArgs)), ("moe", c_void_p), ("moe_x", c_void_p), ("topk_idx", c_void_p),
                ("topk_w", c_void_p), ("y_region", c_void_p), ("moe_out", c_void_p), ("expert", EXPERT_FN),
                ("expert_user", c_void_p), ("fused_step", c_int32)]


_lib = None

# (name, restype, argtypes) for every entry point of include/dcp_capi.h.
_SIGNATURES = [
    ("dcp_last_error", c_char_p, []),
    ("dcp_version", c_char_p, []),
    ("dcp_ctx_create", c_int, [c_int, POINTER(c_void_p)]),
    ("dcp_ctx_destroy", c_int, [c_void_p]),
    ("dcp_ctx_num_sms", c_int, [c_void_p]),
    ("dcp_copy_to_host", c_int, [c_void_p, c_void_p, c_size_t]),
    ("dcp_device_sleep", c_int, [c_void_p, c_int32, c_void_p]),
    ("dcp_attn_workspace_bytes", c_size_t, [c_void_p, c_int32, c_int32, c_int32]),
    ("dcp_splitkv_decode_attn", c_int, [c_void_p, POINTER(AttnArgs), c_void_p]),
    ("dcp_attn_launches_per_call", c_int, []),
    ("dcp_splitkv_decode_attn_f32", c_int, [c_void_p, POINTER(AttnArgs), c_void_p]),
    ("dcp_mla_workspace_bytes", c_size_t, [c_void_p, c_int32]),
    ("dcp_mla_decode_attn", c_int, [c_void_p, POINTER(MlaArgs), c_void_p]),
    ("dcp_mla_launches_per_call", c_int, []),
    ("dcp_mla_set_trace", c_int, [c_void_p]),
    ("dcp_planner_create", c_int, [c_void_p, POINTER(PlannerConfig), POINTER(c_void_p)]),
    ("dcp_planner_destroy", c_int, [c_void_p]),
    ("dcp_planner_enqueue", c_int, [c_void_p, c_void_p, c_void_p, c_int32]),
    ("dcp_planner_step", c_int, [c_void_p, c_void_p]),
    ("dcp_planner_step_result", c_int, [c_void_p] + [c_void_p] * 7),
    ("dcp_planner_finish", c_int, [c_void_p, c_void_p, c_int32, c_void_p]),
    ("dcp_planner_append_token", c_int, [c_void_p, c_void_p, c_int32, c_void_p]),
    ("dcp_planner_placement", c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("dcp_planner_instances", c_int, [c_void_p] + [c_void_p] * 4),
    ("dcp_planner_dump_page_table", c_int64, [c_void_p, c_char_p, c_int64]),
    ("dcp_planner_build_routing", c_int, [c_void_p, c_void_p]),
    ("dcp_planner_dump_routing", c_int64, [c_void_p, c_char_p, c_int64]),
    ("dcp_planner_instance_view", c_int, [c_void_p, c_int32, POINTER(InstanceView)]),
    ("dcp_planner_last_launches", c_int, [c_void_p]),
    ("dcp_xchg_create", c_int, [c_void_p, POINTER(XchgConfig), POINTER(c_void_p)]),
    ("dcp_xchg_destroy", c_int, [c_void_p]),
    ("dcp_xchg_ipc_handle", c_int, [c_void_p, c_void_p]),
    ("dcp_xchg_open_peer_ipc", c_int, [c_void_p, c_int32, c_void_p]),
    ("dcp_xchg_set_peer_local", c_int, [c_void_p, c_int32, c_void_p]),
    ("dcp_xchg_commit", c_int, [c_void_p]),
    ("dcp_xchg_begin_step", c_int, [c_void_p, c_void_p]),
    ("dcp_xchg_buffers", c_int, [c_void_p] + [POINTER(c_void_p)] * 4),
    ("dcp_xchg_write_queries", c_int, [c_void_p, c_void_p, c_int32, c_void_p]),
    ("dcp_route_q", c_int, [c_void_p, POINTER(InstanceView), c_void_p]),
    ("dcp_decode_attn_routed", c_int, [c_void_p, c_void_p, POINTER(InstanceView), POINTER(AttnArgs), c_void_p]),
    ("dcp_decode_step_fused", c_int, [c_void_p, c_void_p, POINTER(InstanceView), POINTER(AttnArgs), c_void_p]),
    ("dcp_decode_attn_routed_f32", c_int, [c_void_p, c_void_p, POINTER(InstanceView), POINTER(AttnArgs), c_void_p]),
    ("dcp_mla_decode_attn_routed", c_int, [c_void_p, c_void_p, POINTER(InstanceView), POINTER(MlaArgs), c_void_p]),
    ("dcp_merge_partials", c_int, [c_void_p, POINTER(InstanceView), c_void_p]),
    ("dcp_xchg_status", c_int, [c_void_p, c_void_p]),
    ("dcp_planner_set_policy", c_int, [c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_int32, c_int32]),
    ("dcp_planner_set_queue", c_int, [c_void_p, c_void_p, c_void_p, c_int32]),
    ("dcp_planner_ucp_rr", c_int, [c_void_p, c_void_p, c_int32, c_int32]),
    ("dcp_planner_allocate", c_int, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p, c_int32]),
    ("dcp_planner_pages", c_int64, [c_void_p, c_int64, c_void_p, c_void_p, c_int64]),
    ("dcp_planner_active_moe", c_int32, [c_void_p, c_void_p, c_void_p, c_int32]),
    ("dcp_planner_rebalance", c_int, [c_void_p, c_void_p, c_int32]),
    ("dcp_planner_load_instances", c_int, [c_void_p] + [c_void_p] * 5),
    ("dcp_water_fill", c_int, [c_void_p, c_int32, c_void_p, c_int64, c_void_p]),
    ("dcp_binding_config", c_int, [c_void_p, c_int32] + [c_void_p] * 4 + [c_int32] + [c_void_p] * 4),
    ("dcp_route_tables", c_int, [c_void_p, c_int32, c_int32, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    ("dcp_shard_attention_batch", c_int, [c_void_p, c_int32, c_int32, c_int32, ctypes.c_double] + [c_void_p] * 9),
    ("dcp_lse_merge_batch", c_int, [c_void_p, c_int32, c_int32, c_int32] + [c_void_p] * 6),
    ("dcp_step_graph_create", c_int, [c_void_p, c_void_p, POINTER(InstanceView), POINTER(AttnArgs),
                                      POINTER(c_void_p)]),
    ("dcp_step_graph_launch", c_int, [c_void_p, c_int32, c_int32, c_void_p]),
    ("dcp_step_graph_count", c_int, [c_void_p, c_void_p]),
    ("dcp_step_graph_destroy", c_int, [c_void_p]),
    ("dcp_kv_append", c_int, [c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_int32, c_void_p]),
    ("dcp_k1_set_trace", c_int, [c_void_p]),
    ("dcp_kv_migrate", c_int, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_int32, c_int32,
                               c_int32, c_void_p]),
    ("dcp_moe_create", c_int, [c_void_p, POINTER(MoeConfig), POINTER(c_void_p)]),
    ("dcp_moe_destroy", c_int, [c_void_p]),
    ("dcp_moe_ipc_handle", c_int, [c_void_p, c_void_p]),
    ("dcp_moe_open_peer_ipc", c_int, [c_void_p, c_int32, c_void_p]),
    ("dcp_moe_set_peer_local", c_int, [c_void_p, c_int32, c_void_p]),
    ("dcp_moe_commit", c_int, [c_void_p]),
    ("dcp_moe_begin_step", c_int, [c_void_p, c_void_p]),
    ("dcp_moe_status", c_int, [c_void_p, c_void_p]),
    ("dcp_moe_receive_regions", c_int, [c_void_p, c_void_p]),
    ("dcp_moe_parity", c_int32, [c_void_p]),
    ("dcp_moe_regions", c_int, [c_void_p, c_int32, POINTER(c_void_p), POINTER(c_void_p)]),
    ("dcp_moe_combine_put_regions", c_int, [c_void_p, c_void_p, c_void_p]),
    ("dcp_moe_meta_width", c_int32, [c_void_p]),
    ("dcp_moe_dispatch", c_int, [c_void_p] + [c_void_p] * 5),
    ("dcp_moe_receive", c_int32, [c_void_p] + [c_void_p] * 4),
    ("dcp_moe_receive_async", c_int, [c_void_p] + [c_void_p] * 3),
    ("dcp_moe_recv_counts_dev", c_void_p, [c_void_p]),
    ("dcp_moe_combine_put", c_int, [c_void_p, c_void_p, c_void_p]),
    ("dcp_moe_combine_reduce", c_int, [c_void_p, c_void_p, c_void_p]),
    ("dcp_moe_combine_fused", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("dcp_moe_expert_identity", c_int, [c_void_p, c_void_p, c_void_p]),
    ("dcp_moe_step_dispatch", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("dcp_moe_step_dispatch_recv", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("dcp_layer_graph_create", c_int, [c_void_p, POINTER(LayerGraphDesc), POINTER(c_void_p)]),
    ("dcp_layer_graph_launch", c_int, [c_void_p, c_int32, c_void_p]),
    ("dcp_layer_graph_info", c_int, [c_void_p, c_void_p, c_void_p]),
    ("dcp_layer_graph_destroy", c_int, [c_void_p]),
]


def exported_symbols():
    return [s[0] for s in _SIGNATURES]


def lib():
    """Load libdcp_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2605_21100_b200.build` "
                              "(no CPU fallback exists)")
        L = ctypes.CDLL(str(LIB_PATH), mode=ctypes.RTLD_GLOBAL)
        for name, res, args in _SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().dcp_last_error().decode(errors="replace")
        raise _CODES.get(rc, RuntimeError)(f"dcp error {rc}: {msg}")


def device_to_numpy(ptr, n, dtype):
    """Copy n elements of `dtype` from a device pointer (dcp_copy_to_host)."""
    import numpy as np
    out = np.zeros(max(int(n), 0), dtype)
    if n:
        check(lib().dcp_copy_to_host(out.ctypes.data, ptr, out.nbytes))
    return out
