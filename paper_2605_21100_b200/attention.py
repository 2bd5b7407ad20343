"""Host-side mirror of the reference attention interface over the device path.

The reference exposes `shard_attention` / `lse_merge` / `sharded_attention_merge`
(attn_merge.hpp:53-121) on contiguous host spans for one query and one head.
On B200 the same math runs batched over a paged bf16 KV pool: every
(shard, q-head) of an instance in one launch of K1 (dcp_splitkv_decode_attn),
with the intra-GPU split combine (K9) fused in.  This wrapper owns the
context and the workspace; tensors are torch CUDA tensors (torch is plumbing
for device memory and streams only).
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import _capi


class DcpContext:
    """One dcp_ctx per CUDA device (mirrors dcp_ctx_create / destroy)."""

    def __init__(self, device: int = 0):
        L = _capi.lib()
        h = ctypes.c_void_p()
        _capi.check(L.dcp_ctx_create(int(device), ctypes.byref(h)))
        self.handle = h
        self.device = device
        self.num_sms = L.dcp_ctx_num_sms(h)

    def close(self):
        if self.handle:
            _capi.lib().dcp_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class DecodeAttention:
    """K1+K9 split-KV paged decode attention (dcp_splitkv_decode_attn).

    kv_pool: bf16 [num_frames, 2, num_kv_heads, page_size, head_dim]
    q:       bf16 [num_shards, num_q_heads, head_dim]
    block_table int32 [P], cu_pages int32 [num_shards+1], shard_len int64 [num_shards],
    page_fill uint8 [P] or None.
    Returns (out fp32 [num_shards, num_q_heads, head_dim], lse fp32 [num_shards, num_q_heads]).
    """

    def __init__(self, ctx: DcpContext, num_q_heads: int, num_kv_heads: int, head_dim: int = 128,
                 page_size: int = 16, max_shards: int = 4096, dtype: str = "bf16"):
        if dtype not in ("bf16", "f32"):
            raise ValueError(f"dtype {dtype!r}")
        self.ctx, self.dtype = ctx, dtype
        self.tdtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.hq, self.hkv, self.d, self.page = num_q_heads, num_kv_heads, head_dim, page_size
        self.max_shards = max_shards
        nbytes = _capi.lib().dcp_attn_workspace_bytes(ctx.handle, max_shards, num_q_heads, head_dim)
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device=f"cuda:{ctx.device}")
        self.args = _capi.AttnArgs()

    def prepare(self, q, kv_pool, block_table, cu_pages, shard_len, page_fill=None, scale=None,
                out=None, lse=None):
        """Fill the argument block once (for repeated / graph-captured launches)."""
        R = q.shape[0]
        if R > self.max_shards:
            raise _capi.DcpInvalidArgument(f"{R} shards > max_shards {self.max_shards}")
        for name, t, dt in (("q", q, self.tdtype), ("kv_pool", kv_pool, self.tdtype),
                            ("block_table", block_table, torch.int32),
                            ("cu_pages", cu_pages, torch.int32), ("shard_len", shard_len, torch.int64)):
            if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
                raise _capi.DcpInvalidArgument(f"{name}: need contiguous CUDA {dt}, got {t.dtype}")
        if out is None:
            out = torch.empty(R, self.hq, self.d, dtype=torch.float32, device=q.device)
        if lse is None:
            lse = torch.empty(R, self.hq, dtype=torch.float32, device=q.device)
        a = self.args
        a.num_shards, a.num_q_heads, a.num_kv_heads = R, self.hq, self.hkv
        a.head_dim, a.page_size = self.d, self.page
        a.num_frames = kv_pool.shape[0]
        a.q, a.kv_pool = q.data_ptr(), kv_pool.data_ptr()
        a.block_table, a.cu_pages, a.shard_len = (block_table.data_ptr(), cu_pages.data_ptr(),
                                                  shard_len.data_ptr())
        a.page_fill = page_fill.data_ptr() if page_fill is not None else None
        a.scale = scale if scale is not None else 1.0 / math.sqrt(self.d)
        a.out, a.lse = out.data_ptr(), lse.data_ptr()
        a.workspace, a.workspace_bytes = self.workspace.data_ptr(), self.workspace.numel()
        self._keep = (q, kv_pool, block_table, cu_pages, shard_len, page_fill, out, lse)
        return out, lse

    def launch(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.ctx.device)
        L = _capi.lib()
        fn = L.dcp_splitkv_decode_attn if self.dtype == "bf16" else L.dcp_splitkv_decode_attn_f32
        _capi.check(fn(self.ctx.handle, ctypes.byref(self.args), ctypes.c_void_p(s.cuda_stream)))

    def __call__(self, *args, stream=None, **kw):
        out, lse = self.prepare(*args, **kw)
        self.launch(stream)
        return out, lse


class MlaDecodeAttention:
    """K10 MLA split-KV paged decode attention (dcp_mla_decode_attn), tcgen05 CTA pairs.

    The DeepSeek-V3 absorbed-latent decode shape (cfg5): 128 q-heads share one
    576-wide cache row per token (512 latent | 64 rope); keys are the whole row,
    values its first 512 columns.  Per (shard, head) the math is the reference's
    shard_attention (attn_merge.hpp:53-82); the reference itself does not model
    MLA.

    kv_pool: bf16 [num_frames, page_size, 576]
    q:       bf16 [num_shards, 128, 576]
    Returns (out fp32 [num_shards, 128, 512], lse fp32 [num_shards, 128]).
    """

    HEADS, LORA, ROPE = 128, 512, 64

    def __init__(self, ctx: DcpContext, page_size: int = 16, max_shards: int = 4096):
        self.ctx, self.page, self.max_shards = ctx, page_size, max_shards
        nbytes = _capi.lib().dcp_mla_workspace_bytes(ctx.handle, max_shards)
        self.workspace = torch.zeros(nbytes, dtype=torch.uint8, device=f"cuda:{ctx.device}")
        self.args = _capi.MlaArgs()

    def prepare(self, q, kv_pool, block_table, cu_pages, shard_len, page_fill=None, scale=None,
                out=None, lse=None):
        R = q.shape[0]
        if R > self.max_shards:
            raise _capi.DcpInvalidArgument(f"{R} shards > max_shards {self.max_shards}")
        for name, t, dt in (("q", q, torch.bfloat16), ("kv_pool", kv_pool, torch.bfloat16),
                            ("block_table", block_table, torch.int32),
                            ("cu_pages", cu_pages, torch.int32), ("shard_len", shard_len, torch.int64)):
            if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
                raise _capi.DcpInvalidArgument(f"{name}: need contiguous CUDA {dt}, got {t.dtype}")
        if out is None:
            out = torch.empty(R, self.HEADS, self.LORA, dtype=torch.float32, device=q.device)
        if lse is None:
            lse = torch.empty(R, self.HEADS, dtype=torch.float32, device=q.device)
        a = self.args
        a.num_shards, a.num_q_heads, a.kv_lora_rank, a.rope_dim = R, self.HEADS, self.LORA, self.ROPE
        a.page_size, a.num_frames = self.page, kv_pool.shape[0]
        a.q, a.kv_pool = q.data_ptr(), kv_pool.data_ptr()
        a.block_table, a.cu_pages, a.shard_len = (block_table.data_ptr(), cu_pages.data_ptr(),
                                                  shard_len.data_ptr())
        a.page_fill = page_fill.data_ptr() if page_fill is not None else None
        # DeepSeek-V3 softmax scale: 1/sqrt(qk_nope_head_dim 128 + qk_rope_head_dim 64)
        a.scale = scale if scale is not None else 1.0 / math.sqrt(192.0)
        a.out, a.lse = out.data_ptr(), lse.data_ptr()
        a.workspace, a.workspace_bytes = self.workspace.data_ptr(), self.workspace.numel()
        self._keep = (q, kv_pool, block_table, cu_pages, shard_len, page_fill, out, lse)
        return out, lse

    def launch(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.ctx.device)
        _capi.check(_capi.lib().dcp_mla_decode_attn(self.ctx.handle, ctypes.byref(self.args),
                                                    ctypes.c_void_p(s.cuda_stream)))

    def __call__(self, *args, stream=None, **kw):
        out, lse = self.prepare(*args, **kw)
        self.launch(stream)
        return out, lse
