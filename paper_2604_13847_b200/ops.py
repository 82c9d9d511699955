"""PyTorch-facing operator layer over the sm_100a kernels (C ABI: include/sb_kernels.h).

PyTorch is plumbing here (device memory, streams, autograd bookkeeping); every computation
is one of this repo's CUDA kernels, called through ctypes with raw device pointers on the
current torch stream. There is no CPU or eager fallback: if the native library is missing
or the tensors are not on a CUDA device the call raises.

Operators (reference stand-ins they replace are cited in include/sb_kernels.h):
  block_pool, block_scores       -- K1 + K2 block scorer (MoBA gate)
  topk_select                    -- K3 per-query-block top-k selector
  coverage_profile, coverage_at_grid -- K4 routing profile / C(k) for the sparsity tuner
  sparse_attn_fwd / sparse_attn_bwd / SparseAttention -- K5 / K6 varlen block-sparse attention
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native

_vp = C.c_void_p


def _lib():
    lib = _native.lib()
    if not getattr(lib, "_sb_kernels_bound", False):
        i, i64, f, sz = C.c_int, C.c_int64, C.c_float, C.c_size_t
        sig = {
            "sb_block_layout_host": (i, [_vp, i, i, _vp, _vp, _vp, _vp, _vp]),
            "sb_block_pool": (i, [_vp, _vp, _vp, i, i, i, i, i, _vp, _vp]),
            "sb_block_scores": (i, [_vp, _vp, _vp, _vp, i, i, i, i, i, f, _vp, _vp]),
            "sb_topk_select": (i, [_vp, _vp, _vp, i, i, i, i, i, _vp, i, i, _vp, _vp, _vp]),
            "sb_coverage_profile_workspace_size": (sz, [i64, i, i, i]),
            "sb_coverage_profile": (i, [_vp, _vp, _vp, i, i, i64, i, i, _vp, _vp, _vp]),
            "sb_coverage_at_grid": (i, [_vp, _vp, i, i, _vp, i, _vp, _vp]),
            "sb_sparse_attn_fwd_workspace_size": (sz, [i, i, i]),
            "sb_sparse_attn_fwd_workspace_size_ex": (sz, [i, i, i, i, i, i]),
            "sb_sparse_attn_bwd_workspace_size_ex": (sz, [i, i, i, i, i, i, i, i, i, i]),
            "sb_sparse_attn_fwd": (i, [_vp, _vp, _vp, _vp, _vp, i, i, i, i, i, i, i, _vp, _vp, i, i, f, _vp, _vp,
                                       _vp, _vp]),
            "sb_sparse_attn_fwd_ex": (i, [_vp, _vp, _vp, _vp, _vp, i, i, i, i, i, i, i, _vp, _vp, i, i, f, _vp, _vp,
                                          _vp, _vp, _vp]),
            "sb_sparse_attn_bwd_workspace_size": (sz, [i, i, i, i, i, i, i]),
            "sb_sparse_attn_bwd": (i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, i, i, i, i, i, i, i, _vp, _vp, i, i,
                                       f, _vp, _vp, _vp, _vp, _vp]),
            "sb_sparse_attn_bwd_ex": (i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, i, i, i, i, i, i, i, _vp, _vp,
                                          i, i, f, _vp, _vp, _vp, _vp, _vp, i]),
            "sb_launch_count": (C.c_uint64, []),
            "sb_last_error": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        lib._sb_kernels_bound = True
    return lib


def _call(name, *args):
    lib = _lib()
    _native.check(getattr(lib, name)(*args), lib.sb_last_error)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need_cuda(*ts):
    dev = None
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise RuntimeError("sparsebalance-b200 ops run on CUDA tensors only (no CPU fallback)")
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise ValueError(f"all tensors must be on one device ({dev} vs {t.device})")
    if dev is not None and dev.index is not None and dev.index != torch.cuda.current_device():
        # kernels launch on the current device's current stream
        raise ValueError(f"tensors are on {dev} but the current CUDA device is {torch.cuda.current_device()} "
                         "(use torch.cuda.device(...))")


def _need(t, name: str, dtype, ndim: int | None = None, shape=None):
    """The kernels read raw data_ptr()s as dense row-major arrays of `dtype`: reject anything
    else (a strided view or an fp16/fp32 tensor would otherwise be misread silently)."""
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (got strides {tuple(t.stride())})")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must have {ndim} dims, got shape {tuple(t.shape)}")
    if shape is not None:
        for a, (got, want) in enumerate(zip(t.shape, shape)):
            if want is not None and got != want:
                raise ValueError(f"{name} dim {a} must be {want}, got shape {tuple(t.shape)}")


def _need_qkv(q, k, v, lay: "VarlenLayout"):
    _need(q, "q", torch.bfloat16, 3, (lay.total_tokens, None, None))
    T, _, D = q.shape
    _need(k, "k", torch.bfloat16, 3, (T, None, D))
    if v is not None:
        _need(v, "v", torch.bfloat16, 3, tuple(k.shape))


def _need_sel(idx, cnt, lay: "VarlenLayout"):
    _need(idx, "idx", torch.int32, 3, (None, lay.nb_total, None))
    _need(cnt, "cnt", torch.int32, 2, (idx.shape[0], lay.nb_total))


def launch_count() -> int:
    return int(_lib().sb_launch_count())


@dataclass
class VarlenLayout:
    """Block geometry of a packed varlen batch (cu_seqlens) at block size B.

    blk_off / tri_off are the prefix sums described in include/sb_kernels.h."""

    cu_seqlens_host: np.ndarray
    block_size: int
    blk_off_host: np.ndarray
    tri_off_host: np.ndarray
    nb_total: int
    tri_total: int
    nb_max: int
    cu_seqlens: torch.Tensor | None = None
    blk_off: torch.Tensor | None = None
    tri_off: torch.Tensor | None = None

    @property
    def nseq(self) -> int:
        return len(self.cu_seqlens_host) - 1

    @property
    def total_tokens(self) -> int:
        return int(self.cu_seqlens_host[-1])

    @property
    def nb_per_seq(self) -> np.ndarray:
        return np.diff(self.blk_off_host)

    @classmethod
    def build(cls, cu_seqlens, block_size: int, device="cuda") -> "VarlenLayout":
        cu = np.ascontiguousarray(np.asarray(cu_seqlens, dtype=np.int32))
        nseq = len(cu) - 1
        blk = np.zeros(nseq + 1, np.int32)
        tri = np.zeros(nseq + 1, np.int64)
        nbt, nbm = C.c_int(), C.c_int()
        trit = C.c_int64()
        _call("sb_block_layout_host", cu.ctypes.data_as(_vp), nseq, block_size, blk.ctypes.data_as(_vp),
              tri.ctypes.data_as(_vp), C.byref(nbt), C.byref(trit), C.byref(nbm))
        lay = cls(cu, block_size, blk, tri, nbt.value, trit.value, nbm.value)
        if device is not None:
            lay.cu_seqlens = torch.from_numpy(cu).to(device)
            lay.blk_off = torch.from_numpy(blk).to(device)
            lay.tri_off = torch.from_numpy(tri).to(device)
        return lay


def block_pool(x: torch.Tensor, lay: VarlenLayout) -> torch.Tensor:
    """K1: Xbar [NB, H, D] fp32 = mean of the valid rows of each block."""
    _need_cuda(x)
    _need(x, "x", torch.bfloat16, 3, (lay.total_tokens, None, None))
    T, H, D = x.shape
    out = torch.empty((lay.nb_total, H, D), dtype=torch.float32, device=x.device)
    _call("sb_block_pool", _ptr(x), _ptr(lay.cu_seqlens), _ptr(lay.blk_off), lay.nseq, lay.nb_total, H, D,
          lay.block_size, _ptr(out), _stream())
    return out


def block_scores(q: torch.Tensor, k: torch.Tensor, lay: VarlenLayout, scale: float | None = None,
                 qbar: torch.Tensor | None = None, kbar: torch.Tensor | None = None) -> torch.Tensor:
    """K1+K2: S [Hq, TRI] fp32, S[h][row(s,i)][j] = scale * <Qbar_i, Kbar_j>, j <= i."""
    _need_cuda(q, k, qbar, kbar)
    _need_qkv(q, k, None, lay)
    Hq, D = q.shape[1], q.shape[2]
    Hkv = k.shape[1]
    scale = 1.0 / math.sqrt(D) if scale is None else scale
    qbar = block_pool(q, lay) if qbar is None else qbar
    kbar = block_pool(k, lay) if kbar is None else kbar
    _need(qbar, "qbar", torch.float32, 3, (lay.nb_total, Hq, D))
    _need(kbar, "kbar", torch.float32, 3, (lay.nb_total, Hkv, D))
    S = torch.empty((Hq, max(1, lay.tri_total)), dtype=torch.float32, device=q.device)
    _call("sb_block_scores", _ptr(qbar), _ptr(kbar), _ptr(lay.blk_off), _ptr(lay.tri_off), lay.nseq, lay.nb_max, Hq,
          Hkv, D, C.c_float(scale), _ptr(S), _stream())
    return S


def topk_select(scores: torch.Tensor, lay: VarlenLayout, k_seq: torch.Tensor, k_max: int, group: int = 1,
                force_diag: bool = True):
    """K3: (idx [Hsel, NB, k_max] int32 ascending, -1 padded; cnt [Hsel, NB] int32)."""
    _need_cuda(scores, k_seq)
    _need(scores, "scores", torch.float32, 2, (None, max(1, lay.tri_total)))
    Hs = scores.shape[0]
    hsel = Hs // group
    k_seq = k_seq.to(torch.int32).contiguous()
    if k_seq.numel() != lay.nseq:
        raise ValueError(f"k_seq must have one entry per sequence ({lay.nseq}), got {k_seq.numel()}")
    idx = torch.empty((hsel, lay.nb_total, k_max), dtype=torch.int32, device=scores.device)
    cnt = torch.empty((hsel, lay.nb_total), dtype=torch.int32, device=scores.device)
    _call("sb_topk_select", _ptr(scores), _ptr(lay.blk_off), _ptr(lay.tri_off), lay.nseq, lay.nb_total, lay.nb_max,
          Hs, group, _ptr(k_seq), k_max, 1 if force_diag else 0, _ptr(idx), _ptr(cnt), _stream())
    return idx, cnt


def coverage_profile(scores: torch.Tensor, lay: VarlenLayout) -> torch.Tensor:
    """K4a: per-sequence routing profile [nseq, nb_max] fp64 (zero padded)."""
    _need_cuda(scores)
    _need(scores, "scores", torch.float32, 2, (None, max(1, lay.tri_total)))
    Hs = scores.shape[0]
    ws = torch.empty(max(1, int(_lib().sb_coverage_profile_workspace_size(lay.tri_total, Hs, lay.nseq, lay.nb_max))),
                     dtype=torch.uint8, device=scores.device)
    prof = torch.empty((lay.nseq, max(1, lay.nb_max)), dtype=torch.float64, device=scores.device)
    _call("sb_coverage_profile", _ptr(scores), _ptr(lay.blk_off), _ptr(lay.tri_off), lay.nseq, lay.nb_total,
          lay.tri_total, lay.nb_max, Hs, _ptr(ws), _ptr(prof), _stream())
    return prof


def coverage_at_grid(profile: torch.Tensor, lay: VarlenLayout, grid) -> torch.Tensor:
    """K4b: C[s][g] = coverage(profile_s, grid[g]) (reference dst.cpp:53-61 arithmetic)."""
    _need_cuda(profile)
    _need(profile, "profile", torch.float64, 2, (lay.nseq, None))
    if isinstance(grid, torch.Tensor) and grid.is_cuda and grid.dtype == torch.int32:
        g = grid
    else:
        g = torch.as_tensor(np.asarray(grid, np.int32), device=profile.device)
    out = torch.empty((lay.nseq, len(g)), dtype=torch.float64, device=profile.device)
    _call("sb_coverage_at_grid", _ptr(profile), _ptr(lay.blk_off), lay.nseq, profile.shape[1], _ptr(g), len(g),
          _ptr(out), _stream())
    return out


def dst_decide(profile: torch.Tensor, lay: VarlenLayout, mb_off: torch.Tensor, k_base: torch.Tensor,
               k_anchor: torch.Tensor, bottleneck: torch.Tensor, grid: torch.Tensor, threshold_p: float):
    """K8 (fixed-base on-device DST): (k_final [n_mb] int32, coverage_drop [n_mb] fp64,
    k_seq [nseq] int32 = min(k_final, nb_s)). All inputs device tensors; mb_off int32 [n_mb+1]
    partitions the layout's sequences into micro-batches."""
    _need_cuda(profile, mb_off, k_base, k_anchor, bottleneck, grid)
    _need(profile, "profile", torch.float64, 2, (lay.nseq, None))
    for t_, n_ in ((mb_off, "mb_off"), (k_base, "k_base"), (k_anchor, "k_anchor"), (bottleneck, "bottleneck"),
                   (grid, "grid")):
        _need(t_, n_, torch.int32, 1)
    n_mb = mb_off.numel() - 1
    k_final = torch.empty(n_mb, dtype=torch.int32, device=profile.device)
    drop = torch.empty(n_mb, dtype=torch.float64, device=profile.device)
    k_seq = torch.empty(lay.nseq, dtype=torch.int32, device=profile.device)
    _call("sb_dst_decide", _ptr(profile), _ptr(lay.blk_off), _ptr(lay.cu_seqlens), profile.shape[1], _ptr(mb_off),
          n_mb, _ptr(k_base), _ptr(k_anchor), _ptr(bottleneck), _ptr(grid), grid.numel(), C.c_double(threshold_p),
          _ptr(k_final), _ptr(drop), _ptr(k_seq), _stream())
    return k_final, drop, k_seq


def sparse_attn_fwd(q, k, v, lay: VarlenLayout, idx, cnt, scale: float | None = None, residual: bool = True):
    """K5: (O [T, Hq, D] bf16, LSE [Hq, T] fp32 natural log). With residual (default) the kernel also
    writes O's bf16 rounding residual, attached as `lse.o_res`; sparse_attn_bwd then forms
    D = rowsum(dO * O) from O + residual (accurate dQ on rows that attend few keys)."""
    _need_cuda(q, k, v, idx, cnt)
    _need_qkv(q, k, v, lay)
    _need_sel(idx, cnt, lay)
    T, Hq, D = q.shape
    Hkv = k.shape[1]
    hsel, _, k_max = idx.shape
    scale = 1.0 / math.sqrt(D) if scale is None else scale
    o = torch.empty_like(q)
    o_res = torch.empty_like(q) if residual else None
    lse = torch.empty((Hq, T), dtype=torch.float32, device=q.device)
    ws = torch.empty(max(16, int(_lib().sb_sparse_attn_fwd_workspace_size_ex(lay.nseq, lay.nb_total, Hq, hsel, k_max,
                                                                            lay.block_size))),
                     dtype=torch.uint8, device=q.device)
    _call("sb_sparse_attn_fwd_ex", _ptr(q), _ptr(k), _ptr(v), _ptr(lay.cu_seqlens), _ptr(lay.blk_off), lay.nseq, T,
          lay.nb_total, Hq, Hkv, D, lay.block_size, _ptr(idx), _ptr(cnt), hsel, k_max, C.c_float(scale), _ptr(o),
          _ptr(o_res), _ptr(lse), _ptr(ws), _stream())
    if o_res is not None:
        lse.o_res = o_res
    return o, lse


SB_BWD_DETERMINISTIC = 1
SB_BWD_FUSED = 2


def sparse_attn_bwd(q, k, v, o, do, lse, lay: VarlenLayout, idx, cnt, scale: float | None = None,
                    o_res=None, fused: bool = False):
    """K6: (dQ, dK, dV) bf16. Default: the bit-deterministic two-pass backward. fused=True (d = B
    = 128): the single pass with dQ reduce-added in fp32 (reproducible to summation order; opt-in,
    it measures slower on B200, see sb_kernels.h)."""
    _need_cuda(q, k, v, o, do, lse, idx, cnt)
    _need_qkv(q, k, v, lay)
    _need_sel(idx, cnt, lay)
    do = do.contiguous()  # autograd may hand a strided / expanded gradient
    _need(o, "o", torch.bfloat16, 3, tuple(q.shape))
    _need(do, "do", torch.bfloat16, 3, tuple(q.shape))
    _need(lse, "lse", torch.float32, 2, (q.shape[1], q.shape[0]))
    o_res = o_res if o_res is not None else getattr(lse, "o_res", None)
    if o_res is not None:
        _need_cuda(o_res)
        _need(o_res, "o_res", torch.bfloat16, 3, tuple(q.shape))
    T, Hq, D = q.shape
    Hkv = k.shape[1]
    hsel, _, k_max = idx.shape
    scale = 1.0 / math.sqrt(D) if scale is None else scale
    flags = SB_BWD_FUSED if fused else SB_BWD_DETERMINISTIC
    ws_bytes = int(_lib().sb_sparse_attn_bwd_workspace_size_ex(lay.nseq, T, lay.nb_total, Hq, Hkv, D, hsel, k_max,
                                                               lay.block_size, flags))
    ws = torch.empty(max(1, ws_bytes), dtype=torch.uint8, device=q.device)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    _call("sb_sparse_attn_bwd_ex", _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(o_res), _ptr(do), _ptr(lse),
          _ptr(lay.cu_seqlens), _ptr(lay.blk_off), lay.nseq, T, lay.nb_total, Hq, Hkv, D, lay.block_size, _ptr(idx),
          _ptr(cnt), hsel, k_max, C.c_float(scale), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), _stream(),
          flags)
    return dq, dk, dv


class SparseAttention(torch.autograd.Function):
    """Autograd wrapper: forward = K5, backward = K6 (recompute from the saved LSE)."""

    @staticmethod
    def forward(ctx, q, k, v, lay, idx, cnt, scale, fused=False):
        o, lse = sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
        ctx.save_for_backward(q, k, v, o, lse, idx, cnt)
        ctx.lay, ctx.scale, ctx.fused = lay, scale, fused
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse, idx, cnt = ctx.saved_tensors
        dq, dk, dv = sparse_attn_bwd(q, k, v, o, do, lse, ctx.lay, idx, cnt, ctx.scale, fused=ctx.fused)
        return dq, dk, dv, None, None, None, None, None


def sparse_attention(q, k, v, lay, idx, cnt, scale=None, fused=False):
    return SparseAttention.apply(q, k, v, lay, idx, cnt, scale, fused)
