"""ctypes binding of oracle/_ref/liboracle.so (sb_oracle.c): the CPU restatement of the device
half. TEST ORACLE / CPU BASELINE ONLY -- see oracle/__init__.py."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise FileNotFoundError(f"{LIB} not built (make -C oracle oracle)")
        _lib = C.CDLL(LIB)
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def set_threads(n: int = 0) -> int:
    return lib().orc_set_threads(int(n))


def layout(cu, bsz):
    cu = np.asarray(cu, np.int32)
    nb = (np.diff(cu) + bsz - 1) // bsz
    blk = np.concatenate([[0], np.cumsum(nb)]).astype(np.int32)
    tri = np.concatenate([[0], np.cumsum(nb.astype(np.int64) * (nb + 1) // 2)]).astype(np.int64)
    return blk, tri


def block_pool(x_bf16: np.ndarray, cu, bsz):
    """x: uint16 [T, H, D] (bf16 bits) -> double [NB, H, D]."""
    cu = np.ascontiguousarray(cu, np.int32)
    blk, _ = layout(cu, bsz)
    T, H, D = x_bf16.shape
    out = np.zeros((int(blk[-1]), H, D), np.float64)
    lib().orc_block_pool(_p(np.ascontiguousarray(x_bf16)), _p(cu), _p(blk), C.c_int(len(cu) - 1), C.c_int(H),
                         C.c_int(D), C.c_int(bsz), _p(out))
    return out


def block_scores(qbar, kbar, cu, bsz, scale):
    blk, tri = layout(cu, bsz)
    _, Hq, D = qbar.shape
    Hkv = kbar.shape[1]
    out = np.zeros((Hq, max(1, int(tri[-1]))), np.float64)
    lib().orc_block_scores(_p(np.ascontiguousarray(qbar)), _p(np.ascontiguousarray(kbar)), _p(blk), _p(tri),
                           C.c_int(len(blk) - 1), C.c_int(Hq), C.c_int(Hkv), C.c_int(D), C.c_double(scale), _p(out))
    return out


def topk_select(scores_f32, cu, bsz, k_seq, k_max, group=1, force_diag=True):
    blk, tri = layout(cu, bsz)
    Hs = scores_f32.shape[0]
    hsel = Hs // group
    idx = np.zeros((hsel, int(blk[-1]), k_max), np.int32)
    cnt = np.zeros((hsel, int(blk[-1])), np.int32)
    k_seq = np.ascontiguousarray(k_seq, np.int32)
    lib().orc_topk_select(_p(np.ascontiguousarray(scores_f32, np.float32)), _p(blk), _p(tri), C.c_int(len(blk) - 1),
                          C.c_int(Hs), C.c_int(group), _p(k_seq), C.c_int(k_max), C.c_int(1 if force_diag else 0),
                          _p(idx), _p(cnt))
    return idx, cnt


def coverage_profile(scores_f32, cu, bsz):
    blk, tri = layout(cu, bsz)
    nb_max = int(np.diff(blk).max()) if len(blk) > 1 else 0
    out = np.zeros((len(blk) - 1, max(1, nb_max)), np.float64)
    lib().orc_coverage_profile(_p(np.ascontiguousarray(scores_f32, np.float32)), _p(blk), _p(tri),
                               C.c_int(len(blk) - 1), C.c_int(max(1, nb_max)), C.c_int(scores_f32.shape[0]), _p(out))
    return out


def coverage_at_grid(profile, cu, bsz, grid):
    blk, _ = layout(cu, bsz)
    g = np.ascontiguousarray(grid, np.int32)
    out = np.zeros((len(blk) - 1, len(g)), np.float64)
    lib().orc_coverage_at_grid(_p(np.ascontiguousarray(profile)), _p(blk), C.c_int(len(blk) - 1),
                               C.c_int(profile.shape[1]), _p(g), C.c_int(len(g)), _p(out))
    return out


def sparse_attn_fwd(q, k, v, cu, bsz, idx, cnt, scale):
    """q,k,v: uint16 bf16 bits [T,H,D] -> (O double [T,Hq,D], LSE double [Hq,T])."""
    cu = np.ascontiguousarray(cu, np.int32)
    blk, _ = layout(cu, bsz)
    T, Hq, D = q.shape
    Hkv = k.shape[1]
    hsel, _, k_max = idx.shape
    o = np.zeros((T, Hq, D), np.float64)
    lse = np.zeros((Hq, T), np.float64)
    lib().orc_sparse_attn_fwd(_p(np.ascontiguousarray(q)), _p(np.ascontiguousarray(k)), _p(np.ascontiguousarray(v)),
                              _p(cu), _p(blk), C.c_int(len(cu) - 1), C.c_int(T), C.c_int(Hq), C.c_int(Hkv), C.c_int(D),
                              C.c_int(bsz), _p(np.ascontiguousarray(idx, np.int32)),
                              _p(np.ascontiguousarray(cnt, np.int32)), C.c_int(hsel), C.c_int(k_max),
                              C.c_double(scale), _p(o), _p(lse))
    return o, lse


def sparse_attn_bwd(q, k, v, o, do, lse, cu, bsz, idx, cnt, scale):
    cu = np.ascontiguousarray(cu, np.int32)
    blk, _ = layout(cu, bsz)
    T, Hq, D = q.shape
    Hkv = k.shape[1]
    hsel, _, k_max = idx.shape
    dq = np.zeros((T, Hq, D), np.float64)
    dk = np.zeros((T, Hkv, D), np.float64)
    dv = np.zeros((T, Hkv, D), np.float64)
    lib().orc_sparse_attn_bwd(_p(np.ascontiguousarray(q)), _p(np.ascontiguousarray(k)), _p(np.ascontiguousarray(v)),
                              _p(np.ascontiguousarray(o, np.float64)), _p(np.ascontiguousarray(do)),
                              _p(np.ascontiguousarray(lse, np.float64)), _p(cu), _p(blk), C.c_int(len(cu) - 1),
                              C.c_int(T), C.c_int(Hq), C.c_int(Hkv), C.c_int(D), C.c_int(bsz),
                              _p(np.ascontiguousarray(idx, np.int32)), _p(np.ascontiguousarray(cnt, np.int32)),
                              C.c_int(hsel), C.c_int(k_max), C.c_double(scale), _p(dq), _p(dk), _p(dv))
    return dq, dk, dv
