"""Test-only checker for full-size shapes: block-sparse causal attention in plain PyTorch fp32 on
the GPU, gathered per q block over the selected key blocks, with autograd for the gradients.

It restates the same semantics as oracle/sb_oracle.c (Eq. 2; diagonal
block causal, keys past the sequence end masked, empty rows -> zero output / LSE -inf), and
is used only where the fp64 C oracle would take minutes (C2 / C3 / C4 / C5 full sizes), on a
subset of heads. Never part of the product path."""
from __future__ import annotations

import math

import torch


def _gather_rows(lists: torch.Tensor, cnts: torch.Tensor, seq0: int, seq_len: int, B: int):
    """lists [n, k_max] key-block indices (local to the sequence, -1 pads), cnts [n] ->
    token index [n, k_max*B] (clamped) and validity mask [n, k_max*B]."""
    n, k_max = lists.shape
    t = torch.arange(B, device=lists.device)
    jb = lists.clamp(min=0)
    tok = jb[:, :, None] * B + t[None, None, :]                     # [n, k_max, B] local token
    slot = torch.arange(k_max, device=lists.device)[None, :, None]
    valid = (slot < cnts[:, None, None]) & (lists[:, :, None] >= 0) & (tok < seq_len)
    tok = torch.where(valid, tok, torch.zeros_like(tok)) + seq0
    return tok.reshape(n, k_max * B), valid.reshape(n, k_max * B), jb


def sparse_attention_ref(q, k, v, do, cu, B, idx, cnt, scale, heads, hsel, chunk=64):
    """fp32 reference for the q heads in `heads`.

    q [T, hq, d], k/v [T, hkv, d], do [T, hq, d] (any float dtype, CUDA); idx [hsel, NB, k_max],
    cnt [hsel, NB] (the selector's output). Returns {h: (o [T, d], lse [T])} and the fp32 grads
    (dq [T, hq, d] for those heads; dk, dv [T, hkv, d] accumulated over those heads only)."""
    T, hq, d = q.shape
    hkv = k.shape[1]
    # TF32 GEMMs: bf16 inputs are exact in TF32 and accumulation stays fp32, so the checker
    # remains ~1e-3 relative -- an order of magnitude inside the 2e-2 bf16 bar it enforces.
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        return _ref(q, k, v, do, cu, B, idx, cnt, scale, heads, hsel, chunk, T, hq, hkv, d)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _ref(q, k, v, do, cu, B, idx, cnt, scale, heads, hsel, chunk, T, hq, hkv, d):
    qf = q.float().detach().requires_grad_(True)
    kf = k.float().detach().requires_grad_(True)
    vf = v.float().detach().requires_grad_(True)
    dof = do.float()
    out = {}
    cu = [int(x) for x in cu]
    nb = [(cu[s + 1] - cu[s] + B - 1) // B for s in range(len(cu) - 1)]
    blk_off = [0]
    for x in nb:
        blk_off.append(blk_off[-1] + x)
    for h in heads:
        hk = h // (hq // hkv)
        srow = h // (hq // hsel)
        o_h = torch.zeros(T, d, device=q.device)
        lse_h = torch.full((T,), -math.inf, device=q.device)
        for s in range(len(cu) - 1):
            seq0, L = cu[s], cu[s + 1] - cu[s]
            for i0 in range(0, nb[s], chunk):
                i1 = min(nb[s], i0 + chunk)
                n = i1 - i0
                lists = idx[srow, blk_off[s] + i0:blk_off[s] + i1].long()
                cnts = cnt[srow, blk_off[s] + i0:blk_off[s] + i1].long()
                tok, valid, _ = _gather_rows(lists, cnts, seq0, L, B)
                qi = torch.arange(i0 * B, i1 * B, device=q.device).reshape(n, B)   # local query pos
                qrow_valid = qi < L
                qtok = torch.where(qrow_valid, qi, torch.zeros_like(qi)) + seq0
                Q = qf[qtok, h]                                                   # [n, B, d]
                K = kf[tok, hk]                                                   # [n, kB, d]
                V = vf[tok, hk]
                S = torch.einsum("nqd,nkd->nqk", Q, K) * scale
                kpos = tok - seq0
                mask = valid[:, None, :] & (kpos[:, None, :] <= qi[:, :, None])
                S = S.masked_fill(~mask, -math.inf)
                m = S.amax(dim=-1, keepdim=True)
                m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
                P = torch.exp(S - m)
                l = P.sum(dim=-1, keepdim=True)
                O = torch.einsum("nqk,nkd->nqd", P / torch.where(l > 0, l, torch.ones_like(l)), V)
                lse = torch.where(l[..., 0] > 0, m[..., 0] + torch.log(l[..., 0]), torch.full_like(l[..., 0], -math.inf))
                dO = dof[qtok, h] * qrow_valid[..., None]
                (O * dO).sum().backward()
                sel = qrow_valid.reshape(-1)
                o_h[qtok.reshape(-1)[sel]] = O.detach().reshape(-1, d)[sel]
                lse_h[qtok.reshape(-1)[sel]] = lse.detach().reshape(-1)[sel]
        out[h] = (o_h, lse_h)
    return out, qf.grad, kf.grad, vf.grad


def assert_close_bf16(got, ref, rel_fro, name=""):
    """The bf16 rule of the device parity tests (tests/tolerance.py)."""
    from tests.tolerance import check_bf16

    return check_bf16(got, ref, name, rel_fro=rel_fro)
