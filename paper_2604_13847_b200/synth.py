"""Synthetic Q/K/V/dO with planted block-routing structure (benchmark and driver inputs).

Plain N(0,1) activations give near-uniform block scores, so a tuner fed by the GPU scorer would
see no sparsity structure at all. The reference has no activations either: its routing comes
from the workload generator, one gamma(alpha) draw per key block, normalised
(draw_profile, proj/core/src/workload.cpp:42-60, alpha from generate_samples :255-265). These
tensors carry that routing: for member sequence s with routing vector r (the generator's
PRE-sort draws, one per key block), every head's queries get a shared direction u (one per kv
head, so a GQA group agrees) and the keys of block j get b_j * u with
b_j = d^(1/4) * max(ln r_j, LN_FLOOR). Block means then give

    Qbar_i . Kbar_j / sqrt(d) = (d^(1/4) * b_j) / sqrt(d) + O(B^-1/2) = ln r_j + noise,

so the scorer's softmax over key blocks reproduces r (renormalised over the causal prefix) and
the K4 coverage profile the tuner reads carries the generator's concentration. A per-layer
softmax temperature (DPStep.layer_scales) then varies it per layer.

This is input synthesis for benchmarks and tests, not part of the product path.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch

LN_FLOOR = -30.0  # gamma draws of tiny alpha underflow to 0; cap their log score


def planted_qkv(lengths: Sequence[int], routing: Sequence[np.ndarray], hq: int, hkv: int, d: int, block: int,
                seed: int, device="cuda", dtype=torch.bfloat16):
    """-> (q, k, v, do) packed [T, H, d]. routing[s] = member s's per-key-block routing vector
    (ceil(L_s / block) entries, e.g. generate_samples(..., sorted=False)[s][layer])."""
    lengths = [int(x) for x in lengths]
    T = sum(lengths)
    g = torch.Generator(device=device).manual_seed(int(seed))
    q = torch.randn((T, hq, d), generator=g, device=device)
    k = torch.randn((T, hkv, d), generator=g, device=device)
    v = torch.randn((T, hkv, d), generator=g, device=device)
    do = torch.randn((T, hq, d), generator=g, device=device)
    u = torch.randn((hkv, d), generator=g, device=device)
    u = u / u.norm(dim=1, keepdim=True)
    a = d ** 0.25
    q += a * u.repeat_interleave(hq // hkv, dim=0)[None]
    # per-token key coefficient: b_j of the token's key block
    coef = np.zeros(T, np.float32)
    pos = 0
    for L, r in zip(lengths, routing):
        nb = (L + block - 1) // block
        r = np.asarray(r, np.float64)
        if len(r) != nb:
            raise ValueError(f"routing vector of {len(r)} entries for a {L}-token sequence at block {block}")
        with np.errstate(divide="ignore"):
            lr = np.maximum(np.log(r), LN_FLOOR)
        coef[pos:pos + L] = np.repeat(a * lr, block)[:L]
        pos += L
    k += torch.from_numpy(coef).to(device)[:, None, None] * u[None]
    return q.to(dtype), k.to(dtype), v.to(dtype), do.to(dtype)


def expected_block_scores(routing: np.ndarray) -> np.ndarray:
    """The planted score of each key block (ln r_j, floored): what Qbar_i . Kbar_j / sqrt(d)
    approaches as the block size grows."""
    with np.errstate(divide="ignore"):
        return np.maximum(np.log(np.asarray(routing, np.float64)), LN_FLOOR)


def layer_scales(num_layers: int, seed: int) -> np.ndarray:
    """Per-layer softmax temperature (fixed seed): exp(U[-0.5, 1.0])."""
    return np.exp(np.random.default_rng(seed).uniform(-0.5, 1.0, size=num_layers))


def d_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
