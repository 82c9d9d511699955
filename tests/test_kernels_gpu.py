"""Device-half parity: the sm_100a kernels (through the C ABI) against the CPU oracle
(oracle/sb_oracle.c, fp64). Tolerances: selections bit-exact on identical fp32 score tensors;
scores / profiles fp32 rules (1e-4 relative); attention outputs and gradients bf16 rules
(2e-2 relative), as BASELINE.json's north_star states."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from tests.tolerance import check_bf16  # noqa: E402

from oracle import device as orc  # noqa: E402


def _bits(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def _rand_bf16(shape, seed, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(shape, generator=g) * scale).to(torch.bfloat16).cuda()


def _layout(cu, B):
    from paper_2604_13847_b200.ops import VarlenLayout

    return VarlenLayout.build(cu, B)


CASES = [
    # cu_seqlens, Hq, Hkv, D, B
    ([0, 4096], 8, 8, 64, 64),           # C1 shape (single 4K sequence, MHA, d64, B64)
    ([0, 300, 1000, 1100], 4, 2, 128, 128),
    ([0, 129, 130, 900], 4, 4, 128, 64),
    ([0, 1000, 1031], 4, 1, 64, 128),
]


@pytest.mark.parametrize("cu,hq,hkv,d,B", CASES)
def test_block_scores_vs_oracle(cu, hq, hkv, d, B):
    from paper_2604_13847_b200 import ops

    T = cu[-1]
    q, k = _rand_bf16((T, hq, d), 1), _rand_bf16((T, hkv, d), 2)
    lay = _layout(cu, B)
    S = ops.block_scores(q, k, lay).cpu().numpy()
    qb, kb = orc.block_pool(_bits(q), cu, B), orc.block_pool(_bits(k), cu, B)
    np.testing.assert_allclose(ops.block_pool(q, lay).cpu().numpy(), qb, rtol=1e-5, atol=1e-6)
    ref = orc.block_scores(qb, kb, cu, B, 1.0 / math.sqrt(d))
    np.testing.assert_allclose(S[:, :lay.tri_total], ref[:, :lay.tri_total], rtol=1e-4, atol=1e-5 * np.abs(ref).max())


def _rand_scores(lay, hs, seed, ties=False, nans=False):
    rng = np.random.default_rng(seed)
    S = rng.standard_normal((hs, max(1, lay.tri_total))).astype(np.float32)
    if ties:
        S = np.round(S * 2) / 2  # many exact ties
    if nans:
        S[rng.random(S.shape) < 0.02] = np.nan
        S[rng.random(S.shape) < 0.02] = -0.0
    return S


@pytest.mark.parametrize("force_diag", [1, 0])
@pytest.mark.parametrize("group", [1, 4])
@pytest.mark.parametrize("ties,nans", [(False, False), (True, False), (True, True)])
def test_topk_select_bitexact(force_diag, group, ties, nans):
    from paper_2604_13847_b200 import ops

    cu = [0, 64 * 70 + 5, 64 * 70 + 5 + 64 * 300, 64 * 70 + 5 + 64 * 300 + 33, 64 * 70 + 5 + 64 * 300 + 33 + 64 * 1500]
    lay = _layout(cu, 64)
    hs = 8
    S = _rand_scores(lay, hs, 7 + group, ties, nans)
    for k_seq in ([1, 2, 3, 4], [16, 8, 1, 40], [71, 301, 1, 1501], [5, 200, 2, 700], [9, 8, 1, 9], [10, 9, 1, 3]):
        k_max = max(k_seq)
        idx, cnt = ops.topk_select(torch.from_numpy(S).cuda(), lay, torch.tensor(k_seq, dtype=torch.int32).cuda(),
                                   k_max, group=group, force_diag=bool(force_diag))
        ridx, rcnt = orc.topk_select(S, cu, 64, k_seq, k_max, group=group, force_diag=bool(force_diag))
        assert np.array_equal(cnt.cpu().numpy(), rcnt)
        assert np.array_equal(idx.cpu().numpy(), ridx)


def test_topk_select_on_reference_routing_scores():
    """Golden: the reference's own routing-score vectors (workload.cpp:42-57, pre-sort), one per
    row; with force_diag=0 the selected set is the top-k and its descending-order sum equals the
    reference's coverage(profile, k) bit-for-bit (dst.cpp:53-61)."""
    from paper_2604_13847_b200 import ops
    from tests.golden_io import load_routing_golden

    g = load_routing_golden()
    for row_scores, sorted_profile, ks, cov in g:
        m = len(row_scores)
        cu = [0, m * 64]
        lay = _layout(cu, 64)
        S = np.full((1, lay.tri_total), -np.inf, np.float32)
        S[0, lay.tri_total - m:] = row_scores.astype(np.float32)  # last row i = m-1 has m entries
        for k, c in zip(ks, cov):
            idx, cnt = ops.topk_select(torch.from_numpy(S).cuda(), lay, torch.tensor([k], dtype=torch.int32).cuda(),
                                       int(k), force_diag=False)
            sel = idx.cpu().numpy()[0, m - 1, :cnt.cpu().numpy()[0, m - 1]]
            vals = np.sort(row_scores[sel])[::-1]
            acc = 0.0
            for v in vals:
                acc += float(v)
            expect = c if k < m else 1.0
            assert (acc if k < m else 1.0) == expect


@pytest.mark.parametrize("cu,hq,hkv,d,B", CASES[:3])
def test_coverage_profile_vs_oracle(cu, hq, hkv, d, B):
    from paper_2604_13847_b200 import ops
    from paper_2604_13847_b200.host import api

    T = cu[-1]
    q, k = _rand_bf16((T, hq, d), 3, 4.0), _rand_bf16((T, hkv, d), 4, 4.0)
    lay = _layout(cu, B)
    S = ops.block_scores(q, k, lay)
    prof = ops.coverage_profile(S, lay).cpu().numpy()
    ref = orc.coverage_profile(S.cpu().numpy(), cu, B)
    np.testing.assert_allclose(prof, ref, atol=2e-6)
    for s, nb in enumerate(lay.nb_per_seq):
        assert abs(prof[s, :nb].sum() - 1.0) < 1e-5
        assert np.all(np.diff(prof[s, :nb]) <= 1e-7)
    grid = [1, 2, 3, 4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 56, 64]
    cov = ops.coverage_at_grid(torch.from_numpy(prof).cuda(), lay, grid).cpu().numpy()
    h = api()
    for s, nb in enumerate(lay.nb_per_seq):
        for gi, kk in enumerate(grid):
            assert cov[s, gi] == h.coverage(prof[s, :nb], kk)  # bit-exact vs host coverage()


def _selection(lay, hsel, keep, seed, force_diag=True):
    """Random scores -> GPU selector (selection is an input of the attention parity test)."""
    from paper_2604_13847_b200 import ops

    S = torch.from_numpy(_rand_scores(lay, hsel, seed)).cuda()
    nb = lay.nb_per_seq
    k_seq = np.maximum(1, np.ceil(keep * nb)).astype(np.int32)
    k_max = int(k_seq.max())
    return ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), k_max, force_diag=force_diag)


ATTN_CASES = [
    # cu, hq, hkv, d, B, hsel_mode, keep
    ([0, 4096], 8, 8, 64, 64, "head", 0.25),           # C1
    ([0, 1000, 1100, 2900], 4, 2, 128, 128, "head", 0.5),
    ([0, 1000, 1100, 2900], 4, 2, 128, 128, "group", 0.3),
    ([0, 77, 700, 2000], 2, 1, 128, 64, "head", 0.4),
    ([0, 33, 1500], 2, 2, 64, 128, "head", 1.0),        # dense
    ([0, 128 * 20], 2, 2, 128, 128, "head", 0.05),      # k = 1: diagonal only
    ([0, 8192, 9000, 12288], 8, 2, 64, 128, "head", 0.3),  # > 1 work item per persistent CTA
]


@pytest.mark.parametrize("cu,hq,hkv,d,B,mode,keep", ATTN_CASES)
def test_sparse_attn_fwd_vs_oracle(cu, hq, hkv, d, B, mode, keep):
    from paper_2604_13847_b200 import ops

    T = cu[-1]
    q, k, v = _rand_bf16((T, hq, d), 11), _rand_bf16((T, hkv, d), 12), _rand_bf16((T, hkv, d), 13)
    lay = _layout(cu, B)
    hsel = hq if mode == "head" else hkv
    idx, cnt = _selection(lay, hsel, keep, 5)
    scale = 1.0 / math.sqrt(d)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    torch.cuda.synchronize()
    ro, rlse = orc.sparse_attn_fwd(_bits(q), _bits(k), _bits(v), cu, B, idx.cpu().numpy(), cnt.cpu().numpy(), scale)
    check_bf16(o, ro, "o", rel_fro=1e-2)
    np.testing.assert_allclose(lse.cpu().numpy(), rlse, atol=2e-3, rtol=1e-4)


BWD_CASES = [
    ([0, 1000, 1100, 2900], 4, 2, 128, 128, "head", 0.5),
    ([0, 1000, 1100, 2900], 4, 2, 128, 128, "group", 0.3),
    ([0, 77, 700, 2000], 2, 1, 128, 64, "head", 0.4),
    ([0, 33, 1500], 2, 2, 64, 128, "head", 1.0),
    ([0, 2048], 4, 4, 64, 64, "head", 0.25),
    ([0, 8192, 9000, 12288], 8, 2, 64, 128, "head", 0.3),   # > 1 work item per persistent CTA
    ([0, 6000, 6100, 9000], 4, 4, 128, 128, "head", 0.5),
]


@pytest.mark.parametrize("cu,hq,hkv,d,B,mode,keep", BWD_CASES)
def test_sparse_attn_bwd_vs_oracle(cu, hq, hkv, d, B, mode, keep):
    from paper_2604_13847_b200 import ops

    T = cu[-1]
    q, k, v = _rand_bf16((T, hq, d), 21), _rand_bf16((T, hkv, d), 22), _rand_bf16((T, hkv, d), 23)
    do = _rand_bf16((T, hq, d), 24)
    lay = _layout(cu, B)
    hsel = hq if mode == "head" else hkv
    idx, cnt = _selection(lay, hsel, keep, 9)
    scale = 1.0 / math.sqrt(d)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    dq, dk, dv = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
    torch.cuda.synchronize()
    ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
    ro, rlse = orc.sparse_attn_fwd(_bits(q), _bits(k), _bits(v), cu, B, ic, cc, scale)
    rdq, rdk, rdv = orc.sparse_attn_bwd(_bits(q), _bits(k), _bits(v), ro, _bits(do), rlse, cu, B, ic, cc, scale)
    for got, ref, name in ((dq, rdq, "dq"), (dk, rdk, "dk"), (dv, rdv, "dv")):
        check_bf16(got, ref, name)


def test_fwd_bwd_large_dynamic_range():
    """Scores spanning hundreds of log2 units: exp2 of x <= -127 must give ~0, not NaN (the
    FMA-pipe exp2 once wrapped its exponent field there), in the fwd and in both bwd passes."""
    from paper_2604_13847_b200 import ops

    cu, hq, d, B = [0, 700, 2000], 2, 128, 128
    T = cu[-1]
    q = (_rand_bf16((T, hq, d), 31).float() * 8).to(torch.bfloat16)  # exact: power-of-two scale
    k, v, do = _rand_bf16((T, hq, d), 32), _rand_bf16((T, hq, d), 33), _rand_bf16((T, hq, d), 34)
    lay = _layout(cu, B)
    idx, cnt = _selection(lay, hq, 0.6, 3)
    scale = 1.0  # std of the scores ~ 90: most exp2 arguments are far below -127
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    dq, dk, dv = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
    torch.cuda.synchronize()
    for t in (o, lse, dq, dk, dv):
        assert torch.isfinite(t.float()).all()
    ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
    ro, rlse = orc.sparse_attn_fwd(_bits(q), _bits(k), _bits(v), cu, B, ic, cc, scale)
    check_bf16(o, ro, "o")
    np.testing.assert_allclose(lse.cpu().numpy(), rlse, atol=2e-3, rtol=1e-4)
    rdq, rdk, rdv = orc.sparse_attn_bwd(_bits(q), _bits(k), _bits(v), ro, _bits(do), rlse, cu, B, ic, cc, scale)
    # Near one-hot softmax rows: the exact dQ / dK of such a row is a cancellation residue
    # (dP_j - D ~ 0 for the dominant key) orders of magnitude below its terms, so fp32 rounding of
    # dP and D sets its relative error; the per-row rule applies to rows above 25 % of the largest
    # row norm here (5 % everywhere else), the global max / Frobenius rules unchanged.
    for got, ref, name in ((dq, rdq, "dq"), (dk, rdk, "dk"), (dv, rdv, "dv")):
        check_bf16(got, ref, name, sig=0.25)


def test_bwd_deterministic():
    from paper_2604_13847_b200 import ops

    cu = [0, 1000, 3000]
    T = cu[-1]
    q, k, v, do = (_rand_bf16((T, 4, 128), s) for s in (31, 32, 33, 34))
    lay = _layout(cu, 128)
    idx, cnt = _selection(lay, 4, 0.5, 3)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
    a = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
    b = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


@pytest.mark.parametrize("hq,hkv,d,B", [(8, 2, 128, 128), (4, 4, 64, 64)])
def test_bwd_split_items_sink_column(hq, hkv, d, B):
    """Column-concentrated selection: every q block selects key block 0 (a sink), with GQA group
    selection, so key block 0's dK/dV item holds every q block x the group's q heads -- far over
    the split cap (attn_bwd.cu dkv_split_kernel). Its chunks' fp32 partials are summed in chunk
    order by dkv_split_reduce_kernel: oracle parity, and bit-identical run to run."""
    from paper_2604_13847_b200 import ops

    cu = [0, 8192, 8300, 12000]
    T = cu[-1]
    q, k, v, do = _rand_bf16((T, hq, d), 41), _rand_bf16((T, hkv, d), 42), _rand_bf16((T, hkv, d), 43), \
        _rand_bf16((T, hq, d), 44)
    lay = _layout(cu, B)
    hsel = hkv
    S = _rand_scores(lay, hsel, 7)
    for s in range(lay.nseq):  # sink: column 0 of every causal row
        for i in range(int(lay.nb_per_seq[s])):
            S[:, lay.tri_off_host[s] + i * (i + 1) // 2] += 50.0
    nb = lay.nb_per_seq
    k_seq = np.minimum(3, nb).astype(np.int32)
    idx, cnt = ops.topk_select(torch.from_numpy(S).cuda(), lay, torch.from_numpy(k_seq).cuda(), 3)
    ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
    assert (ic[:, : int(nb[0]), 0] == 0).all()  # ascending lists: the sink is every row's first entry
    scale = 1.0 / math.sqrt(d)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    a = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
    b = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    ro, rlse = orc.sparse_attn_fwd(_bits(q), _bits(k), _bits(v), cu, B, ic, cc, scale)
    rdq, rdk, rdv = orc.sparse_attn_bwd(_bits(q), _bits(k), _bits(v), ro, _bits(do), rlse, cu, B, ic, cc, scale)
    for got, ref, name in zip(a, (rdq, rdk, rdv), ("dq", "dk", "dv")):
        check_bf16(got, ref, name)


def test_fused_bwd_vs_two_pass():
    """d = B = 128: the opt-in fused single pass against the default deterministic two-pass on the
    same inputs: dK / dV accumulate in TMEM in a fixed order (bit-identical run to run); dQ is
    reduce-added in fp32 across key blocks, so it agrees to fp32 summation order."""
    from paper_2604_13847_b200 import ops

    cu = [0, 1000, 1100, 2900, 6000]
    T = cu[-1]
    q, do = _rand_bf16((T, 8, 128), 71), _rand_bf16((T, 8, 128), 72)
    k, v = _rand_bf16((T, 2, 128), 73), _rand_bf16((T, 2, 128), 74)
    lay = _layout(cu, 128)
    idx, cnt = _selection(lay, 2, 0.4, 5)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt)
    f1 = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, fused=True)
    f2 = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, fused=True)
    det = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt)
    assert torch.equal(f1[1], f2[1]) and torch.equal(f1[2], f2[2])
    for a, b, name in zip(f1, det, ("dq", "dk", "dv")):
        a, b = a.float(), b.float()
        assert ((a - b).norm() / b.norm()).item() < 2e-3, name
        assert (a - b).abs().max().item() <= 1e-2 * b.abs().max().item(), name


def test_autograd_matches_explicit_calls():
    from paper_2604_13847_b200 import ops

    cu = [0, 600, 1300]
    T = cu[-1]
    q, k, v = (_rand_bf16((T, 2, 64), s).requires_grad_(True) for s in (41, 42, 43))
    lay = _layout(cu, 64)
    idx, cnt = _selection(lay, 2, 0.5, 4)
    o = ops.sparse_attention(q, k, v, lay, idx, cnt)
    do = _rand_bf16((T, 2, 64), 44)
    o.backward(do)
    o2, lse = ops.sparse_attn_fwd(q.detach(), k.detach(), v.detach(), lay, idx, cnt)
    dq, dk, dv = ops.sparse_attn_bwd(q.detach(), k.detach(), v.detach(), o2, do, lse, lay, idx, cnt)
    assert torch.equal(o.detach(), o2)
    assert torch.equal(q.grad, dq) and torch.equal(k.grad, dk) and torch.equal(v.grad, dv)


@pytest.mark.parametrize("cu,B", [
    ([0, 300, 300, 1000, 1000, 1129], 128),  # empty sequences in the middle of the pack
    ([0, 1, 2, 66, 194, 195], 64),           # length-1 sequences, exactly B, B + 1
    ([0, 0, 257], 128),                      # leading empty sequence
])
def test_edge_layouts_end_to_end(cu, B):
    """Ragged / empty sequences through scorer -> selector -> fwd -> bwd against the oracle:
    empty sequences own no blocks and no rows; every other row is computed as usual."""
    from paper_2604_13847_b200 import ops

    T = cu[-1]
    hq, hkv, d = 2, 1, 64
    q, k, v, do = _rand_bf16((T, hq, d), 61), _rand_bf16((T, hkv, d), 62), _rand_bf16((T, hkv, d), 63), \
        _rand_bf16((T, hq, d), 64)
    lay = _layout(cu, B)
    scale = 1.0 / math.sqrt(d)
    S = ops.block_scores(q, k, lay, scale)
    rS = orc.block_scores(orc.block_pool(_bits(q), cu, B), orc.block_pool(_bits(k), cu, B), cu, B, scale)
    np.testing.assert_allclose(S.cpu().numpy()[:, :lay.tri_total], rS[:, :lay.tri_total], rtol=1e-4,
                               atol=1e-5 * np.abs(rS).max())
    k_seq = np.full(len(cu) - 1, 2, np.int32)
    idx, cnt = ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), 2, group=hq)
    ridx, rcnt = orc.topk_select(S.cpu().numpy(), cu, B, k_seq, 2, group=hq, force_diag=True)
    assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(cnt.cpu().numpy(), rcnt)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    dq, dk, dv = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale)
    torch.cuda.synchronize()
    ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
    ro, rlse = orc.sparse_attn_fwd(_bits(q), _bits(k), _bits(v), cu, B, ic, cc, scale)
    rdq, rdk, rdv = orc.sparse_attn_bwd(_bits(q), _bits(k), _bits(v), ro, _bits(do), rlse, cu, B, ic, cc, scale)
    for got, ref, name in ((o, ro, "o"), (dq, rdq, "dq"), (dk, rdk, "dk"), (dv, rdv, "dv")):
        check_bf16(got, ref, name)


B256_CASES = [
    ([0, 2048], 2, 2, 128, 0.5),                     # one sequence, 8 blocks
    ([0, 1000, 1100, 2900, 4096], 4, 2, 128, 0.4),   # ragged: partial last blocks, a 100-token sequence
    ([0, 700, 3000], 2, 1, 64, 1.0),                 # dense rows, d64
]


@pytest.mark.parametrize("cu,hq,hkv,d,keep", B256_CASES)
def test_block_256_fwd_bwd_vs_oracle(cu, hq, hkv, d, keep):
    """Block size 256 (the paper's MoBA setting; reference default config.hpp:21):
    scorer -> selector at B = 256, attention through the exact 128-tile re-expression
    (expand256.cu), fwd and bwd against the fp64 oracle run natively at B = 256."""
    from paper_2604_13847_b200 import ops

    B = 256
    T = cu[-1]
    q, k, v, do = _rand_bf16((T, hq, d), 81), _rand_bf16((T, hkv, d), 82), _rand_bf16((T, hkv, d), 83), \
        _rand_bf16((T, hq, d), 84)
    lay = _layout(cu, B)
    scale = 1.0 / math.sqrt(d)
    S = ops.block_scores(q, k, lay, scale)
    rS = orc.block_scores(orc.block_pool(_bits(q), cu, B), orc.block_pool(_bits(k), cu, B), cu, B, scale)
    np.testing.assert_allclose(S.cpu().numpy()[:, :lay.tri_total], rS[:, :lay.tri_total], rtol=1e-4,
                               atol=1e-5 * np.abs(rS).max())
    nb = lay.nb_per_seq
    k_seq = np.maximum(1, np.ceil(keep * nb)).astype(np.int32)
    idx, cnt = ops.topk_select(S, lay, torch.from_numpy(k_seq).cuda(), int(k_seq.max()))
    ridx, rcnt = orc.topk_select(S.cpu().numpy(), cu, B, k_seq, int(k_seq.max()))
    assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(cnt.cpu().numpy(), rcnt)
    o, lse = ops.sparse_attn_fwd(q, k, v, lay, idx, cnt, scale)
    ic, cc = idx.cpu().numpy(), cnt.cpu().numpy()
    ro, rlse = orc.sparse_attn_fwd(_bits(q), _bits(k), _bits(v), cu, B, ic, cc, scale)
    check_bf16(o, ro, "o")
    np.testing.assert_allclose(lse.cpu().numpy(), rlse, atol=2e-3, rtol=1e-4)
    rdq, rdk, rdv = orc.sparse_attn_bwd(_bits(q), _bits(k), _bits(v), ro, _bits(do), rlse, cu, B, ic, cc, scale)
    for fused in (False, True):
        dq, dk, dv = ops.sparse_attn_bwd(q, k, v, o, do, lse, lay, idx, cnt, scale, fused=fused)
        for got, ref, name in ((dq, rdq, "dq"), (dk, rdk, "dk"), (dv, rdv, "dv")):
            check_bf16(got, ref, f"{name} fused={fused}")
