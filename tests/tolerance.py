"""The bf16 parity rule of the device tests (BASELINE.json north_star: "within 2e-2 relative (bf16)").

For an output tensor `got` (rows = (token, head) vectors of the last dim d) against its fp64 /
fp32 reference `ref`:
  * max |got - ref| <= rel * max |ref|                    (relative to the tensor's scale; no floor)
  * per row r with ||ref_r|| > sig * max_r ||ref_r||:
        ||got_r - ref_r|| <= rel * ||ref_r||             (true relative check of every token's own
                                                         output / gradient vector)
  * ||got - ref||_F / ||ref||_F < rel_fro

Why per row and not per element: every tensor-core attention backward rounds dS = P (dP - D) to
bf16 before the dQ / dK GEMMs, and sum_j dS_ij = 0 per query row, so dQ / dK elements are sums
with heavy cancellation. Rounding dS alone (an exact fp64 computation otherwise; 2000 rows x 768
keys, d 128, N(0,1) data) gives 2.4 % elementwise relative error on elements above 5 % of the max
-- a tail statistic over ~10^5 elements -- while each row's error vector is ~0.2-0.5 % of the row
and the relative Frobenius error 0.16 %. The per-row relative L2 rule therefore keeps a wide margin
over the arithmetic any bf16 kernel must do, while a real defect (a wrong or missing block, a lost
column, a mis-scaled row) moves a row by far more than 2 %.
"""
import numpy as np

REL = 2e-2
SIG = 0.05


def check_bf16(got, ref, name="", rel=REL, rel_fro=REL, sig=SIG):
    """Returns (max abs err, worst per-row relative L2 error on significant rows, rel Fro)."""
    if hasattr(got, "detach"):
        got = got.detach().float().cpu().numpy()
    if hasattr(ref, "detach"):
        ref = ref.detach().float().cpu().numpy()
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    assert np.isfinite(got).all(), (name, "non-finite output")
    amax = float(np.abs(ref).max()) if ref.size else 0.0
    err = np.abs(got - ref)
    emax = float(err.max()) if err.size else 0.0
    assert emax <= rel * amax + 1e-30, (name, "max err", emax, "max|ref|", amax)
    d = ref.shape[-1] if ref.ndim else 1
    rr, ee = ref.reshape(-1, d), err.reshape(-1, d)
    rn = np.linalg.norm(rr, axis=1)
    sig_rows = rn > sig * (rn.max() if rn.size else 0.0)
    worst = float((np.linalg.norm(ee[sig_rows], axis=1) / rn[sig_rows]).max()) if sig_rows.any() else 0.0
    assert worst <= rel, (name, "per-row relative L2 error", worst)
    fro = float(np.linalg.norm(got - ref) / max(1e-30, np.linalg.norm(ref)))
    assert fro < rel_fro, (name, "rel Fro", fro)
    return emax, worst, fro
