"""The bf16 parity rule of the device tests (BASELINE.json north_star: "within 2e-2 relative (bf16)").

For an output tensor `got` against its fp64 / fp32 reference `ref`:
  * max |got - ref| <= rel * max |ref|            (relative to the tensor's scale, no absolute floor)
  * |got - ref| <= rel * |ref| for every element with |ref| > sig * max |ref|   (true elementwise
    relative check on the elements that are not near zero; near-zero elements are bounded by the
    first rule only, since their relative error is dominated by bf16 cancellation)
  * ||got - ref||_F / ||ref||_F < rel_fro
"""
import numpy as np

REL = 2e-2
SIG = 0.05


def check_bf16(got, ref, name="", rel=REL, rel_fro=REL, sig=SIG):
    """Returns (max abs err, worst elementwise relative err on significant elements, rel Fro)."""
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
    mask = np.abs(ref) > sig * amax
    worst = float((err[mask] / np.abs(ref[mask])).max()) if mask.any() else 0.0
    assert worst <= rel, (name, "elementwise rel err on |ref| > %.2f max|ref|" % sig, worst)
    fro = float(np.linalg.norm(got - ref) / max(1e-30, np.linalg.norm(ref)))
    assert fro < rel_fro, (name, "rel Fro", fro)
    return emax, worst, fro
