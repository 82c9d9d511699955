"""Closed-loop replay: the DST decisions the measured step driver made on B200
from GPU block-score profiles (driver.py, C3 mix at N = 4, SAB + DST, Mean anchor, p = 0.1,
coverage base, dense 1..256 grid, the committed GPU-measured cost table; iteration 0) replayed on
the host from the profiles the GPU produced: this repo's planner and the compiled reference's
simulate_iteration both reproduce the decisions CSV byte for byte.

Fixture: tests/golden/closed_loop/ (copied from gpurun_out/balance_r2/c3_N4/sab_dst/, the run
logged in profiles/r2/README.md)."""
import os

import numpy as np
import pytest

from paper_2604_13847_b200.host import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "closed_loop")
TABLE = os.path.join(FIX, "cost_table_h32_d128_b128.csv")  # the table that run used
KW = dict(gbs=20, mbs=5, dp=4, anchor="mean", threshold_p=0.1, dst_scope="global", base_mode="coverage",
          dst_grid=list(range(1, 257)), iter_index=0)


def _load():
    z = np.load(os.path.join(FIX, "c3_N4_it0_gpu_profiles.npz"))
    L = int(z["layers"])
    lengths = z["lengths"]
    return lengths, [[z[f"p{i}_{l}"] for l in range(L)] for i in range(len(lengths))], L


def _replay(h, table, tmp_path, name):
    lengths, profs, L = _load()
    est = h.make_estimator(h.default_bin_edges(65536), budget_grid=list(table.budget_grid))
    path = str(tmp_path / name)
    h.plan_step("sab_dst", np.arange(len(lengths)), lengths, profs, num_layers=L, table=table, est=est,
                decisions_csv=path, **KW)
    return open(path, "rb").read()


def test_host_replay_of_gpu_profiles_is_bit_identical(tmp_path):
    """The profiles carry real structure (not uniform) and the replay reproduces the GPU run."""
    lengths, profs, L = _load()
    assert L == 36 and len(lengths) == 20
    k90 = [int(np.searchsorted(np.cumsum(p[0]), 0.9) + 1) for p in profs]
    assert min(k90) < max(k90)  # concentration differs between samples (planted routing)
    h = api()
    table = h.load_table(TABLE)[0]
    got = _replay(h, table, tmp_path, "ours.csv")
    want = open(os.path.join(FIX, "c3_N4_it0_decisions.csv"), "rb").read()
    assert got == want


def test_reference_replay_of_gpu_profiles_is_bit_identical(tmp_path, ref):
    h = api()
    table = h.load_table(TABLE)[0]
    got = _replay(ref, table, tmp_path, "ref.csv")
    want = open(os.path.join(FIX, "c3_N4_it0_decisions.csv"), "rb").read()
    assert got == want
