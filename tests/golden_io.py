"""Readers for the committed golden fixtures in tests/golden (written by oracle/gen_golden.py
from the compiled reference, so they travel to the GPU box where /root/reference is absent)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_routing_golden():
    z = np.load(os.path.join(GOLDEN, "routing_scores.npz"))
    out = []
    for r in range(int(z["n"])):
        out.append((z[f"row{r}"], z[f"sorted{r}"], z[f"ks{r}"], z[f"cov{r}"]))
    return out


def load_host_golden():
    with open(os.path.join(GOLDEN, "host_decisions.json")) as f:
        return json.load(f)
