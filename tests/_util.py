"""Shared helpers for the parity tests (test infrastructure)."""
import os

import numpy as np


def rel_l2(got, ref):
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    den = np.linalg.norm(ref)
    return record(float(np.linalg.norm(got - ref) / (den if den > 0 else 1.0)))


def record(r):
    """With TED_TOL_REPORT=<file>, append the current test's measured error (tolerance audits:
    the bars in the parity tests are set from these)."""
    rep = os.environ.get("TED_TOL_REPORT")
    if rep:
        with open(rep, "a") as f:
            f.write(f"{os.environ.get('PYTEST_CURRENT_TEST', '?').split(' ')[0]}\t{r:.3e}\n")
    return r


def to_dev_bf16(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to("cuda").to(torch.bfloat16)


def from_dev(t):
    import torch
    return t.detach().to(torch.float32).cpu().numpy().astype(np.float64)
