"""Shared helpers for the parity tests (test infrastructure)."""
import numpy as np


def rel_l2(got, ref):
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (den if den > 0 else 1.0))


def to_dev_bf16(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to("cuda").to(torch.bfloat16)


def from_dev(t):
    import torch
    return t.detach().to(torch.float32).cpu().numpy().astype(np.float64)
