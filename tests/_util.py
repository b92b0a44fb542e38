"""Shared helpers: normwise relative error, bf16 rounding, mesh construction."""

from __future__ import annotations

import numpy as np
import torch

# North-star tolerances (BASELINE.json): BF16 with FP32 accumulate vs the f64 oracle.
TOL_BF16 = 2e-2
TOL_FP32 = 1e-3

MESHES = [(1, 1), (1, 2), (2, 2), (2, 4)]


def rel(x, ref) -> float:
    """max|x - ref| / max|ref| (normwise, so near-zero entries do not dominate)."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert x.shape == ref.shape, (x.shape, ref.shape)
    den = max(float(np.max(np.abs(ref))), 1e-30)
    return float(np.max(np.abs(x - ref))) / den


def bf16_round(a) -> np.ndarray:
    return torch.as_tensor(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def mesh(r: int, c: int):
    import paper_2104_05343_b200 as sg

    return sg.create_mesh(sg.MeshConfig(rows=r, cols=c))
