"""Helpers for the -m gpu parity tests (inputs on the device, golden files)."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def require_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def to_dev(ds):
    return (torch.from_numpy(ds.residues.copy()).cuda(), torch.from_numpy(ds.offsets.copy()).cuda())


def load_golden(cfg_idx):
    path = os.path.join(GOLDEN, f"partition_cfg{cfg_idx}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden file for cfg{cfg_idx} not generated")
    with open(os.path.join(GOLDEN, f"partition_cfg{cfg_idx}.json")) as f:
        meta = json.load(f)
    return dict(np.load(path)), meta


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def keys_u64(t: torch.Tensor) -> np.ndarray:
    """device int64 [n][2] (lo, hi) -> uint64 [n][2] (same layout as make_golden.keys_to_u64)."""
    return t.cpu().numpy().view(np.uint64).reshape(-1, 2)


def prof_np(t: torch.Tensor, bins: int) -> np.ndarray:
    return t.cpu().numpy()[:, :bins]


def assert_rel(a, b, tol=1e-12):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.maximum(np.abs(b), 1e-300)
    rel = np.abs(a - b) / den
    rel[(a == b)] = 0.0
    assert rel.max(initial=0.0) <= tol, f"max rel err {rel.max()}"
