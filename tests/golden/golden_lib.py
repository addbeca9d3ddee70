"""Shared helpers of the golden fixtures (no reference import: safe on the GPU box)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

GOLDEN_DIR = os.path.dirname(os.path.abspath(__file__))
FULL_GRAD_MAX = 20000   # K*N up to which gradients/thetas are stored verbatim
N_PROBES = 16
N_SAMPLED = 2048


def seeded_theta(seed: int, k: int, n: int, scale: float, base_seed: int | None = None,
                 base_scale: float = 1.0) -> np.ndarray:
    """theta = base_scale * N(0,1)[base_seed] + scale * N(0,1)[seed] (base optional)."""
    th = scale * np.random.default_rng(seed).normal(size=(k, n))
    if base_seed is not None:
        th = base_scale * np.random.default_rng(base_seed).normal(size=(k, n)) + th
    return th


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def probes(k: int, n: int) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(2024)
    proj = rng.normal(size=(N_PROBES, k * n))
    idx = np.sort(rng.choice(k * n, size=min(N_SAMPLED, k * n), replace=False))
    return proj, idx


def grad_summary(grad: np.ndarray) -> dict:
    proj, idx = probes(*grad.shape)
    flat = grad.ravel()
    return {"norm": np.linalg.norm(flat), "proj": proj @ flat, "idx": idx, "vals": flat[idx]}


def load(name: str):
    return np.load(os.path.join(GOLDEN_DIR, name + ".npz"), allow_pickle=False)


def thetas(z) -> list:
    """Rebuild the theta list of a golden case (verbatim or from its seeds)."""
    out = []
    j = 0
    while f"phi{j}" in z:
        if f"theta{j}" in z:
            out.append(np.array(z[f"theta{j}"]))
        else:
            spec = z[f"theta_spec{j}"]
            seed, k, n, base_seed = (int(v) for v in spec[:4])
            scale, base_scale = float(spec[4]), float(spec[5])
            th = seeded_theta(seed, k, n, scale, None if base_seed < 0 else base_seed, base_scale)
            assert digest(th) == str(z[f"theta_sha{j}"]), "seeded theta does not reproduce"
            out.append(th)
        j += 1
    return out


def points(z) -> np.ndarray:
    """Coordinates of a golden case: its regular grid or the stored pixel subset."""
    m = int(z["grid_m"])
    c = -1.0 + (np.arange(1, 2 * m + 1) - 0.5) / m
    side = c.size
    if "point_index" in z:
        idx = np.asarray(z["point_index"], dtype=np.int64)
    else:
        idx = np.arange(side * side)
    return np.column_stack([c[idx // side], c[idx % side]])
