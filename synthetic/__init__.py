"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the paper's method: it only draws random
numbers (volumes, labels, initial weights) so that both sides of a parity test
see identical inputs.  Recipe:

* volume  x[n,z,y,x] = E(z,y,x) * (0.5 + 0.2*g), g ~ N(0,1) drawn for the whole
  N x D x H x W array in C order with numpy PCG64 ``default_rng(seed)``, float32.
  E is a brain-like ellipsoid centred in the grid with radii
  (36/91, 44/109, 34/91) of (D, H, W) -- ~25% of voxels on the 91x109x91 MNI
  grid inferred from Table 1 (reading X1); background is 0.
* labels  y = rng.integers(0, 2, N) drawn after the volume (2 classes).
* weights (reading X21): conv Kaiming-normal fan-out (std = sqrt(2/(Cout*k^3))),
  BN gamma = 1, beta = 0, FC weight U(-1/sqrt(C), 1/sqrt(C)), all biases 0.
  Drawn tensor by tensor in the canonical parameter order supplied by the caller.
"""
from __future__ import annotations

import numpy as np

RADII_FRAC = (36.0 / 91.0, 44.0 / 109.0, 34.0 / 91.0)


def ellipsoid_mask(D: int, H: int, W: int) -> np.ndarray:
    c = ((D - 1) / 2.0, (H - 1) / 2.0, (W - 1) / 2.0)
    r = (RADII_FRAC[0] * D, RADII_FRAC[1] * H, RADII_FRAC[2] * W)
    z, y, x = np.meshgrid(np.arange(D), np.arange(H), np.arange(W), indexing="ij")
    q = ((z - c[0]) / r[0]) ** 2 + ((y - c[1]) / r[1]) ** 2 + ((x - c[2]) / r[2]) ** 2
    return (q <= 1.0)


def make_batch(N: int, D: int, H: int, W: int, seed: int = 1):
    """Return (x float32 [N,D,H,W], y int32 [N])."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((N, D, H, W))
    E = ellipsoid_mask(D, H, W).astype(np.float64)
    x = (E[None] * (0.5 + 0.2 * g)).astype(np.float32)
    y = rng.integers(0, 2, N).astype(np.int32)
    return x, y


def init_params(tensors, seed: int = 0):
    """tensors: list of (name, shape, kind) in canonical order; kind in
    {'conv', 'bn_gamma', 'bn_beta', 'fc_w', 'bias'}.  Returns list of float32 arrays."""
    rng = np.random.default_rng(seed)
    out = []
    for name, shape, kind in tensors:
        shape = tuple(int(s) for s in shape)
        if kind == "conv":
            fan_out = shape[0] * int(np.prod(shape[2:]))
            a = rng.standard_normal(shape) * np.sqrt(2.0 / fan_out)
        elif kind == "bn_gamma":
            a = np.ones(shape)
        elif kind in ("bn_beta", "bias"):
            a = np.zeros(shape)
        elif kind == "fc_w":
            bound = 1.0 / np.sqrt(shape[1])
            a = rng.uniform(-bound, bound, shape)
        else:
            raise ValueError(kind)
        out.append(a.astype(np.float32))
    return out


def perturb_params(tensors, arrays, seed: int = 2, scale: float = 0.1):
    """Perturb BN affine parameters and biases away from (1, 0, 0) so parity
    tests exercise the gamma/beta/bias paths (gamma=1, beta=0 hide bugs)."""
    rng = np.random.default_rng(seed)
    out = []
    for (name, shape, kind), a in zip(tensors, arrays):
        if kind in ("bn_gamma", "bn_beta", "bias"):
            a = (a + scale * rng.standard_normal(a.shape)).astype(np.float32)
        out.append(a)
    return out
