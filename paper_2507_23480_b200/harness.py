"""Synthetic point-cloud families (``harness.generate_cloud``).

Only the generators are in scope: they produce the
input shapes of the BASELINE.json configs.  Every cloud is float32 (N, 3)
and deterministic given ``seed``.

Families:
  uniform-box        i.i.d. uniform in the unit cube (C1, C5)
  unit-sphere        uniform on the unit sphere surface (C2, ModelNet-like)
  gaussian-clusters  k Gaussian blobs with uniform centres
  room-surfaces      6 faces of a W x D x H metre box plus two interior
                     planes (a partition wall and a table top) -- the
                     S3DIS/ScanNet indoor proxy (C3, C4)
  lidar-rings        concentric rings with equal points per ring, so areal
                     density falls as 1/radius (outdoor proxy)
  lattice            regular grid with spacing 0.1 plus exact duplicates
                     (tie-heavy stress cloud for the bit-exact checks)
"""

from __future__ import annotations

import numpy as np

FAMILIES = ("uniform-box", "unit-sphere", "gaussian-clusters", "room-surfaces",
            "lidar-rings", "lattice")


def _gen(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed) & ((1 << 64) - 1)))


def _room(g: np.random.Generator, N: int, W: float, D: float, H: float) -> np.ndarray:
    # (origin, u-axis, v-axis) rectangles; area-weighted sampling
    planes = [
        ((0, 0, 0), (W, 0, 0), (0, D, 0)),      # floor
        ((0, 0, H), (W, 0, 0), (0, D, 0)),      # ceiling
        ((0, 0, 0), (W, 0, 0), (0, 0, H)),      # wall y=0
        ((0, D, 0), (W, 0, 0), (0, 0, H)),      # wall y=D
        ((0, 0, 0), (0, D, 0), (0, 0, H)),      # wall x=0
        ((W, 0, 0), (0, D, 0), (0, 0, H)),      # wall x=W
        ((0.55 * W, 0, 0), (0, 0.6 * D, 0), (0, 0, H)),          # partition
        ((0.2 * W, 0.3 * D, 0.75), (0.25 * W, 0, 0), (0, 0.3 * D, 0)),  # table
    ]
    o = np.array([p[0] for p in planes], np.float64)
    u = np.array([p[1] for p in planes], np.float64)
    v = np.array([p[2] for p in planes], np.float64)
    area = np.linalg.norm(np.cross(u, v), axis=1)
    which = g.choice(len(planes), size=N, p=area / area.sum())
    a = g.random(N)[:, None]
    b = g.random(N)[:, None]
    pts = o[which] + a * u[which] + b * v[which]
    pts += g.normal(0.0, 0.005, size=pts.shape)  # scanner noise
    return pts


def generate_cloud(family: str, N: int, seed: int = 0, **params) -> np.ndarray:
    if N < 1:
        raise ValueError("N must be >= 1")
    g = _gen(seed)
    if family == "uniform-box":
        pts = g.random((N, 3))
    elif family == "unit-sphere":
        v = g.normal(size=(N, 3))
        pts = v / np.linalg.norm(v, axis=1, keepdims=True)
    elif family == "gaussian-clusters":
        k = int(params.get("k", 8))
        sigma = float(params.get("sigma", 0.05))
        centers = g.random((k, 3))
        pts = centers[g.integers(0, k, N)] + g.normal(0, sigma, (N, 3))
    elif family == "room-surfaces":
        pts = _room(g, N, float(params.get("W", 6.0)), float(params.get("D", 5.0)),
                    float(params.get("H", 3.0)))
    elif family == "lidar-rings":
        rings = int(params.get("rings", 32))
        r = 2.0 + 1.5 * np.arange(rings)
        ring = g.integers(0, rings, N)
        th = g.random(N) * 2 * np.pi
        rad = r[ring] + g.normal(0, 0.02, N)
        pts = np.stack([rad * np.cos(th), rad * np.sin(th), -1.7 + 0.02 * g.normal(size=N)], 1)
    elif family == "lattice":
        side = int(np.ceil(N ** (1.0 / 3.0)))
        ix = np.stack(np.meshgrid(np.arange(side), np.arange(side), np.arange(side),
                                  indexing="ij"), -1).reshape(-1, 3)
        base = ix[:N] * 0.1
        ndup = int(params.get("dups", N // 16))
        if ndup:
            src = g.integers(0, N, ndup)
            dst = g.choice(N, ndup, replace=False)
            base[dst] = base[src]
        pts = base
    else:
        raise ValueError(f"unknown family {family!r}; expected one of {FAMILIES}")
    return np.ascontiguousarray(pts, dtype=np.float32)
