"""SPEC.md module ``baselines`` -- exact FPS on the B200 (K1).

``fps(cloud, n, seed_index)`` follows SPEC.md:124-132 (Algorithm 1 with the
lowest-index tie rule and the duplicate fallback of _kernels.py:65-70); the
random / grid samplers of SPEC.md:144-172 are out of scope.
"""

from __future__ import annotations

import time

import numpy as np

from . import core, engine


def fps(cloud, n: int, seed_index: int = 0):
    """-> (SampleResult, curve float64[n]) with curve[0] = +inf."""
    pc = cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)
    N = pc.n
    if not (1 <= n <= N):
        raise ValueError(f"n must be in [1, {N}], got {n}")
    if not (0 <= seed_index < N):
        raise ValueError(f"seed_index out of range: {seed_index}")
    t0 = time.perf_counter()
    xyz4 = engine.as_xyz4(pc.coords)
    idx, curve, _, _ = engine.fps(xyz4, n, seed_index)
    out = idx[0].cpu().numpy()
    cv = curve[0].cpu().numpy()
    core.add_pair_evals(N * (n - 1))
    return core.SampleResult(out, "fps", {"wall_time_s": time.perf_counter() - t0}), cv


def fps_batch(coords, n: int, seed_index: int = 0):
    """Batched exact FPS on device tensors [B, N, 3] -> (idx [B,n], curve [B,n])."""
    xyz4 = engine.as_xyz4(coords)
    idx, curve, _, _ = engine.fps(xyz4, n, seed_index)
    return idx, curve
