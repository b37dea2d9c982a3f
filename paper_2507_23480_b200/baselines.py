"""SPEC.md module ``baselines`` -- exact FPS on the B200 (K1).

``fps(cloud, n, seed_index)`` follows SPEC.md:124-132 (Algorithm 1 with the
lowest-index tie rule and the duplicate fallback of _kernels.py:65-70) on the
device.  The Table 2 comparison samplers of SPEC.md:144-172 (random, grid,
grid-to-count) are host utilities for API completeness:
they are not on the sampling hot path.
"""

from __future__ import annotations

import math
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


def random_sample(cloud, n: int, rng) -> "core.SampleResult":
    """n distinct indices uniformly without replacement,
    deterministic for a seeded core.Rng (partial Fisher-Yates from the top:
    slot N-1-t swaps with a draw below N-t, as Rng.shuffle)."""
    pc = cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)
    N = pc.n
    if not (1 <= n <= N):
        raise ValueError(f"n must be in [1, {N}], got {n}")
    r = rng if isinstance(rng, core.Rng) else core.Rng(int(rng))
    a = np.arange(N, dtype=np.int64)
    for t in range(n):
        i = N - 1 - t
        j = r.below(i + 1)
        a[i], a[j] = a[j], a[i]
    return core.SampleResult(a[N - n:][::-1].copy(), "random", {})


def grid_sample(cloud, voxel_size: float) -> "core.SampleResult":
    """voxels of edge voxel_size anchored at the bounding-box
    minimum; per occupied voxel the point nearest its voxel's barycenter
    (ties -> lowest index); ordered by voxel key (z-major integer key of the
    voxel coordinates).  float64 arithmetic on the float32 coordinates."""
    if not voxel_size > 0:
        raise ValueError(f"voxel size must be positive, got {voxel_size}")
    pc = cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)
    xyz = pc.coords.astype(np.float64)
    lo = xyz.min(axis=0)
    v = np.floor((xyz - lo) / float(voxel_size)).astype(np.int64)
    dims = v.max(axis=0) + 1
    key = (v[:, 2] * dims[1] + v[:, 1]) * dims[0] + v[:, 0]
    order = np.lexsort((np.arange(pc.n), key))
    ks = key[order]
    starts = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    ends = np.r_[starts[1:], ks.shape[0]]
    out = np.empty(starts.shape[0], np.int64)
    for g, (a, b) in enumerate(zip(starts, ends)):
        members = order[a:b]
        bc = xyz[members].sum(axis=0) / float(b - a)
        d = ((xyz[members] - bc) ** 2).sum(axis=1)
        out[g] = int(members[d == d.min()].min())
    return core.SampleResult(out, "grid", {"voxel_size": float(voxel_size), "voxels": int(out.shape[0])})


def grid_sample_to_count(cloud, target_n: int, tolerance_fraction: float = 0.05) -> "core.SampleResult":
    """bisect the voxel size over [diag/2^20, diag] (at most
    40 iterations) until the count is within tolerance; best-effort result."""
    pc = cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)
    if not (1 <= target_n <= pc.n):
        raise ValueError(f"target_n must be in [1, {pc.n}]")
    xyz = pc.coords.astype(np.float64)
    diag = float(np.linalg.norm(xyz.max(axis=0) - xyz.min(axis=0))) or 1.0
    lo_v, hi_v = diag / 2.0 ** 20, diag
    best, best_err = None, None
    lo_c, hi_c = target_n * (1 - tolerance_fraction), target_n * (1 + tolerance_fraction)
    for _ in range(40):
        mid = math.sqrt(lo_v * hi_v)
        res = grid_sample(pc, mid)
        c = len(res.indices)
        err = abs(c - target_n)
        if best is None or err < best_err:
            best, best_err = res, err
        if lo_c <= c <= hi_c:
            break
        if c > target_n:
            lo_v = mid
        else:
            hi_v = mid
    best.stats["achieved"] = len(best.indices)
    best.stats["target"] = int(target_n)
    return best
