"""SPEC.md module ``quality``: coverage metric on the B200.

avg_min_spacing = mean over samples of the distance to the nearest other
sample; the per-sample minima are exact float64 (K6), the mean is a float64
reduction (tolerance 1e-12 relative vs. a sequential sum, stated in tests).
"""

from __future__ import annotations

import numpy as np
import torch

from . import core, engine


def avg_min_spacing(cloud, sample) -> float:
    pc = cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)
    idx = np.asarray(getattr(sample, "indices", sample), np.int64)
    if idx.shape[0] < 2:
        raise ValueError("need >= 2 samples")
    xyz4 = engine.as_xyz4(pc.coords)
    s = torch.as_tensor(idx, device=xyz4.device).reshape(1, -1)
    d2 = engine.min_spacing_d2(xyz4, s)
    return float(torch.sqrt(d2).mean().item())


def avg_min_spacing_batch(xyz4, samples) -> torch.Tensor:
    """[B] float64 on device."""
    return torch.sqrt(engine.min_spacing_d2(xyz4, samples)).mean(dim=1)


def quality_ratio(cloud, candidate, baseline) -> float:
    b = avg_min_spacing(cloud, baseline)
    if b == 0:
        raise ValueError("zero baseline spacing")
    return 100.0 * avg_min_spacing(cloud, candidate) / b
