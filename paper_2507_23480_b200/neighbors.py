"""SPEC.md module ``neighbors`` on the B200.

Outputs are (idx int64[q, k] (-1 padded), dist float64[q, k] (NaN padded),
cnt int64[q]) ordered by (d2, index) with the strict ``d2 < r^2`` test.
The redundancy-free versions read the exclusion lists built for sampling
and perform no distance evaluations.
"""

from __future__ import annotations

import numpy as np
import torch

from . import core, engine


def _np(t):
    return t.cpu().numpy()


def ball_query_naive(cloud, centroids, R, max_neighbors):
    pc = cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)
    if not R > 0:
        raise ValueError("R must be positive")
    xyz4 = engine.as_xyz4(pc.coords)
    c = torch.as_tensor(np.asarray(centroids, np.int64), device=xyz4.device).reshape(1, -1)
    idx, dist, cnt = engine.ball_query_naive(xyz4, c, R, int(max_neighbors))
    core.add_pair_evals(pc.n * c.shape[1])
    return _np(idx[0]).astype(np.int64), _np(dist[0]), _np(cnt[0]).astype(np.int64)


def rf_ball_query(fp: "engine.FastPoint", R, max_neighbors, centroids=None, cloud_index=0):
    """From a sampled FastPoint pipeline (``mdps(..., return_pipeline=True)``)."""
    cent = None
    if centroids is not None:
        cent = torch.as_tensor(np.asarray(centroids, np.int64), device=fp.device).reshape(1, -1)
        if fp.B != 1:
            raise ValueError("explicit centroids need a single-cloud pipeline")
    idx, dist, cnt = fp.group_rf(R, int(max_neighbors), centroids=cent)
    b = cloud_index
    return _np(idx[b]).astype(np.int64), _np(dist[b]), _np(cnt[b]).astype(np.int64)


def knn_naive(cloud, queries, pool, k):
    pc = cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)
    pool = np.asarray(pool, np.int64)
    if pool.shape[0] == 0:
        raise ValueError("empty pool")
    xyz4 = engine.as_xyz4(pc.coords)
    q = torch.as_tensor(np.asarray(queries, np.int64), device=xyz4.device).reshape(1, -1)
    pl = torch.as_tensor(pool, device=xyz4.device).reshape(1, -1)
    idx, dist, cnt = engine.knn_naive(xyz4, pl, int(k), queries=q)
    core.add_pair_evals(q.shape[1] * pool.shape[0])
    return _np(idx[0]).astype(np.int64), _np(dist[0]), _np(cnt[0]).astype(np.int64)


def rf_knn(fp: "engine.FastPoint", k, queries=None, cloud_index=0):
    """Queries (default: every point) into the sampled set of ``fp``; returns
    (idx, dist, cnt, fallback_count)."""
    q = None
    if queries is not None:
        q = torch.as_tensor(np.asarray(queries, np.int64), device=fp.device).reshape(1, -1)
    idx, dist, cnt, fb = fp.knn_rf(int(k), queries=q)
    b = cloud_index
    return _np(idx[b]).astype(np.int64), _np(dist[b]), _np(cnt[b]).astype(np.int64), int(fb[b].item())
