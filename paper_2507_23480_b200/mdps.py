"""SPEC.md module ``mdps`` -- FastPoint / Minimum Distance Prediction
Sampling on the B200.

``mdps(cloud, n, ...)`` composes extract_prefix -> estimator ->
segment_thresholds -> build_exclusion_lists -> sample_with_predicted_distance
-> early_termination exactly as SPEC.md:425-433 (call stack B of SURVEY.md 3);
all stages run as sm_100a kernels (engine.FastPoint).  The per-stage
functions below expose the same stages to callers that compose them
themselves; they return device-backed results.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import core, engine
from .curve import radius_sq, sampler_boundaries


@dataclass
class ExclusionLists:
    """Host view of one cloud's exclusion CSR (rows sorted by (d2, index))."""

    indptr: np.ndarray
    nbr: np.ndarray
    d2: np.ndarray
    counts: np.ndarray           # [L, N], level rows: nseg segments then extra radii
    r2_levels: np.ndarray
    seg_level_rows: np.ndarray
    extra_radii: tuple
    extra_level_rows: tuple

    def level_of_radius(self, r):
        for rr, row in zip(self.extra_radii, self.extra_level_rows):
            if rr == float(r):
                return row
        raise ValueError(f"radius {r} not baked into exclusion lists; available {list(self.extra_radii)}")


def _cloud(cloud):
    return cloud if isinstance(cloud, core.PointCloud) else core.PointCloud(cloud)


def mdps(cloud, n: int, p: float = 0.1, nseg: int = 6, estimator: str = "power", exponent=None, curve=None,
         seed_index: int = 0, rng=None, extra_radii=(), pick_lowest: bool = False, return_pipeline: bool = False,
         model=None):
    """FastPoint sampling of one cloud.  ``estimator``: 'power' (needs
    ``exponent``, see curve.fit_power_exponent), 'mlp' (needs ``model``, a
    curve.MlpModel or the path of an SPEC.md:357 weight file) or 'curve' (a
    full estimated curve, e.g. the oracle estimator's true FPS curve).
    ``rng`` is a core.Rng (advanced in place) or an integer seed."""
    from . import curve as _curve

    if estimator == "mlp" and model is not None and not isinstance(model, _curve.MlpModel):
        model = _curve.MlpModel.load(model)
    pc = _cloud(cloud)
    r = rng if isinstance(rng, core.Rng) else core.Rng(0 if rng is None else int(rng))
    t0 = time.perf_counter()
    fp = engine.FastPoint(1, pc.n, n, p=p, nseg=nseg, estimator=estimator, exponent=exponent,
                          extra_radii=extra_radii, seed_index=seed_index, pick_lowest=pick_lowest, mlp=model)
    fp.set_points(torch.from_numpy(pc.coords.copy()).to(fp.device))
    fp.set_rng([r.state])
    if estimator == "curve":
        fp.set_curve(np.asarray(curve, np.float64).reshape(1, n))
    fp.sample()
    fp.check()
    idx = fp.out[0].cpu().numpy()
    reached = int(fp.reached.item())
    r.state = int(np.int64(fp.state.item()).view(np.uint64))
    evals = fp.pair_evals()[0]
    core.add_pair_evals(evals)
    stats = {"fps_prefix_iters": fp.k0, "early_term_iters": n - reached, "segments_entered": int(fp.entered.item()),
             "exhausted": bool(fp.exhausted.item()), "thresholds": fp.R[0].cpu().numpy(),
             "wall_time_s": time.perf_counter() - t0, "pair_evals": evals}
    res = core.SampleResult(idx, "mdps", stats)
    if return_pipeline:
        return res, fp
    return res


def build_exclusion_lists(cloud, radii, extra_radii=()):
    """SPEC.md:394-402 on the device; radii are the segment thresholds."""
    from . import _kernels

    pc = _cloud(cloud)
    seg_r2 = [radius_sq(r if r > 0 else 5e-324) for r in radii]
    ext_r2 = [radius_sq(float(r)) for r in extra_radii]
    levels = np.array(seg_r2 + ext_r2, np.float64)
    x, y, z = pc.columns_f64()
    indptr, nbr, d2, counts, evals = _kernels.build_csr(x, y, z, levels)
    core.add_pair_evals(evals + pc.n)
    nseg = len(seg_r2)
    return ExclusionLists(indptr, nbr, d2, counts, levels, np.arange(nseg), tuple(float(r) for r in extra_radii),
                          tuple(range(nseg, nseg + len(ext_r2))))


def sample_with_predicted_distance(n, prefix_idx, excl: ExclusionLists, rng, pick_lowest=False):
    """SPEC.md:404-413 -> (indices with -1 beyond reached, exhausted, reached)."""
    from . import _kernels

    r = rng if isinstance(rng, core.Rng) else core.Rng(int(rng))
    N = excl.indptr.shape[0] - 1
    nseg = len(excl.seg_level_rows)
    out, i, ex, en, st = _kernels.sample_predicted(excl.indptr, excl.nbr, excl.counts, excl.seg_level_rows,
                                                   sampler_boundaries(n, nseg), prefix_idx, n, N,
                                                   np.uint64(r.state), pick_lowest)
    r.state = int(st)
    return out, ex, i


def early_termination(cloud, n, partial_idx, reached, excl: ExclusionLists):
    """seed md from level-1 rows, finish with exact FPS."""
    from . import _kernels

    pc = _cloud(cloud)
    out = np.array(partial_idx, np.int64)
    if reached >= n:
        return core.SampleResult(out[:n], "mdps", {"early_term_iters": 0})
    N = pc.n
    taken = np.zeros(N, np.uint8)
    taken[out[:reached]] = 1
    md = np.full(N, np.inf)
    lvl1 = np.ascontiguousarray(excl.counts[int(excl.seg_level_rows[0])])
    _kernels.earlyterm_scan(excl.indptr, excl.nbr, excl.d2, lvl1, taken, md, 0, N)
    x, y, z = pc.columns_f64()
    curve = np.full(n, np.inf)
    ev = _kernels.fps_loop(x, y, z, md, taken, out, curve, reached, n)
    core.add_pair_evals(ev)
    return core.SampleResult(out, "mdps", {"early_term_iters": n - reached})
