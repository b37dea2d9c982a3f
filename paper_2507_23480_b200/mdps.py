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


def _est_curve(fp, n):
    """The estimated MinDistCurve the radii came from: the
    measured prefix from the device, the tail from the same estimator on
    the host (bit-identical to K2's arithmetic; R_s = est[d_s])."""
    from . import curve as _curve

    pre = fp.curve[0, :fp.k0].cpu().numpy()
    if fp.estimator == "power":
        return _curve.estimate_power(pre, n, fp.exponent)
    if fp.estimator == "mlp":
        return _curve.estimate_mlp(pre, n, fp._mlp_model)
    est = fp.given_curve[0].cpu().numpy().copy()
    est[:fp.k0] = pre
    return est


def mdps(cloud, n: int, p: float = 0.1, nseg: int = 6, estimator: str = "power", exponent=None, curve=None,
         seed_index: int = 0, rng=None, extra_radii=(), pick_lowest: bool = False, return_pipeline: bool = False,
         model=None):
    """FastPoint sampling of one cloud -> (SampleResult,
    estimated MinDistCurve float64[n]).  ``estimator``: 'power' (needs
    ``exponent``, see curve.fit_power_exponent), 'mlp' (needs ``model``, a
    curve.MlpModel or the path of an SPEC.md:357 weight file) or 'curve' (a
    full estimated curve, e.g. the oracle estimator's true FPS curve).
    ``rng`` is a core.Rng (advanced in place) or an integer seed.

    ``stats`` carries the Appendix B.2 latency categories measured with
    device events on the launching stream: ``time_curve_estimation_s``
    (prefix FPS + estimator), ``time_segmentation_s`` (thresholds +
    exclusion lists), ``time_sampling_s`` (bitmap sampler),
    ``time_early_termination_s`` (seeding + FPS tail), plus
    ``wall_time_s`` for the whole call.  ``return_pipeline=True`` appends
    the engine.FastPoint that ran (its device buffers)."""
    from . import curve as _curve

    if estimator == "mlp" and model is not None and not isinstance(model, _curve.MlpModel):
        model = _curve.MlpModel.load(model)
    pc = _cloud(cloud)
    r = rng if isinstance(rng, core.Rng) else core.Rng(0 if rng is None else int(rng))
    t0 = time.perf_counter()
    fp = engine.FastPoint(1, pc.n, n, p=p, nseg=nseg, estimator=estimator, exponent=exponent,
                          extra_radii=extra_radii, seed_index=seed_index, pick_lowest=pick_lowest, mlp=model)
    fp._mlp_model = model
    fp.set_points(torch.from_numpy(pc.coords.copy()).to(fp.device))
    fp.set_rng([r.state])
    if estimator == "curve":
        fp.set_curve(np.asarray(curve, np.float64).reshape(1, n))
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record(st)
    fp._prefix()
    fp._thresholds()  # estimator + segment radii (K2)
    ev[1].record(st)
    fp._exclusion()
    ev[2].record(st)
    fp._sampler()
    ev[3].record(st)
    fp._early_termination()
    ev[4].record(st)
    fp.check()  # capacity status; re-runs with larger buffers if exhausted
    ev[4].synchronize()
    idx = fp.out[0].cpu().numpy()
    reached = int(fp.reached.item())
    r.state = int(np.int64(fp.state.item()).view(np.uint64))
    evals = fp.pair_evals()[0]
    core.add_pair_evals(evals)
    est = _est_curve(fp, n)
    ms = [ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(4)]
    stats = {"fps_prefix_iters": fp.k0, "early_term_iters": n - reached, "segments_entered": int(fp.entered.item()),
             "exhausted": bool(fp.exhausted.item()), "thresholds": fp.R[0].cpu().numpy(),
             # Appendix B.2 categories: curve estimation | segmentation | sampling | early termination
             "time_curve_estimation_s": ms[0], "time_segmentation_s": ms[1], "time_sampling_s": ms[2],
             "time_early_termination_s": ms[3], "wall_time_s": time.perf_counter() - t0, "pair_evals": evals}
    res = core.SampleResult(idx, "mdps", stats)
    if return_pipeline:
        return res, est, fp
    return res, est


def build_exclusion_lists(cloud, thresholds, extra_radii=()):
    """SPEC.md:394-402 on the device.  ``thresholds`` is the
    SegmentedThresholds pair (d, R) of curve.segment_thresholds, or the radii
    R_1 >= ... >= R_nseg alone."""
    from . import _kernels

    pc = _cloud(cloud)
    radii = thresholds[1] if isinstance(thresholds, tuple) and len(thresholds) == 2 else thresholds
    radii = [float(v) for v in np.asarray(radii, np.float64).reshape(-1)]
    if not radii:
        raise ValueError("at least one segment radius")
    seg_r2 = [radius_sq(r if r > 0 else 5e-324) for r in radii]
    ext_r2 = [radius_sq(float(r)) for r in extra_radii]
    if not max(seg_r2 + ext_r2) > 0:
        raise ValueError("non-positive R_max (SPEC.md:399)")
    levels = np.array(seg_r2 + ext_r2, np.float64)
    x, y, z = pc.columns_f64()
    indptr, nbr, d2, counts, evals = _kernels.build_csr(x, y, z, levels)
    core.add_pair_evals(evals + pc.n)
    nseg = len(seg_r2)
    return ExclusionLists(indptr, nbr, d2, counts, levels, np.arange(nseg), tuple(float(r) for r in extra_radii),
                          tuple(range(nseg, nseg + len(ext_r2))))


def sample_with_predicted_distance(cloud, n, prefix_result, excl: ExclusionLists, thresholds=None, rng=0,
                                   pick_lowest=False):
    """SPEC.md:404-413 -> (partial SampleResult, seg_exhausted, last_index_reached).

    ``prefix_result`` is the FPS prefix (a SampleResult from
    curve.extract_prefix, or its index array); ``thresholds`` is accepted
    for the SPEC signature -- the radii are already the level rows of
    ``excl``.  The partial result holds the ``last_index_reached`` samples
    (prefix included)."""
    from . import _kernels

    del thresholds
    pc = _cloud(cloud)
    prefix_idx = np.asarray(getattr(prefix_result, "indices", prefix_result), np.int64)
    r = rng if isinstance(rng, core.Rng) else core.Rng(int(rng))
    N = excl.indptr.shape[0] - 1
    if N != pc.n:
        raise ValueError("exclusion lists were built for another cloud")
    nseg = len(excl.seg_level_rows)
    out, i, ex, en, st = _kernels.sample_predicted(excl.indptr, excl.nbr, excl.counts, excl.seg_level_rows,
                                                   sampler_boundaries(n, nseg), prefix_idx, n, N,
                                                   np.uint64(r.state), pick_lowest)
    r.state = int(st)
    part = core.SampleResult(np.asarray(out[:i], np.int64), "mdps",
                             {"segments_entered": int(en), "fps_prefix_iters": int(prefix_idx.shape[0])})
    return part, bool(ex), int(i)


def early_termination(cloud, n, partial, excl: ExclusionLists):
    """seed md from the level-1 rows of the samples so far,
    finish with exact FPS -> SampleResult (stats.early_term_iters = n - k)."""
    from . import _kernels

    pc = _cloud(cloud)
    part = np.asarray(getattr(partial, "indices", partial), np.int64)
    reached = int(part.shape[0])
    stats = dict(getattr(partial, "stats", None) or {})
    if reached >= n:
        stats["early_term_iters"] = 0
        return core.SampleResult(part[:n].copy(), "mdps", stats)
    N = pc.n
    out = np.full(n, -1, np.int64)
    out[:reached] = part
    taken = np.zeros(N, np.uint8)
    taken[part] = 1
    md = np.full(N, np.inf)
    lvl1 = np.ascontiguousarray(excl.counts[int(excl.seg_level_rows[0])])
    _kernels.earlyterm_scan(excl.indptr, excl.nbr, excl.d2, lvl1, taken, md, 0, N)
    x, y, z = pc.columns_f64()
    curve = np.full(n, np.inf)
    ev = _kernels.fps_loop(x, y, z, md, taken, out, curve, reached, n)
    core.add_pair_evals(ev)
    stats["early_term_iters"] = n - reached
    return core.SampleResult(out, "mdps", stats)
