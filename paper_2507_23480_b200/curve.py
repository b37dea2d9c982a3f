"""Distance-curve helpers (SPEC.md module ``curve``).

The hot-path estimator (power law on the measured prefix, segment radii) runs
on the device in K2 (csrc/sampler.cu); these host functions hold the O(n)
pieces that are fixed before launch -- the prefix length, the i**e table, the
segment positions and sampler boundaries -- and the user-facing full-curve
operations of the SPEC (``estimate_power``, ``segment_thresholds``,
``fit_power_exponent``), which share the exact definitions K2 evaluates:

* k0 = ceil(p * n)
* a  = (sum_{i=1}^{k0-1} v_i * i**e, summed in order) / (k0 - 1)
* est[i] = v[i] for i < k0; min(est[i-1], a / i**e) for i >= k0
                                                      
* d_s = min(floor(n s / nseg), n - 1), R_s = running min of est[d_s]
                                                      
* sampler boundaries = (d_1 .. d_{nseg-1}, n)
* R <= 0 -> 5e-324 and r2 = max(R*R, 5e-324)
"""

from __future__ import annotations

import math

import numpy as np

TINY = 5e-324


def prefix_len(n: int, p: float) -> int:
    if not (0.0 < p < 1.0):
        raise ValueError(f"p must be in (0, 1), got {p}")
    return int(math.ceil(p * n))


def power_table(n: int, exponent: float) -> np.ndarray:
    """i**e as float64 for i in [0, n) (entry 0 unused)."""
    return np.power(np.arange(n, dtype=np.float64), np.float64(exponent))


def threshold_positions(n: int, nseg: int) -> np.ndarray:
    if nseg < 1:
        raise ValueError("nseg must be >= 1")
    if n < nseg + 1:
        raise ValueError(f"curve length n={n} must be >= nseg + 1 = {nseg + 1}")
    return np.array([min(n * s // nseg, n - 1) for s in range(1, nseg + 1)], np.int64)


def sampler_boundaries(n: int, nseg: int) -> np.ndarray:
    return np.array([n * s // nseg for s in range(1, nseg)] + [n], np.int64)


def clamp_radius(R: float) -> float:
    return R if R > 0 else TINY


def radius_sq(R: float) -> float:
    r2 = R * R
    return r2 if r2 > TINY else TINY


def fit_power_exponent(curves) -> float:
    """pooled least squares of log(v_i) on log(i), i >= 1."""
    xs, ys = [], []
    for c in curves:
        c = np.asarray(c, np.float64)
        if c.shape[0] < 9:
            raise ValueError("each curve needs >= 8 finite positions")
        v = c[1:]
        if np.any(~(v > 0)):
            raise ValueError("non-positive curve value")
        xs.append(np.log(np.arange(1, c.shape[0], dtype=np.float64)))
        ys.append(np.log(v))
    X = np.concatenate(xs)
    Y = np.concatenate(ys)
    X0 = X - X.mean()
    slope = float(np.dot(X0, Y - Y.mean()) / np.dot(X0, X0))
    return -slope


def estimate_power(prefix, n: int, exponent: float) -> np.ndarray:
    """Full estimated curve.  The sampling pipeline only
    needs est[d_s] and evaluates those on the device (K2); this host version
    returns the whole curve for users and reports."""
    v = np.asarray(prefix, np.float64)
    k0 = v.shape[0]
    if k0 < 2:
        raise ValueError("prefix needs >= 2 values")
    pw = power_table(max(n, k0), exponent)
    acc = 0.0
    for i in range(1, k0):
        acc = acc + float(v[i]) * float(pw[i])
    amp = acc / float(k0 - 1)
    out = np.empty(n, np.float64)
    out[:min(n, k0)] = v[:min(n, k0)]
    if n > k0:
        tail = amp / pw[k0:n]
        out[k0:n] = np.minimum.accumulate(np.concatenate([[v[k0 - 1]], tail]))[1:]
    return out


def segment_thresholds(curve, nseg: int):
    """SPEC.md:318-326 -> (d int64[nseg], R float64[nseg])."""
    c = np.asarray(curve, np.float64)
    d = threshold_positions(c.shape[0], nseg)
    R = np.minimum.accumulate(c[d])
    return d, R


def resample_curve(values, target_len: int) -> np.ndarray:
    """linear interpolation over normalised abscissa."""
    v = np.asarray(values, np.float64)
    if v.shape[0] < 2:
        raise ValueError("need >= 2 values")
    src = np.linspace(0.0, 1.0, v.shape[0])
    dst = np.linspace(0.0, 1.0, target_len)
    out = np.interp(dst, src, v)
    out[0], out[-1] = v[0], v[-1]
    return out


def estimator_mape(estimated, truth, p: float) -> float:
    """mean |est - truth| / truth over positions > ceil(p n)."""
    e = np.asarray(estimated, np.float64)
    t = np.asarray(truth, np.float64)
    k0 = prefix_len(t.shape[0], p)
    tail_t = t[k0 + 1:] if k0 + 1 < t.shape[0] else t[k0:]
    tail_e = e[k0 + 1:] if k0 + 1 < t.shape[0] else e[k0:]
    if np.any(tail_t == 0):
        raise ValueError("zero truth value in the tail")
    return float(np.mean(np.abs(tail_e - tail_t) / tail_t) * 100.0)
