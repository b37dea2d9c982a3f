"""CPU parity oracle for the FastPoint sampling path.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, by ``__graft_entry__.smoke()``
and by bench.py's ``cpu_baseline`` / ``--impl reference`` legs -- never by
the product package ``paper_2507_23480_b200``.

Two layers:

* ``CKernels`` -- ctypes binding of ``oracle/ps_oracle.c``, a C restatement
  of the reference numba kernels (``pkg/src/pointsample/_kernels.py``).  Its
  methods take and return numpy arrays with the same signatures and in-place
  semantics as the reference kernels, so the reference module itself can be
  swapped in (``tests/golden/make_golden.py`` does exactly that to produce
  the golden fixtures that pin this oracle).
* Module-level functions -- a restatement of the orchestration layer that the
  reference only specifies (SPEC.md modules ``baselines``, ``curve``,
  ``mdps``, ``neighbors``, ``quality``; absent from the reference code).  Each
  cites the SPEC lines it follows.  The ambiguities listed in SURVEY.md
  Appendix B are pinned here and mirrored by the CUDA path:

  - sampler boundaries are segment ends with the last one equal to n
    (SURVEY 0.4); radii look up d_s clamped to n-1;
  - r2 = max(R*R, 5e-324) with R <= 0 clamped to 5e-324;
  - estimate_power: a = sequential-sum mean of v_i * i**e over i in [1, k0),
    tail a / i**e, running min that starts at the last measured value;
    i**e comes from ``power_table`` (numpy float64 power);
  - all neighbor orderings use the key (d2, index).
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libps_oracle.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_f64 = ctypes.c_double

TINY = 5e-324  # smallest positive float64 (SPEC.md:448 clamp)


def build_oracle() -> str:
    """Compile libps_oracle.so with the committed Makefile."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    if not os.path.exists(_LIB_PATH):
        build_oracle()
    lib = ctypes.CDLL(_LIB_PATH)
    lib.ora_sm64_next.restype = ctypes.c_uint64
    lib.ora_sm64_next.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
    lib.ora_fps_loop.restype = _i64
    lib.ora_fps_loop.argtypes = [_f64p, _f64p, _f64p, _i64, _f64p, _u8p, _i64p, _f64p, _i64, _i64]
    lib.ora_fps_update_chunk.restype = None
    lib.ora_fps_update_chunk.argtypes = [_f64p, _f64p, _f64p, _f64, _f64, _f64, _f64p, _i64, _i64,
                                         ctypes.POINTER(_f64), ctypes.POINTER(_i64)]
    lib.ora_fps_loop_mt.restype = _i64
    lib.ora_fps_loop_mt.argtypes = [_f64p, _f64p, _f64p, _i64, _f64p, _u8p, _i64p, _f64p, _i64, _i64, ctypes.c_int32]
    lib.ora_excl_build_mt.restype = ctypes.c_void_p
    lib.ora_excl_build_mt.argtypes = [_f64p, _f64p, _f64p, _i64, _f64, ctypes.c_int32]
    lib.ora_first_untaken.restype = _i64
    lib.ora_first_untaken.argtypes = [_u8p, _i64]
    lib.ora_excl_build.restype = ctypes.c_void_p
    lib.ora_excl_build.argtypes = [_f64p, _f64p, _f64p, _i64, _f64]
    for nm in ("ora_csr_N", "ora_csr_E", "ora_csr_evals"):
        getattr(lib, nm).restype = _i64
        getattr(lib, nm).argtypes = [ctypes.c_void_p]
    lib.ora_csr_copy.restype = None
    lib.ora_csr_copy.argtypes = [ctypes.c_void_p, _i64p, _i64p, _f64p]
    lib.ora_csr_free.restype = None
    lib.ora_csr_free.argtypes = [ctypes.c_void_p]
    lib.ora_level_counts.restype = None
    lib.ora_level_counts.argtypes = [_i64p, _f64p, _i64, _f64p, _i64, _i64p]
    lib.ora_sample_predicted.restype = _i64
    lib.ora_sample_predicted.argtypes = [_i64p, _i64p, _i64p, _i64p, _i64p, _i64, _i64p, _i64, _i64,
                                         _i64, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int32,
                                         _i64p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_i64)]
    lib.ora_earlyterm_scan.restype = None
    lib.ora_earlyterm_scan.argtypes = [_i64p, _i64p, _f64p, _i64p, _u8p, _f64p, _i64, _i64]
    lib.ora_ball_query_naive.restype = None
    lib.ora_ball_query_naive.argtypes = [_f64p, _f64p, _f64p, _i64, _i64p, _i64, _f64, _i64,
                                         _i64p, _f64p, _i64p]
    lib.ora_knn_naive.restype = None
    lib.ora_knn_naive.argtypes = [_f64p, _f64p, _f64p, _i64p, _i64, _i64p, _i64, _i64,
                                  _i64p, _f64p, _i64p]
    lib.ora_min_spacing_d2.restype = None
    lib.ora_min_spacing_d2.argtypes = [_f64p, _f64p, _f64p, _i64p, _i64, _f64p]
    return lib


_LIB = None

# worker threads of the reference's multi-worker form (core.workers,
# core.py:71-101): FPS slices merged by the chunk rule and the
# excl_collect task split.  1 = the serial kernels.  Results are identical.
THREADS = max(1, int(os.environ.get("PS_ORACLE_THREADS", "1")))


def set_threads(t: int) -> int:
    global THREADS
    old, THREADS = THREADS, max(1, int(t))
    return old


def lib():
    global _LIB
    if _LIB is None:
        _LIB = _load()
    return _LIB


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _cf(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# kernel layer (signatures of _kernels.py)


class CKernels:
    """The C restatement behind the reference kernel signatures."""

    name = "c-oracle"

    @staticmethod
    def fps_loop(x, y, z, md, taken, out_idx, curve, k_start, n_total):
        # _kernels.py:35-74
        if THREADS > 1:
            return int(lib().ora_fps_loop_mt(x, y, z, x.shape[0], md, taken, out_idx, curve,
                                             int(k_start), int(n_total), THREADS))
        return int(lib().ora_fps_loop(x, y, z, x.shape[0], md, taken, out_idx, curve,
                                      int(k_start), int(n_total)))

    @staticmethod
    def fps_update_chunk(x, y, z, px, py, pz, md, lo, hi):
        # _kernels.py:77-92
        b = _f64()
        j = _i64()
        lib().ora_fps_update_chunk(x, y, z, px, py, pz, md, int(lo), int(hi),
                                   ctypes.byref(b), ctypes.byref(j))
        return b.value, j.value

    @staticmethod
    def first_untaken(taken):
        # _kernels.py:95-100
        return int(lib().ora_first_untaken(taken, taken.shape[0]))

    @staticmethod
    def excl_build(x, y, z, r2max):
        """excl_collect over all tasks + csr_fill + csr_sort_rows
        (_kernels.py:111-219).  Returns (indptr, nbr, d2, evals)."""
        L = lib()
        h = L.ora_excl_build_mt(x, y, z, x.shape[0], float(r2max), THREADS)
        try:
            N = L.ora_csr_N(h)
            E = L.ora_csr_E(h)
            indptr = np.empty(N + 1, np.int64)
            nbr = np.empty(E, np.int64)
            d2 = np.empty(E, np.float64)
            L.ora_csr_copy(h, indptr, nbr, d2)
            evals = L.ora_csr_evals(h)
        finally:
            L.ora_csr_free(h)
        return indptr, nbr, d2, int(evals)

    @staticmethod
    def csr_level_counts(indptr, d2, r2_levels):
        # _kernels.py:222-234
        N = indptr.shape[0] - 1
        r2 = _cf(r2_levels)
        out = np.empty((r2.shape[0], N), np.int64)
        lib().ora_level_counts(_c64(indptr), _cf(d2), N, r2, r2.shape[0], out)
        return out

    @staticmethod
    def sample_predicted(indptr, nbr_idx, level_counts, seg_level_rows, boundaries,
                         prefix_idx, n_total, N, state, pick_lowest):
        # _kernels.py:251-353
        out = np.empty(int(n_total), np.int64)
        st = ctypes.c_uint64(int(state))
        ex = ctypes.c_int32(0)
        en = _i64(0)
        nseg = int(np.asarray(boundaries).shape[0])
        reached = lib().ora_sample_predicted(
            _c64(indptr), _c64(nbr_idx), _c64(level_counts), _c64(seg_level_rows),
            _c64(boundaries), nseg, _c64(prefix_idx), int(np.asarray(prefix_idx).shape[0]),
            int(n_total), int(N), ctypes.byref(st), 1 if pick_lowest else 0, out,
            ctypes.byref(ex), ctypes.byref(en))
        return out, int(reached), bool(ex.value), int(en.value), np.uint64(st.value)

    @staticmethod
    def earlyterm_scan(indptr, nbr_idx, d2, lvl1_counts, taken, md, lo, hi):
        # _kernels.py:356-367
        lib().ora_earlyterm_scan(_c64(indptr), _c64(nbr_idx), _cf(d2), _c64(lvl1_counts),
                                 taken, md, int(lo), int(hi))


DEFAULT_KERNELS = CKernels


# ---------------------------------------------------------------------------
# core (core.py restated where the path needs it)

_GOLDEN = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def sm64_stream(seed: int, count: int):
    """splitmix64 outputs (core.py:131-133)."""
    s = ctypes.c_uint64(seed & _M64)
    return [int(lib().ora_sm64_next(ctypes.byref(s))) for _ in range(count)]


def columns_f64(coords):
    """core.py:200-207: exact f32 -> f64 widening into three columns."""
    c = np.ascontiguousarray(coords, dtype=np.float32)
    return (np.ascontiguousarray(c[:, 0], np.float64), np.ascontiguousarray(c[:, 1], np.float64),
            np.ascontiguousarray(c[:, 2], np.float64))


# ---------------------------------------------------------------------------
# baselines.fps


def fps(coords, n, seed_index=0, kernels=DEFAULT_KERNELS, k_stop=None):
    """Exact FPS.  Returns (indices i64[n], curve f64[n], md, taken, evals).

    ``k_stop`` < n runs only iterations 1..k_stop-1 (the prefix); the
    returned arrays then hold the first k_stop entries."""
    x, y, z = columns_f64(coords)
    N = x.shape[0]
    if not (1 <= n <= N):
        raise ValueError(f"n must be in [1, {N}], got {n}")
    if not (0 <= seed_index < N):
        raise ValueError(f"seed_index out of range: {seed_index}")
    stop = n if k_stop is None else int(k_stop)
    md = np.full(N, np.inf)
    taken = np.zeros(N, np.uint8)
    out = np.full(n, -1, np.int64)
    curve = np.full(n, np.inf)
    out[0] = seed_index
    taken[seed_index] = 1
    evals = kernels.fps_loop(x, y, z, md, taken, out, curve, 1, stop)
    return out[:stop], curve[:stop], md, taken, int(evals)


def fps_bruteforce_oracle(coords, n, seed_index=0):
    """recompute every min-distance from scratch each step."""
    x, y, z = columns_f64(coords)
    N = x.shape[0]
    if N > 5000:
        raise ValueError("fps_bruteforce_oracle is guarded at N <= 5000")
    out = [int(seed_index)]
    taken = np.zeros(N, bool)
    taken[seed_index] = True
    for _ in range(1, n):
        best, arg = -1.0, -1
        for j in range(N):
            m = math.inf
            for s in out:
                dx = x[j] - x[s]
                dy = y[j] - y[s]
                dz = z[j] - z[s]
                d = dx * dx + dy * dy + dz * dz
                if d < m:
                    m = d
            if m > best:
                best, arg = m, j
        if best <= 0.0 or taken[arg]:
            arg = int(np.flatnonzero(~taken)[0])
        out.append(arg)
        taken[arg] = True
    return np.array(out, np.int64)


# ---------------------------------------------------------------------------
# curve


def prefix_len(n: int, p: float) -> int:
    """k0 = ceil(p * n)."""
    return int(math.ceil(p * n))


def power_table(n: int, exponent: float) -> np.ndarray:
    """i**e for i in [0, n) as float64 (numpy power); entry 0 unused."""
    return np.power(np.arange(n, dtype=np.float64), np.float64(exponent))


def fit_power_exponent(curves) -> float:
    """least squares of log v on log i over i >= 1."""
    xs, ys = [], []
    for c in curves:
        c = np.asarray(c, np.float64)
        i = np.arange(1, c.shape[0])
        v = c[1:]
        if np.any(v <= 0):
            raise ValueError("curve has non-positive values")
        xs.append(np.log(i))
        ys.append(np.log(v))
    X = np.concatenate(xs)
    Y = np.concatenate(ys)
    slope = np.polyfit(X, Y, 1)[0]
    return float(-slope)


def estimate_power(prefix_curve, n: int, exponent: float) -> np.ndarray:
    """SPEC.md:258-266 with SURVEY Appendix B.3 pinned (see module doc)."""
    pre = np.asarray(prefix_curve, np.float64)
    k0 = pre.shape[0]
    if k0 < 2:
        raise ValueError("prefix needs >= 2 values")
    pw = power_table(max(n, k0), exponent)
    s = 0.0
    for i in range(1, k0):
        s = s + float(pre[i]) * float(pw[i])
    a = s / float(k0 - 1)
    est = np.empty(n, np.float64)
    m = min(n, k0)
    est[:m] = pre[:m]
    run = float(pre[k0 - 1])
    for i in range(k0, n):
        t = a / float(pw[i])
        if t < run:
            run = t
        est[i] = run
    return est


def segment_thresholds(curve, nseg: int):
    """SPEC.md:318-326.  Returns (d i64[nseg], R f64[nseg])."""
    if nseg < 1:
        raise ValueError("nseg must be >= 1")
    c = np.asarray(curve, np.float64)
    n = c.shape[0]
    d = np.array([min(n * s // nseg, n - 1) for s in range(1, nseg + 1)], np.int64)
    R = np.empty(nseg, np.float64)
    run = math.inf
    for s in range(nseg):
        v = float(c[d[s]])
        if v < run:
            run = v
        R[s] = run
    return d, R


def sampler_boundaries(n: int, nseg: int) -> np.ndarray:
    """Segment ends: floor(n*s/nseg) for s < nseg, then n."""
    return np.array([n * s // nseg for s in range(1, nseg)] + [n], np.int64)


def clamp_radius(R: float) -> float:
    return R if R > 0 else TINY


def radius_sq(R: float) -> float:
    r2 = R * R
    return r2 if r2 > TINY else TINY


# ---------------------------------------------------------------------------
# mdps


@dataclass
class ExclusionLists:
    indptr: np.ndarray
    nbr: np.ndarray
    d2: np.ndarray
    counts: np.ndarray          # [L, N]
    r2_levels: np.ndarray       # ascending, unique
    seg_level_rows: np.ndarray  # nseg -> level row
    extra_radii: tuple = ()
    extra_level_rows: tuple = ()
    evals: int = 0

    def level_of_radius(self, r: float) -> int:
        for rr, row in zip(self.extra_radii, self.extra_level_rows):
            if rr == r:
                return row
        raise ValueError(f"radius {r} not baked into exclusion lists; available {list(self.extra_radii)}")


def make_levels(R, extra_radii=()):
    """Sorted unique r2 levels; seg rows; extra rows."""
    seg_r2 = [radius_sq(clamp_radius(float(r))) for r in R]
    ext_r2 = []
    for r in extra_radii:
        if not r > 0:
            raise ValueError(f"extra radius must be positive, got {r}")
        ext_r2.append(radius_sq(float(r)))
    levels = np.array(sorted(set(seg_r2 + ext_r2)), np.float64)
    pos = {float(v): i for i, v in enumerate(levels)}
    seg_rows = np.array([pos[v] for v in seg_r2], np.int64)
    ext_rows = tuple(pos[v] for v in ext_r2)
    return levels, seg_rows, ext_rows


def build_exclusion_lists(coords, R, extra_radii=(), kernels=DEFAULT_KERNELS):
    x, y, z = columns_f64(coords)
    levels, seg_rows, ext_rows = make_levels(R, extra_radii)
    r2max = float(levels[-1])
    indptr, nbr, d2, evals = kernels.excl_build(x, y, z, r2max)
    counts = kernels.csr_level_counts(indptr, d2, levels)
    N = x.shape[0]
    return ExclusionLists(indptr, nbr, d2, counts, levels, seg_rows, tuple(float(r) for r in extra_radii),
                          ext_rows, evals + N)


def sample_with_predicted_distance(excl: ExclusionLists, n, prefix_idx, boundaries, rng_state,
                                   pick_lowest=False, kernels=DEFAULT_KERNELS):
    N = excl.indptr.shape[0] - 1
    return kernels.sample_predicted(excl.indptr, excl.nbr, excl.counts, excl.seg_level_rows,
                                    boundaries, np.asarray(prefix_idx, np.int64), n, N,
                                    np.uint64(rng_state), pick_lowest)


def early_termination(coords, n, out, reached, excl: ExclusionLists, kernels=DEFAULT_KERNELS):
    """SPEC.md:415-423.  Completes out[reached:n] in place; returns evals."""
    if reached >= n:
        return 0, None
    x, y, z = columns_f64(coords)
    N = x.shape[0]
    taken = np.zeros(N, np.uint8)
    taken[out[:reached]] = 1
    md = np.full(N, np.inf)
    lvl1 = np.ascontiguousarray(excl.counts[excl.seg_level_rows[0]])
    kernels.earlyterm_scan(excl.indptr, excl.nbr, excl.d2, lvl1, taken, md, 0, N)
    curve = np.full(n, np.inf)
    evals = kernels.fps_loop(x, y, z, md, taken, out, curve, reached, n)
    return int(evals), md


@dataclass
class MdpsResult:
    indices: np.ndarray
    est_curve: np.ndarray
    thresholds: np.ndarray
    d: np.ndarray
    reached: int
    exhausted: bool
    entered: int
    rng_state: int
    excl: ExclusionLists
    evals: int
    stats: dict = field(default_factory=dict)


def mdps(coords, n, p=0.1, nseg=6, estimator="power", exponent=None, curve=None,
         seed_index=0, rng_seed=0, extra_radii=(), pick_lowest=False, kernels=DEFAULT_KERNELS, mlp=None):
    """SPEC.md:425-433 composition (call stack B of SURVEY.md section 3)."""
    N = np.asarray(coords).shape[0]
    if not (1 <= n <= N):
        raise ValueError(f"n must be in [1, {N}]")
    k0 = prefix_len(n, p)
    if k0 < 2:
        raise ValueError("ceil(p*n) must be >= 2")
    k0 = min(k0, n)
    pre_idx, pre_curve, _, _, ev = fps(coords, n, seed_index, kernels, k_stop=k0)
    evals = ev
    if estimator == "power":
        if exponent is None:
            raise ValueError("power estimator needs an exponent")
        est = estimate_power(pre_curve, n, exponent)
    elif estimator == "curve":
        est = np.asarray(curve, np.float64).copy()
        est[:k0] = pre_curve
    elif estimator == "mlp":
        if mlp is None:
            raise ValueError("mlp estimator needs a model")
        est = estimate_mlp(pre_curve, n, mlp)
    else:
        raise ValueError(f"unknown estimator {estimator!r}")
    d, R = segment_thresholds(est, nseg)
    excl = build_exclusion_lists(coords, R, extra_radii, kernels)
    evals += excl.evals
    bnd = sampler_boundaries(n, nseg)
    out, reached, exhausted, entered, state = sample_with_predicted_distance(
        excl, n, pre_idx, bnd, rng_seed, pick_lowest, kernels)
    out = np.array(out, np.int64)
    ev_et, _ = early_termination(coords, n, out, reached, excl, kernels)
    evals += ev_et
    return MdpsResult(out, est, R, d, int(reached), bool(exhausted), int(entered), int(state), excl, evals,
                      {"fps_prefix_iters": k0, "early_term_iters": n - int(reached),
                       "segments_entered": int(entered)})


# ---------------------------------------------------------------------------
# neighbors


def ball_query_naive(coords, centroids, r, k):
    x, y, z = columns_f64(coords)
    c = _c64(centroids)
    n = c.shape[0]
    idx = np.empty((n, k), np.int64)
    dist = np.empty((n, k), np.float64)
    cnt = np.empty(n, np.int64)
    lib().ora_ball_query_naive(x, y, z, x.shape[0], c, n, radius_sq(float(r)), int(k), idx, dist, cnt)
    return idx, dist, cnt


def rf_ball_query(excl: ExclusionLists, r, centroids, k):
    row = excl.level_of_radius(float(r))
    c = _c64(centroids)
    n = c.shape[0]
    idx = np.full((n, k), -1, np.int64)
    dist = np.full((n, k), np.nan)
    cnt = np.empty(n, np.int64)
    for t, p in enumerate(c):
        m = min(int(excl.counts[row, p]), k)
        lo = excl.indptr[p]
        idx[t, :m] = excl.nbr[lo:lo + m]
        dist[t, :m] = np.sqrt(excl.d2[lo:lo + m])
        cnt[t] = m
    return idx, dist, cnt


def knn_naive(coords, queries, pool, k):
    x, y, z = columns_f64(coords)
    q = _c64(queries)
    pl = _c64(pool)
    if pl.shape[0] == 0:
        raise ValueError("empty pool")
    idx = np.empty((q.shape[0], k), np.int64)
    dist = np.empty((q.shape[0], k), np.float64)
    cnt = np.empty(q.shape[0], np.int64)
    lib().ora_knn_naive(x, y, z, q, q.shape[0], pl, pl.shape[0], int(k), idx, dist, cnt)
    return idx, dist, cnt


def rf_knn(coords, excl: ExclusionLists, sampled_mask, queries, k):
    """Level-1 row of the query intersected with the sampled set; brute-force
    fallback over the whole pool when fewer than k candidates remain."""
    mask = np.asarray(sampled_mask, bool)
    pool = np.flatnonzero(mask).astype(np.int64)
    if pool.shape[0] == 0:
        raise ValueError("empty pool")
    row1 = excl.seg_level_rows[0]
    q = _c64(queries)
    idx = np.full((q.shape[0], k), -1, np.int64)
    dist = np.full((q.shape[0], k), np.nan)
    cnt = np.empty(q.shape[0], np.int64)
    fallback = 0
    for t, p in enumerate(q):
        lo = excl.indptr[p]
        m = int(excl.counts[row1, p])
        ent = excl.nbr[lo:lo + m]
        sel = np.flatnonzero(mask[ent])
        if sel.shape[0] >= k:
            sel = sel[:k]
            idx[t] = ent[sel]
            dist[t] = np.sqrt(excl.d2[lo + sel])
            cnt[t] = k
        else:
            fallback += 1
            i2, d2_, c2 = knn_naive(coords, [p], pool, k)
            idx[t] = i2[0]
            dist[t] = d2_[0]
            cnt[t] = c2[0]
    return idx, dist, cnt, fallback


# ---------------------------------------------------------------------------
# quality


def min_spacing_d2(coords, samples):
    x, y, z = columns_f64(coords)
    s = _c64(samples)
    out = np.empty(s.shape[0], np.float64)
    lib().ora_min_spacing_d2(x, y, z, s, s.shape[0], out)
    return out


def avg_min_spacing(coords, samples):
    s = _c64(samples)
    if s.shape[0] < 2:
        raise ValueError("need >= 2 samples")
    return float(np.mean(np.sqrt(min_spacing_d2(coords, s))))


def quality_ratio(coords, candidate, baseline):
    b = avg_min_spacing(coords, baseline)
    if b == 0:
        raise ValueError("zero baseline spacing")
    return 100.0 * avg_min_spacing(coords, candidate) / b


# ---------------------------------------------------------------------------
# multi-stage set abstraction (config C2)


def sa_cascade(coords, strides=(2, 2, 2, 2), radii=None, k=32, first="fastpoint", p=0.1, nseg=6, exponent=None,
               rng_seed=0, kernels=DEFAULT_KERNELS):
    """Stage 0: FastPoint (first="fastpoint") or exact FPS on the cloud, then a
    ball query of radius radii[0] (rf from the exclusion lists, or naive);
    stage s > 0: exact FPS of the previous stage's samples (sample order) and
    a naive ball query of radius radii[s].  Returns per stage
    (indices into that stage's input, group idx, group counts)."""
    radii = tuple(radii) if radii is not None else tuple(0.15 * 1.5 ** s for s in range(len(strides)))
    pts = np.ascontiguousarray(coords, np.float32)
    stages = []
    for s, st in enumerate(strides):
        n = pts.shape[0] // st
        if s == 0 and first == "fastpoint":
            res = mdps(pts, n, p=p, nseg=nseg, estimator="power", exponent=exponent, rng_seed=rng_seed,
                       extra_radii=(radii[0],), kernels=kernels)
            idx = res.indices
            gi, _, gc = rf_ball_query(res.excl, radii[0], idx, k)
        else:
            idx = fps(pts, n, 0, kernels)[0]
            gi, _, gc = ball_query_naive(pts, idx, radii[s], k)
        stages.append((idx, gi, gc))
        pts = np.ascontiguousarray(pts[idx])
    return stages


# ---------------------------------------------------------------------------
# MLP curve estimator, restated independently of the
# product code.  Pinned where the SPEC is silent (SURVEY B):
#   resample: u = (t * (S-1)) / (T-1); i0 = floor(u); frac = u - i0;
#             out = v[i0] + frac * (v[i0+1] - v[i0]); t = T-1 -> v[S-1];
#             T == 1 -> v[0]
#   forward: every dot product summed in input order from 0.0, bias added
#            last, relu(a) = a if a > 0 else 0.0, no FMA
#   estimate: prefix positions 1..k0-1 -> 32 values / v[k0-1] -> forward ->
#             * v[k0-1] -> resampled to the n-k0 tail positions -> running
#             minimum from v[k0-1]


@dataclass
class OracleMlp:
    W1: np.ndarray  # [128, 32]
    b1: np.ndarray
    W2: np.ndarray  # [128, 128]
    b2: np.ndarray
    W3: np.ndarray  # [64, 128]
    b3: np.ndarray


def read_mlp(path) -> OracleMlp:
    """SPEC.md:357 text format: `MLP 32 128 128 64`, then per layer `W r c`
    + r*c floats (row-major) and `B c` + c floats."""
    tok = open(path).read().split()
    if tok[:5] != ["MLP", "32", "128", "128", "64"]:
        raise ValueError("not an MLP 32 128 128 64 file")
    pos = 5
    mats = []
    for _ in range(3):
        if tok[pos] != "W":
            raise ValueError("expected W header")
        r, c = int(tok[pos + 1]), int(tok[pos + 2])
        W = np.array([float(x) for x in tok[pos + 3:pos + 3 + r * c]], np.float64).reshape(r, c)
        pos += 3 + r * c
        if tok[pos] != "B" or int(tok[pos + 1]) != r:
            raise ValueError("expected B header")
        bv = np.array([float(x) for x in tok[pos + 2:pos + 2 + r]], np.float64)
        pos += 2 + r
        mats += [W, bv]
    return OracleMlp(*mats)


def resample_pinned(v, T: int) -> np.ndarray:
    v = [float(x) for x in v]
    S = len(v)
    if S < 2:
        raise ValueError("need >= 2 values")
    out = np.empty(T, np.float64)
    if T == 1:
        out[0] = v[0]
        return out
    for t in range(T):
        u = (float(t) * float(S - 1)) / float(T - 1)
        i0 = int(math.floor(u))
        if i0 >= S - 1:
            out[t] = v[S - 1]
            continue
        frac = u - float(i0)
        out[t] = v[i0] + frac * (v[i0 + 1] - v[i0])
    return out


def mlp_forward_seq(m: OracleMlp, x) -> np.ndarray:
    def layer(W, bv, inp, relu):
        out = np.empty(W.shape[0], np.float64)
        for j in range(W.shape[0]):
            acc = 0.0
            row = W[j]
            for i in range(W.shape[1]):
                acc = acc + float(row[i]) * float(inp[i])
            acc = acc + float(bv[j])
            out[j] = (acc if acc > 0.0 else 0.0) if relu else acc
        return out

    h1 = layer(m.W1, m.b1, x, True)
    h2 = layer(m.W2, m.b2, h1, True)
    return layer(m.W3, m.b3, h2, False)


def estimate_mlp(prefix_curve, n: int, m: OracleMlp) -> np.ndarray:
    v = np.asarray(prefix_curve, np.float64)
    k0 = v.shape[0]
    if k0 < 3:
        raise ValueError("the MLP estimator needs >= 2 finite prefix values (k0 >= 3)")
    scale = float(v[k0 - 1])
    if not scale > 0:
        raise ValueError("last measured prefix value must be > 0")
    x = resample_pinned(v[1:k0], 32)
    x = np.array([float(a) / scale for a in x])
    y = mlp_forward_seq(m, x)
    y = np.array([float(a) * scale for a in y])
    out = np.empty(n, np.float64)
    out[:k0] = v
    if n > k0:
        tail = resample_pinned(y, n - k0)
        run = scale
        for i in range(n - k0):
            if tail[i] < run:
                run = float(tail[i])
            out[k0 + i] = run
    return out
