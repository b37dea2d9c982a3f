"""Batched device pipeline: exact FPS, FastPoint (MDPS) sampling and grouping
for B clouds of N points on one B200, stream-ordered through the C ABI.

This is the hot path.  PyTorch provides device memory, the stream and CUDA
graphs; every computation is one of the sm_100a kernels in csrc/.  The
launch sequence of ``FastPoint.sample`` mirrors call stack (B) of SURVEY.md
section 3:

  K1  ps_fps                      FPS prefix, k0 = ceil(p n) iterations
  K2  ps_thresholds               power-law estimate -> segment radii / levels
  K3a ps_excl_build               exclusion CSR + level counts (one pass)
  K3c ps_sample_predicted         bitmap sampler (greedy-MIS formulation)
  K3d ps_early_termination_prepare + K1 ps_fps_loop(k_start = reached)
  K4a ps_ball_query_rf            grouping from the cached distances

No host synchronisation happens inside ``sample``/``group``; the only host
reads are the capacity status (``check``) and the results the caller asks
for.  All buffers are allocated once, so the whole sequence can be captured
in a CUDA graph (``capture``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .curve import power_table, prefix_len, radius_sq, sampler_boundaries, threshold_positions


def _p(t):
    return 0 if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def as_xyz4(coords, device=None) -> torch.Tensor:
    """[B, N, 3] (or [N, 3]) float32 -> contiguous [B, N, 4] float32 on device."""
    t = torch.as_tensor(coords)
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3 or t.shape[-1] != 3:
        raise ValueError(f"expected (B, N, 3) coordinates, got {tuple(t.shape)}")
    if t.dtype != torch.float32:
        raise ValueError("coordinates must be float32 (PointCloud storage, core.py:183)")
    dev = torch.device(device) if device is not None else (t.device if t.is_cuda else torch.device("cuda"))
    out = torch.zeros(t.shape[0], t.shape[1], 4, dtype=torch.float32, device=dev)
    out[..., :3].copy_(t, non_blocking=True)
    return out


# ---------------------------------------------------------------------------
# exact FPS


class inflight:
    """Context: launches inside it pick their FPS cluster width for
    ``clouds`` clouds in flight across concurrent streams (ps_set_fps_inflight;
    None / 0 = latency mode).  Results are identical either way."""

    def __init__(self, clouds):
        self.clouds = int(clouds or 0)

    def __enter__(self):
        self.old = int(_lib.raw("ps_set_fps_inflight", self.clouds)) if self.clouds else None
        return self

    def __exit__(self, *exc):
        if self.old is not None:
            _lib.raw("ps_set_fps_inflight", self.old)


def fps(xyz4: torch.Tensor, n: int, seed_index: int = 0, k_stop: int | None = None, inflight_clouds=None):
    """Exact FPS on a batch.  Returns (idx int64[B,n],
    curve float64[B,n], md float64[B,N], taken uint8[B,N]).
    ``inflight_clouds``: throughput hint (see ``inflight``)."""
    B, N, _ = xyz4.shape
    if not (1 <= n <= N):
        raise ValueError(f"n must be in [1, {N}], got {n}")
    stop = n if k_stop is None else int(k_stop)
    dev = xyz4.device
    md = torch.empty(B, N, dtype=torch.float64, device=dev)
    taken = torch.empty(B, N, dtype=torch.uint8, device=dev)
    out = torch.full((B, n), -1, dtype=torch.int64, device=dev)
    curve = torch.full((B, n), math.inf, dtype=torch.float64, device=dev)
    with inflight(inflight_clouds):
        _lib.call("ps_fps", _p(xyz4), B, N, _p(md), _p(taken), _p(out), _p(curve), n, stop, int(seed_index), None,
                  _stream())
    return out, curve, md, taken


class SplitMailboxes:
    """Mailboxes of G ranks living on this device ("virtual ranks"):
    the point-split FPS protocol of ps_fps_split exercised on one GPU, each
    rank a thread-block cluster exchanging its shard record through the same
    sequence-tagged global-memory slots that peer GPUs use over NVLink."""

    def __init__(self, B: int, G: int, device=None):
        self.B, self.G = int(B), int(G)
        nbytes = int(_lib.raw("ps_fps_mailbox_bytes", self.B, self.G))
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.boxes = [torch.full((nbytes,), 0xFF, dtype=torch.uint8, device=dev) for _ in range(self.G)]
        self.ptrs = torch.tensor([b.data_ptr() for b in self.boxes], dtype=torch.int64, device=dev)
        self.seq = 0

    def next_seq(self, k_stop: int) -> int:
        """Sequence base for a launch of k_stop iterations (tags stay unique)."""
        if self.seq + k_stop + 1 >= 0xFFFFFFFF:
            for b in self.boxes:
                b.fill_(0xFF)
            self.seq = 0
        base = self.seq
        self.seq += int(k_stop) + 1
        return base


def fps_split(xyz4: torch.Tensor, n: int, G: int, seed_index: int = 0, k_stop: int | None = None,
              mailboxes: SplitMailboxes | None = None):
    """Exact FPS with every cloud split over G virtual ranks on this GPU
    (config C5's point split).  Bit-identical to ``fps`` for any G.  Returns
    (idx, curve, md, taken) like ``fps``."""
    B, N, _ = xyz4.shape
    if not (1 <= n <= N):
        raise ValueError(f"n must be in [1, {N}], got {n}")
    stop = n if k_stop is None else int(k_stop)
    dev = xyz4.device
    mb = mailboxes if mailboxes is not None else SplitMailboxes(B, G, dev)
    if mb.G != G or mb.B != B:
        raise ValueError("mailboxes were made for another (B, G)")
    md = torch.empty(B, N, dtype=torch.float64, device=dev)
    taken = torch.empty(B, N, dtype=torch.uint8, device=dev)
    out = torch.full((B, n), -1, dtype=torch.int64, device=dev)
    curve = torch.full((B, n), math.inf, dtype=torch.float64, device=dev)
    _lib.call("ps_fps_split", _p(xyz4), B, N, _p(md), _p(taken), _p(out), _p(curve), n, stop, int(seed_index),
              G, 0, G, _p(mb.ptrs), mb.next_seq(stop), 0, _stream())
    return out, curve, md, taken


def fps_loop(xyz4, md, taken, out_idx, curve, k_start, n_total, k_start_dev=None):
    B, N, _ = xyz4.shape
    _lib.call("ps_fps_loop", _p(xyz4), B, N, _p(md), _p(taken), _p(out_idx), _p(curve), out_idx.shape[1],
              int(k_start), _p(k_start_dev), int(n_total), _stream())


# ---------------------------------------------------------------------------
# exclusion lists


@dataclass
class DeviceCsr:
    indptr: torch.Tensor   # int64 [B, N+1]
    nbr: torch.Tensor      # int32 [B, cap]
    d2: torch.Tensor       # float64 [B, cap]
    counts: torch.Tensor   # int32 [B, L, N]
    levels: torch.Tensor   # float64 [B, L]
    status: torch.Tensor   # int32 [B]
    work: torch.Tensor     # uint8 workspace
    cap_entries: int
    cap_edges: int
    method: int = 1

    @property
    def L(self):
        return self.counts.shape[1]

    @staticmethod
    def allocate(B, N, L, cap_entries, cap_edges, device, method=1):
        """method 0 = brute-force triangle, 1 = uniform-grid candidates (both
        give the reference CSR: rows sorted by (d2, index)); 2 = grid with a
        fixed row stride cap_entries // N and level-bucketed rows (every
        level's entries form the row prefix; the hot-path layout)."""
        cap_entries = int(min(max(cap_entries, N), (1 << 31) - 1))
        cap_edges = int(max(cap_edges, 1)) if method == 0 else 1
        ws = int(_lib.raw("ps_excl_workspace_bytes", B, N, cap_edges, method))
        return DeviceCsr(
            indptr=torch.zeros(B, N + 1, dtype=torch.int64, device=device),
            # +16 entries of tail padding: row scans use aligned 16-byte loads
            nbr=torch.empty(B * cap_entries + 16, dtype=torch.int32, device=device)[:B * cap_entries].view(
                B, cap_entries),
            d2=torch.empty(B, cap_entries, dtype=torch.float64, device=device),
            counts=torch.empty(B, L, N, dtype=torch.int32, device=device),
            levels=torch.empty(B, L, dtype=torch.float64, device=device),
            status=torch.zeros(B, dtype=torch.int32, device=device),
            work=torch.empty(ws, dtype=torch.uint8, device=device),
            cap_entries=cap_entries, cap_edges=cap_edges, method=int(method))

    def build(self, xyz4):
        B, N, _ = xyz4.shape
        _lib.call("ps_excl_build", _p(xyz4), B, N, _p(self.levels), self.L, self.levels.shape[1], _p(self.indptr),
                  _p(self.nbr), _p(self.d2), _p(self.counts), self.cap_entries, _p(self.work), self.cap_edges,
                  _p(self.status), self.method, _stream())

    def evaluated_pairs(self) -> list[int]:
        """Pair distances the build evaluated per cloud (self pairs excluded)."""
        B, N = self.indptr.shape[0], self.indptr.shape[1] - 1
        if self.method == 0:
            return [N * (N - 1) // 2] * B
        off = int(_lib.raw("ps_excl_grid_evals_offset", B, N))
        cand = self.work[off:off + 8 * B].view(torch.int64).tolist()
        # the grid count pass visits ordered pairs including self: unordered = (c - N) / 2
        return [(int(c) - N) // 2 for c in cand]

    @property
    def stride(self) -> int:
        """Method 2: entries per strided row (rows beyond it spill, see
        ps_excl_row_stride); 0 for the sorted-CSR methods."""
        N = self.indptr.shape[1] - 1
        return int(_lib.raw("ps_excl_row_stride", N, self.cap_entries)) if self.method == 2 else 0

    def overflowed(self) -> bool:
        return bool(int(self.status.max().item()) != 0)

    def row(self, b, i, level=None):
        """Entries of row i (method 2: only the first counts[level] entries are
        defined; pass the widest level)."""
        lo, hi = (int(v) for v in self.indptr[b, i:i + 2].tolist())
        if level is not None:
            hi = lo + int(self.counts[b, level, i].item())
        return self.nbr[b, lo:hi], self.d2[b, lo:hi]


def default_capacity(N: int, n: int) -> tuple[int, int]:
    """CSR entries per cloud: rows average ~14 x stride at the first segment
    radius; start with a generous bound, grow on overflow.
    The method-2 row stride comes out near ``per_point`` and the extra ninth
    is the spill arena for longer rows (ps_excl_row_stride)."""
    stride = max(1, N // max(n, 1))
    per_point = min(N, max(96, 48 * stride))
    cap_entries = N * (-(-per_point * 9 // 8) + 4)
    return cap_entries, max(1, (cap_entries - N) // 2 + 1)


# ---------------------------------------------------------------------------
# FastPoint pipeline


class FastPoint:
    """FastPoint sampling (+ redundancy-free grouping) on a fixed-shape batch.

    Parameters mirror SPEC.md:425-433 ``mdps(cloud, n, {p, nseg, estimator,
    seed_index, rng})``; ``extra_radii`` are ball-query radii baked into the
    exclusion lists."""

    def __init__(self, B, N, n, *, p=0.1, nseg=6, estimator="power", exponent=None, extra_radii=(),
                 seed_index=0, pick_lowest=False, cap_entries=None, excl_method="grid", device="cuda", mlp=None,
                 inflight_clouds=None):
        if not (1 <= n <= N):
            raise ValueError(f"n must be in [1, {N}]")
        if nseg < 1 or nseg > 16:
            raise ValueError("nseg must be in [1, 16]")
        if estimator not in ("power", "curve", "mlp"):
            raise ValueError(f"unknown estimator {estimator!r}")
        if estimator == "mlp" and mlp is None:
            raise ValueError("mlp estimator needs a model (curve.MlpModel)")
        if estimator == "power" and exponent is None:
            raise ValueError("power estimator needs an exponent (fit_power_exponent)")
        self.B, self.N, self.n = int(B), int(N), int(n)
        self.p, self.nseg, self.estimator = float(p), int(nseg), estimator
        self.exponent = None if exponent is None else float(exponent)
        self.extra_radii = tuple(float(r) for r in extra_radii)
        for r in self.extra_radii:
            if not r > 0:
                raise ValueError(f"extra radius must be positive, got {r}")
        if len(self.extra_radii) > 8:
            raise ValueError("at most 8 extra radii")
        self.seed_index = int(seed_index)
        self.pick_lowest = bool(pick_lowest)
        # throughput hint for the FPS launches (prefix, early-termination tail):
        # clouds kept in flight by concurrent pipelines (ps_set_fps_inflight)
        self.inflight_clouds = int(inflight_clouds or 0)
        methods = {"bruteforce": 0, "grid-sorted": 1, "grid": 2}
        if excl_method not in methods:
            raise ValueError(f"excl_method must be one of {sorted(methods)}")
        self.excl_method = methods[excl_method]
        self.device = torch.device(device)
        self.k0 = min(prefix_len(self.n, self.p), self.n)
        if self.k0 < 2:
            raise ValueError("ceil(p*n) must be >= 2 (SPEC.md:240)")
        self.d = threshold_positions(self.n, self.nseg)
        self.boundaries = sampler_boundaries(self.n, self.nseg)
        self.seg_level_rows = np.arange(self.nseg, dtype=np.int32)
        self.extra_r2 = np.array([radius_sq(r) for r in self.extra_radii], np.float64)
        self.L = self.nseg + len(self.extra_radii)
        dev = self.device
        B, N = self.B, self.N
        self.xyz4 = torch.zeros(B, N, 4, dtype=torch.float32, device=dev)
        self.md = torch.empty(B, N, dtype=torch.float64, device=dev)
        self.taken = torch.empty(B, N, dtype=torch.uint8, device=dev)
        self.out = torch.full((B, n), -1, dtype=torch.int64, device=dev)
        self.curve = torch.full((B, n), math.inf, dtype=torch.float64, device=dev)
        self.R = torch.empty(B, self.nseg, dtype=torch.float64, device=dev)
        self.reached = torch.zeros(B, dtype=torch.int64, device=dev)
        self.exhausted = torch.zeros(B, dtype=torch.int32, device=dev)
        self.entered = torch.zeros(B, dtype=torch.int32, device=dev)
        self.state = torch.zeros(B, dtype=torch.int64, device=dev)  # uint64 bit pattern
        self.pow_tab = (torch.as_tensor(power_table(self.n, self.exponent), device=dev)
                        if estimator == "power" else None)
        self.given_curve = torch.zeros(B, n, dtype=torch.float64, device=dev) if estimator == "curve" else None
        self.mlp_w = (torch.as_tensor(mlp.packed(), dtype=torch.float64, device=dev)
                      if estimator == "mlp" else None)
        if estimator == "mlp" and self.k0 < 3:
            raise ValueError("the MLP estimator needs ceil(p*n) >= 3")
        ce, cg = (default_capacity(N, n) if cap_entries is None else (int(cap_entries), int(cap_entries) // 2 + 1))
        self.csr = DeviceCsr.allocate(B, N, self.L, ce, cg, dev, self.excl_method)
        ws = int(_lib.raw("ps_sampler_workspace_bytes", B, N, self.nseg))
        self.samp_ws = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev) if ws else None
        self._bnd_c = np.ascontiguousarray(self.boundaries, np.int64)
        self._rows_c = np.ascontiguousarray(self.seg_level_rows, np.int32)
        self._d_c = np.ascontiguousarray(self.d, np.int64)
        self.graph = None

    # -- inputs ---------------------------------------------------------------
    def set_points(self, coords):
        t = torch.as_tensor(coords)
        if t.dim() == 2:
            t = t.unsqueeze(0)
        if tuple(t.shape) != (self.B, self.N, 3) or t.dtype != torch.float32:
            raise ValueError(f"expected float32 ({self.B}, {self.N}, 3), got {t.dtype} {tuple(t.shape)}")
        self.xyz4[..., :3].copy_(t, non_blocking=True)

    def set_rng(self, seeds):
        """splitmix64 state per cloud (uint64); the sampler advances it in place."""
        s = np.asarray(seeds, dtype=np.uint64).reshape(-1)
        if s.shape[0] == 1:
            s = np.repeat(s, self.B)
        self.state.copy_(torch.from_numpy(s.view(np.int64).copy()), non_blocking=False)
        self._state0 = self.state.clone()

    def set_curve(self, curves):
        if self.given_curve is None:
            raise ValueError("estimator is not 'curve'")
        self.given_curve.copy_(torch.as_tensor(curves, dtype=torch.float64).reshape(self.B, self.n))

    # -- stages -----------------------------------------------------------------
    def _prefix(self):
        with inflight(self.inflight_clouds):
            _lib.call("ps_fps", _p(self.xyz4), self.B, self.N, _p(self.md), _p(self.taken), _p(self.out),
                      _p(self.curve), self.n, self.k0, self.seed_index, None, _stream())

    def _thresholds(self):
        extra = np.ascontiguousarray(self.extra_r2) if len(self.extra_r2) else np.zeros(1)
        if self.estimator == "mlp":
            _lib.call("ps_thresholds_mlp", _p(self.curve), self.n, self.B, self.k0, self.n, self.nseg,
                      self._d_c.ctypes.data, _p(self.mlp_w), extra.ctypes.data, len(self.extra_r2), _p(self.R),
                      _p(self.csr.levels), self.L, _stream())
            return
        mode = 0 if self.estimator == "power" else 1
        _lib.call("ps_thresholds", _p(self.curve), self.n, self.B, self.k0, self.n, self.nseg,
                  self._d_c.ctypes.data, mode, _p(self.pow_tab), _p(self.given_curve), self.n,
                  extra.ctypes.data, len(self.extra_r2), _p(self.R), _p(self.csr.levels), self.L, _stream())

    def _exclusion(self):
        self.csr.build(self.xyz4)

    def _sampler(self):
        c = self.csr
        _lib.call("ps_sample_predicted", _p(c.indptr), _p(c.nbr), c.cap_entries, _p(c.counts), self.L,
                  self._rows_c.ctypes.data, self._bnd_c.ctypes.data, self.nseg, _p(self.out), self.n, self.k0,
                  self.n, self.B, self.N, _p(self.state), 1 if self.pick_lowest else 0, _p(self.reached),
                  _p(self.exhausted), _p(self.entered), _p(self.samp_ws), _p(c.status), _stream())

    def _early_termination(self):
        c = self.csr
        lvl1 = c.counts[:, int(self.seg_level_rows[0]), :]
        _lib.call("ps_early_termination_prepare", _p(c.indptr), _p(c.nbr), _p(c.d2), c.cap_entries, _p(lvl1),
                  self.L * self.N, _p(self.taken), _p(self.md), _p(self.out), self.n, _p(self.reached), self.n,
                  self.B, self.N, _stream())
        with inflight(self.inflight_clouds):
            _lib.call("ps_fps_loop", _p(self.xyz4), self.B, self.N, _p(self.md), _p(self.taken), _p(self.out),
                      _p(self.curve), self.n, 1, _p(self.reached), self.n, _stream())

    def sample(self):
        """Launch the full sampling sequence (no host sync)."""
        if self.graph is not None:
            self.graph.replay()
            return
        self._prefix()
        self._thresholds()
        self._exclusion()
        self._sampler()
        self._early_termination()

    KERNELS_PER_SAMPLE = 1 + 1 + 6 + 1 + 2 + 1  # prefix, thresholds, exclusion (N > 4096), sampler, ET seed, ET FPS

    def capture(self):
        """Capture ``sample`` into a CUDA graph (buffers are static).

        A replay on new points whose exclusion rows outgrow the capacity
        stays safe: rows longer than the stride spill into the arena inside
        the same launch sequence (identical results), and only an exhausted
        arena leaves the error state (``csr.status`` set, sampled indices -1
        past the prefix, ``entered`` -1, rf groups with count -1) that
        ``check`` turns into a rebuild -- it re-runs and re-captures."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.sample()  # warm-up outside capture (sets kernel attributes)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.sample()
        self.graph = g
        return g

    def check(self, max_grow=8):
        """Host read of the exclusion-build status (one int per cloud).  On
        an exhausted capacity: grow the buffers, re-run ``sample`` from the
        RNG state of the last ``set_rng`` (and re-capture the CUDA graph if
        one was captured) until nothing overflows.  Returns True when a
        re-run happened; raises RuntimeError if the capacity cannot grow."""
        reran = False
        had_graph = self.graph is not None
        for _ in range(max_grow):
            if not self.csr.overflowed():
                break
            full = self.N * (self.N + 1) + 16 * self.N  # every pair, any stride rounding
            if self.csr.cap_entries >= min(full, (1 << 31) - 1):
                raise RuntimeError("exclusion lists overflow at the largest capacity")
            grow = min(2 * self.csr.cap_entries, full, (1 << 31) - 1)
            self.csr = DeviceCsr.allocate(self.B, self.N, self.L, grow, grow // 2 + 1, self.device,
                                          self.excl_method)
            self.graph = None
            if getattr(self, "_state0", None) is not None:
                self.state.copy_(self._state0)  # replay from the same RNG state
            self.sample()
            reran = True
        if self.csr.overflowed():
            raise RuntimeError("exclusion lists still overflow after growing the capacity")
        if reran and had_graph:
            if getattr(self, "_state0", None) is not None:
                self.state.copy_(self._state0)
            self.capture()
            if getattr(self, "_state0", None) is not None:
                self.state.copy_(self._state0)
            self.sample()
        return reran

    # -- grouping ---------------------------------------------------------------
    def level_of_radius(self, r: float) -> int:
        for e, rr in enumerate(self.extra_radii):
            if rr == float(r):
                return self.nseg + e
        raise ValueError(f"radius {r} not baked into the exclusion lists; available {list(self.extra_radii)}")

    def group_rf(self, radius, k, centroids=None, out=None):
        """rf_ball_query around the samples (default) -> (idx, dist, cnt)."""
        lvl = self.level_of_radius(radius)
        cent = self.out if centroids is None else centroids
        B, n = cent.shape
        if out is None:
            out = (torch.empty(B, n, k, dtype=torch.int32, device=self.device),
                   torch.empty(B, n, k, dtype=torch.float64, device=self.device),
                   torch.empty(B, n, dtype=torch.int32, device=self.device))
        c = self.csr
        _lib.call("ps_ball_query_rf", _p(c.indptr), _p(c.nbr), _p(c.d2), c.cap_entries, _p(c.counts), self.L, lvl,
                  _p(cent), cent.stride(0), B, self.N, n, int(k), _p(out[0]), _p(out[1]), _p(out[2]), _p(c.status),
                  _stream())
        return out

    def knn_rf(self, k, queries=None):
        """rf_knn from every point (default) into the sampled set."""
        B, N = self.B, self.N
        sampled = torch.zeros(B, N, dtype=torch.uint8, device=self.device)
        sampled.scatter_(1, self.out, 1)
        nq = N if queries is None else queries.shape[1]
        idx = torch.empty(B, nq, k, dtype=torch.int32, device=self.device)
        dist = torch.empty(B, nq, k, dtype=torch.float64, device=self.device)
        cnt = torch.empty(B, nq, dtype=torch.int32, device=self.device)
        fb = torch.zeros(B, dtype=torch.int32, device=self.device)
        c = self.csr
        lvl1 = c.counts[:, int(self.seg_level_rows[0]), :]
        _lib.call("ps_knn_rf", _p(self.xyz4), _p(c.indptr), _p(c.nbr), _p(c.d2), c.cap_entries, _p(lvl1),
                  self.L * N, _p(sampled), _p(queries), 0 if queries is None else queries.stride(0), nq,
                  _p(self.out), self.n, self.n, B, N, int(k), _p(idx), _p(dist), _p(cnt), _p(fb), _p(c.status),
                  _stream())
        return idx, dist, cnt, fb

    # -- accounting ---------------------------------------------------------------
    def pair_evals(self) -> list[int]:
        """Per-cloud pair-distance evaluations: prefix N(k0-1) + exclusion
        (brute force: N(N-1)/2, the SPEC.md:438 accounting; grid: the
        candidate pairs actually evaluated) + N self pairs + early
        termination N(n-i)."""
        reached = self.reached.tolist()
        N = self.N
        excl = self.csr.evaluated_pairs()
        return [N * (self.k0 - 1) + excl[b] + N + N * (self.n - int(r)) for b, r in enumerate(reached)]


def shard_ranges(N: int, G: int) -> list[tuple[int, int]]:
    """Original-index range [lo, hi) of every rank of a point split (the
    partition of ps_fps_split: ceil(N / G) points per rank)."""
    Ns = -(-N // G)
    return [(min(N, g * Ns), min(N, (g + 1) * Ns)) for g in range(G)]


class FastPointSplit(FastPoint):
    """FastPoint with every cloud point-split over G ranks (config C5's MDPS,
    SURVEY.md 8e), here all G ranks on this GPU ("virtual ranks"); the same
    per-rank calls make up pointsplit.PointSplitFastPoint over one process
    per GPU:

      prefix      point-split FPS (ps_fps_split, mailbox exchange), k0 samples
      thresholds  every rank (identical prefix -> identical radii)
      exclusion   row-sharded: rank g builds the rows of its points
                  (ps_excl_build_shard, own spill sub-arena, own status)
      sampler     one rank over all rows (the rows meet on it: here they
                  share one buffer; across GPUs they are gathered)
      early term  every rank seeds md of its points from its own rows
                  (ps_early_termination_shard), then the point-split FPS
                  tail (ps_fps_split_loop from the sampler's reached count)
      grouping    rank g answers the sampled centroids it owns (its rows);
                  the per-rank answers are disjoint and summed

    Results are identical to FastPoint (and the oracle) for any G."""

    def __init__(self, B, N, n, G, **kw):
        super().__init__(B, N, n, **kw)
        if self.excl_method != 2:
            raise ValueError("the row-sharded build uses the method-2 layout (excl_method='grid')")
        self.G = int(G)
        if not (1 <= self.G <= 32):
            raise ValueError("1 <= G <= 32 ranks")
        self.ranges = shard_ranges(self.N, self.G)
        self.mb = SplitMailboxes(self.B, self.G, self.device)
        ws = int(_lib.raw("ps_excl_workspace_bytes", self.B, self.N, 1, 2))
        self.shard_ws = [torch.empty(ws, dtype=torch.uint8, device=self.device) for _ in range(self.G)]
        self.shard_status = torch.zeros(self.G, self.B, dtype=torch.int32, device=self.device)

    def capture(self):
        raise RuntimeError("FastPointSplit tags its mailbox exchanges from the host (ps_fps_split); run it eagerly "
                           "-- ps_fps's internal split is the graph-capturable form")

    def spill_ranges(self):
        spill = self.csr.cap_entries - self.N * self.csr.stride
        per = (spill // self.G) & ~3
        return [(g * per, (g + 1) * per if g < self.G - 1 else spill) for g in range(self.G)]

    def _prefix(self):
        _lib.call("ps_fps_split", _p(self.xyz4), self.B, self.N, _p(self.md), _p(self.taken), _p(self.out),
                  _p(self.curve), self.n, self.k0, self.seed_index, self.G, 0, self.G, _p(self.mb.ptrs),
                  self.mb.next_seq(self.k0), 0, _stream())

    def _exclusion(self):
        c = self.csr
        sp = self.spill_ranges()
        for g, (lo, hi) in enumerate(self.ranges):
            if hi <= lo:
                continue
            _lib.call("ps_excl_build_shard", _p(self.xyz4), self.B, self.N, _p(c.levels), self.L, c.levels.shape[1],
                      lo, hi, sp[g][0], sp[g][1], _p(c.indptr), _p(c.nbr), _p(c.d2), _p(c.counts), c.cap_entries,
                      _p(self.shard_ws[g]), _p(self.shard_status[g]), _stream())
        torch.amax(self.shard_status, dim=0, out=c.status)  # a failed rank fails the cloud

    def _early_termination(self):
        c = self.csr
        lvl1 = c.counts[:, int(self.seg_level_rows[0]), :]
        for lo, hi in self.ranges:
            if hi <= lo:
                continue
            _lib.call("ps_early_termination_shard", _p(c.indptr), _p(c.nbr), _p(c.d2), c.cap_entries, _p(lvl1),
                      self.L * self.N, _p(self.taken), _p(self.md), _p(self.out), self.n, _p(self.reached), self.n,
                      self.B, self.N, lo, hi, _stream())
        _lib.call("ps_fps_split_loop", _p(self.xyz4), self.B, self.N, _p(self.md), _p(self.taken), _p(self.out),
                  _p(self.curve), self.n, 1, _p(self.reached), self.n, self.G, 0, self.G, _p(self.mb.ptrs),
                  self.mb.next_seq(self.n), 0, _stream())

    def group_rf(self, radius, k, centroids=None, out=None):
        """rf_ball_query, centroid-sharded: rank g answers the centroids in its
        point range (the other positions come back as count -1); the disjoint
        answers are summed (index + 1, count + 1, distance)."""
        cent = self.out if centroids is None else centroids
        B, n = cent.shape
        acc_i = torch.zeros(B, n, k, dtype=torch.int32, device=self.device)
        acc_d = torch.zeros(B, n, k, dtype=torch.float64, device=self.device)
        acc_c = torch.zeros(B, n, dtype=torch.int32, device=self.device)
        for lo, hi in self.ranges:
            if hi <= lo:
                continue
            mine = torch.where((cent >= lo) & (cent < hi), cent, torch.full_like(cent, -1))
            gi, gd, gc = FastPoint.group_rf(self, radius, k, centroids=mine)
            own = gc >= 0
            acc_i += torch.where(own[..., None], gi + 1, 0)
            acc_d += torch.where(own[..., None], gd, 0.0)
            acc_c += torch.where(own, gc + 1, 0)
        res = (acc_i - 1, acc_d, acc_c - 1)
        if out is not None:
            for o, r in zip(out, res):
                o.copy_(r)
            return out
        return res


def ball_query_naive(xyz4, centroids, radius, k):
    B, N, _ = xyz4.shape
    n = centroids.shape[1]
    idx = torch.empty(B, n, k, dtype=torch.int32, device=xyz4.device)
    dist = torch.empty(B, n, k, dtype=torch.float64, device=xyz4.device)
    cnt = torch.empty(B, n, dtype=torch.int32, device=xyz4.device)
    _lib.call("ps_ball_query_naive", _p(xyz4), _p(centroids), centroids.stride(0), B, N, n, radius_sq(float(radius)),
              int(k), _p(idx), _p(dist), _p(cnt), _stream())
    return idx, dist, cnt


def knn_naive(xyz4, pool, k, queries=None):
    B, N, _ = xyz4.shape
    nq = N if queries is None else queries.shape[1]
    idx = torch.empty(B, nq, k, dtype=torch.int32, device=xyz4.device)
    dist = torch.empty(B, nq, k, dtype=torch.float64, device=xyz4.device)
    cnt = torch.empty(B, nq, dtype=torch.int32, device=xyz4.device)
    _lib.call("ps_knn_naive", _p(xyz4), _p(queries), 0 if queries is None else queries.stride(0), nq, _p(pool),
              pool.stride(0), pool.shape[1], B, N, int(k), _p(idx), _p(dist), _p(cnt), _stream())
    return idx, dist, cnt


def min_spacing_d2(xyz4, samples):
    B, N, _ = xyz4.shape
    n = samples.shape[1]
    out = torch.empty(B, n, dtype=torch.float64, device=xyz4.device)
    _lib.call("ps_min_spacing", _p(xyz4), _p(samples), samples.stride(0), n, B, N, _p(out), _stream())
    return out


# ---------------------------------------------------------------------------
# multi-stage set abstraction (config C2)


def gather_xyz4(xyz4: torch.Tensor, idx: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """[B, N, 4] points at idx [B, n] (sample order) -> [B, n, 4]."""
    B, N, _ = xyz4.shape
    n = idx.shape[1]
    if out is None:
        out = torch.empty(B, n, 4, dtype=torch.float32, device=xyz4.device)
    _lib.call("ps_gather_xyz4", _p(xyz4), _p(idx), idx.stride(0), B, N, n, _p(out), _stream())
    return out


class SACascade:
    """PointNet++ / PointNeXt set-abstraction sampling cascade on a batch
    (config C2: B clouds of N points, stages of stride ``strides``, ball query
    radius ``radii[s]`` with k neighbours per stage).

    Stage 0 samples the input clouds with FastPoint and groups from the cached
    distances (the paper applies FastPoint to the first layer);
    every later stage runs exact FPS on the previous stage's samples in sample
    order, then a naive ball query.  ``first="fps"`` gives the all-exact
    cascade the paper compares against.  Buffers are static, so ``capture``
    records the whole cascade in one CUDA graph."""

    def __init__(self, B, N, strides=(2, 2, 2, 2), radii=None, k=32, *, first="fastpoint", exponent=None, p=0.1,
                 nseg=6, device="cuda"):
        if first not in ("fastpoint", "fps"):
            raise ValueError("first must be 'fastpoint' or 'fps'")
        radii = tuple(radii) if radii is not None else tuple(0.15 * 1.5 ** s for s in range(len(strides)))
        if len(radii) != len(strides):
            raise ValueError("one radius per stage")
        self.B, self.N, self.k, self.first = int(B), int(N), int(k), first
        self.strides, self.radii = tuple(int(s) for s in strides), tuple(float(r) for r in radii)
        dev = torch.device(device)
        self.device = dev
        self.sizes = [self.N]
        for st in self.strides:
            self.sizes.append(self.sizes[-1] // st)
        if self.sizes[-1] < 1:
            raise ValueError("cascade samples fewer than one point")
        self.xyz = [torch.zeros(B, m, 4, dtype=torch.float32, device=dev) for m in self.sizes]
        self.idx, self.groups, self.fps_bufs = [], [], []
        for s, st in enumerate(self.strides):
            n_in, n = self.sizes[s], self.sizes[s + 1]
            self.groups.append((torch.empty(B, n, k, dtype=torch.int32, device=dev),
                                torch.empty(B, n, k, dtype=torch.float64, device=dev),
                                torch.empty(B, n, dtype=torch.int32, device=dev)))
            if s == 0 and first == "fastpoint":
                self.fp = FastPoint(B, n_in, n, p=p, nseg=nseg, estimator="power", exponent=exponent,
                                    extra_radii=(self.radii[0],), device=dev)
                self.idx.append(self.fp.out)
                self.fps_bufs.append(None)
            else:
                self.fps_bufs.append((torch.empty(B, n_in, dtype=torch.float64, device=dev),
                                      torch.empty(B, n_in, dtype=torch.uint8, device=dev),
                                      torch.full((B, n), math.inf, dtype=torch.float64, device=dev)))
                self.idx.append(torch.full((B, n), -1, dtype=torch.int64, device=dev))
        self.graph = None

    def set_points(self, coords):
        x = as_xyz4(coords, self.device)
        if tuple(x.shape[:2]) != (self.B, self.N):
            raise ValueError(f"expected ({self.B}, {self.N}, 3) coordinates")
        self.xyz[0].copy_(x)
        if self.first == "fastpoint":
            self.fp.set_points(coords)

    def set_rng(self, seeds):
        if self.first == "fastpoint":
            self.fp.set_rng(seeds)

    def run(self):
        """All stages, stream-ordered, no host sync."""
        if self.graph is not None:
            self.graph.replay()
            return
        B, k = self.B, self.k
        for s in range(len(self.strides)):
            n_in, n = self.sizes[s], self.sizes[s + 1]
            x = self.xyz[s]
            gi, gd, gc = self.groups[s]
            if s == 0 and self.first == "fastpoint":
                self.fp.sample()
                self.fp.group_rf(self.radii[0], k, out=self.groups[0])
            else:
                md, taken, curve = self.fps_bufs[s]
                out = self.idx[s]
                _lib.call("ps_fps", _p(x), B, n_in, _p(md), _p(taken), _p(out), _p(curve), n, n, 0, None, _stream())
                _lib.call("ps_ball_query_naive", _p(x), _p(out), out.stride(0), B, n_in, n,
                          radius_sq(self.radii[s]), k, _p(gi), _p(gd), _p(gc), _stream())
            gather_xyz4(x, self.idx[s], out=self.xyz[s + 1])

    def capture(self):
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.run()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run()
        self.graph = g
        return g
