"""Drop-in replacement for the reference kernel layer
``pointsample._kernels`` (/root/reference/pkg/src/pointsample/_kernels.py).

Same 11 public names, positional signatures, numpy in/out and in-place
semantics; the work runs on the B200 through libps_b200.so.  Each call
stages its numpy arguments on the device, launches, and copies results back
into the caller's arrays, so a reference orchestrator can swap the import and
keep working.  Coordinates must be float32-representable float64 columns (what
``PointCloud.columns_f64`` produces, core.py:200-207) -- the device stores
clouds as float32 and widens exactly; anything else raises ValueError.

For batched, stream-ordered use (no per-call copies) see ``engine.py``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .engine import _p, _stream

_U64_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _dev():
    _lib.load(require_device=True)
    return torch.device("cuda")


def _xyz4(x, y, z):
    cols = [np.asarray(c, np.float64) for c in (x, y, z)]
    f = [c.astype(np.float32) for c in cols]
    for a, b in zip(cols, f):
        if not np.array_equal(a, b.astype(np.float64)):
            raise ValueError("coordinates must be float32-representable (PointCloud.columns_f64)")
    host = np.zeros((cols[0].shape[0], 4), np.float32)
    host[:, 0], host[:, 1], host[:, 2] = f
    return torch.from_numpy(host).to(_dev()).unsqueeze(0)


def _to(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(_dev())


def _back(dst: np.ndarray, src: torch.Tensor):
    dst[...] = src.cpu().numpy().reshape(dst.shape).astype(dst.dtype, copy=False)


def _sm64(state):
    """splitmix64 step (_kernels.py:20-28) -> (state, z)."""
    s = (int(state) + int(_U64_GOLDEN)) & ((1 << 64) - 1)
    from .core import mix64

    return np.uint64(s), np.uint64(mix64(s))


# ---- farthest point sampling (_kernels.py:35-100) -----------------------------


def fps_loop(x, y, z, md, taken, out_idx, curve, k_start, n_total):
    N = int(np.asarray(x).shape[0])
    n_total, k_start = int(n_total), int(k_start)
    if k_start >= n_total:
        return 0
    xyz4 = _xyz4(x, y, z)
    d_md, d_tk = _to(md, np.float64), _to(taken, np.uint8)
    d_out, d_cv = _to(out_idx, np.int64), _to(curve, np.float64)
    _lib.call("ps_fps_loop", _p(xyz4), 1, N, _p(d_md), _p(d_tk), _p(d_out), _p(d_cv), d_out.shape[0], k_start, None,
              n_total, _stream())
    _back(md, d_md)
    _back(taken, d_tk)
    _back(out_idx, d_out)
    _back(curve, d_cv)
    return N * (n_total - k_start)


def fps_update_chunk(x, y, z, px, py, pz, md, lo, hi):
    N = int(np.asarray(x).shape[0])
    xyz4 = _xyz4(x, y, z)
    d_md = _to(md, np.float64)
    best = torch.empty(1, dtype=torch.float64, device=xyz4.device)
    arg = torch.empty(1, dtype=torch.int64, device=xyz4.device)
    _lib.call("ps_fps_update_chunk", _p(xyz4), N, float(px), float(py), float(pz), _p(d_md), int(lo), int(hi),
              _p(best), _p(arg), _stream())
    _back(md, d_md)
    return float(best.item()), int(arg.item())


def first_untaken(taken):
    t = _to(taken, np.uint8)
    out = torch.empty(1, dtype=torch.int64, device=t.device)
    _lib.call("ps_first_untaken", _p(t), t.shape[0], _p(out), _stream())
    return int(out.item())


# ---- exclusion lists (_kernels.py:111-234) --------------------------------------


def build_csr(x, y, z, r2_levels, cap_entries=None, method=0):
    """Fused device build: (indptr int64[N+1], nbr int64[E], d2 float64[E],
    counts int64[L, N], evals).  The unit the reference orchestrator forms
    from excl_collect + csr_fill + csr_sort_rows + csr_level_counts.
    method 0 = brute-force triangle, 1 = grid (identical CSR)."""
    if method not in (0, 1):
        raise ValueError("build_csr returns the reference CSR layout: method 0 or 1")
    from .engine import DeviceCsr

    N = int(np.asarray(x).shape[0])
    lv = np.ascontiguousarray(r2_levels, np.float64).reshape(1, -1)
    L = lv.shape[1]
    xyz4 = _xyz4(x, y, z)
    cap = N * min(N, 128) if cap_entries is None else int(cap_entries)
    while True:
        csr = DeviceCsr.allocate(1, N, L, cap, cap // 2 + 1, xyz4.device, method)
        csr.levels.copy_(torch.from_numpy(lv))
        csr.build(xyz4)
        if not csr.overflowed():
            break
        cap = max(2 * cap, int(csr.indptr[0, -1].item()) + N)
    indptr = csr.indptr[0].cpu().numpy()
    E = int(indptr[-1])
    nbr = csr.nbr[0, :E].cpu().numpy().astype(np.int64)
    d2 = csr.d2[0, :E].cpu().numpy()
    counts = csr.counts[0].cpu().numpy().astype(np.int64)
    return indptr, nbr, d2, counts, N * (N - 1) // 2


def excl_collect(x, y, z, klo, khi, r2max, cap_hint):
    """Edges (i, j, d2), i < j, d2 < r2max, for the row-pair tasks [klo, khi)
    in the reference's emission order (task k: row k, then row N-1-k; j
    ascending).  The distances come from the device build; the host only
    reorders them."""
    N = int(np.asarray(x).shape[0])
    indptr, nbr, d2, _, _ = build_csr(x, y, z, [float(r2max)])
    ei, ej, ed = [], [], []
    evals = 0
    for k in range(int(klo), int(khi)):
        for i in ((k,) if N - 1 - k <= k else (k, N - 1 - k)):
            lo, hi = indptr[i], indptr[i + 1]
            js, ds = nbr[lo:hi], d2[lo:hi]
            sel = js > i
            order = np.argsort(js[sel], kind="stable")
            ei.append(np.full(order.shape[0], i, np.int32))
            ej.append(js[sel][order].astype(np.int32))
            ed.append(ds[sel][order])
            evals += N - 1 - i
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.empty(0, dt))
    return cat(ei, np.int32), cat(ej, np.int32), cat(ed, np.float64), evals


def csr_fill(ei, ej, ed, indptr, out_idx, out_d2):
    """Scatter the edges into both rows, self first, edges in emission order
    (_kernels.py:164-185) -- on the device (ps_csr_fill)."""
    indptr = np.asarray(indptr, np.int64)
    N = indptr.shape[0] - 1
    M = int(np.asarray(ei).shape[0])
    E = int(indptr[-1])
    dev = _dev()
    d_ei = _to(ei if M else np.zeros(1), np.int32)
    d_ej = _to(ej if M else np.zeros(1), np.int32)
    d_ed = _to(ed if M else np.zeros(1), np.float64)
    d_ip = _to(indptr, np.int64)
    d_idx = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
    d_d2 = torch.empty(max(E, 1), dtype=torch.float64, device=dev)
    wb = int(_lib.raw("ps_csr_fill_workspace_bytes", M, max(N, 1)))
    work = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    _lib.call("ps_csr_fill", _p(d_ei), _p(d_ej), _p(d_ed), M, _p(d_ip), N, _p(d_idx), _p(d_d2), _p(work), wb,
              _stream())
    out_idx[:E] = d_idx[:E].cpu().numpy()
    out_d2[:E] = d_d2[:E].cpu().numpy()


def csr_sort_rows(indptr, d2, idx):
    """Order every row by (d2, index) on the device, in place."""
    N = indptr.shape[0] - 1
    E = int(indptr[-1])
    if E == 0:
        return
    dev = _dev()
    d_ip = _to(indptr, np.int64).reshape(1, -1)
    d_nb = _to(idx, np.int32).reshape(1, -1)
    d_d2 = _to(d2, np.float64).reshape(1, -1)
    work = torch.empty(4 * N + 512, dtype=torch.uint8, device=dev)
    _lib.call("ps_csr_sort_rows", _p(d_ip), _p(d_nb), _p(d_d2), E, 1, N, _p(work), _stream())
    _back(d2, d_d2[0])
    _back(idx, d_nb[0])


def csr_level_counts(indptr, d2, r2_levels):
    N = indptr.shape[0] - 1
    lv = np.ascontiguousarray(r2_levels, np.float64).reshape(1, -1)
    L = lv.shape[1]
    d_ip = _to(indptr, np.int64).reshape(1, -1)
    d_d2 = _to(d2 if len(d2) else np.zeros(1), np.float64).reshape(1, -1)
    d_lv = _to(lv, np.float64)
    counts = torch.empty(1, L, N, dtype=torch.int32, device=d_ip.device)
    _lib.call("ps_level_counts", _p(d_ip), _p(d_d2), d_d2.shape[1], 1, N, _p(d_lv), L, L, _p(counts), _stream())
    return counts[0].cpu().numpy().astype(np.int64)


# ---- sampler (_kernels.py:241-367) -------------------------------------------------


def sample_predicted(indptr, nbr_idx, level_counts, seg_level_rows, boundaries, prefix_idx, n_total, N, state,
                     pick_lowest):
    N, n_total = int(N), int(n_total)
    dev = _dev()
    prefix = np.asarray(prefix_idx, np.int64)
    k0 = prefix.shape[0]
    E = int(indptr[-1])
    d_ip = _to(indptr, np.int64).reshape(1, -1)
    d_nb = _to(nbr_idx if E else np.zeros(1), np.int32).reshape(1, -1)
    lc = np.asarray(level_counts)
    L = lc.shape[0]
    d_ct = _to(lc, np.int32).reshape(1, L, N)
    out = torch.full((1, max(n_total, 1)), -1, dtype=torch.int64, device=dev)
    if k0:
        out[0, :k0] = torch.from_numpy(prefix)
    st = torch.tensor([np.int64(np.uint64(state).view(np.int64))], dtype=torch.int64, device=dev)
    reached = torch.zeros(1, dtype=torch.int64, device=dev)
    ex = torch.zeros(1, dtype=torch.int32, device=dev)
    en = torch.zeros(1, dtype=torch.int32, device=dev)
    nseg = int(np.asarray(boundaries).shape[0])
    ws = int(_lib.raw("ps_sampler_workspace_bytes", 1, N, nseg))
    work = torch.empty(max(ws, 1), dtype=torch.uint8, device=dev) if ws else None
    rows = np.ascontiguousarray(seg_level_rows, np.int32)
    bnd = np.ascontiguousarray(boundaries, np.int64)
    _lib.call("ps_sample_predicted", _p(d_ip), _p(d_nb), d_nb.shape[1], _p(d_ct), L, rows.ctypes.data,
              bnd.ctypes.data, nseg, _p(out), out.shape[1], k0, n_total, 1, N, _p(st), 1 if pick_lowest else 0,
              _p(reached), _p(ex), _p(en), _p(work), None, _stream())
    o = out[0, :n_total].cpu().numpy()
    state_out = np.uint64(np.int64(st.item()).view(np.uint64))
    return o, int(reached.item()), bool(ex.item()), int(en.item()), state_out


def earlyterm_scan(indptr, nbr_idx, d2, lvl1_counts, taken, md, lo, hi):
    N = indptr.shape[0] - 1
    lo, hi = int(lo), int(hi)
    if hi <= lo:
        return
    E = max(int(indptr[-1]), 1)
    d_ip = _to(indptr, np.int64).reshape(1, -1)
    d_nb = _to(nbr_idx if len(nbr_idx) else np.zeros(1), np.int32).reshape(1, -1)
    d_d2 = _to(d2 if len(d2) else np.zeros(1), np.float64).reshape(1, -1)
    d_c1 = _to(lvl1_counts, np.int32).reshape(1, -1)
    d_tk = _to(taken, np.uint8).reshape(1, -1)
    d_md = _to(md, np.float64).reshape(1, -1)
    _lib.call("ps_earlyterm_scan", _p(d_ip), _p(d_nb), _p(d_d2), E, _p(d_c1), N, _p(d_tk), _p(d_md), 1, N, lo, hi,
              _stream())
    _back(md, d_md[0])
