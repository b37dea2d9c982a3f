"""Generate tests/golden/golden.npz from the REAL reference kernels.

Run in the build container only (it needs /root/reference and numba):

    python tests/golden/make_golden.py

The reference package is copied to a scratch directory first so numba's
``cache=True`` never writes into /root/reference.  The orchestration glue
(SPEC-level composition, absent from the reference code) is
``oracle.oracle``'s, run with the reference kernel module swapped in as the
kernel backend -- so the fixtures pin the C restatement
(oracle/ps_oracle.c) to the reference arithmetic, tie rules, RNG stream and
sampler behaviour.  Large outputs are stored as sha256 digests; small ones
verbatim.
"""

import hashlib
import math
import os
import shutil
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "ps_numba_cache"))
sys.dont_write_bytecode = True

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402


def load_reference():
    src = "/root/reference/pkg/src/pointsample"
    dst = os.path.join(tempfile.gettempdir(), "ps_ref_copy", "pointsample")
    if os.path.exists(dst):
        shutil.rmtree(dst)
    shutil.copytree(src, dst)
    sys.path.insert(0, os.path.dirname(dst))
    from pointsample import _kernels as K  # noqa: E402
    from pointsample import core  # noqa: E402
    return K, core


K, core = load_reference()


class RefKernels:
    """Reference numba kernels behind the oracle's kernel interface."""

    name = "reference"
    fps_loop = staticmethod(K.fps_loop)
    fps_update_chunk = staticmethod(K.fps_update_chunk)
    first_untaken = staticmethod(K.first_untaken)
    csr_level_counts = staticmethod(K.csr_level_counts)
    sample_predicted = staticmethod(K.sample_predicted)
    earlyterm_scan = staticmethod(K.earlyterm_scan)

    @staticmethod
    def excl_build(x, y, z, r2max):
        N = x.shape[0]
        T = (N + 1) // 2
        ei, ej, ed, evals = K.excl_collect(x, y, z, 0, T, r2max, 1024)
        deg = np.ones(N, np.int64)
        np.add.at(deg, ei, 1)
        np.add.at(deg, ej, 1)
        indptr = np.zeros(N + 1, np.int64)
        np.cumsum(deg, out=indptr[1:])
        nbr = np.empty(indptr[-1], np.int64)
        d2 = np.empty(indptr[-1], np.float64)
        K.csr_fill(ei, ej, ed, indptr, nbr, d2)
        K.csr_sort_rows(indptr, d2, nbr)
        return indptr, nbr, d2, int(evals)


def digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return np.frombuffer(h.digest(), np.uint8)


OUT = {}


def put(key, val):
    OUT[key] = np.asarray(val)


def clouds():
    cs = {
        "square4": np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.float32),
        "collinear3": np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], np.float32),
        "dups4": np.array([[0, 0, 0], [0, 0, 0], [1, 0, 0], [1, 0, 0]], np.float32),
        "uniform1000": generate_cloud("uniform-box", 1000, 11),
        "sphere1024": generate_cloud("unit-sphere", 1024, 12),
        "room2000": generate_cloud("room-surfaces", 2000, 13),
        "lattice1728": generate_cloud("lattice", 1728, 14),
        "clusters1500": generate_cloud("gaussian-clusters", 1500, 15),
        "lidar1200": generate_cloud("lidar-rings", 1200, 16),
        "uniform4096": generate_cloud("uniform-box", 4096, 17),
        "dupheavy600": np.repeat(generate_cloud("uniform-box", 200, 18), 3, axis=0),
    }
    return cs


def main():
    cs = clouds()
    for name, c in cs.items():
        put(f"cloud/{name}", c)

    # splitmix64 (core.py:111-133) and Rng.below
    r = core.Rng(0)
    put("rng/seed0", np.array([r.next_u64() for _ in range(8)], np.uint64))
    r = core.Rng(1)
    put("rng/seed1_below10", np.array([r.below(10) for _ in range(5)], np.int64))

    # FPS (full) on every cloud; tie-heavy ones included
    fps_cases = {"square4": 3, "collinear3": 3, "dups4": 4, "uniform1000": 300, "sphere1024": 512,
                 "room2000": 500, "lattice1728": 1728, "clusters1500": 375, "lidar1200": 300,
                 "uniform4096": 1024, "dupheavy600": 600}
    for name, n in fps_cases.items():
        for seed in (0, 7) if cs[name].shape[0] > 7 else (0,):
            idx, curve, md, taken, ev = O.fps(cs[name], n, seed, RefKernels)
            put(f"fps/{name}/n", n)
            put(f"fps/{name}/s{seed}/idx", idx)
            put(f"fps/{name}/s{seed}/curve", curve)
            put(f"fps/{name}/s{seed}/md", digest(md))
            put(f"fps/{name}/s{seed}/evals", ev)

    # exclusion lists + level counts
    excl_cases = [("collinear3", [1.5, 0.5], ()), ("dups4", [0.5], ()),
                  ("uniform1000", [0.12, 0.09, 0.07], (0.1,)), ("room2000", [0.4, 0.3, 0.25], (0.1,)),
                  ("lattice1728", [0.15, 0.1, 0.1000001], (0.2,)), ("clusters1500", [0.05], ()),
                  ("dupheavy600", [0.08, 0.0], ())]
    for t, (name, R, extra) in enumerate(excl_cases):
        e = O.build_exclusion_lists(cs[name], R, extra, RefKernels)
        k = f"excl/{t}"
        put(f"{k}/cloud", name)
        put(f"{k}/R", np.array(R, np.float64))
        put(f"{k}/extra", np.array(extra, np.float64))
        put(f"{k}/levels", e.r2_levels)
        put(f"{k}/seg_rows", e.seg_level_rows)
        put(f"{k}/E", e.indptr[-1])
        put(f"{k}/evals", e.evals)
        put(f"{k}/digest", digest(e.indptr, e.nbr, e.d2, e.counts))
        if cs[name].shape[0] <= 8:
            put(f"{k}/indptr", e.indptr)
            put(f"{k}/nbr", e.nbr)
            put(f"{k}/d2", e.d2)
            put(f"{k}/counts", e.counts)

    # full MDPS pipelines: power / true-curve estimators,
    # random and lowest-index picks, forced early termination
    mdps_cases = [
        ("uniform4096", 1024, dict(estimator="power", exponent=0.4, extra_radii=(0.05,), rng_seed=3)),
        ("uniform4096", 1024, dict(estimator="power", exponent=0.4, pick_lowest=True)),
        ("uniform1000", 250, dict(estimator="curve", rng_seed=5)),
        ("uniform1000", 250, dict(estimator="power", exponent=0.9, rng_seed=1)),  # overestimate -> ET
        ("room2000", 500, dict(estimator="power", exponent=0.45, rng_seed=9, extra_radii=(0.1,))),
        ("sphere1024", 512, dict(estimator="curve", nseg=3, rng_seed=2)),
        ("lattice1728", 432, dict(estimator="curve", rng_seed=4)),
        ("lattice1728", 432, dict(estimator="power", exponent=0.33, rng_seed=4, p=0.2)),
        ("dupheavy600", 600, dict(estimator="curve", rng_seed=6)),
        ("clusters1500", 375, dict(estimator="power", exponent=0.5, nseg=1, rng_seed=8)),
        ("lidar1200", 300, dict(estimator="curve", rng_seed=10, nseg=7)),
        ("collinear3", 3, dict(estimator="curve", nseg=1, p=0.5, rng_seed=5)),
    ]
    for t, (name, n, kw) in enumerate(mdps_cases):
        kw = dict(kw)
        if kw.get("estimator") == "curve":
            _, truth, _, _, _ = O.fps(cs[name], n, 0, RefKernels)
            kw["curve"] = truth
        res = O.mdps(cs[name], n, kernels=RefKernels, **kw)
        k = f"mdps/{t}"
        put(f"{k}/cloud", name)
        put(f"{k}/n", n)
        put(f"{k}/kw", repr({a: b for a, b in kw.items() if a != "curve"}))
        if "curve" in kw:
            put(f"{k}/curve", kw["curve"])
        put(f"{k}/idx", res.indices)
        put(f"{k}/reached", res.reached)
        put(f"{k}/exhausted", res.exhausted)
        put(f"{k}/entered", res.entered)
        put(f"{k}/state", np.uint64(res.rng_state))
        put(f"{k}/R", res.thresholds)
        put(f"{k}/evals", res.evals)
        put(f"{k}/excl_digest", digest(res.excl.indptr, res.excl.nbr, res.excl.d2, res.excl.counts))

    # earlyterm_scan (_kernels.py:356-367) on a partial sample
    e = O.build_exclusion_lists(cs["uniform1000"], [0.1], (), RefKernels)
    taken = np.zeros(1000, np.uint8)
    taken[::7] = 1
    md = np.full(1000, np.inf)
    K.earlyterm_scan(e.indptr, e.nbr, e.d2, e.counts[0], taken, md, 0, 1000)
    put("et/md", md)

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **OUT)
    print(f"wrote {path}: {len(OUT)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
