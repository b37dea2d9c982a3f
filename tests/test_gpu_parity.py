"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle
and the golden vectors of the real reference.  Indices, counts and RNG state
are compared bit-exactly; float64 distances / curves bit-exactly too (same
operation sequence, IEEE sqrt/div)."""

import os

import numpy as np
import pytest

from golden_util import cases, digest, mdps_kwargs
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2507_23480_b200 import _kernels as GK  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402


def gpu_fps(cloud, n, seed=0):
    xyz4 = engine.as_xyz4(cloud)
    idx, curve, md, taken = engine.fps(xyz4, n, seed)
    return idx[0].cpu().numpy(), curve[0].cpu().numpy(), md[0].cpu().numpy(), taken[0].cpu().numpy()


def gpu_mdps(cloud, n, **kw):
    kw = dict(kw)
    est = kw.pop("estimator", "power")
    curve = kw.pop("curve", None)
    rng_seed = kw.pop("rng_seed", 0)
    fp = engine.FastPoint(1, cloud.shape[0], n, estimator=est, **kw)
    fp.set_points(torch.from_numpy(np.ascontiguousarray(cloud)).cuda())
    fp.set_rng([rng_seed])
    if est == "curve":
        fp.set_curve(np.asarray(curve).reshape(1, n))
    fp.sample()
    fp.check()
    return fp


# ---- K1 exact FPS ---------------------------------------------------------------

def test_fps_golden(golden):
    for k in golden.files:
        if not (k.startswith("fps/") and k.endswith("/idx")):
            continue
        _, name, s, _ = k.split("/")
        seed = int(s[1:])
        c = golden[f"cloud/{name}"]
        n = int(golden[f"fps/{name}/n"])
        idx, curve, md, _ = gpu_fps(c, n, seed)
        np.testing.assert_array_equal(idx, golden[k], err_msg=k)
        np.testing.assert_array_equal(curve, golden[f"fps/{name}/s{seed}/curve"], err_msg=k)
        np.testing.assert_array_equal(digest(md), golden[f"fps/{name}/s{seed}/md"], err_msg=k)


@pytest.mark.parametrize("N,n,family", [
    (1, 1, "uniform-box"), (2, 2, "uniform-box"), (37, 37, "lattice"), (300, 75, "unit-sphere"),
    (1024, 512, "unit-sphere"), (4096, 1024, "uniform-box"), (5000, 1250, "lattice"),
    (24000, 6000, "room-surfaces"), (65536, 2048, "uniform-box"), (70001, 600, "gaussian-clusters"),
])
def test_fps_matches_oracle_across_cluster_shapes(N, n, family):
    c = generate_cloud(family, N, N + n)
    idx, curve, md, taken = gpu_fps(c, n, seed=N // 3)
    ri, rc, rmd, rtk, _ = O.fps(c, n, N // 3)
    np.testing.assert_array_equal(idx, ri)
    np.testing.assert_array_equal(curve, rc)
    np.testing.assert_array_equal(md, rmd)
    np.testing.assert_array_equal(taken, rtk)


@pytest.mark.parametrize("C", ["1", "2", "3", "4", "8", "16", "legacy"])
def test_fps_resident_cluster_widths(C, monkeypatch):
    """K1 v2 (resident, spatially sorted, warp-skip) at every cluster width,
    and the legacy register kernel, on tie-heavy and surface clouds."""
    if C == "legacy":
        monkeypatch.setenv("PS_FPS_LEGACY", "1")
    else:
        monkeypatch.setenv("PS_FPS_RESIDENT", "1")
        monkeypatch.setenv("PS_FPS_CLUSTER", C)
    for family, N, n in (("lattice", 4913, 1200), ("room-surfaces", 12000, 3000), ("gaussian-clusters", 9000, 900)):
        c = generate_cloud(family, N, 7)
        if family == "room-surfaces":
            c = c[np.lexsort((c[:, 2], c[:, 1], c[:, 0]))].copy()  # spatially coherent index order
        idx, curve, md, taken = gpu_fps(c, n, seed=N // 5)
        ri, rc, rmd, rtk, _ = O.fps(c, n, N // 5)
        np.testing.assert_array_equal(idx, ri, err_msg=f"{family} C={C}")
        np.testing.assert_array_equal(curve, rc)
        np.testing.assert_array_equal(md, rmd)
        np.testing.assert_array_equal(taken, rtk)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("kernel", ["speculative", "one-sample"])
@pytest.mark.parametrize("C", ["1", "2", "5", "10", "16"])
def test_fps_register_kernels_across_cluster_widths(kernel, C, monkeypatch):
    """Both register-resident exact kernels -- the speculative one (default,
    fps_spec.cu) and the one-exchange-per-sample one (fps.cu) -- at forced
    cluster widths, on tie-heavy (lattice), surface, clustered and
    half-duplicate clouds (the fallback of _kernels.py:65-70 mid-run and at
    the tail), full runs and a run stopped early, against the oracle:
    indices, curve, md and taken bit for bit."""
    monkeypatch.setenv("PS_FPS_CLUSTER", C)
    if kernel == "one-sample":
        monkeypatch.setenv("PS_FPS_NOSPEC", "1")
    else:
        monkeypatch.setenv("PS_FPS_SPEC", "1")  # also at C = 1, 2 (dispatched to one-sample by default)
    dup = generate_cloud("uniform-box", 1500, 3)
    dup = np.concatenate([dup, dup[::2]])[np.random.default_rng(1).permutation(2250)].copy()
    cases = (("lattice", generate_cloud("lattice", 4913, 7), 1200), ("room", generate_cloud("room-surfaces", 12000, 7), 3000),
             ("clusters", generate_cloud("gaussian-clusters", 9000, 7), 900), ("dup", dup, 2250))
    for name, c, n in cases:
        N = len(c)
        for k_stop in (n, max(2, n // 3)):
            xyz4 = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
            idx, curve, md, taken = engine.fps(xyz4, n, seed_index=N // 5, k_stop=k_stop)
            ri, rc, rmd, rtk, _ = O.fps(c, n, N // 5, k_stop=k_stop)
            msg = f"{name} {kernel} C={C} k_stop={k_stop}"
            np.testing.assert_array_equal(idx[0].cpu().numpy()[:k_stop], ri[:k_stop], err_msg=msg)
            np.testing.assert_array_equal(curve[0].cpu().numpy()[:k_stop], rc[:k_stop], err_msg=msg)
            np.testing.assert_array_equal(md[0].cpu().numpy(), rmd, err_msg=msg)
            np.testing.assert_array_equal(taken[0].cpu().numpy(), rtk, err_msg=msg)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("family", ["room-surfaces", "lattice", "half-duplicates"])
def test_fps_speculative_lead_owns_points(family, monkeypatch):
    """The speculative kernel's variant for 3841..4096 points per CTA (the
    lead warp owns points too; C4-sized clouds at C = 16) against the oracle,
    full run and early stop."""
    monkeypatch.setenv("PS_FPS_CLUSTER", "16")
    N = 64000
    if family == "half-duplicates":
        base = generate_cloud("uniform-box", N // 2, 11)
        c = np.concatenate([base, base])[np.random.default_rng(3).permutation(N)].copy()
    else:
        c = generate_cloud(family, N, 11)
    for n, k_stop in ((1200, 1200), (1200, 500)):
        xyz4 = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
        idx, curve, md, taken = engine.fps(xyz4, n, seed_index=N // 9, k_stop=k_stop)
        ri, rc, rmd, rtk, _ = O.fps(c, n, N // 9, k_stop=k_stop)
        msg = f"{family} k_stop={k_stop}"
        np.testing.assert_array_equal(idx[0].cpu().numpy()[:k_stop], ri[:k_stop], err_msg=msg)
        np.testing.assert_array_equal(curve[0].cpu().numpy()[:k_stop], rc[:k_stop], err_msg=msg)
        np.testing.assert_array_equal(md[0].cpu().numpy(), rmd, err_msg=msg)
        np.testing.assert_array_equal(taken[0].cpu().numpy(), rtk, err_msg=msg)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("family", ["room-surfaces", "half-duplicates"])
def test_fps_throughput_width_ten_points_per_thread(family):
    """The throughput-hint width (several batches in flight): C3 clouds at
    5-CTA clusters, 10 points per thread with md in shared memory and the
    lead warp on its own loop -- full run, early stop and a resumed tail,
    bit-exact against the oracle (duplicates exercise the fallback)."""
    N = 24000
    if family == "half-duplicates":
        base = generate_cloud("uniform-box", N // 2, 13)
        c = np.concatenate([base, base])[np.random.default_rng(5).permutation(N)].copy()
    else:
        c = generate_cloud(family, N, 13)
    B = 2
    cl = np.stack([c, generate_cloud("room-surfaces", N, 14)])
    xyz4 = engine.as_xyz4(torch.from_numpy(cl).cuda())
    with engine.inflight(8 * B):
        for n, k_stop in ((1500, 1500), (1500, 600)):
            idx, curve, md, taken = engine.fps(xyz4, n, seed_index=N // 7, k_stop=k_stop)
            for b in range(B):
                ri, rc, rmd, rtk, _ = O.fps(cl[b], n, N // 7, k_stop=k_stop)
                msg = f"{family} cloud {b} k_stop={k_stop}"
                np.testing.assert_array_equal(idx[b].cpu().numpy()[:k_stop], ri[:k_stop], err_msg=msg)
                np.testing.assert_array_equal(curve[b].cpu().numpy()[:k_stop], rc[:k_stop], err_msg=msg)
                np.testing.assert_array_equal(md[b].cpu().numpy(), rmd, err_msg=msg)
                np.testing.assert_array_equal(taken[b].cpu().numpy(), rtk, err_msg=msg)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_fps_small_cloud_kernel(W, monkeypatch):
    """The small-cloud kernel (fps_small.cu: one CTA of W warps per cloud,
    points in registers) at every points-per-lane width it instantiates, on
    tie-heavy, half-duplicate (fallback of _kernels.py:65-70, also when every
    point is taken) and uniform clouds, full runs, early stops and a resumed
    loop (fps_loop from a partial state), against the oracle bit for bit."""
    monkeypatch.setenv("PS_FPS_SMALL_W", str(W))
    rng = np.random.default_rng(W)
    for R in (1, 2, 4, 8, 16):
        N = max(3, W * 32 * R - int(rng.integers(0, W * 16 * R)))
        half = generate_cloud("uniform-box", (N + 1) // 2, 5)
        dup = np.concatenate([half, half])[:N][rng.permutation(N)].copy()
        cases = (("lattice", generate_cloud("lattice", N, 7)), ("dup", dup), ("box", generate_cloud("uniform-box", N, 9)))
        for name, c in cases:
            for n, k_stop in ((N, N), (max(2, N // 2), max(2, N // 5))):
                msg = f"W={W} R={R} N={N} {name} n={n} k_stop={k_stop}"
                xyz4 = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
                seed = N // 3
                idx, curve, md, taken = engine.fps(xyz4, n, seed_index=seed, k_stop=k_stop)
                ri, rc, rmd, rtk, _ = O.fps(c, n, seed, k_stop=k_stop)
                np.testing.assert_array_equal(idx[0].cpu().numpy()[:k_stop], ri[:k_stop], err_msg=msg)
                np.testing.assert_array_equal(curve[0].cpu().numpy()[:k_stop], rc[:k_stop], err_msg=msg)
                np.testing.assert_array_equal(md[0].cpu().numpy(), rmd, err_msg=msg)
                np.testing.assert_array_equal(taken[0].cpu().numpy(), rtk, err_msg=msg)
                if k_stop < n:  # resume to n from the partial state
                    engine.fps_loop(xyz4, md, taken, idx, curve, k_stop, n)
                    ri, rc, rmd, rtk, _ = O.fps(c, n, seed)
                    np.testing.assert_array_equal(idx[0].cpu().numpy(), ri, err_msg=msg + " resumed")
                    np.testing.assert_array_equal(curve[0].cpu().numpy(), rc, err_msg=msg + " resumed")
                    np.testing.assert_array_equal(md[0].cpu().numpy(), rmd, err_msg=msg + " resumed")
                    np.testing.assert_array_equal(taken[0].cpu().numpy(), rtk, err_msg=msg + " resumed")


@pytest.mark.timeout(300)
def test_fps_small_cloud_batches():
    """Default small-cloud dispatch over batches (C2's stage sizes, and 4096
    points at a chip-filling batch, which takes W = 8): every cloud against
    the oracle."""
    for B, N, n in ((32, 1024, 512), (32, 512, 256), (32, 256, 128), (32, 128, 64), (160, 4096, 300), (200, 600, 600)):
        clouds = np.stack([generate_cloud("room-surfaces", N, 40 + b) for b in range(B)])
        xyz4 = engine.as_xyz4(torch.from_numpy(clouds).cuda())
        idx, curve, md, taken = engine.fps(xyz4, n, seed_index=1)
        for b in sorted({0, B // 2, B - 1}):
            ri, rc, rmd, rtk, _ = O.fps(clouds[b], n, 1)
            msg = f"B={B} N={N} cloud {b}"
            np.testing.assert_array_equal(idx[b].cpu().numpy(), ri, err_msg=msg)
            np.testing.assert_array_equal(curve[b].cpu().numpy(), rc, err_msg=msg)
            np.testing.assert_array_equal(md[b].cpu().numpy(), rmd, err_msg=msg)
            np.testing.assert_array_equal(taken[b].cpu().numpy(), rtk, err_msg=msg)


@pytest.mark.timeout(300)
def test_fps_batch_beyond_one_wave():
    """40 clouds of 24000 points: more clusters than fit co-resident, so the
    speculative kernel runs in waves; FastPoint-prefix-length FPS, spot-checked
    clouds against the oracle."""
    B, N, n = 40, 24000, 600
    clouds = np.stack([generate_cloud("room-surfaces", N, 900 + b) for b in range(B)])
    xyz4 = engine.as_xyz4(torch.from_numpy(clouds).cuda())
    idx, curve, md, taken = engine.fps(xyz4, n, seed_index=5)
    for b in (0, 17, 39):
        ri, rc, rmd, rtk, _ = O.fps(clouds[b], n, 5)
        np.testing.assert_array_equal(idx[b].cpu().numpy(), ri, err_msg=f"cloud {b}")
        np.testing.assert_array_equal(curve[b].cpu().numpy(), rc)
        np.testing.assert_array_equal(md[b].cpu().numpy(), rmd)
        np.testing.assert_array_equal(taken[b].cpu().numpy(), rtk)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("case", range(24))
def test_fps_randomized_against_oracle(case, monkeypatch):
    """Seeded random cases for the exact FPS dispatch (speculative register
    kernel, its lead-owns-points variant, the resident kernel, the internal
    virtual-rank split): random N (1 .. 300000), n, seed, early stop, forced
    cluster width, cloud family incl. integer grids (exact md ties) and heavy
    duplicates; indices, curve, md, taken against the oracle bit for bit."""
    rng = np.random.default_rng(1000 + case)
    N = int(rng.choice([1, 2, 7, 33, 500, 1023, 4096, 12000, 24000, 40000, 65000, 120000, 300000]))
    kind = case % 4
    if kind == 0:
        c = generate_cloud("uniform-box", N, 50 + case)
    elif kind == 1:  # integer grid: many exactly tied distances
        c = rng.integers(0, 12, size=(N, 3)).astype(np.float32)
    elif kind == 2:  # heavy duplicates
        base = generate_cloud("room-surfaces", max(1, N // 3), 60 + case)
        c = base[rng.integers(0, base.shape[0], size=N)].copy()
    else:
        c = generate_cloud("gaussian-clusters", N, 70 + case)
    n = int(rng.integers(1, min(N, 1500) + 1))
    k_stop = n if rng.random() < 0.6 else int(rng.integers(1, n + 1))
    seed = int(rng.integers(0, N))
    if N <= 65536 and rng.random() < 0.4:
        monkeypatch.setenv("PS_FPS_CLUSTER", str(int(rng.choice([1, 2, 4, 8, 10, 16]))))
    xyz4 = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
    idx, curve, md, taken = engine.fps(xyz4, n, seed_index=seed, k_stop=k_stop)
    ri, rc, rmd, rtk, _ = O.fps(c, n, seed, k_stop=k_stop)
    msg = f"case {case}: N={N} n={n} k_stop={k_stop} seed={seed} kind={kind}"
    np.testing.assert_array_equal(idx[0].cpu().numpy()[:k_stop], ri[:k_stop], err_msg=msg)
    np.testing.assert_array_equal(curve[0].cpu().numpy()[:k_stop], rc[:k_stop], err_msg=msg)
    np.testing.assert_array_equal(md[0].cpu().numpy(), rmd, err_msg=msg)
    np.testing.assert_array_equal(taken[0].cpu().numpy(), rtk, err_msg=msg)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("family,N,n,G,B", [
    ("room-surfaces", 24000, 3000, 2, 1), ("room-surfaces", 24000, 3000, 4, 2), ("lattice", 4913, 1200, 3, 1),
    ("uniform-box", 200000, 1500, 4, 1), ("gaussian-clusters", 9000, 900, 8, 1), ("uniform-box", 4096, 1024, 1, 1),
])
def test_fps_point_split_virtual_ranks(family, N, n, G, B):
    """C5 point split: every cloud split over G ranks exchanging
    shard records through the mailbox protocol (all ranks on this GPU) is
    bit-identical to the single-rank reference FPS."""
    clouds = np.stack([generate_cloud(family, N, 31 + b) for b in range(B)])
    xyz4 = engine.as_xyz4(torch.from_numpy(clouds).cuda())
    mb = engine.SplitMailboxes(B, G)
    for rep in range(2):  # the second launch reuses the mailboxes (sequence tags)
        idx, curve, md, taken = engine.fps_split(xyz4, n, G, seed_index=N // 7, mailboxes=mb)
        for b in range(B):
            ri, rc, rmd, rtk, _ = O.fps(clouds[b], n, N // 7)
            np.testing.assert_array_equal(idx[b].cpu().numpy(), ri, err_msg=f"{family} G={G} rep={rep}")
            np.testing.assert_array_equal(curve[b].cpu().numpy(), rc)
            np.testing.assert_array_equal(md[b].cpu().numpy(), rmd)
            np.testing.assert_array_equal(taken[b].cpu().numpy(), rtk)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("loop", ["speculative", "one-sample"])
def test_fps_point_split_both_loops(loop, monkeypatch):
    """The resident kernel's two exchange loops (speculative default,
    PS_RES_NOSPEC=1 one sample per exchange) over virtual ranks, with a
    half-duplicate cloud (fallback across ranks) and an early stop."""
    if loop == "one-sample":
        monkeypatch.setenv("PS_RES_NOSPEC", "1")
    base = generate_cloud("room-surfaces", 15000, 21)
    cloud = np.concatenate([base, base[::3]])[np.random.default_rng(2).permutation(20000)].copy()
    xyz4 = engine.as_xyz4(torch.from_numpy(cloud[None]).cuda())
    for G, n, k_stop in ((3, 2000, 2000), (5, 2000, 700), (2, 20000, 20000)):
        idx, curve, md, taken = engine.fps_split(xyz4, n, G, seed_index=77, k_stop=k_stop)
        ri, rc, rmd, rtk, _ = O.fps(cloud, n, 77, k_stop=k_stop)
        msg = f"{loop} G={G} n={n} k_stop={k_stop}"
        np.testing.assert_array_equal(idx[0].cpu().numpy()[:k_stop], ri[:k_stop], err_msg=msg)
        np.testing.assert_array_equal(curve[0].cpu().numpy()[:k_stop], rc[:k_stop], err_msg=msg)
        np.testing.assert_array_equal(md[0].cpu().numpy(), rmd, err_msg=msg)
        np.testing.assert_array_equal(taken[0].cpu().numpy(), rtk, err_msg=msg)


@pytest.mark.timeout(300)
def test_fps_huge_cloud_internal_virtual_split():
    """Clouds beyond one cluster (here N = 300000) run ps_fps as the point
    split over co-resident virtual ranks with internal mailboxes: oracle
    parity for a full prefix, an early stop, and a resumed fps_loop."""
    N, n = 300000, 800
    c = generate_cloud("room-surfaces", N, 33)
    xyz4 = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
    for k_stop in (n, 300):
        idx, curve, md, taken = engine.fps(xyz4, n, seed_index=N // 3, k_stop=k_stop)
        ri, rc, rmd, rtk, _ = O.fps(c, n, N // 3, k_stop=k_stop)
        np.testing.assert_array_equal(idx[0].cpu().numpy()[:k_stop], ri[:k_stop], err_msg=f"k_stop={k_stop}")
        np.testing.assert_array_equal(curve[0].cpu().numpy()[:k_stop], rc[:k_stop])
        np.testing.assert_array_equal(md[0].cpu().numpy(), rmd)
        np.testing.assert_array_equal(taken[0].cpu().numpy(), rtk)
    # resume the early-stopped run to n through the fps_loop drop-in path
    idx, curve, md, taken = engine.fps(xyz4, n, seed_index=N // 3, k_stop=300)
    engine.fps_loop(xyz4, md, taken, idx, curve, 300, n)
    ri, rc, rmd, rtk, _ = O.fps(c, n, N // 3)
    np.testing.assert_array_equal(idx[0].cpu().numpy(), ri)
    np.testing.assert_array_equal(md[0].cpu().numpy(), rmd)


@pytest.mark.timeout(300)
def test_fps_point_split_duplicates_fallback():
    """All-duplicate tails force the lowest-untaken fallback to be exchanged
    across ranks (_kernels.py:65-70)."""
    B, N = 2, 900
    base = generate_cloud("uniform-box", 300, 5)
    clouds = np.stack([np.repeat(base, 3, axis=0)[np.random.default_rng(b).permutation(N)] for b in range(B)])
    xyz4 = engine.as_xyz4(torch.from_numpy(clouds).cuda())
    for G in (2, 3):
        idx, curve, _, _ = engine.fps_split(xyz4, N, G, seed_index=4)
        for b in range(B):
            ri, rc, *_ = O.fps(clouds[b], N, 4)
            np.testing.assert_array_equal(idx[b].cpu().numpy(), ri)
            np.testing.assert_array_equal(curve[b].cpu().numpy(), rc)


def test_fps_batched_and_duplicates():
    B, N = 5, 900
    base = generate_cloud("uniform-box", 300, 5)
    clouds = np.stack([np.repeat(base, 3, axis=0)[np.random.default_rng(b).permutation(N)] for b in range(B)])
    xyz4 = engine.as_xyz4(torch.from_numpy(clouds).cuda())
    idx, curve, _, _ = engine.fps(xyz4, N, 4)  # n = N forces the duplicate fallback
    for b in range(B):
        ri, rc, *_ = O.fps(clouds[b], N, 4)
        np.testing.assert_array_equal(idx[b].cpu().numpy(), ri)
        np.testing.assert_array_equal(curve[b].cpu().numpy(), rc)


def test_fps_loop_resume_dropin():
    c = generate_cloud("room-surfaces", 3000, 9)
    x, y, z = O.columns_f64(c)
    n = 700
    st = {}
    for nm, K in (("gpu", GK), ("ora", O.CKernels)):
        md = np.full(3000, np.inf)
        tk = np.zeros(3000, np.uint8)
        out = np.full(n, -1, np.int64)
        cv = np.full(n, np.inf)
        out[0] = 17
        tk[17] = 1
        e1 = K.fps_loop(x, y, z, md, tk, out, cv, 1, 333)
        e2 = K.fps_loop(x, y, z, md, tk, out, cv, 333, n)
        st[nm] = (md, tk, out, cv, e1 + e2)
    for a, b in zip(st["gpu"], st["ora"]):
        np.testing.assert_array_equal(a, b)


def test_dropin_chunk_and_first_untaken():
    c = generate_cloud("lattice", 2000, 3)
    x, y, z = O.columns_f64(c)
    md_g = np.full(2000, np.inf)
    md_o = md_g.copy()
    for (lo, hi, p) in ((0, 2000, 5), (100, 777, 42), (1500, 2000, 1999), (10, 10, 3)):
        rg = GK.fps_update_chunk(x, y, z, x[p], y[p], z[p], md_g, lo, hi)
        ro = O.CKernels.fps_update_chunk(x, y, z, x[p], y[p], z[p], md_o, lo, hi)
        assert rg == ro
        np.testing.assert_array_equal(md_g, md_o)
    tk = np.ones(2000, np.uint8)
    assert GK.first_untaken(tk) == -1
    tk[1234] = 0
    tk[1999] = 0
    assert GK.first_untaken(tk) == 1234


# ---- K3a/K3b exclusion lists --------------------------------------------------------

def test_excl_golden(golden):
    for t in cases(golden, "excl"):
        k = f"excl/{t}"
        c = golden[f"cloud/{golden[k + '/cloud']}"]
        R = list(golden[f"{k}/R"])
        extra = tuple(golden[f"{k}/extra"])
        levels = golden[f"{k}/levels"]  # oracle layout: sorted unique r2 levels
        x, y, z = O.columns_f64(c)
        for method in (0, 1):
            indptr, nbr, d2, counts, evals = GK.build_csr(x, y, z, levels, method=method)
            assert indptr[-1] == int(golden[f"{k}/E"])
            assert evals + len(c) == int(golden[f"{k}/evals"])
            np.testing.assert_array_equal(digest(indptr, nbr, d2, counts), golden[f"{k}/digest"], err_msg=k)


@pytest.mark.parametrize("family,N,R", [("uniform-box", 6000, 0.05), ("room-surfaces", 8000, 0.2),
                                        ("lattice", 4096, 0.1000001), ("gaussian-clusters", 3000, 0.02),
                                        ("uniform-box", 700, 3.0), ("lidar-rings", 5000, 1e-30)])
def test_excl_matches_oracle(family, N, R):
    c = generate_cloud(family, N, 77)
    e = O.build_exclusion_lists(c, [R, R * 0.8, R * 0.5], (R * 0.6,))
    x, y, z = O.columns_f64(c)
    for method in (0, 1):
        indptr, nbr, d2, counts, _ = GK.build_csr(x, y, z, e.r2_levels, method=method)
        np.testing.assert_array_equal(indptr, e.indptr)
        np.testing.assert_array_equal(nbr, e.nbr)
        np.testing.assert_array_equal(d2, e.d2)
        np.testing.assert_array_equal(counts, e.counts)


def _set_excl_variant(variant, monkeypatch):
    # "auto": the default choice; "2": cells of width R_max / 2 with culled /
    # trimmed candidate rows (the long-row path) forced; "1": cells of width
    # R_max (warp per cell, candidates in registers) forced; "row": the warp-
    # per-point kernel over 3 x 3 cell rows (grid_ell_kernel)
    if variant in ("1", "2"):
        monkeypatch.setenv("PS_GRID_REACH", variant)
    elif variant == "row":
        monkeypatch.setenv("PS_GRID_REACH", "1")
        monkeypatch.setenv("PS_ELL_ROW", "1")


@pytest.mark.parametrize("reach", ["auto", "2", "row"])
@pytest.mark.parametrize("N", [5000, 4096, 1000])
def test_excl_bucketed_rows_match_oracle_sets(N, reach, monkeypatch):
    """Method-2 rows against the oracle's sorted CSR as sets per level, for
    every row kernel (see _set_excl_variant)."""
    _set_excl_variant(reach, monkeypatch)
    # method 2 (hot path): fixed stride, rows bucketed by level -- every
    # level's entries are the row prefix; as sets they equal the reference's.
    # N <= 4096 takes the fused one-CTA grid build, 5000 the multi-kernel one.
    _check_bucketed_rows(generate_cloud("room-surfaces", N, 5), [0.3, 0.25, 0.2, 0.2, 0.15, 0.1], 0.12, 256)


@pytest.mark.parametrize("reach", ["1", "row"])
def test_excl_bucketed_rows_dense(reach, monkeypatch):
    """A dense volume: ~1300 candidates per cell (the cell kernel reloads its
    register window per row), rows above 256 entries (the per-bucket rescan),
    rows beyond the stride (spill arena)."""
    _set_excl_variant(reach, monkeypatch)
    _check_bucketed_rows(generate_cloud("uniform-box", 6000, 8), [0.21, 0.2, 0.17, 0.15, 0.12, 0.1], 0.05, 300)


@pytest.mark.parametrize("variant", ["auto", "1", "row"])
@pytest.mark.parametrize("family,N,R", [("uniform-box", 6000, 0.05), ("lattice", 4096, 0.1000001),
                                        ("gaussian-clusters", 3000, 0.02), ("uniform-box", 700, 3.0),
                                        ("lidar-rings", 5000, 1e-30), ("uniform-box", 1, 0.1),
                                        ("room-surfaces", 7, 0.5)])
def test_excl_bucketed_rows_families(family, N, R, variant, monkeypatch):
    """Method-2 rows for every row kernel on the families of
    test_excl_matches_oracle: lattice ties, dense clusters, a radius above the
    cloud's diameter (every row the whole cloud: rescans), no neighbour at all,
    one- and seven-point clouds."""
    _set_excl_variant(variant, monkeypatch)
    _check_bucketed_rows(generate_cloud(family, N, 77), [R, R * 0.8, R * 0.5], R * 0.6, None)


def test_excl_bucketed_rows_many_levels():
    """Ten levels (eight segments + two baked radii): beyond the cell
    kernel's eight buckets, the build takes the per-row kernel."""
    R = [0.3, 0.28, 0.25, 0.21, 0.18, 0.15, 0.12, 0.1]
    c = generate_cloud("room-surfaces", 5000, 9)
    e = O.build_exclusion_lists(c, R, (0.13, 0.07))
    levels = np.array([O.radius_sq(r) for r in R] + [O.radius_sq(0.13), O.radius_sq(0.07)])
    csr = engine.DeviceCsr.allocate(1, 5000, len(levels), 5000 * 256, 1, torch.device("cuda"), 2)
    csr.levels.copy_(torch.from_numpy(levels.reshape(1, -1)))
    csr.build(engine.as_xyz4(c))
    assert not csr.overflowed()
    counts = csr.counts[0].cpu().numpy()
    pos = {float(v): k for k, v in enumerate(e.r2_levels)}
    for l, lv in enumerate(levels):
        np.testing.assert_array_equal(counts[l], e.counts[pos[float(lv)]])


def _check_bucketed_rows(c, R, extra, cap_per_point):
    N = c.shape[0]
    e = O.build_exclusion_lists(c, R, (extra,))
    if cap_per_point is None:  # room for the longest row in the strided part
        cap_per_point = max(16, int(1.25 * int(e.counts[-1].max())) + 8)
    levels = np.array([O.radius_sq(r) for r in R] + [O.radius_sq(extra)])
    csr = engine.DeviceCsr.allocate(1, N, len(levels), N * cap_per_point, 1, torch.device("cuda"), 2)
    csr.levels.copy_(torch.from_numpy(levels.reshape(1, -1)))
    csr.build(engine.as_xyz4(c))
    assert not csr.overflowed()
    counts = csr.counts[0].cpu().numpy()
    nbr = csr.nbr[0].cpu().numpy()
    d2 = csr.d2[0].cpu().numpy()
    pos = {float(v): k for k, v in enumerate(e.r2_levels)}
    for l, lv in enumerate(levels):
        np.testing.assert_array_equal(counts[l], e.counts[pos[float(lv)]])
    ip = csr.indptr[0].cpu().numpy()
    stride = csr.stride
    assert np.all(ip[:N] % 4 == 0)  # 16-byte aligned rows (strided or spilled)
    for i in range(0, N, 7):
        m = counts[0]  # widest level is R[0]
        a = ip[i]
        assert a == i * stride or (a >= N * stride and m[i] > stride)  # spilled rows are the long ones
        got = sorted(zip(d2[a:a + m[i]].tolist(), nbr[a:a + m[i]].tolist()))
        lo = e.indptr[i]
        ref = list(zip(e.d2[lo:lo + m[i]].tolist(), e.nbr[lo:lo + m[i]].tolist()))
        assert got == ref, i
        for l, lv in enumerate(levels):  # each level is a prefix
            assert np.all(d2[a:a + counts[l][i]] < lv)


def test_excl_prefilter_adversarial():
    # pairs placed at float64 distances straddling r exactly: the float32
    # pre-filter must never drop a pair whose exact d2 is below r2.
    rng = np.random.default_rng(1)
    base = rng.random((400, 3)).astype(np.float32) * 10
    r = np.float64(0.3)
    pts = [base]
    for s in (1 - 1e-7, 1 - 3e-8, 1.0, 1 + 3e-8):
        off = (rng.normal(size=(400, 3)))
        off /= np.linalg.norm(off, axis=1, keepdims=True)
        pts.append((base + (off * r * s)).astype(np.float32))
    c = np.concatenate(pts)
    x, y, z = O.columns_f64(c)
    r2 = [float(r * r)]
    e_ip, e_nb, e_d2, _ = O.CKernels.excl_build(x, y, z, r2[0])
    for method in (0, 1):
        indptr, nbr, d2, counts, _ = GK.build_csr(x, y, z, r2, method=method)
        np.testing.assert_array_equal(indptr, e_ip)
        np.testing.assert_array_equal(nbr, e_nb)
        np.testing.assert_array_equal(d2, e_d2)


def test_dropin_collect_fill_sort_counts():
    c = generate_cloud("uniform-box", 1500, 8)
    x, y, z = O.columns_f64(c)
    r2 = 0.09 ** 2
    N = 1500
    T = (N + 1) // 2
    ei, ej, ed, ev = GK.excl_collect(x, y, z, 0, T, r2, 1024)
    # reference order/semantics restated: rows (k, N-1-k), j ascending
    e = O.build_exclusion_lists(c, [0.09])
    deg = np.ones(N, np.int64)
    np.add.at(deg, ei, 1)
    np.add.at(deg, ej, 1)
    indptr = np.zeros(N + 1, np.int64)
    np.cumsum(deg, out=indptr[1:])
    nbr = np.empty(indptr[-1], np.int64)
    d2 = np.empty(indptr[-1], np.float64)
    GK.csr_fill(ei, ej, ed, indptr, nbr, d2)
    # the fill order itself (before sorting): _kernels.py:164-185 restated
    ref_nbr, ref_d2 = np.empty_like(nbr), np.empty_like(d2)
    cur = indptr[:N].copy()
    ref_nbr[cur], ref_d2[cur] = np.arange(N), 0.0
    cur += 1
    for a, b, d in zip(ei, ej, ed):
        ref_nbr[cur[a]], ref_d2[cur[a]] = b, d
        cur[a] += 1
        ref_nbr[cur[b]], ref_d2[cur[b]] = a, d
        cur[b] += 1
    np.testing.assert_array_equal(nbr, ref_nbr)
    np.testing.assert_array_equal(d2, ref_d2)
    GK.csr_sort_rows(indptr, d2, nbr)
    np.testing.assert_array_equal(indptr, e.indptr)
    np.testing.assert_array_equal(nbr, e.nbr)
    np.testing.assert_array_equal(d2, e.d2)
    assert ev == N * (N - 1) // 2
    np.testing.assert_array_equal(GK.csr_level_counts(indptr, d2, e.r2_levels), e.counts)


# ---- K2/K3c/K3d full FastPoint pipeline --------------------------------------------

@pytest.mark.parametrize("method", ["bruteforce", "grid-sorted", "grid"])
def test_mdps_golden(golden, method):
    for t in cases(golden, "mdps"):
        k = f"mdps/{t}"
        c = golden[f"cloud/{golden[k + '/cloud']}"]
        n = int(golden[f"{k}/n"])
        kw = mdps_kwargs(golden, t)
        fp = gpu_mdps(c, n, excl_method=method, **kw)
        np.testing.assert_array_equal(fp.out[0].cpu().numpy(), golden[f"{k}/idx"], err_msg=k)
        assert int(fp.reached.item()) == int(golden[f"{k}/reached"]), k
        assert bool(fp.exhausted.item()) == bool(golden[f"{k}/exhausted"]), k
        assert int(fp.entered.item()) == int(golden[f"{k}/entered"]), k
        st = int(np.int64(fp.state.item()).view(np.uint64))
        assert st == int(golden[f"{k}/state"]), k
        np.testing.assert_array_equal(fp.R[0].cpu().numpy(), golden[f"{k}/R"], err_msg=k)
        if method == "bruteforce":  # SPEC.md:438 accounting (A7)
            assert fp.pair_evals()[0] == int(golden[f"{k}/evals"]), k
        else:
            assert fp.pair_evals()[0] <= int(golden[f"{k}/evals"]), k


@pytest.mark.parametrize("reach", ["auto", "2", "row"])
@pytest.mark.parametrize("B,N,n,family,nseg,pick", [
    (4, 4096, 1024, "uniform-box", 6, False), (3, 3000, 750, "room-surfaces", 6, True),
    (2, 24000, 6000, "room-surfaces", 6, False), (2, 5000, 1250, "lattice", 4, False),
    (1, 40000, 10000, "uniform-box", 6, False),  # global-memory sampler workspace
])
def test_mdps_batched_matches_oracle(B, N, n, family, nseg, pick, reach, monkeypatch):
    _set_excl_variant(reach, monkeypatch)
    clouds = np.stack([generate_cloud(family, N, 1000 + b) for b in range(B)])
    e = 0.42
    fp = engine.FastPoint(B, N, n, nseg=nseg, exponent=e, extra_radii=(0.1,), pick_lowest=pick)
    fp.set_points(torch.from_numpy(clouds).cuda())
    fp.set_rng([7 + b for b in range(B)])
    fp.sample()
    fp.check()
    gi, gd, gc = fp.group_rf(0.1, 32)
    for b in range(B):
        ref = O.mdps(clouds[b], n, nseg=nseg, exponent=e, rng_seed=7 + b, extra_radii=(0.1,), pick_lowest=pick)
        np.testing.assert_array_equal(fp.out[b].cpu().numpy(), ref.indices, err_msg=f"cloud {b}")
        assert int(fp.reached[b].item()) == ref.reached
        assert int(np.int64(fp.state[b].item()).view(np.uint64)) == ref.rng_state
        oi, od, oc = O.rf_ball_query(ref.excl, 0.1, ref.indices, 32)
        np.testing.assert_array_equal(gi[b].cpu().numpy().astype(np.int64), oi)
        np.testing.assert_array_equal(gd[b].cpu().numpy(), od)
        np.testing.assert_array_equal(gc[b].cpu().numpy().astype(np.int64), oc)


def test_dropin_sampler_and_earlyterm():
    c = generate_cloud("uniform-box", 2500, 4)
    e = O.build_exclusion_lists(c, [0.09, 0.07, 0.06], ())
    prefix = O.fps(c, 60)[0]
    bnd = O.sampler_boundaries(600, 3)
    for pick in (False, True):
        for seed in (0, 123456789):
            g = GK.sample_predicted(e.indptr, e.nbr, e.counts, e.seg_level_rows, bnd, prefix, 600, 2500,
                                    np.uint64(seed), pick)
            o = O.CKernels.sample_predicted(e.indptr, e.nbr, e.counts, e.seg_level_rows, bnd, prefix, 600, 2500,
                                            np.uint64(seed), pick)
            np.testing.assert_array_equal(g[0], o[0])
            assert g[1:] == o[1:]
    taken = np.zeros(2500, np.uint8)
    taken[::5] = 1
    md_g = np.full(2500, np.inf)
    md_o = md_g.copy()
    lv = np.ascontiguousarray(e.counts[e.seg_level_rows[0]])
    GK.earlyterm_scan(e.indptr, e.nbr, e.d2, lv, taken, md_g, 0, 2500)
    O.CKernels.earlyterm_scan(e.indptr, e.nbr, e.d2, lv, taken, md_o, 0, 2500)
    np.testing.assert_array_equal(md_g, md_o)


def test_mdps_cuda_graph_replay_identical():
    B, N, n = 2, 4096, 1024
    clouds = np.stack([generate_cloud("uniform-box", N, 50 + b) for b in range(B)])
    fp = engine.FastPoint(B, N, n, exponent=0.4, extra_radii=(0.05,))
    fp.set_points(torch.from_numpy(clouds).cuda())
    fp.set_rng([1, 2])
    fp.sample()
    first = fp.out.clone()
    fp.capture()
    for _ in range(3):
        fp.set_rng([1, 2])
        fp.out.fill_(-7)
        fp.sample()
        torch.cuda.synchronize()
        assert torch.equal(fp.out, first)


def _dense_cloud(N, n_dup, seed):
    """Uniform box with n_dup copies of one point: n_dup rows of >= n_dup
    entries, far beyond the default row stride."""
    c = generate_cloud("uniform-box", N, seed)
    c[:n_dup] = c[0]
    return c[np.random.default_rng(seed).permutation(N)].copy()


@pytest.mark.timeout(300)
def test_graph_replay_spill_and_exhausted_capacity():
    """A FastPoint CUDA graph captured on an ordinary cloud and replayed on
    new points: (1) rows beyond the stride spill into the arena inside the
    same launch sequence -- replay output equals the oracle, no host step;
    (2) rows beyond the whole arena leave an explicit error state (indices -1
    past the prefix, entered -1, rf counts -1) that survives the replay, and
    check() rebuilds with a larger capacity, re-captures, and then matches."""
    N, n, e, r = 4096, 1024, 0.4, 0.05
    fp = engine.FastPoint(1, N, n, exponent=e, extra_radii=(r,))
    stride = fp.csr.stride
    spill = fp.csr.cap_entries - N * stride
    fp.set_points(torch.from_numpy(generate_cloud("uniform-box", N, 5)[None]).cuda())
    fp.set_rng([9])
    fp.sample()
    fp.check()
    fp.capture()
    grp = (torch.empty(1, n, 16, dtype=torch.int32, device="cuda"),
           torch.empty(1, n, 16, dtype=torch.float64, device="cuda"),
           torch.empty(1, n, dtype=torch.int32, device="cuda"))
    n_spill = stride + stride // 4  # rows of ~n_spill entries: they spill, and fit the arena
    assert n_spill > stride and n_spill * (n_spill + 4) < spill
    n_big = int(1.2 * spill ** 0.5) + stride  # rows beyond the whole arena
    for name, n_dup in (("spill", n_spill), ("exhausted", n_big)):
        c = _dense_cloud(N, n_dup, 17)
        fp.set_points(torch.from_numpy(c[None]).cuda())
        fp.set_rng([9])
        fp.sample()  # graph replay
        fp.group_rf(r, 16, out=grp)
        torch.cuda.synchronize()
        ref = O.mdps(c, n, exponent=e, rng_seed=9, extra_radii=(r,))
        if name == "spill":
            assert not fp.csr.overflowed()
            np.testing.assert_array_equal(fp.out[0].cpu().numpy(), ref.indices, err_msg="spilled rows")
            oi, _, oc = O.rf_ball_query(ref.excl, r, ref.indices, 16)
            np.testing.assert_array_equal(grp[2][0].cpu().numpy().astype(np.int64), oc)
            continue
        assert fp.csr.overflowed()
        out = fp.out[0].cpu().numpy()
        assert np.all(out[fp.k0:] == -1) and int(fp.entered[0].item()) == -1
        assert int(fp.reached[0].item()) == n
        cnt = grp[2][0].cpu().numpy()
        assert np.all(cnt == -1)
        assert fp.check() is True  # grow + re-run + re-capture
        assert fp.graph is not None and not fp.csr.overflowed()
        np.testing.assert_array_equal(fp.out[0].cpu().numpy(), ref.indices, err_msg="after check()")
        fp.set_rng([9])
        fp.out.fill_(-7)
        fp.sample()  # the re-captured graph
        torch.cuda.synchronize()
        np.testing.assert_array_equal(fp.out[0].cpu().numpy(), ref.indices, err_msg="re-captured graph")


def test_ball_query_rf_rejects_k_beyond_128():
    fp = gpu_mdps(generate_cloud("uniform-box", 2000, 3), 500, exponent=0.4, extra_radii=(0.2,))
    with pytest.raises(ValueError, match=r"k must be in \[1, 128\]"):
        fp.group_rf(0.2, 200)
    gi, gd, gc = fp.group_rf(0.2, 128)  # the bound itself: dense rows, exact vs oracle
    ref = O.mdps(generate_cloud("uniform-box", 2000, 3), 500, exponent=0.4, rng_seed=0, extra_radii=(0.2,))
    oi, od, oc = O.rf_ball_query(ref.excl, 0.2, ref.indices, 128)
    assert int(oc.max()) > 64
    np.testing.assert_array_equal(gc[0].cpu().numpy().astype(np.int64), oc)
    np.testing.assert_array_equal(gi[0].cpu().numpy().astype(np.int64), oi)


@pytest.mark.timeout(300)
def test_virtual_split_graph_replay_changing_inputs():
    """ps_fps on a cloud beyond one cluster runs the virtual-rank point split;
    captured in a CUDA graph and replayed on changing points, every replay
    gets fresh mailbox tags (device-side epoch) and matches the oracle."""
    N, n = 300000, 400
    clouds = [generate_cloud(f, N, 8) for f in ("room-surfaces", "uniform-box", "gaussian-clusters")]
    x = engine.as_xyz4(torch.from_numpy(clouds[0][None]).cuda())
    md = torch.empty(1, N, dtype=torch.float64, device="cuda")
    taken = torch.empty(1, N, dtype=torch.uint8, device="cuda")
    out = torch.full((1, n), -1, dtype=torch.int64, device="cuda")
    curve = torch.full((1, n), np.inf, dtype=torch.float64, device="cuda")
    from paper_2507_23480_b200 import _lib

    def run():
        _lib.call("ps_fps", x.data_ptr(), 1, N, md.data_ptr(), taken.data_ptr(), out.data_ptr(), curve.data_ptr(),
                  n, n, 5, None, torch.cuda.current_stream().cuda_stream)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for rep in range(2):
        for c in clouds[1:] + clouds[:1]:
            x[0, :, :3].copy_(torch.from_numpy(c))
            out.fill_(-7)
            g.replay()
            torch.cuda.synchronize()
            ri, rc, *_ = O.fps(c, n, 5)
            np.testing.assert_array_equal(out[0].cpu().numpy(), ri, err_msg=f"replay {rep}")
            np.testing.assert_array_equal(curve[0].cpu().numpy(), rc)


# ---- K4 grouping and K6 quality ------------------------------------------------------

def test_ball_query_naive_and_rf_equal_oracle():
    c = generate_cloud("room-surfaces", 6000, 21)
    cent = O.fps(c, 1500)[0]
    for r, k in ((0.1, 32), (0.25, 64), (0.05, 1)):
        oi, od, oc = O.ball_query_naive(c, cent, r, k)
        xyz4 = engine.as_xyz4(c)
        gi, gd, gc = engine.ball_query_naive(xyz4, torch.from_numpy(cent).cuda().reshape(1, -1), r, k)
        np.testing.assert_array_equal(gi[0].cpu().numpy().astype(np.int64), oi)
        np.testing.assert_array_equal(gd[0].cpu().numpy(), od)
        np.testing.assert_array_equal(gc[0].cpu().numpy().astype(np.int64), oc)
        e = O.build_exclusion_lists(c, [r * 0.5], (r,))
        ri, rd, rc = O.rf_ball_query(e, r, cent, k)
        np.testing.assert_array_equal(ri, oi)  # RF == naive (A2)


def test_knn_naive_and_rf():
    c = generate_cloud("uniform-box", 4000, 31)
    n = 1000
    fp = gpu_mdps(c, n, exponent=0.4)
    pool = fp.out[0].cpu().numpy()
    queries = np.arange(4000)
    for k in (1, 3, 16):
        oi, od, oc = O.knn_naive(c, queries, pool, k)
        xyz4 = engine.as_xyz4(c)
        gi, gd, gc = engine.knn_naive(xyz4, fp.out, k)
        np.testing.assert_array_equal(gi[0].cpu().numpy().astype(np.int64), oi)
        np.testing.assert_array_equal(gd[0].cpu().numpy(), od)
        ri, rd, rc, fb = fp.knn_rf(k)
        np.testing.assert_array_equal(ri[0].cpu().numpy().astype(np.int64), oi)
        np.testing.assert_array_equal(rd[0].cpu().numpy(), od)
    assert int(fb[0].item()) > 0  # k = 16 forces fallbacks


def test_min_spacing_tolerance():
    c = generate_cloud("uniform-box", 5000, 41)
    s = O.fps(c, 1200)[0]
    ref_d2 = O.min_spacing_d2(c, s)
    xyz4 = engine.as_xyz4(c)
    got = engine.min_spacing_d2(xyz4, torch.from_numpy(s).cuda().reshape(1, -1))[0].cpu().numpy()
    np.testing.assert_array_equal(got, ref_d2)  # per-sample minima: exact
    from paper_2507_23480_b200 import quality
    v = quality.avg_min_spacing(c, s)
    assert abs(v - O.avg_min_spacing(c, s)) <= 1e-12 * abs(v)  # mean: reduction order only


def test_errors_are_value_errors():
    with pytest.raises(ValueError):
        engine.FastPoint(1, 100, 10, exponent=None)
    with pytest.raises(ValueError):
        engine.fps(engine.as_xyz4(np.zeros((5, 3), np.float32)), 6)
    fp = gpu_mdps(generate_cloud("uniform-box", 500, 1), 100, exponent=0.4, extra_radii=(0.1,))
    with pytest.raises(ValueError, match="not baked"):
        fp.group_rf(0.2, 8)


# ---- C2: multi-stage set-abstraction cascade -----------------------------

@pytest.mark.timeout(300)
@pytest.mark.parametrize("first", ["fastpoint", "fps"])
def test_sa_cascade_matches_oracle(first):
    """Four stride-2 stages on unit-sphere clouds (C2 shape, B reduced):
    stage 0 FastPoint + rf ball query (or exact FPS + naive), later stages
    exact FPS + naive ball query on the previous samples -- every stage's
    indices, group members and counts bit-identical to the oracle cascade;
    the CUDA-graph replay reproduces them."""
    B, N, k = 3, 1024, 32
    clouds = np.stack([generate_cloud("unit-sphere", N, 70 + b) for b in range(B)])
    exponent = 0.5
    sa = engine.SACascade(B, N, k=k, first=first, exponent=exponent)
    sa.set_points(torch.from_numpy(clouds).cuda())
    sa.set_rng(list(range(B)))
    sa.run()
    torch.cuda.synchronize()
    got = [(sa.idx[s].cpu().numpy(), sa.groups[s][0].cpu().numpy(), sa.groups[s][2].cpu().numpy())
           for s in range(4)]
    for b in range(B):
        ref = O.sa_cascade(clouds[b], k=k, first=first, exponent=exponent, rng_seed=b)
        for s, (ri, rg, rc) in enumerate(ref):
            gi, gg, gc = got[s]
            np.testing.assert_array_equal(gi[b], ri, err_msg=f"stage {s} indices, cloud {b}")
            np.testing.assert_array_equal(gc[b], rc, err_msg=f"stage {s} counts")
            for t in range(len(ri)):
                m = int(rc[t])
                np.testing.assert_array_equal(gg[b, t, :m], rg[t, :m])
    sa.set_rng(list(range(B)))
    sa.capture()
    sa.set_rng(list(range(B)))
    sa.run()
    torch.cuda.synchronize()
    for s in range(4):
        np.testing.assert_array_equal(sa.idx[s].cpu().numpy(), got[s][0])


@pytest.mark.timeout(600)
def test_c4_shape_fastpoint_matches_oracle():
    """C4 cloud shape (N = 65536 -> 16384, room surfaces): FastPoint indices,
    reached count and RF groups bit-identical to the oracle (global-memory
    sampler tables, large-N FPS plan)."""
    N, n = 65536, 16384
    c = generate_cloud("room-surfaces", N, 4242)
    fp = engine.FastPoint(1, N, n, exponent=0.53, extra_radii=(0.1,))
    fp.set_points(torch.from_numpy(c[None]).cuda())
    fp.set_rng([5])
    fp.sample()
    fp.check()
    gi, _, gc = fp.group_rf(0.1, 32)
    ref = O.mdps(c, n, exponent=0.53, rng_seed=5, extra_radii=(0.1,))
    np.testing.assert_array_equal(fp.out[0].cpu().numpy(), ref.indices)
    assert int(fp.reached[0].item()) == ref.reached
    oi, _, oc = O.rf_ball_query(ref.excl, 0.1, ref.indices, 32)
    np.testing.assert_array_equal(gc[0].cpu().numpy(), oc)


# ---- MLP estimator --------------------------------------

@pytest.mark.timeout(300)
def test_mlp_estimator_thresholds_and_sampling_match_oracle():
    """FastPoint with the MLP estimator: K2 evaluates resample -> 32-128-128-64
    MLP -> resample -> running min on the device; radii and sampled indices
    bit-identical to the oracle's estimate_mlp path (model trained briefly on
    exact curves of the family, saved and reloaded in the SPEC.md:357 format)."""
    import tempfile

    from paper_2507_23480_b200 import curve as Cv

    N, n = 6000, 1500
    train = [O.fps(generate_cloud("room-surfaces", N, 500 + i), n)[1] for i in range(3)]
    model, losses = Cv.mlp_train([Cv.mlp_pair(c) for c in train], epochs=20, lr=0.01,
                                 rng=np.random.default_rng(3))
    assert losses[-1] <= losses[0]
    path = tempfile.mktemp(suffix=".mlp")
    model.save(path)
    model = Cv.MlpModel.load(path)
    om = O.read_mlp(path)
    B = 2
    clouds = np.stack([generate_cloud("room-surfaces", N, 600 + b) for b in range(B)])
    fp = engine.FastPoint(B, N, n, estimator="mlp", mlp=model, extra_radii=(0.1,))
    fp.set_points(torch.from_numpy(clouds).cuda())
    fp.set_rng([0, 1])
    fp.sample()
    fp.check()
    for b in range(B):
        ref = O.mdps(clouds[b], n, estimator="mlp", mlp=om, rng_seed=b, extra_radii=(0.1,))
        np.testing.assert_array_equal(fp.R[b].cpu().numpy(), ref.thresholds, err_msg="segment radii")
        np.testing.assert_array_equal(fp.out[b].cpu().numpy(), ref.indices)
        np.testing.assert_array_equal(Cv.estimate_mlp(ref.est_curve[:fp.k0], n, model), ref.est_curve)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("variant", ["global-workspace", "grid-mode", "grid-mode-lattice", "many-levels",
                                     "many-small-clouds", "exhausting"])
def test_sampler_variants_match_oracle(variant, monkeypatch):
    """Sampler code paths beyond the default: the global-memory mode of v4
    (one cluster per cloud, and the grid mode: a cooperative grid slice per
    cloud with a global barrier), 12 segments + 3 baked radii (L = 15 levels),
    a batch of many single-CTA clouds (block barriers), and tight radii that
    exhaust segment pools (entered / exhausted bookkeeping)."""
    B, N, n, nseg, extra, family, e = 3, 6000, 1500, 6, (0.1,), "room-surfaces", 0.45
    if variant == "global-workspace":
        monkeypatch.setenv("PS_SAMPLER_GLOBAL", "1")
        monkeypatch.setenv("PS_SAMPLER_NOGRID", "1")
    elif variant.startswith("grid-mode"):  # cooperative grid of 12 CTAs per cloud, global barrier
        monkeypatch.setenv("PS_SAMPLER_GLOBAL", "1")
        monkeypatch.setenv("PS_SAMPLER_GRID_CTAS", "12")
        if variant.endswith("lattice"):
            family, e = "lattice", 0.9
    elif variant == "many-levels":
        nseg, extra = 12, (0.05, 0.1, 0.2)
    elif variant == "many-small-clouds":
        B, N, n, family = 24, 1500, 400, "unit-sphere"
    elif variant == "exhausting":
        family, e = "lattice", 0.9
    clouds = np.stack([generate_cloud(family, N, 4000 + b) for b in range(B)])
    fp = engine.FastPoint(B, N, n, nseg=nseg, exponent=e, extra_radii=extra)
    fp.set_points(torch.from_numpy(clouds).cuda())
    fp.set_rng([3 + b for b in range(B)])
    fp.sample()
    fp.check()
    for b in range(B):
        ref = O.mdps(clouds[b], n, nseg=nseg, exponent=e, rng_seed=3 + b, extra_radii=extra)
        np.testing.assert_array_equal(fp.out[b].cpu().numpy(), ref.indices, err_msg=f"{variant} cloud {b}")
        assert int(fp.reached[b].item()) == ref.reached
        assert bool(fp.exhausted[b].item()) == ref.exhausted
        assert int(fp.entered[b].item()) == ref.entered
        assert int(np.int64(fp.state[b].item()).view(np.uint64)) == ref.rng_state


@pytest.mark.timeout(240)
def test_point_split_two_processes_cuda_ipc():
    """The one-process-per-GPU point split (pointsplit.PointSplitFPS): two
    processes exchange their cudaMalloc mailboxes through CUDA IPC and peer
    stores; here both live on the same GPU (their kernels alternate by
    time-slicing, hence few iterations).  Identical to the single-rank FPS on
    every rank."""
    import subprocess
    import sys as _sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IPC_N="64")
    port = 29000 + os.getpid() % 1000
    out = subprocess.run([_sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(root, "tools", "ipc_selftest.py")],
                         env=env, capture_output=True, text=True, timeout=200, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("identical to single-rank: True") == 2


@pytest.mark.timeout(300)
def test_point_split_fastpoint_two_processes():
    """pointsplit.PointSplitFastPoint over two processes (both on this GPU,
    gloo for the row transfer / broadcast / all-reduce): identical indices
    and groups to the single-process FastPoint on both ranks, with an
    early-termination tail (low exponent) running through the split FPS."""
    import subprocess
    import sys as _sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = 29500 + os.getpid() % 400
    out = subprocess.run([_sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(root, "tools", "ipc_mdps_selftest.py")],
                         capture_output=True, text=True, timeout=280, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert out.stdout.count("identical to single-process FastPoint: True") == 2
