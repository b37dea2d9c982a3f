"""Config C5 on one GPU (BASELINE.json configs[4]: one cloud, N = 2^20 ->
65536): exact FPS and the whole FastPoint path at full size against the
oracle digests of tests/golden/c5_digest.json (tests/golden/make_c5_digest.py
ran the oracle with the reference's worker split), and FastPoint at
N = 2^18 -> 16384 against the live oracle as well.

The large cloud runs ps_fps as the point split over virtual ranks (the
prefix and the early-termination tail), the grid exclusion build with
fixed-stride rows and a spill arena, the global-memory sampler tables and
the rf ball query -- the single-GPU shape of SURVEY.md 8e's MDPS at C5."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DIG = json.load(open(os.path.join(HERE, "golden", "c5_digest.json")))
PRM = DIG["fastpoint_params"]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_fastpoint(cloud, n, exponent, graph=False):
    N = cloud.shape[0]
    fp = engine.FastPoint(1, N, n, p=PRM["p"], nseg=PRM["nseg"], exponent=exponent, extra_radii=(PRM["radius"],))
    fp.set_points(torch.from_numpy(cloud[None]).cuda())
    fp.set_rng([PRM["rng_seed"]])
    fp.sample()
    fp.check()
    if graph:  # replay a captured graph of the same sequence
        fp.capture()
        fp.set_rng([PRM["rng_seed"]])
        fp.out.fill_(-7)
        fp.sample()
    gi, gd, gc = fp.group_rf(PRM["radius"], PRM["k"])
    torch.cuda.synchronize()
    return fp, gi[0].cpu().numpy().astype(np.int64), gc[0].cpu().numpy().astype(np.int64)


def check_digest(fp, gi, gc, d):
    idx = fp.out[0].cpu().numpy()
    np.testing.assert_array_equal(idx[:16], d["idx_head"])
    np.testing.assert_array_equal(idx[-16:], d["idx_tail"])
    assert sha(idx.astype(np.int64)) == d["idx_sha256"]
    assert int(fp.reached[0].item()) == d["reached"]
    assert int(fp.entered[0].item()) == d["entered"]
    assert bool(fp.exhausted[0].item()) == d["exhausted"]
    np.testing.assert_array_equal(fp.R[0].cpu().numpy(), np.array(d["R"]))
    assert str(int(np.int64(fp.state[0].item()).view(np.uint64))) == d["rng_state"]
    k = PRM["k"]
    members = np.where(np.arange(k)[None, :] < gc[:, None], gi, -1).astype(np.int64)
    assert int(gc.sum()) == d["rf_cnt_sum"]
    assert sha(gc) == d["rf_cnt_sha256"]
    assert sha(members) == d["rf_idx_sha256"]


@pytest.mark.timeout(600)
def test_c5_exact_fps_matches_oracle_digest():
    c = DIG["c5"]
    cloud = generate_cloud(c["family"], c["N"], c["cloud_seed"])
    x = engine.as_xyz4(torch.from_numpy(cloud[None]).cuda())
    idx, curve, _, _ = engine.fps(x, c["n"], c["seed_index"])
    d = DIG["exact_fps"]
    got = idx[0].cpu().numpy()
    np.testing.assert_array_equal(got[:16], d["idx_head"])
    np.testing.assert_array_equal(got[-16:], d["idx_tail"])
    assert sha(got.astype(np.int64)) == d["idx_sha256"]
    assert sha(curve[0].cpu().numpy().astype(np.float64)) == d["curve_sha256"]


@pytest.mark.timeout(900)
def test_fastpoint_2e18_matches_live_oracle_and_digest():
    m = DIG["mid"]
    cloud = generate_cloud(m["family"], m["N"], m["cloud_seed"])
    fp, gi, gc = run_fastpoint(cloud, m["n"], PRM["mid_exponent"])
    check_digest(fp, gi, gc, m["fastpoint"])
    old = O.set_threads(os.cpu_count() or 1)
    try:
        ref = O.mdps(cloud, m["n"], p=PRM["p"], nseg=PRM["nseg"], exponent=PRM["mid_exponent"],
                     rng_seed=PRM["rng_seed"], extra_radii=(PRM["radius"],))
        oi, _, oc = O.rf_ball_query(ref.excl, PRM["radius"], ref.indices, PRM["k"])
    finally:
        O.set_threads(old)
    np.testing.assert_array_equal(fp.out[0].cpu().numpy(), ref.indices)
    np.testing.assert_array_equal(gc, oc)
    for t in range(0, m["n"], 97):
        np.testing.assert_array_equal(gi[t, :gc[t]], oi[t, :oc[t]])


@pytest.mark.timeout(900)
@pytest.mark.parametrize("graph", [False, True])
def test_fastpoint_c5_matches_oracle_digest(graph):
    c = DIG["c5"]
    cloud = generate_cloud(c["family"], c["N"], c["cloud_seed"])
    fp, gi, gc = run_fastpoint(cloud, c["n"], PRM["exponent"], graph=graph)
    check_digest(fp, gi, gc, DIG["fastpoint"])


@pytest.mark.timeout(900)
@pytest.mark.parametrize("case", ["room-24k-G3", "dup-spill-G5", "mid-2e18-G4"])
def test_fastpoint_point_split_matches_single_rank_and_oracle(case):
    """MDPS with every cloud point-split over G virtual ranks (split prefix,
    row-sharded exclusion build with per-rank spill arenas, sampler over the
    joined rows, per-rank early-termination seeding + split FPS tail,
    centroid-sharded rf grouping): identical to the single-rank FastPoint
    and to the oracle."""
    if case == "mid-2e18-G4":
        m = DIG["mid"]
        cloud = generate_cloud(m["family"], m["N"], m["cloud_seed"])
        n, e, G, r = m["n"], PRM["mid_exponent"], 4, PRM["radius"]
    elif case == "room-24k-G3":
        cloud = generate_cloud("room-surfaces", 24000, 77)
        n, e, G, r = 6000, 0.2, 3, 0.1  # low exponent: long early-termination tail
    else:
        cloud = generate_cloud("uniform-box", 30000, 78)
        cloud[:400] = cloud[0]  # dense duplicates: long rows spill
        cloud = cloud[np.random.default_rng(0).permutation(30000)].copy()
        n, e, G, r = 4000, 0.45, 5, 0.05
    B, N = 1, cloud.shape[0]
    seed = PRM["rng_seed"] if case == "mid-2e18-G4" else 3
    fs = engine.FastPointSplit(B, N, n, G, exponent=e, extra_radii=(r,))
    fs.set_points(torch.from_numpy(cloud[None]).cuda())
    fs.set_rng([seed])
    fs.sample()
    fs.check()
    si, sd, sc = fs.group_rf(r, 32)
    fp = engine.FastPoint(B, N, n, exponent=e, extra_radii=(r,))
    fp.set_points(torch.from_numpy(cloud[None]).cuda())
    fp.set_rng([seed])
    fp.sample()
    fp.check()
    gi, gd, gc = fp.group_rf(r, 32)
    torch.cuda.synchronize()
    assert torch.equal(fs.out, fp.out)
    assert torch.equal(fs.reached, fp.reached) and torch.equal(fs.state, fp.state)
    assert torch.equal(sc, gc) and torch.equal(si, gi)
    assert torch.equal(torch.nan_to_num(sd, nan=-1.0), torch.nan_to_num(gd, nan=-1.0))
    if case == "mid-2e18-G4":
        check_digest(fs, si[0].cpu().numpy().astype(np.int64), sc[0].cpu().numpy().astype(np.int64),
                     DIG["mid"]["fastpoint"])
    else:
        ref = O.mdps(cloud, n, exponent=e, rng_seed=3, extra_radii=(r,))
        np.testing.assert_array_equal(fs.out[0].cpu().numpy(), ref.indices)
        if case == "room-24k-G3":
            assert ref.reached < n  # the split tail ran
        else:
            stride = fs.csr.stride
            assert int(fs.csr.counts[0].amax(dim=0).max()) > stride  # spilled rows
