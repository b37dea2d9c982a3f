"""SPEC acceptance properties on the GPU path: A3 sampling
quality, A4 segment-count trend, A6 step-function guarantee, A9 early-
termination share and the overestimating-estimator case, A10 curve
monotonicity.  (A1, A2, A7 and A8 are covered bit-exactly against the oracle
in test_gpu_parity.py / test_oracle_golden.py.)"""

import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2507_23480_b200 import curve, engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

N, STRIDE = 10000, 4
n = N // STRIDE


def batch(family, seeds):
    return torch.from_numpy(np.stack([generate_cloud(family, N, s) for s in seeds])).cuda()


def spacing(xyz4, idx):
    return engine.min_spacing_d2(xyz4, idx).sqrt().mean(dim=1)


def fastpoint(x, estimator, nseg=6, exponent=None, curves=None, seed=0):
    B = x.shape[0]
    fp = engine.FastPoint(B, N, n, nseg=nseg, estimator=estimator, exponent=exponent)
    fp.set_points(x)
    fp.set_rng([seed + b for b in range(B)])
    if curves is not None:
        fp.set_curve(curves)
    fp.sample()
    fp.check()
    return fp


@pytest.fixture(scope="module", params=["uniform-box", "room-surfaces"])
def family_set(request):
    fam = request.param
    x = batch(fam, range(500, 505))
    xyz4 = engine.as_xyz4(x)
    idx, cv, _, _ = engine.fps(xyz4, n)
    held = engine.as_xyz4(batch(fam, range(600, 605)))
    _, hcv, _, _ = engine.fps(held, n)
    e = curve.fit_power_exponent(hcv.cpu().numpy())  # 5 held-out clouds of the family (A3)
    return fam, x, xyz4, idx, cv, e


def test_a3_a4_a9_quality_segments_and_early_termination(family_set):
    fam, x, xyz4, idx, cv, e = family_set
    base = spacing(xyz4, idx)
    # A3: oracle estimator (the true FPS curve), nseg = 6 -> >= 97 %
    fo = fastpoint(x, "curve", curves=cv.cpu().numpy())
    q_oracle = (spacing(xyz4, fo.out) / base).cpu().numpy()
    assert np.all(q_oracle >= 0.97), (fam, q_oracle)
    # A3: power estimator, exponent fitted on 5 held-out clouds -> >= 93 %
    fpw = fastpoint(x, "power", exponent=e)
    q_power = (spacing(xyz4, fpw.out) / base).cpu().numpy()
    assert np.all(q_power >= 0.93), (fam, e, q_power)
    # A4: nseg = 6 at least as good as nseg = 1 per cloud (0.2 % noise floor)
    f1 = fastpoint(x, "curve", nseg=1, curves=cv.cpu().numpy())
    q1 = (spacing(xyz4, f1.out) / base).cpu().numpy()
    assert np.all(q_oracle >= q1 - 0.002), (fam, q_oracle, q1)
    # A9: early termination <= 10 % of n with the oracle estimator
    et = (n - fo.reached.cpu().numpy()) / n
    assert np.all(et <= 0.10), (fam, et)
    # A9: a 2x-overestimating estimator still yields n distinct indices
    f2 = fastpoint(x, "curve", curves=2.0 * cv.cpu().numpy())
    out = f2.out.cpu().numpy()
    for b in range(out.shape[0]):
        assert len(np.unique(out[b])) == n and out[b].min() >= 0 and out[b].max() < N
    assert np.any(f2.reached.cpu().numpy() < n)  # the fallback did run


def test_a10_fps_curves_non_increasing(family_set):
    fam, _, _, _, cv, _ = family_set
    c = cv.cpu().numpy()
    assert np.all(np.isinf(c[:, 0]))
    assert np.all(c[:, 2:] <= c[:, 1:-1]), fam


@pytest.mark.parametrize("family,Nc,nc,e", [("uniform-box", 2000, 500, 0.4), ("room-surfaces", 1800, 450, 0.45),
                                              ("lattice", 1728, 432, 0.6)])
def test_a6_step_function_guarantee(family, Nc, nc, e):
    """Every sample taken by the predicted-distance sampler in segment s lies
    at distance >= R_s from all earlier samples (brute force, float64, the
    strict `<` exclusion predicate).  Segments only advance with the sample
    position or earlier (pool exhausted), so a sample at position t was taken
    in some segment s(t) >= seg_pos(t), non-decreasing in t, with at most
    entered - 1 advances: the check finds the latest such assignment that
    explains every sample and requires it to exist."""
    c = generate_cloud(family, Nc, 11)
    fp = engine.FastPoint(1, Nc, nc, exponent=e)
    fp.set_points(torch.from_numpy(c[None]).cuda())
    fp.set_rng([5])
    fp.sample()
    fp.check()
    out = fp.out[0].cpu().numpy()
    reached = int(fp.reached[0].item())
    R = fp.R[0].cpu().numpy()
    r2 = np.array([O.radius_sq(float(v)) for v in R])
    bnd = curve.sampler_boundaries(nc, len(R))
    k0 = fp.k0
    x, y, z = O.columns_f64(c)
    s_cur = 0
    for t in range(k0, reached):
        while s_cur < len(R) - 1 and t >= bnd[s_cur]:
            s_cur += 1
        j = out[t]
        prev = out[:t]
        d2 = (x[prev] - x[j]) ** 2 + (y[prev] - y[j]) ** 2 + (z[prev] - z[j]) ** 2
        dmin = d2.min()
        # the sample lies outside every earlier sample's level-s ball
        while dmin < r2[s_cur]:
            s_cur += 1  # it can only have been taken in a later segment
            assert s_cur < len(R), f"sample {t} (index {j}) violates every segment radius"
    assert s_cur + 1 <= int(fp.entered[0].item())
