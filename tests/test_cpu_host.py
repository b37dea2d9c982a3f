"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
argument validation works without a device, host-side helpers agree with the
oracle, and the product package never reaches into oracle/."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_23480_b200 import _lib, core, curve, harness

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(REPO, "include", "ps_b200.h")).read()
    return sorted(set(re.findall(r"PS_API\s+[\w\s\*]+?\b(ps_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.ps_version() == 1


def test_validation_without_device():
    lib = _lib.load()
    # B = 0 is rejected before any CUDA call
    rc = lib.ps_fps(None, 0, 10, None, None, None, None, 10, 5, 0, None, None)
    assert rc == _lib.PS_ERR_INVALID
    assert b"invalid batch shape" in lib.ps_last_error()
    rows = np.zeros(6, np.int32)
    bnd = np.array([1, 2, 3, 4, 5, 9], np.int64)  # last != n_total
    rc = lib.ps_sample_predicted(None, None, 0, None, 6, rows.ctypes.data, bnd.ctypes.data, 6, None, 10, 2, 10, 1,
                                 100, None, 0, None, None, None, None, None, None)
    assert rc == _lib.PS_ERR_INVALID
    assert b"last segment boundary" in lib.ps_last_error()
    # rf ball query: the per-warp top-k lists hold 128 entries
    rc = lib.ps_ball_query_rf(None, None, None, 0, None, 7, 6, None, 1, 1, 100, 10, 200, None, None, None, None, None)
    assert rc == _lib.PS_ERR_INVALID and b"k must be in [1, 128]" in lib.ps_last_error()
    # method-2 rows: 16-byte aligned stride, about 1/9 of the capacity left as spill arena
    for N, per in ((24000, 216), (1000, 100), (7, 3)):
        st = lib.ps_excl_row_stride(N, N * per)
        assert st <= per * 8 // 9 and (st % 4 == 0 or st < 4) and N * per - N * st >= N * per // 9 - N
    assert lib.ps_excl_workspace_bytes(2, 100, 50, 0) > 0 and lib.ps_excl_workspace_bytes(2, 100, 1, 1) > 0
    assert 0 < lib.ps_sampler_workspace_bytes(1, 24000, 6) < lib.ps_sampler_workspace_bytes(1, 40000, 6) / 1.5
    assert lib.ps_sampler_workspace_bytes(2, 100000, 6) > 2 * lib.ps_sampler_workspace_bytes(1, 100000, 6) * 0.99


def test_curve_helpers_match_oracle():
    rng = np.random.default_rng(0)
    for n, p, e in ((1024, 0.1, 0.4), (6000, 0.1, 0.45), (300, 0.2, 1.3), (37, 0.3, 0.0)):
        k0 = curve.prefix_len(n, p)
        assert k0 == O.prefix_len(n, p)
        pre = np.concatenate([[math.inf], np.sort(rng.random(k0 - 1))[::-1] + 0.1])
        np.testing.assert_array_equal(curve.estimate_power(pre, n, e), O.estimate_power(pre, n, e))
        est = O.estimate_power(pre, n, e)
        for nseg in (1, 3, 6):
            d, R = curve.segment_thresholds(est, nseg)
            d2, R2 = O.segment_thresholds(est, nseg)
            np.testing.assert_array_equal(d, d2)
            np.testing.assert_array_equal(R, R2)
            np.testing.assert_array_equal(curve.sampler_boundaries(n, nseg), O.sampler_boundaries(n, nseg))
    assert curve.radius_sq(0.0) == O.radius_sq(O.clamp_radius(0.0)) == 5e-324
    i = np.arange(65, dtype=np.float64)
    assert abs(curve.fit_power_exponent([2.0 / np.maximum(i, 1)]) - 1.0) < 1e-9
    np.testing.assert_array_equal(curve.resample_curve([4, 2], 3), [4, 3, 2])
    assert curve.estimator_mape([np.inf, 1, 1, 2, 2], [np.inf, 1, 1, 2, 4], 0.4) == 25.0


def test_core_api():
    r = core.Rng(0)
    assert [r.next_u64() for _ in range(3)] == O.sm64_stream(0, 3)
    assert [core.Rng(1).below(10) for _ in range(1)] == [5]
    r = core.Rng(1)
    assert [r.below(10) for _ in range(5)] == [5, 9, 0, 5, 1]
    with pytest.raises(ValueError):
        core.PointCloud(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        core.PointCloud([[0, 0, np.nan]])
    pc = core.PointCloud([[0, 0, 0], [1, 2, 2]])
    assert not pc.coords.flags.writeable
    core.reset_pair_evals()
    assert core.squared_distance((0, 0, 0), (1, 2, 2)) == 9 and core.pair_evals() == 1
    with core.workers(4):
        assert core.get_workers() == 4
    assert core.get_workers() == 1


def test_cloud_io_roundtrip(tmp_path):
    c = core.PointCloud(harness.generate_cloud("uniform-box", 50, 1))
    for ext in (".pcf", ".xyz"):
        p = str(tmp_path / f"c{ext}")
        core.save_cloud(c, p)
        np.testing.assert_array_equal(core.load_cloud(p).coords, c.coords)
    bad = tmp_path / "bad.xyz"
    bad.write_text("0 0 abc\n")
    with pytest.raises(core.CloudFormatError, match="line 1"):
        core.load_cloud(str(bad))
    core.write_indices_csv(str(tmp_path / "i.csv"), [3, 1, 2])
    assert core.read_indices_csv(str(tmp_path / "i.csv")).tolist() == [3, 1, 2]


def test_harness_families_deterministic():
    for fam in harness.FAMILIES:
        a = harness.generate_cloud(fam, 1000, 5)
        b = harness.generate_cloud(fam, 1000, 5)
        assert a.dtype == np.float32 and a.shape == (1000, 3)
        np.testing.assert_array_equal(a, b)
        assert np.isfinite(a).all()
    u = harness.generate_cloud("uniform-box", 10000, 0)
    assert u.min() >= 0 and u.max() <= 1
    lid = harness.generate_cloud("lidar-rings", 20000, 0)
    r = np.hypot(lid[:, 0], lid[:, 1])
    area_density = np.histogram(r, bins=[2, 10, 20, 30, 45])[0] / np.diff(np.array([2, 10, 20, 30, 45]) ** 2)
    assert np.all(np.diff(area_density) < 0)


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2507_23480_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "ps_oracle" not in txt, f


# ---- MLP estimator host pieces (A8) --------------------------

def test_resample_curve_spec_examples():
    from paper_2507_23480_b200 import curve as Cv

    np.testing.assert_array_equal(Cv.resample_curve([4, 2], 3), [4, 3, 2])
    np.testing.assert_array_equal(Cv.resample_curve([4, 3, 2, 1], 4), [4, 3, 2, 1])
    r = Cv.resample_curve(np.arange(10.0), 32)                                        # SPEC.md:296 (affine)
    assert np.max(np.abs(r - np.linspace(0.0, 9.0, 32))) < 1e-13
    v = np.random.default_rng(0).random(17)
    assert Cv.resample_curve(v, 5)[0] == v[0] and Cv.resample_curve(v, 5)[-1] == v[-1]
    with pytest.raises(ValueError):
        Cv.resample_curve([1.0], 4)


def test_mlp_model_file_roundtrip_and_zero_model(tmp_path):
    from paper_2507_23480_b200 import curve as Cv

    m = Cv.MlpModel.init(np.random.default_rng(4))
    m.save(tmp_path / "m.txt")
    m2 = Cv.MlpModel.load(tmp_path / "m.txt")
    for a, b in zip(m.W + m.b, m2.W + m2.b):
        np.testing.assert_array_equal(a, b)
    assert open(tmp_path / "m.txt").readline().strip() == "MLP 32 128 128 64"
    z = Cv.MlpModel(*[np.zeros_like(a) for k in range(3) for a in (m.W[k], m.b[k])])
    np.testing.assert_array_equal(Cv.mlp_forward_exact(z, np.ones(32)), np.zeros(64))


def test_mlp_gradients_match_finite_differences():
    """SPEC.md:276 / A8(ii): every layer's gradient within 1e-4 relative of
    central differences (eps = 1e-3)."""
    from paper_2507_23480_b200 import curve as Cv

    rng = np.random.default_rng(7)
    m = Cv.MlpModel.init(rng)
    for k in range(3):
        m.b[k] = rng.normal(0, 0.1, m.b[k].shape)
    x, y = rng.normal(size=32), rng.normal(size=64)
    _, g = Cv.mlp_loss_grad(m, x, y)
    eps = 1e-3
    for k in range(3):
        for (r, c) in ((0, 0), (5, 7), (m.W[k].shape[0] - 1, m.W[k].shape[1] - 1)):
            w0 = m.W[k][r, c]
            m.W[k][r, c] = w0 + eps
            lp, _ = Cv.mlp_loss_grad(m, x, y)
            m.W[k][r, c] = w0 - eps
            lm, _ = Cv.mlp_loss_grad(m, x, y)
            m.W[k][r, c] = w0
            fd = (lp - lm) / (2 * eps)
            an = g[2 * k][r, c]
            assert abs(fd - an) <= 1e-4 * max(abs(fd), abs(an), 1e-8), (k, r, c, fd, an)


def test_mlp_train_overfit_determinism_and_zero_lr():
    from paper_2507_23480_b200 import curve as Cv

    c = np.concatenate([[np.inf], 2.0 / np.arange(1, 400) ** 0.6])
    pair = Cv.mlp_pair(c)
    m0 = Cv.MlpModel.init(np.random.default_rng(1))
    l0, _ = Cv.mlp_loss_grad(m0, *pair)
    m1, losses = Cv.mlp_train([pair], epochs=200, lr=0.01, rng=np.random.default_rng(1))
    assert losses[-1] * 10 <= l0
    m2, _ = Cv.mlp_train([pair], epochs=200, lr=0.01, rng=np.random.default_rng(1))
    for a, b in zip(m1.W + m1.b, m2.W + m2.b):
        np.testing.assert_array_equal(a, b)
    m3, _ = Cv.mlp_train([pair], epochs=3, lr=0.0, rng=np.random.default_rng(1))
    for a, b in zip(m0.W + m0.b, m3.W + m3.b):
        np.testing.assert_array_equal(a, b)


def test_estimate_mlp_matches_oracle_and_is_scale_equivariant():
    from oracle import oracle as O
    from paper_2507_23480_b200 import curve as Cv

    m = Cv.MlpModel.init(np.random.default_rng(9))
    prefix = np.concatenate([[np.inf], 3.0 / np.arange(1, 60) ** 0.5])
    import tempfile
    p = tempfile.mktemp()
    m.save(p)
    est = Cv.estimate_mlp(prefix, 600, m)
    np.testing.assert_array_equal(est, O.estimate_mlp(prefix, 600, O.read_mlp(p)))
    np.testing.assert_array_equal(est[:60], prefix)
    assert np.all(np.diff(est[59:]) <= 0)
    est2 = Cv.estimate_mlp(2 * prefix, 600, m)
    np.testing.assert_allclose(est2[60:], 2 * est[60:], rtol=1e-12)


def test_random_and_grid_samplers_spec_examples():
    """SPEC.md:144-171 comparison samplers (host utilities)."""
    from paper_2507_23480_b200 import baselines, core

    cube = np.array([[x, y, z] for x in (0, 1) for y in (0, 1) for z in (0, 1)], np.float32)
    assert len(baselines.grid_sample(cube, 2.0).indices) == 1
    assert sorted(baselines.grid_sample(cube, 0.5).indices.tolist()) == list(range(8))
    two = np.array([[0, 0, 0], [0.1, 0, 0]], np.float32)
    assert baselines.grid_sample(two, 1.0).indices.tolist() == [0]
    with pytest.raises(ValueError):
        baselines.grid_sample(cube, 0.0)
    c = np.random.default_rng(0).random((100, 3), dtype=np.float32)
    r1 = baselines.random_sample(c, 10, core.Rng(5)).indices
    r2 = baselines.random_sample(c, 10, core.Rng(5)).indices
    assert r1.tolist() == r2.tolist() and len(set(r1.tolist())) == 10
    assert sorted(baselines.random_sample(c, 100, core.Rng(1)).indices.tolist()) == list(range(100))
    with pytest.raises(ValueError):
        baselines.random_sample(c, 0, core.Rng(1))
    u = np.random.default_rng(2).random((10000, 3), dtype=np.float32)
    g = baselines.grid_sample_to_count(u, 2500, 0.05)
    assert 2375 <= len(g.indices) <= 2625
    assert baselines.grid_sample_to_count(u[:1], 1).indices.tolist() == [0]


def test_pointsample_import_alias():
    """The reference package name resolves to the B200 modules (drop-in swap
    by import path, pkg/pyproject.toml:6)."""
    import importlib

    ps = importlib.import_module("pointsample")
    from paper_2507_23480_b200 import _kernels as K
    from paper_2507_23480_b200 import core as C

    assert importlib.import_module("pointsample._kernels") is K
    assert ps.core is C
    for name in ("fps_loop", "fps_update_chunk", "first_untaken", "excl_collect", "csr_fill", "csr_sort_rows",
                 "csr_level_counts", "sample_predicted", "earlyterm_scan"):
        assert callable(getattr(K, name)), name
    from pointsample.mdps import early_termination, mdps, sample_with_predicted_distance  # noqa: F401
    from pointsample.curve import extract_prefix, segment_thresholds  # noqa: F401
