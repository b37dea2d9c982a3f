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
                                 100, None, 0, None, None, None, None, None)
    assert rc == _lib.PS_ERR_INVALID
    assert b"last segment boundary" in lib.ps_last_error()
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
