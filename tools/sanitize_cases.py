"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Sizes are tiny so that the
sanitizers' per-access instrumentation finishes in seconds; each case also
checks its result against the oracle so a sanitizer-perturbed schedule that
changes a result is caught too.

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402


def _eq(a, b, msg):
    if not np.array_equal(a, b):
        raise AssertionError(msg)


def _fps(c, n, seed=0, env=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        x = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
        idx, curve, md, taken = engine.fps(x, n, seed)
        ri, rc, *_ = O.fps(c, n, seed)
        _eq(idx[0].cpu().numpy(), ri, f"fps {env}")
        _eq(curve[0].cpu().numpy(), rc, f"fps curve {env}")
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def case_fps_small():
    _fps(generate_cloud("lattice", 700, 1), 300)


def case_fps_spec():
    _fps(generate_cloud("room-surfaces", 6000, 2), 300, 5, {"PS_FPS_CLUSTER": "4", "PS_FPS_SPEC": "1"})


def case_fps_spec_p10():
    # 10 points per thread (md in shared memory, the lead's own loop): 5-CTA clusters of a 24000-point cloud
    _fps(generate_cloud("room-surfaces", 24000, 12), 200, 5, {"PS_SPEC_C": "5"})


def case_fps_cluster():
    _fps(generate_cloud("room-surfaces", 6000, 3), 300, 5, {"PS_FPS_CLUSTER": "4", "PS_FPS_NOSPEC": "1"})


def case_fps_resident():
    _fps(generate_cloud("gaussian-clusters", 6000, 4), 300, 5, {"PS_FPS_CLUSTER": "4", "PS_FPS_RESIDENT": "1"})


def case_fps_split():
    c = generate_cloud("room-surfaces", 8000, 5)
    x = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
    idx, curve, _, _ = engine.fps_split(x, 300, 3, seed_index=7)
    _eq(idx[0].cpu().numpy(), O.fps(c, 300, 7)[0], "fps_split")


def _fastpoint(B, N, n, family, env=None, extra=(0.1,)):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        clouds = np.stack([generate_cloud(family, N, 60 + b) for b in range(B)])
        fp = engine.FastPoint(B, N, n, exponent=0.45, extra_radii=extra)
        fp.set_points(torch.from_numpy(clouds).cuda())
        fp.set_rng(list(range(B)))
        fp.sample()
        fp.check()
        gi, gd, gc = fp.group_rf(extra[0], 16)
        torch.cuda.synchronize()
        for b in range(B):
            ref = O.mdps(clouds[b], n, exponent=0.45, rng_seed=b, extra_radii=extra)
            _eq(fp.out[b].cpu().numpy(), ref.indices, f"mdps {env} cloud {b}")
            oi, _, oc = O.rf_ball_query(ref.excl, extra[0], ref.indices, 16)
            _eq(gc[b].cpu().numpy().astype(np.int64), oc, "rf counts")
        return fp
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def case_mdps_smem():
    _fastpoint(2, 3000, 750, "room-surfaces")


def case_mdps_global():
    _fastpoint(1, 3000, 750, "room-surfaces", {"PS_SAMPLER_GLOBAL": "1"})


def case_mdps_sorted_csr():
    clouds = generate_cloud("uniform-box", 1500, 9)
    for method in ("bruteforce", "grid-sorted"):
        fp = engine.FastPoint(1, 1500, 400, exponent=0.45, extra_radii=(0.1,), excl_method=method)
        fp.set_points(torch.from_numpy(clouds[None]).cuda())
        fp.set_rng([3])
        fp.sample()
        fp.check()
        ref = O.mdps(clouds, 400, exponent=0.45, rng_seed=3, extra_radii=(0.1,))
        _eq(fp.out[0].cpu().numpy(), ref.indices, f"mdps {method}")


def case_grouping():
    c = generate_cloud("room-surfaces", 3000, 11)
    cent = O.fps(c, 700)[0]
    x = engine.as_xyz4(c)
    ct = torch.from_numpy(cent).cuda().reshape(1, -1)
    gi, gd, gc = engine.ball_query_naive(x, ct, 0.2, 32)
    oi, od, oc = O.ball_query_naive(c, cent, 0.2, 32)
    _eq(gi[0].cpu().numpy().astype(np.int64), oi, "bq naive")
    ki, kd, kc = engine.knn_naive(x, ct, 3)
    _eq(ki[0].cpu().numpy().astype(np.int64), O.knn_naive(c, np.arange(3000), cent, 3)[0], "knn naive")
    s = engine.min_spacing_d2(x, ct)
    _eq(s[0].cpu().numpy(), O.min_spacing_d2(c, cent), "min spacing")
    fp = _fastpoint(1, 3000, 700, "room-surfaces")
    fp.knn_rf(3)


def case_cascade():
    B, N = 3, 512
    clouds = np.stack([generate_cloud("unit-sphere", N, 70 + b) for b in range(B)])
    sa = engine.SACascade(B, N, k=16, first="fastpoint", exponent=0.5)
    sa.set_points(torch.from_numpy(clouds).cuda())
    sa.set_rng(list(range(B)))
    sa.run()
    torch.cuda.synchronize()
    ref = O.sa_cascade(clouds[0], k=16, first="fastpoint", exponent=0.5, rng_seed=0)
    _eq(sa.idx[3][0].cpu().numpy(), ref[3][0], "cascade")


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        torch.cuda.synchronize()
        print(f"case {nm}: ok", flush=True)
