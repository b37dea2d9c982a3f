"""Per-phase cycles of the sampler (PS_SAMPLER_TIMING=1) at C2's FastPoint
stage: B=32 unit-sphere clouds, N=1024 -> 512."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

B, N, n = 32, 1024, 512
clouds = np.stack([generate_cloud("unit-sphere", N, 2000 + b) for b in range(B)])
fp = engine.FastPoint(B, N, n, p=0.1, nseg=6, estimator="power", exponent=0.567, extra_radii=(0.15,))
fp.set_points(torch.from_numpy(clouds).cuda())
fp.set_rng(list(range(B)))
fp.sample()
fp.check()
torch.cuda.synchronize()
for env in ({}, {"PS_SAMPLER_NOTINY": "1"}):
    os.environ.pop("PS_SAMPLER_NOTINY", None)
    os.environ.update(env)
    os.environ["PS_SAMPLER_TIMING"] = "1"
    fp.set_rng(list(range(B)))
    fp._sampler()
    torch.cuda.synchronize()
    del os.environ["PS_SAMPLER_TIMING"]
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(10):
        fp.set_rng(list(range(B)))
        fp._sampler()
    e[1].record()
    torch.cuda.synchronize()
    print(env, "sampler", e[0].elapsed_time(e[1]) / 10 * 1e3, "us; reached", fp.reached.tolist()[:8],
          "entered", fp.entered.tolist()[:4], flush=True)
