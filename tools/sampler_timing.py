"""Per-phase cycles of the bitmap sampler at the bench workload (PS_SAMPLER_TIMING=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402

B = bench.B_PER_GPU
clouds = bench.clouds_for(0, B)
fp = engine.FastPoint(B, bench.N, bench.n_SAMPLES, exponent=bench.heldout_exponent(), extra_radii=(bench.RADIUS,))
fp.set_points(torch.from_numpy(clouds).cuda())
fp.set_rng(list(range(B)))
fp.sample()
torch.cuda.synchronize()
os.environ["PS_SAMPLER_TIMING"] = "1"
fp.set_rng(list(range(B)))
fp._sampler()
torch.cuda.synchronize()
print("reached", fp.reached.tolist(), "entered", fp.entered.tolist())
