"""One C4 per-GPU step (B=2 room clouds, N=65536 -> 16384, FastPoint + rf
ball query) bracketed by cudaProfilerStart/Stop for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

B, N, n = 2, 65536, 16384
clouds = np.stack([generate_cloud(bench.FAMILY, N, 3000 + b) for b in range(B)])
fp = engine.FastPoint(B, N, n, p=bench.P, nseg=bench.NSEG, estimator="power", exponent=0.536,
                      extra_radii=(bench.RADIUS,))
fp.set_points(torch.from_numpy(clouds).cuda())
fp.set_rng(list(range(B)))
fp.sample()
fp.check()
fp.group_rf(bench.RADIUS, bench.K)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fp.set_rng(list(range(B)))
fp.sample()
fp.group_rf(bench.RADIUS, bench.K)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("reached", fp.reached.tolist())
