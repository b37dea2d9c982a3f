"""One C2 set-abstraction cascade (B=32, N=1024, FastPoint first) bracketed
by cudaProfilerStart/Stop for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

first = sys.argv[1] if len(sys.argv) > 1 else "fastpoint"
B, N = 32, 1024
clouds = np.stack([generate_cloud("unit-sphere", N, 2000 + b) for b in range(B)])
sa = engine.SACascade(B, N, first=first, exponent=0.567, device="cuda")
sa.set_points(torch.from_numpy(clouds).cuda())
sa.set_rng(list(range(B)))
sa.run()
if first == "fastpoint":
    sa.fp.check()
sa.run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sa.run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
