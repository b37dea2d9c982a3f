"""Time the thresholds stage (FastPoint._thresholds, K2) alone on the bench
batch and on C2's FastPoint stage, median of 50 CUDA-event runs; run once per
library build (PS_B200_LIB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

cases = {"C3": (bench.clouds_for(0, bench.B_PER_GPU), bench.n_SAMPLES, bench.heldout_exponent()),
         "C2": (np.stack([generate_cloud("unit-sphere", 1024, 2000 + b) for b in range(32)]), 512, 0.567)}
for name, (clouds, n, e) in cases.items():
    B, N = clouds.shape[:2]
    fp = engine.FastPoint(B, N, n, p=0.1, nseg=6, estimator="power", exponent=e, extra_radii=(0.1,))
    fp.set_points(torch.from_numpy(clouds).cuda())
    fp.sample()
    fp.check()
    R = fp.R.clone()
    ts = []
    for _ in range(50):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        fp._thresholds()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    ts.sort()
    print(f"{os.environ.get('PS_B200_LIB', 'default')[-20:]} {name}: thresholds {ts[25]:.1f} us (min {ts[0]:.1f}) "
          f"R identical {torch.equal(fp.R, R)}", flush=True)
