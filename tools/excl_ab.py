"""Time the exclusion-row stage (FastPoint._exclusion) alone on the bench
batch, median of 30 CUDA-event-timed runs after the prefix and thresholds;
run once per library build (PS_B200_LIB) to A/B kernel variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402

B = bench.B_PER_GPU
fp = engine.FastPoint(B, bench.N, bench.n_SAMPLES, p=bench.P, nseg=bench.NSEG, estimator="power",
                      exponent=bench.heldout_exponent(), extra_radii=(bench.RADIUS,))
fp.set_points(torch.from_numpy(bench.clouds_for(0, B)).cuda())
fp.sample()
fp.check()
fp._prefix()
fp._thresholds()
for _ in range(3):
    fp._exclusion()
torch.cuda.synchronize()
ts = []
for _ in range(30):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    fp._exclusion()
    e[1].record()
    torch.cuda.synchronize()
    ts.append(e[0].elapsed_time(e[1]))
ts.sort()
print(f"{os.environ.get('PS_B200_LIB', 'default')}: exclusion {1e3 * ts[15]:.1f} us (min {1e3 * ts[0]:.1f})")
