"""rf ball query alone on the C3 bench batch (r = 0.1, k = 32), median of 30
CUDA-event-timed runs; PS_BQ_RF_WARP=1 selects the warp-per-centroid kernel."""
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
out = (torch.empty(B, bench.n_SAMPLES, bench.K, dtype=torch.int32, device="cuda"),
       torch.empty(B, bench.n_SAMPLES, bench.K, dtype=torch.float64, device="cuda"),
       torch.empty(B, bench.n_SAMPLES, dtype=torch.int32, device="cuda"))
for _ in range(3):
    fp.group_rf(bench.RADIUS, bench.K, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    fp.group_rf(bench.RADIUS, bench.K, out=out)
    e[1].record()
    torch.cuda.synchronize()
    ts.append(e[0].elapsed_time(e[1]))
ts.sort()
print(f"{'warp' if os.environ.get('PS_BQ_RF_WARP') else 'pair'}: rf ball query {1e3 * ts[15]:.1f} us (min {1e3 * ts[0]:.1f}), "
      f"checksum {int(out[0].sum())} {float(out[1].nan_to_num(0).sum()):.6f} {int(out[2].sum())}")
