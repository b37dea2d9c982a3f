"""Time the early-termination stage (FastPoint._early_termination: prepare,
mark, push, FPS tail) alone on the bench batch, median of 30 CUDA-event
runs; run once per library build (PS_B200_LIB) to A/B K1 variants.  The
stage is idempotent (it restarts from the sampler's output)."""
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
ref = fp.out.clone()
for _ in range(3):
    fp._early_termination()
torch.cuda.synchronize()
ts = []
for _ in range(30):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    fp._early_termination()
    e[1].record()
    torch.cuda.synchronize()
    ts.append(e[0].elapsed_time(e[1]) * 1e3)
ts.sort()
same = torch.equal(fp.out, ref)
print(f"{os.environ.get('PS_B200_LIB', 'default')}: early termination {ts[15]:.1f} us (min {ts[0]:.1f}) "
      f"out identical {same}", flush=True)
