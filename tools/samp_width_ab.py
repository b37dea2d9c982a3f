"""Sampler stage time (C3 bench batch, latency mode) at the current
PS_SAMPLER_CLUSTER width, median of 21 CUDA-event-timed runs."""
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
fp.set_rng(list(range(B)))
fp.sample()
fp.check()
ref = fp.out.clone()
ts = []
for k in range(24):
    fp.set_rng(list(range(B)))
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    fp._sampler()
    e[1].record()
    torch.cuda.synchronize()
    if k >= 3:
        ts.append(e[0].elapsed_time(e[1]))
fp.set_rng(list(range(B)))
fp.sample()
torch.cuda.synchronize()
ok = torch.equal(fp.out, ref)
ts.sort()
print(f"C={os.environ.get('PS_SAMPLER_CLUSTER', 'default')}: sampler {1e3 * ts[len(ts) // 2]:.1f} us (min {1e3 * ts[0]:.1f}), same indices {ok}")
