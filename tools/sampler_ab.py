"""Time the sampler stage (FastPoint._sampler) alone on the bench batch,
median of 30 CUDA-event-timed runs from the same RNG state; run once per
library build (PS_B200_LIB) to A/B kernel variants."""
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
s0 = fp.state.clone()
fp.state.copy_(s0)
fp._prefix()
fp._thresholds()
fp._exclusion()
torch.cuda.synchronize()
ts = []
ref = None
for _ in range(int(os.environ.get("REPS", "30"))):
    fp.state.copy_(s0)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    fp._sampler()
    e[1].record()
    torch.cuda.synchronize()
    ts.append(e[0].elapsed_time(e[1]))
    if ref is None:
        ref = fp.out.clone()
    assert torch.equal(ref, fp.out)
ts.sort()
print(f"{os.environ.get('PS_B200_LIB', 'default')}: sampler {1e3 * ts[len(ts) // 2]:.1f} us (min {1e3 * ts[0]:.1f})")
