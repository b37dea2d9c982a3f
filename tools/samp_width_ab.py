"""Sampler stage time (C3 bench batch, latency mode; --c4: the C4 per-GPU
share, B=2 room clouds N=65536 -> 16384) at the current PS_SAMPLER_* knobs,
median of 21 CUDA-event-timed runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402

if "--c4" in sys.argv:
    import numpy as np

    from paper_2507_23480_b200.harness import generate_cloud
    B, N, n = 2, 65536, 16384
    clouds = np.stack([generate_cloud(bench.FAMILY, N, 3000 + b) for b in range(B)])
    fp = engine.FastPoint(B, N, n, p=bench.P, nseg=bench.NSEG, estimator="power", exponent=0.536,
                          extra_radii=(bench.RADIUS,))
    fp.set_points(torch.from_numpy(clouds).cuda())
else:
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
knobs = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("PS_SAMPLER")) or "default"
print(f"{knobs}: sampler {1e3 * ts[len(ts) // 2]:.1f} us (min {1e3 * ts[0]:.1f}), same indices {ok}")
