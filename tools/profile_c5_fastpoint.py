"""C5 FastPoint (2^20 -> 65536, uniform box, one GPU): per-stage device
times of one eager run, then one more run bracketed by
cudaProfilerStart/Stop for an ncu launch list (--profile-from-start off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

N, n = bench.C5_N, bench.C5_n
c = generate_cloud("uniform-box", N, 5000)
fp = engine.FastPoint(1, N, n, exponent=bench.C5_EXPONENT, extra_radii=(bench.C5_RADIUS,))
fp.set_points(torch.from_numpy(c[None]).cuda())
seed = torch.zeros(1, dtype=torch.int64, device="cuda")
names = ["fps_prefix", "thresholds", "excl_build", "sampler", "early_term", "rf_ball_query"]
for rep in range(3):
    fp.state.copy_(seed)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record()
    fp._prefix(); ev[1].record()
    fp._thresholds(); ev[2].record()
    fp._exclusion(); ev[3].record()
    fp._sampler(); ev[4].record()
    fp._early_termination(); ev[5].record()
    fp.group_rf(bench.C5_RADIUS, 32); ev[6].record()
    torch.cuda.synchronize()
    fp.check()
    print("stages ms:", {nm: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, nm in enumerate(names)}, flush=True)
print("reached", int(fp.reached[0]), "stride", fp.csr.stride, "cap", fp.csr.cap_entries, flush=True)
torch.cuda.cudart().cudaProfilerStart()
fp.state.copy_(seed)
fp.sample()
fp.group_rf(bench.C5_RADIUS, 32)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
