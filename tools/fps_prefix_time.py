"""Median CUDA-event time of the C3 FPS prefix (600 of 24000, B=8) and of a
full 6000-sample FPS, latency mode (and with --inflight K the throughput-hint
width); env knobs of the FPS kernels apply (A/B of development variants)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402

x = engine.as_xyz4(torch.from_numpy(bench.clouds_for(0, bench.B_PER_GPU)).cuda())
infl = int(sys.argv[sys.argv.index("--inflight") + 1]) if "--inflight" in sys.argv else None
label = os.environ.get("LABEL", "")
res = []
for stop in (600, 6000):
    for _ in range(3):
        engine.fps(x, 6000, k_stop=stop, inflight_clouds=infl)
    torch.cuda.synchronize()
    ts = []
    for _ in range(11):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        engine.fps(x, 6000, k_stop=stop, inflight_clouds=infl)
        e[1].record()
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]))
    ts.sort()
    res.append(ts[5])
print(f"{label} prefix {res[0]*1e3:.1f} us ({res[0]/599*1e3:.3f} us/it)  full {res[1]*1e3:.1f} us ({res[1]/5999*1e3:.3f} us/it)")
