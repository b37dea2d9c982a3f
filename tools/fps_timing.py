"""Per-phase cycle breakdown of the cluster FPS iteration (PS_FPS_TIMING=1)."""
import os
import sys

os.environ["PS_FPS_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402
import numpy as np  # noqa: E402

for N, B, C in ((24000, 8, None), (24000, 8, 8), (4096, 1, None), (1024, 32, None), (65536, 2, None)):
    if C:
        os.environ["PS_FPS_CLUSTER"] = str(C)
    else:
        os.environ.pop("PS_FPS_CLUSTER", None)
    clouds = np.stack([generate_cloud("room-surfaces", N, b) for b in range(B)])
    x = engine.as_xyz4(torch.from_numpy(clouds).cuda())
    for _ in range(2):
        engine.fps(x, min(N // 4, 2000))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    os.environ.pop("PS_FPS_TIMING")
    ev[0].record()
    engine.fps(x, min(N // 4, 2000))
    ev[1].record()
    torch.cuda.synchronize()
    os.environ["PS_FPS_TIMING"] = "1"
    it = min(N // 4, 2000) - 1
    print(f"N={N} B={B} C={C}: {ev[0].elapsed_time(ev[1]) * 1e3 / it:.3f} us/iter", flush=True)
