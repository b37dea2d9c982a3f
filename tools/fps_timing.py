"""Per-phase cycle breakdown of the cluster FPS iteration (PS_FPS_TIMING=1; needs
a library built with `make -C paper_2507_23480_b200/csrc TIMING=1`).

  python tools/fps_timing.py [N B n] ...   (env PS_FPS_CLUSTER / PS_FPS_THREADS honoured)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

cases = [(24000, 8, 6000), (4096, 1, 1024), (1024, 32, 512), (65536, 2, 2000)]
if len(sys.argv) >= 4:
    cases = [tuple(int(v) for v in sys.argv[1:4])]
for N, B, n in cases:
    clouds = np.stack([generate_cloud("room-surfaces", N, b) for b in range(B)])
    x = engine.as_xyz4(torch.from_numpy(clouds).cuda())
    os.environ.pop("PS_FPS_TIMING", None)
    for _ in range(2):
        engine.fps(x, n)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    engine.fps(x, n)
    ev[1].record()
    torch.cuda.synchronize()
    os.environ["PS_FPS_TIMING"] = "1"
    engine.fps(x, min(n, 2000) if os.environ.get("PS_FPS_LATE") else min(n, 300))
    torch.cuda.synchronize()
    print(f"N={N} B={B} n={n} C={os.environ.get('PS_FPS_CLUSTER', 'auto')} T={os.environ.get('PS_FPS_THREADS', '256')}: "
          f"{ev[0].elapsed_time(ev[1]) * 1e3 / (n - 1):.3f} us/iter (full run)", flush=True)
