"""Default dispatch vs one-sample vs no warp-per-cloud kernel, exact FPS by cloud size (B clouds, n = N/2):
us per iteration, CUDA events, to place the dispatch crossover."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

B = int(os.environ.get("B", "32"))
for N in (64, 128, 256, 512, 1024, 2048, 4096):
    import numpy as np
    c = np.stack([generate_cloud("unit-sphere", N, 7 + b) for b in range(B)])
    x = engine.as_xyz4(torch.from_numpy(c).cuda())
    row = []
    for env in ({}, {"PS_FPS_NOSPEC": "1"}, {"PS_FPS_NOWARP": "1"}):
        os.environ.pop("PS_FPS_NOSPEC", None)
        os.environ.pop("PS_FPS_NOWARP", None)
        os.environ.update(env)
        engine.fps(x, N // 2)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(3):
            engine.fps(x, N // 2)
        e[1].record()
        torch.cuda.synchronize()
        row.append(e[0].elapsed_time(e[1]) / 3 * 1e3 / (N // 2 - 1))
    os.environ.pop("PS_FPS_NOSPEC", None)
    os.environ.pop("PS_FPS_NOWARP", None)
    print(f"B={B} N={N:6d}: default {row[0]:.3f} us/it, one-sample {row[1]:.3f}, without warp kernel {row[2]:.3f}", flush=True)
