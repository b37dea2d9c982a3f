"""Small-cloud exact FPS: warps per cloud (PS_FPS_SMALL_W) sweep vs the
kernels without fps_small (PS_FPS_NOSMALL): us per iteration, CUDA events over graph replays,
n = N/2 samples, B clouds (env B, default 32)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

B = int(os.environ.get("B", "32"))


def timed(x, n, env):
    for k in ("PS_FPS_SMALL_W", "PS_FPS_NOSMALL", "PS_FPS_SPEC"):
        os.environ.pop(k, None)
    os.environ.update(env)
    ref = engine.fps(x, n)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # graph replay: no host overhead in the timing
    with torch.cuda.graph(g):
        got = engine.fps(x, n)
    g.replay()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(10):
        g.replay()
    e[1].record()
    torch.cuda.synchronize()
    assert all(torch.equal(u, v) for u, v in zip(got, ref))
    return e[0].elapsed_time(e[1]) / 10 * 1e3 / (n - 1), got


for N in (128, 256, 512, 1024, 2048, 4096):
    c = np.stack([generate_cloud("unit-sphere", N, 7 + b) for b in range(B)])
    x = engine.as_xyz4(torch.from_numpy(c).cuda())
    base, ref = timed(x, N // 2, {"PS_FPS_NOSMALL": "1"})
    cols = [f"without {base:.3f}"]
    t, got = timed(x, N // 2, {"PS_FPS_SPEC": "1"})
    cols.append(f"spec {t:.3f}{'' if all(torch.equal(u, v) for u, v in zip(got, ref)) else ' MISMATCH'}")
    for W in (1, 2, 4, 8):
        if W * 32 * 16 < N:
            continue
        t, got = timed(x, N // 2, {"PS_FPS_SMALL_W": str(W)})
        same = all(torch.equal(u, v) for u, v in zip(got, ref))
        cols.append(f"W{W} {t:.3f}{'' if same else ' MISMATCH'}")
    print(f"B={B} N={N:5d} us/it: " + "  ".join(cols), flush=True)
