"""Register speculative kernel vs resident speculative kernel on C4-sized clouds (us per iteration)."""
import os, sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2507_23480_b200 import engine
from paper_2507_23480_b200.harness import generate_cloud
for N, B in ((32768, 2), (65536, 2), (65536, 4)):
    c = np.stack([generate_cloud("room-surfaces", N, 7 + b) for b in range(B)])
    x = engine.as_xyz4(torch.from_numpy(c).cuda())
    for stop in (N // 40, N // 4):
        row = []
        for env in ({}, {"PS_FPS_RESIDENT": "1"}):
            os.environ.pop("PS_FPS_RESIDENT", None); os.environ.update(env)
            engine.fps(x, N // 4, k_stop=stop); torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record(); engine.fps(x, N // 4, k_stop=stop); e[1].record(); torch.cuda.synchronize()
            row.append(e[0].elapsed_time(e[1]) * 1e3 / (stop - 1))
        os.environ.pop("PS_FPS_RESIDENT", None)
        print(f"N={N} B={B} iters={stop}: register spec {row[0]:.3f} us/it, resident spec {row[1]:.3f} us/it", flush=True)
