"""C5 (single cloud N = 2^20 -> 65536) point-split FPS on one GPU with G
virtual ranks; cross-checked against the single-rank kernel.

  python tools/c5_split.py [n] [G,G,...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_23480_b200 import _lib, engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

N = 1 << 20
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
Gs = [int(g) for g in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 12, 16]
cloud = generate_cloud("uniform-box", N, 5000)
x = engine.as_xyz4(torch.from_numpy(cloud[None]).cuda())
ref = None
for G in Gs:
    import ctypes
    C, P = ctypes.c_int32(), ctypes.c_int32()
    rc = _lib.raw("ps_fps_split_plan", N, 1, G, G, ctypes.byref(C), ctypes.byref(P))
    if rc != 0:
        print(f"G={G}: no co-resident plan ({_lib.raw('ps_last_error').decode()})", flush=True)
        continue
    mb = engine.SplitMailboxes(1, G)
    engine.fps_split(x, n, G, mailboxes=mb, k_stop=min(n, 512))
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    idx, curve, _, _ = engine.fps_split(x, n, G, mailboxes=mb)
    e[1].record()
    torch.cuda.synchronize()
    ms = e[0].elapsed_time(e[1])
    print(f"G={G:2d} (C={C.value}, P={P.value}): {ms:8.1f} ms, {ms * 1e3 / (n - 1):.3f} us/iter, "
          f"{n / ms * 1e3:,.0f} sampled pts/s", flush=True)
    if ref is None:
        t0 = time.time()
        ref = engine.fps(x, n)
        torch.cuda.synchronize()
        print(f"single-rank kernel: {1e3 * (time.time() - t0):.1f} ms (wall)", flush=True)
    same = torch.equal(idx, ref[0]) and torch.equal(curve, ref[1])
    print(f"   identical to single-rank FPS: {same}", flush=True)
