"""Two processes on ONE GPU run the one-process-per-GPU point-split FPS
(pointsplit.PointSplitFPS: cudaMalloc mailboxes, CUDA IPC handles exchanged
with all_gather_object, peer stores) for a few iterations and compare with
the single-rank kernel.  Kernels of different processes only alternate by
time-slicing, so n is tiny.  Launch:

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/ipc_selftest.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_23480_b200 import engine, pointsplit  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

dist.init_process_group("gloo")
rank = dist.get_rank()
torch.cuda.set_device(0)
N, n = 3000, int(os.environ.get("IPC_N", "6"))
cloud = generate_cloud("uniform-box", N, 77)
x = engine.as_xyz4(torch.from_numpy(cloud[None]).cuda())
ps = pointsplit.PointSplitFPS(1, N)
idx, curve, _, _ = ps.run(x, n)
torch.cuda.synchronize()
ref, rc, _, _ = engine.fps(x, n)
ok = torch.equal(idx, ref) and torch.equal(curve, rc)
print(f"rank {rank}: idx {idx[0].tolist()} identical to single-rank: {ok}", flush=True)
ps.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
