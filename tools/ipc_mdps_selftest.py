"""Two processes on ONE GPU run pointsplit.PointSplitFastPoint (C5's MDPS
over one process per GPU: split prefix through CUDA-IPC mailboxes,
row-sharded build with the rows sent to rank 0, sampler on rank 0 and its
result broadcast, per-rank early-termination seeding + split FPS tail,
centroid-sharded grouping) with the gloo backend, and compare with the
single-process FastPoint.  Kernels of the two processes alternate by
time-slicing, so the cloud is small.  Launch:

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 tools/ipc_mdps_selftest.py
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
N, n = int(os.environ.get("MDPS_N", "3000")), int(os.environ.get("MDPS_n", "96"))
e, r = float(os.environ.get("MDPS_E", "0.25")), 0.12
cloud = generate_cloud("uniform-box", N, 79)
x = engine.as_xyz4(torch.from_numpy(cloud[None]).cuda())
ps = pointsplit.PointSplitFastPoint(N, n, exponent=e, extra_radii=(r,))
idx, (gi, gd, gc) = ps.run(x, rng_seed=4, k=16, radius=r)
torch.cuda.synchronize()
fp = engine.FastPoint(1, N, n, exponent=e, extra_radii=(r,))
fp.set_points(torch.from_numpy(cloud[None]).cuda())
fp.set_rng([4])
fp.sample()
fp.check()
ri, rd, rc = fp.group_rf(r, 16)
torch.cuda.synchronize()
ok_i = torch.equal(idx, fp.out[0])
ok_g = (torch.equal(gc, rc[0]) and torch.equal(gi, ri[0])
        and torch.equal(torch.nan_to_num(gd, nan=-1.0), torch.nan_to_num(rd[0], nan=-1.0)))
ok = ok_i and ok_g
if not ok_i:
    bad = (idx != fp.out[0]).nonzero()
    print(f"rank {rank}: first index mismatch at {int(bad[0])}: {idx[int(bad[0]):int(bad[0]) + 6].tolist()} vs "
          f"{fp.out[0, int(bad[0]):int(bad[0]) + 6].tolist()}", flush=True)
if not ok:
    print(f"rank {rank}: split status {ps.fp.csr.status.tolist()} reached {ps.fp.reached.tolist()} entered "
          f"{ps.fp.entered.tolist()} stride {ps.fp.csr.stride} cap {ps.fp.csr.cap_entries}", flush=True)
if not ok_g:
    print(f"rank {rank}: groups differ (cnt equal: {torch.equal(gc, rc[0])})", flush=True)
print(f"rank {rank}: reached {int(fp.reached[0])}/{n}, identical to single-process FastPoint: {ok}", flush=True)
ps.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
