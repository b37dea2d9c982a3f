"""Exact FPS of one 2^20-point cloud to 65536 through ps_fps (internal virtual-rank split)."""
import sys, torch, time
sys.path.insert(0, ".")
from paper_2507_23480_b200 import engine
from paper_2507_23480_b200.harness import generate_cloud
c = generate_cloud("uniform-box", 1 << 20, 5000)
x = engine.as_xyz4(torch.from_numpy(c[None]).cuda())
engine.fps(x, 65536, k_stop=1024); torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record(); idx = engine.fps(x, 65536)[0]; e[1].record(); torch.cuda.synchronize()
print("N=2^20 -> 65536 exact FPS via ps_fps: %.1f ms" % e[0].elapsed_time(e[1]))
