"""Sweep K1 launch shapes (PS_FPS_CLUSTER / PS_FPS_THREADS) on the bench batch:
us per iteration for the FastPoint prefix (k0 iterations) and a full exact FPS."""
import os
import subprocess
import sys

code = r'''
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2507_23480_b200 import engine
x = engine.as_xyz4(torch.from_numpy(bench.clouds_for(0, bench.B_PER_GPU)).cuda())
res = []
for stop in (600, 6000):
    for _ in range(2):
        engine.fps(x, 6000, k_stop=stop)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(3):
        engine.fps(x, 6000, k_stop=stop)
    e[1].record()
    torch.cuda.synchronize()
    res.append(e[0].elapsed_time(e[1]) / 3 * 1e3 / (stop - 1))
print("%.3f %.3f" % tuple(res))
'''
for C in sys.argv[1].split(","):
    for T in sys.argv[2].split(","):
        env = dict(os.environ, PS_FPS_CLUSTER=C, PS_FPS_THREADS=T)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
        print(f"C={C:>2} T={T}: prefix/full us per iter = {out.stdout.strip() or out.stderr.strip()[-200:]}", flush=True)
