"""K1 one-sample kernel vs top-K speculation on the bench batch: us per
iteration for the FastPoint prefix (600) and a full exact FPS (6000), and
index/curve equality of the two kernels."""
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
        o = engine.fps(x, 6000, k_stop=stop)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(3):
        engine.fps(x, 6000, k_stop=stop)
    e[1].record()
    torch.cuda.synchronize()
    res.append(e[0].elapsed_time(e[1]) / 3 * 1e3 / (stop - 1))
idx, curve = engine.fps(x, 6000)[:2]
torch.save((idx.cpu(), curve.cpu()), sys.argv[1])
print("%.3f %.3f" % tuple(res))
'''
outs = {}
for name, extra in (("one-sample", {"PS_FPS_NOSPEC": "1"}), ("spec", {})):
    env = dict(os.environ, **extra)
    path = f"/tmp/fps_{name}.pt"
    out = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True, timeout=300)
    print(f"{name:>10}: prefix/full us per iter = {out.stdout.strip() or out.stderr.strip()[-400:]}", flush=True)
    outs[name] = path
import torch
a = torch.load(outs["one-sample"])
b = torch.load(outs["spec"])
print("indices equal:", torch.equal(a[0], b[0]), " curve bit-equal:", torch.equal(a[1], b[1]))
