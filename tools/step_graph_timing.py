"""One C3 step eager vs CUDA-graph replay, CUDA events around the step, L2 flushed before each."""
import sys, torch, numpy as np
sys.path.insert(0, ".")
import bench
from paper_2507_23480_b200 import engine
B = bench.B_PER_GPU
fp = engine.FastPoint(B, bench.N, bench.n_SAMPLES, p=bench.P, nseg=bench.NSEG, estimator="power",
                      exponent=bench.heldout_exponent(), extra_radii=(bench.RADIUS,))
fp.set_points(torch.from_numpy(bench.clouds_for(0, B)).cuda())
grp = (torch.empty(B, bench.n_SAMPLES, bench.K, dtype=torch.int32, device="cuda"),
       torch.empty(B, bench.n_SAMPLES, bench.K, dtype=torch.float64, device="cuda"),
       torch.empty(B, bench.n_SAMPLES, dtype=torch.int32, device="cuda"))
seeds = torch.arange(B, dtype=torch.int64, device="cuda")
def step():
    fp.state.copy_(seeds)
    fp.sample()
    fp.group_rf(bench.RADIUS, bench.K, out=grp)
for _ in range(3): step()
fp.check(); torch.cuda.synchronize()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def timeit(fn, n=10):
    ts = []
    for _ in range(n):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record(); fn(); e[1].record(); torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]))
    return np.median(ts)
print("eager step (one event pair): %.3f ms" % timeit(step))
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
print("graph step: %.3f ms" % timeit(g.replay))
