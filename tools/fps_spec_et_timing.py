"""K1 speculation counters for a FastPoint run (prefix + early-termination tail); TIMING=1 build."""
import os, sys
sys.path.insert(0, ".")
import torch, bench
from paper_2507_23480_b200 import engine
B = bench.B_PER_GPU
fp = engine.FastPoint(B, bench.N, bench.n_SAMPLES, p=bench.P, nseg=bench.NSEG, estimator="power",
                      exponent=bench.heldout_exponent(), extra_radii=(bench.RADIUS,))
fp.set_points(torch.from_numpy(bench.clouds_for(0, B)).cuda())
fp.sample(); fp.check(); torch.cuda.synchronize()
os.environ["PS_FPS_TIMING"] = "1"
print("reached", fp.reached.tolist(), file=sys.stderr)
fp.sample(); torch.cuda.synchronize()
c = fp.curve[0].cpu().numpy(); r = int(fp.reached[0])
print("curve around reached:", c[r-5:r+3], file=sys.stderr)
