#!/bin/bash
# Sampler stage at the bench batch for several cluster widths (PS_SAMPLER_CLUSTER).
for c in "$@"; do
  PS_SAMPLER_CLUSTER=$c python - <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2507_23480_b200 import engine
B = bench.B_PER_GPU
fp = engine.FastPoint(B, bench.N, bench.n_SAMPLES, p=bench.P, nseg=bench.NSEG, estimator="power",
                      exponent=bench.heldout_exponent(), extra_radii=(bench.RADIUS,))
fp.set_points(torch.from_numpy(bench.clouds_for(0, B)).cuda())
fp.set_rng(list(range(B)))
st0 = fp.state.clone()
fp.sample(); fp.check()
ref = fp.out.clone()
ts = []
for _ in range(20):
    fp.state.copy_(st0)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record(); fp._sampler(); e[1].record(); torch.cuda.synchronize()
    ts.append(e[0].elapsed_time(e[1]) * 1e3)
ts.sort()
fp._early_termination(); torch.cuda.synchronize()
print(f"C={os.environ['PS_SAMPLER_CLUSTER']}: sampler {ts[10]:.1f} us (min {ts[0]:.1f}) out identical {torch.equal(fp.out, ref)}", flush=True)
PY
done
