"""Early-termination share and coverage quality of the C3 bench batch under
the estimator choices: power-law exponents fitted on 2 and
5 held-out clouds, a sweep around them, and the MLP estimator trained on
held-out exact curves.  One B200; quality = avg min spacing
of FastPoint / exact FPS."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import curve, engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

B, N, n = bench.B_PER_GPU, bench.N, bench.n_SAMPLES
clouds = bench.clouds_for(0, B)
x = torch.from_numpy(clouds).cuda()
held = np.stack([generate_cloud(bench.FAMILY, N, 99000 + i) for i in range(16)])
_, cv, _, _ = engine.fps(engine.as_xyz4(torch.from_numpy(held).cuda()), n)
cv = cv.cpu().numpy()
e2, e5, e16 = (curve.fit_power_exponent(cv[:k]) for k in (2, 5, 16))
print(f"fitted exponent: 2 clouds {e2:.6f}, 5 clouds {e5:.6f}, 16 clouds {e16:.6f}", flush=True)
xyz4 = engine.as_xyz4(x)
exact_idx, _, _, _ = engine.fps(xyz4, n)
sp_x = engine.min_spacing_d2(xyz4, exact_idx).sqrt().mean(dim=1)


def run(label, **kw):
    fp = engine.FastPoint(B, N, n, p=bench.P, nseg=bench.NSEG, extra_radii=(bench.RADIUS,), **kw)
    fp.set_points(x)
    fp.set_rng(list(range(B)))
    fp.sample()
    fp.check()
    ts = []
    for _ in range(5):
        fp.set_rng(list(range(B)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fp.sample()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    q = (engine.min_spacing_d2(xyz4, fp.out).sqrt().mean(dim=1) / sp_x).cpu().numpy()
    et = (n - fp.reached.cpu().numpy()) / n
    print(f"{label:28s} ET {100 * et.mean():5.2f}% (max {100 * et.max():5.2f}%)  quality {q.mean():.4f} "
          f"(min {q.min():.4f})  sample {np.median(ts):.3f} ms", flush=True)


for e in sorted({round(e2, 6), round(e5, 6), round(e16, 6), 0.50, 0.52, 0.55, 0.57, 0.60}):
    run(f"power e={e}", estimator="power", exponent=e)
t0 = time.time()
pairs = [curve.mlp_pair(c) for c in cv]
model, losses = curve.mlp_train(pairs, epochs=int(os.environ.get("MLP_EPOCHS", "60")), lr=0.01,
                                rng=np.random.default_rng(1))
print(f"MLP trained on 16 curves: loss {losses[0]:.3e} -> {losses[-1]:.3e} ({time.time() - t0:.0f} s)", flush=True)
run("mlp (16 curves)", estimator="mlp", mlp=model)
