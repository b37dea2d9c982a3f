"""One FastPoint + grouping step at the bench workload, bracketed by
cudaProfilerStart/Stop so that `ncu --profile-from-start off` captures only
the step's kernels (warm-up and set-up stay outside).

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches.csv python tools/profile_step.py
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:fps_cluster -o gpurun_out/prof python tools/profile_step.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402


def main():
    exact = "--exact" in sys.argv
    # --inflight K: the FPS cluster width of K clouds in flight (the bench's
    # concurrent chains; default 8 x 5)
    infl = int(sys.argv[sys.argv.index("--inflight") + 1]) if "--inflight" in sys.argv else None
    B = bench.B_PER_GPU
    clouds = bench.clouds_for(0, B)
    fp = engine.FastPoint(B, bench.N, bench.n_SAMPLES, p=bench.P, nseg=bench.NSEG, estimator="power",
                          exponent=bench.heldout_exponent(), extra_radii=(bench.RADIUS,), inflight_clouds=infl)
    fp.set_points(torch.from_numpy(clouds).cuda())
    for _ in range(2):
        fp.set_rng(list(range(B)))
        fp.sample()
        fp.group_rf(bench.RADIUS, bench.K)
        if exact:
            idx, *_ = engine.fps(fp.xyz4, bench.n_SAMPLES)
            engine.ball_query_naive(fp.xyz4, idx, bench.RADIUS, bench.K)
    fp.check()
    torch.cuda.synchronize()
    fp.set_rng(list(range(B)))
    torch.cuda.profiler.start()
    fp.sample()
    fp.group_rf(bench.RADIUS, bench.K)
    if exact:
        idx, *_ = engine.fps(fp.xyz4, bench.n_SAMPLES)
        engine.ball_query_naive(fp.xyz4, idx, bench.RADIUS, bench.K)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("reached", fp.reached.tolist(), "E", fp.csr.indptr[:, -1].tolist())


if __name__ == "__main__":
    main()
