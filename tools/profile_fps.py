"""Exact FPS on the bench batch (8 x 24000 -> 6000) inside a cudaProfilerStart/Stop range."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402

clouds = bench.clouds_for(0, bench.B_PER_GPU)
x = engine.as_xyz4(torch.from_numpy(clouds).cuda())
engine.fps(x, bench.n_SAMPLES)
torch.cuda.synchronize()
torch.cuda.profiler.start()
engine.fps(x, bench.n_SAMPLES)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
