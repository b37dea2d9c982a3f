"""One exact FPS call on B small clouds (for ncu): N, B from the env."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

N = int(os.environ.get("N", "1024"))
B = int(os.environ.get("B", "32"))
c = np.stack([generate_cloud("unit-sphere", N, 7 + b) for b in range(B)])
x = engine.as_xyz4(torch.from_numpy(c).cuda())
for _ in range(2):
    engine.fps(x, N // 2)
torch.cuda.synchronize()
