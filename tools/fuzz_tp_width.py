"""Randomized parity of exact FPS at the throughput-hint widths (10 points per
thread, md in shared memory, the lead on its own loop) against the oracle:
random family / N / seed / n / k_stop, two clouds per batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fams = ["room-surfaces", "uniform-box", "gaussian-clusters", "lattice", "unit-sphere"]
bad = 0
for i in range(cases):
    N = int(rng.integers(9000, 48001))
    fam = fams[int(rng.integers(len(fams)))]
    cl = np.stack([generate_cloud(fam, N, int(rng.integers(1 << 30))) for _ in range(2)])
    if rng.random() < 0.3:  # duplicated points
        cl[1, N // 2:] = cl[1, :N - N // 2]
    n = int(rng.integers(200, 1500))
    k_stop = n if rng.random() < 0.6 else int(rng.integers(1, n + 1))
    seed = int(rng.integers(N))
    x = engine.as_xyz4(torch.from_numpy(cl).cuda())
    with engine.inflight(64):
        idx, curve, md, taken = engine.fps(x, n, seed_index=seed, k_stop=k_stop)
    ok = True
    for b in range(2):
        ri, rc, rmd, rtk, _ = O.fps(cl[b], n, seed, k_stop=k_stop)
        ok &= np.array_equal(idx[b].cpu().numpy()[:k_stop], ri[:k_stop])
        ok &= np.array_equal(curve[b].cpu().numpy()[:k_stop], rc[:k_stop])
        ok &= np.array_equal(md[b].cpu().numpy(), rmd) and np.array_equal(taken[b].cpu().numpy(), rtk)
    bad += 0 if ok else 1
    print(f"case {i}: {fam} N={N} n={n} k_stop={k_stop} seed={seed} {'ok' if ok else 'MISMATCH'}", flush=True)
print(f"{cases - bad}/{cases} bit-exact")
sys.exit(1 if bad else 0)
