"""A/B K1 variants on the bench batch in one process: environment settings
given as KEY=VAL[,KEY=VAL] arguments (e.g. PS_FPS_CLUSTER=12), against the
default and PS_FPS_NOSPEC=1 (one-sample kernel).  Prints us/iteration
for the FastPoint prefix (600) and a full exact FPS (6000), and whether the
indices/curve equal the one-sample kernel's."""
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2507_23480_b200 import engine  # noqa: E402

x = engine.as_xyz4(torch.from_numpy(bench.clouds_for(0, bench.B_PER_GPU)).cuda())


def run(env):
    for k in ("PS_FPS_NOSPEC", "PS_FPS_CLUSTER", "PS_FPS_THREADS", "PS_SPEC_TARGET"):
        os.environ.pop(k, None)
    os.environ.update(env)
    res = []
    for stop in (600, 6000):
        for _ in range(2):
            engine.fps(x, 6000, k_stop=stop)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            e[0].record()
            engine.fps(x, 6000, k_stop=stop)
            e[1].record()
            torch.cuda.synchronize()
            ts.append(e[0].elapsed_time(e[1]) * 1e3 / (stop - 1))
        res.append(sorted(ts)[2])
    idx, curve = engine.fps(x, 6000)[:2]
    return res, idx, curve


variants = [("one-sample", {"PS_FPS_NOSPEC": "1"}), ("default", {})]
for v in sys.argv[1:]:  # KEY=VAL[,KEY=VAL...] environment variants
    variants.append((v, dict(kv.split("=", 1) for kv in v.split(","))))
ref = None
for name, env in variants:
    (p, f), idx, curve = run(env)
    if ref is None:
        ref = (idx, curve)
    ok = torch.equal(idx, ref[0]) and torch.equal(curve, ref[1])
    print(f"{name:>24}: prefix {p:.3f} us/it  full {f:.3f} us/it  bit-equal {ok}", flush=True)
