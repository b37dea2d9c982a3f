"""C2 cascade (bench.bench_c2_cascade) with and without the small-cloud FPS
kernel (PS_FPS_NOSMALL), interleaved."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for rep in range(2):
    for env in ({"PS_FPS_NOSMALL": "1"}, {}):
        os.environ.pop("PS_FPS_NOSMALL", None)
        os.environ.update(env)
        r = bench.bench_c2_cascade("cuda", 10)
        print(json.dumps({"env": env, **{k: r[k] for k in ("fastpoint_first_ms", "all_exact_fps_ms", "speedup_vs_exact")}}),
              flush=True)
