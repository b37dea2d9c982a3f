"""Generate tests/golden/c5_digest.json: oracle digests at config C5 size.

Config C5 (BASELINE.json configs[4]) is one uniform-box cloud of N = 2^20
points sampled to n = 65536.  The oracle (oracle/ps_oracle.c, itself pinned
to the reference kernels by tests/golden/golden.npz) is run here with the
reference's multi-worker split (PS_ORACLE_THREADS, identical results), and
the outputs are stored as sha256 digests plus a few verbatim entries:

* exact FPS 2^20 -> 65536 (baselines.fps; fps_loop,
  _kernels.py:35-74): indices and curve;
* FastPoint (mdps) at the same size -- power estimator
  with an exponent fitted offline on a held-out cloud, the rf ball query
  radius baked in -- indices,
  reached / entered / exhausted, radii, final RNG state and the rf ball
  query counts and members (neighbors.rf_ball_query);
* FastPoint at N = 2^18 -> 16384 (the size the GPU suite also checks
  against the live oracle).

    python tests/golden/make_c5_digest.py            # ~10 min on 8 threads

The GPU tests compare the CUDA path with these digests; nothing here reads
/root/reference.
"""

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2507_23480_b200.harness import generate_cloud  # noqa: E402

C5_N, C5_n, C5_SEED = 1 << 20, 65536, 5000
# exponents fitted offline (curve.fit_power_exponent) on the
# exact FPS curves of held-out uniform-box clouds (seeds 5100 at 2^20, 5200-5201
# at 2^18), so that early termination stays as short as the estimator allows
FP_RNG, FP_RADIUS, FP_K = 0, 0.04, 32
C5_EXPONENT, MID_EXPONENT = 0.368508, 0.376902
MID_N, MID_n, MID_SEED = 1 << 18, 16384, 5001


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fastpoint_digest(cloud, n, exponent):
    t = time.time()
    r = O.mdps(cloud, n, p=0.1, nseg=6, estimator="power", exponent=exponent, rng_seed=FP_RNG,
               extra_radii=(FP_RADIUS,))
    gi, gd, gc = O.rf_ball_query(r.excl, FP_RADIUS, r.indices, FP_K)
    members = np.where(np.arange(FP_K)[None, :] < gc[:, None], gi, -1).astype(np.int64)
    return {
        "idx_sha256": sha(r.indices.astype(np.int64)), "idx_head": r.indices[:16].tolist(),
        "idx_tail": r.indices[-16:].tolist(), "reached": r.reached, "entered": r.entered,
        "exhausted": r.exhausted, "R": [float(v) for v in r.thresholds], "rng_state": str(r.rng_state),
        "rf_cnt_sha256": sha(gc.astype(np.int64)), "rf_idx_sha256": sha(members),
        "rf_cnt_sum": int(gc.sum()), "entries": int(r.excl.indptr[-1]), "seconds": time.time() - t,
    }


def main():
    O.set_threads(int(os.environ.get("PS_ORACLE_THREADS", os.cpu_count() or 1)))
    out = {"generator": "tests/golden/make_c5_digest.py", "oracle_threads": O.THREADS,
           "c5": {"family": "uniform-box", "N": C5_N, "n": C5_n, "cloud_seed": C5_SEED, "seed_index": 0},
           "fastpoint_params": {"p": 0.1, "nseg": 6, "estimator": "power", "exponent": C5_EXPONENT,
                                "mid_exponent": MID_EXPONENT, "rng_seed": FP_RNG, "radius": FP_RADIUS, "k": FP_K}}
    cloud = generate_cloud("uniform-box", C5_N, C5_SEED)
    t = time.time()
    idx, curve, _, _, _ = O.fps(cloud, C5_n, 0)
    out["exact_fps"] = {"idx_sha256": sha(idx.astype(np.int64)), "curve_sha256": sha(curve.astype(np.float64)),
                        "idx_head": idx[:16].tolist(), "idx_tail": idx[-16:].tolist(),
                        "curve_last": float(curve[-1]), "seconds": time.time() - t}
    print("exact fps", out["exact_fps"]["seconds"], flush=True)
    mid = generate_cloud("uniform-box", MID_N, MID_SEED)
    out["mid"] = {"family": "uniform-box", "N": MID_N, "n": MID_n, "cloud_seed": MID_SEED,
                  "fastpoint": fastpoint_digest(mid, MID_n, MID_EXPONENT)}
    print("mid fastpoint", out["mid"]["fastpoint"]["seconds"], flush=True)
    out["fastpoint"] = fastpoint_digest(cloud, C5_n, C5_EXPONENT)
    print("c5 fastpoint", out["fastpoint"]["seconds"], flush=True)
    with open(os.path.join(HERE, "c5_digest.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
