"""K1 speculation counters (make TIMING=1 build, PS_B200_LIB=<that .so> PS_FPS_TIMING=1):
exchanges, samples per exchange and per-phase lead-warp cycles for the prefix and a full FPS,
in latency mode and with the throughput hint (--inflight K)."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2507_23480_b200 import engine
x = engine.as_xyz4(torch.from_numpy(bench.clouds_for(0, bench.B_PER_GPU)).cuda())
infl = int(sys.argv[sys.argv.index("--inflight") + 1]) if "--inflight" in sys.argv else None
for stop in (600, 6000):
    engine.fps(x, 6000, k_stop=stop, inflight_clouds=infl)
    torch.cuda.synchronize()
