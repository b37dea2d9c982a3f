"""Benchmark: FastPoint sampling + grouping at N=24k on B200 (BASELINE.json
metric "sampled pts/sec & us/cloud for FPS+ball-query at N=24k, 1-8 B200").

Workload (BASELINE.json configs[2], "C3"): per GPU a batch of B=8 synthetic
room-surface clouds (6 x 5 x 3 m, S3DIS-shape), N = 24000, stride 4 ->
n = 6000 samples, FastPoint p = 0.1, nseg = 6, power-law estimator (exponent
fitted offline on held-out clouds), then redundancy-free ball query r = 0.1 m,
k = 32 from the cached distances.  One step = one pass of that path over the
batch.  The exact-FPS + naive-ball-query B200 path is timed beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: launched by torch.distributed.run; each rank samples its own batch
(batch sharding, no data-path collective; "scaling": "weak").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

B_PER_GPU, N, STRIDE = 8, 24000, 4
n_SAMPLES = N // STRIDE
P, NSEG, RADIUS, K = 0.1, 6, 0.1, 32
FAMILY = "room-surfaces"
METRIC = "sampled pts/sec & us/cloud for FPS+ball-query at N=24k, 1-8 B200"
UNIT = "sampled pts/s"
WORKLOAD = ("C3 PointNeXt-L S3DIS-shape: B=8 clouds/GPU, N=24000 -> n=6000 (stride 4), FastPoint "
            "(p=0.1, nseg=6, power estimator) + rf ball_query r=0.1 k=32")


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def shard_seeds(rank: int, B: int):
    """Cloud seeds of one rank's shard: disjoint across ranks (batch sharding,
    no data-path collective)."""
    return [1000 * 3 + rank * B + b for b in range(B)]


def clouds_for(rank: int, B: int, n_points: int = N):
    from paper_2507_23480_b200.harness import generate_cloud

    return np.stack([generate_cloud(FAMILY, n_points, s) for s in shard_seeds(rank, B)])


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank time over the job (the contract's timing rule)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


HELDOUT = 5  # held-out clouds of the family for the exponent fit (A3)


def heldout_exponent():
    """Offline exponent fit on 5 held-out clouds of the
    family (the A3 protocol), from exact GPU FPS curves --
    outside every timed region."""
    import torch

    from paper_2507_23480_b200 import curve, engine
    from paper_2507_23480_b200.harness import generate_cloud

    held = np.stack([generate_cloud(FAMILY, N, 99000 + i) for i in range(HELDOUT)])
    _, cv, _, _ = engine.fps(engine.as_xyz4(torch.from_numpy(held).cuda()), n_SAMPLES)
    return curve.fit_power_exponent(cv.cpu().numpy())


def heldout_exponent_cpu():
    """Same offline fit as heldout_exponent(), from the CPU oracle's exact FPS
    curves (bit-identical to the GPU's), for the reference arm."""
    from oracle import oracle as O
    from paper_2507_23480_b200 import curve
    from paper_2507_23480_b200.harness import generate_cloud

    curves = [O.fps(generate_cloud(FAMILY, N, 99000 + i), n_SAMPLES)[1] for i in range(HELDOUT)]
    return curve.fit_power_exponent(curves)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the
    timed region (written to a temp file: nvidia-smi block-buffers pipes)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        import tempfile

        fd, self.path = tempfile.mkstemp(prefix="ps_clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)  # first sample before the timed region starts
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        sm, mx, reasons, util = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            lines = open(self.path).read().splitlines()
            os.unlink(self.path)
        except (OSError, TypeError):
            lines = []
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                s, m, u = float(f[0]), float(f[1]), float(f[6])
            except ValueError:
                continue
            mx = m
            util.append(u)
            sm.append(s)
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "samples_loaded": len(loaded)}


def peaks():
    try:
        return json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except OSError:
        return {}


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path (oracle port) on the host cores


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_run(clouds, exponent, threads):
    """The reference's CPU path on `threads` host threads: one cloud per pool
    thread (the kernels release the GIL, like the reference's nogil numba
    kernels) and, when there are more threads than clouds, the reference's
    per-cloud worker split of FPS and excl_collect (core.workers,
    core.py:71-101) over the rest."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    B = clouds.shape[0]
    pool = max(1, min(threads, B))
    old = O.set_threads(max(1, threads // pool))

    def one(b):
        r = O.mdps(clouds[b], n_SAMPLES, p=P, nseg=NSEG, estimator="power", exponent=exponent, rng_seed=b,
                   extra_radii=(RADIUS,))
        O.rf_ball_query(r.excl, RADIUS, r.indices, K)
        return r.indices

    try:
        t0 = time.perf_counter()
        with ThreadPoolExecutor(pool) as ex:
            out = list(ex.map(one, range(B)))
        return time.perf_counter() - t0, out
    finally:
        O.set_threads(old)


def cpu_baseline(clouds, exponent, gpu_idx, runs):
    """threads = 1 and threads = os.cpu_count(), one
    warm-up then the median of `runs` timed runs each, CPU model named; the
    indices are checked against the GPU run of the same batch."""
    res = {}
    match = None
    for t in sorted({1, os.cpu_count() or 1}):
        cpu_run(clouds[:1], exponent, 1)  # warm-up (oracle load, page-in)
        times = []
        for _ in range(max(1, runs)):
            dt, idx = cpu_run(clouds, exponent, t)
            times.append(dt)
        if match is None and gpu_idx is not None:
            match = all(np.array_equal(idx[b], gpu_idx[b]) for b in range(clouds.shape[0]))
        med = statistics.median(times)
        res[t] = {"value": clouds.shape[0] * n_SAMPLES / med, "median_s": med, "runs_s": times}
    tmax = max(res)
    return {"value": res[tmax]["value"], "unit": UNIT, "cores": tmax, "kind": "port",
            "cpu": cpu_model(), "threads_1": res[1], f"threads_{tmax}": res[tmax],
            "sample": (f"the rank-0 batch ({clouds.shape[0]} clouds) FastPoint + rf ball query per run, one cloud per "
                       "thread plus the reference's per-cloud worker split; warm-up + median of "
                       f"{max(1, runs)} runs per thread count"),
            "indices_bit_exact_vs_gpu": match}


def workload_config(ws: int, exponent: float) -> dict:
    """The workload both arms run (identical in their JSON lines)."""
    return {"workload": WORKLOAD, "family": FAMILY, "B_per_gpu": B_PER_GPU, "B": B_PER_GPU,
            "global_batch": B_PER_GPU * ws, "N": N, "n": n_SAMPLES, "p": P, "nseg": NSEG, "radius": RADIUS, "k": K,
            "exponent": round(exponent, 6), "parallelism": f"batch-shard x{ws}"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    clouds = clouds_for(0, B_PER_GPU)
    exponent = heldout_exponent_cpu()
    threads = os.cpu_count() or 1
    for _ in range(max(args.warmup, 0)):
        cpu_run(clouds[:1], exponent, 1)
    times = []
    for _ in range(args.steps):
        dt, _ = cpu_run(clouds, exponent, threads)
        times.append(dt)
    t = sum(times)
    value = B_PER_GPU * n_SAMPLES * args.steps / t
    sample = (f"{B_PER_GPU} clouds x (FastPoint + rf ball query) per step on all {threads} host threads: one cloud "
              "per pool thread plus the reference's per-cloud worker split")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(ws, exponent),
            "us_per_cloud": 1e6 * t / (args.steps * B_PER_GPU),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


L2_BYTES = 126 << 20  # B200 L2 (126 MB)


def input_ring(rank: int, B: int):
    """Distinct input batches whose float32 coordinates together exceed L2,
    so that no timed step re-reads an input batch L2 still holds (the
    contract's alternative to a flush).  Batch 0 is the rank's shard batch."""
    per = B * N * 3 * 4
    R = -(-int(1.25 * L2_BYTES) // per)
    from paper_2507_23480_b200.harness import generate_cloud

    ring = [clouds_for(rank, B)]
    for k in range(1, R):
        ring.append(np.stack([generate_cloud(FAMILY, N, 7_000_000 + (rank * R + k) * B + b) for b in range(B)]))
    return np.stack(ring)  # [R, B, N, 3]


class Chain:
    """One FastPoint pipeline (buffers, stream, CUDA graph of sample + rf
    grouping) -- the unit the bench runs S of concurrently."""

    def __init__(self, B, exponent, dev, seeds, inflight=None):
        import torch

        from paper_2507_23480_b200 import engine

        self.fp = engine.FastPoint(B, N, n_SAMPLES, p=P, nseg=NSEG, estimator="power", exponent=exponent,
                                   extra_radii=(RADIUS,), device=dev, inflight_clouds=inflight)
        self.grp = (torch.empty(B, n_SAMPLES, K, dtype=torch.int32, device=dev),
                    torch.empty(B, n_SAMPLES, K, dtype=torch.float64, device=dev),
                    torch.empty(B, n_SAMPLES, dtype=torch.int32, device=dev))
        self.seed_t = torch.tensor(seeds, dtype=torch.int64, device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        self.graph = None

    def body(self):
        self.fp.state.copy_(self.seed_t)
        self.fp.sample()
        self.fp.group_rf(RADIUS, K, out=self.grp)

    def capture(self):
        import torch

        from paper_2507_23480_b200 import _lib

        s = self.stream
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.body()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.fp.check()
        g = torch.cuda.CUDAGraph()
        k0 = _lib.launch_count()
        with torch.cuda.graph(g, stream=s):
            self.body()
        self.kernels = _lib.launch_count() - k0  # our kernels per replay (ps_launch_count)
        self.graph = g


def run_chains(chains, steps, feed, after=None):
    """Steps round-robin over the chains' streams (step s on chain s % S):
    feed(chain, s) enqueues the step's input, the graph the step, after(chain,
    s) its output.  Device wall time between events around the whole loop."""
    import torch

    main = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for c in chains:
        c.stream.wait_event(a)
    for s in range(steps):
        c = chains[s % len(chains)]
        with torch.cuda.stream(c.stream):
            feed(c, s)
            c.graph.replay()
            if after is not None:
                after(c, s)
    for c in chains:
        main.wait_stream(c.stream)
    b.record(main)
    b.synchronize()
    return a.elapsed_time(b)


def main_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2507_23480_b200 import _lib, engine

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    B = B_PER_GPU
    ring_h = input_ring(rank, B)
    R = ring_h.shape[0]
    clouds = ring_h[0]
    exponent = heldout_exponent()
    S = max(1, args.streams)
    seeds = [rank * B + b for b in range(B)]  # sampler RNG seeds (clouds: shard_seeds)
    # throughput hint: S chains keep B * S clouds in flight (FPS cluster width)
    chains = [Chain(B, exponent, dev, seeds, inflight=B * S if S > 1 else None) for _ in range(S)]
    ring_d = torch.from_numpy(ring_h).to(dev)  # [R, B, N, 3] resident inputs
    for c in chains:
        c.fp.set_points(ring_d[0])
        c.capture()
    fp = chains[0].fp
    stream = torch.cuda.current_stream()

    # ---- stage breakdown: one chain, per-stage events, L2 flushed between steps ----
    # stage_ms: each stage alone at its latency-mode width (the FastPoint a
    # single chain runs); stage_ms_inflight: the same with the chains'
    # throughput-hint FPS width
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stages = ["fps_prefix", "thresholds", "excl_build", "sampler", "early_term", "rf_ball_query"]
    lat_chain = Chain(B, exponent, dev, seeds)

    def staged(ch, events):
        f = ch.fp
        f.state.copy_(ch.seed_t)
        events[0].record(stream)
        f._prefix()
        events[1].record(stream)
        f._thresholds()
        events[2].record(stream)
        f._exclusion()
        events[3].record(stream)
        f._sampler()
        events[4].record(stream)
        f._early_termination()
        events[5].record(stream)
        f.group_rf(RADIUS, K, out=ch.grp)
        events[6].record(stream)

    def breakdown(ch):
        ch.fp.set_points(ring_d[0])
        for _ in range(max(args.warmup, 3)):
            staged(ch, [torch.cuda.Event(enable_timing=True) for _ in range(7)])
        torch.cuda.synchronize()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in range(args.steps)]
        for s in range(args.steps):
            ch.fp.set_points(ring_d[s % R])
            flush.zero_()  # L2 flush between steps, outside the events
            staged(ch, ev[s])
        torch.cuda.synchronize()
        sm = np.array([[ev[s][i].elapsed_time(ev[s][i + 1]) for i in range(6)] for s in range(args.steps)])
        return {nm: float(sm[:, i].mean()) for i, nm in enumerate(stages)}

    per_stage = breakdown(lat_chain)
    per_stage_inflight = breakdown(chains[0])
    fp.set_points(ring_d[0])
    del flush

    # ---- headline: S concurrent chains, steps back to back, inputs cold (ring > L2) ----
    def feed_dev(c, s):
        c.fp.set_points(ring_d[s % R])

    for _ in range(max(args.warmup, 3)):
        run_chains(chains, S, feed_dev)
    launches0 = _lib.launch_count()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_ms = run_chains(chains, args.steps, feed_dev)
    # eager calls count themselves; each graph replay launches the kernels its
    # capture counted
    launches = (_lib.launch_count() - launches0) + sum(
        chains[s % S].kernels for s in range(args.steps))
    t_ms = max_over_ranks(t_ms, dev)
    value = ws * B * n_SAMPLES * args.steps / (t_ms / 1e3)
    # one chain alone in latency mode (no cross-step overlap, widest FPS
    # clusters), same loop
    lat = lat_chain
    lat.fp.set_points(ring_d[0])
    lat.capture()
    run_chains([lat], 2, feed_dev)
    t1_ms = max_over_ranks(run_chains([lat], args.steps, feed_dev), dev)
    del lat, lat_chain

    # results of the last step of each chain: valid (status clear) and
    # identical to a fresh un-captured run of the same batch
    for c in chains:
        if c.fp.csr.overflowed():
            raise RuntimeError("exclusion capacity exhausted in a timed replay")
    last = args.steps - 1
    fp.set_points(ring_d[last % R])
    chains[0].body()
    torch.cuda.synchronize()
    cl = chains[last % S]
    replay_ok = bool(torch.equal(cl.fp.out, fp.out)) if cl is not chains[0] else True
    fp.set_points(ring_d[0])
    chains[0].body()
    torch.cuda.synchronize()
    reached = fp.reached.cpu().numpy()

    # ---- exact-FPS + naive ball query comparator, same loop and ring ---------------------
    class ExactChain:
        def __init__(self, inflight):
            self.x4 = torch.zeros(B, N, 4, dtype=torch.float32, device=dev)
            self.stream = torch.cuda.Stream(device=dev)
            self.graph = None
            self.inflight = inflight

        def body(self):
            idx, _, _, _ = engine.fps(self.x4, n_SAMPLES, inflight_clouds=self.inflight)
            self.out = engine.ball_query_naive(self.x4, idx, RADIUS, K)
            self.idx = idx

    ex = [ExactChain(B * S if S > 1 else None) for _ in range(S)] + [ExactChain(None)]  # last: latency mode
    for c in ex:
        c.x4[..., :3].copy_(ring_d[0])
        c.stream.wait_stream(stream)
        with torch.cuda.stream(c.stream):
            c.body()
        stream.wait_stream(c.stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=c.stream):
            c.body()
        c.graph = g

    def feed_exact(c, s):
        c.x4[..., :3].copy_(ring_d[s % R])

    run_chains(ex[:S], S, feed_exact)
    exact_ms = max_over_ranks(run_chains(ex[:S], args.steps, feed_exact), dev) / args.steps
    run_chains(ex[S:], 2, feed_exact)
    exact1_ms = max_over_ranks(run_chains(ex[S:], args.steps, feed_exact), dev) / args.steps
    # kernel split of the exact path (latency mode, per-kernel events)
    fps_ms, bqn_ms = [], []
    x4 = ex[S].x4
    for s in range(min(args.steps, 5)):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        idx, _, _, _ = engine.fps(x4, n_SAMPLES)
        e1.record(stream)
        engine.ball_query_naive(x4, idx, RADIUS, K)
        e2.record(stream)
        torch.cuda.synchronize()
        fps_ms.append(e0.elapsed_time(e1))
        bqn_ms.append(e1.elapsed_time(e2))
    del ex

    # ---- end to end through the public API: pinned host in, results out ---------
    # every step uploads its batch from pinned host memory (the ring), runs
    # set_points + sample + group_rf, and downloads indices, groups and the
    # exclusion status; chains run concurrently on their streams, so one
    # chain's copies overlap the others' kernels
    host_ring = torch.from_numpy(ring_h).pin_memory()
    d_stage = [torch.empty(B, N, 3, dtype=torch.float32, device=dev) for _ in range(S)]
    host_idx = [torch.empty(B, n_SAMPLES, dtype=torch.int64).pin_memory() for _ in range(S)]
    host_grp = [torch.empty(B, n_SAMPLES, K, dtype=torch.int32).pin_memory() for _ in range(S)]
    host_st = [torch.empty(B, dtype=torch.int32).pin_memory() for _ in range(S)]
    h2d = B * N * 3 * 4
    d2h = host_idx[0].numel() * 8 + host_grp[0].numel() * 4 + B * 4
    ci = {id(c): i for i, c in enumerate(chains)}

    def feed_host(c, s):
        i = ci[id(c)]
        d_stage[i].copy_(host_ring[s % R], non_blocking=True)
        c.fp.set_points(d_stage[i])

    def out_host(c, s):
        i = ci[id(c)]
        host_idx[i].copy_(c.fp.out, non_blocking=True)
        host_grp[i].copy_(c.grp[0], non_blocking=True)
        host_st[i].copy_(c.fp.csr.status, non_blocking=True)

    run_chains(chains, S, feed_host, out_host)
    if ws > 1:
        dist.barrier()
    e2e_ms = max_over_ranks(run_chains(chains, args.steps, feed_host, out_host), dev)
    e2e_value = ws * B * n_SAMPLES * args.steps / (e2e_ms / 1e3)
    if any(int(h.max()) != 0 for h in host_st):
        raise RuntimeError("exclusion capacity exhausted during the e2e run (status set)")
    # the last step's downloaded indices equal a fresh run on its batch
    fp.set_points(ring_d[last % R])
    chains[0].body()
    torch.cuda.synchronize()
    e2e_ok = bool(np.array_equal(host_idx[last % S].numpy(), fp.out.cpu().numpy()))
    fp.set_points(ring_d[0])
    chains[0].body()
    torch.cuda.synchronize()

    # ---- quality and early termination on the rank-0 batch --------
    exact_idx, _, _, _ = engine.fps(fp.xyz4, n_SAMPLES)
    sp_f = engine.min_spacing_d2(fp.xyz4, fp.out).sqrt().mean(dim=1)
    sp_x = engine.min_spacing_d2(fp.xyz4, exact_idx).sqrt().mean(dim=1)
    quality = (sp_f / sp_x).cpu().numpy()
    et_frac = (n_SAMPLES - reached) / n_SAMPLES

    # ---- roofline for the dominant kernel ------------------------------------------
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    dom = max(per_stage, key=per_stage.get)
    k0 = fp.k0
    E = int(fp.csr.counts.amax(dim=1).sum().item())  # entries of the widest level, all clouds
    alg = {  # algorithmic bytes per launch
        "fps_prefix": 28.0 * N * (k0 - 1) * B,
        "excl_build": 12.0 * E + 4.0 * N * fp.L * B + 16.0 * N * B,
        "sampler": 4.0 * E + 4.0 * N * fp.L * B,
        "early_term": 28.0 * N * float(np.sum(n_SAMPLES - reached)) + 12.0 * E,
        "rf_ball_query": 24.0 * n_SAMPLES * K * B,
        "thresholds": 8.0 * n_SAMPLES * B,
    }
    achieved = alg[dom] / (per_stage[dom] / 1e3) / 1e9
    traffic = None
    for rnd in ("r02", "r01"):
        try:  # measured DRAM bytes per launch from the committed ncu --set full capture
            traffic = json.load(open(os.path.join(REPO, "profiles", rnd, "traffic.json"))).get(dom)
            if traffic is not None:
                break
        except (OSError, ValueError):
            pass
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "algorithmic_bytes": alg[dom],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in pk else "fallback 6.65 TB/s",
                "note": ("algorithmic bytes per SURVEY 8d (28 B per point-iteration for FPS, the bytes a kernel "
                         "streaming xyz/md every iteration would move); K1 keeps xyz/md in registers (measured "
                         "DRAM traffic ~1000x lower) and certifies several samples per exchange, so frac compares "
                         "it with such a streaming kernel at HBM speed -- it is bound by its exchange/pick "
                         "latency chain, not by DRAM")}
    if dom == "fps_prefix":
        # the bound that actually applies: one cluster exchange (DSMEM send + wait, 400-600 SM cycles measured,
        # profiles/r01 micro_sync.log) per group of certified picks; picks per exchange from the instrumented
        # build (profiles/r02/fps_spec_phase_cycles.log)
        picks_per_ex = 4.87
        us_per_sample = per_stage[dom] * 1e3 / max(k0 - 1, 1)
        cyc_ex = us_per_sample * picks_per_ex * pk.get("sm_max_mhz", 1965.0)
        roofline["latency_model"] = {
            "us_per_sample": us_per_sample, "picks_per_exchange": picks_per_ex,
            "sm_cycles_per_exchange": cyc_ex, "exchange_floor_cycles": 500.0,
            "frac": 500.0 / cyc_ex,
            "note": "fraction of each exchange spent in the unavoidable cluster round trip; the rest is the lead "
                    "warp's serial pick chain (~550-700 cycles per certified pick)"}

    # ---- other configs ------------------------------------------------------------------
    c5 = c5f = c2 = c4 = None
    if not args.no_c5 and ws == 1:
        c5 = bench_c5_virtual(dev)
        c5f = bench_c5_fastpoint(dev)
    elif args.c5_split and ws > 1:
        c5 = bench_c5_split(dev, ws)
    if not args.no_extra and ws == 1:
        c2 = bench_c2_cascade(dev, args.steps)
        c4 = bench_c4(dev, args.steps)

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(clouds, exponent, fp.out.cpu().numpy(), args.cpu_runs)

    if rank == 0:
        ms_step = t_ms / args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(ws, exponent),
            "method": {"streams": S,
                       "l2": (f"inputs larger than L2: a ring of {R} distinct batches "
                              f"({R * B * N * 12 / 2**20:.0f} MiB of float32 coordinates) cycled step by step; "
                              "stage breakdown: 512 MiB flush between steps")},
            "timing": (f"device events around the whole loop of K steps (steps back to back on {S} streams, "
                       "step s on stream s % S, each step = set_points + one CUDA graph of sample + rf grouping)"),
            "us_per_cloud": 1e3 * ms_step / B,
            "one_stream": {"ms_per_step": t1_ms / args.steps, "value": ws * B * n_SAMPLES / (t1_ms / args.steps / 1e3),
                           "note": "one chain, latency-mode FPS cluster width, steps back to back"},
            "stage_ms": per_stage,
            "stage_sum_ms": float(sum(per_stage.values())),
            "stage_ms_inflight": per_stage_inflight,
            "stage_note": ("stage_ms: one chain, each stage alone at its latency-mode width (FPS: widest "
                           "co-resident clusters); stage_ms_inflight: the same stages with the throughput-hint FPS "
                           "width the concurrent chains use; timeline: profiles/r02/timeline_c3_5chains.txt"),
            "exact_fps_path": {"ms_per_step": exact_ms, "ms_per_step_one_stream": exact1_ms,
                               "fps_ms": float(np.mean(fps_ms)), "ball_query_naive_ms": float(np.mean(bqn_ms)),
                               "value": ws * B * n_SAMPLES / (exact_ms / 1e3), "us_per_cloud": 1e3 * exact_ms / B,
                               "kernels": "fps_spec (speculative exact FPS) + bq_naive, same loop, ring and streams"},
            "speedup_vs_exact_fps": exact_ms / ms_step,
            "speedup_vs_exact_fps_one_stream": exact1_ms / (t1_ms / args.steps),
            "speedup_vs_exact_fps_kernel_only": float(np.mean(fps_ms)) / (t1_ms / args.steps),
            "quality_ratio": {"mean": float(np.mean(quality)), "min": float(np.min(quality)),
                              "def": "avg_min_spacing(FastPoint) / avg_min_spacing(exact FPS), SPEC.md:573-581"},
            "early_term_frac": {"mean": float(np.mean(et_frac)), "max": float(np.max(et_frac)),
                                "def": "(n - reached) / n, SPEC.md:703"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms / args.steps, "results_match_device": e2e_ok and replay_ok,
                    "note": (f"pinned H2D of the step's batch (ring of {R}) + set_points + sample + group_rf + D2H of "
                             f"indices, groups and exclusion status, every step, {S} chains on their own streams "
                             "(copies of one overlap the kernels of the others)")},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "c5_point_split": c5,
            "c5_fastpoint": c5f,
            "c2_cascade": c2,
            "c4_large_clouds": c4,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


C5_N, C5_n = 1 << 20, 65536


def _time_graph(fn, reps=10):
    import torch

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def bench_c2_cascade(dev, steps):
    """C2: B=32 unit-sphere clouds, N=1024, four stride-2 set-abstraction
    stages (1024->512->256->128->64), ball query r_s = 0.15*1.5^s, k=32:
    FastPoint on stage 0 (rf grouping) + exact FPS later vs all-exact FPS +
    naive grouping; each cascade one CUDA graph, inputs resident."""
    import torch

    from paper_2507_23480_b200 import curve, engine
    from paper_2507_23480_b200.harness import generate_cloud

    B, Nc = 32, 1024
    held = np.stack([generate_cloud("unit-sphere", Nc, 77000 + i) for i in range(HELDOUT)])
    _, cv, _, _ = engine.fps(engine.as_xyz4(torch.from_numpy(held).to(dev)), Nc // 2)
    e = curve.fit_power_exponent(cv.cpu().numpy())
    clouds = np.stack([generate_cloud("unit-sphere", Nc, 2000 + b) for b in range(B)])
    res = {}
    for first in ("fastpoint", "fps"):
        sa = engine.SACascade(B, Nc, first=first, exponent=e, device=dev)
        sa.set_points(torch.from_numpy(clouds).to(dev))
        sa.set_rng(list(range(B)))
        sa.run()
        sa.fp.check() if first == "fastpoint" else None
        sa.capture()
        res[first] = _time_graph(sa.run, max(steps, 5))
    return {"workload": "C2: B=32 unit-sphere clouds N=1024, 4 SA stages stride 2 (->512->256->128->64), "
                        "r_s=0.15*1.5^s, k=32", "exponent": round(e, 6),
            "fastpoint_first_ms": res["fastpoint"], "all_exact_fps_ms": res["fps"],
            "us_per_cloud": 1e3 * res["fastpoint"] / B, "speedup_vs_exact": res["fps"] / res["fastpoint"],
            "sampled_pts_per_s": B * (512 + 256 + 128 + 64) / (res["fastpoint"] / 1e3),
            "timing": "CUDA graph replay, mean of >=5"}


def bench_c4(dev, steps):
    """C4 per-GPU share at 8 GPUs: B=2 room clouds N=65536 -> n=16384
    FastPoint + rf ball query (r=0.1, k=32) vs exact FPS + naive ball query."""
    import torch

    from paper_2507_23480_b200 import curve, engine
    from paper_2507_23480_b200.harness import generate_cloud

    B, Nc, nc = 2, 65536, 16384
    held = np.stack([generate_cloud(FAMILY, Nc, 88000 + i) for i in range(HELDOUT)])
    _, cv, _, _ = engine.fps(engine.as_xyz4(torch.from_numpy(held).to(dev)), nc)
    e = curve.fit_power_exponent(cv.cpu().numpy())
    clouds = np.stack([generate_cloud(FAMILY, Nc, 3000 + b) for b in range(B)])
    fp = engine.FastPoint(B, Nc, nc, p=P, nseg=NSEG, estimator="power", exponent=e, extra_radii=(RADIUS,), device=dev)
    fp.set_points(torch.from_numpy(clouds).to(dev))
    grp = (torch.empty(B, nc, K, dtype=torch.int32, device=dev), torch.empty(B, nc, K, dtype=torch.float64, device=dev),
           torch.empty(B, nc, dtype=torch.int32, device=dev))
    seeds = torch.arange(B, dtype=torch.int64, device=dev)

    def ours():
        fp.state.copy_(seeds)
        fp.sample()
        fp.group_rf(RADIUS, K, out=grp)

    ours()
    fp.check()
    ms = _time_graph(ours, max(2, min(steps, 5)))

    def exact():
        idx, _, _, _ = engine.fps(fp.xyz4, nc)
        engine.ball_query_naive(fp.xyz4, idx, RADIUS, K)

    exact()
    ms_x = _time_graph(exact, 2)
    return {"workload": "C4 per-GPU share at 8 GPUs: B=2 room clouds N=65536 -> n=16384, FastPoint + rf ball "
                        "query r=0.1 k=32", "ms": ms, "us_per_cloud": 1e3 * ms / B,
            "sampled_pts_per_s": B * nc / (ms / 1e3), "exact_fps_path_ms": ms_x, "speedup_vs_exact": ms_x / ms,
            "exponent": round(e, 6)}


def bench_c5_virtual(dev, G=None):
    """C5: exact FPS of one N = 2^20 uniform-box cloud to n = 65536, the cloud
    split over G ranks that exchange shard headers and candidate sets through
    the NVLink mailbox protocol (one exchange per certified run of samples)
    -- here all ranks on this GPU (virtual ranks;
    the one-process-per-GPU run is pointsplit.PointSplitFPS).  Timed with CUDA
    events on the launching stream; inputs resident."""
    import ctypes

    import torch

    from paper_2507_23480_b200 import _lib, engine
    from paper_2507_23480_b200.harness import generate_cloud

    cloud = generate_cloud("uniform-box", C5_N, 5000)
    x = engine.as_xyz4(torch.from_numpy(cloud[None]).to(dev))
    cands = [G] if G else [10, 12, 16, 8]
    for g in cands:
        C, Pp = ctypes.c_int32(), ctypes.c_int32()
        if _lib.raw("ps_fps_split_plan", C5_N, 1, g, g, ctypes.byref(C), ctypes.byref(Pp)) == 0:
            G = g
            break
    else:
        return {"unavailable": "no co-resident virtual-rank plan"}
    mb = engine.SplitMailboxes(1, G, dev)
    engine.fps_split(x, C5_n, G, mailboxes=mb, k_stop=1024)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    idx, curve, _, _ = engine.fps_split(x, C5_n, G, mailboxes=mb)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ok = bool(torch.all(idx >= 0).item()) and int(torch.unique(idx).numel()) == C5_n and bool(
        torch.all(curve[0, 2:] <= curve[0, 1:-1]).item())
    return {"workload": "C5: 1 cloud N=2^20 uniform-box -> n=65536 exact FPS, point split", "ranks": G,
            "cluster_ctas": C.value, "points_per_thread": Pp.value, "mode": "virtual ranks on one GPU",
            "ms": ms, "us_per_iter": 1e3 * ms / (C5_n - 1), "sampled_pts_per_s": C5_n / (ms / 1e3),
            "checks": "distinct indices, non-increasing curve" if ok else "FAILED property checks",
            "parity": "bit-identical to the single-rank kernel (tests/test_gpu_parity.py, tools/c5_split.py)"}


C5_EXPONENT, C5_RADIUS = 0.368508, 0.04  # tests/golden/make_c5_digest.py (fitted on a held-out cloud)


def bench_c5_fastpoint(dev, reps=3):
    """C5 FastPoint on one GPU: one N = 2^20 uniform-box cloud -> n = 65536,
    p = 0.1, nseg = 6, power estimator, rf ball query r = 0.04 k = 32 -- the
    prefix and the early-termination tail run as the point split over
    virtual ranks inside ps_fps.  One CUDA graph per sample + grouping,
    inputs resident, device events; against exact FPS + naive ball query on
    the same cloud.  Indices are compared with the oracle digest."""
    import hashlib

    import torch

    from paper_2507_23480_b200 import engine
    from paper_2507_23480_b200.harness import generate_cloud

    cloud = generate_cloud("uniform-box", C5_N, 5000)
    fp = engine.FastPoint(1, C5_N, C5_n, p=P, nseg=NSEG, exponent=C5_EXPONENT, extra_radii=(C5_RADIUS,), device=dev)
    fp.set_points(torch.from_numpy(cloud[None]).to(dev))
    grp = (torch.empty(1, C5_n, K, dtype=torch.int32, device=dev),
           torch.empty(1, C5_n, K, dtype=torch.float64, device=dev),
           torch.empty(1, C5_n, dtype=torch.int32, device=dev))
    seed = torch.zeros(1, dtype=torch.int64, device=dev)

    def body():
        fp.state.copy_(seed)
        fp.sample()
        fp.group_rf(C5_RADIUS, K, out=grp)

    body()
    torch.cuda.synchronize()
    fp.check()
    # stage breakdown (one eager run, events on the launching stream)
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    fp.state.copy_(seed)
    ev[0].record(st)
    fp._prefix()
    ev[1].record(st)
    fp._thresholds()
    ev[2].record(st)
    fp._exclusion()
    ev[3].record(st)
    fp._sampler()
    ev[4].record(st)
    fp._early_termination()
    ev[5].record(st)
    fp.group_rf(C5_RADIUS, K, out=grp)
    ev[6].record(st)
    torch.cuda.synchronize()
    stage_ms = {nm: ev[i].elapsed_time(ev[i + 1]) for i, nm in enumerate(
        ["fps_prefix", "thresholds", "excl_build", "sampler", "early_term", "rf_ball_query"])}
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    g.replay()
    ms = _time_graph(g.replay, reps)
    try:
        dig = json.load(open(os.path.join(REPO, "tests", "golden", "c5_digest.json")))["fastpoint"]["idx_sha256"]
    except (OSError, ValueError, KeyError):
        dig = None
    got = hashlib.sha256(fp.out[0].cpu().numpy().astype(np.int64).tobytes()).hexdigest()
    reached = int(fp.reached[0].item())

    def exact():
        idx, _, _, _ = engine.fps(fp.xyz4, C5_n)
        engine.ball_query_naive(fp.xyz4, idx, C5_RADIUS, K)

    exact()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    idx, _, _, _ = engine.fps(fp.xyz4, C5_n)
    e1.record()
    engine.ball_query_naive(fp.xyz4, idx, C5_RADIUS, K)
    e2.record()
    torch.cuda.synchronize()
    fps_ms, bq_ms = e0.elapsed_time(e1), e1.elapsed_time(e2)
    return {"workload": "C5 FastPoint: 1 cloud N=2^20 uniform-box -> n=65536, p=0.1, nseg=6, power estimator "
                        f"(e={C5_EXPONENT}), rf ball query r={C5_RADIUS} k={K}; one GPU",
            "ms": ms, "stage_ms": stage_ms, "sampled_pts_per_s": C5_n / (ms / 1e3), "reached": reached,
            "early_term_frac": (C5_n - reached) / C5_n, "entries": int(fp.csr.counts[0].amax(dim=0).sum().item()),
            "exact_fps_ms": fps_ms, "ball_query_naive_ms": bq_ms,
            "speedup_vs_exact_fps": (fps_ms + bq_ms) / ms, "speedup_vs_exact_fps_kernel_only": fps_ms / ms,
            "indices_match_oracle_digest": (got == dig) if dig else None,
            "timing": f"CUDA graph replay (sample + rf grouping), mean of {reps}; exact path eager, one run"}


def bench_c5_split(dev, ws):
    """C5 over the job's GPUs, one process per GPU (pointsplit.PointSplitFPS:
    cudaMalloc mailboxes mapped into every peer through CUDA IPC, NVLink
    stores; no NCCL on the data path).  Device time, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2507_23480_b200 import engine, pointsplit
    from paper_2507_23480_b200.harness import generate_cloud

    cloud = generate_cloud("uniform-box", C5_N, 5000)
    x = engine.as_xyz4(torch.from_numpy(cloud[None]).to(dev))
    ps = pointsplit.PointSplitFPS(1, C5_N, device=dev)
    ps.run(x, C5_n, k_stop=1024)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    idx, curve, _, _ = ps.run(x, C5_n)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), dev)
    ok = int(torch.unique(idx).numel()) == C5_n
    dist.barrier()
    ps.close()
    # C5 FastPoint over the same ranks (pointsplit.PointSplitFastPoint: split
    # prefix + tail, row-sharded build, rows to rank 0 for the sampler,
    # centroid-sharded grouping); host-timed collectives included
    mp = pointsplit.PointSplitFastPoint(C5_N, C5_n, exponent=C5_EXPONENT, extra_radii=(C5_RADIUS,), device=dev)
    mp.run(x, 0, K, C5_RADIUS)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    fidx, _ = mp.run(x, 0, K, C5_RADIUS)
    e1.record()
    torch.cuda.synchronize()
    fms = max_over_ranks(e0.elapsed_time(e1), dev)
    import hashlib

    try:
        dig = json.load(open(os.path.join(REPO, "tests", "golden", "c5_digest.json")))["fastpoint"]["idx_sha256"]
    except (OSError, ValueError, KeyError):
        dig = None
    got = hashlib.sha256(fidx.cpu().numpy().astype(np.int64).tobytes()).hexdigest()
    mp.close()
    return {"workload": "C5: 1 cloud N=2^20 uniform-box -> n=65536 exact FPS, point split", "ranks": ws,
            "mode": "one process per GPU, CUDA-IPC mailboxes over NVLink", "ms": ms,
            "us_per_iter": 1e3 * ms / (C5_n - 1), "sampled_pts_per_s": C5_n / (ms / 1e3),
            "checks": "distinct indices" if ok else "FAILED property checks",
            "fastpoint_ms": fms, "fastpoint_sampled_pts_per_s": C5_n / (fms / 1e3),
            "fastpoint_matches_oracle_digest": (got == dig) if dig else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=256)  # 8 chains x 32 steps: past the ramp-up, ~0.14 s timed
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 point-split line")
    ap.add_argument("--no-extra", action="store_true", help="skip the C2 / C4 objects")
    ap.add_argument("--streams", type=int, default=8, help="concurrent FastPoint chains (streams)")
    ap.add_argument("--cpu-runs", type=int, default=5, help="timed CPU-baseline runs per thread setting (median)")
    ap.add_argument("--c5-split", action="store_true",
                    help="N > 1: also run C5 point-split over the job's GPUs (CUDA IPC + NVLink)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
