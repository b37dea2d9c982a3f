"""Timeline of the bench's concurrent C3 loop: S FastPoint chains on their own
streams (step s on chain s % S), every stage bracketed by CUDA events (eager
launches instead of the bench's graph replays, same kernels and widths).
Prints per-step stage intervals and an ASCII Gantt chart (one row per chain,
10 us per character) -- the evidence that one chain's FPS prefix overlaps the
others' exclusion rows / sampler / early termination.

  python tools/timeline.py [--streams S] [--steps K]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

S = int(sys.argv[sys.argv.index("--streams") + 1]) if "--streams" in sys.argv else 5
K = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 15
dev = torch.device("cuda", 0)
B = bench.B_PER_GPU
ring = torch.from_numpy(bench.input_ring(0, B)).to(dev)
R = ring.shape[0]
e = bench.heldout_exponent()
chains = [bench.Chain(B, e, dev, list(range(B)), inflight=B * S if S > 1 else None) for _ in range(S)]
for c in chains:
    c.fp.set_points(ring[0])
    with torch.cuda.stream(c.stream):
        c.body()
torch.cuda.synchronize()
for c in chains:
    c.fp.check()
names = ["prefix", "thresh", "excl", "sampler", "et", "bq"]
marks = "PTXSEB"


def step(c, ev):
    fp = c.fp
    fp.state.copy_(c.seed_t)
    ev[0].record()
    fp._prefix()
    ev[1].record()
    fp._thresholds()
    ev[2].record()
    fp._exclusion()
    ev[3].record()
    fp._sampler()
    ev[4].record()
    fp._early_termination()
    ev[5].record()
    fp.group_rf(bench.RADIUS, bench.K, out=c.grp)
    ev[6].record()


def run(record):
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for c in chains:
        c.stream.wait_event(t0)
    evs = []
    for s in range(K):
        c = chains[s % S]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        with torch.cuda.stream(c.stream):
            c.fp.set_points(ring[s % R])
            step(c, ev)
        evs.append((s % S, ev))
    for c in chains:
        torch.cuda.current_stream().wait_stream(c.stream)
    torch.cuda.synchronize()
    return t0, evs


run(False)
t0, evs = run(True)
rows = []
for ci, ev in evs:
    ts = [t0.elapsed_time(x) * 1e3 for x in ev]  # us
    rows.append((ci, ts))
end = max(r[1][-1] for r in rows)
print(f"# tools/timeline.py: S={S} chains, K={K} steps of the C3 batch (B={B}, N={bench.N} -> {bench.n_SAMPLES}),"
      f" eager launches; {end:.0f} us in total = {end / K:.0f} us per step")
print("# step chain  " + "  ".join(f"{n:>14s}" for n in names) + "   (start-end, us)")
for s, (ci, ts) in enumerate(rows):
    print(f"{s:6d} {ci:5d}  " + "  ".join(f"{ts[i]:6.0f}-{ts[i + 1]:6.0f}" for i in range(6)))
res = 10.0
width = int(end / res) + 1
print(f"\n# Gantt, {res:.0f} us per character: " + ", ".join(f"{m}={n}" for m, n in zip(marks, names)) + ", . idle")
for ci in range(S):
    line = ["."] * width
    for c, ts in rows:
        if c != ci:
            continue
        for i in range(6):
            a, b = int(ts[i] / res), int(ts[i + 1] / res)
            for x in range(a, max(a + 1, b)):
                if x < width:
                    line[x] = marks[i]
    print(f"chain {ci}: " + "".join(line))
# overlap: fraction of the time more than one chain is inside a stage
busy = [0] * width
for ci, ts in rows:
    for x in range(int(ts[0] / res), int(ts[6] / res) + 1):
        if x < width:
            busy[x] += 1
print(f"\n# chains busy per 10 us slot: mean {sum(busy) / width:.2f}, max {max(busy)}")
