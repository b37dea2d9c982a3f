"""Group compute-sanitizer racecheck hazards by (kind, source pair)."""
import collections
import re
import sys

for path in sys.argv[1:]:
    pairs = collections.Counter()
    cur = None
    for ln in open(path, errors="replace"):
        m = re.search(r"(Error|Warning): (.*?)hazard detected", ln)
        if m:
            if cur:
                pairs[(cur[0], tuple(cur[1]))] += 1
            cur = [m.group(1) + ": " + m.group(2).strip(), []]
            continue
        m = re.search(r"(Read|Write) Thread .* at (?:void )?([\w:]+?)(?:<|\().* in (\S+:\d+)", ln)
        if m and cur is not None:
            cur[1].append(f"{m.group(1)} {m.group(3)}")
    if cur:
        pairs[(cur[0], tuple(cur[1]))] += 1
    print(f"== {path}")
    for (k, locs), c in pairs.most_common():
        print(f"  {c:4d}  {k:55s} {' | '.join(locs)}")
