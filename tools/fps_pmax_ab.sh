#!/bin/bash
# FPS prefix / full run at forced cluster widths with more points per thread (PS_SPEC_PMAX=13), C3 batch:
# SM-time per cloud = C x time
export PS_SPEC_PMAX=13
for C in 6 5 4 6 5 4; do
  LABEL="C=$C" PS_SPEC_C=$C python tools/fps_prefix_time.py 2>&1 | tail -1
done
unset PS_SPEC_PMAX
LABEL="default-latency" python tools/fps_prefix_time.py 2>&1 | tail -1
LABEL="default-inflight40" python tools/fps_prefix_time.py --inflight 40 2>&1 | tail -1
