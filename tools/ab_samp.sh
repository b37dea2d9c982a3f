#!/bin/bash
# sampler A/B: build_ab/base (HEAD) vs the working-tree lib (flattened P1 push, and PS_SAMPLER_PUSH_GROUPED=1), interleaved
L0=build_ab/base/paper_2507_23480_b200/libps_b200.so
for rep in 1 2; do
  for v in base new grp; do
    unset PS_B200_LIB PS_SAMPLER_PUSH_GROUPED
    [ $v = base ] && export PS_B200_LIB=$L0
    [ $v = grp ] && export PS_SAMPLER_PUSH_GROUPED=1
    echo "$v C3 $(python tools/samp_width_ab.py 2>/dev/null | tail -1)"
  done
done
unset PS_B200_LIB PS_SAMPLER_PUSH_GROUPED
PS_SAMPLER_TIMING=1 python tools/sampler_timing.py 2>&1 | tail -3
