#!/bin/bash
# sampler A/B: build_ab/base (HEAD) vs the working-tree lib (and PS_SAMPLER_NOD16=1), interleaved
L0=build_ab/base/paper_2507_23480_b200/libps_b200.so
for rep in 1 2; do
  for v in base new no16; do
    unset PS_B200_LIB PS_SAMPLER_NOD16
    [ $v = base ] && export PS_B200_LIB=$L0
    [ $v = no16 ] && export PS_SAMPLER_NOD16=1
    echo "$v C3 $(python tools/samp_width_ab.py 2>/dev/null | tail -1)"
  done
done
unset PS_B200_LIB PS_SAMPLER_NOD16
PS_SAMPLER_TIMING=1 python tools/sampler_timing.py 2>&1 | tail -3
