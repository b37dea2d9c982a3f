#!/bin/bash
# loop barrier variants: __syncthreads (build_ab/sync, HEAD) vs the working tree (producer-consumer named barriers)
for rep in 1 2; do
  for v in sync named2; do
    if [ $v = named2 ]; then unset PS_B200_LIB; else export PS_B200_LIB=build_ab/$v/paper_2507_23480_b200/libps_b200.so; fi
    for C in 5 6; do LABEL="$v C=$C" PS_SPEC_C=$C python tools/fps_prefix_time.py 2>&1 | tail -1; done
    LABEL="$v latency" python tools/fps_prefix_time.py 2>&1 | tail -1
  done
done
