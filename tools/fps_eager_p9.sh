#!/bin/bash
# eager record refresh from P = 8 (working tree) vs from P = 10 (build_ab/p10): C3 at 6-CTA clusters (P = 9), C4
L0=build_ab/p10/paper_2507_23480_b200/libps_b200.so
for rep in 1 2; do
  for v in p10 p8; do
    if [ $v = p10 ]; then export PS_B200_LIB=$L0; else unset PS_B200_LIB; fi
    LABEL="$v C=6" PS_SPEC_C=6 python tools/fps_prefix_time.py 2>&1 | tail -1
    echo "$v c4 $(python -c "
import sys; sys.argv=['x']
import bench, json
print(json.dumps({k: round(v,4) if isinstance(v,float) else v for k,v in bench.bench_c4('cuda', 10).items() if k in ('ms','exact_fps_path_ms')}))
" 2>/dev/null | tail -1)"
  done
done
