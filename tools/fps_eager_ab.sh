#!/bin/bash
# eager warp-record refresh (working tree) vs phase-B-only refresh (build_ab/noeager)
L0=build_ab/noeager/paper_2507_23480_b200/libps_b200.so
for rep in 1 2; do
  for v in noeager eager; do
    if [ $v = noeager ]; then export PS_B200_LIB=$L0; else unset PS_B200_LIB; fi
    for C in 5; do LABEL="$v C=$C" PS_SPEC_C=$C python tools/fps_prefix_time.py 2>&1 | tail -1; done
    LABEL="$v latency" python tools/fps_prefix_time.py 2>&1 | tail -1
  done
done
q() { python bench.py --no-extra --no-c5 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), '1s', round(d['one_stream']['ms_per_step'],4), 'pre', round(d['stage_ms']['fps_prefix'],4), 'et', round(d['stage_ms']['early_term'],4))"; }
for rep in 1 2; do export PS_B200_LIB=$L0; q noeager; unset PS_B200_LIB; q eager; done
