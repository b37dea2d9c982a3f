#!/bin/bash
# sampler A/B: build_ab/base (HEAD) vs the working tree (pair-mode MIS first pass) vs PS_SAMPLER_NOPAIR=1
L0=build_ab/base/paper_2507_23480_b200/libps_b200.so
for rep in 1 2; do
  for v in base new nopair; do
    unset PS_B200_LIB PS_SAMPLER_NOPAIR
    [ $v = base ] && export PS_B200_LIB=$L0
    [ $v = nopair ] && export PS_SAMPLER_NOPAIR=1
    echo "$v C3 $(python tools/samp_width_ab.py 2>/dev/null | tail -1)"
  done
done
unset PS_B200_LIB PS_SAMPLER_NOPAIR
PS_SAMPLER_TIMING=1 python tools/sampler_timing.py 2>&1 | tail -3
q() { python bench.py --no-extra --no-c5 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), '1s', round(d['one_stream']['ms_per_step'],4), 'samp', round(d['stage_ms']['sampler'],4))"; }
for rep in 1 2; do q new; PS_SAMPLER_NOPAIR=1 q nopair; done
