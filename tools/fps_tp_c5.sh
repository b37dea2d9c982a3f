#!/bin/bash
# C3 throughput bench: default chooser vs forced FPS widths (PS_SPEC_C)
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), '1-stream', round(d['one_stream']['ms_per_step'],4), 'infl', {k: round(v,3) for k,v in d['stage_ms_inflight'].items()})"; }
for rep in 1 2; do
  q default
  PS_SPEC_C=5 q forced5
  PS_SPEC_C=6 q forced6
done
