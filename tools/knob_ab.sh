#!/bin/bash
# env-knob / chain-count A/B on the C3 bench (--no-extra), two passes
q() { python bench.py --no-extra --no-c5 --no-cpu $2 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), '1s', round(d['one_stream']['ms_per_step'],4))"; }
for rep in 1 2; do
  q default ""
  PS_SAMPLER_POLL=64 q samp_poll64 ""
  PS_SAMPLER_POLL=256 q samp_poll256 ""
  PS_SPEC_POLL_NS=64 q fps_poll64 ""
  PS_SPEC_POLL_NS=16 q fps_poll16 ""
  q streams10 "--streams 10"
  q streams12 "--streams 12"
done
