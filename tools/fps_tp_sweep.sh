# C3 throughput with the shared-memory resident FPS kernel (fps_res.cu) at small cluster widths,
# speculative and one-sample, vs the default (fps_spec, throughput-hint width)
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value']/1e6,2), round(d['ms_per_step'],3), '1-stream', round(d['one_stream']['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items()}, 'ET', round(d['early_term_frac']['mean'],4))"; }
q default
for c in 2 3 4; do
  PS_FPS_RESIDENT=1 PS_FPS_CLUSTER=$c q res-spec-C$c
  PS_FPS_RESIDENT=1 PS_RES_NOSPEC=1 PS_FPS_CLUSTER=$c q res-nospec-C$c
done
