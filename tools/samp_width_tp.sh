for c in 7 6; do PS_SAMPLER_CLUSTER=$c python tools/samp_width_ab.py; done
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 30 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$L', round(d['value']/1e6,2), round(d['ms_per_step'],3), 'samp', round(d['stage_ms']['sampler'],3))"; }
for r in 1 2; do L=default q; L=samp7 PS_SAMPLER_CLUSTER=7 q; done
