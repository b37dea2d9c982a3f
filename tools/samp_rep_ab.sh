timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do python tools/samp_width_ab.py; done
python tools/samp_width_ab.py --c4
python tools/sampler_timing_c2.py 2>&1 | tail -1
PS_SAMPLER_TIMING=1 python tools/sampler_timing.py 2>&1 | tail -3
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), '1-stream', round(d['one_stream']['ms_per_step'],4), 'samp', round(d['stage_ms']['sampler'],4))"; }
q rep; q rep
