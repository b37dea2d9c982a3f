# fps_spec with 9 points per thread (no points on the lead warp) vs the lead owning points (PS_SPEC_NOP9=1) at C=6
PS_FPS_CLUSTER=6 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fps or mdps_batched" 2>&1 | tail -1
for r in 1 2; do
LABEL=p9-C6 PS_FPS_CLUSTER=6 python tools/fps_prefix_time.py
LABEL=lead-C6 PS_SPEC_NOP9=1 PS_FPS_CLUSTER=6 python tools/fps_prefix_time.py
done
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), '1-stream', round(d['one_stream']['ms_per_step'],4), 'infl', round(d['stage_ms_inflight']['fps_prefix'],4), round(d['stage_ms_inflight']['early_term'],4))"; }
for r in 1 2; do q p9; PS_SPEC_NOP9=1 q lead; done
