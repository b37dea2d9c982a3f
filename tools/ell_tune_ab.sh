python -m pytest tests/test_gpu_parity.py -x -q -k "excl or mdps_batched or bucketed" 2>&1 | tail -1
PS_ELL_C32=1 python -m pytest tests/test_gpu_parity.py -x -q -k "bucketed" 2>&1 | tail -1
python tools/excl_ab.py; PS_ELL_C32=1 python tools/excl_ab.py
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 30 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value']/1e6,2), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,2), '1-stream', round(d['one_stream']['ms_per_step'],3), 'excl', round(d['stage_ms']['excl_build'],3))"; }
q c16; PS_ELL_C32=1 q c32; q c16; PS_ELL_C32=1 q c32
ncu --set full --import-source on --clock-control none -k regex:grid_ell --launch-skip 3 -c 1 -o gpurun_out/ell_tune python tools/excl_ab.py > /dev/null 2>&1
