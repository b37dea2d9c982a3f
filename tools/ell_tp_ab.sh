# C3 throughput (bench, 5 chains) with the cell kernel (default) vs the row kernel (PS_ELL_ROW=1), interleaved x2
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 30 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value']/1e6,2), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,2), '1-stream', round(d['one_stream']['ms_per_step'],3), 'excl', round(d['stage_ms']['excl_build'],3))"; }
python -m pytest tests/test_gpu_parity.py -x -q -k "excl or mdps_batched" 2>&1 | tail -1
for r in 1 2; do q cell; PS_ELL_ROW=1 q row; done
ncu --set full --import-source on --clock-control none -k regex:grid_ell --launch-skip 3 -c 1 -o gpurun_out/ell_cell python tools/excl_ab.py > /dev/null 2>&1
