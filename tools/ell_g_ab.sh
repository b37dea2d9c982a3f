# exclusion rows: G rows per warp (PS_ELL_G; 3 = two rows per warp in 2-warp CTAs) -- parity, stage time, C3 throughput
for G in 2 3 4; do
  PS_ELL_G=$G python -m pytest tests/test_gpu_parity.py -x -q -k "excl or mdps_batched" 2>&1 | tail -1
  PS_ELL_G=$G python tools/excl_ab.py
done
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 30 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value']/1e6,2), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,2), '1-stream', round(d['one_stream']['ms_per_step'],3), 'excl', round(d['stage_ms']['excl_build'],3))"; }
for r in 1 2; do for G in 2 3 4; do PS_ELL_G=$G q G$G; done; done
PS_ELL_G=4 ncu --set full --import-source on --clock-control none -k regex:grid_ell --launch-skip 3 -c 1 -o gpurun_out/ell_g4 python tools/excl_ab.py > /dev/null 2>&1
