#!/bin/bash
# grid_ell_cell occupancy variants (PS_ELL_V): exclusion stage alone and C3 throughput
q() { python bench.py --no-extra --no-c5 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), 'excl', round(d['stage_ms']['excl_build'],4))"; }
for rep in 1 2; do
  for v in 2 4 5 6; do
    echo "V=$v $(PS_ELL_V=$v python tools/excl_ab.py 2>/dev/null | tail -1)"
    PS_ELL_V=$v q "V=$v"
  done
done
