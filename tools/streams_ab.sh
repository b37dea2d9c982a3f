q() { python bench.py --no-extra --no-c5 --no-cpu --steps 20 --warmup 5 "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$L', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2))"; }
for r in 1 2 3; do L=S5 q --streams 5; L=S6 q --streams 6; L=S8 q --streams 8; done
