# C3 throughput vs forced FPS width and chains after the round-2 kernel changes
q() { python bench.py --no-extra --no-c5 --no-cpu --steps 30 "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$L', round(d['value']/1e6,2), round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']/1e6,2))"; }
L=default q
for c in 7 8; do L=C$c PS_FPS_CLUSTER=$c q; done
L=S4 q --streams 4; L=S6 q --streams 6; L=S8 q --streams 8
L=default q
