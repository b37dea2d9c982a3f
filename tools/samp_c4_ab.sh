python tools/samp_width_ab.py --c4
PS_SAMPLER_GRID_CTAS=32 python tools/samp_width_ab.py --c4
PS_SAMPLER_GRID_CTAS=48 python tools/samp_width_ab.py --c4
for c in 8 12 16; do PS_SAMPLER_NOGRID=1 PS_SAMPLER_CLUSTER=$c python tools/samp_width_ab.py --c4; done
