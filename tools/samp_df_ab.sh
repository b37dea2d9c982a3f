# sampler MIS: dataflow (default) vs barrier-separated rounds (PS_SAMPLER_ROUNDS=1)
timeout 600 python -m pytest tests -m gpu -q -x -k "mdps or sampler or golden or cascade or c5 or acceptance or split" 2>&1 | tail -1
python tools/samp_width_ab.py; PS_SAMPLER_ROUNDS=1 python tools/samp_width_ab.py
python tools/samp_width_ab.py --c4; PS_SAMPLER_ROUNDS=1 python tools/samp_width_ab.py --c4
PS_SAMPLER_TIMING=1 python tools/sampler_timing.py 2>&1 | tail -2
