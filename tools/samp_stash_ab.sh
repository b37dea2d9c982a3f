python -m pytest tests -m gpu -q -x -k "mdps or sampler or golden or cascade or c5 or acceptance or split or dropin" 2>&1 | tail -1 > gpurun_out/t.log
python tools/samp_width_ab.py >> gpurun_out/t.log; python tools/samp_width_ab.py >> gpurun_out/t.log
python tools/samp_width_ab.py --c4 >> gpurun_out/t.log
PS_SAMPLER_TIMING=1 python tools/sampler_timing.py 2>&1 | tail -3 >> gpurun_out/t.log
cat gpurun_out/t.log
