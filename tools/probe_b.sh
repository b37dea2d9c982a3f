#!/bin/bash
# sampler per-phase cycles (C3), C2 cascade launch list, small-cloud FPS per-iteration times
set -x
mkdir -p gpurun_out
timeout 300 python tools/sampler_timing.py > gpurun_out/samp_timing.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c2_launches.csv python tools/profile_c2.py > gpurun_out/c2_prof.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c2_launches_exact.csv python tools/profile_c2.py exact >> gpurun_out/c2_prof.log 2>&1
timeout 300 python tools/c2_ab.py > gpurun_out/c2_ab.log 2>&1
