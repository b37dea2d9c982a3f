# round-2 evidence: bench line, step launch lists (latency-mode and inflight widths), full-set capture of the step
python bench.py --steps 30 > gpurun_out/bench_final.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step_inflight.csv python tools/profile_step.py --inflight 40 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/step_full python tools/profile_step.py > /dev/null 2>&1
ls -la gpurun_out
