# round-2 evidence: GPU tests, smoke, bench line, step launch lists (latency-mode and inflight widths),
# full-set capture of the step, C4 launch list
python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -1 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_final.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step_inflight.csv python tools/profile_step.py --inflight 40 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/step_full python tools/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/profile_c4.py > /dev/null 2>&1
ls gpurun_out | head -30
