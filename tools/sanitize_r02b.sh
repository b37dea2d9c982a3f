#!/bin/bash
# sanitizers over the kernels changed late in round 2 (split lead loop / P = 10, sampler push)
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize_b; mkdir -p $OUT
for t in memcheck racecheck synccheck initcheck; do
  for c in fps_spec_p10 fps_spec mdps_smem; do
    extra="--kernel-name-exclude kns=at6native"
    [ "$t" = "racecheck" ] && extra="$extra --racecheck-report all"
    [ "$t" = "memcheck" ] && extra="$extra --leak-check no"
    [ "$t" = "initcheck" ] && extra=""
    timeout 600 compute-sanitizer --tool $t $extra python tools/sanitize_cases.py $c > $OUT/${t}_${c}.log 2>&1
    echo "$t $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/${t}_${c}.log | tail -1)" | tee -a $OUT/summary.txt
  done
done
