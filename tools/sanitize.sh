#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py, one process per (tool, case),
# each bounded by a timeout; logs under gpurun_out/sanitize/.
#   bash tools/sanitize.sh [tool ...]    (default: memcheck racecheck synccheck initcheck)
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p $OUT
TOOLS=${@:-memcheck racecheck synccheck initcheck}
CASES=$(python -c "import sys; sys.argv=['x']; exec(open('tools/sanitize_cases.py').read().split('CASES =')[0]); print(' '.join(k[5:] for k in list(globals()) if k.startswith('case_')))" 2>/dev/null)
[ -z "$CASES" ] && CASES="fps_small fps_spec fps_cluster fps_resident fps_split mdps_smem mdps_global mdps_sorted_csr grouping cascade"
for t in $TOOLS; do
  # torch's own kernels are not checked (their writes still count as
  # initialisation for initcheck, which therefore checks every kernel)
  extra="--kernel-name-exclude kns=at6native"
  [ "$t" = "racecheck" ] && extra="$extra --racecheck-report all"
  [ "$t" = "memcheck" ] && extra="$extra --leak-check no"
  [ "$t" = "initcheck" ] && extra=""
  for c in $CASES; do
    log=$OUT/${t}_${c}.log
    timeout ${SAN_TIMEOUT:-600} compute-sanitizer --tool $t $extra \
        python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" $log | tail -2 | tr '\n' ' ')
    echo "$t $c rc=$rc $summ" | tee -a $OUT/summary.txt
  done
done
