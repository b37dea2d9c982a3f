python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
SAN_TIMEOUT=900 bash tools/sanitize.sh memcheck racecheck > /dev/null 2>&1; grep -E "mdps|grouping" gpurun_out/sanitize/summary.txt
