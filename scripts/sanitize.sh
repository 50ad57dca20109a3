#!/bin/bash
# compute-sanitizer over the GPU path: memcheck / racecheck / synccheck /
# initcheck on __graft_entry__.smoke() (correction + overlap + CORRELATION on
# a small 2-process trace) and memcheck on a golden-vector test subset.
# Logs -> gpurun_out/sanitize_<tool>.log (summaries copied to profiles/).
cd "$(dirname "$0")/.."
export XS_NO_GRAPHS=${XS_NO_GRAPHS:-0}
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/sanitize_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_${tool}_smoke.log >> gpurun_out/sanitize_summary.txt
done
timeout 2400 $CS --tool memcheck python -m pytest -q -x -m gpu tests/test_gpu_overlap.py tests/test_gpu_edge.py \
  -k "not single_pid_span" > gpurun_out/sanitize_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?" | tee -a gpurun_out/sanitize_summary.txt
tail -3 gpurun_out/sanitize_memcheck_tests.log >> gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck; do
  timeout 1200 $CS --tool $tool python scripts/sanitize_medium.py > gpurun_out/sanitize_${tool}_medium.log 2>&1
  echo "$tool medium rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_${tool}_medium.log >> gpurun_out/sanitize_summary.txt
done
