#!/bin/bash
# compute-sanitizer memcheck / racecheck over the window-carry paths (device
# correction with residue / clip carries, sequential windows of an oversized
# process) and the correction suite with the 16-byte slab records.
cd "$(dirname "$0")/.."
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
timeout 1500 $CS --tool memcheck python -m pytest -q -x -m gpu tests/test_gpu_windows.py tests/test_gpu_huge_process.py \
  > gpurun_out/sanitize_memcheck_windows.log 2>&1
echo "memcheck windows rc=$?" | tee gpurun_out/sanitize_windows_summary.txt
tail -3 gpurun_out/sanitize_memcheck_windows.log >> gpurun_out/sanitize_windows_summary.txt
timeout 1500 $CS --tool memcheck python -m pytest -q -x -m gpu tests/test_gpu_correct.py \
  > gpurun_out/sanitize_memcheck_correct.log 2>&1
echo "memcheck correct rc=$?" | tee -a gpurun_out/sanitize_windows_summary.txt
tail -3 gpurun_out/sanitize_memcheck_correct.log >> gpurun_out/sanitize_windows_summary.txt
timeout 1500 $CS --tool racecheck --racecheck-report all python -m pytest -q -x -m gpu tests/test_gpu_windows.py \
  -k "instant and ddpg1" > gpurun_out/sanitize_racecheck_windows.log 2>&1
echo "racecheck windows rc=$?" | tee -a gpurun_out/sanitize_windows_summary.txt
tail -3 gpurun_out/sanitize_racecheck_windows.log >> gpurun_out/sanitize_windows_summary.txt
