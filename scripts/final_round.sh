#!/bin/bash
# Round-end measurement on one B200: GPU suite, smoke, bench lines (configs
# 2/5/3), the reference arm, and the ncu launch list of the default bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputest.log 2>&1; echo rc=$? >> gpurun_out/final_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
timeout 600 python bench.py --config 5 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_c2.log 2>&1
timeout 1500 python -X faulthandler bench.py --config 3 > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
tail -2 gpurun_out/final_gputest.log; tail -1 gpurun_out/final_smoke.log
