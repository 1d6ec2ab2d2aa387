#!/bin/bash
# full evidence pass: GPU tests (+ printed parity figures), smoke, bench, lag-kernel ncu, bench launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_round.sh
timeout 300 python -m pytest tests/test_gpu_ndft_i8.py tests/test_gpu_ndft_tc.py -q -s -p no:cacheprovider -k "c2 or C2" > gpurun_out/parity_print.log 2>&1
bash tools/gpu_prof_lag.sh
B="python bench.py --steps 3 --warmup 3 --no-extras --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
