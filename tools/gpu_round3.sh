#!/bin/bash
# evidence pass: GPU tests, smoke, bench, ncu of the changed kernels, bench launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_round.sh
timeout 300 python -m pytest tests/test_gpu_ndft_i8.py tests/test_gpu_ndft_tc.py -q -s -p no:cacheprovider -k "c2 or C2" > gpurun_out/parity_print.log 2>&1
SPECS="tc8fused:k_ndft_i8:ndft_tc8:c64 lagi8:k_lag_i8:map:c64 lagi8_5:k_lag_i8:map5:c64 cprep5:k_lag_cprep:map5:c64" bash tools/gpu_prof_lag.sh
B="python bench.py --steps 3 --warmup 3 --no-extras --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 300 python tools/time_map_blocks.py > gpurun_out/map_blocks.log 2>&1
