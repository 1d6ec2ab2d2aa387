#!/bin/bash
# final evidence pass: GPU tests, smoke, bench, ncu of the Doppler kernel, bench launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_round.sh
SPECS="doppler5:k_doppler:map5:c64" bash tools/gpu_prof_lag.sh
B="python bench.py --steps 3 --warmup 3 --no-extras --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
