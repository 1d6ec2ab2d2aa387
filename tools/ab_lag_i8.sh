#!/bin/bash
# lag stage: int8 (default) vs bf16x2 (SA_LAG_KIND=bf16) kernels, C4 and C5, device-resident
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lag_tc.py -q -x -p no:cacheprovider 2>&1 | tail -15
for k in i8 bf16; do
  for c5 in 0 1; do
    SA_LAG_KIND=$k C5=$c5 timeout 300 python tools/time_map.py 2>&1 | sed "s/^/$k /" | grep -v complex128
  done
done
