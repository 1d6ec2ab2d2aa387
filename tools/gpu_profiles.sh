#!/bin/bash
# Round-end evidence: bench line, ncu launch list of the bench command, and
# ncu --set full captures of the hot kernels (each preceded by a clean run).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-extras --no-e2e --no-cpu"
$B > gpurun_out/plain_bench.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
bash tools/gpu_prof.sh ndft_tc:k_ndft_tc:ndft_tc:c64 ndft:k_ndft_fast:ndft:c64 ndft64:k_ndft_fast:ndft:c128 \
    nlfft64k:k_nlfft64k:nlfft:c64 nlfft64k_c128:k_nlfft64k:nlfft:c128 \
    nlfft64k_dif:k_nlfft64k:nlfft_dif:c64 lag:k_lag_tc:map:c64 detect:k_peaks_tile:detect:c64
