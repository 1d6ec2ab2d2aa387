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
    ndft_i8:k_ndft_i8:ndft_tc:c128 i8prep:k_i8_prep:ndft_tc:c128 \
    nlfft64k:k_nlfft64k:nlfft:c64 nlfft64k_c128:k_nlfft64k:nlfft:c128 nlfft64k_dif:k_nlfft64k:nlfft_dif:c64 \
    nlfft64k_dif_c128:k_nlfft64k:nlfft_dif:c128 lag:k_lag_tc:map:c64 lag5:k_lag_tc:map5:c64 \
    doppler5:k_doppler:map5:c64 detect:k_peaks_tile:detect:c64
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB return limit)
python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep --out gpurun_out/round_kernels > gpurun_out/summary.log 2>&1
mkdir -p gpurun_out/src
for r in gpurun_out/prof_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page source --csv --print-source cuda,sass > gpurun_out/src/$b.csv 2>/dev/null
  gzip -f gpurun_out/src/$b.csv
done
rm -f gpurun_out/prof_*.ncu-rep
du -sh gpurun_out
