#!/bin/bash
# ncu --set full of the lag-stage kernels (C4, C5 maps) + source-level CSVs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/src
bash tools/gpu_prof.sh ${SPECS:-lagi8:k_lag_i8:map:c64 lagi8_5:k_lag_i8:map5:c64}
python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep --out gpurun_out/lag_kernels > gpurun_out/summary.log 2>&1
for r in gpurun_out/prof_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page source --csv --print-source cuda,sass > gpurun_out/src/$b.csv 2>/dev/null
  ncu -i $r --page raw --csv > gpurun_out/src/$b.raw.csv 2>/dev/null
  gzip -f gpurun_out/src/$b.csv gpurun_out/src/$b.raw.csv
done
rm -f gpurun_out/prof_*.ncu-rep
