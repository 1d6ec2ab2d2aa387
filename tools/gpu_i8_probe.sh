bash tools/ab_i8_kernels.sh base noepi nomma
bash tools/gpu_prof.sh i8c64:k_ndft_i8:ndft_tc8:c64 i8prep64:k_i8_prep:ndft_tc8:c64 i8c128:k_ndft_i8:ndft_tc:c128
python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep --out gpurun_out/i8_kernels > gpurun_out/summary.log 2>&1
mkdir -p gpurun_out/src
for r in gpurun_out/prof_*.ncu-rep; do b=$(basename $r .ncu-rep); ncu -i $r --page source --csv --print-source cuda,sass > gpurun_out/src/$b.csv 2>/dev/null; gzip -f gpurun_out/src/$b.csv; ncu -i $r --page raw --csv > gpurun_out/src/$b.raw.csv 2>/dev/null; done
rm -f gpurun_out/prof_*.ncu-rep
cat gpurun_out/i8_kernels.md
