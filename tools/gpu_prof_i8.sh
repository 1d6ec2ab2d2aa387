cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-extras --no-e2e --no-cpu"
$B > gpurun_out/plain_bench.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
bash tools/gpu_prof.sh ndft_i8_c64:k_ndft_i8:ndft_tc8:c64 i8prep_c64:k_i8_prep:ndft_tc8:c64 ndft_i8:k_ndft_i8:ndft_tc:c128 i8prep:k_i8_prep:ndft_tc:c128
python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep --out gpurun_out/round_kernels > gpurun_out/summary.log 2>&1
mkdir -p gpurun_out/src
for r in gpurun_out/prof_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page source --csv --print-source cuda,sass > gpurun_out/src/$b.csv 2>/dev/null
  gzip -f gpurun_out/src/$b.csv
done
rm -f gpurun_out/prof_*.ncu-rep
