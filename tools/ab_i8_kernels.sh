# per-kernel times (ncu launch list) of the C2 tc paths in library variants (tools/variants/NAME.so)
for l in "$@"; do
  for cfg in "c128 tc" "c64 tc8"; do set -- $cfg
    SA_LIB_PATH=$PWD/tools/variants/$l.so SA_DT=$1 SA_MODE=$2 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/time_i8_c128_once.py 2>/dev/null | grep -E "k_i8_prep|k_ndft_i8" | awk -F'","' -v l=$l '{split($5,a,"(");print l, a[1], $NF}' | tail -2
  done
done
