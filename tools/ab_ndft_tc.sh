#!/bin/bash
# Interleaved A/B timing of the C2 NDFT (complex64, mode tc) across library builds:
#   tools/ab_ndft_tc.sh [-r ROUNDS] lib1.so lib2.so ...
cd "$(dirname "$0")/.."
rounds=3
while getopts "r:" o; do case $o in r) rounds=$OPTARG;; esac; done
shift $((OPTIND - 1))
for r in $(seq $rounds); do
  for l in "$@"; do
    SA_LIB_PATH=$PWD/$l timeout 300 python - <<'PY' | sed "s|^|$l |"
import torch
import paper_1402_0532_b200 as sa
x = torch.randn(65536, 1024, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
for mode in ("tc",):
    for _ in range(2): sa.ndft_batch(x, out=y, mode=mode)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): sa.ndft_batch(x, out=y, mode=mode)
    e1.record(); torch.cuda.synchronize()
    print(f"{mode} {e0.elapsed_time(e1) / 5:.3f} ms")
PY
  done
done | sort | awk '{k=$1" "$2; v=$3; if(!(k in m)||v<m[k])m[k]=v; a[k]=a[k]" "v} END{for(k in m)print k, "min", m[k], "all", a[k]}' | sort
