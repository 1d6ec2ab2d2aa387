#!/bin/bash
# Interleaved A/B timing of the C4 lag stage (complex64) across library builds:
#   tools/ab_lag.sh [-r ROUNDS] lib1.so lib2.so ...
cd "$(dirname "$0")/.."
rounds=3
while getopts "r:" o; do case $o in r) rounds=$OPTARG;; esac; done
shift $((OPTIND - 1))
for r in $(seq $rounds); do
  for l in "$@"; do
    SA_LIB_PATH=$PWD/$l timeout 300 python - <<'PY' | sed "s|^|$l |"
import torch
from paper_1402_0532_b200 import _native
from paper_1402_0532_b200.workloads import c4_scene
sc = c4_scene()
s = torch.from_numpy(sc.surv).to(torch.complex64).cuda(); r = torch.from_numpy(sc.ref).to(torch.complex64).cuda()
z = torch.empty((1024, 512), dtype=torch.complex64, device="cuda")
def lag():
    _native.check(_native.lib().sa_ambiguity_integrate(_native.SA_C64, _native.ptr(s), _native.ptr(r), s.numel(),
                  r.numel(), 0, 1024, 512, 1, 0, _native.ptr(z), _native.stream_ptr()))
for _ in range(5): lag()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(50): lag()
e1.record(); torch.cuda.synchronize()
print(f"lag {e0.elapsed_time(e1) / 50:.4f} ms")
PY
  done
done | sort | awk '{k=$1" "$2; v=$3; if(!(k in m)||v<m[k])m[k]=v; a[k]=a[k]" "v} END{for(k in m)print k, "min", m[k], "all", a[k]}' | sort
