#!/bin/bash
# Interleaved A/B timing of the 2^16 NL-FFT across library builds, with an output
# hash per build (all builds must agree bit for bit):
#   tools/ab_nlfft_check.sh [-d "complex64:dit"] [-r ROUNDS] lib1.so lib2.so ...
cd "$(dirname "$0")/.."
cases="complex64:dit"; rounds=3
while getopts "d:r:" o; do case $o in d) cases=$OPTARG;; r) rounds=$OPTARG;; esac; done
shift $((OPTIND - 1))
for r in $(seq $rounds); do
  for l in "$@"; do
    SA_NLFFT_IMPL=cluster SA_LIB_PATH=$PWD/$l timeout 300 python - $r $cases <<'PY' 2>&1 | sed "s|^|$l |"
import sys, hashlib, torch
import paper_1402_0532_b200 as sa
rnd = int(sys.argv[1])
for c in sys.argv[2:]:
    dt, var = c.split(":")
    g = torch.Generator(device="cuda"); g.manual_seed(7)
    x = torch.randn(4096, 65536, dtype=getattr(torch, dt), device="cuda", generator=g); y = torch.empty_like(x)
    for _ in range(3): sa.nfft_batch(x, out=y, variant=var)
    torch.cuda.synchronize()
    if rnd == 1:
        h = hashlib.sha256(y.view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"{dt} {var} hash {h}")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(30): sa.nfft_batch(x, out=y, variant=var)
    e1.record(); torch.cuda.synchronize()
    print(f"{dt} {var} {e0.elapsed_time(e1) / 30:.3f} ms")
    del x, y
PY
  done
done | tee gpurun_out/ab_nlfft_raw.txt | grep -v hash | sort | awk '{k=$1" "$2" "$3; v=$4; if(!(k in m)||v<m[k])m[k]=v; a[k]=a[k]" "v} END{for(k in m)print k, "min", m[k], "all", a[k]}' | sort
grep hash gpurun_out/ab_nlfft_raw.txt
