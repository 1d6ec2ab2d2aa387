#!/bin/bash
# C2 complex128 int8 tensor-core NDFT (mode "tc") timing for library variants tools/variants/NAME.so ("base": in-tree)
cd "$(dirname "$0")/.."
for l in "$@"; do
  if [ "$l" = base ]; then L=""; else L=$PWD/tools/variants/$l.so; fi
  SA_LIB_PATH=$L timeout 200 python - <<'PY' 2>&1 | sed "s|^|$l |"
import torch, paper_1402_0532_b200 as sa
x = torch.randn(65536, 1024, dtype=torch.complex128, device="cuda"); y = torch.empty_like(x)
for _ in range(3): sa.ndft_batch(x, out=y, mode="tc")
best = 1e9
for r in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): sa.ndft_batch(x, out=y, mode="tc")
    e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 5)
print(f"C2 c128 tc {best:.3f} ms")
PY
done
