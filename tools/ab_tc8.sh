# C2 complex64 tc8 timing (device-resident, CUDA events) for library variants tools/variants/NAME.so
for l in "$@"; do
  SA_LIB_PATH=$PWD/tools/variants/$l.so timeout 200 python - <<'PY' 2>&1 | sed "s|^|$l |"
import torch, paper_1402_0532_b200 as sa
x = torch.randn(65536, 1024, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): sa.ndft_batch(x, out=y, mode="tc8")
best = 1e9
for r in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): sa.ndft_batch(x, out=y, mode="tc8")
    e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 10)
print(f"C2 c64 tc8 {best:.3f} ms")
PY
done
