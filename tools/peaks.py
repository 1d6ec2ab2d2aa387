"""Measure CUDA-core FMA peaks (FFMA, FFMA2 packed, DFMA) with sa_fma_peak."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1402_0532_b200 import _native
lib = _native.lib()
sms = torch.cuda.get_device_properties(0).multi_processor_count
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
res = {}
for name, d, iters, lanes in (("ffma", 0, 4096, 1), ("ffma2", 2, 4096, 2), ("dfma", 1, 512, 1)):
    for occ in (4, 8):
        blocks = sms * occ
        best = 0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); _native.check(lib.sa_fma_peak(d, iters, _native.ptr(sink), blocks, _native.stream_ptr())); e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e-3
            best = max(best, 2 * blocks * 256 * iters * 16 * 8 * lanes / t / 1e12)
        res[f"{name}_occ{occ}"] = round(best, 2)
print(json.dumps(res))
