"""Time sa_map_peaks (tile + select kernels) on a C5-shaped device map, 4 maps cycled
(> L2): python tools/time_detect.py [k ...]  (SA_LIB_PATH selects a library build)."""
import ctypes
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
from paper_1402_0532_b200 import _native  # noqa: E402

rows, cols = 4096, 2048
for dt, cdt in (("c64", torch.complex64), ("c128", torch.complex128)):
    g = torch.Generator(device="cuda").manual_seed(14020539)
    maps = [torch.randn(rows, cols, dtype=cdt, device="cuda", generator=g) for _ in range(4)]
    for k in [int(a) for a in sys.argv[1:]] or [8]:
        need = ctypes.c_int64()
        _native.check(_native.lib().sa_peaks_workspace_bytes(rows, cols, k, ctypes.byref(need)))
        ws = torch.empty(need.value, dtype=torch.uint8, device="cuda")
        idx = torch.empty(k, dtype=torch.int64, device="cuda")
        mag = torch.empty(k, dtype=torch.float64, device="cuda")
        cnt = torch.empty(1, dtype=torch.int32, device="cuda")
        d = _native.SA_C64 if dt == "c64" else _native.SA_C128

        def step(i):
            _native.check(_native.lib().sa_map_peaks(d, _native.ptr(maps[i % 4]), rows, cols, k, _native.ptr(idx),
                                                     _native.ptr(mag), _native.ptr(cnt), _native.ptr(ws), need.value,
                                                     _native.stream_ptr()))
        for i in range(4):
            step(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for i in range(40):
            step(i)
        e1.record()
        torch.cuda.synchronize()
        print(f"{dt} k={k} {e0.elapsed_time(e1) / 40 * 1e3:.1f} us")
