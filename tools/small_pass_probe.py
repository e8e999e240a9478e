"""Fixed vs size-dependent cost of one CGS block-dot pass at small n (development probe)."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2602_21958_b200 import _device, _native  # noqa: E402

lib = _native.lib()
s = _device.stream_ptr()
out = (ctypes.c_double * 32)()
for n in (64, 4096, 49600, 400000):
    V = [torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(31)]
    w = torch.randn(n, dtype=torch.float64, device="cuda")
    for k in (4, 31):
        ptrs = (ctypes.c_void_p * k)(*[v.data_ptr() for v in V[:k]])
        for _ in range(20):
            lib.rtk_block_dot(ptrs, k, _device.ptr(w), n, out, s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            lib.rtk_block_dot(ptrs, k, _device.ptr(w), n, out, s)
        el = (time.perf_counter() - t0) / 200
        print(f"n={n:7d} k={k:2d}: {el * 1e6:7.1f} us per call (incl. D2H + sync)", flush=True)
