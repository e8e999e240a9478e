"""Bandwidth of the CGS2 block-dot pass and of a GMRES(30) cycle at cfg2 size (development probe)."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import _device, _native, configs  # noqa: E402

n = 65536000
lib = _native.lib()
V = [torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(31)]
w = torch.randn(n, dtype=torch.float64, device="cuda")
out = (ctypes.c_double * 32)()
s = _device.stream_ptr()
for k in (1, 8, 16, 31):
    ptrs = (ctypes.c_void_p * k)(*[v.data_ptr() for v in V[:k]])
    lib.rtk_block_dot(ptrs, k, _device.ptr(w), n, out, s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        lib.rtk_block_dot(ptrs, k, _device.ptr(w), n, out, s)
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / 5
    print(f"block_dot k={k:2d}: {el * 1e3:7.2f} ms  {(k + 1) * 8 * n / el / 1e9:7.0f} GB/s", flush=True)
p = configs.slab_problem(2)
b = torch.randn(n, dtype=torch.float64, device="cuda")
P.gmres(p, b, P.SolveConfig(rel_tol=1e-30, max_iter=30, restart=30))   # warm the memory pool
best = 1e9
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-30, max_iter=30, restart=30))
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
el = best
orth = sum((3 * (j + 1) + 7) * 8 * n for j in range(30))
print(f"gmres30 x30: {el * 1e3:.1f} ms, {el / 30 * 1e3:.2f} ms/it, orth ~{orth / (el - 31 * 0.42e-3) / 1e9:.0f} GB/s")
