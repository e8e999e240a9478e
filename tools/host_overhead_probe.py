"""Host-side cost of one rtk_apply_A at cfg1 size (GPU idle before each call), its device span,
and the back-to-back rate (development probe)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2602_21958_b200 import _device, _native, configs  # noqa: E402

p = configs.slab_problem(1)
n = p.n_total
lib = _native.lib()
h = p.device()
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s = _device.stream_ptr()
for _ in range(20):
    lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, s)
torch.cuda.synchronize()
host = []
for _ in range(200):
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, s)
    host.append(time.perf_counter_ns() - t0)
host.sort()
print(f"rtk_apply_A host time: median {host[100] / 1e3:.1f} us, min {host[0] / 1e3:.1f} us")
ev0 = torch.cuda.Event(enable_timing=True)
ev1 = torch.cuda.Event(enable_timing=True)
gt = []
for _ in range(50):
    torch.cuda.synchronize()
    ev0.record()
    lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, s)
    ev1.record()
    torch.cuda.synchronize()
    gt.append(ev0.elapsed_time(ev1) * 1e3)
gt.sort()
print(f"rtk_apply_A device span (single call, idle GPU): median {gt[25]:.1f} us")
t0 = time.perf_counter()
for _ in range(2000):
    lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, s)
torch.cuda.synchronize()
print(f"back-to-back: {(time.perf_counter() - t0) / 2000 * 1e6:.1f} us/matvec")
