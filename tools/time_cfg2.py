"""Time the cfg2 matvec and its kernels (development tool): argv = formal solver (default ie).
Environment switches of the library (RTK_SIGMA_DIRECT, RTK_SIGMA_UNFUSED, ...) apply."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_21958_b200 import _device, _native, configs  # noqa: E402

fs = sys.argv[1] if len(sys.argv) > 1 else "ie"
p = configs.slab_problem(2, formal_solver=fs)
n = p.n_total
x = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
y = torch.empty_like(x)
h = p.device()
lib = _native.lib()
sp = _device.stream_ptr()
for _ in range(5):
    _native.check(lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sp))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 30
e0.record()
for _ in range(reps):
    _native.check(lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sp))
e1.record()
torch.cuda.synchronize()
buf = (ctypes.c_float * 3)()
acc = [0.0, 0.0, 0.0]
for _ in range(10):
    _native.check(lib.rtk_profile_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sp, buf))
    for k in range(3):
        acc[k] += buf[k] / 10
print(f"{fs}: matvec {e0.elapsed_time(e1) / reps * 1e3:.1f} us; sigma {acc[0] * 1e3:.1f} us, redistribute {acc[1] * 1e3:.1f} us, "
      f"sweep {acc[2] * 1e3:.1f} us; checksum {float(y.double().sum()):.12e}")
