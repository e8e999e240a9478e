"""cfg2 exponential-sweep timing (per-kernel CUDA events through rtk_profile_apply_A), dev tool."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_21958_b200 import _device, _native, configs  # noqa: E402

for fs in sys.argv[1:] or ("exp_linear", "exp_parabolic"):
    p = configs.slab_problem(2, formal_solver=fs)
    n = p.n_total
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
    y = torch.empty_like(x)
    h = p.device()
    ms = (ctypes.c_float * 3)()
    lib = _native.lib()
    tot = []
    for i in range(13):
        _native.check(lib.rtk_profile_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, _device.stream_ptr(), ms))
        if i >= 3:
            tot.append(ms[2])
    t = float(np.median(tot))
    b = 16 * n + 8 * 2 * 512 * 2000
    print(f"{fs:14s} sweep {t*1e3:7.1f} us  {b/t/1e6:6.0f} GB/s  frac {b/t/1e6/6548:.3f}", flush=True)
