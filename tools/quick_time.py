"""Quick cfg1/cfg2 matvec timing with per-kernel CUDA events (development tool)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import _device, _native, configs  # noqa: E402

for cfg in (1, 2):
    for fs in ("ie", "exp_linear", "exp_parabolic"):
        p = configs.slab_problem(cfg, formal_solver=fs)
        n = p.n_total
        x = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
        y = torch.empty_like(x)
        h = p.device()
        ms = (ctypes.c_float * 3)()
        lib = _native.lib()
        for _ in range(3):
            _native.check(lib.rtk_profile_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, _device.stream_ptr(), ms))
        tot = np.zeros(3)
        K = 10
        for _ in range(K):
            _native.check(lib.rtk_profile_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, _device.stream_ptr(), ms))
            tot += np.array(list(ms))
        tot /= K
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(K):
            P.apply_A(p, x)
        s1.record()
        torch.cuda.synchronize()
        full = s0.elapsed_time(s1) / K
        nf, ns, nm = p.grid.n_freq, p.grid.n_space, 2
        sweep_bytes = 16 * n + 8 * nm * nf * ns
        mom_bytes = 8 * n + 8 * nm * nf * ns
        gflop = 2 * nf * nf * nm * ns / 1e9
        print(f"cfg{cfg} {fs:14s} N={n:>10d} matvec {full*1e3:9.1f} us  moments {tot[0]*1e3:8.1f} us "
              f"({mom_bytes/tot[0]/1e6:7.0f} GB/s)  R {tot[1]*1e3:8.1f} us ({gflop/tot[1]:6.2f} TF/s)  "
              f"sweep {tot[2]*1e3:8.1f} us ({sweep_bytes/tot[2]/1e6:7.0f} GB/s)  GDOF/s {n/full/1e6:7.1f}", flush=True)
