"""Where does a cfg1 GMRES iteration spend its time?  (development probe)"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import _device, _native, configs  # noqa: E402

p = configs.slab_problem(1)
n = p.n_total
lib = _native.lib()
h = p.device()
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
s = _device.stream_ptr()
for _ in range(10):
    lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(1000):
    lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, s)
torch.cuda.synchronize()
print(f"matvec loop (no sync): {(time.perf_counter() - t0) * 1e3:.3f} us/matvec")
t0 = time.perf_counter()
for _ in range(200):
    lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, s)
    torch.cuda.synchronize()
print(f"matvec + sync: {(time.perf_counter() - t0) * 1e6 / 200:.1f} us/matvec")
out = np.zeros(1)
t0 = time.perf_counter()
for _ in range(200):
    lib.rtk_dot(_device.ptr(x), _device.ptr(y), n, _device.dptr(out), s)
print(f"rtk_dot (incl. workspace init): {(time.perf_counter() - t0) * 1e6 / 200:.1f} us")
b = P.build_rhs(p, device=True)
for restart, its in ((30, 30), (30, 60), (30, 120), (None, 30), (None, 60)):
    cfg = P.SolveConfig(rel_tol=1e-30, max_iter=its, restart=restart)
    P.gmres(p, b, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = P.gmres(p, b, cfg)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    print(f"gmres restart={restart} iters={rep.iterations}: {el * 1e3:.2f} ms  = {el / rep.iterations * 1e6:.1f} us/iter")
