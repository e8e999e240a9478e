import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2602_21958_b200 import _device, _native, configs
lib = _native.lib()
for ns in (2000, 1848, 1780, 1716, 1023, 990):
    p = configs.slab_problem(2, n_space=ns)
    n = p.n_total
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    h = p.device(); sp = _device.stream_ptr()
    buf = (ctypes.c_float * 3)(); acc = [0.0]*3
    for _ in range(3): lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sp)
    for _ in range(10):
        lib.rtk_profile_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, sp, buf)
        for k in range(3): acc[k] += buf[k] / 10
    print(f"n_space {ns}: sigma {acc[0]*1e3:.1f} us  ({acc[0]*1e6/ns:.1f} ns/point), sweep {acc[2]*1e3:.1f} us")
    del p, x, y, h
    torch.cuda.empty_cache()
