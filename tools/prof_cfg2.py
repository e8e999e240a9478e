"""Small driver for ncu: a few cfg2 matvecs (formal solver from argv[1], default ie)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_21958_b200 import _device, _native, configs  # noqa: E402

fs = sys.argv[1] if len(sys.argv) > 1 else "ie"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = configs.slab_problem(2, formal_solver=fs)
n = p.n_total
x = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).cuda()
y = torch.empty_like(x)
h = p.device()
lib = _native.lib()
for _ in range(reps):
    _native.check(lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, _device.stream_ptr()))
torch.cuda.synchronize()
print("ok")
