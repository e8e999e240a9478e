"""cfg2 matvec timing through apply_A (CUDA events over 50 back-to-back matvecs), dev tool."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

p = configs.slab_problem(2)
x = torch.from_numpy(np.random.default_rng(0).standard_normal(p.n_total)).cuda()
for _ in range(5):
    P.apply_A(p, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    P.apply_A(p, x)
e1.record()
torch.cuda.synchronize()
print(f"matvec {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
