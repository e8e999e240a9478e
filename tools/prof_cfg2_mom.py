"""ncu driver: a few cfg2 moment-layout matvecs."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

p = configs.slab_problem(2, layout="moments")
u = torch.randn(p.n_total, dtype=torch.float64, device="cuda")
for _ in range(3):
    P.apply_A(p, u)
torch.cuda.synchronize()
print("ok")
