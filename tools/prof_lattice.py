"""ncu driver: one lattice matvec of a config (argv[1] = 3|4|5)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200.configs import LATTICE_CONFIGS as CFGS  # noqa: E402
from paper_2602_21958_b200 import lattice as L  # noqa: E402

cfg = int(sys.argv[1])
p = L.lattice_problem(seed=21958 + cfg, **CFGS[cfg])
x = torch.randn(p.n_total, dtype=torch.float64, device="cuda")
y = P.apply_A(p, x)
torch.cuda.synchronize()
print("ok")
