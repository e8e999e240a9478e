"""ncu driver: a few GMRES(30) Arnoldi iterations on cfg2 (524 MB vectors), argv[1] = cgs2 | mgs,
argv[2] = iterations (default 10).  Profile the Krylov kernels with
  ncu -k regex:'cgs_pass|mgs_pass|scale_kernel|combine' ..."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

orth = sys.argv[1] if len(sys.argv) > 1 else "cgs2"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p = configs.slab_problem(2)
b = torch.randn(p.n_total, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-30, max_iter=its, restart=30, orthogonalization=orth))
torch.cuda.synchronize()
print("ok", rep.iterations, rep.matvecs)
