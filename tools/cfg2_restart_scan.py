"""cfg2 moment layout: time-to-1e-8 for several GMRES restart lengths (development probe)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

p = configs.slab_problem(2, layout="moments")
b = P.build_rhs(p, device=True)
P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=400, restart=400))   # warm the pool
for restart in [int(a) for a in sys.argv[1:]] or [100, 200, 400, 800]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=8000, restart=restart))
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    print(f"GMRES({restart}) its={rep.iterations} conv={rep.converged} time={el:.2f}s true={rep.true_residual:.2e}",
          flush=True)
