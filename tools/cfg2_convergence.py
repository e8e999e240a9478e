"""Convergence of device GMRES on cfg2 in the moment layout (long unrestarted bases)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

p = configs.slab_problem(2, layout="moments")
b = P.build_rhs(p, device=True)
for restart, its in ((30, 3000), (None, 3000)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=its, restart=restart))
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    h = rep.residual_history
    marks = {k: h[k - 1] for k in (10, 100, 300, 1000, 2000, 3000) if k <= len(h)}
    print(f"cfg2 moments GMRES({restart}) its={rep.iterations} conv={rep.converged} time={el:.1f}s "
          f"true={rep.true_residual:.3e} {marks}", flush=True)
