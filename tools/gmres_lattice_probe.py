"""Convergence of device GMRES on the multi-D configs (development probe)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import lattice as L  # noqa: E402
from tools.time_lattice import CFGS  # noqa: E402

for cfg, restart, its in ((3, 30, 300), (4, 30, 300), (5, 20, 60)):
    p = L.lattice_problem(seed=21958 + cfg, **CFGS[cfg])
    b = P.build_rhs(p, device=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=its, restart=restart))
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    h = rep.residual_history
    print(f"cfg{cfg} GMRES({restart}) its={rep.iterations} conv={rep.converged} time={el:.1f}s "
          f"true_res={rep.true_residual:.3e} hist[9,29,59,-1]={[h[i] for i in (9, 29, 59) if i < len(h)] + [h[-1]]}",
          flush=True)
    del p, b, rep
    torch.cuda.empty_cache()
