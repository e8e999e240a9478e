"""Long (unrestarted / large-restart) device GMRES on cfg4 to a 1e-8 residual (probe)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import lattice as L  # noqa: E402
from paper_2602_21958_b200.configs import LATTICE_CONFIGS as CFGS  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
its = int(sys.argv[2]) if len(sys.argv) > 2 else 400
restart = int(sys.argv[3]) if len(sys.argv) > 3 else None
p = L.lattice_problem(seed=21958 + cfg, **CFGS[cfg])
b = P.build_rhs(p, device=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=its, restart=restart))
torch.cuda.synchronize()
el = time.perf_counter() - t0
h = rep.residual_history
print(f"cfg{cfg} GMRES({restart}) its={rep.iterations} conv={rep.converged} time={el:.1f}s "
      f"true_res={rep.true_residual:.3e} hist={[float('%.2e' % h[i]) for i in range(0, len(h), max(1, len(h) // 12))]}",
      flush=True)
