"""Unrestarted GMRES on cfg2 (moment layout, n = 2.05 M): time for growing iteration counts and the
implied CGS2 bandwidth of the late iterations (development probe)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

p = configs.slab_problem(2, layout="moments")
n = p.n_total
b = P.build_rhs(p, device=True)
P.gmres(p, b, P.SolveConfig(rel_tol=1e-30, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 20, restart=None))
prev = None
for its in (100, 200, 400, 800):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.gmres(p, b, P.SolveConfig(rel_tol=1e-30, max_iter=its, restart=None))
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    line = f"its={its:4d} {el:7.3f} s"
    if prev:
        j0, t_prev = prev
        dt = el - t_prev
        # passes over the basis per iteration j: 4 (j+1) vector reads (+ w traffic); count 4 passes
        byts = sum(4 * (j + 1) * 8 * n for j in range(j0, its))
        line += f"  increment {dt:6.3f} s  ~{byts / dt / 1e9:6.0f} GB/s over 4 passes"
    print(line, flush=True)
    prev = (its, el)
