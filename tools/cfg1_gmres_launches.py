"""A few cfg1 GMRES(30) iterations, for an ncu launch list (per-kernel GPU durations)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

p = configs.slab_problem(1)
b = P.build_rhs(p, device=True)
P.gmres(p, b, P.SolveConfig(rel_tol=1e-30, max_iter=30, restart=30))
t0 = time.perf_counter()
rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-30, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 20, restart=30))
print(f"{rep.iterations} its in {(time.perf_counter() - t0) * 1e3:.2f} ms")
