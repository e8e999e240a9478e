import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_2602_21958_b200 as P
from paper_2602_21958_b200 import configs
p = configs.slab_problem(2)
x = np.random.default_rng(0).standard_normal(p.n_total)
for _ in range(2): y = P.apply_A(p, x)
t0 = time.perf_counter()
for _ in range(5): y = P.apply_A(p, x)
print("numpy apply_A per call ms", (time.perf_counter() - t0) / 5 * 1e3)
