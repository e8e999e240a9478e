"""Time the lattice matvec at the BASELINE config sizes (development tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import lattice as L  # noqa: E402

from paper_2602_21958_b200.configs import LATTICE_CONFIGS as CFGS  # noqa: E402


def main():
  which = [int(a) for a in sys.argv[1:]] or [3, 4, 5]
  for cfg in which:
    kw = dict(CFGS[cfg])
    import os
    if os.environ.get("FS"):
        kw["formal_solver"] = os.environ["FS"]
    if os.environ.get("LAYOUT"):
        kw["layout"] = os.environ["LAYOUT"]
    if os.environ.get("CHARS"):
        kw["characteristics"] = os.environ["CHARS"]
    t0 = time.time()
    p = L.lattice_problem(seed=21958 + cfg, **kw)
    p.device()
    setup = time.time() - t0
    x = torch.randn(p.n_total, dtype=torch.float64, device="cuda")
    y = P.apply_A(p, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3 if cfg == 5 else 5
    e0.record()
    for _ in range(reps):
        y = P.apply_A(p, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    dof = p.n_space * p.n_dirs * p.n_freq
    print(f"cfg{cfg} {kw['layout']:9s} unknowns={p.n_total:>11d} DOF={dof:>11d} setup {setup:6.1f}s  matvec {ms:9.2f} ms"
          f"  {dof / ms / 1e6:8.2f} GDOF/s", flush=True)
    del p, x, y
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
