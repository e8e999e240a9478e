"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone, both at once
(the ceiling of the e2e matvec rate, which moves 524 MB each way per cfg2 matvec)."""
import time

import torch

n = 65536000
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1 = torch.cuda.Stream()
s2 = torch.cuda.Stream()
gb = 8 * n / 1e9


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t_both = timed(both)
print(f"H2D {gb / t_h2d:6.1f} GB/s   D2H {gb / t_d2h:6.1f} GB/s   both at once: {t_both * 1e3:6.2f} ms "
      f"({2 * gb / t_both:6.1f} GB/s total) -> e2e ceiling {1 / t_both:6.1f} matvec/s")
