"""CPU oracle for the (I - Lambda Sigma) hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference package ``rtkrylov`` (the code
behind arXiv 2602.21958) for the path that the B200 build accelerates:
``apply_A`` (R/operator.py:48-53), its Lambda sweeps (R/_kernels.py:37-54,
R/transfer.py:88-147) and Sigma moment contractions (R/scattering.py:126-148),
``build_rhs`` (R/operator.py:56-64) and the GMRES driver (R/krylov.py:56-177),
plus the oracle extensions the BASELINE configs need and the reference lacks
(dipole x PRD kernel, exponential formal solvers, periodic lattice long
characteristics, moment layout).  R/ = /root/reference/pkg/src/rtkrylov/.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg / ``--impl reference`` arm may import this package, and only as the
checker or the timed CPU baseline.  The product package
``paper_2602_21958_b200`` never imports it.

Pinning: the reference-restated parts are pinned against golden vectors
produced by running the reference itself (``tests/golden/make_golden.py`` ->
``tests/golden/ref_goldens.npz``).  The extensions (PRD matrix, exp
integrators, lattice LC, moment layout) have no reference implementation;
they are pinned only through reduction identities that tie them to the
reference (R = ones -> LegendreKernel, R = phi phi' -> CRDKernel, IE lattice
on axis-aligned rays -> 0/1 selection, ...) and through analytic known
answers -- see DESIGN.md "Parity".
"""

from oracle.rt_oracle import *  # noqa: F401,F403
