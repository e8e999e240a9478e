"""Build product-side problems from the golden (reference) setups, and the oracle
description of any product problem, so both run on identical setup arrays."""
import numpy as np

import paper_2602_21958_b200 as P
from oracle import rt_oracle as ro
from tests import _golden as G


def lorentzian(nu):
    return 1.0 / (np.pi * (np.asarray(nu, dtype=float) ** 2 + 1.0))


def gauss(nu):
    nu = np.asarray(nu, dtype=float)
    return np.exp(-nu * nu) / np.sqrt(np.pi)


PROFILES = {"mono": None, "coherent": lorentzian, "crd": lorentzian, "log_legendre": gauss, "log_crd": gauss,
            "cfg1_legendre": gauss, "cfg1_crd": gauss}


def product_from_golden(key, formal_solver="ie"):
    z = G.load()
    prof = PROFILES[key]
    grid = P.Grid(z[f"{key}/t_nodes"], z[f"{key}/mu"], z[f"{key}/ang_w"], z[f"{key}/nu"], z[f"{key}/freq_w"], prof)
    kind = str(z[f"{key}/kernel"])
    if kind == "LegendreKernel":
        kernel = P.LegendreKernel(tuple(z[f"{key}/coefficients"]))
    elif kind == "CRDKernel":
        kernel = P.CRDKernel(prof)
    else:
        kernel = P.CoherentKernel(prof)
    scat = P.ScatteringOperator(grid, kernel, z[f"{key}/gamma"])
    tr = P.build_transfer(grid, 0.0, 0.0, formal_solver=formal_solver)
    tr.inflow = np.array(z[f"{key}/inflow"])
    return P.RTProblem(grid, tr, scat, thermal=z[f"{key}/thermal"])


def oracle_desc(problem):
    """Oracle description of a product problem (same arrays, independent arithmetic)."""
    return ro.desc_from_problem(problem)


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
