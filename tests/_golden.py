"""Load the reference golden vectors (tests/golden/ref_goldens.npz) as oracle descriptions."""
import os

import numpy as np

from oracle import rt_oracle as ro

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_goldens.npz")
CASES = ("mono", "coherent", "crd", "log_legendre", "log_crd", "cfg1_legendre", "cfg1_crd")
_cache = {}


def load():
    if "z" not in _cache:
        z = np.load(GOLDEN)
        _cache["z"] = {k: z[k] for k in z.files}
    return _cache["z"]


def general_kernel(z, key):
    kind = str(z[f"{key}/kernel"])
    mu, phi, fw = z[f"{key}/mu"], z[f"{key}/phi"], z[f"{key}/freq_w"]
    if kind == "LegendreKernel":
        return ro.legendre_as_general(z[f"{key}/coefficients"], mu, phi.size)
    if kind == "CRDKernel":
        return ro.crd_as_general(phi, mu)
    if kind == "CoherentKernel":
        return ro.coherent_as_general(phi, fw, mu)
    raise KeyError(kind)


def desc(key, formal_solver="ie"):
    z = load()
    Y, c, R = general_kernel(z, key)
    return ro.SlabDesc(t_nodes=z[f"{key}/t_nodes"], mu=z[f"{key}/mu"], ang_w=z[f"{key}/ang_w"],
                       nu=z[f"{key}/nu"], freq_w=z[f"{key}/freq_w"], phi=z[f"{key}/phi"],
                       ybasis=Y, coeffs=c, R=R, gamma=z[f"{key}/gamma"], thermal=z[f"{key}/thermal"],
                       inflow=z[f"{key}/inflow"], formal_solver=formal_solver)


def gmres_cases(key):
    z = load()
    names = sorted({k.split("/")[1] for k in z if k.startswith(f"{key}/gmres_")})
    out = []
    for n in names:
        pre = f"{key}/{n}"
        tol, max_iter, restart, reorth = z[f"{pre}/cfg"]
        out.append(dict(name=n, b=z[f"{pre}/b"], solution=z[f"{pre}/solution"],
                        iterations=int(z[f"{pre}/iterations"]), history=z[f"{pre}/history"],
                        converged=bool(z[f"{pre}/converged"]), true_residual=float(z[f"{pre}/true_residual"]),
                        rel_tol=float(tol), max_iter=int(max_iter),
                        restart=None if restart < 0 else int(restart), reorthogonalize=bool(reorth)))
    return out


def gmres_band(key, name):
    """Iteration counts of the unmodified reference on 16 ulp-perturbed right-hand sides
    (tests/golden/make_gmres_bands.py) for a restarted golden case."""
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_gmres_bands.npz"))
    return z[f"{key}/{name}/iterations"]
