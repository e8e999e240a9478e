"""Multi-D (2D slab / 3D box) problems on a periodic lattice, applied on the B200.

BASELINE configs 3-5 need 3D directions, x(/y)-periodic domains and
polychromatic dipole x PRD scattering, which the reference's 2D code cannot
express (R/multidim.py: in-plane azimuths only, monochromatic, non-periodic).
This module keeps the reference's multi-D pattern -- parallel characteristic
lines per direction, line-node recursion, Cartesian <-> line interpolators
(R/multidim.py:127-360) -- on a periodic lattice family; the
operator is defined in oracle/lattice.py and DESIGN.md section 11.

Unknown layouts: 'intensity' (I[s][a][f], the reference's layout) or
'moments' (u[s][l][f], redistributed dipole moments; mandatory at configs
4-5 where an intensity vector is 8-66 GB).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from paper_2602_21958_b200 import _device, _native
from paper_2602_21958_b200.quadrature import gauss_legendre, legendre_basis, trapezoid
from paper_2602_21958_b200.redistribution import gaussian_profile, prd_matrix

LAYOUTS = {"intensity": 0, "moments": 1}
# real dipole harmonics: p(W, W') = 1 + P2(W.W')/2 = sum_k C_k Y_k(W) Y_k(W')
DIPOLE_3D_COEFFS = (1.0, 0.5, 1.5, 1.5, 0.375, 0.375)


class LatticeDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("n_dirs", ctypes.c_int32), ("n_freq", ctypes.c_int32), ("n_moments", ctypes.c_int32),
                ("formal_solver", ctypes.c_int32), ("layout", ctypes.c_int32),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double)] + \
               [(n, _native.c_double_p) for n in ("omega", "dir_w", "phi", "freq_w", "ybasis", "coeffs",
                                                   "redistribution", "gamma", "chi", "inflow_top",
                                                   "inflow_bottom")] + \
               [("characteristics", ctypes.c_int32)]

CHARACTERISTICS = {"long": 0, "short": 1, "hybrid": 2}


def product_quadrature(n_polar: int, n_azimuth: int):
    """Half-interval Gauss-Legendre polar cosines (as R/grid.py:137-140) x equidistant
    azimuths (j + 1/2) 2 pi / n_az (the reference's offset, R/multidim.py:57).
    Returns omega (n_dirs, 3) polar-major, weights summing to 4 pi."""
    dn = gauss_legendre(n_polar // 2, -1.0, 0.0)
    up = gauss_legendre(n_polar // 2, 0.0, 1.0)
    mu = np.concatenate([dn.nodes, up.nodes])
    wmu = np.concatenate([dn.weights, up.weights])
    phi = 2.0 * math.pi * (np.arange(n_azimuth) + 0.5) / n_azimuth
    mm, pp = np.meshgrid(mu, phi, indexing="ij")
    s = np.sqrt(1.0 - mm * mm)
    omega = np.stack([s * np.cos(pp), s * np.sin(pp), mm], axis=-1).reshape(-1, 3)
    w = (wmu[:, None] * np.full(n_azimuth, 2.0 * math.pi / n_azimuth)[None, :]).reshape(-1)
    return omega, w


def dipole_harmonics(omega: np.ndarray) -> np.ndarray:
    """Y (6, n_dirs): 1, P2(mu), mu s cos phi, mu s sin phi, s^2 cos 2phi, s^2 sin 2phi."""
    ox, oy, mu = omega[:, 0], omega[:, 1], omega[:, 2]
    return np.stack([np.ones_like(mu), 0.5 * (3 * mu * mu - 1), mu * ox, mu * oy, ox * ox - oy * oy,
                     2 * ox * oy])


def lognormal_field(shape, sigma: float, corr_len: float, seed: int) -> np.ndarray:
    """exp(sigma g - sigma^2/2), g a unit-variance Gaussian random field: white noise
    FFT-filtered with a Gaussian of the given correlation length (cells), periodic."""
    rng = np.random.default_rng(seed)
    white = rng.standard_normal(shape)
    k = np.meshgrid(*[np.fft.fftfreq(n) for n in shape], indexing="ij")
    k2 = sum(kk * kk for kk in k)
    filt = np.exp(-0.5 * (2 * math.pi) ** 2 * k2 * corr_len ** 2)
    g = np.real(np.fft.ifftn(np.fft.fftn(white) * filt))
    g = (g - g.mean()) / g.std()
    return np.exp(sigma * g - 0.5 * sigma * sigma)


def stratified_opacity(nz: int, dz: float = 1.0, t_top: float = 1e-4, t_bottom: float = 1e4) -> np.ndarray:
    """Exponential vertical stratification: kappa0(z_k) = c t_k with t_k log-spaced
    t_top..t_bottom (k = 0 top), so the vertical optical depth spans t_top..t_bottom."""
    c = math.log(t_bottom / t_top) / ((nz - 1) * dz)
    t = t_top * np.exp(c * dz * np.arange(nz))
    return c * t


@dataclass
class LatticeProblem:
    nx: int
    ny: int
    nz: int
    omega: np.ndarray
    dir_w: np.ndarray
    nu: np.ndarray
    freq_w: np.ndarray
    phi: np.ndarray
    ybasis: np.ndarray
    coeffs: np.ndarray
    R: np.ndarray
    gamma: np.ndarray           # (n_space, n_freq)
    chi: np.ndarray             # (n_space,)
    thermal: np.ndarray         # (n_space, n_freq)
    inflow_top: np.ndarray
    inflow_bottom: np.ndarray
    layout: str = "intensity"
    formal_solver: str = "ie"
    characteristics: str = "long"   # "long" | "short" | "hybrid" (short for steep, long for grazing directions)
    dx: float = 1.0
    dy: float = 1.0
    dz: float = 1.0
    descriptor: dict = field(default_factory=dict)
    _handle: object = field(default=None, repr=False, compare=False)

    @property
    def n_space(self):
        return self.nx * self.ny * self.nz

    @property
    def n_dirs(self):
        return self.omega.shape[0]

    @property
    def n_freq(self):
        return self.nu.size

    @property
    def n_mom(self):
        return self.ybasis.shape[0]

    @property
    def n_total(self):
        per = self.n_mom if self.layout == "moments" else self.n_dirs
        return self.n_space * per * self.n_freq

    def device(self):
        if self._handle is None:
            self._handle = _LatticeHandle(self)
        return self._handle


class _LatticeHandle:
    def __init__(self, p: LatticeProblem):
        _device.require_cuda()
        lib = _native.lib()
        self._keep = {n: np.ascontiguousarray(getattr(p, n), dtype=float) for n in
                      ("omega", "dir_w", "phi", "freq_w", "ybasis", "coeffs", "R", "gamma", "chi", "inflow_top",
                       "inflow_bottom")}
        d = LatticeDesc()
        d.nx, d.ny, d.nz = p.nx, p.ny, p.nz
        d.n_dirs, d.n_freq, d.n_moments = p.n_dirs, p.n_freq, p.n_mom
        if p.formal_solver not in ("ie", "exp_linear", "exp_parabolic"):
            raise ValueError("formal_solver must be 'ie', 'exp_linear' or 'exp_parabolic'")
        d.formal_solver = _native.FS_CODES[p.formal_solver]
        d.layout = LAYOUTS[p.layout]
        if p.characteristics not in CHARACTERISTICS:
            raise ValueError(f"characteristics must be one of {sorted(CHARACTERISTICS)}, not {p.characteristics!r}")
        d.characteristics = CHARACTERISTICS[p.characteristics]
        d.dx, d.dy, d.dz = p.dx, p.dy, p.dz
        for name, key in (("omega", "omega"), ("dir_w", "dir_w"), ("phi", "phi"), ("freq_w", "freq_w"),
                          ("ybasis", "ybasis"), ("coeffs", "coeffs"), ("redistribution", "R"), ("gamma", "gamma"),
                          ("chi", "chi"), ("inflow_top", "inflow_top"), ("inflow_bottom", "inflow_bottom")):
            setattr(d, name, _device.dptr(self._keep[key]))
        h = ctypes.c_void_p()
        _native.check(lib.rtk_problem_create_lattice(ctypes.byref(d), ctypes.byref(h)))
        self.h = h
        self.n_total = int(lib.rtk_problem_n_total(h))
        self._lib = lib

    def set_inflow(self, inflow):  # pragma: no cover - lattice inflow is fixed at creation
        raise ValueError("lattice inflow is fixed at creation")

    def set_tuning(self, key: str, value: int):
        """Select a kernel variant of this handle (rtk_problem_set_tuning)."""
        _native.check(self._lib.rtk_problem_set_tuning(self.h, key.encode(), int(value)))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self._lib.rtk_problem_destroy(h)
            except Exception:  # pragma: no cover
                pass
            self.h = None


def lattice_problem(nx: int, ny: int, nz: int, n_polar: int, n_azimuth: int, n_freq: int, x_max: float = 5.0,
                    eps: float = 1e-4, sigma: float = 0.5, corr_len: float = 8.0, seed: int = 0,
                    layout: str = "intensity", formal_solver: str = "ie", coherence: float = 0.5,
                    bottom_inflow: float = 1.0, t_range=(1e-4, 1e4),
                    characteristics: str = "long") -> LatticeProblem:
    """Seeded lattice problem: log-normal opacity on an exponential stratification, dipole x PRD
    scattering with gamma = (1 - eps) / (4 pi phi), thermal eps B (B = 1), zero incident
    intensity at the top and B at the bottom."""
    omega, w = product_quadrature(n_polar, n_azimuth)
    fr = trapezoid(n_freq, -x_max, x_max)
    nu, fw = fr.nodes, fr.weights
    phi = gaussian_profile(nu)
    R = prd_matrix(nu, fw, phi, coherence)
    Y = dipole_harmonics(omega)
    c = np.array(DIPOLE_3D_COEFFS)
    kappa0 = stratified_opacity(nz, 1.0, *t_range)
    rho = lognormal_field((nz, ny, nx), sigma, corr_len, seed)
    chi = (kappa0[:, None, None] * rho).reshape(-1)
    n_space = nx * ny * nz
    gamma = np.broadcast_to((1.0 - eps) / (4.0 * math.pi * phi)[None, :], (n_space, n_freq)).copy()
    thermal = np.full((n_space, n_freq), eps)
    return LatticeProblem(nx=nx, ny=ny, nz=nz, omega=omega, dir_w=w, nu=nu, freq_w=fw, phi=phi, ybasis=Y,
                          coeffs=c, R=R, gamma=gamma, chi=chi, thermal=thermal, inflow_top=np.zeros(n_freq),
                          inflow_bottom=np.full(n_freq, bottom_inflow), layout=layout, formal_solver=formal_solver,
                          characteristics=characteristics, descriptor=dict(eps=eps, sigma=sigma, corr_len=corr_len, seed=seed, coherence=coherence))


def lattice_apply_A(problem: LatticeProblem, v):
    """y = v - Lambda Sigma v (intensity layout) or u - R_w M Lambda S(u) (moment layout)."""
    n = problem.n_total
    h = problem.device()
    if not _device.is_tensor(v):
        # host arrays go through the library's staged host path (pinned chunks, overlapped copies)
        arr = np.ascontiguousarray(np.asarray(v, dtype=float).reshape(-1))
        if arr.size != n:
            raise ValueError(f"expected length {n}, got {arr.size}")
        out = np.empty(n)
        _native.check(_native.lib().rtk_apply_A_host(h.h, _device.dptr(arr), _device.dptr(out), n,
                                                     _device.stream_ptr()))
        return out
    x, kind = _device.to_device(v, n)
    y = _device.empty(n)
    _native.check(_native.lib().rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, _device.stream_ptr()))
    return _device.from_device(y, kind)


def lattice_build_rhs(problem: LatticeProblem, device: bool = False):
    """b = Lambda thermal + inflow term (intensity layout) or its redistributed moments."""
    n = problem.n_total
    h = problem.device()
    th, _ = _device.to_device(problem.thermal.reshape(-1), problem.n_space * problem.n_freq)
    b = _device.empty(n)
    _native.check(_native.lib().rtk_build_rhs(h.h, _device.ptr(th), _device.ptr(b), n, 0, _device.stream_ptr()))
    return b if device else b.cpu().numpy()
