"""Periodic-lattice long characteristics (2D slab / 3D box) -- TEST INFRASTRUCTURE ONLY.

EXTENSION of the reference's multi-D pattern.  The reference's 2D operator
(R/multidim.py:127-360) traces parallel characteristic lines per direction,
marches the implicit-Euler recursion along them (R/_kernels.py:90-99) and
couples lines and Cartesian nodes through two interpolators (T_CR, T_RC;
P:397-421).  BASELINE configs 3-5 need 3D directions, x(/y)-periodic domains
and polychromatic dipole x PRD scattering, which the reference cannot express
(SURVEY.md section 0), so this module DEFINES the operator the B200 build
implements:

* nodes (i, j, k) with spacing dx, dy, dz; x (and y) periodic; layer k = 0 is the
  top (small depth), k = nz-1 the bottom; space index s = (k * ny + j) * nx + i;
* one line per horizontal node and direction ("lattice family"): the line that
  enters at column (lx, ly) of its entry layer (top for Omega_z < 0, bottom for
  Omega_z > 0) sits, after t layer steps, at (lx + t sx, ly + t sy) with
  sx = Omega_x dz / (|Omega_z| dx), sy = Omega_y dz / (|Omega_z| dy)  (sy = 0 in 2D);
* between two layers the line is split into n_sub = max(1, ceil(max(|sx|,|sy|)))
  equal sub-segments (each moves <= 1 cell horizontally, like the reference's
  <= 1-cell arc nodes, R/multidim.py:143-145); opacity and source are sampled at
  sub-nodes by trilinear interpolation (T_CR): bilinear in the layer, linear
  between the two layers; dt = len * (chi_a + chi_b) / 2 per sub-segment;
* the recursion per sub-segment is the reference IE (R/_kernels.py:96) or the
  exp-linear extension, on dtau = phi_f dt; exp-parabolic (Kunasz-Auer) updates the
  point P_j of a line from P_{j-1}, P_j and the downwind P_{j+1}: the next sub-node of
  the step, or for a step's last point (the crossing of the next layer) the point one
  sub-segment beyond it, P_n + s / n_sub between the next two layers; the line's last
  segment (exit layer) uses the linear weights, as in the 1D sweep;
* line values at a layer go back to the nodes of that layer by bilinear
  interpolation from the four surrounding lines (T_RC, rows sum to one).

Characteristics (TRIP chooses short or long
characteristics by ray inclination):
* "long" (default): the lattice family above;
* "short": every layer step restarts each direction's lines at the nodes: the
  characteristic through node c of layer t+1 starts at its upwind point c - (sx, sy)
  on layer t with the bilinear interpolate of layer t's node values there, and is
  integrated with the same n_sub sub-segments / T_CR sampling up to the node; no T_RC
  (the line ends on the node);
* "hybrid": short characteristics for steep directions (max(|sx|, |sy|) <= 1: the
  upwind point lies in the adjacent cell), long ones for grazing directions.
Vertical (integer-shift) directions give identical results in all three.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from oracle.rt_oracle import _linear_weights, _parabolic_weights


@dataclass
class LatticeDesc:
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    omega: np.ndarray        # (n_dirs, 3)
    dir_w: np.ndarray        # (n_dirs,)
    phi: np.ndarray          # (n_freq,)
    freq_w: np.ndarray       # (n_freq,)
    ybasis: np.ndarray       # (n_mom, n_dirs)
    coeffs: np.ndarray       # (n_mom,)
    R: np.ndarray            # (n_freq, n_freq)
    gamma: np.ndarray        # (n_space, n_freq)
    chi: np.ndarray          # (n_space,)
    inflow_top: np.ndarray   # (n_freq,)
    inflow_bottom: np.ndarray
    thermal: np.ndarray      # (n_space, n_freq) isotropic thermal source
    formal_solver: str = "ie"
    characteristics: str = "long"   # "long" | "short" | "hybrid"

    @property
    def n_space(self):
        return self.nx * self.ny * self.nz

    @property
    def n_dirs(self):
        return self.omega.shape[0]

    @property
    def n_freq(self):
        return self.phi.size

    @property
    def n_mom(self):
        return self.ybasis.shape[0]


def direction_geometry(d: LatticeDesc, a: int):
    """(down, sx, sy, n_sub, sub_len) for direction a."""
    ox, oy, oz = d.omega[a]
    down = oz < 0
    sx = ox * d.dz / (abs(oz) * d.dx)
    sy = (oy * d.dz / (abs(oz) * d.dy)) if d.ny > 1 else 0.0
    n_sub = max(1, int(math.ceil(max(abs(sx), abs(sy)) - 1e-12)))
    length = d.dz / abs(oz)          # 3D path length per layer (the slab is y-invariant, not 2D-transport)
    return down, sx, sy, n_sub, length / n_sub


def uses_short_characteristics(d: LatticeDesc, a: int) -> bool:
    """Short characteristics for direction a under d.characteristics."""
    if d.characteristics == "short":
        return True
    if d.characteristics == "hybrid":
        return direction_geometry(d, a)[3] == 1
    if d.characteristics != "long":
        raise ValueError(f"characteristics must be 'long', 'short' or 'hybrid', not {d.characteristics!r}")
    return False


def _bilinear_sample(field_layer, X, Y):
    """field_layer (ny, nx, ...) periodic; X, Y arrays of positions (cell units)."""
    ny, nx = field_layer.shape[:2]
    fx0 = np.floor(X)
    fy0 = np.floor(Y)
    ax = X - fx0
    ay = Y - fy0
    i0 = fx0.astype(np.int64) % nx
    j0 = fy0.astype(np.int64) % ny
    i1 = (i0 + 1) % nx
    j1 = (j0 + 1) % ny
    ex = (slice(None),) + (None,) * (field_layer.ndim - 2)
    ax = ax[ex]
    ay = ay[ex]
    return ((1 - ax) * (1 - ay) * field_layer[j0, i0] + ax * (1 - ay) * field_layer[j0, i1]
            + (1 - ax) * ay * field_layer[j1, i0] + ax * ay * field_layer[j1, i1])


def lattice_transfer(d: LatticeDesc, S: np.ndarray, with_boundary: bool = False, solver: str = None) -> np.ndarray:
    """Lambda on a source S[s, a, f] -> I[s, a, f] (homogeneous unless with_boundary)."""
    solver = solver or d.formal_solver
    nx, ny, nz, na, nf = d.nx, d.ny, d.nz, d.n_dirs, d.n_freq
    S4 = S.reshape(nz, ny, nx, na, nf)
    chi3 = d.chi.reshape(nz, ny, nx)
    out = np.empty((nz, ny, nx, na, nf))
    ly, lx = np.meshgrid(np.arange(ny, dtype=float), np.arange(nx, dtype=float), indexing="ij")
    lx = lx.ravel()
    ly = ly.ravel()
    gi, gj = lx.copy(), ly.copy()           # grid columns, same enumeration as lines
    for a in range(na):
        down, sx, sy, n_sub, sub_len = direction_geometry(d, a)
        short = uses_short_characteristics(d, a)
        if with_boundary:
            inflow = d.inflow_top if down else d.inflow_bottom
            state = np.tile(np.asarray(inflow, dtype=float), (nx * ny, 1))
        else:
            state = np.zeros((nx * ny, nf))
        for t in range(nz):
            k = t if down else nz - 1 - t
            if short:
                # lines end on the nodes: node values are the line values
                grid_vals = state
            else:
                # T_RC: node (i, j) from the four lines around it at this layer
                u = gi - t * sx
                v = gj - t * sy
                grid_vals = _bilinear_sample(state.reshape(ny, nx, nf), u, v)
            out[k].reshape(ny * nx, na, nf)[:, a, :] = grid_vals
            if t == nz - 1:
                break
            k2 = k + 1 if down else k - 1
            Sa = S4[k, :, :, a, :]
            Sb = S4[k2, :, :, a, :]
            if short:
                # restart at the upwind point of each node of layer k2, from layer k's nodes
                state = _bilinear_sample(state.reshape(ny, nx, nf), gi - sx, gj - sy)
            # sample points of the step: m = 0 .. n_sub (+ the downwind point beyond the step for
            # exp-parabolic, when a further layer step exists)
            pts = []
            for m in range(n_sub + 1):
                if short:
                    X = gi + (m / n_sub - 1.0) * sx
                    Y = gj + (m / n_sub - 1.0) * sy
                else:
                    tt = t + m / n_sub
                    X = lx + tt * sx
                    Y = ly + tt * sy
                wz = m / n_sub
                s_m = (1 - wz) * _bilinear_sample(Sa, X, Y) + wz * _bilinear_sample(Sb, X, Y)
                c_m = (1 - wz) * _bilinear_sample(chi3[k], X, Y) + wz * _bilinear_sample(chi3[k2], X, Y)
                pts.append((s_m, c_m, X, Y))
            down_pt = None
            if solver == "exp_parabolic" and t < nz - 2:
                k3 = k2 + 1 if down else k2 - 1
                X = pts[-1][2] + sx / n_sub
                Y = pts[-1][3] + sy / n_sub
                wz = 1.0 / n_sub
                s_x = (1 - wz) * _bilinear_sample(S4[k2, :, :, a, :], X, Y) + wz * _bilinear_sample(
                    S4[k3, :, :, a, :], X, Y)
                c_x = (1 - wz) * _bilinear_sample(chi3[k2], X, Y) + wz * _bilinear_sample(chi3[k3], X, Y)
                down_pt = (s_x, c_x)
            for m in range(1, n_sub + 1):
                (prev_S, prev_chi), (s_m, c_m) = pts[m - 1][:2], pts[m][:2]
                dtau = d.phi[None, :] * (sub_len * (prev_chi + c_m) * 0.5)[:, None]
                nxt = pts[m + 1][:2] if m < n_sub else down_pt
                if solver == "ie":
                    state = (state + dtau * s_m) / (1.0 + dtau)
                elif solver == "exp_parabolic" and nxt is not None:
                    s_d, c_d = nxt
                    dd = d.phi[None, :] * (sub_len * (c_m + c_d) * 0.5)[:, None]
                    att, wu, wc, wd = _parabolic_weights(dtau, dd)
                    state = att * state + wu * prev_S + wc * s_m + wd * s_d
                elif solver in ("exp_linear", "exp_parabolic"):
                    att, wu, wc = _linear_weights(dtau)
                    state = att * state + wu * prev_S + wc * s_m
                else:
                    raise ValueError(f"unknown formal solver {solver!r}")
    return out.reshape(d.n_space, na, nf)


def source_from_moments(d: LatticeDesc, u: np.ndarray) -> np.ndarray:
    """S[s,a,f] = gamma[s,f] sum_k c_k Y_k(a) u[s,k,f]  (u: redistributed moments)."""
    u = u.reshape(d.n_space, d.n_mom, d.n_freq)
    cy = d.coeffs[:, None] * d.ybasis                      # (n_mom, n_dirs)
    return d.gamma[:, None, :] * np.einsum("ka,skf->saf", cy, u)


def moments_of(d: LatticeDesc, I: np.ndarray) -> np.ndarray:
    """m[s,k,f] = sum_a w_a Y_k(a) I[s,a,f]."""
    return np.einsum("ka,saf->skf", d.ybasis * d.dir_w[None, :], I.reshape(d.n_space, d.n_dirs, d.n_freq))


def redistribute(d: LatticeDesc, m: np.ndarray) -> np.ndarray:
    """u[s,k,f] = sum_g R[f,g] w_g m[s,k,g]."""
    return np.einsum("fg,skg->skf", d.R * d.freq_w[None, :], m)


def apply_sigma(d: LatticeDesc, I: np.ndarray) -> np.ndarray:
    return source_from_moments(d, redistribute(d, moments_of(d, I))).reshape(-1)


def apply_A_intensity(d: LatticeDesc, x: np.ndarray) -> np.ndarray:
    """Intensity layout: y = x - Lambda Sigma x, x[s, a, f]."""
    S = apply_sigma(d, x).reshape(d.n_space, d.n_dirs, d.n_freq)
    return x - lattice_transfer(d, S).reshape(-1)


def apply_A_moments(d: LatticeDesc, u: np.ndarray) -> np.ndarray:
    """Moment layout: y = u - R_w M Lambda S(u), u[s, k, f]."""
    S = source_from_moments(d, u)
    I = lattice_transfer(d, S)
    return u - redistribute(d, moments_of(d, I)).reshape(-1)


def thermal_source(d: LatticeDesc) -> np.ndarray:
    return np.broadcast_to(d.thermal[:, None, :], (d.n_space, d.n_dirs, d.n_freq)).copy()


def build_rhs_intensity(d: LatticeDesc) -> np.ndarray:
    return lattice_transfer(d, thermal_source(d), with_boundary=True).reshape(-1)


def build_rhs_moments(d: LatticeDesc) -> np.ndarray:
    I = lattice_transfer(d, thermal_source(d), with_boundary=True)
    return redistribute(d, moments_of(d, I)).reshape(-1)


def desc_from_lattice_problem(p) -> LatticeDesc:
    """Oracle description of a product-side LatticeProblem (same setup arrays, duck-typed)."""
    return LatticeDesc(nx=p.nx, ny=p.ny, nz=p.nz, dx=p.dx, dy=p.dy, dz=p.dz, omega=np.asarray(p.omega),
                       dir_w=np.asarray(p.dir_w), phi=np.asarray(p.phi), freq_w=np.asarray(p.freq_w),
                       ybasis=np.asarray(p.ybasis), coeffs=np.asarray(p.coeffs), R=np.asarray(p.R),
                       gamma=np.asarray(p.gamma), chi=np.asarray(p.chi), inflow_top=np.asarray(p.inflow_top),
                       inflow_bottom=np.asarray(p.inflow_bottom), thermal=np.asarray(p.thermal),
                       formal_solver=p.formal_solver,
                       characteristics=getattr(p, "characteristics", "long"))


def apply_A(d: LatticeDesc, layout: str, x):
    return apply_A_moments(d, x) if layout == "moments" else apply_A_intensity(d, x)


def build_rhs(d: LatticeDesc, layout: str):
    return build_rhs_moments(d) if layout == "moments" else build_rhs_intensity(d)


def real_dipole_harmonics(omega):
    """Oracle restatement of the real l = 0, 2 harmonics with p = 1 + P2(W.W')/2 = sum_k c_k Y_k Y_k'."""
    ox, oy, mu = omega[:, 0], omega[:, 1], omega[:, 2]
    Y = np.stack([np.ones_like(mu), 1.5 * mu * mu - 0.5, mu * ox, mu * oy, ox * ox - oy * oy, 2 * ox * oy])
    return Y, np.array([1.0, 0.5, 1.5, 1.5, 0.375, 0.375])
