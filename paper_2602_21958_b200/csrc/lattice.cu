// Periodic-lattice long-characteristics transfer for the 2D slab / 3D box
// configurations (BASELINE configs 3-5).  The operator is defined in
// oracle/lattice.py; it generalises the reference's
// 2D long characteristics (R/multidim.py:127-360): one line per
// horizontal node and direction, <= 1-cell sub-steps with trilinear T_CR
// sampling of opacity and source, the IE / exp-linear recursion
// (R/_kernels.py:90-99), and bilinear T_RC back to the nodes of each layer.
//
// Kernels:
//  * lattice_int_smem_kernel (intensity layout, cfg3): one CTA per (direction, sector-aligned
//    4-frequency chunk) marches ALL lines of that direction through ALL layers in one launch;
//    source / x planes staged by cp.async rings, line values double-buffered in shared memory
//    for the T_RC gather (one barrier per layer step).  Output y = x - I (or I).
//    lattice_int_kernel is its fallback for layers too large for shared memory.
//  * lattice_mom_tile_kernel (moment layout, cfg4/5; IE, exp-linear, exp-parabolic LC):
//    layer-synchronous, one launch per layer step; a CTA owns a tile of lines and a frequency
//    pair and loops over the directions, sampling the source from shared-memory windows of the
//    pair-major planes written by lattice_splane_pm_kernel; angular moments accumulate in
//    registers in a fixed order (no atomics); line states live in a double-buffered
//    [dir][pair][line] array.  The source is rebuilt from the moment unknown u per layer.
//  * lattice_mom_group_kernel (+ lattice_splane_kernel): the per-item moment kernel, one thread
//    per (line, frequency pair[, direction group]) reading through L1/L2 -- exp-parabolic with
//    short characteristics, odd padded N_nu, oversized windows, and the parity-test variants.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "formal.cuh"
#include "rtk_internal.cuh"

namespace rtk {
namespace {

constexpr int kFC = 4;            // frequencies per CTA in the intensity kernel
constexpr int kIntThreads = 256;
#ifndef RTK_INT_MINB
#define RTK_INT_MINB 2   // CTAs per SM the shared-memory intensity kernel is compiled for
#endif

__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// bilinear stencil of a horizontal position (periodic): 4 node indices + weights
struct Stencil {
    int c00, c10, c01, c11;
    double w00, w10, w01, w11;
};

// Lattice regularity: every line of a direction has the same fractional offset at a
// given (layer step, sub-node), so the interpolation weights and the integer shift
// are warp-uniform; only the line's own column enters per lane.
struct Shift {
    int bx, by;       // floor(offset) mod n
    double ax, ay;    // fractional part
};

__host__ __device__ __forceinline__ Shift shift_of(double offx, double offy, int nx, int ny) {
    Shift s;
    const double fx = floor(offx), fy = floor(offy);
    s.ax = offx - fx;
    s.ay = offy - fy;
    s.bx = static_cast<int>(fx - nx * floor(fx / nx));
    s.by = static_cast<int>(fy - ny * floor(fy / ny));
    if (s.bx >= nx) s.bx -= nx;   // guard the rounding edge of floor(fx / nx)
    if (s.by >= ny) s.by -= ny;
    if (s.bx < 0) s.bx += nx;
    if (s.by < 0) s.by += ny;
    return s;
}

__device__ __forceinline__ Stencil stencil_at(int lx, int ly, const Shift& sh, int nx, int ny) {
    int i0 = lx + sh.bx;
    if (i0 >= nx) i0 -= nx;
    int j0 = ly + sh.by;
    if (j0 >= ny) j0 -= ny;
    const int i1 = (i0 + 1 == nx) ? 0 : i0 + 1, j1 = (j0 + 1 == ny) ? 0 : j0 + 1;
    Stencil s;
    s.c00 = j0 * nx + i0;
    s.c10 = j0 * nx + i1;
    s.c01 = j1 * nx + i0;
    s.c11 = j1 * nx + i1;
    s.w00 = (1 - sh.ax) * (1 - sh.ay);
    s.w10 = sh.ax * (1 - sh.ay);
    s.w01 = (1 - sh.ax) * sh.ay;
    s.w11 = sh.ax * sh.ay;
    return s;
}

// SC restart: value at the upwind point c - s of node c, bilinear from a [nxy][stride] plane
__device__ __forceinline__ Shift restart_shift(const LatDir& D) {
    Shift sh;
    sh.bx = D.rbx;
    sh.by = D.rby;
    sh.ax = D.rax;
    sh.ay = D.ray;
    return sh;
}

struct LatArgs {
    const LatDir* dirs;
    const Shift* sub_shift;   // [dir: shift_off + t * (n_sub + 1) + m] sub-node shifts
    const Shift* gat_shift;   // [dir * nz + t] T_RC gather shifts
    const Shift* down_shift;  // [dir * nz + t] exp-parabolic downwind point of step t's last sub-node
    const double* dtab;       // sub-segment optical paths (moment layout), see lattice_dtab_kernel
    const double* chi;      // [n_space]
    const double* phi;      // [n_freq]
    const double* src;      // SRC_VEC: S[s][a][f]; SRC_ISO: thermal[s][f]; SRC_U: u[s][l][f]
    const double* gamma;    // [s][f] (SRC_U)
    const double* x;        // OUT_X_MINUS
    double* y;
    const double* inflow_top;     // [n_freq] or null
    const double* inflow_bottom;
    int nx, ny, nz, n_dirs, n_freq, n_mom;
    int a0, a1;               // direction range of this call (sharded operator); default all
    int64_t nxy;
    int total_sub;            // sum over directions of (n_sub + 1): one step's sub-node shifts
};

enum LatSrc { LSRC_VEC = 0, LSRC_ISO = 1, LSRC_U = 2 };

// One formal-solver pass of a line between two layers.  The line sits at horizontal
// position (lx + t sx, ly + t sy) on the start layer; chi_a/chi_b are the opacity
// planes and Sa/Sb the source planes (node c at Sa[c * ss]) of the start and end layers.
template <int FS>
__device__ __forceinline__ double advance_line(const LatDir& D, const Shift* __restrict__ sub, double acc, int lx,
                                               int ly, int t, int nx, int ny, const double* __restrict__ chi_a,
                                               const double* __restrict__ chi_b, const double* __restrict__ Sa,
                                               const double* __restrict__ Sb, int64_t ss, double phi_f) {
    double prev_s = 0.0, prev_c = 0.0;
    for (int m = 0; m <= D.n_sub; ++m) {
        const double wz = static_cast<double>(m) / D.n_sub;
        const Shift sh = sub[m];   // warp-uniform, precomputed at setup (same arithmetic as shift_of)
        const Stencil st = stencil_at(lx, ly, sh, nx, ny);
        const double ca = st.w00 * __ldg(chi_a + st.c00) + st.w10 * __ldg(chi_a + st.c10) +
                          st.w01 * __ldg(chi_a + st.c01) + st.w11 * __ldg(chi_a + st.c11);
        const double cb = st.w00 * __ldg(chi_b + st.c00) + st.w10 * __ldg(chi_b + st.c10) +
                          st.w01 * __ldg(chi_b + st.c01) + st.w11 * __ldg(chi_b + st.c11);
        const double sa = st.w00 * __ldg(Sa + st.c00 * ss) + st.w10 * __ldg(Sa + st.c10 * ss) +
                          st.w01 * __ldg(Sa + st.c01 * ss) + st.w11 * __ldg(Sa + st.c11 * ss);
        const double sb = st.w00 * __ldg(Sb + st.c00 * ss) + st.w10 * __ldg(Sb + st.c10 * ss) +
                          st.w01 * __ldg(Sb + st.c01 * ss) + st.w11 * __ldg(Sb + st.c11 * ss);
        const double c_m = (1 - wz) * ca + wz * cb;
        const double s_m = (1 - wz) * sa + wz * sb;
        if (m > 0) {
            const double dtau = phi_f * (D.sub_len * (prev_c + c_m) * 0.5);
            if (FS == RTK_FS_IE) {
                const double r = rcp_nr(1.0 + dtau);
                acc = fma(acc, r, (dtau * s_m) * r);
            } else {
                const ExpLin w = exp_linear_weights(dtau);
                acc = fma(acc, w.att, w.wu * prev_s + w.wc * s_m);
            }
        }
        prev_s = s_m;
        prev_c = c_m;
    }
    return acc;
}

// Shared-memory planes of the intensity kernel are pair-major: frequency q of node c sits at
// pidx(c, q) = [q / 2][c][q % 2], so a warp's double2 loads of consecutive nodes are
// contiguous (bank-conflict-free LDS.128; node-major [c][kFC] put lanes 32 B apart).
__device__ __forceinline__ int pidx(int c, int q, int nxy) { return (q >> 1) * 2 * nxy + 2 * c + (q & 1); }

// Shared-memory variant of advance_line for kFC frequencies at once: the geometry
// (shift, stencil, trilinear opacity, dt) is computed once per line and sub-node and
// reused for the kFC frequencies of the chunk.  Planes: chi [nxy], S [nxy][kFC].
// DT: dt of sub-segment m comes from the precomputed table (dtl = entry of (direction,
// step, line), stride nxy; prefetched one sub-node ahead) instead of the opacity planes.
// PLANAR (ny = 1, the 2D slab): sy = 0, so the stencil's second row has weight exactly 0
// and only two corners per layer are read (half the shared-memory traffic; same result).
// Sub-node table of one (direction, layer step), built once per CTA and step from the Shift
// table: integer shift plus the trilinear corner weights with wz = m / n_sub folded in
// (plane a: (1 - wz) w_xy, plane b: wz w_xy), so a thread spends no division, no weight
// products and 4 (planar) or 8 FMAs per sample and frequency.
struct SubW {
    int bx, by;
    double a00, a10, a01, a11, b00, b10, b01, b11;
};
__device__ __forceinline__ SubW subw_of(const Shift& sh, int m, int n_sub) {
    const double wz = static_cast<double>(m) / n_sub;
    const double w00 = (1 - sh.ax) * (1 - sh.ay), w10 = sh.ax * (1 - sh.ay), w01 = (1 - sh.ax) * sh.ay,
                 w11 = sh.ax * sh.ay;
    SubW w;
    w.bx = sh.bx;
    w.by = sh.by;
    w.a00 = (1 - wz) * w00;
    w.a10 = (1 - wz) * w10;
    w.a01 = (1 - wz) * w01;
    w.a11 = (1 - wz) * w11;
    w.b00 = wz * w00;
    w.b10 = wz * w10;
    w.b01 = wz * w01;
    w.b11 = wz * w11;
    return w;
}

template <int FS, bool DT, bool PLANAR>
__device__ __forceinline__ void advance_line_smem4(const LatDir& D, const SubW* __restrict__ sub,
                                                   double (&acc)[kFC], int lx, int ly, int t, int nx, int ny,
                                                   const double* chi_a, const double* chi_b,
                                                   const double* Sa, const double* Sb, const double (&phi)[kFC],
                                                   const double* __restrict__ dtl, int nxy) {
    double prev_s[kFC], prev_c = 0.0;
#pragma unroll
    for (int q = 0; q < kFC; ++q) prev_s[q] = 0.0;
    double dt_next = DT ? __ldg(dtl) : 0.0;
    // IE with tabulated dt needs no sample at the step's first point (its source enters only
    // the exponential solvers' upwind term, its opacity only the on-the-fly dt)
    for (int m = (FS == RTK_FS_IE && DT) ? 1 : 0; m <= D.n_sub; ++m) {
        const SubW W = sub[m];   // warp-uniform
        int i0 = lx + W.bx;
        if (i0 >= nx) i0 -= nx;
        const int i1 = (i0 + 1 == nx) ? 0 : i0 + 1;
        int c00, c10, c01 = 0, c11 = 0;
        if (PLANAR) {
            c00 = i0;
            c10 = i1;
        } else {
            int j0 = ly + W.by;
            if (j0 >= ny) j0 -= ny;
            const int j1 = (j0 + 1 == ny) ? 0 : j0 + 1;
            c00 = j0 * nx + i0;
            c10 = j0 * nx + i1;
            c01 = j1 * nx + i0;
            c11 = j1 * nx + i1;
        }
        double dt = 0.0, c_m = 0.0;
        if (DT) {
            if (m > 0) {
                dt = dt_next;
                if (m < D.n_sub) dt_next = __ldg(dtl + static_cast<int64_t>(m) * nxy);
            }
        } else {
            c_m = PLANAR ? (W.a00 * chi_a[c00] + W.a10 * chi_a[c10]) + (W.b00 * chi_b[c00] + W.b10 * chi_b[c10])
                         : (W.a00 * chi_a[c00] + W.a10 * chi_a[c10] + W.a01 * chi_a[c01] + W.a11 * chi_a[c11]) +
                               (W.b00 * chi_b[c00] + W.b10 * chi_b[c10] + W.b01 * chi_b[c01] + W.b11 * chi_b[c11]);
            dt = D.sub_len * (prev_c + c_m) * 0.5;
        }
        const double2* pa = reinterpret_cast<const double2*>(Sa);
        const double2* pb = reinterpret_cast<const double2*>(Sb);
#pragma unroll
        for (int h = 0; h < kFC / 2; ++h) {
            const int hh = h * nxy;
            const double2 p00 = pa[hh + c00], p10 = pa[hh + c10], q00 = pb[hh + c00], q10 = pb[hh + c10];
            double s2[2];
            if (PLANAR) {
                s2[0] = (W.a00 * p00.x + W.a10 * p10.x) + (W.b00 * q00.x + W.b10 * q10.x);
                s2[1] = (W.a00 * p00.y + W.a10 * p10.y) + (W.b00 * q00.y + W.b10 * q10.y);
            } else {
                const double2 p01 = pa[hh + c01], p11 = pa[hh + c11], q01 = pb[hh + c01], q11 = pb[hh + c11];
                s2[0] = (W.a00 * p00.x + W.a10 * p10.x + W.a01 * p01.x + W.a11 * p11.x) +
                        (W.b00 * q00.x + W.b10 * q10.x + W.b01 * q01.x + W.b11 * q11.x);
                s2[1] = (W.a00 * p00.y + W.a10 * p10.y + W.a01 * p01.y + W.a11 * p11.y) +
                        (W.b00 * q00.y + W.b10 * q10.y + W.b01 * q01.y + W.b11 * q11.y);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int q = 2 * h + e;
                if (m > 0) {
                    const double dtau = phi[q] * dt;
                    if (FS == RTK_FS_IE) {
                        const double r = rcp_nr(1.0 + dtau);
                        acc[q] = fma(acc[q], r, (dtau * s2[e]) * r);
                    } else {
                        const ExpLin w = exp_linear_weights(dtau);
                        acc[q] = fma(acc[q], w.att, w.wu * prev_s[q] + w.wc * s2[e]);
                    }
                }
                prev_s[q] = s2[e];
            }
        }
        prev_c = c_m;
    }
}

// Exp-parabolic (Kunasz-Auer) variant of advance_line_smem4 (oracle/lattice.py): the point
// P_m of the step is updated from P_{m-1}, P_m and the downwind P_{m+1}; for the step's last
// point the downwind is one sub-segment beyond the crossing (shift dsh, planes b / c of the
// next two layers), or, on the line's last step (no plane c), the linear weights are used.
// Samples are streamed one ahead; dt comes from the opacity planes (same arithmetic as the
// dt table, so LC results equal the table-driven kernels').
template <bool PLANAR>
struct ParSample {
    double s[kFC];
    double c;
};

template <bool PLANAR>
__device__ __forceinline__ void sample_planes(ParSample<PLANAR>& o, const Stencil& st, double wz,
                                              const double* chi_a, const double* chi_b, const double* Sa,
                                              const double* Sb, int nxy) {
    const double ca = PLANAR ? st.w00 * chi_a[st.c00] + st.w10 * chi_a[st.c10]
                             : st.w00 * chi_a[st.c00] + st.w10 * chi_a[st.c10] + st.w01 * chi_a[st.c01] +
                                   st.w11 * chi_a[st.c11];
    const double cb = PLANAR ? st.w00 * chi_b[st.c00] + st.w10 * chi_b[st.c10]
                             : st.w00 * chi_b[st.c00] + st.w10 * chi_b[st.c10] + st.w01 * chi_b[st.c01] +
                                   st.w11 * chi_b[st.c11];
    o.c = (1 - wz) * ca + wz * cb;
#pragma unroll
    for (int q = 0; q < kFC; ++q) {
        const double pa = PLANAR ? st.w00 * Sa[pidx(st.c00, q, nxy)] + st.w10 * Sa[pidx(st.c10, q, nxy)]
                                 : st.w00 * Sa[pidx(st.c00, q, nxy)] + st.w10 * Sa[pidx(st.c10, q, nxy)] +
                                       st.w01 * Sa[pidx(st.c01, q, nxy)] + st.w11 * Sa[pidx(st.c11, q, nxy)];
        const double pb = PLANAR ? st.w00 * Sb[pidx(st.c00, q, nxy)] + st.w10 * Sb[pidx(st.c10, q, nxy)]
                                 : st.w00 * Sb[pidx(st.c00, q, nxy)] + st.w10 * Sb[pidx(st.c10, q, nxy)] +
                                       st.w01 * Sb[pidx(st.c01, q, nxy)] + st.w11 * Sb[pidx(st.c11, q, nxy)];
        o.s[q] = (1 - wz) * pa + wz * pb;
    }
}

template <bool PLANAR>
__device__ __forceinline__ void advance_line_smem4_par(const LatDir& D, const Shift* __restrict__ sub, Shift dsh,
                                                       double (&acc)[kFC], int lx, int ly, int nx, int ny,
                                                       const double* chi_a, const double* chi_b,
                                                       const double* chi_c, const double* Sa, const double* Sb,
                                                       const double* Sc, const double (&phi)[kFC], int nxy) {
    ParSample<PLANAR> prev, cur, nxt;
    sample_planes<PLANAR>(prev, stencil_at(lx, ly, sub[0], nx, ny), 0.0, chi_a, chi_b, Sa, Sb, nxy);
    sample_planes<PLANAR>(cur, stencil_at(lx, ly, sub[1], nx, ny), 1.0 / D.n_sub, chi_a, chi_b, Sa, Sb, nxy);
    for (int m = 1; m <= D.n_sub; ++m) {
        const bool down = m < D.n_sub || Sc != nullptr;
        if (m < D.n_sub)
            sample_planes<PLANAR>(nxt, stencil_at(lx, ly, sub[m + 1], nx, ny), static_cast<double>(m + 1) / D.n_sub,
                                  chi_a, chi_b, Sa, Sb, nxy);
        else if (Sc != nullptr)
            sample_planes<PLANAR>(nxt, stencil_at(lx, ly, dsh, nx, ny), 1.0 / D.n_sub, chi_b, chi_c, Sb, Sc, nxy);
        const double dtu = D.sub_len * (prev.c + cur.c) * 0.5;
        const double dtd = D.sub_len * (cur.c + nxt.c) * 0.5;
#pragma unroll
        for (int q = 0; q < kFC; ++q) {
            if (down) {
                const ExpPar w = exp_parabolic_weights_bf(phi[q] * dtu, phi[q] * dtd);
                acc[q] = fma(acc[q], w.att, w.wu * prev.s[q] + w.wc * cur.s[q] + w.wd * nxt.s[q]);
            } else {
                const ExpLin w = exp_linear_weights_bf(phi[q] * dtu);
                acc[q] = fma(acc[q], w.att, w.wu * prev.s[q] + w.wc * cur.s[q]);
            }
        }
        prev = cur;
        cur = nxt;
    }
}

// Intensity layout, small layers (nxy <= ~1000, e.g. the 2D slab): one CTA per
// (direction, 4-frequency chunk), one thread per line handling the 4 frequencies.
// The source / opacity planes the lines cross and the x plane of the y = x - v gather
// are staged in shared memory by cp.async two layer steps ahead (rings of 3 and 2),
// so the global-memory latency of the plane loads overlaps the line march.
__device__ __forceinline__ void cp_async16_d(double* dst, const double* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src));
}

template <int FS, int SRC, int OUT, bool DT, bool PLANAR>
__global__ void __launch_bounds__(kIntThreads, RTK_INT_MINB) lattice_int_smem_kernel(LatArgs A, int with_inflow, int max_sub,
                                                                       int fchunk_slack, int vec16) {
    extern __shared__ __align__(16) double sm[];
    const int nxy = static_cast<int>(A.nxy);
    constexpr bool XM = (OUT == OUT_X_MINUS);
    double* lines0 = sm;                        // [2][nxy][kFC] line values: step t reads buffer t % 2, writes the other
    constexpr bool PAR = FS == RTK_FS_EXP_PARABOLIC;
    constexpr int RING = PAR ? 4 : 3;           // source / opacity plane ring (PAR reads layer t + 2)
    double* splane = lines0 + 2 * nxy * kFC;    // [RING][nxy][kFC]
    double* cplane = splane + RING * nxy * kFC; // [RING][nxy]      (opacity; unused with DT)
    double* xplane = cplane + ((RING * nxy + 1) & ~1);   // [2][nxy][kFC]   (XM only; 16-byte aligned for double2)
    double* seeds = xplane + 2 * nxy * kFC;     // [nxy][kFC] SC restart values
    Shift* shs0 = reinterpret_cast<Shift*>(seeds + nxy * kFC);  // [2][max_sub + 1] shifts of a step (exp-parabolic)
    SubW* sws0 = reinterpret_cast<SubW*>(shs0 + 2 * (max_sub + 1));   // [2][max_sub + 1] folded sub-node tables
    // Frequency chunks are cut at 32-byte sectors of the [node][direction][frequency] vectors:
    // with (n_dirs n_freq) % 4 == 0 the row of (node, direction a) starts (a n_freq) % 4
    // doubles past a sector boundary for every node, so the chunks of direction a start at
    // f0 = 4 j - (a n_freq) % 4 (the first and last ones partial) and each chunk's 4 doubles
    // are exactly one sector of src, x and y (an odd N_nu otherwise makes 3 of 4 directions
    // straddle two sectors per chunk: measured 1.85x the algorithmic DRAM traffic at cfg3).
    const int nfc = (A.n_freq + fchunk_slack + kFC - 1) / kFC;
    const int a = blockIdx.x / nfc;
    const int f0 = (blockIdx.x % nfc) * kFC - (fchunk_slack ? (a * A.n_freq) % kFC : 0);
    const int qlo = max(0, -f0), qhi = min(kFC, A.n_freq - f0);   // valid frequencies: f0 + [qlo, qhi)
    if (qhi <= qlo) return;
    const LatDir D = A.dirs[a];
    double phi[kFC], inflow[kFC];
#pragma unroll
    for (int q = 0; q < kFC; ++q) {
        const int f = f0 + q;
        const bool fv = f >= 0 && f < A.n_freq;
        phi[q] = fv ? A.phi[f] : 0.0;
        const double* in = D.down ? A.inflow_top : A.inflow_bottom;
        inflow[q] = (with_inflow && fv && in) ? in[f] : 0.0;
    }
    auto layer_of = [&](int t) { return D.down ? t : A.nz - 1 - t; };
    // source + opacity planes of layer k into ring slot r (asynchronous)
    auto issue_planes = [&](int k, int r) {
        const int64_t base = static_cast<int64_t>(k) * A.nxy;
        double* sp = splane + r * nxy * kFC;
        double* cp = cplane + r * nxy;
        // one (node, frequency pair) per iteration: a 16-byte copy when the pair is whole and
        // the chunks are sector-aligned (vec16), else per element
        for (int e = threadIdx.x; e < nxy * (kFC / 2); e += blockDim.x) {
            const int c = e / (kFC / 2), q = 2 * (e - c * (kFC / 2));
            const bool v0 = q >= qlo && q < qhi, v1 = q + 1 >= qlo && q + 1 < qhi;
            double* d = sp + pidx(c, q, nxy);
            const double* gsrc = SRC == LSRC_VEC ? A.src + ((base + c) * A.n_dirs + a) * A.n_freq + f0 + q
                                                 : A.src + (base + c) * A.n_freq + f0 + q;
            if (SRC == LSRC_VEC && vec16 && v0 && v1) {
                cp_async16_d(d, gsrc);
            } else {
                if (v0) cp_async8(d, gsrc);
                else d[0] = 0.0;
                if (v1) cp_async8(d + 1, gsrc + 1);
                else d[1] = 0.0;
            }
        }
        if (!DT)
            for (int c = threadIdx.x; c < nxy; c += blockDim.x) cp_async8(cp + c, A.chi + base + c);
    };
    auto issue_x = [&](int k, int r) {
        if (!XM) return;
        const int64_t base = static_cast<int64_t>(k) * A.nxy;
        double* xp = xplane + r * nxy * kFC;
        for (int e = threadIdx.x; e < nxy * (kFC / 2); e += blockDim.x) {
            const int c = e / (kFC / 2), q = 2 * (e - c * (kFC / 2));
            const bool v0 = q >= qlo && q < qhi, v1 = q + 1 >= qlo && q + 1 < qhi;
            double* d = xp + pidx(c, q, nxy);
            const double* gsrc = A.x + ((base + c) * A.n_dirs + a) * A.n_freq + f0 + q;
            if (vec16 && v0 && v1) {
                cp_async16_d(d, gsrc);
            } else {
                if (v0) cp_async8(d, gsrc);
                if (v1) cp_async8(d + 1, gsrc + 1);
            }
        }
    };
    auto commit = []() { asm volatile("cp.async.commit_group;\n" ::); };
    for (int e = threadIdx.x; e < nxy * kFC; e += blockDim.x) lines0[pidx(e / kFC, e % kFC, nxy)] = inflow[e % kFC];
    // sub-node table of step t into buffer t % 2 (staged one step ahead; the step's top barrier
    // orders it before its readers)
    auto stage_sub = [&](int t) {
        if (t >= A.nz - 1) return;
        for (int m = threadIdx.x; m <= D.n_sub; m += blockDim.x) {
            const Shift sh = A.sub_shift[D.shift_off + t * (D.n_sub + 1) + m];
            if (PAR) shs0[(t & 1) * (max_sub + 1) + m] = sh;
            else sws0[(t & 1) * (max_sub + 1) + m] = subw_of(sh, m, D.n_sub);
        }
    };
    stage_sub(0);
    // prologue: group 0 = planes(t=0) + x(t=0); group 1 = planes(t=1) + x(t=1)
    issue_planes(layer_of(0), 0);
    issue_x(layer_of(0), 0);
    commit();
    if (A.nz > 1) {
        issue_planes(layer_of(1), 1);
        issue_x(layer_of(1), 1);
    }
    commit();
    if (PAR && A.nz > 2) issue_planes(layer_of(2), 2);
    if (PAR) commit();
    static_assert(kIntThreads % (kFC / 2) == 0, "a thread keeps its frequency pair across gather iterations");
    const int gj0 = (static_cast<int>(threadIdx.x) / (kFC / 2)) / A.nx,
              gi0 = static_cast<int>(threadIdx.x) / (kFC / 2) - gj0 * A.nx;
    int gnbx, gnby;
    double gnax, gnay;
    {
        const Shift g0 = A.gat_shift[a * A.nz];
        gnbx = g0.bx;
        gnby = g0.by;
        gnax = g0.ax;
        gnay = g0.ay;
    }
    for (int t = 0; t < A.nz; ++t) {
        const int k = layer_of(t);
        // groups committed so far: t + 2 (steps 0..t+1); step t needs groups 0..t+1 (planes t and
        // t+1, x of t): all but none may stay pending
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        // prefetch for step t+1: planes of layer t+2 into the slot last used at step t-1, x of t+1
        if (t + RING - 1 < A.nz) issue_planes(layer_of(t + RING - 1), (t + RING - 1) % RING);
        if (t + 1 < A.nz && t > 0) issue_x(layer_of(t + 1), (t + 1) & 1);
        commit();
        stage_sub(t + 1);
        double* lines = lines0 + (t & 1) * nxy * kFC;          // written by the previous step's march
        double* lines_out = lines0 + ((t + 1) & 1) * nxy * kFC;
        const Shift* shs = shs0 + (t & 1) * (max_sub + 1);
        const SubW* sws = sws0 + (t & 1) * (max_sub + 1);
        // next step's sub-segment paths of this thread's lines into L1 (the march reads them one
        // sub-node ahead only, which left their L2 latency exposed)
        if (DT && t + 2 < A.nz) {
            const double* dn = A.dtab + D.dtab_off + static_cast<int64_t>(t + 1) * D.n_sub * A.nxy;
            for (int c = threadIdx.x; c < nxy; c += blockDim.x)
                for (int m = 0; m < D.n_sub; ++m)
                    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(dn + static_cast<int64_t>(m) * A.nxy + c));
        }
        // T_RC gather: one thread per (node, frequency) for coalesced y writes; the node's (i, j)
        // advance incrementally (blockDim.x / kFC nodes per iteration) instead of by division
        Shift gsh;
        gsh.bx = gnbx;
        gsh.by = gnby;
        gsh.ax = gnax;
        gsh.ay = gnay;
        if (t + 1 < A.nz) {
            const Shift* gn = A.gat_shift + a * A.nz + t + 1;
            gnbx = gn->bx;
            gnby = gn->by;
            gnax = gn->ax;
            gnay = gn->ay;
        }
        const double* xp = xplane + (t & 1) * nxy * kFC;
        int gi = gi0, gj = gj0;
        for (int e = threadIdx.x; e < nxy * (kFC / 2); e += blockDim.x) {
            const int c = e / (kFC / 2), q = 2 * (e - c * (kFC / 2));   // frequency pair (q, q + 1) of node c
            const int j = gj, i = gi;
            gi += kIntThreads / (kFC / 2);
            while (gi >= A.nx) {
                gi -= A.nx;
                ++gj;
            }
            const Stencil st = stencil_at(i, j, gsh, A.nx, A.ny);
            const double2* lp = reinterpret_cast<const double2*>(lines) + (q >> 1) * nxy;   // pair-major planes
            const double2 l00 = lp[st.c00], l10 = lp[st.c10], l01 = lp[st.c01], l11 = lp[st.c11];
            double2 v;
            v.x = st.w00 * l00.x + st.w10 * l10.x + st.w01 * l01.x + st.w11 * l11.x;
            v.y = st.w00 * l00.y + st.w10 * l10.y + st.w01 * l01.y + st.w11 * l11.y;
            if (XM) {
                const double2 xv = reinterpret_cast<const double2*>(xp)[(q >> 1) * nxy + c];
                v.x = xv.x - v.x;
                v.y = xv.y - v.y;
            }
            const bool v0 = q >= qlo && q < qhi, v1 = q + 1 >= qlo && q + 1 < qhi;
            double* yo = A.y + ((static_cast<int64_t>(k) * A.nxy + c) * A.n_dirs + a) * A.n_freq + f0 + q;
            if (vec16 && v0 && v1) {
                *reinterpret_cast<double2*>(yo) = v;
            } else {
                if (v0) yo[0] = v.x;
                if (v1) yo[1] = v.y;
            }
        }
        if (t == A.nz - 1) break;
        if (D.sc) {
            // short characteristics: every line restarts at its node's upwind point on this layer
            const Shift rsh = restart_shift(D);
            for (int e = threadIdx.x; e < nxy * kFC; e += blockDim.x) {
                const int c = e / kFC, q = e - c * kFC;
                const int j = c / A.nx, i = c - j * A.nx;
                const Stencil st = stencil_at(i, j, rsh, A.nx, A.ny);
                seeds[pidx(c, q, nxy)] = st.w00 * lines[pidx(st.c00, q, nxy)] + st.w10 * lines[pidx(st.c10, q, nxy)] +
                                         st.w01 * lines[pidx(st.c01, q, nxy)] + st.w11 * lines[pidx(st.c11, q, nxy)];
            }
        }
        // The march writes the OTHER line buffer, so the gather above needs no barrier before it
        // (one barrier per layer step); only the SC restart values cross threads here.
        if (D.sc) __syncthreads();
        const double* start = D.sc ? seeds : lines;
        const double* Sa = splane + (t % RING) * nxy * kFC;
        const double* Sb = splane + ((t + 1) % RING) * nxy * kFC;
        const double* ca = cplane + (t % RING) * nxy;
        const double* cb = cplane + ((t + 1) % RING) * nxy;
        const bool has_c = PAR && t + 2 < A.nz;
        const double* Sc = has_c ? splane + ((t + 2) % RING) * nxy * kFC : nullptr;
        const double* cc = has_c ? cplane + ((t + 2) % RING) * nxy : nullptr;
        const Shift dsh = PAR ? A.down_shift[a * A.nz + t] : Shift{};
        for (int c = threadIdx.x; c < nxy; c += blockDim.x) {
            const int ly = c / A.nx, lx = c - ly * A.nx;
            double acc[kFC];
#pragma unroll
            for (int q = 0; q < kFC; ++q) acc[q] = start[pidx(c, q, nxy)];
            if (PAR)
                advance_line_smem4_par<PLANAR>(D, shs, dsh, acc, lx, ly, A.nx, A.ny, ca, cb, cc, Sa, Sb, Sc, phi, nxy);
            else
            advance_line_smem4<FS, DT, PLANAR>(D, sws, acc, lx, ly, t, A.nx, A.ny, ca, cb, Sa, Sb, phi,
                                       DT ? A.dtab + D.dtab_off + static_cast<int64_t>(t) * D.n_sub * A.nxy + c : nullptr,
                                       nxy);
#pragma unroll
            for (int q = 0; q < kFC; ++q) lines_out[pidx(c, q, nxy)] = acc[q];
        }
    }
}

// ---------------- intensity layout: one CTA per (direction, frequency chunk) ----------------
template <int FS, int SRC, int OUT>
__global__ void __launch_bounds__(kIntThreads) lattice_int_kernel(LatArgs A, int with_inflow) {
    extern __shared__ double lines[];   // [nxy][kFC]
    const int nfc = (A.n_freq + kFC - 1) / kFC;
    const int a = blockIdx.x / nfc;
    const int f0 = (blockIdx.x % nfc) * kFC;
    const int fq = threadIdx.x % kFC;
    const int f = f0 + fq;
    const bool fvalid = f < A.n_freq;
    const int slots = blockDim.x / kFC;
    const int slot = threadIdx.x / kFC;
    const LatDir D = A.dirs[a];
    const double phi_f = fvalid ? A.phi[f] : 0.0;
    double inflow = 0.0;
    if (with_inflow && fvalid) {
        const double* in = D.down ? A.inflow_top : A.inflow_bottom;
        inflow = in ? in[f] : 0.0;
    }
    for (int l = slot; l < A.nxy; l += slots) lines[l * kFC + fq] = inflow;
    for (int t = 0; t < A.nz; ++t) {
        const int k = D.down ? t : A.nz - 1 - t;
        __syncthreads();
        // T_RC gather for the nodes of layer k
        const Shift gsh = A.gat_shift[a * A.nz + t];
        for (int c = slot; c < A.nxy; c += slots) {
            const int j = c / A.nx, i = c - j * A.nx;
            const Stencil st = stencil_at(i, j, gsh, A.nx, A.ny);
            const double v = st.w00 * lines[st.c00 * kFC + fq] + st.w10 * lines[st.c10 * kFC + fq] +
                             st.w01 * lines[st.c01 * kFC + fq] + st.w11 * lines[st.c11 * kFC + fq];
            if (fvalid) {
                const int64_t idx = ((static_cast<int64_t>(k) * A.nxy + c) * A.n_dirs + a) * A.n_freq + f;
                A.y[idx] = (OUT == OUT_X_MINUS) ? A.x[idx] - v : v;
            }
        }
        if (t == A.nz - 1) break;
        __syncthreads();
        const int k2 = D.down ? k + 1 : k - 1;
        // source planes of layers k and k2 for (a, f): S[s][a][f] (VEC) or thermal[s][f] (ISO)
        const int64_t ss = (SRC == LSRC_VEC) ? static_cast<int64_t>(A.n_dirs) * A.n_freq : A.n_freq;
        const int64_t off = (SRC == LSRC_VEC) ? static_cast<int64_t>(a) * A.n_freq + f : f;
        const double* Sa = A.src + static_cast<int64_t>(k) * A.nxy * ss + off;
        const double* Sb = A.src + static_cast<int64_t>(k2) * A.nxy * ss + off;
        const double* chi_a = A.chi + static_cast<int64_t>(k) * A.nxy;
        const double* chi_b = A.chi + static_cast<int64_t>(k2) * A.nxy;
        for (int c = slot; c < A.nxy; c += slots) {
            const int ly = c / A.nx, lx = c - ly * A.nx;
            double acc = lines[c * kFC + fq];   // long characteristics only (SC: smem kernel)
            if (fvalid)
                acc = advance_line<FS>(D, A.sub_shift + D.shift_off + t * (D.n_sub + 1), acc, lx, ly, t, A.nx, A.ny,
                                       chi_a, chi_b, Sa, Sb, ss, phi_f);
            lines[c * kFC + fq] = acc;
        }
    }
}

// F frequencies per thread (F even): the lattice geometry (shift, stencil, trilinear
// opacity, dt) is frequency-independent and computed once for the group; the internal
// planes use the even pitch fp so each group moves as F/2 16-byte loads.
// Trilinear opacity at sub-node m of a line (T_CR on the two opacity planes).
__device__ __forceinline__ double chi_at(const Stencil& st, double wz, const double* __restrict__ chi_a,
                                         const double* __restrict__ chi_b) {
    const double ca = st.w00 * __ldg(chi_a + st.c00) + st.w10 * __ldg(chi_a + st.c10) +
                      st.w01 * __ldg(chi_a + st.c01) + st.w11 * __ldg(chi_a + st.c11);
    const double cb = st.w00 * __ldg(chi_b + st.c00) + st.w10 * __ldg(chi_b + st.c10) +
                      st.w01 * __ldg(chi_b + st.c01) + st.w11 * __ldg(chi_b + st.c11);
    return (1 - wz) * ca + wz * cb;
}

// DTAB: the frequency-independent sub-segment optical paths dt are read from the
// precomputed [dir][layer step][sub-segment][line] table (one coalesced load instead of
// eight opacity samples); dtab points at (direction, step t, line) and has stride nxy.
template <int FS, int F, bool DTAB>
__device__ __forceinline__ void advance_lineF(const LatDir& D, const Shift* __restrict__ sub, double (&acc)[F],
                                              int lx, int ly, int t, int nx, int ny, const double* __restrict__ chi_a,
                                              const double* __restrict__ chi_b, const double2* __restrict__ Sa,
                                              const double2* __restrict__ Sb, int64_t ss, const double (&phi)[F],
                                              const double* __restrict__ dtab, int64_t nxy) {
    double prev_s[F], prev_c = 0.0;
#pragma unroll
    for (int q = 0; q < F; ++q) prev_s[q] = 0.0;
    for (int m = 0; m <= D.n_sub; ++m) {
        const double wz = static_cast<double>(m) / D.n_sub;
        const Shift sh = sub[m];   // warp-uniform, precomputed at setup (same arithmetic as shift_of)
        const Stencil st = stencil_at(lx, ly, sh, nx, ny);
        double dt = 0.0, c_m = 0.0;
        if (DTAB) {
            if (m > 0) dt = __ldg(dtab + static_cast<int64_t>(m - 1) * nxy);
        } else {
            c_m = chi_at(st, wz, chi_a, chi_b);
            dt = D.sub_len * (prev_c + c_m) * 0.5;
        }
#pragma unroll
        for (int h = 0; h < F / 2; ++h) {
            const double2 a00 = __ldg(Sa + st.c00 * ss + h), a10 = __ldg(Sa + st.c10 * ss + h);
            const double2 a01 = __ldg(Sa + st.c01 * ss + h), a11 = __ldg(Sa + st.c11 * ss + h);
            const double2 b00 = __ldg(Sb + st.c00 * ss + h), b10 = __ldg(Sb + st.c10 * ss + h);
            const double2 b01 = __ldg(Sb + st.c01 * ss + h), b11 = __ldg(Sb + st.c11 * ss + h);
            double s2[2];
            s2[0] = (1 - wz) * (st.w00 * a00.x + st.w10 * a10.x + st.w01 * a01.x + st.w11 * a11.x) +
                    wz * (st.w00 * b00.x + st.w10 * b10.x + st.w01 * b01.x + st.w11 * b11.x);
            s2[1] = (1 - wz) * (st.w00 * a00.y + st.w10 * a10.y + st.w01 * a01.y + st.w11 * a11.y) +
                    wz * (st.w00 * b00.y + st.w10 * b10.y + st.w01 * b01.y + st.w11 * b11.y);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int q = 2 * h + e;
                if (m > 0) {
                    const double dtau = phi[q] * dt;
                    if (FS == RTK_FS_IE) {
                        const double r = rcp_nr(1.0 + dtau);
                        acc[q] = fma(acc[q], r, (dtau * s2[e]) * r);
                    } else {
                        const ExpLin w = exp_linear_weights(dtau);
                        acc[q] = fma(acc[q], w.att, w.wu * prev_s[q] + w.wc * s2[e]);
                    }
                }
                prev_s[q] = s2[e];
            }
        }
        prev_c = c_m;
    }
}

// Exp-parabolic advance of a line over one layer step in the moment layout (oracle/lattice.py):
// point m is updated from m - 1, m and the downwind m + 1; the downwind of the step's last
// point lies one sub-segment beyond the crossing (shift dsh, planes Sb / Sc of the next two
// layers, dt from the opacity: chi_a / chi_b / chi_c are the three layers), or the linear
// weights apply on the line's last step (Sc == nullptr).  Interior dt from the table.
template <int F>
__device__ __forceinline__ void sample_s2(double (&out)[F], const Stencil& st, double wz, const double2* __restrict__ Sa,
                                          const double2* __restrict__ Sb, int64_t ss) {
#pragma unroll
    for (int h = 0; h < F / 2; ++h) {
        const double2 a00 = __ldg(Sa + st.c00 * ss + h), a10 = __ldg(Sa + st.c10 * ss + h);
        const double2 a01 = __ldg(Sa + st.c01 * ss + h), a11 = __ldg(Sa + st.c11 * ss + h);
        const double2 b00 = __ldg(Sb + st.c00 * ss + h), b10 = __ldg(Sb + st.c10 * ss + h);
        const double2 b01 = __ldg(Sb + st.c01 * ss + h), b11 = __ldg(Sb + st.c11 * ss + h);
        out[2 * h] = (1 - wz) * (st.w00 * a00.x + st.w10 * a10.x + st.w01 * a01.x + st.w11 * a11.x) +
                     wz * (st.w00 * b00.x + st.w10 * b10.x + st.w01 * b01.x + st.w11 * b11.x);
        out[2 * h + 1] = (1 - wz) * (st.w00 * a00.y + st.w10 * a10.y + st.w01 * a01.y + st.w11 * a11.y) +
                         wz * (st.w00 * b00.y + st.w10 * b10.y + st.w01 * b01.y + st.w11 * b11.y);
    }
}

template <int F>
__device__ __forceinline__ void advance_lineF_par(int n_sub, double sub_len, const Shift* __restrict__ sub, Shift dsh,
                                                  double (&acc)[F], int lx, int ly, int nx, int ny,
                                                  const double2* __restrict__ Sa, const double2* __restrict__ Sb,
                                                  const double2* __restrict__ Sc, int64_t ss, const double (&phi)[F],
                                                  const double* __restrict__ dtab, int64_t nxy,
                                                  const double* __restrict__ chi_a, const double* __restrict__ chi_b,
                                                  const double* __restrict__ chi_c, bool dt_next_tab) {
    const double inv_n = 1.0 / n_sub;
    double sp[F], sc[F], sn[F];
    sample_s2<F>(sp, stencil_at(lx, ly, sub[0], nx, ny), 0.0, Sa, Sb, ss);
    sample_s2<F>(sc, stencil_at(lx, ly, sub[1], nx, ny), inv_n, Sa, Sb, ss);
    double dtu = __ldg(dtab);
    for (int m = 1; m <= n_sub; ++m) {
        const bool down = m < n_sub || Sc != nullptr;
        double dtd = 0.0;
        if (m < n_sub) {
            sample_s2<F>(sn, stencil_at(lx, ly, sub[m + 1], nx, ny), static_cast<double>(m + 1) / n_sub, Sa, Sb, ss);
            dtd = __ldg(dtab + static_cast<int64_t>(m) * nxy);
        } else if (Sc != nullptr) {
            const Stencil sx = stencil_at(lx, ly, dsh, nx, ny);
            sample_s2<F>(sn, sx, inv_n, Sb, Sc, ss);
            if (dt_next_tab) {
                // LC: the downwind segment is the line's first sub-segment of step t + 1, whose
                // table entry follows this step's last (same shifts, same arithmetic)
                dtd = __ldg(dtab + static_cast<int64_t>(n_sub) * nxy);
            } else {
                const double cn = chi_at(stencil_at(lx, ly, sub[n_sub], nx, ny), 1.0, chi_a, chi_b);
                dtd = sub_len * (cn + chi_at(sx, inv_n, chi_b, chi_c)) * 0.5;
            }
        }
#pragma unroll
        for (int q = 0; q < F; ++q) {
            if (down) {
                const ExpPar w = exp_parabolic_weights_bf(phi[q] * dtu, phi[q] * dtd);
                acc[q] = fma(acc[q], w.att, w.wu * sp[q] + w.wc * sc[q] + w.wd * sn[q]);
            } else {
                const ExpLin w = exp_linear_weights_bf(phi[q] * dtu);
                acc[q] = fma(acc[q], w.att, w.wu * sp[q] + w.wc * sc[q]);
            }
            sp[q] = sc[q];
            sc[q] = sn[q];
        }
        dtu = dtd;
    }
}

// dt table: dtab[D.dtab_off + (t * n_sub + m - 1) * nxy + c] = sub_len (chi(m-1) + chi(m)) / 2,
// computed with the same expressions as the on-the-fly path.
__global__ void lattice_dtab_kernel(const LatDir* __restrict__ dirs, const Shift* __restrict__ sub_shift,
                                    const double* __restrict__ chi, double* __restrict__ dtab, int n_dirs, int nx,
                                    int ny, int nz) {
    const int64_t nxy = static_cast<int64_t>(nx) * ny;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int a = blockIdx.y;
    if (tid >= nxy * (nz - 1) || a >= n_dirs) return;
    const int t = static_cast<int>(tid / nxy);
    const int c = static_cast<int>(tid - static_cast<int64_t>(t) * nxy);
    const LatDir D = dirs[a];
    const int k = D.down ? t : nz - 1 - t;
    const int k2 = D.down ? k + 1 : k - 1;
    const int ly = c / nx, lx = c - ly * nx;
    const Shift* sub = sub_shift + D.shift_off + t * (D.n_sub + 1);
    double prev_c = 0.0;
    for (int m = 0; m <= D.n_sub; ++m) {
        const double wz = static_cast<double>(m) / D.n_sub;
        const Stencil st = stencil_at(lx, ly, sub[m], nx, ny);
        const double c_m = chi_at(st, wz, chi + static_cast<int64_t>(k) * nxy, chi + static_cast<int64_t>(k2) * nxy);
        if (m > 0)
            dtab[D.dtab_off + (static_cast<int64_t>(t) * D.n_sub + m - 1) * nxy + c] = D.sub_len * (prev_c + c_m) * 0.5;
        prev_c = c_m;
    }
}

// thread = (line c, frequency group q of F): f = F q .. F q + F - 1 (the tail may be padding).
// Directions are processed hemisphere by hemisphere so only NM x F moment accumulators
// are live; layer t gets the down part, layer nz-1-t the up part.
struct StepDir {
    int down, n_sub, sub_pref, sc;
    long long dtab;        // this step's first dt-table entry of the direction
    double wy[8];
};

// DG direction groups: the CTA is DG x IPB threads, thread (dgi, item) handles directions
// a = dgi, dgi + DG, ... of item (line, frequency group) blockIdx.x * IPB + item, and the DG
// partial moments of an item are summed in shared memory in dgi order (deterministic).  A
// layer step has only nxy * fp / F items (cfg4: 65,536 = 14 warps per SM); DG = 8 gives the
// SMs 8x the warps to hide the L2 latency of the gathers with.
template <int FS, int NM, int F, int DG>
__global__ void __launch_bounds__(DG == 1 ? 128 : 256, DG == 1 ? 5 : 3)
    lattice_mom_group_kernel(LatArgs A, int t, const double* __restrict__ st_in,
                                                                 double* __restrict__ st_out, double* __restrict__ mom,
                                                                 int with_inflow, int fp,
                                                                 const double* __restrict__ plane_cur,
                                                                 const double* __restrict__ plane_next,
                                                                 const double* __restrict__ plane_nn) {
    const int ng = (fp + F - 1) / F;       // groups per line
    const int hp = fp >> 1;                // double2 per line in the [dir][line][fp] planes
    // this step's direction metadata and shifts, staged once per CTA in shared memory (the
    // per-direction / per-sub-node lookups are warp-uniform and sat on the load-latency chain)
    extern __shared__ double mo_s[];       // [NM][F][blockDim] accumulators, then the tables
    StepDir* sdir = reinterpret_cast<StepDir*>(mo_s + NM * F * blockDim.x);
    Shift* sgat = reinterpret_cast<Shift*>(sdir + A.n_dirs);
    Shift* srst = sgat + A.n_dirs;          // SC restart shifts
    Shift* ssub = srst + A.n_dirs;
    for (int a = threadIdx.x; a < A.n_dirs; a += blockDim.x) {
        const LatDir& D = A.dirs[a];
        StepDir sd;
        sd.down = D.down;
        sd.n_sub = D.n_sub;
        sd.sub_pref = D.sub_pref;
        sd.sc = D.sc;
        sd.dtab = D.dtab_off + static_cast<int64_t>(t) * D.n_sub * A.nxy;
        srst[a] = restart_shift(D);
#pragma unroll
        for (int l = 0; l < NM; ++l) sd.wy[l] = D.wy[l];
        sdir[a] = sd;
        sgat[a] = A.gat_shift[a * A.nz + t];
    }
    if (t < A.nz - 1) {
        for (int e = threadIdx.x; e < A.total_sub; e += blockDim.x) {
            // entry e belongs to the direction whose prefix range holds it
            int lo = 0, hi = A.n_dirs - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (A.dirs[mid].sub_pref <= e) lo = mid;
                else hi = mid - 1;
            }
            const LatDir& D = A.dirs[lo];
            ssub[e] = A.sub_shift[D.shift_off + t * (D.n_sub + 1) + (e - D.sub_pref)];
        }
    }
    __syncthreads();
    const int ipb = blockDim.x / DG;                 // items per CTA
    const int dgi = threadIdx.x / ipb;               // direction group of this thread
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * ipb + (threadIdx.x - dgi * ipb);
    const bool item_ok = tid < A.nxy * ng;
    if (DG == 1 && !item_ok) return;
    const int c = item_ok ? static_cast<int>(tid / ng) : 0;
    const int g = static_cast<int>(tid - static_cast<int64_t>(c) * ng);
    const int f0 = F * g;
    const int j = c / A.nx, i = c - j * A.nx;
    double phi[F], in_top[F], in_bot[F];
    bool fv[F];
#pragma unroll
    for (int q = 0; q < F; ++q) {
        const int f = f0 + q;
        fv[q] = f < A.n_freq;
        phi[q] = fv[q] ? A.phi[f] : 0.0;
        in_top[q] = (with_inflow && fv[q] && A.inflow_top) ? A.inflow_top[f] : 0.0;
        in_bot[q] = (with_inflow && fv[q] && A.inflow_bottom) ? A.inflow_bottom[f] : 0.0;
    }
    // the last group of a line may reach past fp when F does not divide fp: clamp its loads
    const bool full_group = f0 + F <= fp;
    const int64_t plane2 = A.nxy * static_cast<int64_t>(hp);
    const double2* sin2 = reinterpret_cast<const double2*>(st_in);
    double2* sout2 = reinterpret_cast<double2*>(st_out);
    const double2* pc2 = reinterpret_cast<const double2*>(plane_cur);
    const double2* pn2 = reinterpret_cast<const double2*>(plane_next);
    const double2* pnn2 = reinterpret_cast<const double2*>(plane_nn);   // exp-parabolic, may be null
    const int g2 = f0 >> 1;               // first double2 of the group within a line
    for (int hemi = 0; hemi < 2; ++hemi) {       // 0: down (layer t), 1: up (layer nz-1-t)
        const int k = hemi == 0 ? t : A.nz - 1 - t;
        // moment accumulators live in shared memory ([l][q][thread], conflict-free) to keep
        // registers for the loads in flight (occupancy)
        auto mo = [&](int l, int q) -> double& { return mo_s[(l * F + q) * blockDim.x + threadIdx.x]; };
#pragma unroll
        for (int l = 0; l < NM; ++l)
#pragma unroll
            for (int q = 0; q < F; ++q) mo(l, q) = 0.0;
        for (int a = A.a0 + dgi; a < A.a1 && item_ok; a += DG) {
            const StepDir& D = sdir[a];
            if ((D.down != 0) != (hemi == 0)) continue;
            const double2* sa = sin2 + a * plane2 + g2;
            double v[F];
            if (t == 0) {
#pragma unroll
                for (int q = 0; q < F; ++q) v[q] = hemi == 0 ? in_top[q] : in_bot[q];
            } else {
                const Stencil st = stencil_at(i, j, sgat[a], A.nx, A.ny);
#pragma unroll
                for (int h = 0; h < F / 2; ++h) {
                    if (!full_group && g2 + h >= hp) {
                        v[2 * h] = v[2 * h + 1] = 0.0;
                        continue;
                    }
                    const double2 s00 = sa[st.c00 * hp + h], s10 = sa[st.c10 * hp + h];
                    const double2 s01 = sa[st.c01 * hp + h], s11 = sa[st.c11 * hp + h];
                    v[2 * h] = st.w00 * s00.x + st.w10 * s10.x + st.w01 * s01.x + st.w11 * s11.x;
                    v[2 * h + 1] = st.w00 * s00.y + st.w10 * s10.y + st.w01 * s01.y + st.w11 * s11.y;
                }
            }
#pragma unroll
            for (int l = 0; l < NM; ++l) {
                const double w = D.wy[l];
#pragma unroll
                for (int q = 0; q < F; ++q) mo(l, q) = fma(w, v[q], mo(l, q));
            }
            if (t < A.nz - 1) {
                const int k2 = hemi == 0 ? k + 1 : k - 1;
                double acc[F];
                if (D.sc && t > 0) {
                    // short characteristics: restart at the upwind point of node c (bilinear
                    // from the previous step's node values = line values)
                    const Stencil rs = stencil_at(i, j, srst[a], A.nx, A.ny);
#pragma unroll
                    for (int h = 0; h < F / 2; ++h) {
                        if (!full_group && g2 + h >= hp) {
                            acc[2 * h] = acc[2 * h + 1] = 0.0;
                            continue;
                        }
                        const double2 s00 = sa[rs.c00 * hp + h], s10 = sa[rs.c10 * hp + h];
                        const double2 s01 = sa[rs.c01 * hp + h], s11 = sa[rs.c11 * hp + h];
                        acc[2 * h] = rs.w00 * s00.x + rs.w10 * s10.x + rs.w01 * s01.x + rs.w11 * s11.x;
                        acc[2 * h + 1] = rs.w00 * s00.y + rs.w10 * s10.y + rs.w01 * s01.y + rs.w11 * s11.y;
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < F / 2; ++h) {
                        double2 s2;
                        if (t == 0) s2 = hemi == 0 ? make_double2(in_top[2 * h], in_top[2 * h + 1])
                                                    : make_double2(in_bot[2 * h], in_bot[2 * h + 1]);
                        else s2 = (!full_group && g2 + h >= hp) ? make_double2(0.0, 0.0)
                                                                : sa[static_cast<int64_t>(c) * hp + h];
                        acc[2 * h] = s2.x;
                        acc[2 * h + 1] = s2.y;
                    }
                }
                LatDir Dl;
                Dl.n_sub = D.n_sub;
                constexpr bool PAR = FS == RTK_FS_EXP_PARABOLIC;
                const int k3 = hemi == 0 ? k2 + 1 : k2 - 1;
                const Shift dsh = PAR ? A.down_shift[a * A.nz + t] : Shift{};
                const double* chk = A.chi + static_cast<int64_t>(k) * A.nxy;
                const double* chk2 = A.chi + static_cast<int64_t>(k2) * A.nxy;
                const double* chk3 = pnn2 ? A.chi + static_cast<int64_t>(k3) * A.nxy : nullptr;
                if (PAR && full_group) {
                    advance_lineF_par<F>(D.n_sub, A.dirs[a].sub_len, ssub + D.sub_pref, dsh, acc, i, j, A.nx, A.ny,
                                         pc2 + a * plane2 + g2, pn2 + a * plane2 + g2,
                                         pnn2 ? pnn2 + a * plane2 + g2 : nullptr, hp, phi, A.dtab + D.dtab + c, A.nxy,
                                         chk, chk2, chk3, !D.sc);
#pragma unroll
                    for (int h = 0; h < F / 2; ++h)
                        sout2[a * plane2 + static_cast<int64_t>(c) * hp + g2 + h] = make_double2(acc[2 * h], acc[2 * h + 1]);
                } else if (PAR) {
                    for (int h = 0; h < F / 2 && g2 + h < hp; ++h) {
                        double ap[2] = {acc[2 * h], acc[2 * h + 1]};
                        const double pp[2] = {phi[2 * h], phi[2 * h + 1]};
                        advance_lineF_par<2>(D.n_sub, A.dirs[a].sub_len, ssub + D.sub_pref, dsh, ap, i, j, A.nx, A.ny,
                                             pc2 + a * plane2 + g2 + h, pn2 + a * plane2 + g2 + h,
                                             pnn2 ? pnn2 + a * plane2 + g2 + h : nullptr, hp, pp,
                                             A.dtab + D.dtab + c, A.nxy, chk, chk2, chk3, !D.sc);
                        sout2[a * plane2 + static_cast<int64_t>(c) * hp + g2 + h] = make_double2(ap[0], ap[1]);
                    }
                } else if (full_group) {
                    advance_lineF<FS, F, true>(Dl, ssub + D.sub_pref, acc, i, j, t, A.nx, A.ny, nullptr, nullptr,
                                               pc2 + a * plane2 + g2, pn2 + a * plane2 + g2, hp, phi,
                                               A.dtab + D.dtab + c, A.nxy);
#pragma unroll
                    for (int h = 0; h < F / 2; ++h)
                        sout2[a * plane2 + static_cast<int64_t>(c) * hp + g2 + h] = make_double2(acc[2 * h], acc[2 * h + 1]);
                } else {
                    // tail group: process as pairs within the pitch
                    for (int h = 0; h < F / 2 && g2 + h < hp; ++h) {
                        double ap[2] = {acc[2 * h], acc[2 * h + 1]};
                        const double pp[2] = {phi[2 * h], phi[2 * h + 1]};
                        advance_lineF<FS, 2, true>(Dl, ssub + D.sub_pref, ap, i, j, t, A.nx, A.ny, nullptr, nullptr,
                                                   pc2 + a * plane2 + g2 + h, pn2 + a * plane2 + g2 + h, hp, pp,
                                                   A.dtab + D.dtab + c, A.nxy);
                        sout2[a * plane2 + static_cast<int64_t>(c) * hp + g2 + h] = make_double2(ap[0], ap[1]);
                    }
                }
            }
        }
        if (DG > 1) {
            // partial moments of the DG direction groups, summed by group 0 in dgi order
            __syncthreads();
            if (dgi == 0 && item_ok) {
#pragma unroll
                for (int l = 0; l < NM; ++l)
#pragma unroll
                    for (int q = 0; q < F; ++q) {
                        double sum = mo(l, q);
                        for (int g2i = 1; g2i < DG; ++g2i) sum += mo_s[(l * F + q) * blockDim.x + threadIdx.x + g2i * ipb];
                        mo(l, q) = sum;
                    }
            }
            __syncthreads();
            if (dgi != 0 || !item_ok) continue;
        }
        // step t is the first visit of layers t and nz-1-t iff t < nz-1-t; the middle layer
        // (odd nz) gets both parts in this thread, up added to down
        const bool first = (hemi == 0) ? (t <= A.nz - 1 - t) : (t < A.nz - 1 - t);
        double* out = mom + (static_cast<int64_t>(k) * A.nxy + c) * NM * fp + f0;
#pragma unroll
        for (int l = 0; l < NM; ++l) {
#pragma unroll
            for (int q = 0; q < F; ++q) {
                if (f0 + q >= fp) continue;
                const double val = fv[q] ? mo(l, q) : 0.0;
                double* o = out + static_cast<int64_t>(l) * fp + q;
                *o = first ? val : *o + val;
            }
        }
    }
}

// Source planes: for every direction a, S_a on the layers its march visits at offsets
// o = 0, 1, 2 from step t (down: t + o, up: nz - 1 - t - o) into plane_o, for the offsets in
// fill_mask (bit o); S = gamma sum_l c_l Y_l(a) u_l (SRC_U) or the isotropic thermal source
// (SRC_ISO).  Layout plane[a][c][f] (the per-item kernels; the tiled kernel's pair-major planes
// come from lattice_splane_pm_kernel below).  Offset 2 is the exp-parabolic downwind plane.
template <int SRC, int NM>
__global__ void __launch_bounds__(256) lattice_splane_kernel(LatArgs A, int t, double* __restrict__ plane0,
                                                              double* __restrict__ plane1,
                                                              double* __restrict__ plane2, int fill_mask, int fp) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= A.nxy * fp) return;
    const int64_t c = tid / fp;
    const int fpad = static_cast<int>(tid - c * fp);
    const bool fvalid = fpad < A.n_freq;
    const int f = fvalid ? fpad : 0;
    const int64_t plane = A.nxy * fp;
    double* planes[3] = {plane0, plane1, plane2};

    // q = 2 o + (0: down, 1: up)
    double uval[6][NM], g[6];
    bool use[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const int o = q >> 1;
        const int layer = (q & 1) ? A.nz - 1 - t - o : t + o;
        use[q] = ((fill_mask >> o) & 1) && layer >= 0 && layer < A.nz;
        g[q] = 0.0;
#pragma unroll
        for (int l = 0; l < NM; ++l) uval[q][l] = 0.0;
        if (!use[q]) continue;
        const int64_t sidx = static_cast<int64_t>(layer) * A.nxy + c;
        if (SRC == LSRC_U) {
#pragma unroll
            for (int l = 0; l < NM; ++l) uval[q][l] = __ldg(A.src + (sidx * NM + l) * A.n_freq + f);
            g[q] = __ldg(A.gamma + sidx * A.n_freq + f);
        } else {
            g[q] = __ldg(A.src + sidx * A.n_freq + f);
        }
    }
    for (int a = A.a0; a < A.a1; ++a) {
        const LatDir& D = A.dirs[a];
        const int qd = D.down ? 0 : 1;
        double cy[NM];
#pragma unroll
        for (int l = 0; l < NM; ++l) cy[l] = D.cy[l];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            if ((q & 1) != qd || !use[q]) continue;
            double v;
            if (SRC == LSRC_U) {
                v = 0.0;
#pragma unroll
                for (int l = 0; l < NM; ++l) v = fma(cy[l], uval[q][l], v);
                v *= g[q];
            } else {
                v = g[q];
            }
            const int64_t idx = a * plane + c * fp + fpad;
            planes[q >> 1][idx] = fvalid ? v : 0.0;
        }
    }
}

// Pair-major source planes for the tiled moment kernel: thread = (frequency pair, node), node
// fastest, so each direction's plane is written with one coalesced 16-byte store per thread
// (the generic kernel above: 8-byte stores and ~60 instructions per value).  The per-direction
// coefficients c_l Y_l(a) and the hemisphere flags sit in shared memory; the node's moments
// (both frequencies of the pair) are loaded once per hemisphere and reused by its directions.
// Same arithmetic as lattice_splane_kernel (v = (sum_l cy_l u_l) gamma in l order).
template <int SRC, int NM>
__global__ void __launch_bounds__(256) lattice_splane_pm_kernel(LatArgs A, int t, double2* __restrict__ plane0,
                                                                 double2* __restrict__ plane1,
                                                                 double2* __restrict__ plane2, int fill_mask, int fp) {
    extern __shared__ __align__(16) double spm[];
    const int nd = A.a1 - A.a0;
    double* cys = spm;                                         // [nd][NM]
    int* downs = reinterpret_cast<int*>(cys + nd * NM);        // [nd]
    for (int e = threadIdx.x; e < nd * NM; e += blockDim.x) cys[e] = A.dirs[A.a0 + e / NM].cy[e % NM];
    for (int e = threadIdx.x; e < nd; e += blockDim.x) downs[e] = A.dirs[A.a0 + e].down;
    __syncthreads();
    const int hp = fp >> 1;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= A.nxy * hp) return;
    const int pr = static_cast<int>(tid / A.nxy);
    const int64_t c = tid - pr * A.nxy;
    const int f0 = 2 * pr, f1 = 2 * pr + 1;
    const bool v0 = f0 < A.n_freq, v1 = f1 < A.n_freq;
    const int64_t plane = A.nxy * hp;   // double2 per direction
    double2* planes[3] = {plane0, plane1, plane2};
    for (int o = 0; o < 3; ++o) {
        if (!((fill_mask >> o) & 1)) continue;
        double2* out = planes[o] + pr * A.nxy + c;
        for (int hm = 0; hm < 2; ++hm) {
            const int layer = hm ? A.nz - 1 - t - o : t + o;
            if (layer < 0 || layer >= A.nz) continue;
            const int64_t sidx = static_cast<int64_t>(layer) * A.nxy + c;
            double u0[NM], u1[NM], g0, g1;
            if (SRC == LSRC_U) {
#pragma unroll
                for (int l = 0; l < NM; ++l) {
                    const double* up = A.src + (sidx * NM + l) * A.n_freq;
                    u0[l] = v0 ? __ldg(up + f0) : 0.0;
                    u1[l] = v1 ? __ldg(up + f1) : 0.0;
                }
                g0 = v0 ? __ldg(A.gamma + sidx * A.n_freq + f0) : 0.0;
                g1 = v1 ? __ldg(A.gamma + sidx * A.n_freq + f1) : 0.0;
            } else {
                g0 = v0 ? __ldg(A.src + sidx * A.n_freq + f0) : 0.0;
                g1 = v1 ? __ldg(A.src + sidx * A.n_freq + f1) : 0.0;
            }
#pragma unroll 4
            for (int i = 0; i < nd; ++i) {
                if ((downs[i] != 0) != (hm == 0)) continue;
                double s0, s1;
                if (SRC == LSRC_U) {
                    const double* cy = cys + i * NM;
                    s0 = 0.0;
                    s1 = 0.0;
#pragma unroll
                    for (int l = 0; l < NM; ++l) {
                        s0 = fma(cy[l], u0[l], s0);
                        s1 = fma(cy[l], u1[l], s1);
                    }
                    s0 *= g0;
                    s1 *= g1;
                } else {
                    s0 = g0;
                    s1 = g1;
                }
                out[(A.a0 + i) * plane] = make_double2(v0 ? s0 : 0.0, v1 ? s1 : 0.0);
            }
        }
    }
}

// ---------------- moment layout, tiled: one CTA per (tile of lines, frequency pair) ----------------
//
// lattice_mom_tile_kernel (IE / exp-linear).  Every line of a direction samples the source at
// the same fractional offset at a given (layer step, sub-node), so for a TX x TY tile of lines
// the samples of one step lie in one (TX + span_x + 1) x (TY + span_y + 1) window of the two
// source planes the step crosses (span = the whole-cell shift range of the step, <= |s| + 1).
// The CTA stages that window of direction a + 1 (both planes, one frequency pair, double2 in
// the pair-major [dir][pair][node] plane layout) and the direction's sub-node table with
// cp.async while it marches direction a out of shared memory: a sample is 8 LDS.128 from
// 32-bit addresses instead of 8 L1/L2 gathers with 64-bit address arithmetic.  The T_RC node
// gather (once per direction and step) reads the [dir][pair][line] line states from global.
// Moments accumulate in registers over one hemisphere's directions (fixed order); with DGZ > 1
// direction groups (gridDim.z) the groups' partial moments go to a scratch array that
// lattice_mom_reduce_kernel sums in group order (deterministic).
struct TileHdr {
    int fx, fy;   // window origin: min over the step's sub-nodes of floor(offset), wrapped mod (nx, ny)
    int w, h;     // window extent (nodes)
};
struct TileSub {
    int dx, dy;           // sub-node offset within the window (unwrapped)
    // trilinear weights of the eight corners: plane a (the step's start layer) carries
    // (1 - wz) w_xy, plane b wz w_xy, with w_xy the bilinear weights of stencil_at and
    // wz = m / n_sub (folded on the host: 8 FMAs per sample and frequency instead of 11)
    double a00, a10, a01, a11, b00, b10, b01, b11;
    double pad;
};
static_assert(sizeof(TileSub) == 80, "TileSub is staged as five 16-byte words");
constexpr int kTileSubW = sizeof(TileSub) / 16;

struct TileArgs {
    const TileHdr* hdr;     // [dir][step]
    const TileSub* sub;     // indexed like the sub-node Shift table: shift_off + t (n_sub + 1) + m
    const int* order;       // direction order: this call's down directions, then its up directions
    int n_order, n_down;    // entries of order; the first n_down are Omega_z < 0
    int region_cap;         // double2 per staged plane window (max over directions)
    int sub_cap;            // max n_sub + 1
    int ntx;                // tiles along x
    int dgz;                // direction groups (gridDim.z)
    int n_stages;           // window stages in shared memory (3 when they fit, else 2)
    double* scratch;        // DGZ > 1: [group][hemi][line][NM][fp]
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

// per-direction metadata of one launch (one layer step), staged in shared memory once so the
// per-direction control flow never waits on a global load
struct TileDir {
    int n_sub, sc, shift_off, down;
    long long dtab;          // this step's first dt-table entry of the direction
    TileHdr hdr;             // this step's window
    Shift gat;               // this step's T_RC gather shift
    double wy[RTK_MAX_MOMENTS];
};

#ifndef RTK_TILE_MINB
#define RTK_TILE_MINB 2
#endif
#ifndef RTK_TILE_TX3
#define RTK_TILE_TX3 16   // tile of lines on 3D lattices (2D slabs: 128 x 1)
#define RTK_TILE_TY3 16
#endif
template <int FS, int NM, int TX, int TY>
__global__ void __launch_bounds__(TX * TY, FS == RTK_FS_EXP_PARABOLIC
                                               ? 1
                                               : (TX * TY >= 256 ? RTK_TILE_MINB : 2 * RTK_TILE_MINB))
    lattice_mom_tile_kernel(LatArgs A, TileArgs T, int t, const double2* __restrict__ st_in,
                            double2* __restrict__ st_out, double* __restrict__ mom, int with_inflow, int fp,
                            const double2* __restrict__ plane_cur, const double2* __restrict__ plane_next,
                            const double2* __restrict__ plane_nn) {
    constexpr int NT = TX * TY;
    // Exp-parabolic (long characteristics): a third window (layer t + 2) for the downwind sample
    // one sub-segment beyond the crossing, whose table entry n_sub + 1 carries the weights of
    // planes b / c; plane_nn == nullptr on the line's last step (linear weights there).
    constexpr bool PAR = FS == RTK_FS_EXP_PARABOLIC;
    constexpr int NW = PAR ? 3 : 2;   // staged windows per direction
    const int hp = fp >> 1;
    const int g = blockIdx.y;                    // frequency pair
    const int tile = blockIdx.x;
    const int tyi = tile / T.ntx;
    const int ty0 = tyi * TY, tx0 = (tile - tyi * T.ntx) * TX;
    const int llx = static_cast<int>(threadIdx.x) % TX, lly = static_cast<int>(threadIdx.x) / TX;
    const int lx = tx0 + llx, ly = ty0 + lly;
    const bool line_ok = lx < A.nx && ly < A.ny;
    const int c = line_ok ? ly * A.nx + lx : 0;
    const int64_t plane2 = A.nxy * static_cast<int64_t>(hp);   // double2 per direction plane
    const int nsteps = A.nz - 1;
    const bool march = t < nsteps;
    const int z = blockIdx.z;
    const int n_mine = T.n_order > z ? (T.n_order - z + T.dgz - 1) / T.dgz : 0;

    extern __shared__ __align__(16) double2 tsm[];
    // [TileDir x n_mine][stage 0: window a, window b, sub table][stage 1: ...]
    TileDir* tdir = reinterpret_cast<TileDir*>(tsm);
    double2* stages = tsm + (n_mine * sizeof(TileDir) + 15) / 16;
    const int stage_d2 = NW * T.region_cap + T.sub_cap * kTileSubW;
    for (int e = threadIdx.x; e < n_mine; e += NT) {
        const int a = T.order[z + e * T.dgz];
        const LatDir& D = A.dirs[a];
        TileDir td;
        td.n_sub = D.n_sub;
        td.sc = D.sc;
        td.shift_off = D.shift_off;
        td.down = D.down;
        td.dtab = D.dtab_off + static_cast<long long>(t) * D.n_sub * A.nxy;
        td.hdr = march ? T.hdr[static_cast<int64_t>(a) * nsteps + t] : TileHdr{0, 0, 0, 0};
        td.gat = A.gat_shift[a * A.nz + t];
#pragma unroll
        for (int l = 0; l < RTK_MAX_MOMENTS; ++l) td.wy[l] = D.wy[l];
        tdir[e] = td;
    }
    __syncthreads();

    double phi[2], in_top[2], in_bot[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int f = 2 * g + q;
        const bool fv = f < A.n_freq;
        phi[q] = fv ? A.phi[f] : 0.0;
        in_top[q] = (with_inflow && fv && A.inflow_top) ? A.inflow_top[f] : 0.0;
        in_bot[q] = (with_inflow && fv && A.inflow_bottom) ? A.inflow_bottom[f] : 0.0;
    }

    // stage the window of this CTA's it-th direction into stage st (cp.async; caller commits):
    // a warp per window row, lanes along the row; the wrap is a conditional subtraction (a
    // window narrower than the lattice) or a modulo (tiny periodic lattices)
    auto stage = [&](int it, int st) {
        const int a = T.order[z + it * T.dgz];
        const TileDir& D = tdir[it];
        int gx0 = tx0 + D.hdr.fx;
        if (gx0 >= A.nx) gx0 -= A.nx;
        int gy0 = ty0 + D.hdr.fy;
        if (gy0 >= A.ny) gy0 -= A.ny;
        const double2* pa = plane_cur + a * plane2 + static_cast<int64_t>(g) * A.nxy;
        const double2* pb = plane_next + a * plane2 + static_cast<int64_t>(g) * A.nxy;
        const double2* pc = (PAR && plane_nn) ? plane_nn + a * plane2 + static_cast<int64_t>(g) * A.nxy : nullptr;
        double2* wa = stages + st * stage_d2;
        double2* wb = wa + T.region_cap;
        double2* wc = wb + T.region_cap;   // PAR only
        const int w = D.hdr.w, h = D.hdr.h;
        const bool small = w <= A.nx && h <= A.ny;
        const int cx = static_cast<int>(threadIdx.x) & 31;
        for (int ry = static_cast<int>(threadIdx.x) >> 5; ry < h; ry += NT / 32) {
            int gy = gy0 + ry;
            gy = small ? (gy >= A.ny ? gy - A.ny : gy) : gy % A.ny;
            const double2* ra = pa + gy * A.nx;
            const double2* rb = pb + gy * A.nx;
            for (int rx = cx; rx < w; rx += 32) {
                int gx = gx0 + rx;
                gx = small ? (gx >= A.nx ? gx - A.nx : gx) : gx % A.nx;
                cp_async16(wa + ry * w + rx, ra + gx);
                cp_async16(wb + ry * w + rx, rb + gx);
                if (PAR && pc) cp_async16(wc + ry * w + rx, pc + gy * A.nx + gx);
            }
        }
        // sub-node table of (direction, step): n_sub + 2 entries (the last one is the exp-parabolic
        // downwind sample), stored after the direction's preceding (n_sub + 2)-entry steps
        const int n_sub2 = D.n_sub + 2;
        const double2* src = reinterpret_cast<const double2*>(
            T.sub + D.shift_off + static_cast<int64_t>(a) * nsteps + static_cast<int64_t>(t) * n_sub2);
        double2* dst = wa + NW * T.region_cap;
        const int n_copy = PAR ? n_sub2 : n_sub2 - 1;
        for (int e = threadIdx.x; e < kTileSubW * n_copy; e += NT) cp_async16(dst + e, src + e);
    };

    // global operands of a direction, loaded one direction ahead into registers: the T_RC
    // gather corners of node c, the line's own state (or the SC restart corners) and its first dt
    struct Pre {
        double2 g00, g10, g01, g11;   // gather corners (t > 0)
        double2 s00;                  // own state (LC; SC restarts are gathered in place)
        double dt0;                   // first sub-segment's dt
    };
    auto prefetch = [&](int it, Pre& P) {
        if (!line_ok || t == 0) return;
        const int a = T.order[z + it * T.dgz];
        const TileDir& D = tdir[it];
        const double2* lin = st_in + a * plane2 + static_cast<int64_t>(g) * A.nxy;
        const Stencil sg = stencil_at(lx, ly, D.gat, A.nx, A.ny);
        P.g00 = lin[sg.c00];
        P.g10 = lin[sg.c10];
        P.g01 = lin[sg.c01];
        P.g11 = lin[sg.c11];
        if (!march) return;
        if (!D.sc) P.s00 = lin[c];
        const double* dtl = A.dtab + D.dtab + c;
        P.dt0 = __ldg(dtl);
        // the direction's remaining sub-segment paths into L1 (the march reads one per sub-node;
        // loaded only one sub-node ahead they were the kernel's largest stall: 24% of samples)
        for (int m = 1; m < D.n_sub; ++m)
            asm volatile("prefetch.global.L1 [%0];\n" ::"l"(dtl + static_cast<int64_t>(m) * A.nxy));
    };

    if (march && n_mine > 0) stage(0, 0);
    asm volatile("cp.async.commit_group;\n" ::);
    Pre cur;
    if (n_mine > 0) prefetch(0, cur);

    double mo[NM][2];
#pragma unroll
    for (int l = 0; l < NM; ++l) mo[l][0] = mo[l][1] = 0.0;
    int hemi = 0;   // hemisphere of the accumulated moments (0: down, layer t; 1: up, layer nz-1-t)

    auto flush = [&](int hm) {
        const int k = hm == 0 ? t : A.nz - 1 - t;
        if (line_ok) {
            if (T.dgz > 1) {
                double* o = T.scratch + ((static_cast<int64_t>(z) * 2 + hm) * A.nxy + c) * NM * fp + 2 * g;
#pragma unroll
                for (int l = 0; l < NM; ++l)
                    *reinterpret_cast<double2*>(o + static_cast<int64_t>(l) * fp) = make_double2(mo[l][0], mo[l][1]);
            } else {
                // step t is the first visit of layers t and nz-1-t iff t < nz-1-t; the middle layer
                // (odd nz) gets both parts from this thread, up added to down
                const bool first = (hm == 0) ? (t <= A.nz - 1 - t) : (t < A.nz - 1 - t);
                double* o = mom + (static_cast<int64_t>(k) * A.nxy + c) * NM * fp + 2 * g;
#pragma unroll
                for (int l = 0; l < NM; ++l) {
                    double2* op = reinterpret_cast<double2*>(o + static_cast<int64_t>(l) * fp);
                    double2 v = make_double2(mo[l][0], mo[l][1]);
                    if (!first) {
                        const double2 old = *op;
                        v.x += old.x;
                        v.y += old.y;
                    }
                    if (2 * g + 1 >= A.n_freq) v.y = 0.0;   // pad column of an odd N_nu stays zero
                    *op = v;
                }
            }
        }
#pragma unroll
        for (int l = 0; l < NM; ++l) mo[l][0] = mo[l][1] = 0.0;
    };

    for (int it = 0; it < n_mine; ++it) {
        const int i = z + it * T.dgz;
        const int a = T.order[i];
        const int hm = i < T.n_down ? 0 : 1;
        if (hm != hemi) {
            flush(hemi);
            hemi = hm;
        }
        // prefetch the next direction's window into the next stage, then wait for this one.  With
        // three stages the refilled stage was last read two iterations ago, and every thread has
        // passed the barrier below since, so one barrier per direction suffices; with two stages
        // (windows too large for three) a second barrier ends the iteration.
        const int st = it % T.n_stages;
        if (march && it + 1 < n_mine) stage(it + 1, (it + 1) % T.n_stages);
        asm volatile("cp.async.commit_group;\n" ::);
        Pre nxt;
        if (it + 1 < n_mine) prefetch(it + 1, nxt);   // global loads in flight across this direction
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();

        const TileDir& D = tdir[it];
        if (line_ok) {
            double v0, v1;
            if (t == 0) {
                v0 = hm == 0 ? in_top[0] : in_bot[0];
                v1 = hm == 0 ? in_top[1] : in_bot[1];
            } else {
                // T_RC weights (the corner values were loaded one direction ahead by prefetch)
                const double gax = D.gat.ax, gay = D.gat.ay;
                const double w00 = (1 - gax) * (1 - gay), w10 = gax * (1 - gay), w01 = (1 - gax) * gay, w11 = gax * gay;
                v0 = w00 * cur.g00.x + w10 * cur.g10.x + w01 * cur.g01.x + w11 * cur.g11.x;
                v1 = w00 * cur.g00.y + w10 * cur.g10.y + w01 * cur.g01.y + w11 * cur.g11.y;
            }
#pragma unroll
            for (int l = 0; l < NM; ++l) {
                mo[l][0] = fma(D.wy[l], v0, mo[l][0]);
                mo[l][1] = fma(D.wy[l], v1, mo[l][1]);
            }
            if (march) {
                double acc0, acc1;
                if (t == 0) {
                    acc0 = hm == 0 ? in_top[0] : in_bot[0];
                    acc1 = hm == 0 ? in_top[1] : in_bot[1];
                } else if (D.sc) {
                    // short characteristics: restart at the upwind point of node c
                    const double2* lin = st_in + a * plane2 + static_cast<int64_t>(g) * A.nxy;
                    const Stencil rs = stencil_at(lx, ly, restart_shift(A.dirs[a]), A.nx, A.ny);
                    const double2 r00 = lin[rs.c00], r10 = lin[rs.c10], r01 = lin[rs.c01], r11 = lin[rs.c11];
                    acc0 = rs.w00 * r00.x + rs.w10 * r10.x + rs.w01 * r01.x + rs.w11 * r11.x;
                    acc1 = rs.w00 * r00.y + rs.w10 * r10.y + rs.w01 * r01.y + rs.w11 * r11.y;
                } else {
                    acc0 = cur.s00.x;
                    acc1 = cur.s00.y;
                }
                const int w = D.hdr.w;
                const double2* wa = stages + st * stage_d2;
                const double2* wb = wa + T.region_cap;
                const TileSub* sb = reinterpret_cast<const TileSub*>(wa + NW * T.region_cap);
                const double* dtl = A.dtab + D.dtab + c;
                const int n_sub = D.n_sub;
                double ps0 = 0.0, ps1 = 0.0;
                double dt_next = t == 0 ? __ldg(dtl) : cur.dt0;
                if (PAR) {
                    // Kunasz-Auer along the line (advance_lineF_par / oracle/lattice.py): point m is
                    // updated from the samples at m - 1, m and the downwind m + 1; the downwind of
                    // the step's last point lies one sub-segment beyond the crossing (windows b / c,
                    // table entry n_sub + 1; its dt is the line's first entry of step t + 1, which
                    // follows this step's last), or the linear weights apply on the last step.
                    const double2* wc = wb + T.region_cap;
                    auto samp = [&](int m, const double2* pa_, const double2* pb_, double& o0, double& o1) {
                        const TileSub S = sb[m];
                        const int o = (lly + S.dy) * w + llx + S.dx;
                        const double2 a00 = pa_[o], a10 = pa_[o + 1], a01 = pa_[o + w], a11 = pa_[o + w + 1];
                        const double2 b00 = pb_[o], b10 = pb_[o + 1], b01 = pb_[o + w], b11 = pb_[o + w + 1];
                        o0 = (S.a00 * a00.x + S.a10 * a10.x + S.a01 * a01.x + S.a11 * a11.x) +
                             (S.b00 * b00.x + S.b10 * b10.x + S.b01 * b01.x + S.b11 * b11.x);
                        o1 = (S.a00 * a00.y + S.a10 * a10.y + S.a01 * a01.y + S.a11 * a11.y) +
                             (S.b00 * b00.y + S.b10 * b10.y + S.b01 * b01.y + S.b11 * b11.y);
                    };
                    const bool has_c = plane_nn != nullptr;
                    double sp0, sp1, sc0, sc1, sn0 = 0.0, sn1 = 0.0;
                    samp(0, wa, wb, sp0, sp1);
                    samp(1, wa, wb, sc0, sc1);
                    double dtu = dt_next;
                    for (int m = 1; m <= n_sub; ++m) {
                        const bool down = m < n_sub || has_c;
                        double dtd = 0.0;
                        if (m < n_sub) {
                            samp(m + 1, wa, wb, sn0, sn1);
                            dtd = __ldg(dtl + static_cast<int64_t>(m) * A.nxy);
                        } else if (has_c) {
                            samp(n_sub + 1, wb, wc, sn0, sn1);
                            dtd = __ldg(dtl + static_cast<int64_t>(n_sub) * A.nxy);
                        }
                        if (down) {
                            const ExpPar w0 = exp_parabolic_weights_bf(phi[0] * dtu, phi[0] * dtd);
                            const ExpPar w1 = exp_parabolic_weights_bf(phi[1] * dtu, phi[1] * dtd);
                            acc0 = fma(acc0, w0.att, w0.wu * sp0 + w0.wc * sc0 + w0.wd * sn0);
                            acc1 = fma(acc1, w1.att, w1.wu * sp1 + w1.wc * sc1 + w1.wd * sn1);
                        } else {
                            const ExpLin w0 = exp_linear_weights_bf(phi[0] * dtu), w1 = exp_linear_weights_bf(phi[1] * dtu);
                            acc0 = fma(acc0, w0.att, w0.wu * sp0 + w0.wc * sc0);
                            acc1 = fma(acc1, w1.att, w1.wu * sp1 + w1.wc * sc1);
                        }
                        sp0 = sc0;
                        sp1 = sc1;
                        sc0 = sn0;
                        sc1 = sn1;
                        dtu = dtd;
                    }
                } else
                for (int m = (FS == RTK_FS_IE ? 1 : 0); m <= n_sub; ++m) {
                    const TileSub S = sb[m];
                    const int o = (lly + S.dy) * w + llx + S.dx;
                    const double2 a00 = wa[o], a10 = wa[o + 1], a01 = wa[o + w], a11 = wa[o + w + 1];
                    const double2 b00 = wb[o], b10 = wb[o + 1], b01 = wb[o + w], b11 = wb[o + w + 1];
                    const double s0 = (S.a00 * a00.x + S.a10 * a10.x + S.a01 * a01.x + S.a11 * a11.x) +
                                      (S.b00 * b00.x + S.b10 * b10.x + S.b01 * b01.x + S.b11 * b11.x);
                    const double s1 = (S.a00 * a00.y + S.a10 * a10.y + S.a01 * a01.y + S.a11 * a11.y) +
                                      (S.b00 * b00.y + S.b10 * b10.y + S.b01 * b01.y + S.b11 * b11.y);
                    if (m > 0) {
                        const double dt = dt_next;
                        if (m < n_sub) dt_next = __ldg(dtl + static_cast<int64_t>(m) * A.nxy);   // one ahead
                        const double d0 = phi[0] * dt, d1 = phi[1] * dt;
                        if (FS == RTK_FS_IE) {
                            const double r0 = rcp_nr(1.0 + d0), r1 = rcp_nr(1.0 + d1);
                            acc0 = fma(acc0, r0, (d0 * s0) * r0);
                            acc1 = fma(acc1, r1, (d1 * s1) * r1);
                        } else {
                            const ExpLin w0 = exp_linear_weights(d0), w1 = exp_linear_weights(d1);
                            acc0 = fma(acc0, w0.att, w0.wu * ps0 + w0.wc * s0);
                            acc1 = fma(acc1, w1.att, w1.wu * ps1 + w1.wc * s1);
                        }
                    }
                    ps0 = s0;
                    ps1 = s1;
                }
                st_out[a * plane2 + static_cast<int64_t>(g) * A.nxy + c] = make_double2(acc0, acc1);
            }
        }
        cur = nxt;
        if (T.n_stages == 2) __syncthreads();   // stage st is refilled by the next iteration's prefetch
    }
    flush(hemi);
    if (hemi == 0) flush(1);   // no up direction in this CTA: its (zero) part is still written
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// DGZ > 1: mom of the step's two layers = sum over the direction groups in group order
template <int NM>
__global__ void lattice_mom_reduce_kernel(const double* __restrict__ scratch, double* __restrict__ mom, int t, int nz,
                                          int64_t nxy, int fp, int dgz, int n_freq) {
    const int64_t per = nxy * NM * fp;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= per) return;
    const int f = static_cast<int>(e % fp);
    for (int hm = 0; hm < 2; ++hm) {
        const int k = hm == 0 ? t : nz - 1 - t;
        const bool first = (hm == 0) ? (t <= nz - 1 - t) : (t < nz - 1 - t);
        double sum = 0.0;
        for (int zz = 0; zz < dgz; ++zz) sum += scratch[(static_cast<int64_t>(zz) * 2 + hm) * per + e];
        if (f >= n_freq) sum = 0.0;
        double* o = mom + static_cast<int64_t>(k) * per + e;
        *o = first ? sum : *o + sum;
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Window and sub-node tables of the tiled moment kernel, per (direction, layer step): the
// same offsets and floor/fraction arithmetic as the Shift tables (shift_of), kept unwrapped
// so a tile's samples index one window.
static int setup_tile_tables(Problem& p, const rtk_lattice_desc* d, const std::vector<LatDir>& dirs) {
    p.lat_tile_tx = d->ny > 1 ? RTK_TILE_TX3 : 128;
    p.lat_tile_ty = d->ny > 1 ? RTK_TILE_TY3 : 1;
    const int nsteps = d->nz - 1;
    std::vector<TileHdr> hdr(static_cast<size_t>(d->n_dirs) * std::max(1, nsteps));
    size_t n_sub_total = 0;
    // n_sub + 2 entries per (direction, step): sub-nodes 0..n_sub, then the exp-parabolic downwind
    // sample; direction a's block starts at shift_off + a nsteps (one extra entry per earlier step)
    for (int a = 0; a < d->n_dirs; ++a)
        n_sub_total = std::max<size_t>(n_sub_total, dirs[a].shift_off + static_cast<size_t>(a) * nsteps +
                                                        static_cast<size_t>(nsteps) * (dirs[a].n_sub + 2));
    std::vector<TileSub> sub(std::max<size_t>(1, n_sub_total));
    const bool par = d->formal_solver == RTK_FS_EXP_PARABOLIC;
    p.lat_region_cap = 0;
    p.lat_sub_cap = 0;
    p.h_lat_down.assign(d->n_dirs, 0);
    for (int a = 0; a < d->n_dirs; ++a) {
        const LatDir& D = dirs[a];
        p.h_lat_down[a] = D.down;
        p.lat_sub_cap = std::max(p.lat_sub_cap, D.n_sub + 2);
        for (int t = 0; t < nsteps; ++t) {
            int fxmin = 0, fxmax = 0, fymin = 0, fymax = 0;
            // entry n_sub + 1: the downwind point of the step's last sub-node (exp-parabolic, LC:
            // the line at t + 1 + 1 / n_sub, as the Shift table's down_shift); it widens the
            // window only for exp-parabolic problems
            const int n_ent = D.n_sub + 2;
            std::vector<double> fxs(n_ent), fys(n_ent), oxs(n_ent), oys(n_ent);
            for (int m = 0; m < n_ent; ++m) {
                if (m == D.n_sub + 1 && !par) break;
                const double tt = m == D.n_sub + 1
                                      ? (D.sc ? 1.0 / D.n_sub : t + 1.0 + 1.0 / D.n_sub)
                                      : (D.sc ? static_cast<double>(m) / D.n_sub - 1.0 : t + static_cast<double>(m) / D.n_sub);
                oxs[m] = tt * D.sx;
                oys[m] = tt * D.sy;
                fxs[m] = std::floor(oxs[m]);
                fys[m] = std::floor(oys[m]);
                const int fx = static_cast<int>(fxs[m]), fy = static_cast<int>(fys[m]);
                if (m == 0 || fx < fxmin) fxmin = fx;
                if (m == 0 || fx > fxmax) fxmax = fx;
                if (m == 0 || fy < fymin) fymin = fy;
                if (m == 0 || fy > fymax) fymax = fy;
            }
            TileHdr& H = hdr[static_cast<size_t>(a) * nsteps + t];
            H.fx = ((fxmin % d->nx) + d->nx) % d->nx;
            H.fy = ((fymin % d->ny) + d->ny) % d->ny;
            H.w = p.lat_tile_tx + (fxmax - fxmin) + 1;
            H.h = p.lat_tile_ty + (fymax - fymin) + 1;
            p.lat_region_cap = std::max(p.lat_region_cap, H.w * H.h);
            for (int m = 0; m < n_ent; ++m) {
                TileSub& S = sub[D.shift_off + static_cast<size_t>(a) * nsteps + static_cast<size_t>(t) * n_ent + m];
                if (m == D.n_sub + 1 && !par) {
                    S = TileSub{};
                    break;
                }
                S.dx = static_cast<int>(fxs[m]) - fxmin;
                S.dy = static_cast<int>(fys[m]) - fymin;
                S.pad = 0.0;
                const double ax = oxs[m] - fxs[m], ay = oys[m] - fys[m];
                const double w00 = (1 - ax) * (1 - ay), w10 = ax * (1 - ay), w01 = (1 - ax) * ay, w11 = ax * ay;
                // the downwind sample interpolates between layers t + 1 and t + 2 at wz = 1 / n_sub
                const double wz = m == D.n_sub + 1 ? 1.0 / D.n_sub : m * (1.0 / D.n_sub);
                S.a00 = (1 - wz) * w00;
                S.a10 = (1 - wz) * w10;
                S.a01 = (1 - wz) * w01;
                S.a11 = (1 - wz) * w11;
                S.b00 = wz * w00;
                S.b10 = wz * w10;
                S.b01 = wz * w01;
                S.b11 = wz * w11;
            }
        }
    }
    RTK_CUDA_TRY(cudaMalloc(&p.lat_tile_hdr, sizeof(TileHdr) * hdr.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.lat_tile_hdr, hdr.data(), sizeof(TileHdr) * hdr.size(), cudaMemcpyHostToDevice));
    RTK_CUDA_TRY(cudaMalloc(&p.lat_tile_sub, sizeof(TileSub) * sub.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.lat_tile_sub, sub.data(), sizeof(TileSub) * sub.size(), cudaMemcpyHostToDevice));
    RTK_CUDA_TRY(cudaMalloc(&p.lat_order, sizeof(int) * d->n_dirs));
    p.lat_region_cap = (p.lat_region_cap + 1) / 2 * 2;   // keep the stages 32-byte aligned

    return RTK_OK;
}

// ---------------------------------------------------------------------------
int setup_lattice(Problem& p, const rtk_lattice_desc* d) {
    std::vector<LatDir> dirs(d->n_dirs);
    for (int a = 0; a < d->n_dirs; ++a) {
        const double ox = d->omega[3 * a], oy = d->omega[3 * a + 1], oz = d->omega[3 * a + 2];
        LatDir& D = dirs[a];
        D.down = oz < 0 ? 1 : 0;
        D.sx = ox * d->dz / (std::fabs(oz) * d->dx);
        D.sy = d->ny > 1 ? oy * d->dz / (std::fabs(oz) * d->dy) : 0.0;
        D.n_sub = std::max(1, static_cast<int>(std::ceil(std::max(std::fabs(D.sx), std::fabs(D.sy)) - 1e-12)));
        D.sub_len = d->dz / std::fabs(oz) / D.n_sub;
        D.sc = d->characteristics == RTK_CHAR_SHORT || (d->characteristics == RTK_CHAR_HYBRID && D.n_sub == 1);
        const Shift rs = shift_of(-D.sx, -D.sy, d->nx, d->ny);
        D.rbx = rs.bx;
        D.rby = rs.by;
        D.rax = rs.ax;
        D.ray = rs.ay;
        for (int l = 0; l < 8; ++l) {
            const bool in = l < d->n_moments;
            D.wy[l] = in ? d->dir_w[a] * d->ybasis[l * d->n_dirs + a] : 0.0;
            D.cy[l] = in ? d->coeffs[l] * d->ybasis[l * d->n_dirs + a] : 0.0;
        }
    }
    // warp-uniform interpolation shifts, tabulated once (same arithmetic as the device's shift_of)
    std::vector<Shift> sub, gat(static_cast<size_t>(d->n_dirs) * d->nz), dsh(gat.size());
    p.lat_total_sub = 0;
    for (int a = 0; a < d->n_dirs; ++a) {
        LatDir& D = dirs[a];
        D.sub_pref = p.lat_total_sub;
        p.lat_total_sub += D.n_sub + 1;
    }
    for (int a = 0; a < d->n_dirs; ++a) {
        LatDir& D = dirs[a];
        D.shift_off = static_cast<int>(sub.size());
        // LC: line c sits at c + (t + m / n_sub) s; SC: the characteristic ending on node c
        // starts at c - s, sub-node m at c + (m / n_sub - 1) s, and node values are the line
        // values (identity gather)
        for (int t = 0; t < d->nz - 1; ++t)
            for (int m = 0; m <= D.n_sub; ++m) {
                const double tt = D.sc ? static_cast<double>(m) / D.n_sub - 1.0 : t + static_cast<double>(m) / D.n_sub;
                sub.push_back(shift_of(tt * D.sx, tt * D.sy, d->nx, d->ny));
            }
        for (int t = 0; t < d->nz; ++t) {
            gat[static_cast<size_t>(a) * d->nz + t] = D.sc ? shift_of(0.0, 0.0, d->nx, d->ny)
                                                           : shift_of(-t * D.sx, -t * D.sy, d->nx, d->ny);
            // exp-parabolic: one sub-segment beyond the step's last point (LC: the line at
            // t + 1 + 1/n_sub; SC: the node + s / n_sub)
            const double td = D.sc ? 1.0 / D.n_sub : t + 1.0 + 1.0 / D.n_sub;
            dsh[static_cast<size_t>(a) * d->nz + t] = shift_of(td * D.sx, td * D.sy, d->nx, d->ny);
        }
    }
    if (sub.empty()) sub.push_back(Shift{});
    RTK_CUDA_TRY(cudaMalloc(&p.lat_sub_shift, sizeof(Shift) * sub.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.lat_sub_shift, sub.data(), sizeof(Shift) * sub.size(), cudaMemcpyHostToDevice));
    RTK_CUDA_TRY(cudaMalloc(&p.lat_gat_shift, sizeof(Shift) * gat.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.lat_gat_shift, gat.data(), sizeof(Shift) * gat.size(), cudaMemcpyHostToDevice));
    RTK_CUDA_TRY(cudaMalloc(&p.lat_down_shift, sizeof(Shift) * dsh.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.lat_down_shift, dsh.data(), sizeof(Shift) * dsh.size(), cudaMemcpyHostToDevice));
    int64_t dtab_count = 0;
    const int64_t nxy = static_cast<int64_t>(d->nx) * d->ny;
    for (auto& D : dirs) {
        D.dtab_off = dtab_count;
        dtab_count += static_cast<int64_t>(D.n_sub) * (d->nz - 1) * nxy;
    }
    RTK_CUDA_TRY(cudaMalloc(&p.lat_dirs, sizeof(LatDir) * dirs.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.lat_dirs, dirs.data(), sizeof(LatDir) * dirs.size(), cudaMemcpyHostToDevice));
    p.lat_max_sub = 0;
    p.lat_any_sc = false;
    for (const auto& D : dirs) {
        p.lat_max_sub = std::max(p.lat_max_sub, D.n_sub);
        p.lat_any_sc = p.lat_any_sc || D.sc;
    }
    const bool small_layers = sizeof(double) * nxy * (10 * kFC + 3) <= 160 * 1024;
    if (d->layout == RTK_LAYOUT_MOMENTS || small_layers) {
        // frequency-independent sub-segment optical paths, streamed by the moment-layout sweep and
        // by the shared-memory intensity kernel (optional there: without it the opacity is sampled)
        cudaError_t e = cudaMalloc(&p.lat_dtab, sizeof(double) * std::max<int64_t>(1, dtab_count));
        if (e != cudaSuccess && d->layout != RTK_LAYOUT_MOMENTS) {
            cudaGetLastError();
            p.lat_dtab = nullptr;
            return RTK_OK;
        }
        if (e != cudaSuccess) return cuda_status(e, "lattice dt table");
        dim3 grid(static_cast<unsigned>((nxy * (d->nz - 1) + 255) / 256), d->n_dirs);
        lattice_dtab_kernel<<<grid, 256>>>(p.lat_dirs, reinterpret_cast<const Shift*>(p.lat_sub_shift), p.lat_chi,
                                           p.lat_dtab, d->n_dirs, d->nx, d->ny, d->nz);
        RTK_LAUNCH_CHECK("lattice_dtab_kernel");
        RTK_CUDA_TRY(cudaDeviceSynchronize());
    }
    if (d->layout == RTK_LAYOUT_MOMENTS) {
        if (int rc = setup_tile_tables(p, d, dirs)) return rc;
    }
    return RTK_OK;
}

static LatArgs lat_args(const Problem& p, const double* src, const double* x, double* y) {
    LatArgs A;
    A.dirs = p.lat_dirs;
    A.sub_shift = reinterpret_cast<const Shift*>(p.lat_sub_shift);
    A.gat_shift = reinterpret_cast<const Shift*>(p.lat_gat_shift);
    A.down_shift = reinterpret_cast<const Shift*>(p.lat_down_shift);
    A.dtab = p.lat_dtab;
    A.total_sub = p.lat_total_sub;
    A.chi = p.lat_chi;
    A.phi = p.phi;
    A.src = src;
    A.gamma = p.gamma;
    A.x = x;
    A.y = y;
    A.inflow_top = p.lat_in_top;
    A.inflow_bottom = p.lat_in_bot;
    A.nx = p.lat_nx;
    A.ny = p.lat_ny;
    A.nz = p.lat_nz;
    A.n_dirs = p.n_angles;
    A.n_freq = p.n_freq;
    A.n_mom = p.n_mom;
    A.nxy = static_cast<int64_t>(p.lat_nx) * p.lat_ny;
    A.a0 = 0;
    A.a1 = p.n_angles;
    return A;
}

template <int FS, int SRC, int OUT>
static int launch_int(const Problem& p, const LatArgs& A, int with_inflow, cudaStream_t s) {
    constexpr int ring = FS == RTK_FS_EXP_PARABOLIC ? 4 : 3;
    // [2] line buffers, source ring, opacity ring, [2] x planes, SC seeds, [2] sub-node tables
    const size_t smem_planes = sizeof(double) * (A.nxy * (2 * kFC + ring * kFC + ring + 2 * kFC + kFC) + 1) +
                               2 * (sizeof(Shift) + sizeof(SubW)) * (p.lat_max_sub + 1);
    if (FS == RTK_FS_EXP_PARABOLIC && (smem_planes > 160 * 1024 || p.tune.lat_no_smem))
        return set_error(RTK_ERESOURCE, "exp-parabolic in the intensity layout needs the shared-memory kernel "
                                        "(small layers); use the moment layout");
    if (smem_planes <= 160 * 1024 && !p.tune.lat_no_smem) {
        // the parabolic march samples the opacity planes (its downwind segment is not in the table)
        const bool dt = A.dtab != nullptr && !p.tune.lat_no_dtab && FS != RTK_FS_EXP_PARABOLIC;
        const bool planar = A.ny == 1 && !p.tune.lat_no_planar;
        auto kern = dt ? (planar ? lattice_int_smem_kernel<FS, SRC, OUT, true, true>
                                 : lattice_int_smem_kernel<FS, SRC, OUT, true, false>)
                       : (planar ? lattice_int_smem_kernel<FS, SRC, OUT, false, true>
                                 : lattice_int_smem_kernel<FS, SRC, OUT, false, false>);
        if (int rc = ensure_smem_for(kern, smem_planes)) return rc;
        // sector-aligned frequency chunks (see the kernel) when every (node, direction) row
        // has the same offset within a 32-byte sector
        const bool aligned_rows = (static_cast<int64_t>(A.n_dirs) * A.n_freq) % kFC == 0 && A.n_freq % kFC != 0 &&
                                  (SRC != LSRC_VEC || reinterpret_cast<uintptr_t>(A.src) % 32 == 0) &&
                                  (A.y == nullptr || reinterpret_cast<uintptr_t>(A.y) % 32 == 0) &&
                                  (A.x == nullptr || reinterpret_cast<uintptr_t>(A.x) % 32 == 0);
        const int slack = aligned_rows ? kFC - 1 : 0;
        const int nfc = (A.n_freq + slack + kFC - 1) / kFC;
        // whole frequency pairs move as 16-byte words when they are 16-byte aligned in src, x
        // and y: always with sector-aligned chunks, else with an even N_nu and aligned bases
        const bool ptr16 = (SRC != LSRC_VEC || reinterpret_cast<uintptr_t>(A.src) % 16 == 0) &&
                           (A.y == nullptr || reinterpret_cast<uintptr_t>(A.y) % 16 == 0) &&
                           (A.x == nullptr || reinterpret_cast<uintptr_t>(A.x) % 16 == 0);
        const int vec16 = (aligned_rows || (A.n_freq % 2 == 0 && ptr16)) ? 1 : 0;
        kern<<<A.n_dirs * nfc, kIntThreads, smem_planes, s>>>(A, with_inflow, p.lat_max_sub, slack, vec16);
        RTK_LAUNCH_CHECK("lattice_int_smem_kernel");
        return RTK_OK;
    }
    if (p.lat_any_sc)
        return set_error(RTK_ERESOURCE, "short characteristics in the intensity layout need the shared-memory kernel "
                                        "(small layers); use the moment layout");
    const size_t smem = sizeof(double) * A.nxy * kFC;
    auto kern = lattice_int_kernel<FS, SRC, OUT>;
    if (int rc = ensure_smem_for(kern, smem)) return rc;
    const int nfc = (A.n_freq + kFC - 1) / kFC;
    kern<<<A.n_dirs * nfc, kIntThreads, smem, s>>>(A, with_inflow);
    RTK_LAUNCH_CHECK("lattice_int_kernel");
    return RTK_OK;
}

// intensity layout transfer: y = x - Lambda S (OUT_X_MINUS) or y = Lambda S (+ inflow)
int lattice_transfer_intensity(const Problem& p, int src_mode, int out_mode, bool with_inflow, const double* src,
                               const double* x, double* y, cudaStream_t s) {
    LatArgs A = lat_args(p, src, x, y);
    const int wi = with_inflow ? 1 : 0;
    if (static_cast<size_t>(A.nxy) * kFC * sizeof(double) > 200 * 1024)
        return set_error(RTK_ERESOURCE, "intensity-layout lattice limited to 6400 horizontal nodes; use the moment layout");
#define RTK_LAT_INT(FS)                                                                                   \
    do {                                                                                                  \
        if (src_mode == LSRC_VEC && out_mode == OUT_X_MINUS) return launch_int<FS, LSRC_VEC, OUT_X_MINUS>(p, A, wi, s); \
        if (src_mode == LSRC_VEC && out_mode == OUT_ACC) return launch_int<FS, LSRC_VEC, OUT_ACC>(p, A, wi, s);         \
        if (src_mode == LSRC_ISO && out_mode == OUT_ACC) return launch_int<FS, LSRC_ISO, OUT_ACC>(p, A, wi, s);         \
    } while (0)
    if (p.fs == RTK_FS_IE) RTK_LAT_INT(RTK_FS_IE);
    else if (p.fs == RTK_FS_EXP_PARABOLIC) RTK_LAT_INT(RTK_FS_EXP_PARABOLIC);
    else RTK_LAT_INT(RTK_FS_EXP_LINEAR);
#undef RTK_LAT_INT
    return set_error(RTK_EINVAL, "lattice: unsupported source/output mode");
}

template <int FS, int SRC, int NM, int DG>
static int launch_mom_steps_dg(const Problem& p, const LatArgs& A, bool with_inflow, double* mom, cudaStream_t s) {
    const unsigned pblocks = static_cast<unsigned>((A.nxy * p.fp + 255) / 256);
    constexpr int F = 2;   // F = 4 measured slower (176 registers, 1 block/SM; cfg5 854 vs 487 ms)
    // DG = 1: 128-thread blocks spread the nxy * fp / F items of a step evenly over the SMs;
    // DG > 1: 32 items x DG direction groups per block
    const int mb = DG == 1 ? 128 : 32 * DG;
    const int ipb = mb / DG;
    const size_t mom_smem = sizeof(double) * NM * F * mb + sizeof(StepDir) * A.n_dirs +
                            sizeof(Shift) * (2 * A.n_dirs + A.total_sub);
    auto kern = lattice_mom_group_kernel<FS, NM, F, DG>;
    if (int rc = ensure_smem_for(kern, mom_smem)) return rc;
    const unsigned sblocks = static_cast<unsigned>((A.nxy * ((p.fp + F - 1) / F) + ipb - 1) / ipb);
    double* a = p.lat_state[0];
    double* b = p.lat_state[1];
    constexpr bool PAR = FS == RTK_FS_EXP_PARABOLIC;
    constexpr int ring = PAR ? 3 : 2;   // source planes: current, next (and after next)
    for (int t = 0; t < A.nz; ++t) {
        double* cur = p.lat_splane[t % ring];
        double* nxt = p.lat_splane[(t + 1) % ring];
        double* nn = PAR ? p.lat_splane[(t + 2) % ring] : nullptr;
        if (t < A.nz - 1) {
            // step 0 fills every plane of the ring; later steps only the newest one
            const int mask = PAR ? (t == 0 ? 7 : 4) : (t == 0 ? 3 : 2);
            lattice_splane_kernel<SRC, NM><<<pblocks, 256, 0, s>>>(A, t, cur, nxt, nn, mask, p.fp);
            RTK_LAUNCH_CHECK("lattice_splane_kernel");
        }
        kern<<<sblocks, mb, mom_smem, s>>>(A, t, a, b, mom, with_inflow ? 1 : 0, p.fp, cur, nxt,
                                           PAR && t + 2 < A.nz ? nn : nullptr);
        RTK_LAUNCH_CHECK("lattice_mom_group_kernel");
        double* tmp = a;
        a = b;
        b = tmp;
    }
    return RTK_OK;
}

// Tiled path (IE / exp-linear): per layer step the pair-major source planes, the tiled
// moment kernel over (tiles x frequency pairs x direction groups) and, with several
// direction groups, the ordered reduction of their partial moments.  -1: not applicable.
template <int FS, int SRC, int NM, int TX, int TY>
static int launch_mom_tiles_t(const Problem& p, const LatArgs& A, bool with_inflow, double* mom, cudaStream_t s) {
    const int hp = p.fp / 2;
    const int ntx = (A.nx + TX - 1) / TX, nty = (A.ny + TY - 1) / TY;
    const int ntiles = ntx * nty;
    // direction order of this call's range: down directions, then up
    if (p.lat_order_a0 != A.a0 || p.lat_order_a1 != A.a1) {
        p.h_lat_order.clear();
        for (int pass = 0; pass < 2; ++pass)
            for (int a = A.a0; a < A.a1; ++a)
                if ((p.h_lat_down[a] != 0) == (pass == 0)) p.h_lat_order.push_back(a);
        int nd = 0;
        for (int a = A.a0; a < A.a1; ++a) nd += p.h_lat_down[a] ? 1 : 0;
        p.lat_order_down = nd;
        if (!p.h_lat_order.empty())
            RTK_CUDA_TRY(cudaMemcpyAsync(p.lat_order, p.h_lat_order.data(), sizeof(int) * p.h_lat_order.size(),
                                         cudaMemcpyHostToDevice, s));
        p.lat_order_a0 = A.a0;
        p.lat_order_a1 = A.a1;
    }
    const int n_order = static_cast<int>(p.h_lat_order.size());
    // direction groups: enough CTAs for ~6 per SM (148 SMs), at most 8 and one per direction
    // (16 groups measured no faster on cfg3's 2 tiles x 21 pairs: 22.7 vs 22.2 ms -- a layer step
    // there is bound by the per-direction latency chain, not by occupancy)
    int dgz = p.tune.lat_dgz;
    if (dgz <= 0) {
        const int64_t ctas = static_cast<int64_t>(ntiles) * hp;
        dgz = static_cast<int>(std::min<int64_t>(8, std::max<int64_t>(1, (148 * 6 + ctas - 1) / ctas)));
    }
    dgz = std::max(1, std::min(dgz, std::max(1, n_order)));
    constexpr bool PAR = FS == RTK_FS_EXP_PARABOLIC;
    const size_t stage_d2 = (PAR ? 3 : 2) * static_cast<size_t>(p.lat_region_cap) +
                            kTileSubW * static_cast<size_t>(p.lat_sub_cap);
    const int per_cta = (n_order + dgz - 1) / dgz;
    const size_t dir_bytes = (per_cta * sizeof(TileDir) + 15) / 16 * 16;
    // IE / exp-linear: two CTAs per SM (110 KB each); exp-parabolic: one CTA per SM (its register
    // count allows no more), so its three windows may take up to 200 KB
    const size_t smem_cap = (PAR ? 200 : 110) * 1024;
    int n_stages = 3;
    size_t smem = n_stages * stage_d2 * sizeof(double2) + dir_bytes;
    if (smem > smem_cap) {
        n_stages = 2;
        smem = n_stages * stage_d2 * sizeof(double2) + dir_bytes;
    }
    if (smem > smem_cap) return -1;   // very grazing directions on large tiles: per-item kernel
    TileArgs T;
    T.hdr = reinterpret_cast<const TileHdr*>(p.lat_tile_hdr);
    T.sub = reinterpret_cast<const TileSub*>(p.lat_tile_sub);
    T.order = p.lat_order;
    T.n_order = n_order;
    T.n_down = p.lat_order_down;
    T.region_cap = p.lat_region_cap;
    T.sub_cap = p.lat_sub_cap;
    T.ntx = ntx;
    T.dgz = dgz;
    T.n_stages = n_stages;
    T.scratch = nullptr;
    if (dgz > 1) {
        const size_t need = static_cast<size_t>(dgz) * 2 * A.nxy * NM * p.fp;
        if (p.lat_scratch_count < need) {
            if (p.lat_scratch) cudaFreeAsync(p.lat_scratch, s);
            p.lat_scratch = nullptr;
            p.lat_scratch_count = 0;
            RTK_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&p.lat_scratch), sizeof(double) * need, s));
            p.lat_scratch_count = need;
        }
        T.scratch = p.lat_scratch;
    }
    auto kern = lattice_mom_tile_kernel<FS, NM, TX, TY>;
    if (int rc = ensure_smem_for(kern, smem)) return rc;
    const unsigned pmblocks = static_cast<unsigned>((A.nxy * hp + 255) / 256);
    const size_t pm_smem = static_cast<size_t>(A.a1 - A.a0) * (NM * sizeof(double) + sizeof(int));
    double2* a = reinterpret_cast<double2*>(p.lat_state[0]);
    double2* b = reinterpret_cast<double2*>(p.lat_state[1]);
    const dim3 grid(static_cast<unsigned>(ntiles), static_cast<unsigned>(hp), static_cast<unsigned>(dgz));
    constexpr int ring = PAR ? 3 : 2;   // source planes: current, next (and the one after, exp-parabolic)
    for (int t = 0; t < A.nz; ++t) {
        double* cur = p.lat_splane[t % ring];
        double* nxt = p.lat_splane[(t + 1) % ring];
        double* nn = PAR ? p.lat_splane[(t + 2) % ring] : nullptr;
        if (t < A.nz - 1) {
            // step 0 fills every plane of the ring; later steps only the newest one
            const int mask = PAR ? (t == 0 ? 7 : 4) : (t == 0 ? 3 : 2);
            lattice_splane_pm_kernel<SRC, NM><<<pmblocks, 256, pm_smem, s>>>(
                A, t, reinterpret_cast<double2*>(cur), reinterpret_cast<double2*>(nxt), reinterpret_cast<double2*>(nn),
                mask, p.fp);
            RTK_LAUNCH_CHECK("lattice_splane_pm_kernel");
        }
        kern<<<grid, TX * TY, smem, s>>>(A, T, t, a, b, mom, with_inflow ? 1 : 0, p.fp,
                                         reinterpret_cast<const double2*>(cur), reinterpret_cast<const double2*>(nxt),
                                         PAR && t + 2 < A.nz ? reinterpret_cast<const double2*>(nn) : nullptr);
        RTK_LAUNCH_CHECK("lattice_mom_tile_kernel");
        if (dgz > 1) {
            const int64_t per = A.nxy * NM * p.fp;
            lattice_mom_reduce_kernel<NM><<<static_cast<unsigned>((per + 255) / 256), 256, 0, s>>>(
                p.lat_scratch, mom, t, A.nz, A.nxy, p.fp, dgz, A.n_freq);
            RTK_LAUNCH_CHECK("lattice_mom_reduce_kernel");
        }
        std::swap(a, b);
    }
    return RTK_OK;
}

template <int FS, int SRC, int NM>
static int launch_mom_tiles(const Problem& p, const LatArgs& A, bool with_inflow, double* mom, cudaStream_t s) {
    if (p.tune.lat_no_tile || !p.lat_tile_hdr || (p.fp & 1)) return -1;
    // exp-parabolic: long characteristics only (the short-characteristics downwind segment needs
    // the opacity planes, which the tiled kernel does not stage)
    if (FS == RTK_FS_EXP_PARABOLIC && (p.lat_any_sc || !p.lat_splane[2])) return -1;
    if (p.lat_tile_ty == 1) return launch_mom_tiles_t<FS, SRC, NM, 128, 1>(p, A, with_inflow, mom, s);
    return launch_mom_tiles_t<FS, SRC, NM, RTK_TILE_TX3, RTK_TILE_TY3>(p, A, with_inflow, mom, s);
}

template <int FS, int SRC, int NM>
static int launch_mom_steps(const Problem& p, const LatArgs& A, bool with_inflow, double* mom, cudaStream_t s) {
    {
        const int rc = launch_mom_tiles<FS, SRC, NM>(p, A, with_inflow, mom, s);
        if (rc != -1) return rc;
    }
    // direction groups only where a step has too few items to fill the SMs: measured cfg4
    // (65,536 items) 45.0 -> 41.3 ms with DG = 8; cfg5 (344,064 items) is slower with it
    const int64_t items = A.nxy * ((p.fp + 1) / 2);
    const int dg = p.tune.lat_dg ? p.tune.lat_dg : (items <= 131072 ? 8 : 1);
    if (dg == 1) return launch_mom_steps_dg<FS, SRC, NM, 1>(p, A, with_inflow, mom, s);
    if (dg == 4) return launch_mom_steps_dg<FS, SRC, NM, 4>(p, A, with_inflow, mom, s);
    return launch_mom_steps_dg<FS, SRC, NM, 8>(p, A, with_inflow, mom, s);
}

template <int FS, int SRC>
static int dispatch_mom_nm(const Problem& p, const LatArgs& A, bool with_inflow, double* mom, cudaStream_t s) {
    switch (p.n_mom) {
        case 1: return launch_mom_steps<FS, SRC, 1>(p, A, with_inflow, mom, s);
        case 2: return launch_mom_steps<FS, SRC, 2>(p, A, with_inflow, mom, s);
        case 3: return launch_mom_steps<FS, SRC, 3>(p, A, with_inflow, mom, s);
        case 4: return launch_mom_steps<FS, SRC, 4>(p, A, with_inflow, mom, s);
        case 5: return launch_mom_steps<FS, SRC, 5>(p, A, with_inflow, mom, s);
        case 6: return launch_mom_steps<FS, SRC, 6>(p, A, with_inflow, mom, s);
        case 7: return launch_mom_steps<FS, SRC, 7>(p, A, with_inflow, mom, s);
        case 8: return launch_mom_steps<FS, SRC, 8>(p, A, with_inflow, mom, s);
        default: return set_error(RTK_EINVAL, "lattice: unsupported number of moments");
    }
}

// moment layout: mom[s][l][f] = sum_a w_a Y_l(a) (Lambda S)(s, a, f); S from u (SRC_U) or thermal (SRC_ISO)
int lattice_transfer_moments(const Problem& p, int src_mode, bool with_inflow, const double* src, double* mom,
                             cudaStream_t s, int a0, int a1) {
    LatArgs A = lat_args(p, src, nullptr, nullptr);
    if (a1 >= 0) {   // partial moments over directions [a0, a1) (direction-sharded operator)
        A.a0 = a0;
        A.a1 = a1;
    }
    if (p.fs == RTK_FS_IE) {
        if (src_mode == LSRC_U) return dispatch_mom_nm<RTK_FS_IE, LSRC_U>(p, A, with_inflow, mom, s);
        return dispatch_mom_nm<RTK_FS_IE, LSRC_ISO>(p, A, with_inflow, mom, s);
    }
    if (p.fs == RTK_FS_EXP_PARABOLIC) {
        if (src_mode == LSRC_U) return dispatch_mom_nm<RTK_FS_EXP_PARABOLIC, LSRC_U>(p, A, with_inflow, mom, s);
        return dispatch_mom_nm<RTK_FS_EXP_PARABOLIC, LSRC_ISO>(p, A, with_inflow, mom, s);
    }
    if (src_mode == LSRC_U) return dispatch_mom_nm<RTK_FS_EXP_LINEAR, LSRC_U>(p, A, with_inflow, mom, s);
    return dispatch_mom_nm<RTK_FS_EXP_LINEAR, LSRC_ISO>(p, A, with_inflow, mom, s);
}

}  // namespace rtk
