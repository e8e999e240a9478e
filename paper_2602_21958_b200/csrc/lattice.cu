// Periodic-lattice long-characteristics transfer for the 2D slab / 3D box
// configurations (BASELINE configs 3-5).  The operator is defined in
// oracle/lattice.py; it generalises the reference's
// 2D long characteristics (R/multidim.py:127-360): one line per
// horizontal node and direction, <= 1-cell sub-steps with trilinear T_CR
// sampling of opacity and source, the IE / exp-linear recursion
// (R/_kernels.py:90-99), and bilinear T_RC back to the nodes of each layer.
//
// Two kernels:
//  * lattice_int_kernel  (intensity layout, cfg3): one CTA per (direction,
//    4-frequency chunk) marches ALL lines of that direction through ALL layers
//    in one launch; line values are exchanged through shared memory for the
//    T_RC gather (two barriers per layer).  Output y = x - I (or I).
//  * lattice_mom_step_kernel (moment layout, cfg4/5): layer-synchronous, one
//    launch per layer step; one thread per (line, frequency) loops over every
//    direction, advancing the line and gathering the node value of the layer,
//    and accumulates the angular moments in registers (deterministic order,
//    no atomics).  Line states live in a double-buffered [dir][line][freq]
//    array.  The source is rebuilt on the fly from the moment unknown u.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "formal.cuh"
#include "rtk_internal.cuh"

namespace rtk {
namespace {

constexpr int kFC = 4;            // frequencies per CTA in the intensity kernel
constexpr int kIntThreads = 256;

__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ int wrap(int v, int n) {
    v %= n;
    return v < 0 ? v + n : v;
}

// bilinear stencil of a horizontal position (periodic): 4 column indices + weights
struct Stencil {
    int c00, c10, c01, c11;
    double w00, w10, w01, w11;
};

__device__ __forceinline__ Stencil stencil(double X, double Y, int nx, int ny) {
    const double fx = floor(X), fy = floor(Y);
    const double ax = X - fx, ay = Y - fy;
    const int i0 = wrap(static_cast<int>(fx), nx), j0 = wrap(static_cast<int>(fy), ny);
    const int i1 = (i0 + 1 == nx) ? 0 : i0 + 1, j1 = (j0 + 1 == ny) ? 0 : j0 + 1;
    Stencil s;
    s.c00 = j0 * nx + i0;
    s.c10 = j0 * nx + i1;
    s.c01 = j1 * nx + i0;
    s.c11 = j1 * nx + i1;
    s.w00 = (1 - ax) * (1 - ay);
    s.w10 = ax * (1 - ay);
    s.w01 = (1 - ax) * ay;
    s.w11 = ax * ay;
    return s;
}

struct LatArgs {
    const LatDir* dirs;
    const double* chi;      // [n_space]
    const double* phi;      // [n_freq]
    const double* src;      // SRC_VEC: S[s][a][f]; SRC_ISO: thermal[s][f]; SRC_U: u[s][l][f]
    const double* gamma;    // [s][f] (SRC_U)
    const double* x;        // OUT_X_MINUS
    double* y;
    const double* inflow_top;     // [n_freq] or null
    const double* inflow_bottom;
    int nx, ny, nz, n_dirs, n_freq, n_mom;
    int64_t nxy;
};

enum LatSrc { LSRC_VEC = 0, LSRC_ISO = 1, LSRC_U = 2 };

// One formal-solver pass of a line between two layers.  The line sits at horizontal
// position (lx + t sx, ly + t sy) on the start layer; chi_a/chi_b are the opacity
// planes and Sa/Sb the source planes (node c at Sa[c * ss]) of the start and end layers.
template <int FS>
__device__ __forceinline__ double advance_line(const LatDir& D, double acc, double lx, double ly, int t, int nx,
                                               int ny, const double* __restrict__ chi_a,
                                               const double* __restrict__ chi_b, const double* __restrict__ Sa,
                                               const double* __restrict__ Sb, int64_t ss, double phi_f) {
    double prev_s = 0.0, prev_c = 0.0;
    const double inv_sub = 1.0 / D.n_sub;
    for (int m = 0; m <= D.n_sub; ++m) {
        const double tt = t + static_cast<double>(m) / D.n_sub;
        // no FMA contraction: same rounding as the oracle's lx + tt * sx
        const double X = __dadd_rn(lx, __dmul_rn(tt, D.sx)), Y = __dadd_rn(ly, __dmul_rn(tt, D.sy));
        const double wz = static_cast<double>(m) / D.n_sub;
        const Stencil st = stencil(X, Y, nx, ny);
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
    (void)inv_sub;
    return acc;
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
    for (int64_t l = slot; l < A.nxy; l += slots) lines[l * kFC + fq] = inflow;
    for (int t = 0; t < A.nz; ++t) {
        const int k = D.down ? t : A.nz - 1 - t;
        __syncthreads();
        // T_RC gather for the nodes of layer k
        for (int64_t c = slot; c < A.nxy; c += slots) {
            const int i = static_cast<int>(c % A.nx), j = static_cast<int>(c / A.nx);
            const Stencil st = stencil(i - t * D.sx, j - t * D.sy, A.nx, A.ny);
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
        for (int64_t c = slot; c < A.nxy; c += slots) {
            const double lx = static_cast<double>(c % A.nx), ly = static_cast<double>(c / A.nx);
            double acc = lines[c * kFC + fq];
            if (fvalid) acc = advance_line<FS>(D, acc, lx, ly, t, A.nx, A.ny, chi_a, chi_b, Sa, Sb, ss, phi_f);
            lines[c * kFC + fq] = acc;
        }
    }
}

// ---------------- moment layout: layer-synchronous step ----------------
// thread = (line c, frequency f); loops over all directions.  NM moments, compile-time.
template <int FS, int NM>
__global__ void __launch_bounds__(256) lattice_mom_step_kernel(LatArgs A, int t, const double* __restrict__ st_in,
                                                                double* __restrict__ st_out, double* __restrict__ mom,
                                                                int with_inflow, int fp,
                                                                const double* __restrict__ plane_cur,
                                                                const double* __restrict__ plane_next) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= A.nxy * A.n_freq) return;
    const int f = static_cast<int>(tid % A.n_freq);
    const int64_t c = tid / A.n_freq;
    const int i = static_cast<int>(c % A.nx), j = static_cast<int>(c / A.nx);
    const double phi_f = A.phi[f];
    double m_dn[NM], m_up[NM];
#pragma unroll
    for (int l = 0; l < NM; ++l) m_dn[l] = m_up[l] = 0.0;
    const int k_dn = t, k_up = A.nz - 1 - t;
    const int64_t plane = A.nxy * A.n_freq;
    const double in_top = (with_inflow && A.inflow_top) ? A.inflow_top[f] : 0.0;
    const double in_bot = (with_inflow && A.inflow_bottom) ? A.inflow_bottom[f] : 0.0;
    for (int a = 0; a < A.n_dirs; ++a) {
        const LatDir& D = A.dirs[a];
        const bool down = D.down != 0;
        const double sx = D.sx, sy = D.sy;
        double wy[NM];
#pragma unroll
        for (int l = 0; l < NM; ++l) wy[l] = D.wy[l];
        const double* sin_a = st_in + a * plane;
        // T_RC gather for node (i, j) at this direction's current layer
        double v;
        if (t == 0) {
            v = down ? in_top : in_bot;
        } else {
            const Stencil st = stencil(i - t * sx, j - t * sy, A.nx, A.ny);
            v = st.w00 * sin_a[st.c00 * A.n_freq + f] + st.w10 * sin_a[st.c10 * A.n_freq + f] +
                st.w01 * sin_a[st.c01 * A.n_freq + f] + st.w11 * sin_a[st.c11 * A.n_freq + f];
        }
        if (down) {
#pragma unroll
            for (int l = 0; l < NM; ++l) m_dn[l] = fma(wy[l], v, m_dn[l]);
        } else {
#pragma unroll
            for (int l = 0; l < NM; ++l) m_up[l] = fma(wy[l], v, m_up[l]);
        }
        // advance own line (c) to the next layer
        if (t < A.nz - 1) {
            const int k = down ? t : A.nz - 1 - t;
            const int k2 = down ? k + 1 : k - 1;
            double acc = (t == 0) ? (down ? in_top : in_bot) : sin_a[c * A.n_freq + f];
            const LatDir Dl = D;
            acc = advance_line<FS>(Dl, acc, static_cast<double>(i), static_cast<double>(j), t, A.nx, A.ny,
                                   A.chi + static_cast<int64_t>(k) * A.nxy, A.chi + static_cast<int64_t>(k2) * A.nxy,
                                   plane_cur + a * plane + f, plane_next + a * plane + f, A.n_freq, phi_f);
            st_out[a * plane + c * A.n_freq + f] = acc;
        }
    }
    // layer k receives its down part at step k and its up part at step nz-1-k: the later step adds
    double* out_dn = mom + (static_cast<int64_t>(k_dn) * A.nxy + c) * NM * fp + f;   // pitch fp (GEMM operand)
    double* out_up = mom + (static_cast<int64_t>(k_up) * A.nxy + c) * NM * fp + f;
    if (k_dn == k_up) {
#pragma unroll
        for (int l = 0; l < NM; ++l) out_dn[static_cast<int64_t>(l) * fp] = m_dn[l] + m_up[l];
    } else {
        // step t is the first visit of both layers t and nz-1-t iff t < nz-1-t
        const bool first = k_dn < k_up;
#pragma unroll
        for (int l = 0; l < NM; ++l) {
            const int64_t o = static_cast<int64_t>(l) * fp;
            out_dn[o] = first ? m_dn[l] : out_dn[o] + m_dn[l];
            out_up[o] = first ? m_up[l] : out_up[o] + m_up[l];
        }
    }
}

// Source planes: for every direction a, S_a on the layer it reaches next (down: t+1,
// up: nz-2-t), and at t = 0 also on its entry layer; S = gamma sum_l c_l Y_l(a) u_l
// (SRC_U) or the isotropic thermal source (SRC_ISO).  Layout plane[a][c][f].
template <int SRC, int NM>
__global__ void __launch_bounds__(256) lattice_splane_kernel(LatArgs A, int t, double* __restrict__ plane_cur,
                                                              double* __restrict__ plane_next, int fill_cur) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= A.nxy * A.n_freq) return;
    const int f = static_cast<int>(tid % A.n_freq);
    const int64_t c = tid / A.n_freq;
    const int64_t plane = A.nxy * A.n_freq;
    // layers: [0] down-current, [1] up-current, [2] down-next, [3] up-next
    const int layers[4] = {t, A.nz - 1 - t, t + 1, A.nz - 2 - t};
    double uval[4][NM], g[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (q < 2 && !fill_cur) {
            g[q] = 0.0;
#pragma unroll
            for (int l = 0; l < NM; ++l) uval[q][l] = 0.0;
            continue;
        }
        const int64_t sidx = static_cast<int64_t>(layers[q]) * A.nxy + c;
        if (SRC == LSRC_U) {
#pragma unroll
            for (int l = 0; l < NM; ++l) uval[q][l] = __ldg(A.src + (sidx * NM + l) * A.n_freq + f);
            g[q] = __ldg(A.gamma + sidx * A.n_freq + f);
        } else {
            g[q] = __ldg(A.src + sidx * A.n_freq + f);
        }
    }
    for (int a = 0; a < A.n_dirs; ++a) {
        const LatDir& D = A.dirs[a];
        const int qd = D.down ? 0 : 1;
        double cy[NM];
#pragma unroll
        for (int l = 0; l < NM; ++l) cy[l] = D.cy[l];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((q & 1) != qd || (q < 2 && !fill_cur)) continue;
            double v;
            if (SRC == LSRC_U) {
                v = 0.0;
#pragma unroll
                for (int l = 0; l < NM; ++l) v = fma(cy[l], uval[q][l], v);
                v *= g[q];
            } else {
                v = g[q];
            }
            double* dst = (q < 2) ? plane_cur : plane_next;
            dst[a * plane + c * A.n_freq + f] = v;
        }
    }
}

}  // namespace

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
        for (int l = 0; l < 8; ++l) {
            const bool in = l < d->n_moments;
            D.wy[l] = in ? d->dir_w[a] * d->ybasis[l * d->n_dirs + a] : 0.0;
            D.cy[l] = in ? d->coeffs[l] * d->ybasis[l * d->n_dirs + a] : 0.0;
        }
    }
    RTK_CUDA_TRY(cudaMalloc(&p.lat_dirs, sizeof(LatDir) * dirs.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.lat_dirs, dirs.data(), sizeof(LatDir) * dirs.size(), cudaMemcpyHostToDevice));
    return RTK_OK;
}

static LatArgs lat_args(const Problem& p, const double* src, const double* x, double* y) {
    LatArgs A;
    A.dirs = p.lat_dirs;
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
    return A;
}

template <int FS, int SRC, int OUT>
static int launch_int(const Problem& p, const LatArgs& A, int with_inflow, cudaStream_t s) {
    const size_t smem = sizeof(double) * A.nxy * kFC;
    auto kern = lattice_int_kernel<FS, SRC, OUT>;
    if (smem > 48 * 1024) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
            cudaSuccess)
            return set_error(RTK_ERESOURCE, "lattice line plane does not fit in shared memory");
    }
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
    else RTK_LAT_INT(RTK_FS_EXP_LINEAR);
#undef RTK_LAT_INT
    return set_error(RTK_EINVAL, "lattice: unsupported source/output mode");
}

template <int FS, int SRC, int NM>
static int launch_mom_steps(const Problem& p, const LatArgs& A, bool with_inflow, double* mom, cudaStream_t s) {
    const int64_t threads = A.nxy * A.n_freq;
    const unsigned blocks = static_cast<unsigned>((threads + 255) / 256);
    double* a = p.lat_state[0];
    double* b = p.lat_state[1];
    for (int t = 0; t < A.nz; ++t) {
        double* cur = p.lat_splane[t & 1];
        double* nxt = p.lat_splane[(t + 1) & 1];
        if (t < A.nz - 1) {
            lattice_splane_kernel<SRC, NM><<<blocks, 256, 0, s>>>(A, t, cur, nxt, t == 0 ? 1 : 0);
            RTK_LAUNCH_CHECK("lattice_splane_kernel");
        }
        lattice_mom_step_kernel<FS, NM><<<blocks, 256, 0, s>>>(A, t, a, b, mom, with_inflow ? 1 : 0, p.fp, cur, nxt);
        RTK_LAUNCH_CHECK("lattice_mom_step_kernel");
        double* tmp = a;
        a = b;
        b = tmp;
    }
    return RTK_OK;
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
                             cudaStream_t s) {
    LatArgs A = lat_args(p, src, nullptr, nullptr);
    if (p.fs == RTK_FS_IE) {
        if (src_mode == LSRC_U) return dispatch_mom_nm<RTK_FS_IE, LSRC_U>(p, A, with_inflow, mom, s);
        return dispatch_mom_nm<RTK_FS_IE, LSRC_ISO>(p, A, with_inflow, mom, s);
    }
    if (src_mode == LSRC_U) return dispatch_mom_nm<RTK_FS_EXP_LINEAR, LSRC_U>(p, A, with_inflow, mom, s);
    return dispatch_mom_nm<RTK_FS_EXP_LINEAR, LSRC_ISO>(p, A, with_inflow, mom, s);
}

}  // namespace rtk
