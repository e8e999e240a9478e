// K1: the 1D formal-solver sweep fused with the source reconstruction and the
// operator output.  Replaces apply_transfer + sweep_down/sweep_up
// (R/transfer.py:134-141, R/_kernels.py:70-88) and, for apply_A, the
// `gamma_table * ((moments*d) @ basis)` expansion (R/scattering.py:136) and
// `v - (...)` (R/operator.py:53): S is rebuilt on the fly from the source
// moments and never written to HBM.
//
// Mapping: one thread per ray (a, f), rays flattened in the reference order
// (a-major, f-minor), so at every march step a warp touches one contiguous
// 256-byte run of the space-major vector.  Each thread streams its inputs
// (x, dt, source moments) through a private D-stage cp.async ring in shared
// memory, so D steps of loads are in flight per thread without holding
// registers; the loop-carried chain is one FMA per step.
#include <cuda_runtime.h>

#include "formal.cuh"
#include "rtk_internal.cuh"

namespace rtk {
namespace {

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct SweepArgs {
    const double* dt;
    const double* phi;
    const double* inv_mu;
    const int* dir_sign;
    const double* yb;       // [n_mom][n_angles]
    const double* gmom;     // [n_space][n_mom][n_freq]
    const double* gray;     // per-ray gamma [n_space][n_rays] or nullptr
    const double* src;      // [n_total] for SRC_VECTOR
    const double* x;        // [n_total] for OUT_X_MINUS
    const double* inflow;   // [n_rays] or nullptr
    double* y;
    int64_t n_space;
    int64_t n_rays;
    int n_angles, n_freq, n_mom, fp;
};

constexpr int kThreads = 128;

// slots per ring stage: 0 = dt, 1 = x (OUT_X_MINUS), 2 = per-ray gamma, 3.. = moments / src
template <int SRC, int NM>
struct Slots {
    static constexpr int kSrc = (SRC == SRC_MOMENTS) ? NM : (SRC == SRC_VECTOR ? 1 : 0);
    static constexpr int kCount = 3 + kSrc;
};

template <int FS, int NM, int SRC, int OUT, int D>
__global__ void __launch_bounds__(kThreads) sweep1d_kernel(SweepArgs A) {
    extern __shared__ double ring[];
    constexpr int NS = Slots<SRC, NM>::kCount;
    const int tid = threadIdx.x;
    const int64_t ray = static_cast<int64_t>(blockIdx.x) * kThreads + tid;
    const bool valid = ray < A.n_rays;
    const int a = valid ? static_cast<int>(ray / A.n_freq) : 0;
    const int f = valid ? static_cast<int>(ray % A.n_freq) : 0;
    const int64_t n = A.n_space;
    const bool down = valid ? (A.dir_sign[a] < 0) : true;
    const double phi_f = A.phi[f];
    const double inv_mu = A.inv_mu[a];
    const bool gray = (SRC == SRC_MOMENTS) && A.gray != nullptr;
    double ya[NM > 0 ? NM : 1];
#pragma unroll
    for (int k = 0; k < (NM > 0 ? NM : 1); ++k) ya[k] = (SRC == SRC_MOMENTS && k < NM) ? A.yb[k * A.n_angles + a] : 0.0;

    auto slot = [&](int stage, int s) -> double* { return ring + (stage * NS + s) * kThreads + tid; };

    // issue the async copies feeding march node j into ring stage j % D
    auto issue = [&](int64_t j, int st) {
        if (valid && j < n) {
            const int64_t i = down ? j : n - 1 - j;
            if (j < n - 1) {
                const int64_t seg = down ? j : n - 2 - j;
                cp_async8(slot(st, 0), A.dt + seg);
            }
            if (OUT == OUT_X_MINUS) cp_async8(slot(st, 1), A.x + i * A.n_rays + ray);
            if (SRC == SRC_MOMENTS) {
                if (gray) cp_async8(slot(st, 2), A.gray + i * A.n_rays + ray);
                const double* g = A.gmom + i * (int64_t)NM * A.fp + f;
#pragma unroll
                for (int k = 0; k < NM; ++k) cp_async8(slot(st, 3 + k), g + (int64_t)k * A.fp);
            } else if (SRC == SRC_VECTOR) {
                cp_async8(slot(st, 3), A.src + i * A.n_rays + ray);
            }
        }
        cp_commit();
    };

    auto source = [&](int st) -> double {
        if (SRC == SRC_MOMENTS) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < NM; ++k) s = fma(ya[k], *slot(st, 3 + k), s);
            if (gray) s *= *slot(st, 2);
            return s;
        } else if (SRC == SRC_VECTOR) {
            return *slot(st, 3);
        }
        return 0.0;
    };

    // prologue: D-1 stages in flight
    for (int j = 0; j < D - 1; ++j) issue(j, j);

    double acc = (A.inflow != nullptr && valid) ? A.inflow[ray] : 0.0;
    double s_prev = 0.0, d_prev = 0.0, s_saved = 0.0;
    int st = 0;                       // ring stage of node j
    for (int64_t j = 0; j < n; ++j) {
        const int st_next = (st + 1 == D) ? 0 : st + 1;
        issue(j + D - 1, st == 0 ? D - 1 : st - 1);
        if (FS == RTK_FS_EXP_PARABOLIC) cp_wait<D - 2>(); else cp_wait<D - 1>();
        const double s_cur = (FS == RTK_FS_EXP_PARABOLIC && j >= 2) ? s_saved : source(st);
        const double d_cur = (j < n - 1) ? phi_f * *slot(st, 0) * inv_mu : 0.0;
        if (j > 0) {
            if (FS == RTK_FS_IE) {
                const double r = 1.0 / (1.0 + d_prev);
                acc = fma(acc, r, (d_prev * s_cur) * r);
            } else if (FS == RTK_FS_EXP_PARABOLIC && j < n - 1) {
                const double s_next = source(st_next);
                const ExpPar w = exp_parabolic_weights(d_prev, d_cur);
                acc = fma(acc, w.att, w.wu * s_prev + w.wc * s_cur + w.wd * s_next);
                s_saved = s_next;
            } else {
                const ExpLin w = exp_linear_weights(d_prev);
                acc = fma(acc, w.att, w.wu * s_prev + w.wc * s_cur);
            }
        }
        if (valid) {
            const int64_t i = down ? j : n - 1 - j;
            const double out = (OUT == OUT_X_MINUS) ? (*slot(st, 1) - acc) : acc;
            A.y[i * A.n_rays + ray] = out;
        }
        s_prev = s_cur;
        d_prev = d_cur;
        st = st_next;
    }
    cp_wait<0>();
}

template <int FS, int NM, int SRC, int OUT>
int launch_t(const SweepArgs& A, cudaStream_t s) {
    constexpr int D = (NM <= 2) ? 16 : (NM <= 4 ? 10 : 6);
    constexpr int NS = Slots<SRC, NM>::kCount;
    const size_t smem = static_cast<size_t>(D) * NS * kThreads * sizeof(double);
    auto kern = sweep1d_kernel<FS, NM, SRC, OUT, D>;
    if (int rc = ensure_smem_for(kern, smem)) return rc;
    const unsigned blocks = static_cast<unsigned>((A.n_rays + kThreads - 1) / kThreads);
    kern<<<blocks, kThreads, smem, s>>>(A);
    RTK_LAUNCH_CHECK("sweep1d_kernel");
    return RTK_OK;
}

template <int FS, int SRC, int OUT>
int dispatch_nm(int nm, const SweepArgs& A, cudaStream_t s) {
    if (SRC != SRC_MOMENTS) return launch_t<FS, 1, SRC, OUT>(A, s);
    switch (nm) {
        case 1: return launch_t<FS, 1, SRC, OUT>(A, s);
        case 2: return launch_t<FS, 2, SRC, OUT>(A, s);
        case 3: return launch_t<FS, 3, SRC, OUT>(A, s);
        case 4: return launch_t<FS, 4, SRC, OUT>(A, s);
        case 5: return launch_t<FS, 5, SRC, OUT>(A, s);
        case 6: return launch_t<FS, 6, SRC, OUT>(A, s);
        case 7: return launch_t<FS, 7, SRC, OUT>(A, s);
        case 8: return launch_t<FS, 8, SRC, OUT>(A, s);
        default: return set_error(RTK_EINVAL, "sweep: unsupported number of moments");
    }
}

template <int FS>
int dispatch_mode(int src_mode, int out_mode, int nm, const SweepArgs& A, cudaStream_t s) {
    if (src_mode == SRC_MOMENTS && out_mode == OUT_X_MINUS) return dispatch_nm<FS, SRC_MOMENTS, OUT_X_MINUS>(nm, A, s);
    if (src_mode == SRC_VECTOR && out_mode == OUT_ACC) return dispatch_nm<FS, SRC_VECTOR, OUT_ACC>(nm, A, s);
    if (src_mode == SRC_ZERO && out_mode == OUT_ACC) return dispatch_nm<FS, SRC_ZERO, OUT_ACC>(nm, A, s);
    return set_error(RTK_EINVAL, "sweep: unsupported source/output mode");
}

}  // namespace

int launch_sweep(const Problem& p, int src_mode, int out_mode, bool with_inflow,
                 const double* src_vec, const double* x, double* y, cudaStream_t s) {
    if (p.n_rays == 0 || p.n_space == 0) return RTK_OK;
    SweepArgs A;
    A.dt = p.dt;
    A.phi = p.phi;
    A.inv_mu = p.inv_mu;
    A.dir_sign = p.dir_sign;
    A.yb = p.yb;
    A.gmom = p.gmom;
    A.gray = p.gamma_per_ray ? p.gamma : nullptr;
    A.src = src_vec;
    A.x = x;
    A.inflow = with_inflow ? p.inflow : nullptr;
    A.y = y;
    A.n_space = p.n_space;
    A.n_rays = p.n_rays;
    A.n_angles = p.n_angles;
    A.n_freq = p.n_freq;
    A.n_mom = p.n_mom;
    A.fp = p.fp;
    switch (p.fs) {
        case RTK_FS_IE: return dispatch_mode<RTK_FS_IE>(src_mode, out_mode, p.n_mom, A, s);
        case RTK_FS_EXP_LINEAR: return dispatch_mode<RTK_FS_EXP_LINEAR>(src_mode, out_mode, p.n_mom, A, s);
        case RTK_FS_EXP_PARABOLIC: return dispatch_mode<RTK_FS_EXP_PARABOLIC>(src_mode, out_mode, p.n_mom, A, s);
        default: return set_error(RTK_EINVAL, "unknown formal solver");
    }
}

}  // namespace rtk
