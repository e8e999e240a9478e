// 1D slab in the moment layout: the unknown is the redistributed
// dipole moment vector u[i][k][f] (2 N_nu N_s values, 16 MB at cfg2 instead of 524 MB),
// and the operator is
//     y = u - R_w M Lambda S(u),   S[i,a,f] = gamma[i,f] sum_k c_k Y_k(a) u[i,k,f],
// i.e. R_w M of the reference's A = I - Lambda Sigma (R/operator.py:48-53) applied in
// the moment coordinates; no intensity-sized array is touched.
//
// Kernel: one CTA per (hemisphere group of 8 directions, 16-frequency tile); a producer
// warp streams TMA boxes of G = c gamma u and dt per stage of U march steps into a
// shared-memory ring; 128 consumer threads (one per ray) march the recursion and, once
// per stage, reduce their contributions w_a Y_k(a) I over the CTA's 8 directions in
// shared memory and store one partial-moment row per direction group.  A second kernel
// sums the groups in fixed order (deterministic) before the R contraction.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "formal.cuh"
#include "rtk_internal.cuh"
#include "tma.cuh"

namespace rtk {
namespace {

constexpr int kMF = 16;                 // frequencies per CTA
constexpr int kMD = 8;                  // directions per CTA
constexpr int kMC = kMF * kMD;          // consumer threads
constexpr int kMThreads = kMC + 32;
constexpr int kMU = 8;                  // march steps per stage
constexpr int kMS = 4;                  // stages
constexpr int kMDtPad = 4;

__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n)); }

__host__ __device__ constexpr int r128(int b) { return (b + 127) / 128 * 128; }

template <int NM>
struct MLayout {
    static constexpr int kG = r128(kMU * NM * kMF * 8);        // G box [U*NM rows][16 f]
    static constexpr int kDt = r128((kMU + 2) * 8);            // dt box
    static constexpr int kStage = kG + kDt;
    static constexpr int kRed = kMU * NM * kMD * kMF;          // doubles per reduction buffer
};

struct MomArgs {
    const MomCta* ctas;
    const double* phi;
    const double* inv_mu;
    const double* yb;      // [n_mom][n_angles]
    const double* wy;      // [n_mom][n_angles]  w_a Y_k(a)
    double* partial;       // [n_groups][n_space][n_mom][fp]
    int64_t n_space;
    int n_angles, n_freq, fp;
};

template <int FS, int NM>
__global__ void __launch_bounds__(kMThreads) sweep1d_mom_kernel(const __grid_constant__ CUtensorMap gmap,
                                                                const __grid_constant__ CUtensorMap dtmap, MomArgs A) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMS;
    double* red = reinterpret_cast<double*>(smem + 128);                       // [2][U][NM][kMD][kMF]
    unsigned char* stages = smem + 128 + 2 * MLayout<NM>::kRed * 8;
    const MomCta cta = A.ctas[blockIdx.x];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n = A.n_space;
    const int Q = static_cast<int>((n + kMU - 1) / kMU);
    const bool down = cta.down != 0;
    if (tid == 0) {
        for (int s = 0; s < kMS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kMC / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kMC / 32) {   // producer
        if (lane == 0) {
            prefetch_tensormap(&gmap);
            prefetch_tensormap(&dtmap);
            const uint32_t tx = static_cast<uint32_t>(kMU * NM * kMF * 8 + (kMU + 2) * 8);
            for (int q = 0; q < Q; ++q) {
                const int s = q % kMS;
                if (q >= kMS) mbar_wait(&empty[s], ((q / kMS) - 1) & 1);
                unsigned char* st = stages + s * MLayout<NM>::kStage;
                const int r0 = down ? q * kMU : static_cast<int>(n) - kMU - q * kMU;
                mbar_arrive_expect_tx(&full[s], tx);
                tma_load_2d(st, &gmap, cta.f0, r0 * NM, &full[s]);
                const int want = (down ? r0 - 1 : r0) + kMDtPad;
                tma_load_1d(st + MLayout<NM>::kG, &dtmap, want & ~1, &full[s]);
            }
        }
        return;
    }

    // consumer: ray (direction a = a0 + d, frequency f = f0 + fl)
    const int d = tid / kMF, fl = tid % kMF;
    const int f = cta.f0 + fl;
    const bool valid = d < cta.nd && f < A.n_freq;
    const int a = cta.a0 + (d < cta.nd ? d : 0);
    const double phi_f = f < A.n_freq ? A.phi[f] : 0.0;
    const double inv_mu = A.inv_mu[a];
    double yk[NM], wk[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) {
        yk[k] = A.yb[k * A.n_angles + a];
        wk[k] = valid ? A.wy[k * A.n_angles + a] : 0.0;
    }
    double acc = 0.0, s_prev = 0.0;
    double* part = A.partial + static_cast<int64_t>(cta.group) * n * NM * A.fp;
    for (int q = 0; q < Q; ++q) {
        const int s = q % kMS;
        mbar_wait(&full[s], (q / kMS) & 1);
        const unsigned char* st = stages + s * MLayout<NM>::kStage;
        const double* gs = reinterpret_cast<const double*>(st);
        const double* dts = reinterpret_cast<const double*>(st + MLayout<NM>::kG);
        const int r0 = down ? q * kMU : static_cast<int>(n) - kMU - q * kMU;
        const int dt_off = ((down ? r0 - 1 : r0) + kMDtPad) & 1;
        double* rb = red + (q & 1) * MLayout<NM>::kRed;
#pragma unroll
        for (int uu = 0; uu < kMU; ++uu) {
            const int j = q * kMU + uu;
            const int u = down ? uu : kMU - 1 - uu;     // box row of march step j
            double sv = 0.0;
#pragma unroll
            for (int k = 0; k < NM; ++k) sv = fma(yk[k], gs[(u * NM + k) * kMF + fl], sv);
            if (j > 0 && j < n) {
                const double dd = phi_f * dts[u + dt_off] * inv_mu;
                if (FS == RTK_FS_IE) {
                    const double r = rcp_nr(1.0 + dd);
                    acc = fma(acc, r, (dd * sv) * r);
                } else {
                    const ExpLin w = exp_linear_weights(dd);
                    acc = fma(acc, w.att, w.wu * s_prev + w.wc * sv);
                }
            }
            s_prev = sv;
#pragma unroll
            for (int k = 0; k < NM; ++k) rb[((u * NM + k) * kMD + d) * kMF + fl] = wk[k] * acc;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        named_sync(1, kMC);   // the stage's contributions are in rb
        // reduce over the CTA's directions in fixed order and store the stage's rows
        for (int o = tid; o < kMU * NM * kMF; o += kMC) {
            const int u = o / (NM * kMF), rem = o - u * NM * kMF, k = rem / kMF, ff = rem - k * kMF;
            const int row = r0 + u;
            const int fo = cta.f0 + ff;
            if (row < 0 || row >= n || fo >= A.n_freq) continue;
            double sum = 0.0;
#pragma unroll
            for (int dd = 0; dd < kMD; ++dd) sum += rb[((u * NM + k) * kMD + dd) * kMF + ff];
            part[(static_cast<int64_t>(row) * NM + k) * A.fp + fo] = sum;
        }
    }
}

// m[i][k][f] = sum_g partial[g][i][k][f]  (fixed order over the direction groups)
__global__ void sum_groups_kernel(const double* __restrict__ partial, double* __restrict__ mom, int64_t count,
                                  int n_groups) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += stride) {
        double s = 0.0;
        for (int g = 0; g < n_groups; ++g) s += partial[g * count + e];
        mom[e] = s;
    }
}

// G[i][k][f] = c_k gamma[i,f] u[i][k][f]   (u: user vector, pitch n_freq; G: pitch fp)
__global__ void fold_source_kernel(const double* __restrict__ u, const double* __restrict__ gamma,
                                   const double* __restrict__ coeffs, double* __restrict__ G, int64_t n_space,
                                   int n_mom, int n_freq, int fp) {
    const int64_t count = n_space * n_mom * fp;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += stride) {
        const int64_t row = e / fp;
        const int f = static_cast<int>(e - row * fp);
        const int64_t i = row / n_mom;
        const int k = static_cast<int>(row - i * n_mom);
        G[e] = f < n_freq ? coeffs[k] * gamma[i * n_freq + f] * u[row * n_freq + f] : 0.0;
    }
}

template <int FS, int NM>
int launch_mom_t(const Problem& p, cudaStream_t s) {
    MomArgs A;
    A.ctas = p.mom_ctas;
    A.phi = p.phi;
    A.inv_mu = p.inv_mu;
    A.yb = p.yb;
    A.wy = p.wy;
    A.partial = p.mom_partial;
    A.n_space = p.n_space;
    A.n_angles = p.n_angles;
    A.n_freq = p.n_freq;
    A.fp = p.fp;
    const size_t smem = 128 + 2 * MLayout<NM>::kRed * 8 + kMS * MLayout<NM>::kStage;
    auto kern = sweep1d_mom_kernel<FS, NM>;
    if (int rc = ensure_smem_for(kern, smem)) return rc;
    kern<<<p.mom_n_ctas, kMThreads, smem, s>>>(p.mom_gmap, p.tma_dtmap_mom, A);
    RTK_LAUNCH_CHECK("sweep1d_mom_kernel");
    return RTK_OK;
}

unsigned eblocks(int64_t n) {
    int64_t b = (n + 255) / 256;
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8)));
}

}  // namespace

int slab_moment_fold(const Problem& p, const double* u, cudaStream_t s) {
    fold_source_kernel<<<eblocks(p.n_space * p.n_mom * p.fp), 256, 0, s>>>(u, p.gamma, p.coeffs, p.gmom, p.n_space,
                                                                         p.n_mom, p.n_freq, p.fp);
    RTK_LAUNCH_CHECK("fold_source_kernel");
    return RTK_OK;
}

// mom = M Lambda S(u) for the slab moment layout (no boundary term)
int slab_moment_transfer(const Problem& p, const double* u, cudaStream_t s) {
    int rc = slab_moment_fold(p, u, s);
    if (rc) return rc;
    switch (p.fs) {
        case RTK_FS_IE:
            rc = p.n_mom == 1 ? launch_mom_t<RTK_FS_IE, 1>(p, s)
                              : (p.n_mom == 2 ? launch_mom_t<RTK_FS_IE, 2>(p, s) : launch_mom_t<RTK_FS_IE, 3>(p, s));
            break;
        case RTK_FS_EXP_LINEAR:
            rc = p.n_mom == 1 ? launch_mom_t<RTK_FS_EXP_LINEAR, 1>(p, s)
                              : (p.n_mom == 2 ? launch_mom_t<RTK_FS_EXP_LINEAR, 2>(p, s)
                                              : launch_mom_t<RTK_FS_EXP_LINEAR, 3>(p, s));
            break;
        default: return set_error(RTK_EINVAL, "moment layout supports the IE and exp-linear formal solvers");
    }
    if (rc) return rc;
    const int64_t count = p.n_space * p.n_mom * p.fp;
    sum_groups_kernel<<<eblocks(count), 256, 0, s>>>(p.mom_partial, p.mom, count, p.mom_n_groups);
    RTK_LAUNCH_CHECK("sum_groups_kernel");
    return RTK_OK;
}

// CTA table (8 same-hemisphere directions x 16 frequencies per CTA) and the TMA maps
int setup_slab_moments(Problem& p) {
    if (p.n_mom > 3) return set_error(RTK_EINVAL, "the slab moment layout supports at most 3 kernel moments");
    if (p.fs == RTK_FS_EXP_PARABOLIC)
        return set_error(RTK_EINVAL, "the slab moment layout supports the IE and exp-linear formal solvers");
    std::vector<MomCta> ctas;
    int group = 0;
    int a = 0;
    while (a < p.n_angles) {
        const int sign = p.h_mu[a] < 0;
        int b = a;
        while (b < p.n_angles && b - a < kMD && (p.h_mu[b] < 0) == sign) ++b;
        for (int f0 = 0; f0 < p.n_freq; f0 += kMF) {
            MomCta c;
            c.a0 = a;
            c.nd = b - a;
            c.down = sign;
            c.f0 = f0;
            c.group = group;
            ctas.push_back(c);
        }
        ++group;
        a = b;
    }
    p.mom_n_groups = group;
    p.mom_n_ctas = static_cast<int>(ctas.size());
    RTK_CUDA_TRY(cudaMalloc(&p.mom_ctas, sizeof(MomCta) * ctas.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.mom_ctas, ctas.data(), sizeof(MomCta) * ctas.size(), cudaMemcpyHostToDevice));
    // partial moments are written only for valid (row, f) entries; zero the pad columns once
    const size_t pcount = static_cast<size_t>(group) * p.n_space * p.n_mom * p.fp;
    RTK_CUDA_TRY(cudaMalloc(&p.mom_partial, sizeof(double) * pcount));
    RTK_CUDA_TRY(cudaMemset(p.mom_partial, 0, sizeof(double) * pcount));
    // G box: [U * n_mom rows][16 f] over G[n_space * n_mom][fp]
    const uint64_t gd[2] = {static_cast<uint64_t>(p.fp), static_cast<uint64_t>(p.n_space * p.n_mom)};
    const uint64_t gs[1] = {static_cast<uint64_t>(p.fp) * 8};
    const uint32_t gb[2] = {kMF, static_cast<uint32_t>(kMU * p.n_mom)};
    if (!encode_f64_map(&p.mom_gmap, p.gmom, 2, gd, gs, gb)) return set_error(RTK_ECUDA, "tensor map (moment G)");
    std::vector<double> hdt(static_cast<size_t>(p.n_space - 1 + 2 * kMDtPad), 0.0);
    RTK_CUDA_TRY(cudaMemcpy(hdt.data() + kMDtPad, p.dt, sizeof(double) * (p.n_space - 1), cudaMemcpyDeviceToHost));
    RTK_CUDA_TRY(cudaMalloc(&p.dtpad_mom, sizeof(double) * hdt.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.dtpad_mom, hdt.data(), sizeof(double) * hdt.size(), cudaMemcpyHostToDevice));
    const uint64_t dd[1] = {static_cast<uint64_t>(hdt.size())};
    const uint32_t db[1] = {static_cast<uint32_t>(kMU + 2)};
    if (!encode_f64_map(&p.tma_dtmap_mom, p.dtpad_mom, 1, dd, nullptr, db))
        return set_error(RTK_ECUDA, "tensor map (moment dt)");
    return RTK_OK;
}

}  // namespace rtk
