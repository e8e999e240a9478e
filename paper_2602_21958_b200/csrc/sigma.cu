// K2: the scattering operator Sigma = Gamma Psi W in moment form
// (R/scattering.py:126-148), split as
//   K2a  m[i,k,f]  = sum_a w_a Y_k(a) x[i,a,f]            angular moments  (HBM-bound)
//   K2b  G[i,k,f]  = c_k gamma[i,f] sum_g R[f,g] w_g m[i,k,g]  redistribution (FP64 GEMM)
// G is the "source moment" array the sweep kernel expands on the fly
// (S[i,a,f] = sum_k Y_k(a) G[i,k,f]).  K2b is a (n_space*n_mom x n_freq) x
// (n_freq x n_freq) GEMM; K = n_freq.
#include <cuda_runtime.h>

#include "rtk_internal.cuh"

namespace rtk {
namespace {

constexpr int kMomThreads = 256;

// one thread per (i, f); loops over the n_angles directions (coalesced in f)
template <int NM>
__global__ void __launch_bounds__(kMomThreads) moments_kernel(const double* __restrict__ x, const double* __restrict__ wy,
                                                              double* __restrict__ mom, int64_t n_space, int n_angles,
                                                              int n_freq, int fp) {
    extern __shared__ double s_wy[];
    for (int t = threadIdx.x; t < NM * n_angles; t += blockDim.x) s_wy[t] = wy[t];
    pdl_prologue();   // w Y is problem data; x comes from the preceding kernel
    __syncthreads();
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_space * n_freq) return;
    const int64_t i = t / n_freq;
    const int f = static_cast<int>(t - i * n_freq);
    const int64_t n_rays = static_cast<int64_t>(n_angles) * n_freq;
    const double* xp = x + i * n_rays + f;
    double acc[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) acc[k] = 0.0;
    int a = 0;
    for (; a + 4 <= n_angles; a += 4) {
        const double v0 = __ldg(xp + (int64_t)(a + 0) * n_freq);
        const double v1 = __ldg(xp + (int64_t)(a + 1) * n_freq);
        const double v2 = __ldg(xp + (int64_t)(a + 2) * n_freq);
        const double v3 = __ldg(xp + (int64_t)(a + 3) * n_freq);
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            const double* w = s_wy + k * n_angles + a;
            acc[k] = fma(w[0], v0, acc[k]);
            acc[k] = fma(w[1], v1, acc[k]);
            acc[k] = fma(w[2], v2, acc[k]);
            acc[k] = fma(w[3], v3, acc[k]);
        }
    }
    for (; a < n_angles; ++a) {
        const double v = __ldg(xp + (int64_t)a * n_freq);
#pragma unroll
        for (int k = 0; k < NM; ++k) acc[k] = fma(s_wy[k * n_angles + a], v, acc[k]);
    }
    double* out = mom + i * NM * fp + f;
#pragma unroll
    for (int k = 0; k < NM; ++k) out[(int64_t)k * fp] = acc[k];
}

// Paired-frequency variant (n_freq even): one thread per (i, f pair), 16-byte streaming
// loads, 8 directions' loads issued before their FMAs (128 bytes in flight per thread), so
// the reduction streams x at HBM speed (cfg2: 84.7 us = 0.97 of HBM, vs 97 us for the
// 8-byte kernel above).
template <int NM>
__global__ void __launch_bounds__(kMomThreads) moments_pair_kernel(const double* __restrict__ x,
                                                                   const double* __restrict__ wy,
                                                                   double* __restrict__ mom, int64_t n_space,
                                                                   int n_angles, int n_freq, int fp) {
    extern __shared__ double s_wy[];
    for (int t = threadIdx.x; t < NM * n_angles; t += blockDim.x) s_wy[t] = wy[t];
    pdl_prologue();   // w Y is problem data; x comes from the preceding kernel
    __syncthreads();
    const int hf = n_freq >> 1;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_space * hf) return;
    const int64_t i = t / hf;
    const int h = static_cast<int>(t - i * hf);
    const int64_t n_rays = static_cast<int64_t>(n_angles) * n_freq;
    const double2* xp = reinterpret_cast<const double2*>(x + i * n_rays) + h;
    double2 acc[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) acc[k] = make_double2(0.0, 0.0);
    int a = 0;
    for (; a + 8 <= n_angles; a += 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(xp + static_cast<int64_t>(a + u) * hf);
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                const double w = s_wy[k * n_angles + a + u];
                acc[k].x = fma(w, v[u].x, acc[k].x);
                acc[k].y = fma(w, v[u].y, acc[k].y);
            }
    }
    for (; a < n_angles; ++a) {
        const double2 v = __ldcs(xp + static_cast<int64_t>(a) * hf);
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            const double w = s_wy[k * n_angles + a];
            acc[k].x = fma(w, v.x, acc[k].x);
            acc[k].y = fma(w, v.y, acc[k].y);
        }
    }
    double2* out = reinterpret_cast<double2*>(mom + i * NM * fp) + h;
#pragma unroll
    for (int k = 0; k < NM; ++k) out[static_cast<int64_t>(k) * (fp >> 1)] = acc[k];
}

// GEMM epilogues (Epilogue in rtk_internal.cuh)
__device__ __forceinline__ double epilogue(int epi, double acc, double ck, const double* gamma, int64_t gidx,
                                           const double* U, int64_t uidx) {
    switch (epi) {
        case EPI_GAMMA: return ck * acc * gamma[gidx];
        case EPI_COEF: return ck * acc;
        case EPI_SUB: return U[uidx] - acc;
        default: return acc;
    }
}

// ---- K2b: Out[c][f] = sum_g A[c][g] * B[g][f];  A = mom (rows c = (i,k)), B = rwt ----
constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
constexpr int kGemmThreads = (BM / TM) * (BN / TN);  // 256

__global__ void __launch_bounds__(kGemmThreads) redistribute_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                                    double* __restrict__ C, const double* __restrict__ gamma,
                                                                    const double* __restrict__ coeffs, int64_t M, int N, int K,
                                                                    int n_mom, int epi, int ld, int ldc,
                                                                    const double* __restrict__ U, int ldu) {
    __shared__ double As[BK][BM + 1];
    __shared__ double Bs[BK][BN];
    const int tx = threadIdx.x % (BN / TN);
    const int ty = threadIdx.x / (BN / TN);
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * BM;
    const int col0 = blockIdx.y * BN;
    double acc[TM][TN];
#pragma unroll
    for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[r][c] = 0.0;

    for (int k0 = 0; k0 < K; k0 += BK) {
        // A tile: BM x BK, stored transposed
        for (int t = threadIdx.x; t < BM * BK; t += kGemmThreads) {
            const int r = t / BK, kk = t % BK;
            const int64_t gr = row0 + r;
            const int gk = k0 + kk;
            As[kk][r] = (gr < M && gk < K) ? A[gr * ld + gk] : 0.0;
        }
        for (int t = threadIdx.x; t < BK * BN; t += kGemmThreads) {
            const int kk = t / BN, c = t % BN;
            const int gk = k0 + kk, gc = col0 + c;
            Bs[kk][c] = (gk < K && gc < N) ? B[static_cast<int64_t>(gk) * ld + gc] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            double a[TM], b[TN];
#pragma unroll
            for (int r = 0; r < TM; ++r) a[r] = As[kk][ty * TM + r];
#pragma unroll
            for (int c = 0; c < TN; ++c) b[c] = Bs[kk][tx + c * (BN / TN)];
#pragma unroll
            for (int r = 0; r < TM; ++r)
#pragma unroll
                for (int c = 0; c < TN; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < TM; ++r) {
        const int64_t gr = row0 + ty * TM + r;
        if (gr >= M) continue;
        const int64_t i = gr / n_mom;
        const int k = static_cast<int>(gr - i * n_mom);
        const double ck = coeffs[k];
#pragma unroll
        for (int c = 0; c < TN; ++c) {
            const int gc = col0 + tx + c * (BN / TN);
            if (gc >= N) continue;
            C[gr * ldc + gc] = epilogue(epi, acc[r][c], ck, gamma, i * N + gc, U, gr * ldu + gc);
        }
    }
}

// Few rows (cfg1-sized problems: M = 200): a block stages the whole K x N B operand and its
// rows of A in shared memory with one round of coalesced loads, then each thread forms one
// output from shared memory.  (The tiled kernel would launch ceil(M / 64) CTAs.)
constexpr int kSmallRows = 8;
__global__ void __launch_bounds__(256) redistribute_small_kernel(const double* __restrict__ A,
                                                                 const double* __restrict__ B, double* __restrict__ C,
                                                                 const double* __restrict__ gamma,
                                                                 const double* __restrict__ coeffs, int64_t M, int N,
                                                                 int K, int n_mom, int epi, int ld, int ldc,
                                                                 const double* __restrict__ U, int ldu) {
    extern __shared__ double sm_small[];
    double* Bs = sm_small;                 // [K][N]
    double* As = sm_small + K * N;         // [kSmallRows][K]
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kSmallRows;
    const int rows = static_cast<int>(M - r0 < kSmallRows ? M - r0 : kSmallRows);
    for (int t = threadIdx.x; t < K * N; t += blockDim.x) {
        const int g = t / N, c = t - g * N;
        Bs[t] = __ldg(B + static_cast<int64_t>(g) * ld + c);
    }
    pdl_prologue();   // R is problem data; A (the moments) comes from the preceding kernel
    for (int t = threadIdx.x; t < rows * K; t += blockDim.x) {
        const int rr = t / K, g = t - rr * K;
        As[t] = __ldg(A + (r0 + rr) * ld + g);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < rows * N; t += blockDim.x) {
        const int rr = t / N, c = t - rr * N;
        // one accumulator in ascending g: the tiled kernel's summation order, so results are
        // identical (restarted GMRES on the slow CRD cases is sensitive to the last bit)
        double acc = 0.0;
        for (int g = 0; g < K; ++g) acc = fma(As[rr * K + g], Bs[g * N + c], acc);
        const int64_t r = r0 + rr;
        const int64_t i = r / n_mom;
        C[r * ldc + c] = epilogue(epi, acc, coeffs[r - i * n_mom], gamma, i * N + c, U, r * ldu + c);
    }
}

// ---- K2b on the FP64 tensor pipe: mma.sync m8n8k4 f64 (DMMA) -------------------
// tcgen05 has no f64 kind on sm_100a, so FP64 tensor work is the warp-level
// DMMA path.  CTA tile 64 (rows c) x 128 (cols f), K staged 16 at a time in a
// 3-stage cp.async ring; 8 warps in a 2 x 4 arrangement, 32 x 32 per warp
// (4 x 4 m8n8 accumulators).  Row pitches 20 / 132 doubles keep the fragment
// loads bank-conflict free.
namespace dmma {
constexpr int BM = 64, BN = 128, BK = 16, SA = BK + 4, SB = BN + 4, STAGES = 3, THREADS = 256;
constexpr size_t kSmem = sizeof(double) * STAGES * (BM * SA + BK * SB);

__device__ __forceinline__ void cp16(double* dst, const double* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp8(double* dst, const double* src, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void mma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// VEC = 2: 16-byte copies (K and N even); VEC = 1: 8-byte copies (any shape)
template <int VEC>
__global__ void __launch_bounds__(THREADS, 2) redistribute_dmma_kernel(const double* __restrict__ A,
                                                                       const double* __restrict__ B,
                                                                       double* __restrict__ C,
                                                                       const double* __restrict__ gamma,
                                                                       const double* __restrict__ coeffs, int64_t M,
                                                                       int N, int K, int n_mom, int epi, int ld, int ldc,
                                                                       const double* __restrict__ U, int ldu) {
    extern __shared__ double smem[];
    double* As = smem;                          // [STAGES][BM][SA]
    double* Bs = smem + STAGES * BM * SA;       // [STAGES][BK][SB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 2, wn = warp & 3;
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * BM;
    const int col0 = blockIdx.y * BN;
    const int KT = (K + BK - 1) / BK;

    auto load = [&](int st, int k0) {
        double* as = As + st * BM * SA;
        double* bs = Bs + st * BK * SB;
        if (VEC == 2) {
            for (int t = tid; t < BM * BK / 2; t += THREADS) {
                const int r = t / (BK / 2), c = (t % (BK / 2)) * 2;
                const int64_t gr = row0 + r;
                const int gk = k0 + c;
                const bool v = gr < M && gk < K;
                cp16(as + r * SA + c, v ? A + gr * ld + gk : A, v);
            }
            for (int t = tid; t < BK * BN / 2; t += THREADS) {
                const int r = t / (BN / 2), c = (t % (BN / 2)) * 2;
                const int gk = k0 + r, gc = col0 + c;
                const bool v = gk < K && gc < N;
                cp16(bs + r * SB + c, v ? B + static_cast<int64_t>(gk) * ld + gc : B, v);
            }
        } else {
            for (int t = tid; t < BM * BK; t += THREADS) {
                const int r = t / BK, c = t % BK;
                const int64_t gr = row0 + r;
                const int gk = k0 + c;
                const bool v = gr < M && gk < K;
                cp8(as + r * SA + c, v ? A + gr * ld + gk : A, v);
            }
            for (int t = tid; t < BK * BN; t += THREADS) {
                const int r = t / BN, c = t % BN;
                const int gk = k0 + r, gc = col0 + c;
                const bool v = gk < K && gc < N;
                cp8(bs + r * SB + c, v ? B + static_cast<int64_t>(gk) * ld + gc : B, v);
            }
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < KT) load(s, s * BK);
        asm volatile("cp.async.commit_group;\n" ::);
    }
    const int g = lane >> 2, q = lane & 3;
    for (int kt = 0; kt < KT; ++kt) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 2));
        __syncthreads();
        const int st = kt % STAGES;
        const double* as = As + st * BM * SA + (wm * 32 + g) * SA + q;
        const double* bs = Bs + st * BK * SB + q * SB + wn * 32 + g;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = as[i * 8 * SA + kk];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = bs[kk * SB + j * 8];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) mma(acc[i][j], af[i], bf[j]);
        }
        const int nk = kt + STAGES - 1;
        if (nk < KT) load(nk % STAGES, nk * BK);
        asm volatile("cp.async.commit_group;\n" ::);
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    // epilogue: G = c_k * gamma[i,f] * acc
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gr = row0 + wm * 32 + i * 8 + g;
        if (gr >= M) continue;
        const int64_t si = gr / n_mom;
        const double ck = coeffs[gr - si * n_mom];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gc = col0 + wn * 32 + j * 8 + 2 * q;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (gc + e >= N) continue;
                C[gr * ldc + gc + e] = epilogue(epi, acc[i][j][e], ck, gamma, si * N + gc + e, U, gr * ldu + gc + e);
            }
        }
    }
}
}  // namespace dmma

// S[i,a,f] = sum_k Y_k(a) G[i,k,f]  (* per-ray gamma)  (+ thermal)
__global__ void expand_kernel(const double* __restrict__ gmom, const double* __restrict__ yb,
                              const double* __restrict__ gray, const double* __restrict__ thermal,
                              double* __restrict__ out, int64_t n_total, int n_angles, int n_freq, int n_mom, int fp) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_total) return;
    const int64_t n_rays = static_cast<int64_t>(n_angles) * n_freq;
    const int64_t i = t / n_rays;
    const int64_t ray = t - i * n_rays;
    const int a = static_cast<int>(ray / n_freq);
    const int f = static_cast<int>(ray - static_cast<int64_t>(a) * n_freq);
    const double* g = gmom + i * n_mom * fp + f;
    double s = 0.0;
    for (int k = 0; k < n_mom; ++k) s = fma(yb[k * n_angles + a], g[(int64_t)k * fp], s);
    if (gray) s *= gray[t];
    if (thermal) s += thermal[t];
    out[t] = s;
}

// Same expansion, one thread per (node i, frequency f) looping over the directions: the
// n_mom source moments are loaded once, Y comes from shared memory, and the writes of a
// direction are contiguous in f (no 64-bit index divisions per element).
template <int NM>
__global__ void __launch_bounds__(256) expand_nodes_kernel(const double* __restrict__ gmom, const double* __restrict__ yb,
                                                           const double* __restrict__ gray,
                                                           const double* __restrict__ thermal, double* __restrict__ out,
                                                           int64_t n_space, int n_angles, int n_freq, int fp) {
    extern __shared__ double s_yb[];   // [NM][n_angles]
    for (int t = threadIdx.x; t < NM * n_angles; t += blockDim.x) s_yb[t] = yb[t];
    __syncthreads();
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n_space * n_freq) return;
    const int64_t i = t / n_freq;
    const int f = static_cast<int>(t - i * n_freq);
    double g[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) g[k] = __ldg(gmom + (i * NM + k) * fp + f);
    const int64_t n_rays = static_cast<int64_t>(n_angles) * n_freq;
    const int64_t base = i * n_rays + f;
    for (int a = 0; a < n_angles; ++a) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < NM; ++k) v = fma(s_yb[k * n_angles + a], g[k], v);
        const int64_t idx = base + static_cast<int64_t>(a) * n_freq;
        if (gray) v *= __ldg(gray + idx);
        if (thermal) v += __ldg(thermal + idx);
        __stcs(out + idx, v);
    }
}

template <int NM>
int launch_expand_nodes(const Problem& p, const double* thermal, double* out, cudaStream_t s) {
    const int64_t work = p.n_space * p.n_freq;
    const unsigned blocks = static_cast<unsigned>((work + 255) / 256);
    const size_t smem = sizeof(double) * NM * p.n_angles;
    expand_nodes_kernel<NM><<<blocks, 256, smem, s>>>(p.gmom, p.yb, p.gamma_per_ray ? p.gamma : nullptr, thermal, out,
                                                      p.n_space, p.n_angles, p.n_freq, p.fp);
    RTK_LAUNCH_CHECK("expand_nodes_kernel");
    return RTK_OK;
}

template <int NM>
int launch_moments_t(const Problem& p, const double* x, cudaStream_t s) {
    const size_t smem = sizeof(double) * NM * p.n_angles;
    if ((p.n_freq & 1) == 0 && !p.tune.moments_scalar) {
        const int64_t work = p.n_space * (p.n_freq / 2);
        const unsigned blocks = static_cast<unsigned>((work + kMomThreads - 1) / kMomThreads);
        RTK_CUDA_TRY(launch_pdl(moments_pair_kernel<NM>, blocks, kMomThreads, smem, s, x, p.wy, p.mom, p.n_space,
                                p.n_angles, p.n_freq, p.fp));
        RTK_LAUNCH_CHECK("moments_pair_kernel");
        return RTK_OK;
    }
    const int64_t work = p.n_space * p.n_freq;
    const unsigned blocks = static_cast<unsigned>((work + kMomThreads - 1) / kMomThreads);
    RTK_CUDA_TRY(launch_pdl(moments_kernel<NM>, blocks, kMomThreads, smem, s, x, p.wy, p.mom, p.n_space, p.n_angles,
                            p.n_freq, p.fp));
    RTK_LAUNCH_CHECK("moments_kernel");
    return RTK_OK;
}

}  // namespace

int launch_moments(const Problem& p, const double* x, cudaStream_t s) {
    switch (p.n_mom) {
        case 1: return launch_moments_t<1>(p, x, s);
        case 2: return launch_moments_t<2>(p, x, s);
        case 3: return launch_moments_t<3>(p, x, s);
        case 4: return launch_moments_t<4>(p, x, s);
        case 5: return launch_moments_t<5>(p, x, s);
        case 6: return launch_moments_t<6>(p, x, s);
        case 7: return launch_moments_t<7>(p, x, s);
        case 8: return launch_moments_t<8>(p, x, s);
        default: return set_error(RTK_EINVAL, "moments: unsupported number of moments");
    }
}

int launch_redistribute_ex(const Problem& p, const double* A, double* C, int ldc, int epi, const double* U, int ldu,
                           cudaStream_t s, int64_t nodes, const double* gamma) {
    const int64_t M = (nodes < 0 ? p.n_space : nodes) * p.n_mom;
    if (!gamma) gamma = p.gamma;
    if (p.n_freq >= 64) {
        if (int rc = ensure_smem_for(dmma::redistribute_dmma_kernel<2>, dmma::kSmem)) return rc;
        dim3 grid(static_cast<unsigned>((M + dmma::BM - 1) / dmma::BM), (p.n_freq + dmma::BN - 1) / dmma::BN);
        // pitch fp is even: 16-byte copies always legal; pad column/row entries are zero
        dmma::redistribute_dmma_kernel<2><<<grid, dmma::THREADS, dmma::kSmem, s>>>(
            A, p.rwt, C, gamma, p.coeffs, M, p.n_freq, p.n_freq, p.n_mom, epi, p.fp, ldc, U, ldu);
        RTK_LAUNCH_CHECK("redistribute_dmma_kernel");
        return RTK_OK;
    }
    if (M * p.n_freq <= (int64_t(1) << 18)) {
        const unsigned blocks = static_cast<unsigned>((M + kSmallRows - 1) / kSmallRows);
        const size_t smem = sizeof(double) * (static_cast<size_t>(p.n_freq) * p.n_freq + kSmallRows * p.n_freq);
        RTK_CUDA_TRY(launch_pdl(redistribute_small_kernel, blocks, 256, smem, s, A, p.rwt, C, gamma, p.coeffs, M,
                                p.n_freq, p.n_freq, p.n_mom, epi, p.fp, ldc, U, ldu));
        RTK_LAUNCH_CHECK("redistribute_small_kernel");
        return RTK_OK;
    }
    dim3 grid(static_cast<unsigned>((M + BM - 1) / BM), (p.n_freq + BN - 1) / BN);
    redistribute_kernel<<<grid, kGemmThreads, 0, s>>>(A, p.rwt, C, gamma, p.coeffs, M, p.n_freq, p.n_freq, p.n_mom,
                                                      epi, p.fp, ldc, U, ldu);
    RTK_LAUNCH_CHECK("redistribute_kernel");
    return RTK_OK;
}

int launch_redistribute(const Problem& p, cudaStream_t s) {
    return launch_redistribute_ex(p, p.mom, p.gmom, p.fp, p.gamma_per_ray ? EPI_COEF : EPI_GAMMA, nullptr, 0, s);
}

int launch_expand_source(const Problem& p, const double* thermal, double* out, cudaStream_t s) {
    if (p.n_mom * p.n_angles <= 6144) {   // Y table fits the default shared-memory window
        switch (p.n_mom) {
            case 1: return launch_expand_nodes<1>(p, thermal, out, s);
            case 2: return launch_expand_nodes<2>(p, thermal, out, s);
            case 3: return launch_expand_nodes<3>(p, thermal, out, s);
            case 4: return launch_expand_nodes<4>(p, thermal, out, s);
            case 5: return launch_expand_nodes<5>(p, thermal, out, s);
            case 6: return launch_expand_nodes<6>(p, thermal, out, s);
            case 7: return launch_expand_nodes<7>(p, thermal, out, s);
            case 8: return launch_expand_nodes<8>(p, thermal, out, s);
            default: break;
        }
    }
    const int64_t n_int = p.n_space * p.n_rays;   // intensity-layout length (n_total differs in the moment layout)
    const unsigned blocks = static_cast<unsigned>((n_int + 255) / 256);
    expand_kernel<<<blocks, 256, 0, s>>>(p.gmom, p.yb, p.gamma_per_ray ? p.gamma : nullptr, thermal, out, n_int,
                                         p.n_angles, p.n_freq, p.n_mom, p.fp);
    RTK_LAUNCH_CHECK("expand_kernel");
    return RTK_OK;
}

}  // namespace rtk
