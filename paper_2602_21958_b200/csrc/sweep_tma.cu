// K1 (TMA variant): the apply_A sweep y = x - Lambda S with S expanded on the fly
// from the source moments G.  Replaces apply_transfer + sweep_down/sweep_up +
// the Legendre/PRD expansion + `v - (...)` (R/transfer.py:134-141,
// R/_kernels.py:70-88, R/scattering.py:136, R/operator.py:53).
//
// Warp-specialised CTA: 4 consumer warps own 128 rays (one ray per thread,
// rays of one hemisphere, consecutive in the reference's a-major/f-minor
// order, so a march step touches one contiguous 1 KB run of x and of y); one
// producer warp streams, per stage of U march steps, three TMA tensor boxes
// into shared memory: x[rows][130 rays], G[rows*n_mom][f-window] and dt[rows].
// S stages are in flight (mbarrier full/empty ring), so no per-thread load
// instruction touches L1 and the loop-carried chain is one FMA per step.
// Measured on sm_100a: a TMA box whose innermost start coordinate is not a
// multiple of 16 bytes (or is negative) faults with "illegal instruction", so
// boxes start at the even coordinate below the wanted one (x box 130 wide,
// dt box 6 long over a front-padded dt copy) and threads read at an offset.
#include <cuda.h>
#include <cuda_runtime.h>

#include "formal.cuh"
#include "rtk_internal.cuh"
#include "tma.cuh"

namespace rtk {

bool encode_f64_map(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* stride_bytes,
                    const uint32_t* box) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return false;
        fn = reinterpret_cast<Fn>(p);
    }
    if (rank < 1 || rank > 3) return false;
    cuuint64_t gd[3] = {dims[0], rank > 1 ? dims[1] : 1, rank > 2 ? dims[2] : 1};
    cuuint64_t gs[2] = {rank > 1 ? stride_bytes[0] : 0, rank > 2 ? stride_bytes[1] : 0};
    cuuint32_t bd[3] = {box[0], rank > 1 ? box[1] : 1, rank > 2 ? box[2] : 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), gd, gs, bd, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 2D f64 map with 128-byte swizzle (box inner extent must be 16 doubles)
bool encode_f64_map_sw128(CUtensorMap* map, const void* base, const uint64_t* dims, uint64_t row_stride_bytes,
                          const uint32_t* box) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return false;
        fn = reinterpret_cast<Fn>(p);
    }
    cuuint64_t gd[2] = {dims[0], dims[1]};
    cuuint64_t gs[1] = {row_stride_bytes};
    cuuint32_t bd[2] = {box[0], box[1]};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), gd, gs, bd, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

namespace {

constexpr int kRaysPerCta = 128;
constexpr int kXW = kRaysPerCta + 2;   // x box width (covers an odd ray0)
// dt box length is U + 2 (U steps plus the parity offset)
constexpr int kDtPad = 4;              // leading zeros in the padded dt copy
constexpr int kConsumerWarps = kRaysPerCta / 32;
constexpr int kTmaThreads = kRaysPerCta + 32;

__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

struct TmaArgs {
    const TmaCta* ctas;
    const double* phi;
    const double* inv_mu;
    const double* yb;      // [n_mom][n_angles]
    double* y;
    int64_t n_space;
    int64_t n_rays;
    int n_angles, n_freq, gw;
};

__host__ __device__ constexpr int round128(int bytes) { return (bytes + 127) / 128 * 128; }

template <int NM, int U>
struct Layout {
    static constexpr int kX = round128(U * kXW * 8);
    __host__ __device__ static int g_bytes(int gw) { return round128(U * NM * gw * 8); }
    static constexpr int kDtW = U + 2;
    static constexpr int kDt = round128(kDtW * 8);
    // the exp-parabolic stage carries two more dt-shaped rows (qc, qd of the hemisphere)
    __host__ __device__ static int stage_bytes(int gw, bool par = false) { return kX + g_bytes(gw) + (par ? 3 : 1) * kDt; }
};

struct SweepState {
    double acc, s_prev;
    double* yp;
};

template <int NM>
struct ConsumerCtx {
    int xoff, gcol, gw;
    double phi_f, inv_mu, rc2;   // rc2 = 1 / (phi_f inv_mu)^2 (exp-parabolic tables)
    bool valid;
    double yk[NM];
};

// U march steps of one stage.  DOWN: box row u = step uu (ascending i); up: u = U-1-uu.
// CHECK: first/last stage (node 0 has no segment; rows beyond the slab are skipped).
// Exponential solvers: the stage's weights are computed first, branch-free
// (exp_linear_weights_bf), so the U weight evaluations are independent instruction
// streams the scheduler interleaves; the recursion then runs over them.
template <int FS, int NM, int U, bool DOWN, bool CHECK>
__device__ __forceinline__ void consume(const ConsumerCtx<NM>& c, SweepState& st, const double* __restrict__ xs,
                                        const double* __restrict__ gs, const double* __restrict__ dts, int q,
                                        int64_t n, int64_t step) {
    const double* gcol = gs + c.gcol;
    double w0[U], w1[U], w2[U];
    if (FS != RTK_FS_IE) {
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const ExpLin w = exp_linear_weights_bf(c.phi_f * dts[DOWN ? uu : U - 1 - uu] * c.inv_mu);
            w0[uu] = w.att;
            w1[uu] = w.wu;
            w2[uu] = w.wc;
        }
    }
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
        const int j = q * U + uu;
        if (CHECK && j >= n) break;
        const int u = DOWN ? uu : U - 1 - uu;
        const double xv = xs[u * kXW + c.xoff];
        double sv = 0.0;
#pragma unroll
        for (int k = 0; k < NM; ++k) sv = fma(c.yk[k], gcol[(u * NM + k) * c.gw], sv);
        if (!CHECK || j > 0) {
            if (FS == RTK_FS_IE) {
                const double d = c.phi_f * dts[u] * c.inv_mu;
                const double r = rcp_nr(1.0 + d);
                st.acc = fma(st.acc, r, (d * sv) * r);
            } else {
                st.acc = fma(st.acc, w0[uu], w1[uu] * st.s_prev + w2[uu] * sv);
            }
        }
        st.s_prev = sv;
        if (c.valid) *st.yp = xv - st.acc;
        st.yp += step;
    }
}

// Exp-parabolic needs the downwind source S_{j+1}: node j-1 is finalised while node j
// is being read (one-node delay), the last node with the linear weights afterwards.
struct ParState {
    double acc, s_m2, s_m1, d_m2, x_m1;
    double* yp;   // node to be finalised next
};

template <int NM, int U, bool DOWN, bool CHECK>
__device__ __forceinline__ void consume_par(const ConsumerCtx<NM>& c, ParState& st, const double* __restrict__ xs,
                                            const double* __restrict__ gs, const double* __restrict__ dts,
                                            const double* __restrict__ qcs, const double* __restrict__ qds, int q,
                                            int64_t n, int64_t step) {
    const double* gcol = gs + c.gcol;
    // optical depths of the segments into each step's node, then the stage's weights
    // (update at step uu uses the segments into nodes j-1 and j; qcs / qds hold the Lagrange
    // denominators of that segment pair at the position of the segment into node j)
    double din[U], w0[U], w1[U], w2[U], w3[U];
#pragma unroll
    for (int uu = 0; uu < U; ++uu) din[uu] = c.phi_f * dts[DOWN ? uu : U - 1 - uu] * c.inv_mu;
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
        const int u = DOWN ? uu : U - 1 - uu;
        const ExpPar w = exp_parabolic_weights_tab(uu == 0 ? st.d_m2 : din[uu - 1], din[uu], c.rc2, qcs[u], qds[u]);
        w0[uu] = w.att;
        w1[uu] = w.wu;
        w2[uu] = w.wc;
        w3[uu] = w.wd;
    }
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
        const int j = q * U + uu;
        if (CHECK && j >= n) break;
        const int u = DOWN ? uu : U - 1 - uu;
        const double xv = xs[u * kXW + c.xoff];
        double sv = 0.0;
#pragma unroll
        for (int k = 0; k < NM; ++k) sv = fma(c.yk[k], gcol[(u * NM + k) * c.gw], sv);
        if (CHECK && j == 0) {
            if (c.valid) *st.yp = xv - st.acc;
            st.yp += step;
            st.s_m1 = sv;
            st.x_m1 = xv;
            continue;
        }
        if (!(CHECK && j == 1)) {
            st.acc = fma(st.acc, w0[uu], w1[uu] * st.s_m2 + w2[uu] * st.s_m1 + w3[uu] * sv);
            if (c.valid) *st.yp = st.x_m1 - st.acc;
            st.yp += step;
        }
        st.s_m2 = st.s_m1;
        st.s_m1 = sv;
        st.d_m2 = din[uu];
        st.x_m1 = xv;
    }
}

template <int FS, int NM, int U, int S>
__global__ void __launch_bounds__(kTmaThreads) sweep1d_tma_kernel(const __grid_constant__ CUtensorMap xmap,
                                                                  const __grid_constant__ CUtensorMap gmap,
                                                                  const __grid_constant__ CUtensorMap dtmap,
                                                                  const __grid_constant__ CUtensorMap qcmap_dn,
                                                                  const __grid_constant__ CUtensorMap qdmap_dn,
                                                                  const __grid_constant__ CUtensorMap qcmap_up,
                                                                  const __grid_constant__ CUtensorMap qdmap_up,
                                                                  TmaArgs A) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    unsigned char* stages = smem + 128;
    const int gbytes = Layout<NM, U>::g_bytes(A.gw);
    constexpr bool PAR = FS == RTK_FS_EXP_PARABOLIC;
    const int sbytes = Layout<NM, U>::stage_bytes(A.gw, PAR);

    const TmaCta cta = A.ctas[blockIdx.x];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t n = A.n_space;
    const int Q = static_cast<int>((n + U - 1) / U);
    const bool down = cta.down != 0;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kConsumerWarps) {
        // ---------------- producer warp ----------------
        if (lane == 0) {
            // programmatic dependent launch: the prologue above overlapped the tail of the
            // kernel that produced G; wait for it to complete before streaming G
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            prefetch_tensormap(&xmap);
            prefetch_tensormap(&gmap);
            prefetch_tensormap(&dtmap);
            const uint32_t tx = static_cast<uint32_t>(U * kXW * 8 + U * NM * A.gw * 8 +
                                                      (PAR ? 3 : 1) * Layout<NM, U>::kDtW * 8);
            if (PAR) {
                prefetch_tensormap(down ? &qcmap_dn : &qcmap_up);
                prefetch_tensormap(down ? &qdmap_dn : &qdmap_up);
            }
            for (int q = 0; q < Q; ++q) {
                const int s = q % S;
                if (q >= S) mbar_wait(&empty[s], ((q / S) - 1) & 1);
                unsigned char* st = stages + s * sbytes;
                const int r0 = down ? q * U : static_cast<int>(n) - U - q * U;   // first box row
                mbar_arrive_expect_tx(&full[s], tx);
                tma_load_2d(st, &xmap, cta.ray0 & ~1, r0, &full[s]);
                tma_load_2d(st + Layout<NM, U>::kX, &gmap, cta.f0, r0 * NM, &full[s]);
                // dt_pad[kDtPad + i] = dt[i]; down rows need dt[r0 - 1 + u], up rows dt[r0 + u]
                const int want = (down ? r0 - 1 : r0) + kDtPad;
                tma_load_1d(st + Layout<NM, U>::kX + gbytes, &dtmap, want & ~1, &full[s]);
                if (PAR) {   // same box as dt: entry i of the tables belongs to segment i
                    unsigned char* qb = st + Layout<NM, U>::kX + gbytes + Layout<NM, U>::kDt;
                    tma_load_1d(qb, down ? &qcmap_dn : &qcmap_up, want & ~1, &full[s]);
                    tma_load_1d(qb + Layout<NM, U>::kDt, down ? &qdmap_dn : &qdmap_up, want & ~1, &full[s]);
                }
            }
        }
        return;
    }

    // ---------------- consumer warps: one ray per thread ----------------
    const bool valid = tid < cta.nr;
    const int64_t ray = cta.ray0 + tid;
    const int a = valid ? static_cast<int>(ray / A.n_freq) : 0;
    const int f = valid ? static_cast<int>(ray - static_cast<int64_t>(a) * A.n_freq) : 0;
    const int gcol = f - cta.f0;
    const int xoff = tid + (cta.ray0 & 1);
    const double phi_f = A.phi[f];
    const double inv_mu = A.inv_mu[a];
    double yk[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) yk[k] = A.yb[k * A.n_angles + a];
    SweepState st{0.0, 0.0, A.y + (down ? 0 : (n - 1) * A.n_rays) + ray};
    ParState ps{0.0, 0.0, 0.0, 0.0, 0.0, st.yp};
    const int64_t step = down ? A.n_rays : -A.n_rays;
    ConsumerCtx<NM> c2;
    c2.xoff = xoff;
    c2.gcol = gcol;
    c2.gw = A.gw;
    c2.phi_f = phi_f;
    c2.inv_mu = inv_mu;
    c2.rc2 = 1.0 / ((phi_f * inv_mu) * (phi_f * inv_mu));
    c2.valid = valid;
#pragma unroll
    for (int k = 0; k < NM; ++k) c2.yk[k] = yk[k];
    // first and last stage carry the boundary checks; the body runs check-free, with the
    // march direction resolved at compile time
    for (int q = 0; q < Q; ++q) {
        const int s = q % S;
        mbar_wait(&full[s], (q / S) & 1);
        const unsigned char* stg = stages + s * sbytes;
        const double* xs = reinterpret_cast<const double*>(stg);
        const double* gs = reinterpret_cast<const double*>(stg + Layout<NM, U>::kX);
        const double* dts = reinterpret_cast<const double*>(stg + Layout<NM, U>::kX + gbytes);
        const int r0 = down ? q * U : static_cast<int>(n) - U - q * U;
        const int dt_off = ((down ? r0 - 1 : r0) + kDtPad) & 1;
        const bool edge = (q == 0) || (q == Q - 1);
        if (FS == RTK_FS_EXP_PARABOLIC) {
            const double* qcs = dts + Layout<NM, U>::kDt / 8 + dt_off;
            const double* qds = qcs + Layout<NM, U>::kDt / 8;
            if (down) {
                if (edge) consume_par<NM, U, true, true>(c2, ps, xs, gs, dts + dt_off, qcs, qds, q, n, step);
                else consume_par<NM, U, true, false>(c2, ps, xs, gs, dts + dt_off, qcs, qds, q, n, step);
            } else {
                if (edge) consume_par<NM, U, false, true>(c2, ps, xs, gs, dts + dt_off, qcs, qds, q, n, step);
                else consume_par<NM, U, false, false>(c2, ps, xs, gs, dts + dt_off, qcs, qds, q, n, step);
            }
        } else if (down) {
            if (edge) consume<FS, NM, U, true, true>(c2, st, xs, gs, dts + dt_off, q, n, step);
            else consume<FS, NM, U, true, false>(c2, st, xs, gs, dts + dt_off, q, n, step);
        } else {
            if (edge) consume<FS, NM, U, false, true>(c2, st, xs, gs, dts + dt_off, q, n, step);
            else consume<FS, NM, U, false, false>(c2, st, xs, gs, dts + dt_off, q, n, step);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (FS == RTK_FS_EXP_PARABOLIC && n >= 2) {   // last node: linear weights on the last segment
        const ExpLin w = exp_linear_weights(ps.d_m2);
        ps.acc = fma(ps.acc, w.att, w.wu * ps.s_m2 + w.wc * ps.s_m1);
        if (valid) *ps.yp = ps.x_m1 - ps.acc;
    }
}

template <int FS, int NM, int U, int S>
int launch_tma_us(const Problem& p, const double* x, double* y, cudaStream_t s);

template <int FS, int NM>
int launch_tma_t(const Problem& p, const double* x, double* y, cudaStream_t s) {
    if (p.tma_u == 8) return launch_tma_us<FS, NM, 8, 4>(p, x, y, s);
    return launch_tma_us<FS, NM, 4, (NM <= 2) ? 8 : 4>(p, x, y, s);
}

template <int FS, int NM, int U, int S>
int launch_tma_us(const Problem& p, const double* x, double* y, cudaStream_t s) {
    CUtensorMap xmap;
    const uint64_t xd[2] = {static_cast<uint64_t>(p.n_rays), static_cast<uint64_t>(p.n_space)};
    const uint64_t xs[1] = {static_cast<uint64_t>(p.n_rays) * 8};
    const uint32_t xb[2] = {kXW, U};
    if (!encode_f64_map(&xmap, x, 2, xd, xs, xb)) return set_error(RTK_ECUDA, "sweep: x tensor-map encoding failed");
    TmaArgs A;
    A.ctas = p.tma_ctas;
    A.phi = p.phi;
    A.inv_mu = p.inv_mu;
    A.yb = p.yb;
    A.y = y;
    A.n_space = p.n_space;
    A.n_rays = p.n_rays;
    A.n_angles = p.n_angles;
    A.n_freq = p.n_freq;
    A.gw = p.tma_gw;
    const size_t smem = 128 + static_cast<size_t>(S) * Layout<NM, U>::stage_bytes(p.tma_gw, FS == RTK_FS_EXP_PARABOLIC);
    auto kern = sweep1d_tma_kernel<FS, NM, U, S>;
    if (int rc = ensure_smem_for(kern, smem)) return rc;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.gridDim = dim3(p.tma_n_ctas);
    cfg.blockDim = dim3(kTmaThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RTK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, xmap, p.tma_gmap, p.tma_dtmap, p.tma_qmap[0], p.tma_qmap[1],
                                    p.tma_qmap[2], p.tma_qmap[3], A));
    RTK_LAUNCH_CHECK("sweep1d_tma_kernel");
    return RTK_OK;
}

template <int FS>
int dispatch_tma(const Problem& p, const double* x, double* y, cudaStream_t s) {
    switch (p.n_mom) {
        case 1: return launch_tma_t<FS, 1>(p, x, y, s);
        case 2: return launch_tma_t<FS, 2>(p, x, y, s);
        case 3: return launch_tma_t<FS, 3>(p, x, y, s);
        case 4: return launch_tma_t<FS, 4>(p, x, y, s);
        default: return -1;
    }
}

}  // namespace

// returns RTK_OK, an error code, or -1 when the TMA path does not apply to this problem's
// shape (fixed at setup) or to an x that is not 16-byte aligned (TMA global addresses must be)
int launch_sweep_tma(const Problem& p, const double* x, double* y, cudaStream_t s) {
    if (!p.tma_ready || p.gamma_per_ray) return -1;
    if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return -1;
    if (p.fs == RTK_FS_IE) return dispatch_tma<RTK_FS_IE>(p, x, y, s);
    if (p.fs == RTK_FS_EXP_LINEAR) return dispatch_tma<RTK_FS_EXP_LINEAR>(p, x, y, s);
    if (p.fs == RTK_FS_EXP_PARABOLIC) return dispatch_tma<RTK_FS_EXP_PARABOLIC>(p, x, y, s);
    return -1;
}

// Host setup: CTA table (hemisphere-uniform ray groups) and the G / dt tensor maps.
int setup_tma(Problem& p) {
    p.tma_ready = false;
    if ((p.n_rays % 2) != 0 || p.n_space < 2 || p.n_mom > 4) return RTK_OK;
    std::vector<TmaCta> ctas;
    const int nf = p.n_freq;
    if (nf >= kRaysPerCta) {
        p.tma_gw = kRaysPerCta;
        for (int a = 0; a < p.n_angles; ++a)
            for (int f0 = 0; f0 < nf; f0 += kRaysPerCta) {
                TmaCta c;
                c.ray0 = a * nf + f0;
                c.nr = std::min(kRaysPerCta, nf - f0);
                c.down = p.h_mu[a] < 0 ? 1 : 0;
                c.f0 = f0;
                ctas.push_back(c);
            }
    } else {
        p.tma_gw = p.fp;
        const int per = kRaysPerCta / nf;
        int a = 0;
        while (a < p.n_angles) {
            const int sign = p.h_mu[a] < 0;
            int b = a;
            while (b < p.n_angles && b - a < per && (p.h_mu[b] < 0) == sign) ++b;
            TmaCta c;
            c.ray0 = a * nf;
            c.nr = (b - a) * nf;
            c.down = sign;
            c.f0 = 0;
            ctas.push_back(c);
            a = b;
        }
    }
    const uint64_t gd[2] = {static_cast<uint64_t>(p.fp), static_cast<uint64_t>(p.n_space * p.n_mom)};
    const uint64_t gs[1] = {static_cast<uint64_t>(p.fp) * 8};
    p.tma_u = p.n_mom <= 2 ? 8 : 4;   // march steps per pipeline stage (U = 8: 96% of HBM on cfg2)
    const uint32_t gb[2] = {static_cast<uint32_t>(p.tma_gw), static_cast<uint32_t>(p.tma_u * p.n_mom)};
    // front/back zero-padded copy of dt so every dt box starts at an even, non-negative coordinate
    std::vector<double> hdt(static_cast<size_t>(p.n_space - 1 + 2 * kDtPad), 0.0);
    RTK_CUDA_TRY(cudaMemcpy(hdt.data() + kDtPad, p.dt, sizeof(double) * (p.n_space - 1), cudaMemcpyDeviceToHost));
    RTK_CUDA_TRY(cudaMalloc(&p.dtpad, sizeof(double) * hdt.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.dtpad, hdt.data(), sizeof(double) * hdt.size(), cudaMemcpyHostToDevice));
    const uint64_t dd[1] = {static_cast<uint64_t>(hdt.size())};
    const uint32_t db[1] = {static_cast<uint32_t>(p.tma_u + 2)};
    if (!encode_f64_map(&p.tma_gmap, p.gmom, 2, gd, gs, gb)) return set_error(RTK_ECUDA, "sweep: G tensor map");
    if (!encode_f64_map(&p.tma_dtmap, p.dtpad, 1, dd, nullptr, db)) return set_error(RTK_ECUDA, "sweep: dt tensor map");
    {
        // Exp-parabolic Lagrange denominators, indexed like dtpad (entry kDtPad + i = segment i,
        // between nodes i and i + 1).  The update that finalises a node uses the segment pair
        // around it; the table entry sits at the pair's LATER segment in march order:
        //   down, entry i: (u, d) = (dt[i-1], dt[i]);   up, entry i: (u, d) = (dt[i+1], dt[i]);
        //   qc = 1 / (u d),  qd = 1 / (d (u + d)).  Pairs reaching outside the slab are never
        // used by the kernel (first update skipped, last node linear); they hold 0.
        const int64_t nseg = p.n_space - 1;
        const size_t len = (hdt.size() + 1) / 2 * 2;   // table stride: tensor-map bases must be 16-byte aligned
        std::vector<double> tab(4 * len, 0.0);
        auto dtv = [&](int64_t i) { return hdt[kDtPad + i]; };
        for (int64_t i = 0; i < nseg; ++i) {
            if (i >= 1) {
                const double u = dtv(i - 1), d = dtv(i);
                tab[0 * len + kDtPad + i] = 1.0 / (u * d);
                tab[1 * len + kDtPad + i] = 1.0 / (d * (u + d));
            }
            if (i + 1 < nseg) {
                const double u = dtv(i + 1), d = dtv(i);
                tab[2 * len + kDtPad + i] = 1.0 / (u * d);
                tab[3 * len + kDtPad + i] = 1.0 / (d * (u + d));
            }
        }
        RTK_CUDA_TRY(cudaMalloc(&p.par_tab, sizeof(double) * tab.size()));
        RTK_CUDA_TRY(cudaMemcpy(p.par_tab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
        for (int k = 0; k < 4; ++k)
            if (!encode_f64_map(&p.tma_qmap[k], p.par_tab + k * len, 1, dd, nullptr, db))
                return set_error(RTK_ECUDA, "sweep: exp-parabolic table tensor map");
    }
    RTK_CUDA_TRY(cudaMalloc(&p.tma_ctas, sizeof(TmaCta) * ctas.size()));
    RTK_CUDA_TRY(cudaMemcpy(p.tma_ctas, ctas.data(), sizeof(TmaCta) * ctas.size(), cudaMemcpyHostToDevice));
    p.tma_n_ctas = static_cast<int>(ctas.size());
    p.tma_ready = true;
    return RTK_OK;
}

}  // namespace rtk
