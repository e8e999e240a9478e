// K2 fused: angular moments + dense redistribution in ONE kernel, so the HBM
// stream of the intensity vector (K2a) overlaps the FP64 tensor-pipe GEMM (K2b)
// instead of running after it (R/scattering.py:126-148 for the operator;
// sigma.cu for the unfused pair, which stays the general path).
//
//   m[i,k,g] = sum_a w_a Y_k(a) x[i,a,g]                (reduction over directions)
//   G[i,k,f] = c_k gamma[i,f] sum_g R[f,g] w_g m[i,k,g]  (DMMA, K = n_freq)
//
// Work decomposition (n_mom = 2, n_freq = 128 * CN, CN = 1..4):
// * a thread-block CLUSTER of CN CTAs owns an M block of SP space points (GEMM rows
//   2 SP of an 8 MT-row block; SP is chosen per problem so the blocks split evenly
//   over the co-resident clusters) and the whole frequency range; CTA rank r
//   computes output columns [BN r, BN r + BN).  Two shapes: BN = 128 with up to 31
//   points (default), and BN = 256 with up to 16 points (clusters half as large,
//   opt-in: measured slower);
// * K (= source frequency g) is walked in KT = BN / 8 steps of BK = 8 CN columns.  In
//   each step CTA r reduces ITS 8 columns of x for the SP points: a producer lane
//   streams x[SP points][16 directions][8 columns] boxes with TMA into a ring (no
//   register staging), 8 reducer warps sum the directions into the 64 x 8 moment
//   slice, which is written into the CTA's A stage and pushed to the other CTAs of
//   the cluster with bulk DSMEM copies that complete on their a_full mbarriers;
// * the producer warp's second lane streams the R^T tile of the step (BK x 128, L2-resident) with
//   TMA (128-byte swizzle: one 16-column box per MMA warp, conflict-light
//   fragment loads);
// * 8 MMA warps wait a_full / b_full, run m8n8k4 f64 MMAs (each warp 64 rows x 16
//   columns) and release the stages through mbarriers (a_empty cluster-wide);
// * clusters are persistent over M blocks (grid = co-resident clusters).
// No named barriers on the MMA side: every hand-off is an mbarrier, so the three
// streams (x, R, MMA) drift independently within the ring depths.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "rtk_internal.cuh"
#include "tma.cuh"

namespace rtk {
namespace {
namespace fused {

constexpr int NM = 2;
constexpr int KS = 8;                  // source columns reduced per CTA per K step
constexpr int PA = KS;                 // A slice row pitch; columns XOR-swizzled by 4 on rows with bit 1 set
constexpr int AC = 16;                 // directions per x box
// 16 warps = 4 per SM sub-partition, so the register cap is 128 (17 warps would cap it at 96)
constexpr int MMA_WARPS = 8, RED_WARPS = 7;
constexpr int THREADS = 32 * (MMA_WARPS + RED_WARPS + 1);   // + producer warp (lane 0: x, lane 1: R^T)
constexpr int RED0 = 32 * MMA_WARPS;   // first reducer thread
constexpr int XPROD = 32 * (MMA_WARPS + RED_WARPS);
constexpr int BPROD = XPROD + 1;
constexpr int MAX_ANGLES = 256;
constexpr unsigned kMmaNapNs = 200;    // see the MMA loop
constexpr size_t kSmemLimit = 232448;

// Variant: CN CTAs per cluster, MT m8 tiles of GEMM rows (2 SP <= 8 MT), NT n8 tiles per
// MMA warp (BN = 64 NT output columns per CTA).  (CN, 8, 2): 31 points x 128 columns;
// (CN, 4, 4): 16 points x 256 columns -- half the cluster size for the same N_nu, so
// clusters of 2 tile every GPC (all 148 SMs) where clusters of 4 leave 16 SMs idle.
template <int CN, int MT_, int NT_>
struct Cfg {
    static constexpr int MT = MT_, NT = NT_;
    static constexpr int ROWS = 8 * MT;                      // rows >= 2 SP are computed but never stored
    static constexpr int SPMAX = MT == 8 ? 31 : 4 * MT;      // space points per M block (runtime SP <= SPMAX)
    static constexpr int NSP = (SPMAX + RED_WARPS - 1) / RED_WARPS;   // points per reducer warp
    static constexpr int BN = 8 * NT * MMA_WARPS;            // output columns per CTA
    static constexpr int KT = BN / KS;                       // K steps (n_freq = BN CN, BK = KS CN)
    static constexpr int SLICE = ROWS * PA;                  // doubles per A slice
    static constexpr int XBOX = KS * AC * SPMAX;             // doubles per x ring slot
    static constexpr int XS = MT == 8 ? 4 : 6;               // x ring stages
    static constexpr int AS = MT == 8 ? 2 : 4;               // A ring stages
    static constexpr int BS = MT == 8 ? 2 : 3;               // R^T tile ring stages
    static constexpr int BK = KS * CN;
    static constexpr size_t a_elems = static_cast<size_t>(CN) * SLICE;   // one A stage
    static constexpr size_t b_elems = static_cast<size_t>(BK) * BN;      // one R^T stage (BN / 16 swizzled boxes)
    static size_t smem_bytes(int n_apad) {
        return 1024 /* alignment slack */ +
               sizeof(double) * (BS * b_elems + static_cast<size_t>(XS) * XBOX + AS * a_elems +
                                 NM * static_cast<size_t>(n_apad)) +
               2 * (AS + XS + BS) * sizeof(uint64_t);
    }
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_rank(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t remote_bar) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void bulk_to_peer(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t remote_bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "r"(src), "r"(bytes), "r"(remote_bar)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void red_bar() { asm volatile("bar.sync 2, %0;\n" ::"n"(32 * RED_WARPS) : "memory"); }
__device__ __forceinline__ void mma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int CN, int MT_, int NT_>
__global__ void __launch_bounds__(THREADS, 1)
    sigma_fused_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap rmap,
                       const double* __restrict__ wy, const double* __restrict__ gamma,
                       const double* __restrict__ coeffs, double* __restrict__ G, int n_space, int n_angles, int fp,
                       int gamma_mode, int SP) {
    using C = Cfg<CN, MT_, NT_>;
    constexpr int BK = C::BK, MT = C::MT, NT = C::NT, BN = C::BN, KT = C::KT, SLICE = C::SLICE, XBOX = C::XBOX;
    // let the sweep (launched with programmatic stream serialization) start its prologue on
    // free SMs; it waits (griddepcontrol.wait) for this grid before reading G
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    constexpr int XS = C::XS, AS = C::AS, BS = C::BS, NSP = C::NSP;
    const int n_freq = BN * CN;
    const int n_chunks = (n_angles + AC - 1) / AC;
    const int n_apad = n_chunks * AC;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment (swizzled TMA boxes) as an OFFSET on the shared array, so the compiler
    // keeps the shared address space and emits LDS / STS (rounding the pointer through an integer
    // made every fragment and x load a generic LD.E on the long scoreboard)
    double* Bs = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u));
    double* Xs = Bs + BS * C::b_elems;                  // [XS][SP][AC][KS]    (TMA boxes, slot pitch XBOX)
    double* As = Xs + XS * XBOX;                        // [AS][CN][ROWS][PA]  (slice r from CTA r)
    double* wys = As + AS * C::a_elems;                 // [NM][n_apad] (zero padded)
    uint64_t* bars = reinterpret_cast<uint64_t*>(wys + NM * n_apad);
    uint64_t* a_full = bars;                            // [AS] 1 arrival (+ tx of the CN-1 peer slices)
    uint64_t* a_empty = a_full + AS;                    // [AS] CN * 8 arrivals (MMA warps of the cluster)
    uint64_t* x_full = a_empty + AS;                    // [XS] TMA tx
    uint64_t* x_empty = x_full + XS;                    // [XS] 8 arrivals (reducer warps)
    uint64_t* b_full = x_empty + XS;                    // [BS] TMA tx
    uint64_t* b_empty = b_full + BS;                    // [BS] 8 arrivals (MMA warps)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int cid = blockIdx.x / CN, ncl = gridDim.x / CN;
    const int nblk = (n_space + SP - 1) / SP;
    const int my_blocks = cid < nblk ? (nblk - 1 - cid) / ncl + 1 : 0;
    const int total = my_blocks * KT;

    for (int t = tid; t < NM * n_apad; t += THREADS) {
        const int k = t / n_apad, a = t - k * n_apad;
        wys[t] = a < n_angles ? wy[k * n_angles + a] : 0.0;
    }
    if (tid == 0) {
        for (int s = 0; s < AS; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], CN * MMA_WARPS);
        }
        for (int s = 0; s < XS; ++s) {
            mbar_init(&x_full[s], 1);
            mbar_init(&x_empty[s], RED_WARPS);
        }
        for (int s = 0; s < BS; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], MMA_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __syncthreads();
    cluster_sync_all();   // peers' barriers are initialised before anyone signals them

    if (tid == XPROD) {
        // ---------------- producer X: x boxes [SP][AC][KS] ----------------
        prefetch_tensormap(&xmap);
        const uint64_t pol = policy_evict_first();   // x is streamed once; keep R^T and gamma in L2
        int it = 0;
        for (int n = 0; n < total; ++n) {
            const int blk = cid + (n / KT) * ncl, j = n % KT;
            for (int c = 0; c < n_chunks; ++c, ++it) {
                const int st = it % XS;
                if (it >= XS) mbar_wait(&x_empty[st], ((it / XS) + 1) & 1);
                mbar_arrive_expect_tx(&x_full[st], KS * AC * SP * sizeof(double));
                tma_load_3d_hint(Xs + st * XBOX, &xmap, j * BK + static_cast<int>(rank) * KS, c * AC, blk * SP,
                                 &x_full[st], pol);
            }
        }
    } else if (tid == BPROD) {
        // ---------------- producer B: R^T tile of the step, 8 swizzled 16-column boxes ----------------
        prefetch_tensormap(&rmap);
        for (int n = 0; n < total; ++n) {
            const int st = n % BS, j = n % KT;
            if (n >= BS) mbar_wait(&b_empty[st], ((n / BS) + 1) & 1);
            mbar_arrive_expect_tx(&b_full[st], C::b_elems * sizeof(double));
            for (int bx = 0; bx < BN / 16; ++bx)
                tma_load_2d(Bs + st * C::b_elems + bx * 16 * BK, &rmap, static_cast<int>(rank) * BN + bx * 16,
                            j * BK, &b_full[st]);
        }
    } else if (warp >= MMA_WARPS && warp < MMA_WARPS + RED_WARPS) {
        // ---------------- reducers: x boxes -> 64 x 8 moment slice -> cluster A stages ----------------
        const int rw = warp - MMA_WARPS;
        const int aq = lane >> 3, f = lane & 7;
        const int nsp = (SP - rw + RED_WARPS - 1) / RED_WARPS;   // local points rw, rw + RED_WARPS, ... below SP
        int it = 0;
        for (int n = 0; n < total; ++n) {
            const int buf = n % AS;
            double acc[NSP][NM];
#pragma unroll
            for (int s = 0; s < NSP; ++s) acc[s][0] = acc[s][1] = 0.0;
            for (int c = 0; c < n_chunks; ++c, ++it) {
                const int st = it % XS;
                mbar_wait(&x_full[st], (it / XS) & 1);
                const double* xb = Xs + st * XBOX;
                const double* w0 = wys + c * AC;
                const double* w1 = wys + n_apad + c * AC;
#pragma unroll
                for (int t = 0; t < AC / 4; ++t) {
                    const int a = aq + 4 * t;
                    const double wa = w0[a], wb = w1[a];
#pragma unroll
                    for (int s = 0; s < NSP; ++s) {
                        if (s < nsp) {
                            const double v = xb[((rw + RED_WARPS * s) * AC + a) * KS + f];
                            acc[s][0] = fma(wa, v, acc[s][0]);
                            acc[s][1] = fma(wb, v, acc[s][1]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&x_empty[st]);
            }
#pragma unroll
            for (int s = 0; s < NSP; ++s)
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    acc[s][k] += __shfl_xor_sync(0xffffffffu, acc[s][k], 8);
                    acc[s][k] += __shfl_xor_sync(0xffffffffu, acc[s][k], 16);
                }
            // the A stage is free once every MMA warp of the cluster has consumed step n - AS and
            // the bulk copies of our slice from step n - AS have been read out
            if (n >= AS) mbar_wait(&a_empty[buf], ((n / AS) + 1) & 1);
            if (tid == RED0) asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(AS - 1) : "memory");
            red_bar();
            double* slice = As + buf * C::a_elems + rank * SLICE;
            if (aq == 0) {
#pragma unroll
                for (int s = 0; s < NSP; ++s)
                    if (s < nsp) {
                        const int r = 2 * (rw + RED_WARPS * s);   // rows r, r + 1 share the swizzle (bit 1)
                        const int cs = f ^ (((r >> 1) & 1) << 2);
                        slice[r * PA + cs] = acc[s][0];
                        slice[(r + 1) * PA + cs] = acc[s][1];
                    }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            red_bar();
            if (tid == RED0) {
                const uint32_t src = smem_addr(slice);
#pragma unroll
                for (int d = 1; d < CN; ++d) {
                    const uint32_t peer = (rank + d) % CN;
                    bulk_to_peer(map_rank(src, peer), src, SLICE * sizeof(double),
                                 map_rank(smem_addr(&a_full[buf]), peer));
                }
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                mbar_arrive_expect_tx(&a_full[buf], (CN - 1) * SLICE * sizeof(double));
            }
        }
        if (tid == RED0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    } else if (warp < MMA_WARPS) {
        // ---------------- MMA warps: G tile (ROWS x BN) += A (ROWS x BK) * R^T tile (BK x BN) ----------------
        const int g = lane >> 2, q = lane & 3;
        const int col_w = warp * 8 * NT;              // = swizzled boxes warp NT/2 .. of the R^T stage
        const int sw = ((g >> 1) & 1) << 2;           // A-slice column swizzle of rows 8 i + g
        // fragment offsets for the two kk % 8 phases (0, 4): A slice column and swizzled R^T chunk
        const int aoff0 = q ^ sw, aoff1 = (4 + q) ^ sw;
        const int boff00 = ((g >> 1) ^ q) << 1, boff01 = ((4 + (g >> 1)) ^ q) << 1;
        const int boff10 = ((g >> 1) ^ (4 + q)) << 1, boff11 = ((4 + (g >> 1)) ^ (4 + q)) << 1;
        double acc[MT][NT][2];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int jn = 0; jn < NT; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;
        for (int n = 0; n < total; ++n) {
            const int j = n % KT, bst = n % BS, buf = n % AS;
            mbar_wait(&b_full[bst], (n / BS) & 1);
            mbar_wait(&a_full[buf], (n / AS) & 1);
            const double* abuf = As + buf * C::a_elems + g * PA;
            const double* bbox = Bs + bst * C::b_elems + warp * (NT / 2) * 16 * BK + q * 16 + (g & 1);
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                // R^T row kk + q of the box, 128-byte swizzle on (kk + q) % 8 = (kk & 4) + q
                const bool hi = (kk & 4) != 0;
                const double* as = abuf + (kk / KS) * SLICE + (hi ? aoff1 : aoff0);
                const double* br = bbox + kk * 16;
                double af[MT], bf[NT];
#pragma unroll
                for (int i = 0; i < MT; ++i) af[i] = as[i * 8 * PA];
#pragma unroll
                for (int jn = 0; jn < NT; ++jn)   // n8 tile jn: box jn / 2, chunk half jn % 2
                    bf[jn] = br[(jn >> 1) * 16 * BK + ((jn & 1) ? (hi ? boff11 : boff01) : (hi ? boff10 : boff00))];
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int jn = 0; jn < NT; ++jn) mma(acc[i][jn], af[i], bf[jn]);
                // FP64-pipe fairness: DMMA and the reducers' DFMA share one pipe per SM sub-partition,
                // and two MMA warps issuing back-to-back DMMAs (16 cycles each) starve the reducer
                // warps, so the next A slice is produced only while the MMA warps wait for it (ncu:
                // reducers stalled on `math`, MMA warps 38% on a_full).  A 200 ns nap after every
                // 32 DMMAs of a warp hands the pipe to the reducers: 140.0 -> 131.0 us at cfg2
                // (measured: 20-300 ns and adaptive naps within 1%, every 16 DMMAs or 600 ns slower).
                if ((kk + 4) % 8 == 0) __nanosleep(kMmaNapNs);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&b_empty[bst]);
#pragma unroll
                for (int d = 0; d < CN; ++d) arrive_remote(map_rank(smem_addr(&a_empty[buf]), d));
            }
            if (j == KT - 1) {
                const int blk = cid + (n / KT) * ncl;
                // epilogue: G[i,k,f] = c_k (gamma[i,f]) acc, two m-tiles at a time so the gamma
                // loads of a group are in flight together
#pragma unroll
                for (int i0 = 0; i0 < MT; i0 += 2) {
                    double2 gm[2][NT];
#pragma unroll
                    for (int di = 0; di < 2; ++di) {
                        const int r = (i0 + di) * 8 + g;
                        const int sp = blk * SP + (r >> 1);
                        const bool ok = gamma_mode && (r >> 1) < SP && sp < n_space;
#pragma unroll
                        for (int jn = 0; jn < NT; ++jn) {
                            const int col = static_cast<int>(rank) * BN + col_w + jn * 8 + 2 * q;
                            gm[di][jn] = ok ? __ldg(reinterpret_cast<const double2*>(
                                                  gamma + static_cast<int64_t>(sp) * n_freq + col))
                                            : make_double2(1.0, 1.0);
                        }
                    }
#pragma unroll
                    for (int di = 0; di < 2; ++di) {
                        const int i = i0 + di;
                        const int r = i * 8 + g;
                        const int sp = blk * SP + (r >> 1), k = r & 1;
                        if ((r >> 1) < SP && sp < n_space) {
                            const double ck = coeffs[k];
#pragma unroll
                            for (int jn = 0; jn < NT; ++jn) {
                                const int col = static_cast<int>(rank) * BN + col_w + jn * 8 + 2 * q;
                                *reinterpret_cast<double2*>(G + (static_cast<int64_t>(sp) * NM + k) * fp + col) =
                                    make_double2(ck * acc[i][jn][0] * gm[di][jn].x, ck * acc[i][jn][1] * gm[di][jn].y);
                            }
                        }
#pragma unroll
                        for (int jn = 0; jn < NT; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;
                    }
                }
            }
        }
    }
    __syncwarp();
    cluster_sync_all();   // no CTA leaves while peers may still copy into / signal its shared memory
}

template <int CN, int MT, int NT>
int launch_t(const Problem& p, const double* x, cudaStream_t s) {
    using C = Cfg<CN, MT, NT>;
    auto kernel = sigma_fused_kernel<CN, MT, NT>;
    const int n_apad = (p.n_angles + AC - 1) / AC * AC;
    const size_t smem = C::smem_bytes(n_apad);
    if (smem > kSmemLimit) return -1;
    // co-resident clusters of this instantiation at this smem size, per device
    const int cache_slot = static_cast<int>(smem);
    int max_clusters = device_cache_get(reinterpret_cast<const void*>(kernel), cache_slot);
    if (max_clusters <= 0) {
        if (int rc = ensure_smem_for(kernel, smem)) return rc;
        cudaLaunchConfig_t qc = {};
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = CN;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.gridDim = dim3(CN * 148);
        qc.blockDim = dim3(THREADS);
        qc.dynamicSmemBytes = smem;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int nc = 0;
        RTK_CUDA_TRY(cudaOccupancyMaxActiveClusters(&nc, kernel, &qc));
        if (nc <= 0) return -1;   // this cluster shape cannot be resident on the device
        max_clusters = nc;
        device_cache_put(reinterpret_cast<const void*>(kernel), cache_slot, nc);
    }
    // block size: the fewest rounds over the co-resident clusters, then the smallest SP
    // that keeps that round count (balanced blocks), then as few clusters as possible
    const int64_t rounds = (p.n_space + static_cast<int64_t>(C::SPMAX) * max_clusters - 1) /
                           (static_cast<int64_t>(C::SPMAX) * max_clusters);
    const int sp = static_cast<int>((p.n_space + rounds * max_clusters - 1) / (rounds * max_clusters));
    const int nblk = static_cast<int>((p.n_space + sp - 1) / sp);
    const int ncl = static_cast<int>((nblk + rounds - 1) / rounds);
    CUtensorMap xmap, rmap;
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(p.n_freq), static_cast<uint64_t>(p.n_angles),
                                  static_cast<uint64_t>(p.n_space)};
        const uint64_t strides[2] = {sizeof(double) * p.n_freq, sizeof(double) * p.n_rays};
        const uint32_t box[3] = {KS, AC, static_cast<uint32_t>(sp)};
        if (!encode_f64_map(&xmap, x, 3, dims, strides, box)) return set_error(RTK_ECUDA, "sigma: x tensor map");
        const uint64_t rd[2] = {static_cast<uint64_t>(p.fp), static_cast<uint64_t>(p.n_freq)};
        const uint32_t rb[2] = {16, static_cast<uint32_t>(C::BK)};
        if (!encode_f64_map_sw128(&rmap, p.rwt, rd, sizeof(double) * p.fp, rb))
            return set_error(RTK_ECUDA, "sigma: R tensor map");
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CN;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CN * ncl);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RTK_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, xmap, rmap, static_cast<const double*>(p.wy),
                                    static_cast<const double*>(p.gamma), static_cast<const double*>(p.coeffs), p.gmom,
                                    static_cast<int>(p.n_space), p.n_angles, p.fp, p.gamma_per_ray ? 0 : 1, sp));
    RTK_LAUNCH_CHECK("sigma_fused_kernel");
    return RTK_OK;
}

}  // namespace fused
}  // namespace

// -1: shape not covered (caller runs the unfused moments + redistribution pair)
int launch_sigma_fused(const Problem& p, const double* x, cudaStream_t s) {
    if (p.kind != KIND_SLAB && p.kind != KIND_LATTICE) return -1;
    if (p.n_mom != fused::NM || p.n_freq % 128 != 0 || p.fp != p.n_freq) return -1;
    if (p.n_angles > fused::MAX_ANGLES || p.n_space > (1 << 30)) return -1;
    if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return -1;
    if (p.tune.sigma_unfused) return -1;
    // 128-column CTAs (clusters of N_nu / 128).  A 256-column shape (clusters of N_nu / 256,
    // tiling all 148 SMs) measured slower on cfg2 (166 vs 146 us: twice the K steps per
    // block, each with a cluster hand-off) and was removed.
    switch (p.n_freq / 128) {
        case 1: return fused::launch_t<1, 8, 2>(p, x, s);
        case 2: return fused::launch_t<2, 8, 2>(p, x, s);
        case 3: return fused::launch_t<3, 8, 2>(p, x, s);
        case 4: return fused::launch_t<4, 8, 2>(p, x, s);
        default: return -1;
    }
}

// Sigma up to the source moments G: fused kernel where it applies, else K2a + K2b.
int launch_sigma(const Problem& p, const double* x, cudaStream_t s) {
    const int rc = launch_sigma_fused(p, x, s);
    if (rc != -1) return rc;
    if (int r = launch_moments(p, x, s)) return r;
    return launch_redistribute(p, s);
}

}  // namespace rtk
