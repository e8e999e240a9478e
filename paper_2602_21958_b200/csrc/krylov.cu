// K3: Krylov solvers on device vectors.  GMRES and BiCGStab with the
// reference's exact control flow (R/krylov.py:56-256); the vectors (Krylov
// basis, iterate, residual) stay in HBM and only scalars cross to the host.
//
// Arnoldi orthogonalisation (rtk_solve_cfg.orthogonalization):
//  * MGS / MGS2 -- the reference's modified Gram-Schmidt (R/krylov.py:98-104), one
//    sweep, or two with reorthogonalize=True: one streaming pass per basis vector,
//    pass i  w <- w - h_{i-1} v_{i-1} ; h_i = v_i . w   (h_{i-1} read on the device);
//  * CGS2 -- classical Gram-Schmidt with one reorthogonalisation pass, fused into
//    three streaming passes over the whole basis:
//      pass 1  h1 = V^T w
//      pass 2  w <- w - V h1 ;  h2 = V^T w          (same sweep over V)
//      pass 3  w <- w - V h2 ;  ||w||^2
// followed by v_{j+1} = w / ||w||.  Every reduction is a fixed-shape
// two-level tree (warp shuffle -> block -> last-block serial sum over block
// partials in index order), so results are bitwise reproducible run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <new>
#include <vector>

#include "rtk_internal.cuh"

namespace rtk {
namespace {

constexpr int kRedThreads = 256;
constexpr int kMaxRedBlocks = 592;   // 4 x 148 SMs
constexpr int KMAX = 32;             // basis vectors handled per pass (restart <= 31 runs fully fused)
constexpr int kFinChunk = 64;        // block partials staged per round trip by the last block
constexpr int kLookahead = 3;        // Arnoldi iterations the device may run ahead of the host

enum PassMode { MODE_DOT = 0, MODE_UPDATE_DOT = 1, MODE_UPDATE_NORM = 2, MODE_UPDATE = 3 };

}  // namespace

struct KrylovWorkspace {
    double* partials = nullptr;      // [KMAX][kMaxRedBlocks]
    unsigned* counter = nullptr;
    double* dev_scalars = nullptr;   // device-side coefficient / result scratch
    double* pinned = nullptr;        // host pinned scratch
    int dev_cap = 0, pin_cap = 0;
    double* look_dev = nullptr;      // GMRES look-ahead column slots (device / pinned host)
    double* look_pin = nullptr;
    int look_cap = 0;
    int device = -1;                 // the device the buffers live on
    ~KrylovWorkspace() {
        if (partials) cudaFree(partials);
        if (counter) cudaFree(counter);
        if (dev_scalars) cudaFree(dev_scalars);
        if (pinned) cudaFreeHost(pinned);
        if (look_dev) cudaFree(look_dev);
        if (look_pin) cudaFreeHost(look_pin);
    }
    int reserve_look(int count) {
        if (count <= look_cap) return RTK_OK;
        if (look_dev) cudaFree(look_dev);
        if (look_pin) cudaFreeHost(look_pin);
        look_dev = nullptr;
        look_pin = nullptr;
        look_cap = 0;
        RTK_CUDA_TRY(cudaMalloc(&look_dev, sizeof(double) * count * 2));
        RTK_CUDA_TRY(cudaMallocHost(&look_pin, sizeof(double) * count * 2));
        look_cap = count * 2;
        return RTK_OK;
    }
    int init() {
        RTK_CUDA_TRY(cudaGetDevice(&device));
        RTK_CUDA_TRY(cudaMalloc(&partials, sizeof(double) * KMAX * kMaxRedBlocks));
        RTK_CUDA_TRY(cudaMalloc(&counter, sizeof(unsigned)));
        RTK_CUDA_TRY(cudaMemset(counter, 0, sizeof(unsigned)));
        if (int rc = reserve_scalars(4 * KMAX)) return rc;
        return reserve_pinned(4 * KMAX);
    }
    int reserve_scalars(int count) {
        if (count <= dev_cap) return RTK_OK;
        if (dev_scalars) cudaFree(dev_scalars);
        dev_cap = count * 2;
        RTK_CUDA_TRY(cudaMalloc(&dev_scalars, sizeof(double) * dev_cap));
        return RTK_OK;
    }
    int reserve_pinned(int count) {
        if (count <= pin_cap) return RTK_OK;
        if (pinned) cudaFreeHost(pinned);
        pin_cap = count * 2;
        RTK_CUDA_TRY(cudaMallocHost(&pinned, sizeof(double) * pin_cap));
        return RTK_OK;
    }
};

void destroy_krylov_workspace(KrylovWorkspace* w) { delete w; }

namespace {

// one full wave: 148 SMs x resident blocks of the pass kernel for this bucket size
int red_blocks(int64_t n, int kb = 4) {
    const int per_sm = kb <= 8 ? 4 : (kb <= 16 ? 2 : 1);
    int64_t b = (n + kRedThreads * 4 - 1) / (kRedThreads * 4);
    if (b < 1) b = 1;
    if (b > 148 * per_sm) b = 148 * per_sm;
    return static_cast<int>(b);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order reduction of nk per-thread accumulators over the grid: warp shuffle ->
// block (warp order) -> block partials; the last block to arrive sums the partials in
// block-index order and writes out[0..nk).  Bitwise reproducible for a given grid size.
template <int NACC>
__device__ __forceinline__ void block_reduce_finish(const double* acc, int nk, double* partials, unsigned* counter,
                                                    double* out) {
    __shared__ double red[kRedThreads / 32][KMAX];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NACC; ++k) {
        if (k < nk) {
            const double s = warp_sum(acc[k]);
            if (lane == 0) red[warp][k] = s;
        }
    }
    __syncthreads();
    if (threadIdx.x < nk) {
        double s = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) s += red[w][threadIdx.x];
        partials[threadIdx.x * kMaxRedBlocks + blockIdx.x] = s;
    }
    // last block to finish sums the block partials in index order
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned ticket = atomicAdd(counter, 1u);
        is_last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        // the partials are staged in shared memory 64 blocks at a time by the whole block (one
        // L2 round trip per chunk instead of one per 8 blocks), then thread k sums row k in
        // block-index order: the same sequential sum, so results do not depend on the staging
        __shared__ double fin[KMAX][kFinChunk + 1];
        const unsigned nb = gridDim.x;
        double total = 0.0;
        for (unsigned b0 = 0; b0 < nb; b0 += kFinChunk) {
            const unsigned cnt = min(static_cast<unsigned>(kFinChunk), nb - b0);
#pragma unroll 8
            for (int e = threadIdx.x; e < nk * kFinChunk; e += kRedThreads) {
                const int k = e / kFinChunk, bb = e - k * kFinChunk;
                if (bb < static_cast<int>(cnt)) fin[k][bb] = __ldcg(partials + k * kMaxRedBlocks + b0 + bb);
            }
            __syncthreads();
            if (threadIdx.x < nk)
                for (unsigned bb = 0; bb < cnt; ++bb) total += fin[threadIdx.x][bb];
            __syncthreads();
        }
        if (threadIdx.x < nk) out[threadIdx.x] = total;
        if (threadIdx.x == 0) *counter = 0u;
    }
}

struct PassArgs {
    const double* v[KMAX];      // basis vectors of this pass
    int kc;                     // how many of them
    const double* coef;         // device coefficients (update modes), length kc
    double* w;                  // vector updated in place (update modes) / read (dot)
    const double* x;            // second operand for MODE_DOT when w is null... (unused)
    int64_t n;
    double* partials;
    unsigned* counter;
    double* out;                // device results: kc dots, or 1 norm^2
};

// KB = compile-time bucket >= kc: all KB loads of an element are issued back to back
// (predicated off beyond kc), so each thread keeps KB independent requests in flight.
template <int MODE, int KB, int VEC>
__global__ void __launch_bounds__(kRedThreads) cgs_pass_kernel(PassArgs P) {
    constexpr int NACC = (MODE == MODE_UPDATE_NORM) ? 1 : KB;
    // programmatic dependent launch: this grid may start while its predecessor drains; wait
    // for the predecessor's completion before any global access, and let the next pass launch
    pdl_prologue();
    __shared__ double coef[KMAX];
    if (threadIdx.x < KMAX) coef[threadIdx.x] = (MODE != MODE_DOT && threadIdx.x < P.kc) ? P.coef[threadIdx.x] : 0.0;
    __syncthreads();
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;

    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (VEC == 2) {
        // element pairs: 16-byte loads halve the load instructions per byte (all operands 16-byte aligned)
        const int64_t n2 = P.n >> 1;
        for (int64_t e = t0; e < n2; e += stride) {
            double2 vv[KB];
#pragma unroll
            for (int k = 0; k < KB; ++k)
                vv[k] = (k < P.kc) ? __ldg(reinterpret_cast<const double2*>(P.v[k]) + e) : make_double2(0.0, 0.0);
            double2 we = reinterpret_cast<double2*>(P.w)[e];
            if (MODE != MODE_DOT) {
#pragma unroll
                for (int k = 0; k < KB; ++k) {
                    we.x = fma(-coef[k], vv[k].x, we.x);
                    we.y = fma(-coef[k], vv[k].y, we.y);
                }
                reinterpret_cast<double2*>(P.w)[e] = we;
            }
            if (MODE == MODE_UPDATE_NORM) {
                acc[0] = fma(we.x, we.x, acc[0]);
                acc[0] = fma(we.y, we.y, acc[0]);
            } else if (MODE != MODE_UPDATE) {
#pragma unroll
                for (int k = 0; k < KB; ++k) {
                    acc[k] = fma(vv[k].x, we.x, acc[k]);
                    acc[k] = fma(vv[k].y, we.y, acc[k]);
                }
            }
        }
    }
    // scalar elements: everything (VEC == 1) or the odd tail element (VEC == 2)
    for (int64_t e = (VEC == 2 ? (P.n & ~int64_t(1)) + t0 : t0); e < P.n; e += stride) {
        double vv[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) vv[k] = (k < P.kc) ? __ldg(P.v[k] + e) : 0.0;
        double we = P.w[e];
        if (MODE != MODE_DOT) {
#pragma unroll
            for (int k = 0; k < KB; ++k) we = fma(-coef[k], vv[k], we);
            P.w[e] = we;
        }
        if (MODE == MODE_UPDATE_NORM) {
            acc[0] = fma(we, we, acc[0]);
        } else if (MODE != MODE_UPDATE) {
#pragma unroll
            for (int k = 0; k < KB; ++k) acc[k] = fma(vv[k], we, acc[k]);
        }
    }
    if (MODE == MODE_UPDATE) return;
    block_reduce_finish<NACC>(acc, (MODE == MODE_UPDATE_NORM) ? 1 : P.kc, P.partials, P.counter, P.out);
}

// One modified Gram-Schmidt step (R/krylov.py:98-104, one basis vector per pass):
//   MGS_DOT          out = d . w                         (first vector of a sweep)
//   MGS_UPDATE_DOT   w <- w - (*coef) u ;  out = d . w   (finish v_{i-1}, start v_i)
//   MGS_UPDATE_NORM  w <- w - (*coef) u ;  out = ||w||^2 (last vector)
// The coefficient is the previous pass's result, read on the device (no host round trip).
enum MgsMode { MGS_DOT = 0, MGS_UPDATE_DOT = 1, MGS_UPDATE_NORM = 2 };
struct MgsArgs {
    const double* u;       // vector to subtract (update modes)
    const double* coef;    // its coefficient, device
    const double* d;       // vector to dot with (dot modes)
    double* w;
    int64_t n;
    double* partials;
    unsigned* counter;
    double* out;
};

template <int MODE, int VEC>
__global__ void __launch_bounds__(kRedThreads) mgs_pass_kernel(MgsArgs P) {
    pdl_prologue();
    const double c = (MODE == MGS_DOT) ? 0.0 : *P.coef;
    double acc[1] = {0.0};
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (VEC == 2) {
        const int64_t n2 = P.n >> 1;
        for (int64_t e = t0; e < n2; e += stride) {
            double2 we = reinterpret_cast<double2*>(P.w)[e];
            if (MODE != MGS_DOT) {
                const double2 uu = __ldg(reinterpret_cast<const double2*>(P.u) + e);
                we.x = fma(-c, uu.x, we.x);
                we.y = fma(-c, uu.y, we.y);
                reinterpret_cast<double2*>(P.w)[e] = we;
            }
            if (MODE == MGS_UPDATE_NORM) {
                acc[0] = fma(we.x, we.x, acc[0]);
                acc[0] = fma(we.y, we.y, acc[0]);
            } else {
                const double2 dd = __ldg(reinterpret_cast<const double2*>(P.d) + e);
                acc[0] = fma(dd.x, we.x, acc[0]);
                acc[0] = fma(dd.y, we.y, acc[0]);
            }
        }
    }
    for (int64_t e = (VEC == 2 ? (P.n & ~int64_t(1)) + t0 : t0); e < P.n; e += stride) {
        double we = P.w[e];
        if (MODE != MGS_DOT) {
            we = fma(-c, __ldg(P.u + e), we);
            P.w[e] = we;
        }
        acc[0] = (MODE == MGS_UPDATE_NORM) ? fma(we, we, acc[0]) : fma(__ldg(P.d + e), we, acc[0]);
    }
    block_reduce_finish<1>(acc, 1, P.partials, P.counter, P.out);
}

// y = a * x  (a read from device: 1/sqrt(norm2) or a host scalar)
__global__ void scale_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n, double a,
                             const double* __restrict__ norm2) {
    pdl_prologue();
    // an exactly zero norm (Arnoldi breakdown) gives a zero vector instead of 0/0 = NaN: a
    // look-ahead iteration enqueued past a breakdown then runs on finite data
    const double s = norm2 ? sqrt(*norm2) : a;
    const double r = s != 0.0 ? 1.0 / s : 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // 16-byte accesses, four in flight per thread (one 8-byte load per iteration left the
    // kernel latency-bound at 4.3 TB/s in ncu); the division keeps numpy's v = w / h bits
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
    const int64_t n2 = vec ? n / 2 : 0;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    double2* y2 = reinterpret_cast<double2*>(y);
    int64_t e = tid;
    for (; e + 3 * stride < n2; e += 4 * stride) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(x2 + e + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            v[u].x = s != 0.0 ? v[u].x / s : v[u].x * r;
            v[u].y = s != 0.0 ? v[u].y / s : v[u].y * r;
            y2[e + u * stride] = v[u];
        }
    }
    for (; e < n2; e += stride) {
        double2 v = x2[e];
        v.x = s != 0.0 ? v.x / s : v.x * r;
        v.y = s != 0.0 ? v.y / s : v.y * r;
        y2[e] = v;
    }
    for (int64_t k = 2 * n2 + tid; k < n; k += stride) y[k] = s != 0.0 ? x[k] / s : x[k] * r;
}

// out = base + sum_k y_k V_k  (the reference's _combine, R/krylov.py:173-177, added to x)
struct CombineArgs {
    const double* v[KMAX];
    double y[KMAX];
    int kc;
    const double* base;   // may be null (then 0)
    double* out;
    int64_t n;
};
__global__ void combine_kernel(CombineArgs C) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < C.n; e += stride) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (k < C.kc) s = fma(C.y[k], __ldg(C.v[k] + e), s);
        C.out[e] = (C.base ? C.base[e] : 0.0) + s;
    }
}

// out = a - b
__global__ void sub_kernel(const double* a, const double* b, double* out,
                           int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride) out[e] = a[e] - b[e];
}

// BiCGStab updates (R/krylov.py:211-233), same operation order as numpy
__global__ void bicg_p_kernel(const double* __restrict__ r, double* __restrict__ p, const double* __restrict__ v,
                              double beta, double omega, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride)
        p[e] = r[e] + beta * (p[e] - omega * v[e]);
}
__global__ void axpy_out_kernel(const double* x, double a, const double* y,
                                double* out, int64_t n) {   // out = x + a*y
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride)
        out[e] = x[e] + a * y[e];
}
__global__ void bicg_x_kernel(double* __restrict__ x, double alpha, const double* __restrict__ p, double omega,
                              const double* __restrict__ s, int64_t n) {   // x = x + alpha p + omega s
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride)
        x[e] = (x[e] + alpha * p[e]) + omega * s[e];
}

unsigned elem_blocks(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return static_cast<unsigned>(b);
}

// ---------------------------------------------------------------------------

// Stream-ordered allocations from the device's default memory pool, kept cached
// (release threshold = max), so per-solve buffers cost no cudaMalloc after warm-up.
int pool_alloc(double** p, size_t count, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        configured = true;
    }
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(double) * (count > 0 ? count : 1), s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return e == cudaErrorMemoryAllocation ? set_error(RTK_ERESOURCE, "device memory exhausted (Krylov workspace)")
                                              : cuda_status(e, "cudaMallocAsync");
    }
    return RTK_OK;
}

// Reduction scratch (block partials, counter, column slots, pinned staging) reused across
// solves -- its allocation, cudaMallocHost in particular, costs milliseconds.  A solve on a
// problem handle uses the handle's own workspace (created on the handle's first solve);
// callable solves and the exported BLAS-1 use one per (host thread, device).  Either way the
// buffers belong to the device that is current when they are created and are rebuilt if
// the same owner is later used on another device.
int bind_workspace(KrylovWorkspace*& slot, KrylovWorkspace** out) {
    int dev = 0;
    RTK_CUDA_TRY(cudaGetDevice(&dev));
    if (slot && slot->device != dev) {
        delete slot;
        slot = nullptr;
    }
    if (!slot) {
        auto* w = new (std::nothrow) KrylovWorkspace();
        if (!w) return set_error(RTK_ERESOURCE, "host allocation failed (Krylov workspace)");
        if (int rc = w->init()) {
            delete w;
            return rc;
        }
        slot = w;
    }
    *out = slot;
    return RTK_OK;
}

int acquire_workspace(Problem* owner, KrylovWorkspace** out) {
    if (owner) return bind_workspace(owner->krylov_ws, out);
    struct PerDevice {
        std::map<int, KrylovWorkspace*> by_dev;
        ~PerDevice() {
            for (auto& kv : by_dev) delete kv.second;
        }
    };
    thread_local PerDevice tl;
    int dev = 0;
    RTK_CUDA_TRY(cudaGetDevice(&dev));
    return bind_workspace(tl.by_dev[dev], out);
}

bool graphs_enabled() {
    static const bool on = !getenv_flag("RTK_GMRES_NO_GRAPH");   // A/B switch, read once per process
    return on;
}

class Engine {
   public:
    explicit Engine(cudaStream_t s, Problem* owner = nullptr) : s_(s), owner_(owner) {}
    int init() { return acquire_workspace(owner_, &wsp_); }

    // results (dots or norm^2) land in out_dev[0 .. k)
    int pass(int mode, const double* const* V, int k, const double* coef_dev, double* w, int64_t n, double* out_dev) {
        PassArgs P;
        for (int i = 0; i < KMAX; ++i) P.v[i] = (i < k) ? V[i] : nullptr;
        P.kc = k;
        P.coef = coef_dev;
        P.w = w;
        P.x = nullptr;
        P.n = n;
        P.partials = wsp_->partials;
        P.counter = wsp_->counter;
        P.out = out_dev;
        const int kb = k <= 4 ? 4 : (k <= 8 ? 8 : (k <= 16 ? 16 : 32));
        const int blocks = red_blocks(n, kb);
        RTK_CUDA_TRY(k <= 4 ? launch_pass<4>(mode, blocks, P)
                            : k <= 8 ? launch_pass<8>(mode, blocks, P)
                                     : k <= 16 ? launch_pass<16>(mode, blocks, P) : launch_pass<32>(mode, blocks, P));
        RTK_LAUNCH_CHECK("cgs_pass_kernel");
        return RTK_OK;
    }

    template <int KB>
    cudaError_t launch_pass(int mode, int blocks, const PassArgs& P) {
        bool aligned = (reinterpret_cast<uintptr_t>(P.w) & 15) == 0;
        for (int k = 0; k < P.kc; ++k) aligned = aligned && (reinterpret_cast<uintptr_t>(P.v[k]) & 15) == 0;
        return aligned ? launch_pass_v<KB, 2>(mode, blocks, P) : launch_pass_v<KB, 1>(mode, blocks, P);
    }
    template <int KB, int VEC>
    cudaError_t launch_pass_v(int mode, int blocks, const PassArgs& P) {
        switch (mode) {
            case MODE_DOT: return launch_pdl(cgs_pass_kernel<MODE_DOT, KB, VEC>, blocks, kRedThreads, 0, s_, P);
            case MODE_UPDATE_DOT: return launch_pdl(cgs_pass_kernel<MODE_UPDATE_DOT, KB, VEC>, blocks, kRedThreads, 0, s_, P);
            case MODE_UPDATE_NORM: return launch_pdl(cgs_pass_kernel<MODE_UPDATE_NORM, KB, VEC>, blocks, kRedThreads, 0, s_, P);
            default: return launch_pdl(cgs_pass_kernel<MODE_UPDATE, KB, VEC>, blocks, kRedThreads, 0, s_, P);
        }
    }

    // host-visible dot product x.y (fixed-order reduction)
    int dot(const double* x, const double* y, int64_t n, double* out) {
        const double* V[1] = {x};
        int rc = pass(MODE_DOT, V, 1, nullptr, const_cast<double*>(y), n, wsp_->dev_scalars);
        if (rc) return rc;
        RTK_CUDA_TRY(cudaMemcpyAsync(wsp_->pinned, wsp_->dev_scalars, sizeof(double), cudaMemcpyDeviceToHost, s_));
        RTK_CUDA_TRY(cudaStreamSynchronize(s_));
        *out = wsp_->pinned[0];
        return RTK_OK;
    }
    int norm(const double* x, int64_t n, double* out) {
        double d;
        int rc = dot(x, x, n, &d);
        *out = std::sqrt(d);
        return rc;
    }

    // Asynchronous CGS2 step: h1 -> slot[0, jp1), h2 -> slot[jp1, 2 jp1), ||w||^2 -> slot[2 jp1];
    // nothing crosses to the host here (the caller copies the slot back when it needs it).
    int cgs2_enqueue(const std::vector<double*>& V, int jp1, double* w, int64_t n, double* slot) {
        int rc;
        double* h1 = slot;
        double* h2 = slot + jp1;
        double* nrm = slot + 2 * jp1;
        if (jp1 <= KMAX) {
            if ((rc = pass(MODE_DOT, V.data(), jp1, nullptr, w, n, h1))) return rc;
            if ((rc = pass(MODE_UPDATE_DOT, V.data(), jp1, h1, w, n, h2))) return rc;
            return pass(MODE_UPDATE_NORM, V.data(), jp1, h2, w, n, nrm);
        }
        for (int k0 = 0; k0 < jp1; k0 += KMAX)
            if ((rc = pass(MODE_DOT, V.data() + k0, std::min(KMAX, jp1 - k0), nullptr, w, n, h1 + k0))) return rc;
        for (int k0 = 0; k0 < jp1; k0 += KMAX)
            if ((rc = pass(MODE_UPDATE, V.data() + k0, std::min(KMAX, jp1 - k0), h1 + k0, w, n, nullptr))) return rc;
        for (int k0 = 0; k0 < jp1; k0 += KMAX)
            if ((rc = pass(MODE_DOT, V.data() + k0, std::min(KMAX, jp1 - k0), nullptr, w, n, h2 + k0))) return rc;
        for (int k0 = 0; k0 < jp1; k0 += KMAX) {
            const int kc = std::min(KMAX, jp1 - k0);
            const bool last = k0 + kc >= jp1;
            if ((rc = pass(last ? MODE_UPDATE_NORM : MODE_UPDATE, V.data() + k0, kc, h2 + k0, w, n,
                           last ? nrm : nullptr)))
                return rc;
        }
        return RTK_OK;
    }

    int mgs_pass(int mode, const double* u, const double* coef, const double* d, double* w, int64_t n, double* out) {
        MgsArgs P;
        P.u = u;
        P.coef = coef;
        P.d = d;
        P.w = w;
        P.n = n;
        P.partials = wsp_->partials;
        P.counter = wsp_->counter;
        P.out = out;
        bool aligned = (reinterpret_cast<uintptr_t>(w) & 15) == 0;
        if (u) aligned = aligned && (reinterpret_cast<uintptr_t>(u) & 15) == 0;
        if (d) aligned = aligned && (reinterpret_cast<uintptr_t>(d) & 15) == 0;
        const int blocks = red_blocks(n, 4);
        cudaError_t e;
        if (aligned) {
            e = mode == MGS_DOT ? launch_pdl(mgs_pass_kernel<MGS_DOT, 2>, blocks, kRedThreads, 0, s_, P)
                : mode == MGS_UPDATE_DOT ? launch_pdl(mgs_pass_kernel<MGS_UPDATE_DOT, 2>, blocks, kRedThreads, 0, s_, P)
                                         : launch_pdl(mgs_pass_kernel<MGS_UPDATE_NORM, 2>, blocks, kRedThreads, 0, s_, P);
        } else {
            e = mode == MGS_DOT ? launch_pdl(mgs_pass_kernel<MGS_DOT, 1>, blocks, kRedThreads, 0, s_, P)
                : mode == MGS_UPDATE_DOT ? launch_pdl(mgs_pass_kernel<MGS_UPDATE_DOT, 1>, blocks, kRedThreads, 0, s_, P)
                                         : launch_pdl(mgs_pass_kernel<MGS_UPDATE_NORM, 1>, blocks, kRedThreads, 0, s_, P);
        }
        RTK_CUDA_TRY(e);
        RTK_LAUNCH_CHECK("mgs_pass_kernel");
        return RTK_OK;
    }

    // Modified Gram-Schmidt, one sweep (sweeps = 1) or two (reorthogonalize, sweeps = 2), the
    // reference's loop order (R/krylov.py:98-104): h1 -> slot[0, jp1), h2 -> slot[jp1, 2 jp1)
    // (second sweep only), ||w||^2 -> slot[2 jp1].
    int mgs_enqueue(const std::vector<double*>& V, int jp1, double* w, int64_t n, double* slot, int sweeps) {
        int rc;
        const double* prev_u = nullptr;
        const double* prev_c = nullptr;
        for (int sw = 0; sw < sweeps; ++sw) {
            double* h = slot + sw * jp1;
            for (int i = 0; i < jp1; ++i) {
                const int mode = prev_u ? MGS_UPDATE_DOT : MGS_DOT;
                if ((rc = mgs_pass(mode, prev_u, prev_c, V[i], w, n, h + i))) return rc;
                prev_u = V[i];
                prev_c = h + i;
            }
        }
        return mgs_pass(MGS_UPDATE_NORM, prev_u, prev_c, nullptr, w, n, slot + 2 * jp1);
    }

    // Arnoldi orthogonalisation of w against V[0, jp1) by the configured method
    int orth_enqueue(int orth, const std::vector<double*>& V, int jp1, double* w, int64_t n, double* slot) {
        if (orth == RTK_ORTH_CGS2) return cgs2_enqueue(V, jp1, w, n, slot);
        return mgs_enqueue(V, jp1, w, n, slot, orth == RTK_ORTH_MGS2 ? 2 : 1);
    }

    // y = x / sqrt(*norm2_dev)  (the norm stays on the device)
    int scale_dev(const double* x, double* y, int64_t n, const double* norm2_dev) {
        RTK_CUDA_TRY(launch_pdl(scale_kernel, elem_blocks(n), 256, 0, s_, x, y, n, 1.0, norm2_dev));
        RTK_LAUNCH_CHECK("scale_kernel");
        return RTK_OK;
    }

    int scale(const double* x, double* y, int64_t n, double a) {
        RTK_CUDA_TRY(launch_pdl(scale_kernel, elem_blocks(n), 256, 0, s_, x, y, n, a, static_cast<const double*>(nullptr)));
        RTK_LAUNCH_CHECK("scale_kernel");
        return RTK_OK;
    }

    // out = base + sum_k y_k V_k
    int combine(const std::vector<double*>& V, const std::vector<double>& y, const double* base, double* out,
                int64_t n) {
        const int m = static_cast<int>(y.size());
        const double* cur_base = base;
        for (int k0 = 0; k0 < m || k0 == 0; k0 += KMAX) {
            CombineArgs C;
            const int kc = std::min(KMAX, m - k0);
            for (int i = 0; i < KMAX; ++i) {
                C.v[i] = (i < kc) ? V[k0 + i] : nullptr;
                C.y[i] = (i < kc) ? y[k0 + i] : 0.0;
            }
            C.kc = kc > 0 ? kc : 0;
            C.base = cur_base;
            C.out = out;
            C.n = n;
            combine_kernel<<<elem_blocks(n), 256, 0, s_>>>(C);
            RTK_LAUNCH_CHECK("combine_kernel");
            cur_base = out;
            if (m == 0) break;
        }
        return RTK_OK;
    }

    int sub(const double* a, const double* b, double* out, int64_t n) {
        sub_kernel<<<elem_blocks(n), 256, 0, s_>>>(a, b, out, n);
        RTK_LAUNCH_CHECK("sub_kernel");
        return RTK_OK;
    }

    KrylovWorkspace* wsp_ = nullptr;

   private:
    cudaStream_t s_;
    Problem* owner_;
};

struct DevBuf {
    double* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    int alloc(int64_t n, cudaStream_t st) {
        s = st;
        return pool_alloc(&p, static_cast<size_t>(n), st);
    }
};

struct Basis {
    std::vector<double*> v;
    cudaStream_t s = nullptr;
    explicit Basis(cudaStream_t st) : s(st) {}
    ~Basis() {
        for (double* p : slabs)
            if (p) cudaFreeAsync(p, s);
    }
    std::vector<double*> slabs;   // allocations; vectors are carved from them
    int ensure(size_t count, int64_t n, size_t hint = 0) {
        // grow in slabs of several vectors (pool growth per 16 MB vector is slow for long
        // unrestarted solves); `hint` = the cycle length, so a restarted cycle is one slab
        const size_t pitch = (static_cast<size_t>(n) + 31) / 32 * 32;   // 256-byte aligned vectors
        while (v.size() < count) {
            size_t want = hint > v.size() ? hint - v.size() : 0;
            want = std::max(want, count - v.size());
            want = std::max<size_t>(want, std::min<size_t>(64, std::max<size_t>(1, v.size())));
            double* p = nullptr;
            while (pool_alloc(&p, pitch * want, s) != RTK_OK) {
                cudaGetLastError();
                if (want <= count - v.size())
                    return set_error(RTK_ERESOURCE, "Krylov basis does not fit in device memory (" +
                                                        std::to_string(v.size()) + " vectors allocated)");
                want = std::max(count - v.size(), want / 2);
            }
            slabs.push_back(p);
            for (size_t i = 0; i < want; ++i) v.push_back(p + i * pitch);
        }
        return RTK_OK;
    }
};

void solve_upper(const std::vector<std::vector<double>>& h_cols, const std::vector<double>& g, int m,
                 std::vector<double>& y) {
    // R/krylov.py:161-170
    y.assign(m, 0.0);
    for (int i = m - 1; i >= 0; --i) {
        double s = g[i];
        for (int k = i + 1; k < m; ++k) s -= h_cols[k][i] * y[k];
        y[i] = s / h_cols[i][i];
    }
}

struct History {
    double* out;
    int cap;
    int count = 0;
    std::vector<double> all;
    void push(double v) { all.push_back(v); }
    void flush(rtk_solve_report* rep) {
        const int n = static_cast<int>(all.size());
        const int w = n < cap ? n : cap;
        if (out)
            for (int i = 0; i < w; ++i) out[i] = all[i];
        rep->n_history = w;
    }
};

// One restart cycle of Arnoldi (matvec, CGS2, next basis vector, column read-back) captured
// as a CUDA graph and replayed every cycle: a cycle's pointers never change (fixed basis
// slab, w, per-iteration column slots), and for small problems the launch overhead of the
// ~10 kernels per iteration dominates the GPU work (cfg1: 65 us per iteration).
struct CycleGraph {
    cudaStream_t gs = nullptr;
    cudaStream_t side = nullptr;      // column read-backs, forked off the Arnoldi chain
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaEvent_t> evs;     // evs[j]: column j is in its pinned slot
    cudaEvent_t start = nullptr, done = nullptr;
    bool ready = false, failed = false;
    int64_t launches = 0;             // kernels per replay (counted during the capture)
    ~CycleGraph() {
        if (exec) cudaGraphExecDestroy(exec);
        for (auto e : evs) cudaEventDestroy(e);
        if (start) cudaEventDestroy(start);
        if (done) cudaEventDestroy(done);
        if (fork) cudaEventDestroy(fork);
        if (join) cudaEventDestroy(join);
        if (side) cudaStreamDestroy(side);
        if (gs) cudaStreamDestroy(gs);
    }
};

int resolve_orth(const rtk_solve_cfg* cfg, int* orth) {
    switch (cfg->orthogonalization) {
        case RTK_ORTH_REFERENCE: *orth = cfg->reorthogonalize ? RTK_ORTH_MGS2 : RTK_ORTH_MGS; return RTK_OK;
        case RTK_ORTH_MGS:
        case RTK_ORTH_MGS2:
        case RTK_ORTH_CGS2: *orth = cfg->orthogonalization; return RTK_OK;
        default: return set_error(RTK_EINVAL, "unknown orthogonalization");
    }
}

int gmres_impl(rtk_matvec_fn apply, void* ctx, int64_t n, const double* b, double* x, const rtk_solve_cfg* cfg,
               rtk_solve_report* rep, double* hist_out, int hist_cap, cudaStream_t s, Problem* owner) {
    if (!cfg || !rep || !b || !x) return set_error(RTK_EINVAL, "null argument");
    if (!(cfg->rel_tol > 0)) return set_error(RTK_EINVAL, "rel_tol must be positive");
    if (cfg->max_iter < 1) return set_error(RTK_EINVAL, "max_iter must be >= 1");
    int orth;
    if (int e = resolve_orth(cfg, &orth)) return e;
    const bool two_sweeps = orth != RTK_ORTH_MGS;   // h = h1 + h2
    // Look-ahead only for the library's own matvec: a user callable sees exactly the
    // reference's sequence of calls (no speculative applications past a stop or breakdown).
    const int window = apply == rtk_problem_matvec ? kLookahead : 1;
    *rep = rtk_solve_report{};
    History hist{hist_out, hist_cap};
    Engine E(s, owner);
    int rc;
    if ((rc = E.init())) return rc;
    int matvecs = 0;
    auto A = [&](const double* in, double* out) -> int {
        ++matvecs;
        int r = apply(ctx, in, out, n, s);
        if (r) return r;
        return RTK_OK;
    };
    cudaEvent_t look_ev[kLookahead];
    for (auto& e : look_ev) RTK_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            for (int q = 0; q < kLookahead; ++q) cudaEventDestroy(e[q]);
        }
    } ev_guard{look_ev};
    // column read-backs run on a side stream forked after the CGS2 passes, so the next
    // matvec on s does not queue behind the device-to-host copy; slot q is rewritten only
    // after the host consumed its previous column (look-ahead window), and the side stream
    // is drained before returning
    struct SideStream {
        cudaStream_t st = nullptr;
        cudaEvent_t fork = nullptr;
        ~SideStream() {
            if (st) {
                cudaStreamSynchronize(st);
                cudaStreamDestroy(st);
            }
            if (fork) cudaEventDestroy(fork);
        }
    } side;
    RTK_CUDA_TRY(cudaStreamCreateWithFlags(&side.st, cudaStreamNonBlocking));
    RTK_CUDA_TRY(cudaEventCreateWithFlags(&side.fork, cudaEventDisableTiming));
    int spec_matvecs = 0;   // look-ahead matvecs whose iterations were discarded (not reported)
    const double tol = cfg->rel_tol;
    double b_norm;
    if ((rc = E.norm(b, n, &b_norm))) return rc;
    RTK_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    if (b_norm == 0.0) {   // R/krylov.py:64-68
        hist.push(0.0);
        hist.flush(rep);
        rep->iterations = 0;
        rep->converged = 1;
        rep->true_residual = 0.0;
        RTK_CUDA_TRY(cudaStreamSynchronize(s));
        return RTK_OK;
    }
    DevBuf r, w, cand;
    if ((rc = r.alloc(n, s)) || (rc = w.alloc(n, s)) || (rc = cand.alloc(n, s))) return rc;
    RTK_CUDA_TRY(cudaMemcpyAsync(r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    int total = 0;
    const int cycle = cfg->restart > 0 ? cfg->restart : cfg->max_iter;
    Basis V(s);
    std::vector<double> col, y;
    // graph replay of whole cycles: the library's own matvec only (a user callback may
    // synchronise), restarted GMRES with short cycles, small vectors (launch-bound regime)
    // (capturing + instantiating costs ~1 ms, so only solves allowed several cycles use it)
    const bool graph_ok = apply == rtk_problem_matvec && cfg->restart > 0 && cycle <= 64 && n <= (int64_t(1) << 23) &&
                          cfg->max_iter >= 3 * cycle && graphs_enabled();
    CycleGraph G;
    const int slot_max = 2 * (cycle + 1) + 1;
    auto finish = [&](int iters, bool conv, bool brk, double tr) {
        rep->iterations = iters;
        rep->converged = conv ? 1 : 0;
        rep->breakdown = brk ? 1 : 0;
        rep->true_residual = tr;
        rep->matvecs = matvecs - spec_matvecs;
        hist.flush(rep);
    };
    while (total < cfg->max_iter) {
        double beta;
        if ((rc = E.norm(r.p, n, &beta))) return rc;
        if (beta / b_norm <= tol) {   // R/krylov.py:77-83
            hist.push(beta / b_norm);
            finish(total > 1 ? total : 1, true, false, beta / b_norm);
            return RTK_OK;
        }
        const size_t hint = static_cast<size_t>(std::min(cycle + 1, 64));
        if ((rc = V.ensure(1, n, hint))) return rc;
        if ((rc = E.scale(r.p, V.v[0], n, beta))) return rc;
        std::vector<std::vector<double>> h_cols;
        std::vector<double> cs, sn, g{beta};
        bool breakdown = false;
        const int steps = std::min(cycle, cfg->max_iter - total);
        // Arnoldi look-ahead: the device runs up to kLookahead iterations ahead of the host's
        // Givens / convergence bookkeeping (the next basis vector only needs ||w||, which stays
        // on the device), so the GPU never idles on the per-iteration column read-back.  Work
        // enqueued past a stopping iteration is discarded; results are those of the
        // sequential loop (same kernels, same operands, same order).
        const bool use_graph = graph_ok && !G.failed && steps == cycle;
        // slots: graph mode keeps one per iteration of the cycle (fixed size, captured pointers)
        const int slot_sz = use_graph ? slot_max : 2 * (steps + 1) + 1;
        if ((rc = E.wsp_->reserve_look(std::max(kLookahead, graph_ok ? cycle : 0) * slot_max))) return rc;
        double* dslots = E.wsp_->look_dev;
        double* pslots = E.wsp_->look_pin;
        int next = 0;
        if (use_graph && !G.ready) {
            if ((rc = V.ensure(cycle + 1, n, hint))) return rc;
            RTK_CUDA_TRY(cudaStreamCreateWithFlags(&G.gs, cudaStreamNonBlocking));
            RTK_CUDA_TRY(cudaEventCreateWithFlags(&G.start, cudaEventDisableTiming));
            RTK_CUDA_TRY(cudaEventCreateWithFlags(&G.done, cudaEventDisableTiming));
            RTK_CUDA_TRY(cudaStreamCreateWithFlags(&G.side, cudaStreamNonBlocking));
            RTK_CUDA_TRY(cudaEventCreateWithFlags(&G.fork, cudaEventDisableTiming));
            RTK_CUDA_TRY(cudaEventCreateWithFlags(&G.join, cudaEventDisableTiming));
            G.evs.resize(cycle, nullptr);
            for (auto& e : G.evs) RTK_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            // the first matvec of a problem may configure kernels (attributes, occupancy queries):
            // do it outside the capture, on scratch
            RTK_CUDA_TRY(cudaStreamSynchronize(s));
            if ((rc = apply(ctx, V.v[0], cand.p, n, G.gs))) return rc;
            RTK_CUDA_TRY(cudaStreamSynchronize(G.gs));
            Engine Eg(G.gs, owner);
            if ((rc = Eg.init())) return rc;
            cudaGraph_t graph = nullptr;
            const int64_t l0 = rtk_kernel_launch_count();
            bool ok = cudaStreamBeginCapture(G.gs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            for (int jj = 0; ok && jj < cycle; ++jj) {
                double* dslot = dslots + static_cast<size_t>(jj) * slot_max;
                // the column's read-back (copy + external event) branches off after the CGS2
                // passes, so the next matvec does not wait for the device-to-host copy
                ok = apply(ctx, V.v[jj], w.p, n, G.gs) == RTK_OK &&
                     Eg.orth_enqueue(orth, V.v, jj + 1, w.p, n, dslot) == RTK_OK &&
                     cudaEventRecord(G.fork, G.gs) == cudaSuccess &&
                     cudaStreamWaitEvent(G.side, G.fork, 0) == cudaSuccess &&
                     cudaMemcpyAsync(pslots + static_cast<size_t>(jj) * slot_max, dslot,
                                     sizeof(double) * (2 * (jj + 1) + 1), cudaMemcpyDeviceToHost, G.side) == cudaSuccess &&
                     cudaEventRecordWithFlags(G.evs[jj], G.side, cudaEventRecordExternal) == cudaSuccess &&
                     Eg.scale_dev(w.p, V.v[jj + 1], n, dslot + 2 * (jj + 1)) == RTK_OK;
            }
            // join the read-back branch (also when the capture failed part-way: the side stream
            // must leave capture mode with the origin stream)
            const bool joined = cudaEventRecord(G.join, G.side) == cudaSuccess &&
                                cudaStreamWaitEvent(G.gs, G.join, 0) == cudaSuccess;
            ok = ok && joined;
            const cudaError_t ec = cudaStreamEndCapture(G.gs, &graph);
            ok = ok && ec == cudaSuccess && graph != nullptr &&
                 cudaGraphInstantiate(&G.exec, graph, 0) == cudaSuccess;
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            G.launches = rtk_kernel_launch_count() - l0;
            count_launch(static_cast<int>(-G.launches));   // captured, not launched
            G.ready = ok;
            G.failed = !ok;
        }
        const bool graph_cycle = use_graph && G.ready;
        if (graph_cycle) {
            RTK_CUDA_TRY(cudaEventRecord(G.start, s));
            RTK_CUDA_TRY(cudaStreamWaitEvent(G.gs, G.start, 0));
            RTK_CUDA_TRY(cudaGraphLaunch(G.exec, G.gs));
            RTK_CUDA_TRY(cudaEventRecord(G.done, G.gs));
            RTK_CUDA_TRY(cudaStreamWaitEvent(s, G.done, 0));   // later work on s sees the whole cycle
            count_launch(static_cast<int>(G.launches));
            next = steps;
        }
        int j = 0;
        while (j < steps) {
            while (!graph_cycle && next < steps && next - j < window) {
                const int q = next % kLookahead;
                double* dslot = dslots + static_cast<size_t>(q) * slot_sz;
                if ((rc = A(V.v[next], w.p))) return rc;
                if ((rc = E.orth_enqueue(orth, V.v, next + 1, w.p, n, dslot))) return rc;
                RTK_CUDA_TRY(cudaEventRecord(side.fork, s));
                RTK_CUDA_TRY(cudaStreamWaitEvent(side.st, side.fork, 0));
                RTK_CUDA_TRY(cudaMemcpyAsync(pslots + static_cast<size_t>(q) * slot_sz, dslot,
                                             sizeof(double) * (2 * (next + 1) + 1), cudaMemcpyDeviceToHost, side.st));
                RTK_CUDA_TRY(cudaEventRecord(look_ev[q], side.st));
                if ((rc = V.ensure(next + 2, n, hint))) return rc;
                if ((rc = E.scale_dev(w.p, V.v[next + 1], n, dslot + 2 * (next + 1)))) return rc;
                ++next;
            }
            {
                const int q = graph_cycle ? j : j % kLookahead;
                RTK_CUDA_TRY(cudaEventSynchronize(graph_cycle ? G.evs[j] : look_ev[q]));
                if (graph_cycle) ++matvecs;   // the replayed matvec of iteration j is consumed
                const double* hs = pslots + static_cast<size_t>(q) * slot_sz;
                col.assign(j + 2, 0.0);
                for (int i = 0; i <= j; ++i) col[i] = two_sweeps ? hs[i] + hs[j + 1 + i] : hs[i];
                col[j + 1] = std::sqrt(hs[2 * (j + 1)]);
            }
            breakdown = col[j + 1] < 1e-14 * b_norm;
            // Givens (R/krylov.py:109-122), host scalars
            for (int i = 0; i < j; ++i) {
                const double tmp = cs[i] * col[i] + sn[i] * col[i + 1];
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
                col[i] = tmp;
            }
            const double denom = std::hypot(col[j], col[j + 1]);
            const double cj = denom != 0.0 ? col[j] / denom : 1.0;
            const double sj = denom != 0.0 ? col[j + 1] / denom : 0.0;
            cs.push_back(cj);
            sn.push_back(sj);
            col[j] = denom;
            h_cols.emplace_back(col.begin(), col.begin() + j + 1);
            g.push_back(-sj * g[j]);
            g[j] = cj * g[j];
            ++total;
            ++j;
            const double rel = std::fabs(g[j]) / b_norm;
            hist.push(rel);
            if (rel <= tol || breakdown) {   // R/krylov.py:129-147
                spec_matvecs = graph_cycle ? 0 : next - j;   // look-ahead iterations not (yet) consumed
                solve_upper(h_cols, g, j, y);
                if ((rc = E.combine(V.v, y, x, cand.p, n))) return rc;
                if ((rc = A(cand.p, w.p))) return rc;
                if ((rc = E.sub(b, w.p, w.p, n))) return rc;
                double tn;
                if ((rc = E.norm(w.p, n, &tn))) return rc;
                const double true_rel = tn / b_norm;
                if (true_rel <= 10.0 * tol) {
                    if (breakdown) hist.all.back() = true_rel;
                    RTK_CUDA_TRY(cudaMemcpyAsync(x, cand.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
                    RTK_CUDA_TRY(cudaStreamSynchronize(s));
                    finish(total, true, breakdown, true_rel);
                    return RTK_OK;
                }
                if (breakdown) {
                    RTK_CUDA_TRY(cudaMemcpyAsync(x, cand.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
                    RTK_CUDA_TRY(cudaStreamSynchronize(s));
                    finish(total, false, true, true_rel);
                    return RTK_OK;
                }
                spec_matvecs = 0;            // continuing: the look-ahead iterations will be consumed
            }
        }
        // cycle exhausted: x += V y ; r = b - A x   (R/krylov.py:149-152)
        solve_upper(h_cols, g, j, y);
        if ((rc = E.combine(V.v, y, x, x, n))) return rc;
        if ((rc = A(x, w.p))) return rc;
        if ((rc = E.sub(b, w.p, r.p, n))) return rc;
    }
    double rn;
    if ((rc = E.norm(r.p, n, &rn))) return rc;
    finish(total, false, false, rn / b_norm);
    RTK_CUDA_TRY(cudaStreamSynchronize(s));
    return RTK_OK;
}

int bicgstab_impl(rtk_matvec_fn apply, void* ctx, int64_t n, const double* b, double* x, const rtk_solve_cfg* cfg,
                  rtk_solve_report* rep, double* hist_out, int hist_cap, cudaStream_t s, Problem* owner) {
    // R/krylov.py:180-256
    if (!cfg || !rep || !b || !x) return set_error(RTK_EINVAL, "null argument");
    if (!(cfg->rel_tol > 0)) return set_error(RTK_EINVAL, "rel_tol must be positive");
    if (cfg->max_iter < 1) return set_error(RTK_EINVAL, "max_iter must be >= 1");
    *rep = rtk_solve_report{};
    History hist{hist_out, hist_cap};
    Engine E(s, owner);
    int rc;
    if ((rc = E.init())) return rc;
    int matvecs = 0;
    auto A = [&](const double* in, double* out) -> int {
        ++matvecs;
        return apply(ctx, in, out, n, s);
    };
    const double eps = 1e-30, tol = cfg->rel_tol;
    double b_norm;
    if ((rc = E.norm(b, n, &b_norm))) return rc;
    RTK_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    if (b_norm == 0.0) {
        hist.push(0.0);
        hist.flush(rep);
        rep->converged = 1;
        RTK_CUDA_TRY(cudaStreamSynchronize(s));
        return RTK_OK;
    }
    DevBuf r, rsh, v, p, sv, t;
    if ((rc = r.alloc(n, s)) || (rc = rsh.alloc(n, s)) || (rc = v.alloc(n, s)) || (rc = p.alloc(n, s)) ||
        (rc = sv.alloc(n, s)) || (rc = t.alloc(n, s)))
        return rc;
    RTK_CUDA_TRY(cudaMemcpyAsync(r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    RTK_CUDA_TRY(cudaMemcpyAsync(rsh.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    RTK_CUDA_TRY(cudaMemsetAsync(v.p, 0, sizeof(double) * n, s));
    RTK_CUDA_TRY(cudaMemsetAsync(p.p, 0, sizeof(double) * n, s));
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    bool breakdown = false, converged = false;
    int it = 0;
    const unsigned nb = elem_blocks(n);
    while (it < cfg->max_iter) {
        double rho;
        if ((rc = E.dot(rsh.p, r.p, n, &rho))) return rc;
        if (std::fabs(rho) < eps) {
            breakdown = true;
            break;
        }
        if (it == 0) {
            RTK_CUDA_TRY(cudaMemcpyAsync(p.p, r.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        } else {
            const double beta = (rho / rho_prev) * (alpha / omega);
            bicg_p_kernel<<<nb, 256, 0, s>>>(r.p, p.p, v.p, beta, omega, n);
            RTK_LAUNCH_CHECK("bicg_p_kernel");
        }
        if ((rc = A(p.p, v.p))) return rc;
        double denom;
        if ((rc = E.dot(rsh.p, v.p, n, &denom))) return rc;
        if (std::fabs(denom) < eps) {
            breakdown = true;
            break;
        }
        alpha = rho / denom;
        axpy_out_kernel<<<nb, 256, 0, s>>>(r.p, -alpha, v.p, sv.p, n);   // s = r - alpha v
        RTK_LAUNCH_CHECK("axpy_out_kernel");
        ++it;
        double s_norm;
        if ((rc = E.norm(sv.p, n, &s_norm))) return rc;
        if (s_norm / b_norm <= tol) {
            axpy_out_kernel<<<nb, 256, 0, s>>>(x, alpha, p.p, x, n);
            RTK_LAUNCH_CHECK("axpy_out_kernel");
            hist.push(s_norm / b_norm);
            converged = true;
            break;
        }
        if ((rc = A(sv.p, t.p))) return rc;
        double tt;
        if ((rc = E.dot(t.p, t.p, n, &tt))) return rc;
        if (tt < eps) {
            breakdown = true;
            break;
        }
        double ts;
        if ((rc = E.dot(t.p, sv.p, n, &ts))) return rc;
        omega = ts / tt;
        if (std::fabs(omega) < eps) {
            breakdown = true;
            break;
        }
        bicg_x_kernel<<<nb, 256, 0, s>>>(x, alpha, p.p, omega, sv.p, n);
        RTK_LAUNCH_CHECK("bicg_x_kernel");
        axpy_out_kernel<<<nb, 256, 0, s>>>(sv.p, -omega, t.p, r.p, n);   // r = s - omega t
        RTK_LAUNCH_CHECK("axpy_out_kernel");
        rho_prev = rho;
        double rn;
        if ((rc = E.norm(r.p, n, &rn))) return rc;
        hist.push(rn / b_norm);
        if (rn / b_norm <= tol) {
            converged = true;
            break;
        }
    }
    if ((rc = A(x, t.p))) return rc;
    if ((rc = E.sub(b, t.p, t.p, n))) return rc;
    double tn;
    if ((rc = E.norm(t.p, n, &tn))) return rc;
    const double true_rel = tn / b_norm;
    if (converged) converged = true_rel <= 10.0 * tol;
    if (hist.all.empty()) hist.push(true_rel);
    rep->iterations = it;
    rep->converged = converged ? 1 : 0;
    rep->breakdown = breakdown ? 1 : 0;
    rep->true_residual = true_rel;
    rep->matvecs = matvecs;
    hist.flush(rep);
    RTK_CUDA_TRY(cudaStreamSynchronize(s));
    return RTK_OK;
}

}  // namespace
}  // namespace rtk

extern "C" {

int rtk_gmres(rtk_matvec_fn apply, void* ctx, int64_t n, const double* b, double* x, const rtk_solve_cfg* cfg,
              rtk_solve_report* rep, double* hist, int32_t cap, void* stream) {
    if (!apply) return rtk::set_error(RTK_EINVAL, "null matvec");
    return rtk::gmres_impl(apply, ctx, n, b, x, cfg, rep, hist, cap, static_cast<cudaStream_t>(stream), nullptr);
}

int rtk_gmres_problem(rtk_problem* p, const double* b, double* x, const rtk_solve_cfg* cfg, rtk_solve_report* rep,
                      double* hist, int32_t cap, void* stream) {
    if (!p) return rtk::set_error(RTK_EINVAL, "null problem handle");
    return rtk::gmres_impl(rtk_problem_matvec, p, rtk_problem_n_total(p), b, x, cfg, rep, hist, cap,
                           static_cast<cudaStream_t>(stream), rtk::problem_impl(p));
}

int rtk_bicgstab(rtk_matvec_fn apply, void* ctx, int64_t n, const double* b, double* x, const rtk_solve_cfg* cfg,
                 rtk_solve_report* rep, double* hist, int32_t cap, void* stream) {
    if (!apply) return rtk::set_error(RTK_EINVAL, "null matvec");
    return rtk::bicgstab_impl(apply, ctx, n, b, x, cfg, rep, hist, cap, static_cast<cudaStream_t>(stream),
                              apply == rtk_problem_matvec ? rtk::problem_impl(static_cast<rtk_problem*>(ctx)) : nullptr);
}

int rtk_dot(const double* x, const double* y, int64_t n, double* out_host, void* stream) {
    rtk::Engine E(static_cast<cudaStream_t>(stream));
    int rc = E.init();
    if (rc) return rc;
    return E.dot(x, y, n, out_host);
}

int rtk_block_dot(const double* const* vecs_host, int32_t k, const double* w, int64_t n, double* out_host,
                  void* stream) {
    rtk::Engine E(static_cast<cudaStream_t>(stream));
    int rc = E.init();
    if (rc) return rc;
    for (int k0 = 0; k0 < k; k0 += rtk::KMAX) {
        const int kc = std::min(rtk::KMAX, k - k0);
        if ((rc = E.pass(rtk::MODE_DOT, vecs_host + k0, kc, nullptr, const_cast<double*>(w), n, E.wsp_->dev_scalars)))
            return rc;
        RTK_CUDA_TRY(cudaMemcpyAsync(out_host + k0, E.wsp_->dev_scalars, sizeof(double) * kc, cudaMemcpyDeviceToHost,
                                     static_cast<cudaStream_t>(stream)));
        RTK_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    }
    return RTK_OK;
}

}  // extern "C"
