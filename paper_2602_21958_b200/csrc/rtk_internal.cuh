// Internal declarations shared by the librtk_b200 translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "rtk_b200.h"

namespace rtk {

// ---- error plumbing -------------------------------------------------------
int set_error(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);
void count_launch(int n = 1);

#define RTK_CUDA_TRY(expr)                                   \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return ::rtk::cuda_status(_e, #expr); \
    } while (0)

#define RTK_LAUNCH_CHECK(what)                               \
    do {                                                     \
        ::rtk::count_launch();                               \
        cudaError_t _e = cudaGetLastError();                 \
        if (_e != cudaSuccess) return ::rtk::cuda_status(_e, what); \
    } while (0)

// ---- device-resident slab operator ---------------------------------------
//
// HBM layout (all float64):
//   dt      [n_space-1]          t_{i+1} - t_i
//   phi     [n_freq]             profile at frequency nodes
//   inv_mu  [n_angles]           1/|mu_a|
//   wy      [n_mom][n_angles]    w_a * Y_k(a)      (moment reduction weights)
//   yb      [n_mom][n_angles]    Y_k(a)            (source reconstruction)
//   rwt     [n_freq][n_freq]     rwt[g][f] = R[f][g] * w_g   (K-major B operand)
//   gamma   [n_space][n_freq] * coeff folded at use, or [n_space][n_rays]
//   inflow  [n_rays]
// workspace:
//   mom     [n_space][n_mom][fp]   angular moments m          (fp = n_freq rounded up to even,
//   gmom    [n_space][n_mom][fp]   G = c_k gamma R w m         so TMA row pitches are 16-byte multiples;
//   rwt     [n_freq][fp]                                       pad columns stay zero)
struct TmaCta {
    int ray0;    // first ray (a-major, f-minor) of the CTA
    int nr;      // rays in the CTA (<= 128), all of one hemisphere
    int down;    // 1: mu < 0, march surface -> depth
    int f0;      // first column of the G box
};

// per-direction lattice geometry (lattice.cu)
struct LatDir {
    int down;         // Omega_z < 0: enters at the top layer
    int n_sub;        // sub-segments per layer step
    int shift_off;    // first entry of this direction in the sub-node shift table
    long long dtab_off;   // first entry of this direction in the dt table (moment layout)
    int sub_pref;     // sum of (n_sub + 1) over the preceding directions (one step's shift block)
    double sx, sy;    // horizontal cells moved per layer step
    double sub_len;   // path length of one sub-segment
    double wy[8];     // w_a Y_l(a)   (moment accumulation)
    double cy[8];     // c_l Y_l(a)   (source expansion)
    int sc;           // short characteristics: lines restart at each node's upwind point every step
    int rbx, rby;     // SC restart gather: integer part of (-sx, -sy) mod (nx, ny) ...
    double rax, ray;  // ... and its fractional part (same arithmetic as shift_of)
};

enum ProblemKind { KIND_SLAB = 1, KIND_LATTICE = 2 };

// Per-problem kernel-selection switches.  Initialised ONCE when the problem is created
// (tuning_from_env: the RTK_* variables, for A/B measurements) and overridable per handle
// through rtk_problem_set_tuning (tests select each shipped kernel variant this way).
// Launchers read only this struct, never the environment.
struct Tuning {
    int disable_tma = 0;      // "disable_tma"      RTK_DISABLE_TMA: 1D sweeps take the cp.async kernel (sweep1d.cu)
    int lat_dg = 0;           // "lattice_dg"       RTK_LAT_DG: direction groups of the lattice moment kernel (0 auto, 1/4/8)
    int lat_no_smem = 0;      // "lattice_no_smem"  RTK_LATTICE_NO_SMEM: intensity layout without the shared-memory kernel
    int lat_no_dtab = 0;      // "lattice_no_dtab"  RTK_LATTICE_NO_DTAB: sample opacity instead of the dt table
    int lat_no_planar = 0;    // "lattice_no_planar" RTK_LATTICE_NO_PLANAR: 2D slabs through the 3D sampling path
    int moments_scalar = 0;   // "moments_scalar"   RTK_MOMENTS_SCALAR: 8-byte moment kernel instead of the pair kernel
    int sigma_unfused = 0;    // "sigma_unfused"    RTK_SIGMA_UNFUSED: K2a + K2b instead of the fused Sigma kernel
    int lat_no_tile = 0;      // "lattice_no_tile"  RTK_LATTICE_NO_TILE: moment layout through the per-item gather
                              //                    kernel (lattice_mom_group_kernel) instead of the tiled one
    int lat_dgz = 0;          // "lattice_dgz"      RTK_LAT_DGZ: direction groups of the tiled kernel (0 auto, 1..8)
};
Tuning tuning_from_env();
// 0 ok, 1 unknown key
int tuning_set(Tuning& t, const char* key, int64_t value);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-DEVICE attribute: this records
// the largest size set per (kernel, current device) and sets it when a launch needs more.
// Returns RTK_OK or a CUDA status (with the error message set).
int ensure_smem(const void* func, size_t bytes);
template <typename F>
int ensure_smem_for(F* func, size_t bytes) {
    return ensure_smem(reinterpret_cast<const void*>(func), bytes);
}
// per-(kernel, device) cached integer (e.g. co-resident clusters of a launch shape); -1 if unset
int device_cache_get(const void* func, int slot);
void device_cache_put(const void* func, int slot, int value);
enum Layout { LAYOUT_INTENSITY = 0, LAYOUT_MOMENTS = 1 };

struct MomCta {
    int a0, nd, down, f0, group;   // 1D moment-layout sweep: directions [a0, a0+nd), 16-frequency tile at f0
};

struct KrylovWorkspace;   // krylov.cu

struct Problem {
    int kind = KIND_SLAB;
    Tuning tune;
    KrylovWorkspace* krylov_ws = nullptr;   // reduction scratch of solves on this handle (owned)
    int layout = LAYOUT_INTENSITY;
    int64_t n_space = 0;
    int n_angles = 0, n_freq = 0, n_mom = 0, fs = 0, gamma_per_ray = 0, fp = 0;
    int64_t n_rays = 0, n_total = 0;
    std::vector<double> h_mu, h_coeffs;
    std::vector<double> h_inflow;   // host copy of the uploaded inflow (set_inflow skips unchanged uploads)
    double *dt = nullptr, *phi = nullptr, *inv_mu = nullptr, *wy = nullptr, *yb = nullptr;
    double *rwt = nullptr, *gamma = nullptr, *coeffs = nullptr, *inflow = nullptr;
    int* dir_sign = nullptr;     // [n_angles] -1 down (mu<0), +1 up
    double *mom = nullptr, *gmom = nullptr;
    double *host_x = nullptr, *host_y = nullptr;   // lazily allocated device staging for *_host calls
    double *host_x2 = nullptr, *host_y2 = nullptr; // second staging pair (batched host calls)
    static constexpr int64_t kStageChunk = int64_t(1) << 22;   // 32 MB pinned chunks for pageable host buffers
    double* stage[2] = {nullptr, nullptr};
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    cudaStream_t io[2] = {nullptr, nullptr};
    cudaEvent_t io_done[2] = {nullptr, nullptr};
    // TMA sweep path (sweep_tma.cu)
    bool tma_ready = false;
    int tma_n_ctas = 0, tma_gw = 0, tma_u = 4;
    TmaCta* tma_ctas = nullptr;
    double* dtpad = nullptr;
    double* par_tab = nullptr;                   // exp-parabolic Lagrange denominators (4 padded tables, sweep_tma.cu)
    // lattice (multi-D) state
    int lat_nx = 0, lat_ny = 0, lat_nz = 0;
    LatDir* lat_dirs = nullptr;
    double *lat_chi = nullptr, *lat_in_top = nullptr, *lat_in_bot = nullptr;
    double* lat_state[2] = {nullptr, nullptr};   // [dir][line][freq] line values (moment layout)
    double* lat_src = nullptr;                   // full source vector (intensity layout)
    double* lat_zero = nullptr;                  // [n_space][n_freq] zeros (boundary-only RHS)
    double* lat_splane[3] = {nullptr, nullptr, nullptr};  // [dir][line][freq] source planes (moment layout ring)
    // slab moment layout (sweep_mom.cu)
    MomCta* mom_ctas = nullptr;
    int mom_n_ctas = 0, mom_n_groups = 0;
    double* mom_partial = nullptr;               // [group][n_space][n_mom][fp]
    double* dtpad_mom = nullptr;
    CUtensorMap mom_gmap, tma_dtmap_mom;
    void* lat_sub_shift = nullptr;               // Shift table (lattice.cu), sub-nodes
    void* lat_gat_shift = nullptr;               // Shift table, T_RC gathers
    void* lat_down_shift = nullptr;              // Shift table, exp-parabolic downwind points
    double* lat_dtab = nullptr;                  // [dir][t][m][line] sub-segment optical paths
    int lat_max_sub = 0;                         // largest sub-segment count over the directions
    bool lat_any_sc = false;   // some direction uses short characteristics
    int lat_total_sub = 0;                       // sum over directions of (n_sub + 1)
    // tiled moment kernel (lattice.cu lattice_mom_tile_kernel)
    void* lat_tile_hdr = nullptr;                // TileHdr [dir][step]
    void* lat_tile_sub = nullptr;                // TileSub, indexed like lat_sub_shift
    int lat_tile_tx = 0, lat_tile_ty = 0;        // lines per tile
    int lat_region_cap = 0, lat_sub_cap = 0;     // staged window (double2) / sub-node table capacity
    std::vector<int> h_lat_down;                 // per direction: Omega_z < 0
    // launch-time workspace of the (logically const) operator application
    int* lat_order = nullptr;                    // device direction order of the current range
    mutable std::vector<int> h_lat_order;
    mutable int lat_order_a0 = -1, lat_order_a1 = -1, lat_order_down = 0;
    mutable double* lat_scratch = nullptr;       // per-group partial moments (direction groups > 1)
    mutable size_t lat_scratch_count = 0;
    CUtensorMap tma_gmap, tma_dtmap;
    CUtensorMap tma_qmap[4];                     // par_tab: [down: qc, qd | up: qc, qd]
    ~Problem();
};

// ---- kernel launchers (return status) --------------------------------------
// sigma.cu
int launch_moments(const Problem& p, const double* x, cudaStream_t s);
int launch_redistribute(const Problem& p, cudaStream_t s);            // mom -> gmom
int launch_sigma_fused(const Problem& p, const double* x, cudaStream_t s);   // x -> gmom; -1: not applicable
int launch_sigma(const Problem& p, const double* x, cudaStream_t s);         // x -> gmom (fused or K2a + K2b)
int launch_expand_source(const Problem& p, const double* thermal, double* out, cudaStream_t s);
// sweep1d.cu
enum SweepSrc { SRC_MOMENTS = 0, SRC_VECTOR = 1, SRC_ZERO = 2 };
enum SweepOut { OUT_X_MINUS = 0, OUT_ACC = 1 };
int launch_sweep(const Problem& p, int src_mode, int out_mode, bool with_inflow,
                 const double* src_vec, const double* x, double* y, cudaStream_t s);
// sweep_tma.cu
int setup_tma(Problem& p);
int launch_sweep_tma(const Problem& p, const double* x, double* y, cudaStream_t s);   // -1: not applicable
// sweep_mom.cu
int setup_slab_moments(Problem& p);
int slab_moment_transfer(const Problem& p, const double* u, cudaStream_t s);   // p.mom = M Lambda S(u)
int slab_moment_fold(const Problem& p, const double* u, cudaStream_t s);       // p.gmom = c gamma u
bool encode_f64_map(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* stride_bytes,
                    const uint32_t* box);
// lattice.cu
int setup_lattice(Problem& p, const rtk_lattice_desc* d);
int lattice_transfer_intensity(const Problem& p, int src_mode, int out_mode, bool with_inflow, const double* src,
                               const double* x, double* y, cudaStream_t s);
int lattice_transfer_moments(const Problem& p, int src_mode, bool with_inflow, const double* src, double* mom,
                             cudaStream_t s, int a0 = 0, int a1 = -1);
// sigma.cu GEMM epilogues: C = c_k gamma acc | c_k acc | U - acc | acc
enum Epilogue { EPI_GAMMA = 0, EPI_COEF = 1, EPI_SUB = 2, EPI_PLAIN = 3 };
int launch_redistribute_ex(const Problem& p, const double* A, double* C, int ldc, int epi, const double* U, int ldu,
                           cudaStream_t s, int64_t nodes = -1, const double* gamma = nullptr);
// krylov.cu
void destroy_krylov_workspace(KrylovWorkspace* w);
Problem* problem_impl(rtk_problem* p);
int apply_A_dev(Problem& p, const double* x, double* y, cudaStream_t s);
int sweep_apply(const Problem& p, const double* x, double* y, cudaStream_t s);
bool getenv_flag(const char* name);

// Programmatic dependent launch (Krylov passes, moment reductions, small redistribution).
__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// Programmatic dependent launch on (default); RTK_NO_PDL=1 (read once per process, an A/B
// measurement switch) launches plainly.
bool pdl_enabled();

// launch with programmatic stream serialization (the kernel starts with pdl_prologue)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned blocks, int threads, size_t smem, cudaStream_t s,
                       Args... args) {
    const bool off = !pdl_enabled();
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

int upload(double** dst, const double* src, size_t count);

}  // namespace rtk
