/*
 * rtk_b200.h -- C ABI of the B200-native (I - Lambda Sigma) operator and its GMRES driver.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * rtkrylov (arXiv 2602.21958).  R/ = /root/reference/pkg/src/rtkrylov/.
 * Every entry point names the reference interface it replaces.  Plain C
 * types only: host arrays are `const double*` + sizes, device vectors are raw
 * device pointers (float64, the reference's space-major layout
 * index = i_space * n_rays + a * n_freq + f, R/grid.py:83-88), streams are
 * `void*` (a cudaStream_t, NULL = the legacy default stream).
 *
 * Status codes: 0 ok, 1 invalid argument (Python: ValueError), 2 resource or
 * capacity (ResourceLimitError, R/errors.py:6-7), 3 CUDA error (RuntimeError).
 * rtk_last_error_message() returns the thread's last message.
 * Non-convergence of a solve is a report flag, never an error
 * (R/krylov.py:154-158).
 */
#ifndef RTK_B200_H
#define RTK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTK_OK 0
#define RTK_EINVAL 1
#define RTK_ERESOURCE 2
#define RTK_ECUDA 3

/* formal solvers (R/_kernels.py:70-88 is IE; the exponential ones are new) */
#define RTK_FS_IE 0
#define RTK_FS_EXP_LINEAR 1
#define RTK_FS_EXP_PARABOLIC 2

#define RTK_MAX_MOMENTS 8

/* unknown layout of slab and lattice problems */
#define RTK_LAYOUT_INTENSITY 0
#define RTK_LAYOUT_MOMENTS 1


typedef struct rtk_problem rtk_problem;

/*
 * 1D plane-parallel slab.  Replaces the state held by Grid (R/grid.py:63-112),
 * TransferOperator (R/transfer.py:65-104) and ScatteringOperator
 * (R/scattering.py:74-100).  Sigma is the separable kernel
 *   Psi[(a,f),(a',f')] = sum_k coeffs[k] ybasis[k][a] ybasis[k][a'] * R[f][f']
 * which expresses LegendreKernel (ybasis = P_l(mu), R = 1), CRDKernel
 * (ybasis = 1, R = phi phi'), CoherentKernel (R = diag(phi / w_f)) and the
 * dipole x PRD kernel (ybasis = P_0, P_2; coeffs = 1, 1/2).
 */
typedef struct rtk_slab_desc {
    int64_t n_space;
    int32_t n_angles;
    int32_t n_freq;
    int32_t n_moments;        /* rows of ybasis, 1..RTK_MAX_MOMENTS */
    int32_t formal_solver;    /* RTK_FS_* */
    int32_t gamma_per_ray;    /* 0: gamma[n_space][n_freq]; 1: gamma[n_space][n_angles*n_freq] (R/grid.py:107-112) */
    int32_t layout;           /* RTK_LAYOUT_INTENSITY (the reference's I[i][a][f]) or RTK_LAYOUT_MOMENTS
                                 (u[i][k][f] = sum_g R w_g m, m = sum_a w_a Y_k(a) I; 2 N_nu N_s values for
                                 the dipole kernel; IE / exp-linear, n_moments <= 3, gamma[n_space][n_freq]) */
    const double* t_nodes;        /* [n_space] strictly increasing optical-depth scale (R/grid.py:68) */
    const double* mu;             /* [n_angles] direction cosines, none zero */
    const double* ang_w;          /* [n_angles] angular weights */
    const double* phi;            /* [n_freq] profile at the frequency nodes */
    const double* freq_w;         /* [n_freq] frequency weights */
    const double* ybasis;         /* [n_moments][n_angles] */
    const double* coeffs;         /* [n_moments] */
    const double* redistribution; /* [n_freq][n_freq] R(nu, nu') */
    const double* gamma;          /* see gamma_per_ray */
    const double* inflow;         /* [n_angles*n_freq] boundary intensity per ray, or NULL for 0 (R/transfer.py:101-103) */
} rtk_slab_desc;

/*
 * Periodic-lattice long characteristics on a 2D slab (ny = 1, y-invariant,
 * periodic in x) or a 3D box (periodic in x and y): BASELINE configs 3-5.
 * Generalises the reference's 2D long characteristics (R/multidim.py:127-360;
 * operator defined in oracle/lattice.py and DESIGN.md section 11).  Nodes
 * s = (k*ny + j)*nx + i, k = 0 the top layer.  Unknown layout:
 *   RTK_LAYOUT_INTENSITY: I[s][a][f]  (n_total = n_space*n_dirs*n_freq)
 *   RTK_LAYOUT_MOMENTS:   u[s][l][f]  redistributed angular moments
 *                         u = sum_g R w_g m,  m = sum_a w_a Y_l(a) I
 *                         (n_total = n_space*n_moments*n_freq);
 *                         S[s][a][f] = gamma[s][f] sum_l coeffs[l] Y_l(a) u[s][l][f].
 * For lattice problems rtk_build_rhs takes thermal as [n_space][n_freq]
 * (isotropic thermal source).
 */
/* Characteristics of a lattice problem (TRIP chooses by ray inclination):
 * LONG   lines of the lattice family carry their values through all layers (T_RC to nodes);
 * SHORT  each layer step restarts at the upwind point of every node (bilinear from the
 *        previous layer's nodes) and integrates to the node with the same sub-segments;
 * HYBRID SHORT for steep directions (upwind point in the adjacent cell, n_sub = 1), LONG
 *        for grazing ones. */
#define RTK_CHAR_LONG 0
#define RTK_CHAR_SHORT 1
#define RTK_CHAR_HYBRID 2

typedef struct rtk_lattice_desc {
    int32_t nx, ny, nz;
    int32_t n_dirs;
    int32_t n_freq;
    int32_t n_moments;            /* 1..RTK_MAX_MOMENTS */
    int32_t formal_solver;        /* RTK_FS_IE, RTK_FS_EXP_LINEAR or RTK_FS_EXP_PARABOLIC */
    int32_t layout;               /* RTK_LAYOUT_* */
    double dx, dy, dz;
    const double* omega;          /* [n_dirs][3] unit vectors, omega_z != 0 */
    const double* dir_w;          /* [n_dirs] quadrature weights */
    const double* phi;            /* [n_freq] */
    const double* freq_w;         /* [n_freq] */
    const double* ybasis;         /* [n_moments][n_dirs] */
    const double* coeffs;         /* [n_moments] */
    const double* redistribution; /* [n_freq][n_freq] */
    const double* gamma;          /* [n_space][n_freq] */
    const double* chi;            /* [n_space] frequency-integrated opacity at nodes */
    const double* inflow_top;     /* [n_freq] incident on omega_z < 0 rays at k = 0, or NULL (0) */
    const double* inflow_bottom;  /* [n_freq] incident on omega_z > 0 rays at k = nz-1, or NULL (0) */
    int32_t characteristics;      /* RTK_CHAR_*: long (lattice family), short, or hybrid by inclination */
} rtk_lattice_desc;

const char* rtk_last_error_message(void);
int rtk_version(void);
/* Number of this library's kernels launched since load (bench / evidence counter). */
int64_t rtk_kernel_launch_count(void);

/* Build the device-resident operator: ONE host->device upload of the tables
 * (dt, phi, 1/|mu|, w*Y, R*w, gamma, inflow) plus the matvec workspace.
 * Replaces build_grid/build_transfer/build_scattering + RTProblem
 * (R/grid.py:115-150, R/transfer.py:88-104, R/scattering.py:85-100,
 * R/operator.py:28-45). */
int rtk_problem_create_slab(const rtk_slab_desc* desc, rtk_problem** out);
/* Multi-D lattice problem (configs 3-5); replaces CartesianGrid2D + build_transfer_2d
 * + build_scattering + RTProblem for the multi-D path (R/multidim.py:33-81, 322-360). */
int rtk_problem_create_lattice(const rtk_lattice_desc* desc, rtk_problem** out);
int rtk_problem_destroy(rtk_problem* p);
int64_t rtk_problem_n_total(const rtk_problem* p);
/* Re-upload inflow after a host-side edit (T/test_operator.py:88-110 mutate it).  Ordered
 * on `stream` after earlier work there; a no-op when the values are unchanged. */
int rtk_problem_set_inflow(rtk_problem* p, const double* inflow_host, int64_t n_rays, void* stream);
/* Kernel-variant selection of one handle (initialised at creation from the RTK_* environment
 * variables, read once then): "disable_tma", "lattice_dg" (0 auto, 1, 4, 8),
 * "lattice_no_smem", "lattice_no_dtab", "lattice_no_planar", "moments_scalar",
 * "sigma_unfused".  Every variant computes the same operator (tests run each one against
 * the oracle).  No reference counterpart.  Unknown key or value: RTK_EINVAL. */
int rtk_problem_set_tuning(rtk_problem* p, const char* key, int64_t value);

/* y = x - Lambda(Sigma x)  -- apply_A, R/operator.py:48-53.  x, y device, length n. */
int rtk_apply_A(rtk_problem* p, const double* x_dev, double* y_dev, int64_t n, void* stream);
/* apply_A with CUDA events between its kernels: ms_out[0..2] = moments, redistribution,
 * sweep durations (ms) on `stream` (synchronises).  When moments and redistribution ran
 * as the single fused kernel, ms_out[0] is its duration and ms_out[1] = -1.
 * Measurement hook for bench.py. */
int rtk_profile_apply_A(rtk_problem* p, const double* x_dev, double* y_dev, int64_t n, void* stream,
                        float* ms_out);
/* Same, host buffers in and out (H2D + matvec + D2H); the e2e path of the drop-in. */
int rtk_apply_A_host(rtk_problem* p, const double* x_host, double* y_host, int64_t n, void* stream);
/* Batched host-buffer apply_A: y_k = A x_k for k < count.  Two device buffer pairs and two
 * streams alternate, so the H2D copy of x_{k+1} overlaps the D2H copy of y_k (PCIe is full
 * duplex).  Host buffers should be pinned for the copies to be asynchronous. */
int rtk_apply_A_host_batch(rtk_problem* p, const double* const* x_host, double* const* y_host, int32_t count,
                           int64_t n);
/* Moment-layout problems: intensities I = Lambda(S(u) + thermal) + inflow term from a
 * moment vector u (the returned intensities of a moment-layout solve); thermal_dev and
 * I_dev are intensity-layout vectors of n_intensity = n_space * n_rays entries. */
int rtk_intensity_from_moments(rtk_problem* p, const double* u_dev, const double* thermal_dev, double* I_dev,
                               int64_t n_intensity, void* stream);
/* Direction sharding: a rank holds a problem built on ITS directions and the
 * matching slice of x.  rtk_partial_moments writes m[i][k][f] = sum_{a in this problem}
 * w_a Y_k(a) x[i,a,f] (n_m = n_space * n_moments * n_freq); after the moments of all ranks
 * are summed (one all-reduce), rtk_apply_A_with_moments returns y = x - Lambda Sigma x for
 * this problem's rays with Sigma built from the summed m.  Slab, intensity layout. */
int rtk_partial_moments(rtk_problem* p, const double* x_dev, double* m_dev, int64_t n_m, void* stream);
int rtk_apply_A_with_moments(rtk_problem* p, const double* x_dev, const double* m_dev, int64_t n_m, double* y_dev,
                             int64_t n, void* stream);
/* Direction sharding of a LATTICE problem in the moment layout (configs 4-5): every rank
 * holds the full problem and the full (replicated) unknown u; it transfers only the
 * directions [a0, a1).  rtk_lattice_partial_moments writes the partial angular moments
 * m[s][l][f] = sum_{a0 <= a < a1} w_a Y_l(a) (Lambda S(u))(s, a, f) (n_m = n_space *
 * n_moments * n_freq = n_total); after the moments of all ranks are summed (one
 * all-reduce), rtk_lattice_apply_with_moments returns y = u - R_w m.  The sum over a
 * partition of the directions is apply_A (rtk_apply_A) of the whole problem. */
int rtk_lattice_partial_moments(rtk_problem* p, const double* u_dev, double* m_dev, int64_t n_m, int32_t a0,
                                int32_t a1, void* stream);
int rtk_lattice_apply_with_moments(rtk_problem* p, const double* u_dev, const double* m_dev, int64_t n_m,
                                   double* y_dev, int64_t n, void* stream);
/* Space-sharded finish of the same operator (Krylov vectors sharded by space): for the node
 * block [node0, node1) (n_b = (node1 - node0) * n_moments * n_freq values, the block's slices
 * of u, of the fully summed moments m, and of y), y_b = u_b - R_w m_b.  With the partial
 * moments of all ranks reduce-scattered by space, the blocks of all ranks form apply_A. */
int rtk_lattice_apply_with_moments_nodes(rtk_problem* p, const double* u_dev, const double* m_dev, int64_t node0,
                                         int64_t node1, double* y_dev, void* stream);
/* s = Sigma x -- apply_scattering, R/scattering.py:126-148. */
int rtk_apply_sigma(rtk_problem* p, const double* x_dev, double* s_dev, int64_t n, void* stream);
/* y = Lambda s (homogeneous part) -- apply_transfer, R/transfer.py:134-141. */
int rtk_apply_lambda(rtk_problem* p, const double* s_dev, double* y_dev, int64_t n, void* stream);
/* y = boundary (inflow) term -- boundary_term, R/transfer.py:144-147 (overflow-free recursion). */
int rtk_boundary(rtk_problem* p, double* y_dev, int64_t n, void* stream);
/* b = Lambda thermal + boundary, or ones -- build_rhs, R/operator.py:56-64. */
int rtk_build_rhs(rtk_problem* p, const double* thermal_dev, double* b_dev, int64_t n,
                  int32_t override_ones, void* stream);
/* s = Sigma I + thermal (returned source function; no reference helper, R/operator.py:35). */
int rtk_source_function(rtk_problem* p, const double* intensity_dev, const double* thermal_dev,
                        double* s_dev, int64_t n, void* stream);

/* ---------------- Krylov (R/krylov.py) ---------------- */

/* Matvec callback: y = A x on device vectors, on `stream`; returns a status code. */
typedef int (*rtk_matvec_fn)(void* ctx, const double* x_dev, double* y_dev, int64_t n, void* stream);

/* Arnoldi orthogonalisation of rtk_gmres / rtk_gmres_problem:
 * REFERENCE  the reference's choice (R/krylov.py:98-104): modified Gram-Schmidt, one sweep,
 *            or two when reorthogonalize != 0 (MGS / MGS2);
 * MGS, MGS2  explicitly;
 * CGS2       classical Gram-Schmidt + one reorthogonalisation, fused into three streaming
 *            passes over the whole basis (fewest bytes and launches per iteration). */
#define RTK_ORTH_REFERENCE 0
#define RTK_ORTH_MGS 1
#define RTK_ORTH_MGS2 2
#define RTK_ORTH_CGS2 3

typedef struct rtk_solve_cfg {       /* SolveConfig, R/krylov.py:21-35 */
    double rel_tol;
    int32_t max_iter;
    int32_t restart;                 /* <= 0: no restart (SolveConfig.restart = None) */
    int32_t reorthogonalize;         /* second Gram-Schmidt sweep (SolveConfig.reorthogonalize) */
    int32_t orthogonalization;       /* RTK_ORTH_*; RTK_ORTH_REFERENCE follows reorthogonalize */
} rtk_solve_cfg;

typedef struct rtk_solve_report {    /* SolveReport, R/krylov.py:38-46 (solution stays on device) */
    int32_t iterations;
    int32_t converged;
    int32_t breakdown;
    int32_t n_history;               /* entries written to history_host (<= history_cap) */
    double true_residual;
    int32_t matvecs;                 /* total operator applications incl. restart/true-residual ones */
    int32_t reserved;
} rtk_solve_report;

/* Restarted GMRES with the reference's exact control flow (R/krylov.py:56-158):
 * x0 = 0, Givens least squares, recurrence-residual stop, true-residual guard
 * at 10 tol, breakdown at 1e-14 ||b||.  Arnoldi by cfg->orthogonalization with
 * deterministic device reductions; the Krylov basis stays in HBM.  x_dev
 * receives the solution.  A callable `apply` is invoked exactly in the
 * reference's order (no look-ahead); the library's own rtk_problem_matvec
 * lets the device run up to three Arnoldi steps ahead of the host. */
int rtk_gmres(rtk_matvec_fn apply, void* ctx, int64_t n, const double* b_dev, double* x_dev,
              const rtk_solve_cfg* cfg, rtk_solve_report* report,
              double* history_host, int32_t history_cap, void* stream);
/* Same, with the problem's own fused matvec (no callback crossing). */
int rtk_gmres_problem(rtk_problem* p, const double* b_dev, double* x_dev,
                      const rtk_solve_cfg* cfg, rtk_solve_report* report,
                      double* history_host, int32_t history_cap, void* stream);
/* BiCGStab (R/krylov.py:180-256) on device vectors. */
int rtk_bicgstab(rtk_matvec_fn apply, void* ctx, int64_t n, const double* b_dev, double* x_dev,
                 const rtk_solve_cfg* cfg, rtk_solve_report* report,
                 double* history_host, int32_t history_cap, void* stream);
/* rtk_matvec_fn adapter: ctx is an rtk_problem*. */
int rtk_problem_matvec(void* problem, const double* x_dev, double* y_dev, int64_t n, void* stream);

/* Device BLAS-1 used by the Krylov driver, exported for tests: deterministic
 * fixed-order reductions, result written to host. */
int rtk_dot(const double* x_dev, const double* y_dev, int64_t n, double* out_host, void* stream);
int rtk_block_dot(const double* const* vecs_host, int32_t k, const double* w_dev, int64_t n,
                  double* out_host, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RTK_B200_H */
