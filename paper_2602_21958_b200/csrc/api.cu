// C-ABI entry points of librtk_b200 (declared in include/rtk_b200.h): problem
// lifetime, operator applications, RHS.  R/ = /root/reference/pkg/src/rtkrylov/.
#include <cuda_runtime.h>

#include <algorithm>
#include <thread>
#include <vector>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "rtk_internal.cuh"

struct rtk_problem {
    rtk::Problem impl;
};

namespace rtk {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_status(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) return RTK_ERESOURCE;
    return RTK_ECUDA;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

Problem::~Problem() {
    if (krylov_ws) destroy_krylov_workspace(krylov_ws);
    double* bufs[] = {dt, phi, inv_mu, wy, yb, rwt, gamma, coeffs, inflow, mom, gmom, host_x, host_y, host_x2, host_y2};
    for (auto st : io)
        if (st) cudaStreamDestroy(st);
    for (auto ev : io_done)
        if (ev) cudaEventDestroy(ev);
    for (double* b : bufs)
        if (b) cudaFree(b);
    if (dir_sign) cudaFree(dir_sign);
    for (int b = 0; b < 2; ++b) {
        if (stage[b]) cudaFreeHost(stage[b]);
        if (stage_ev[b]) cudaEventDestroy(stage_ev[b]);
    }
    if (tma_ctas) cudaFree(tma_ctas);
    if (dtpad) cudaFree(dtpad);
    if (par_tab) cudaFree(par_tab);
    if (lat_dirs) cudaFree(lat_dirs);
    if (mom_ctas) cudaFree(mom_ctas);
    if (mom_partial) cudaFree(mom_partial);
    if (dtpad_mom) cudaFree(dtpad_mom);
    if (lat_sub_shift) cudaFree(lat_sub_shift);
    if (lat_gat_shift) cudaFree(lat_gat_shift);
    if (lat_down_shift) cudaFree(lat_down_shift);
    if (lat_dtab) cudaFree(lat_dtab);
    if (lat_tile_hdr) cudaFree(lat_tile_hdr);
    if (lat_tile_sub) cudaFree(lat_tile_sub);
    if (lat_order) cudaFree(lat_order);
    if (lat_scratch) cudaFree(lat_scratch);
    double* lat[] = {lat_chi, lat_in_top, lat_in_bot, lat_state[0], lat_state[1], lat_src, lat_zero, lat_splane[0],
                     lat_splane[1], lat_splane[2]};
    for (double* b : lat)
        if (b) cudaFree(b);
}

bool getenv_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] && v[0] != '0';
}

static int getenv_int(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] ? std::atoi(v) : 0;
}

Tuning tuning_from_env() {
    Tuning t;
    t.disable_tma = getenv_flag("RTK_DISABLE_TMA");
    t.lat_dg = getenv_int("RTK_LAT_DG");
    t.lat_no_smem = getenv_flag("RTK_LATTICE_NO_SMEM");
    t.lat_no_dtab = getenv_flag("RTK_LATTICE_NO_DTAB");
    t.lat_no_planar = getenv_flag("RTK_LATTICE_NO_PLANAR");
    t.moments_scalar = getenv_flag("RTK_MOMENTS_SCALAR");
    t.sigma_unfused = getenv_flag("RTK_SIGMA_UNFUSED");
    t.lat_no_tile = getenv_flag("RTK_LATTICE_NO_TILE");
    t.lat_dgz = getenv_int("RTK_LAT_DGZ");
    return t;
}

int tuning_set(Tuning& t, const char* key, int64_t value) {
    const std::string k = key ? key : "";
    const int v = static_cast<int>(value);
    if (k == "disable_tma") t.disable_tma = v;
    else if (k == "lattice_dg") {
        if (v != 0 && v != 1 && v != 4 && v != 8) return 1;
        t.lat_dg = v;
    } else if (k == "lattice_no_smem") t.lat_no_smem = v;
    else if (k == "lattice_no_dtab") t.lat_no_dtab = v;
    else if (k == "lattice_no_planar") t.lat_no_planar = v;
    else if (k == "moments_scalar") t.moments_scalar = v;
    else if (k == "sigma_unfused") t.sigma_unfused = v;
    else if (k == "lattice_no_tile") t.lat_no_tile = v;
    else if (k == "lattice_dgz") {
        if (v < 0 || v > 8) return 1;
        t.lat_dgz = v;
    } else return 1;
    return 0;
}

bool pdl_enabled() {
    static const bool on = !getenv_flag("RTK_NO_PDL");
    return on;
}

namespace {
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, size_t> g_smem_set;              // (kernel, device) -> bytes set
std::map<std::pair<const void*, int>, std::map<int, int>> g_dev_cache;   // (kernel, device) -> slot -> value
}  // namespace

int ensure_smem(const void* func, size_t bytes) {
    if (bytes <= 48 * 1024) return RTK_OK;
    int dev = 0;
    RTK_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& have = g_smem_set[{func, dev}];
    if (have >= bytes) return RTK_OK;
    RTK_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    have = bytes;
    return RTK_OK;
}

int device_cache_get(const void* func, int slot) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_dev_cache.find({func, dev});
    if (it == g_dev_cache.end()) return -1;
    auto jt = it->second.find(slot);
    return jt == it->second.end() ? -1 : jt->second;
}

void device_cache_put(const void* func, int slot, int value) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_attr_mu);
    g_dev_cache[{func, dev}][slot] = value;
}

int upload(double** dst, const double* src, size_t count) {
    if (count == 0) count = 1;
    RTK_CUDA_TRY(cudaMalloc(dst, count * sizeof(double)));
    if (src) RTK_CUDA_TRY(cudaMemcpy(*dst, src, count * sizeof(double), cudaMemcpyHostToDevice));
    else RTK_CUDA_TRY(cudaMemset(*dst, 0, count * sizeof(double)));
    return RTK_OK;
}

// The TMA sweep where the problem's shape admits it (launch_sweep_tma returns -1 only for
// shapes it does not cover, decided at setup; a failing TMA launch is an error, never a
// silent switch to the slower kernel); otherwise, or with tune.disable_tma, the cp.async sweep.
int sweep_apply(const Problem& p, const double* x, double* y, cudaStream_t s) {
    if (!p.tune.disable_tma) {
        const int rc = launch_sweep_tma(p, x, y, s);
        if (rc != -1) return rc;
    }
    return launch_sweep(p, SRC_MOMENTS, OUT_X_MINUS, false, nullptr, x, y, s);
}

int apply_A_dev(Problem& p, const double* x, double* y, cudaStream_t s) {
    int rc;
    if (p.kind == KIND_SLAB && p.layout == LAYOUT_MOMENTS) {
        if ((rc = slab_moment_transfer(p, x, s))) return rc;
        return launch_redistribute_ex(p, p.mom, y, p.n_freq, EPI_SUB, x, p.n_freq, s);
    }
    if (p.kind == KIND_LATTICE) {
        if (p.layout == LAYOUT_MOMENTS) {
            if ((rc = lattice_transfer_moments(p, 2 /*LSRC_U*/, false, x, p.mom, s))) return rc;
            return launch_redistribute_ex(p, p.mom, y, p.n_freq, EPI_SUB, x, p.n_freq, s);
        }
        if ((rc = launch_sigma(p, x, s))) return rc;
        if ((rc = launch_expand_source(p, nullptr, p.lat_src, s))) return rc;
        return lattice_transfer_intensity(p, 0 /*LSRC_VEC*/, OUT_X_MINUS, false, p.lat_src, x, y, s);
    }
    if ((rc = launch_sigma(p, x, s))) return rc;
    return sweep_apply(p, x, y, s);
}

}  // namespace rtk

using rtk::Problem;
using rtk::set_error;

static int check_n(const rtk_problem* p, int64_t n) {
    if (!p) return set_error(RTK_EINVAL, "null problem handle");
    if (n != p->impl.n_total)
        return set_error(RTK_EINVAL, "expected length " + std::to_string(p->impl.n_total) + ", got " + std::to_string(n));
    return RTK_OK;
}

namespace rtk {
Problem* problem_impl(rtk_problem* p) { return p ? &p->impl : nullptr; }
}  // namespace rtk

extern "C" {

const char* rtk_last_error_message(void) { return rtk::g_last_error.c_str(); }

int rtk_version(void) { return 1; }

int64_t rtk_kernel_launch_count(void) { return rtk::g_launches.load(); }

int rtk_problem_create_slab(const rtk_slab_desc* d, rtk_problem** out) {
    if (!d || !out) return set_error(RTK_EINVAL, "null argument");
    *out = nullptr;
    if (d->n_space < 2) return set_error(RTK_EINVAL, "need at least 2 space nodes");
    if (d->n_angles < 1 || d->n_freq < 1) return set_error(RTK_EINVAL, "need at least one angle and one frequency");
    if (d->n_moments < 1 || d->n_moments > RTK_MAX_MOMENTS)
        return set_error(RTK_EINVAL, "n_moments must be in 1.." + std::to_string(RTK_MAX_MOMENTS));
    if (d->formal_solver < RTK_FS_IE || d->formal_solver > RTK_FS_EXP_PARABOLIC)
        return set_error(RTK_EINVAL, "unknown formal solver");
    if (!d->t_nodes || !d->mu || !d->ang_w || !d->phi || !d->freq_w || !d->ybasis || !d->coeffs ||
        !d->redistribution || !d->gamma)
        return set_error(RTK_EINVAL, "missing description array");
    for (int64_t i = 0; i + 1 < d->n_space; ++i)
        if (!(d->t_nodes[i + 1] > d->t_nodes[i])) return set_error(RTK_EINVAL, "t_nodes must be strictly increasing");
    for (int a = 0; a < d->n_angles; ++a)
        if (d->mu[a] == 0.0) return set_error(RTK_EINVAL, "mu = 0 is not an admissible direction");

    rtk_problem* h = new (std::nothrow) rtk_problem();
    if (!h) return set_error(RTK_ERESOURCE, "host allocation failed");
    Problem& p = h->impl;
    p.tune = rtk::tuning_from_env();
    p.n_space = d->n_space;
    p.n_angles = d->n_angles;
    p.n_freq = d->n_freq;
    p.n_mom = d->n_moments;
    p.fs = d->formal_solver;
    p.gamma_per_ray = d->gamma_per_ray ? 1 : 0;
    p.layout = d->layout == RTK_LAYOUT_MOMENTS ? rtk::LAYOUT_MOMENTS : rtk::LAYOUT_INTENSITY;
    if (d->layout != RTK_LAYOUT_INTENSITY && d->layout != RTK_LAYOUT_MOMENTS) {
        delete h;
        return set_error(RTK_EINVAL, "unknown layout");
    }
    if (p.layout == rtk::LAYOUT_MOMENTS && p.gamma_per_ray) {
        delete h;
        return set_error(RTK_EINVAL, "the moment layout needs a mu-independent gamma");
    }
    p.n_rays = static_cast<int64_t>(p.n_angles) * p.n_freq;
    p.n_total = p.n_space * p.n_rays;
    p.fp = (p.n_freq + 1) / 2 * 2;
    if (p.layout == rtk::LAYOUT_MOMENTS) p.n_total = p.n_space * p.n_mom * p.n_freq;
    p.h_mu.assign(d->mu, d->mu + p.n_angles);
    p.h_coeffs.assign(d->coeffs, d->coeffs + p.n_mom);

    // host-side table preparation (setup only, once per problem)
    std::vector<double> dt(p.n_space - 1), inv_mu(p.n_angles), wy(p.n_mom * p.n_angles);
    std::vector<double> rwt(static_cast<size_t>(p.n_freq) * p.fp, 0.0);
    std::vector<int> sign(p.n_angles);
    for (int64_t i = 0; i + 1 < p.n_space; ++i) dt[i] = d->t_nodes[i + 1] - d->t_nodes[i];
    for (int a = 0; a < p.n_angles; ++a) {
        inv_mu[a] = 1.0 / std::fabs(d->mu[a]);
        sign[a] = d->mu[a] < 0 ? -1 : 1;
    }
    for (int k = 0; k < p.n_mom; ++k)
        for (int a = 0; a < p.n_angles; ++a) wy[k * p.n_angles + a] = d->ang_w[a] * d->ybasis[k * p.n_angles + a];
    for (int f = 0; f < p.n_freq; ++f)
        for (int g = 0; g < p.n_freq; ++g)
            rwt[static_cast<size_t>(g) * p.fp + f] = d->redistribution[static_cast<size_t>(f) * p.n_freq + g] * d->freq_w[g];

    int rc = RTK_OK;
    const size_t gamma_count = static_cast<size_t>(p.n_space) * (p.gamma_per_ray ? p.n_rays : p.n_freq);
    const size_t mom_count = static_cast<size_t>(p.n_space) * p.n_mom * p.fp;
    if (!rc) rc = rtk::upload(&p.dt, dt.data(), dt.size());
    if (!rc) rc = rtk::upload(&p.phi, d->phi, p.n_freq);
    if (!rc) rc = rtk::upload(&p.inv_mu, inv_mu.data(), inv_mu.size());
    if (!rc) rc = rtk::upload(&p.wy, wy.data(), wy.size());
    if (!rc) rc = rtk::upload(&p.yb, d->ybasis, static_cast<size_t>(p.n_mom) * p.n_angles);
    if (!rc) rc = rtk::upload(&p.rwt, rwt.data(), rwt.size());
    if (!rc) rc = rtk::upload(&p.gamma, d->gamma, gamma_count);
    if (!rc) rc = rtk::upload(&p.coeffs, d->coeffs, p.n_mom);
    if (!rc) rc = rtk::upload(&p.inflow, d->inflow, p.n_rays);
    if (d->inflow) p.h_inflow.assign(d->inflow, d->inflow + p.n_rays);
    else p.h_inflow.assign(static_cast<size_t>(p.n_rays), 0.0);
    if (!rc) rc = rtk::upload(&p.mom, nullptr, mom_count);
    if (!rc) rc = rtk::upload(&p.gmom, nullptr, mom_count);
    if (!rc) {
        cudaError_t e = cudaMalloc(&p.dir_sign, sizeof(int) * p.n_angles);
        if (e == cudaSuccess) e = cudaMemcpy(p.dir_sign, sign.data(), sizeof(int) * p.n_angles, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) rc = rtk::cuda_status(e, "dir_sign upload");
    }
    if (!rc) rc = p.layout == rtk::LAYOUT_MOMENTS ? rtk::setup_slab_moments(p) : rtk::setup_tma(p);
    if (rc) {
        delete h;
        return rc;
    }
    *out = h;
    return RTK_OK;
}

int rtk_problem_create_lattice(const rtk_lattice_desc* d, rtk_problem** out) {
    if (!d || !out) return set_error(RTK_EINVAL, "null argument");
    *out = nullptr;
    if (d->nx < 1 || d->ny < 1 || d->nz < 2) return set_error(RTK_EINVAL, "lattice needs nx, ny >= 1 and nz >= 2");
    if (d->n_dirs < 1 || d->n_freq < 1) return set_error(RTK_EINVAL, "need at least one direction and frequency");
    if (d->n_moments < 1 || d->n_moments > RTK_MAX_MOMENTS)
        return set_error(RTK_EINVAL, "n_moments must be in 1.." + std::to_string(RTK_MAX_MOMENTS));
    if (d->formal_solver != RTK_FS_IE && d->formal_solver != RTK_FS_EXP_LINEAR &&
        d->formal_solver != RTK_FS_EXP_PARABOLIC)
        return set_error(RTK_EINVAL, "unknown formal solver");
    if (d->layout != RTK_LAYOUT_INTENSITY && d->layout != RTK_LAYOUT_MOMENTS)
        return set_error(RTK_EINVAL, "unknown layout");
    if (!(d->dx > 0 && d->dy > 0 && d->dz > 0)) return set_error(RTK_EINVAL, "spacings must be positive");
    if (d->characteristics != RTK_CHAR_LONG && d->characteristics != RTK_CHAR_SHORT &&
        d->characteristics != RTK_CHAR_HYBRID)
        return set_error(RTK_EINVAL, "characteristics must be RTK_CHAR_LONG, _SHORT or _HYBRID");
    if (!d->omega || !d->dir_w || !d->phi || !d->freq_w || !d->ybasis || !d->coeffs || !d->redistribution ||
        !d->gamma || !d->chi)
        return set_error(RTK_EINVAL, "missing description array");
    for (int a = 0; a < d->n_dirs; ++a)
        if (d->omega[3 * a + 2] == 0.0) return set_error(RTK_EINVAL, "omega_z = 0 is not an admissible direction");
    rtk_problem* h = new (std::nothrow) rtk_problem();
    if (!h) return set_error(RTK_ERESOURCE, "host allocation failed");
    Problem& p = h->impl;
    p.tune = rtk::tuning_from_env();
    p.kind = rtk::KIND_LATTICE;
    p.layout = d->layout;
    p.lat_nx = d->nx;
    p.lat_ny = d->ny;
    p.lat_nz = d->nz;
    p.n_space = static_cast<int64_t>(d->nx) * d->ny * d->nz;
    p.n_angles = d->n_dirs;
    p.n_freq = d->n_freq;
    p.n_mom = d->n_moments;
    p.fs = d->formal_solver;
    p.fp = (p.n_freq + 1) / 2 * 2;
    p.n_rays = static_cast<int64_t>(p.n_angles) * p.n_freq;
    p.n_total = p.layout == rtk::LAYOUT_MOMENTS ? p.n_space * p.n_mom * p.n_freq : p.n_space * p.n_rays;
    p.h_coeffs.assign(d->coeffs, d->coeffs + p.n_mom);
    std::vector<double> wy(p.n_mom * p.n_angles), rwt(static_cast<size_t>(p.n_freq) * p.fp, 0.0);
    for (int k = 0; k < p.n_mom; ++k)
        for (int a = 0; a < p.n_angles; ++a) wy[k * p.n_angles + a] = d->dir_w[a] * d->ybasis[k * p.n_angles + a];
    for (int f = 0; f < p.n_freq; ++f)
        for (int g = 0; g < p.n_freq; ++g)
            rwt[static_cast<size_t>(g) * p.fp + f] = d->redistribution[static_cast<size_t>(f) * p.n_freq + g] * d->freq_w[g];
    const size_t mom_count = static_cast<size_t>(p.n_space) * p.n_mom * p.fp;
    int rc = RTK_OK;
    if (!rc) rc = rtk::upload(&p.phi, d->phi, p.n_freq);
    if (!rc) rc = rtk::upload(&p.wy, wy.data(), wy.size());
    if (!rc) rc = rtk::upload(&p.yb, d->ybasis, static_cast<size_t>(p.n_mom) * p.n_angles);
    if (!rc) rc = rtk::upload(&p.rwt, rwt.data(), rwt.size());
    if (!rc) rc = rtk::upload(&p.gamma, d->gamma, static_cast<size_t>(p.n_space) * p.n_freq);
    if (!rc) rc = rtk::upload(&p.coeffs, d->coeffs, p.n_mom);
    if (!rc) rc = rtk::upload(&p.lat_chi, d->chi, p.n_space);
    if (!rc) rc = rtk::upload(&p.lat_in_top, d->inflow_top, p.n_freq);
    if (!rc) rc = rtk::upload(&p.lat_in_bot, d->inflow_bottom, p.n_freq);
    if (!rc) rc = rtk::upload(&p.mom, nullptr, mom_count);
    if (!rc && p.layout == rtk::LAYOUT_INTENSITY) {
        rc = rtk::upload(&p.gmom, nullptr, mom_count);
        if (!rc) rc = rtk::upload(&p.lat_src, nullptr, static_cast<size_t>(p.n_space) * p.n_rays);
    }
    if (!rc && p.layout == rtk::LAYOUT_MOMENTS) {
        const size_t plane = static_cast<size_t>(p.n_angles) * d->nx * d->ny * p.fp;   // pitch fp (pairs)
        rc = rtk::upload(&p.lat_state[0], nullptr, plane);
        if (!rc) rc = rtk::upload(&p.lat_state[1], nullptr, plane);
        if (!rc) rc = rtk::upload(&p.lat_splane[0], nullptr, plane);
        if (!rc) rc = rtk::upload(&p.lat_splane[1], nullptr, plane);
        // exp-parabolic reads the plane after next (downwind point of a step's last sub-node)
        if (!rc && d->formal_solver == RTK_FS_EXP_PARABOLIC) rc = rtk::upload(&p.lat_splane[2], nullptr, plane);
    }
    if (!rc) rc = rtk::upload(&p.lat_zero, nullptr, static_cast<size_t>(p.n_space) * p.n_freq);
    if (!rc) rc = rtk::setup_lattice(p, d);
    if (rc) {
        delete h;
        return rc;
    }
    *out = h;
    return RTK_OK;
}

int rtk_problem_destroy(rtk_problem* p) {
    delete p;
    return RTK_OK;
}

int64_t rtk_problem_n_total(const rtk_problem* p) { return p ? p->impl.n_total : -1; }

int rtk_problem_set_inflow(rtk_problem* p, const double* inflow_host, int64_t n_rays, void* stream) {
    if (!p) return set_error(RTK_EINVAL, "null problem handle");
    if (p->impl.kind == rtk::KIND_LATTICE) return set_error(RTK_EINVAL, "lattice inflow is fixed at creation");
    if (n_rays != p->impl.n_rays) return set_error(RTK_EINVAL, "inflow length must equal n_rays");
    Problem& q = p->impl;
    std::vector<double> want(static_cast<size_t>(n_rays), 0.0);
    if (inflow_host) std::memcpy(want.data(), inflow_host, sizeof(double) * n_rays);
    if (want == q.h_inflow) return RTK_OK;   // unchanged: no upload
    // stream-ordered after every earlier kernel on `stream` that may still read the old inflow;
    // the host copy `want` must outlive the transfer, so wait for it before returning
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    RTK_CUDA_TRY(cudaMemcpyAsync(q.inflow, want.data(), sizeof(double) * n_rays, cudaMemcpyHostToDevice, s));
    RTK_CUDA_TRY(cudaStreamSynchronize(s));
    q.h_inflow.swap(want);
    return RTK_OK;
}

int rtk_problem_set_tuning(rtk_problem* p, const char* key, int64_t value) {
    if (!p) return set_error(RTK_EINVAL, "null problem handle");
    if (rtk::tuning_set(p->impl.tune, key, value))
        return set_error(RTK_EINVAL, std::string("unknown tuning key or value: ") + (key ? key : "(null)"));
    return RTK_OK;
}

int rtk_apply_A(rtk_problem* p, const double* x, double* y, int64_t n, void* stream) {
    int rc = check_n(p, n);
    if (rc) return rc;
    return rtk::apply_A_dev(p->impl, x, y, static_cast<cudaStream_t>(stream));
}

int rtk_profile_apply_A(rtk_problem* p, const double* x, double* y, int64_t n, void* stream, float* ms_out) {
    int rc = check_n(p, n);
    if (rc) return rc;
    if (!ms_out) return set_error(RTK_EINVAL, "null ms_out");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (p->impl.kind == rtk::KIND_LATTICE || p->impl.layout == rtk::LAYOUT_MOMENTS) {   // whole operator (ms_out[2])
        cudaEvent_t e0, e1;
        RTK_CUDA_TRY(cudaEventCreate(&e0));
        RTK_CUDA_TRY(cudaEventCreate(&e1));
        RTK_CUDA_TRY(cudaEventRecord(e0, s));
        rc = rtk::apply_A_dev(p->impl, x, y, s);
        RTK_CUDA_TRY(cudaEventRecord(e1, s));
        RTK_CUDA_TRY(cudaEventSynchronize(e1));
        ms_out[0] = ms_out[1] = 0.0f;
        cudaEventElapsedTime(&ms_out[2], e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return rc;
    }
    cudaEvent_t ev[4];
    for (auto& e : ev) RTK_CUDA_TRY(cudaEventCreate(&e));
    // one untimed matvec first: the timed kernels and events are then enqueued while the GPU is
    // busy, so the first interval does not include the host's launch latency (tensor-map
    // encoding + cudaLaunchKernelEx on an idle stream added 10-70 us to it)
    rc = rtk::apply_A_dev(p->impl, x, y, s);
    RTK_CUDA_TRY(cudaEventRecord(ev[0], s));
    bool fused = false;
    if (!rc) {
        rc = rtk::launch_sigma_fused(p->impl, x, s);
        fused = rc != -1;
        if (!fused) rc = rtk::launch_moments(p->impl, x, s);
    }
    RTK_CUDA_TRY(cudaEventRecord(ev[1], s));
    if (!rc && !fused) rc = rtk::launch_redistribute(p->impl, s);
    RTK_CUDA_TRY(cudaEventRecord(ev[2], s));
    if (!rc) rc = p->impl.kind == rtk::KIND_SLAB ? rtk::sweep_apply(p->impl, x, y, s) : RTK_OK;
    RTK_CUDA_TRY(cudaEventRecord(ev[3], s));
    RTK_CUDA_TRY(cudaEventSynchronize(ev[3]));
    for (int k = 0; k < 3; ++k) cudaEventElapsedTime(&ms_out[k], ev[k], ev[k + 1]);
    if (fused) ms_out[1] = -1.0f;   // moments and redistribution ran as one kernel, timed in ms_out[0]
    for (auto& e : ev) cudaEventDestroy(e);
    return rc;
}

int rtk_problem_matvec(void* ctx, const double* x, double* y, int64_t n, void* stream) {
    return rtk_apply_A(static_cast<rtk_problem*>(ctx), x, y, n, stream);
}

namespace {
bool is_pageable(const void* ptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// host memcpy split over the machine's cores (pageable <-> pinned staging)
void parallel_copy(void* dst, const void* src, size_t bytes) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const size_t per = (bytes / hw + 63) / 64 * 64;
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < hw && t * per < bytes; ++t)
        pool.emplace_back([=] {
            const size_t off = t * per;
            std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, std::min(per, bytes - off));
        });
    std::memcpy(dst, src, std::min(per, bytes));
    for (auto& th : pool) th.join();
}
}  // namespace

namespace rtk {
// Pageable user buffers (e.g. a numpy array through the drop-in apply_A): the copies go
// through two pinned chunks owned by the problem, so the multithreaded host memcpy of one
// chunk overlaps the DMA of the other (cudaMemcpy from pageable memory would stage through
// the driver's small bounce buffers one thread at a time: ~6x slower at cfg2).
int staged_h2d(Problem& q, double* dst_dev, const double* src, int64_t n, cudaStream_t s) {
    const int64_t chunk = Problem::kStageChunk;
    for (int64_t i0 = 0, c = 0; i0 < n; i0 += chunk, ++c) {
        const int b = static_cast<int>(c & 1);
        const int64_t cnt = std::min(chunk, n - i0);
        RTK_CUDA_TRY(cudaEventSynchronize(q.stage_ev[b]));   // the DMA out of this chunk is done
        parallel_copy(q.stage[b], src + i0, sizeof(double) * cnt);
        RTK_CUDA_TRY(cudaMemcpyAsync(dst_dev + i0, q.stage[b], sizeof(double) * cnt, cudaMemcpyHostToDevice, s));
        RTK_CUDA_TRY(cudaEventRecord(q.stage_ev[b], s));
    }
    return RTK_OK;
}

int staged_d2h(Problem& q, double* dst, const double* src_dev, int64_t n, cudaStream_t s) {
    const int64_t chunk = Problem::kStageChunk;
    const int64_t nch = (n + chunk - 1) / chunk;
    auto issue = [&](int64_t c) -> int {
        const int b = static_cast<int>(c & 1);
        const int64_t i0 = c * chunk, cnt = std::min(chunk, n - i0);
        RTK_CUDA_TRY(cudaMemcpyAsync(q.stage[b], src_dev + i0, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s));
        RTK_CUDA_TRY(cudaEventRecord(q.stage_ev[b], s));
        return RTK_OK;
    };
    int rc;
    if ((rc = issue(0))) return rc;
    for (int64_t c = 0; c < nch; ++c) {
        const int b = static_cast<int>(c & 1);
        RTK_CUDA_TRY(cudaEventSynchronize(q.stage_ev[b]));
        if (c + 1 < nch && (rc = issue(c + 1))) return rc;   // next chunk's DMA overlaps this memcpy
        const int64_t i0 = c * chunk, cnt = std::min(chunk, n - i0);
        parallel_copy(dst + i0, q.stage[b], sizeof(double) * cnt);
    }
    return RTK_OK;
}

int ensure_staging(Problem& q) {
    for (int b = 0; b < 2; ++b) {
        if (!q.stage[b]) RTK_CUDA_TRY(cudaMallocHost(&q.stage[b], sizeof(double) * Problem::kStageChunk));
        if (!q.stage_ev[b]) {
            RTK_CUDA_TRY(cudaEventCreateWithFlags(&q.stage_ev[b], cudaEventDisableTiming));
            RTK_CUDA_TRY(cudaEventRecord(q.stage_ev[b], 0));
        }
    }
    return RTK_OK;
}
}  // namespace rtk

int rtk_apply_A_host(rtk_problem* p, const double* x_host, double* y_host, int64_t n, void* stream) {
    int rc = check_n(p, n);
    if (rc) return rc;
    Problem& q = p->impl;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!q.host_x) RTK_CUDA_TRY(cudaMalloc(&q.host_x, sizeof(double) * q.n_total));
    if (!q.host_y) RTK_CUDA_TRY(cudaMalloc(&q.host_y, sizeof(double) * q.n_total));
    const bool stage_in = is_pageable(x_host), stage_out = is_pageable(y_host);
    if ((stage_in || stage_out) && (rc = rtk::ensure_staging(q))) return rc;
    if (stage_in) {
        if ((rc = rtk::staged_h2d(q, q.host_x, x_host, n, s))) return rc;
    } else {
        RTK_CUDA_TRY(cudaMemcpyAsync(q.host_x, x_host, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    }
    if ((rc = rtk::apply_A_dev(q, q.host_x, q.host_y, s))) return rc;
    if (stage_out) {
        if ((rc = rtk::staged_d2h(q, y_host, q.host_y, n, s))) return rc;
    } else {
        RTK_CUDA_TRY(cudaMemcpyAsync(y_host, q.host_y, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    }
    RTK_CUDA_TRY(cudaStreamSynchronize(s));
    return RTK_OK;
}

int rtk_apply_A_host_batch(rtk_problem* p, const double* const* xs, double* const* ys, int32_t count, int64_t n) {
    int rc = check_n(p, n);
    if (rc) return rc;
    if (count < 0 || (count > 0 && (!xs || !ys))) return set_error(RTK_EINVAL, "bad batch arguments");
    Problem& q = p->impl;
    if (!q.host_x) RTK_CUDA_TRY(cudaMalloc(&q.host_x, sizeof(double) * q.n_total));
    if (!q.host_y) RTK_CUDA_TRY(cudaMalloc(&q.host_y, sizeof(double) * q.n_total));
    if (!q.host_x2) RTK_CUDA_TRY(cudaMalloc(&q.host_x2, sizeof(double) * q.n_total));
    if (!q.host_y2) RTK_CUDA_TRY(cudaMalloc(&q.host_y2, sizeof(double) * q.n_total));
    if (!q.io[0]) {
        for (auto& st : q.io) RTK_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        for (auto& ev : q.io_done) RTK_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    const size_t bytes = sizeof(double) * n;
    for (int k = 0; k < count; ++k) {
        const int b = k & 1;
        cudaStream_t st = q.io[b];
        double* dx = b ? q.host_x2 : q.host_x;
        double* dy = b ? q.host_y2 : q.host_y;
        RTK_CUDA_TRY(cudaMemcpyAsync(dx, xs[k], bytes, cudaMemcpyHostToDevice, st));
        // the two streams share the operator's workspace (moments, G): serialise the compute parts
        if (k > 0) RTK_CUDA_TRY(cudaStreamWaitEvent(st, q.io_done[1 - b], 0));
        if ((rc = rtk::apply_A_dev(q, dx, dy, st))) return rc;
        RTK_CUDA_TRY(cudaEventRecord(q.io_done[b], st));
        RTK_CUDA_TRY(cudaMemcpyAsync(ys[k], dy, bytes, cudaMemcpyDeviceToHost, st));
    }
    for (auto st : q.io) RTK_CUDA_TRY(cudaStreamSynchronize(st));
    return RTK_OK;
}

int rtk_intensity_from_moments(rtk_problem* p, const double* u, const double* thermal, double* I, int64_t n_int,
                               void* stream) {
    if (!p) return set_error(RTK_EINVAL, "null problem handle");
    Problem& q = p->impl;
    if (q.kind != rtk::KIND_SLAB || q.layout != rtk::LAYOUT_MOMENTS)
        return set_error(RTK_EINVAL, "intensity_from_moments needs a slab problem in the moment layout");
    if (n_int != q.n_space * q.n_rays) return set_error(RTK_EINVAL, "intensity length must be n_space * n_rays");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // G = c gamma u (pitch fp) -> S = sum_k Y_k G + thermal (intensity layout, into I) -> I = Lambda S + inflow
    int rc = rtk::slab_moment_fold(q, u, s);
    if (rc) return rc;
    double* tmp = nullptr;
    RTK_CUDA_TRY(cudaMalloc(&tmp, sizeof(double) * n_int));
    rc = rtk::launch_expand_source(q, thermal, tmp, s);
    if (!rc) rc = rtk::launch_sweep(q, rtk::SRC_VECTOR, rtk::OUT_ACC, true, tmp, nullptr, I, s);
    cudaError_t e = cudaStreamSynchronize(s);
    cudaFree(tmp);
    if (!rc && e != cudaSuccess) rc = rtk::cuda_status(e, "intensity_from_moments");
    return rc;
}

static int check_shard(const rtk_problem* p, int64_t n_m) {
    if (!p) return set_error(RTK_EINVAL, "null problem handle");
    const Problem& q = p->impl;
    if (q.kind != rtk::KIND_SLAB || q.layout != rtk::LAYOUT_INTENSITY)
        return set_error(RTK_EINVAL, "direction sharding needs a slab problem in the intensity layout");
    if (n_m != q.n_space * q.n_mom * q.n_freq)
        return set_error(RTK_EINVAL, "moment array must hold n_space * n_moments * n_freq values");
    return RTK_OK;
}

static int check_lattice_shard(const rtk_problem* p, int64_t n_m) {
    if (!p) return set_error(RTK_EINVAL, "null problem handle");
    const Problem& q = p->impl;
    if (q.kind != rtk::KIND_LATTICE || q.layout != rtk::LAYOUT_MOMENTS)
        return set_error(RTK_EINVAL, "lattice direction sharding needs a lattice problem in the moment layout");
    if (n_m != q.n_space * q.n_mom * q.n_freq)
        return set_error(RTK_EINVAL, "moment array must hold n_space * n_moments * n_freq values");
    return RTK_OK;
}

int rtk_lattice_partial_moments(rtk_problem* p, const double* u, double* m, int64_t n_m, int32_t a0, int32_t a1,
                                void* stream) {
    int rc = check_lattice_shard(p, n_m);
    if (rc) return rc;
    const Problem& q = p->impl;
    if (a0 < 0 || a1 > q.n_angles || a0 >= a1) return set_error(RTK_EINVAL, "direction range must satisfy 0 <= a0 < a1 <= n_dirs");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((rc = rtk::lattice_transfer_moments(q, 2 /*LSRC_U*/, false, u, q.mom, s, a0, a1))) return rc;
    RTK_CUDA_TRY(cudaMemcpy2DAsync(m, sizeof(double) * q.n_freq, q.mom, sizeof(double) * q.fp,
                                   sizeof(double) * q.n_freq, q.n_space * q.n_mom, cudaMemcpyDeviceToDevice, s));
    return RTK_OK;
}

int rtk_lattice_apply_with_moments(rtk_problem* p, const double* u, const double* m, int64_t n_m, double* y,
                                   int64_t n, void* stream) {
    int rc = check_lattice_shard(p, n_m);
    if (rc) return rc;
    if ((rc = check_n(p, n))) return rc;
    Problem& q = p->impl;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    RTK_CUDA_TRY(cudaMemcpy2DAsync(q.mom, sizeof(double) * q.fp, m, sizeof(double) * q.n_freq,
                                   sizeof(double) * q.n_freq, q.n_space * q.n_mom, cudaMemcpyDeviceToDevice, s));
    return rtk::launch_redistribute_ex(q, q.mom, y, q.n_freq, rtk::EPI_SUB, u, q.n_freq, s);
}

int rtk_lattice_apply_with_moments_nodes(rtk_problem* p, const double* u, const double* m, int64_t node0,
                                         int64_t node1, double* y, void* stream) {
    int rc = check_lattice_shard(p, p ? p->impl.n_total : 0);
    if (rc) return rc;
    Problem& q = p->impl;
    if (node0 < 0 || node1 > q.n_space || node0 >= node1)
        return set_error(RTK_EINVAL, "node range must satisfy 0 <= node0 < node1 <= n_space");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t nodes = node1 - node0;
    RTK_CUDA_TRY(cudaMemcpy2DAsync(q.mom, sizeof(double) * q.fp, m, sizeof(double) * q.n_freq,
                                   sizeof(double) * q.n_freq, nodes * q.n_mom, cudaMemcpyDeviceToDevice, s));
    return rtk::launch_redistribute_ex(q, q.mom, y, q.n_freq, rtk::EPI_SUB, u, q.n_freq, s, nodes,
                                       q.gamma + node0 * q.n_freq);
}

int rtk_partial_moments(rtk_problem* p, const double* x, double* m, int64_t n_m, void* stream) {
    int rc = check_shard(p, n_m);
    if (rc) return rc;
    const Problem& q = p->impl;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((rc = rtk::launch_moments(q, x, s))) return rc;   // -> q.mom, row pitch fp
    RTK_CUDA_TRY(cudaMemcpy2DAsync(m, sizeof(double) * q.n_freq, q.mom, sizeof(double) * q.fp,
                                   sizeof(double) * q.n_freq, q.n_space * q.n_mom, cudaMemcpyDeviceToDevice, s));
    return RTK_OK;
}

int rtk_apply_A_with_moments(rtk_problem* p, const double* x, const double* m, int64_t n_m, double* y, int64_t n,
                             void* stream) {
    int rc = check_shard(p, n_m);
    if (rc) return rc;
    if ((rc = check_n(p, n))) return rc;
    Problem& q = p->impl;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    RTK_CUDA_TRY(cudaMemcpy2DAsync(q.mom, sizeof(double) * q.fp, m, sizeof(double) * q.n_freq,
                                   sizeof(double) * q.n_freq, q.n_space * q.n_mom, cudaMemcpyDeviceToDevice, s));
    if ((rc = rtk::launch_redistribute(q, s))) return rc;   // G from the summed moments
    return rtk::sweep_apply(q, x, y, s);
}

int rtk_apply_sigma(rtk_problem* p, const double* x, double* s_out, int64_t n, void* stream) {
    int rc = check_n(p, n);
    if (rc) return rc;
    if (p->impl.layout == rtk::LAYOUT_MOMENTS) return set_error(RTK_EINVAL, "apply_sigma needs the intensity layout");
    if (p->impl.kind == rtk::KIND_SLAB && p->impl.layout == rtk::LAYOUT_MOMENTS)
        return set_error(RTK_EINVAL, "apply_sigma needs the intensity layout");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((rc = rtk::launch_sigma(p->impl, x, s))) return rc;
    return rtk::launch_expand_source(p->impl, nullptr, s_out, s);
}

int rtk_source_function(rtk_problem* p, const double* intensity, const double* thermal, double* s_out, int64_t n,
                        void* stream) {
    int rc = check_n(p, n);
    if (rc) return rc;
    if (p->impl.kind == rtk::KIND_LATTICE) return set_error(RTK_EINVAL, "source_function is implemented for slabs");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((rc = rtk::launch_sigma(p->impl, intensity, s))) return rc;
    return rtk::launch_expand_source(p->impl, thermal, s_out, s);
}

int rtk_apply_lambda(rtk_problem* p, const double* src, double* y, int64_t n, void* stream) {
    int rc = check_n(p, n);
    if (rc) return rc;
    if (p->impl.kind == rtk::KIND_SLAB && p->impl.layout == rtk::LAYOUT_MOMENTS)
        return set_error(RTK_EINVAL, "apply_lambda needs the intensity layout");
    if (p->impl.kind == rtk::KIND_LATTICE) {
        if (p->impl.layout == rtk::LAYOUT_MOMENTS) return set_error(RTK_EINVAL, "apply_lambda needs the intensity layout");
        return rtk::lattice_transfer_intensity(p->impl, 0, rtk::OUT_ACC, false, src, nullptr, y,
                                               static_cast<cudaStream_t>(stream));
    }
    return rtk::launch_sweep(p->impl, rtk::SRC_VECTOR, rtk::OUT_ACC, false, src, nullptr, y,
                             static_cast<cudaStream_t>(stream));
}

int rtk_boundary(rtk_problem* p, double* y, int64_t n, void* stream) {
    int rc = check_n(p, n);
    if (rc) return rc;
    if (p->impl.kind == rtk::KIND_SLAB && p->impl.layout == rtk::LAYOUT_MOMENTS)
        return set_error(RTK_EINVAL, "boundary needs the intensity layout");
    if (p->impl.kind == rtk::KIND_LATTICE) return rtk_build_rhs(p, nullptr, y, n, 0, stream);
    return rtk::launch_sweep(p->impl, rtk::SRC_ZERO, rtk::OUT_ACC, true, nullptr, nullptr, y,
                             static_cast<cudaStream_t>(stream));
}

int rtk_build_rhs(rtk_problem* p, const double* thermal, double* b, int64_t n, int32_t override_ones, void* stream) {
    int rc = check_n(p, n);
    if (rc) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (override_ones) {
        // b = 1 (named benchmark mode, R/operator.py:62-63)
        std::vector<double> ones(static_cast<size_t>(n), 1.0);
        RTK_CUDA_TRY(cudaMemcpyAsync(b, ones.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
        RTK_CUDA_TRY(cudaStreamSynchronize(s));
        return RTK_OK;
    }
    if (p->impl.kind == rtk::KIND_LATTICE) {
        const double* th = thermal ? thermal : p->impl.lat_zero;   // [n_space][n_freq] isotropic
        if (p->impl.layout == rtk::LAYOUT_MOMENTS) {
            if ((rc = rtk::lattice_transfer_moments(p->impl, 1 /*LSRC_ISO*/, true, th, p->impl.mom, s))) return rc;
            return rtk::launch_redistribute_ex(p->impl, p->impl.mom, b, p->impl.n_freq, rtk::EPI_PLAIN, nullptr, 0, s);
        }
        return rtk::lattice_transfer_intensity(p->impl, 1 /*LSRC_ISO*/, rtk::OUT_ACC, true, th, nullptr, b, s);
    }
    if (p->impl.layout == rtk::LAYOUT_MOMENTS) {
        // b_u = R_w M (Lambda thermal + inflow term): through a transient intensity vector (one-time setup)
        Problem& q = p->impl;
        double* tmp = nullptr;
        RTK_CUDA_TRY(cudaMalloc(&tmp, sizeof(double) * q.n_space * q.n_rays));
        if (thermal) rc = rtk::launch_sweep(q, rtk::SRC_VECTOR, rtk::OUT_ACC, true, thermal, nullptr, tmp, s);
        else rc = rtk::launch_sweep(q, rtk::SRC_ZERO, rtk::OUT_ACC, true, nullptr, nullptr, tmp, s);
        if (!rc) rc = rtk::launch_moments(q, tmp, s);
        if (!rc) rc = rtk::launch_redistribute_ex(q, q.mom, b, q.n_freq, rtk::EPI_PLAIN, nullptr, 0, s);
        cudaError_t e = cudaStreamSynchronize(s);
        cudaFree(tmp);
        if (!rc && e != cudaSuccess) rc = rtk::cuda_status(e, "moment RHS");
        return rc;
    }
    // one recursion carrying the inflow value: Lambda thermal + decay * inflow
    if (thermal)
        return rtk::launch_sweep(p->impl, rtk::SRC_VECTOR, rtk::OUT_ACC, true, thermal, nullptr, b, s);
    return rtk::launch_sweep(p->impl, rtk::SRC_ZERO, rtk::OUT_ACC, true, nullptr, nullptr, b, s);
}

}  // extern "C"
