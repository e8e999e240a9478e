/*
 * C + OpenMP restatement of the reference 1D matvec y = x - Lambda(Sigma x)
 * -- TEST INFRASTRUCTURE / CPU BASELINE ONLY (see oracle/__init__.py).
 *
 * R/ = /root/reference/pkg/src/rtkrylov/.  Follows:
 *   apply_A                  R/operator.py:48-53
 *   apply_scattering (moment form)  R/scattering.py:126-148
 *   apply_transfer + sweeps  R/transfer.py:134-141, R/_kernels.py:70-88 (IE, division form)
 *   exp-linear / exp-parabolic: oracle extension, same weights and small-d
 *   branch as oracle/rt_oracle.py::exp_weights.
 * Parallelised over space nodes (moments, redistribution) and over
 * (direction, frequency block) ray groups (sweeps); vectorises over frequency.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define THRESH 0.05

/* h1 = e1/d^2, h2 = e2/d^3: 8-term Taylor series (csrc/formal.cuh, rt_oracle.py::exp_weights) */
static double h1(double d) {
    static const double c[8] = {1.0 / 2, -1.0 / 6, 1.0 / 24, -1.0 / 120, 1.0 / 720, -1.0 / 5040, 1.0 / 40320,
                                -1.0 / 362880};
    double acc = c[7];
    for (int k = 6; k >= 0; --k) acc = acc * d + c[k];
    return acc;
}

static double h2(double d) {
    static const double c[8] = {2.0 / 6, -2.0 / 24, 2.0 / 120, -2.0 / 720, 2.0 / 5040, -2.0 / 40320, 2.0 / 362880,
                                -2.0 / 3628800};
    double acc = c[7];
    for (int k = 6; k >= 0; --k) acc = acc * d + c[k];
    return acc;
}

/* att = e^-d, e0, e1, e2 (csrc/formal.cuh): series below THRESH, exp(-d) and closed forms above */
static void exp_w(double d, double* att, double* e0, double* e1, double* e2) {
    if (d < THRESH) {
        *e1 = d * d * h1(d);
        *e2 = d * d * d * h2(d);
        *e0 = d - *e1;
        *att = 1.0 - *e0;
    } else {
        *att = exp(-d);
        *e0 = 1.0 - *att;
        *e1 = d - *e0;
        *e2 = d * d - 2.0 * *e1;
    }
}

int rto_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * gamma: [n_space][n_freq]; ybasis: [n_mom][n_angles]; R: [n_freq][n_freq];
 * fs: 0 IE, 1 exp-linear, 2 exp-parabolic.  Work buffers allocated here.
 */
int rto_apply_A_slab(int64_t n_space, int n_angles, int n_freq, int n_mom, int fs, const double* t_nodes,
                     const double* mu, const double* ang_w, const double* phi, const double* freq_w,
                     const double* ybasis, const double* coeffs, const double* R, const double* gamma,
                     const double* x, double* y, int nthreads) {
    const int64_t n_rays = (int64_t)n_angles * n_freq;
    double* m = (double*)malloc(sizeof(double) * n_space * n_mom * n_freq);
    double* G = (double*)malloc(sizeof(double) * n_space * n_mom * n_freq);
    double* rw = (double*)malloc(sizeof(double) * n_freq * n_freq);
    if (!m || !G || !rw) {
        free(m);
        free(G);
        free(rw);
        return 2;
    }
    for (int f = 0; f < n_freq; ++f)
        for (int g = 0; g < n_freq; ++g) rw[(size_t)f * n_freq + g] = R[(size_t)f * n_freq + g] * freq_w[g];
    if (nthreads <= 0) nthreads = rto_max_threads();

    /* moments m[i,k,f] = sum_a w_a Y_k(a) x[i,a,f]; then G = c_k gamma sum_g R w m */
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t i = 0; i < n_space; ++i) {
        double* mi = m + i * n_mom * n_freq;
        memset(mi, 0, sizeof(double) * n_mom * n_freq);
        for (int a = 0; a < n_angles; ++a) {
            const double* xa = x + i * n_rays + (int64_t)a * n_freq;
            for (int k = 0; k < n_mom; ++k) {
                const double wy = ang_w[a] * ybasis[k * n_angles + a];
                double* mk = mi + k * n_freq;
                for (int f = 0; f < n_freq; ++f) mk[f] += wy * xa[f];
            }
        }
        double* Gi = G + i * n_mom * n_freq;
        for (int k = 0; k < n_mom; ++k) {
            const double* mk = mi + k * n_freq;
            for (int f = 0; f < n_freq; ++f) {
                const double* rf = rw + (size_t)f * n_freq;
                double s = 0.0;
                for (int g = 0; g < n_freq; ++g) s += rf[g] * mk[g];
                Gi[k * n_freq + f] = coeffs[k] * gamma[i * n_freq + f] * s;
            }
        }
    }

    /* sweeps: one task per (direction, block of 64 frequencies) */
    const int FB = 64;
    const int nfb = (n_freq + FB - 1) / FB;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
    for (int task = 0; task < n_angles * nfb; ++task) {
        const int a = task / nfb;
        const int f0 = (task % nfb) * FB;
        const int nf = (f0 + FB <= n_freq) ? FB : n_freq - f0;
        const int down = mu[a] < 0;
        double acc[64], sp[64], sc[64], sn[64];
        for (int q = 0; q < nf; ++q) acc[q] = 0.0;
        for (int64_t j = 0; j < n_space; ++j) {
            const int64_t i = down ? j : n_space - 1 - j;
            const int64_t ip = down ? j - 1 : n_space - j;   /* previous node */
            const int64_t in = down ? j + 1 : n_space - 2 - j; /* next node */
            for (int q = 0; q < nf; ++q) {
                const int f = f0 + q;
                double s = 0.0;
                for (int k = 0; k < n_mom; ++k) s += ybasis[k * n_angles + a] * G[(i * n_mom + k) * n_freq + f];
                sc[q] = s;
            }
            if (j > 0) {
                const double dt = down ? t_nodes[j] - t_nodes[j - 1] : t_nodes[ip] - t_nodes[i];
                const double dtn = (j + 1 < n_space) ? (down ? t_nodes[j + 1] - t_nodes[j] : t_nodes[i] - t_nodes[in]) : 0.0;
                for (int q = 0; q < nf; ++q) {
                    const int f = f0 + q;
                    const double d = phi[f] * dt / fabs(mu[a]);   /* (phi dt)/abs(mu), R/grid.py:104-105 */
                    if (fs == 0) {
                        acc[q] = (acc[q] + d * sc[q]) / (1.0 + d);
                    } else {
                        double att, e0, e1, e2;
                        exp_w(d, &att, &e0, &e1, &e2);
                        if (fs == 2 && j + 1 < n_space) {
                            double s = 0.0;
                            for (int k = 0; k < n_mom; ++k) s += ybasis[k * n_angles + a] * G[(in * n_mom + k) * n_freq + f];
                            sn[q] = s;
                            const double dd = phi[f] * dtn / fabs(mu[a]);
                            const double su = d + dd;
                            const double r = 1.0 / (d * dd * su);
                            const double wu = e0 + (e2 - (dd + 2.0 * d) * e1) * (dd * r);
                            const double wc = (su * e1 - e2) * (su * r);
                            const double wd = (e2 - d * e1) * (d * r);
                            acc[q] = att * acc[q] + wu * sp[q] + wc * sc[q] + wd * sn[q];
                        } else {
                            double wc;
                            if (d < THRESH) {
                                wc = d * h1(d);
                                e0 = d - d * wc;
                                att = 1.0 - e0;
                            } else {
                                wc = (d - e0) / d;
                            }
                            const double wu = e0 - wc;
                            acc[q] = att * acc[q] + wu * sp[q] + wc * sc[q];
                        }
                    }
                }
            }
            const double* xi = x + i * n_rays + (int64_t)a * n_freq + f0;
            double* yi = y + i * n_rays + (int64_t)a * n_freq + f0;
            for (int q = 0; q < nf; ++q) {
                yi[q] = xi[q] - acc[q];
                sp[q] = sc[q];
            }
        }
    }
    free(m);
    free(G);
    free(rw);
    return 0;
}
