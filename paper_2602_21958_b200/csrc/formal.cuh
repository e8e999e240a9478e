// Formal-solver step weights shared by every sweep kernel.
//
// IE is the reference's implicit Euler (R/_kernels.py:70-88):
//     acc <- (acc + d S_c) / (1 + d)
// evaluated as acc * r + (d S_c) r with r = 1/(1+d), so the only operation on
// the loop-carried chain is one FMA (<= 1 ulp per step from the division form;
// the recursion is contractive, so it does not accumulate).
//
// EXP_LINEAR (Olson-Kunasz) and EXP_PARABOLIC (Kunasz-Auer) are EXTENSIONS
// with e_k = int_0^d t^k e^{-(d-t)} dt: below EXP_SERIES_THRESHOLD e1, e2 come from
// their Taylor series (no transcendental, expm1-free and cancellation-free), above it
// from exp(-d) and the closed forms.  The CPU oracle (oracle/rt_oracle.py:
// exp_weights, oracle/rt_oracle_c.c) restates the same formulas.
#pragma once

#define RTK_EXP_SERIES_THRESHOLD 0.05

namespace rtk {

// h1(d) = e1 / d^2 = sum_{n=2}^{9} (-1)^n d^(n-2) / n!      (truncation < 1e-17 relative for d < 0.05)
__host__ __device__ __forceinline__ double e1_over_d2(double d) {
    double acc = -1.0 / 362880;
    acc = acc * d + 1.0 / 40320;
    acc = acc * d - 1.0 / 5040;
    acc = acc * d + 1.0 / 720;
    acc = acc * d - 1.0 / 120;
    acc = acc * d + 1.0 / 24;
    acc = acc * d - 1.0 / 6;
    acc = acc * d + 1.0 / 2;
    return acc;
}

// h2(d) = e2 / d^3 = 2 sum_{n=3}^{10} (-1)^(n+1) d^(n-3) / n!
__host__ __device__ __forceinline__ double e2_over_d3(double d) {
    double acc = -2.0 / 3628800;
    acc = acc * d + 2.0 / 362880;
    acc = acc * d - 2.0 / 40320;
    acc = acc * d + 2.0 / 5040;
    acc = acc * d - 2.0 / 720;
    acc = acc * d + 2.0 / 120;
    acc = acc * d - 2.0 / 24;
    acc = acc * d + 2.0 / 6;
    return acc;
}

struct ExpLin {
    double att, wu, wc;
};
struct ExpPar {
    double att, wu, wc, wd;
};

// Linear (Olson-Kunasz) weights, two paths (restated by rt_oracle.py::exp_weights /
// _linear_weights and rt_oracle_c.c):
//   d < 0.05 : w_c = d h1(d), e0 = d - d w_c, att = 1 - e0      (Taylor series, no transcendental)
//   else     : att = exp(-d), e0 = 1 - att, w_c = (d - e0) / d  (e0 loses <= 5e-15 relative at d = 0.05)
//   w_u = e0 - w_c
// Most (ray, segment) pairs of a wide-profile line are in the series path, which costs a
// third of the transcendental path (measured: a single expm1 path for every d was 30% slower).
__device__ __forceinline__ ExpLin exp_linear_weights(double d) {
    ExpLin w;
    double e0;
    if (d < RTK_EXP_SERIES_THRESHOLD) {
        w.wc = d * e1_over_d2(d);
        e0 = d - d * w.wc;
        w.att = 1.0 - e0;
    } else {
        w.att = exp(-d);
        e0 = 1.0 - w.att;
        w.wc = (d - e0) / d;
    }
    w.wu = e0 - w.wc;
    return w;
}

// exp(-d) for d >= 0 without the library call's special-case handling: d log2(e) =
// k + f, exp(-d) = 2^-k e^r with r = k ln2 - d in [-ln2/2, ln2/2] (Cody-Waite split of
// ln2), e^r by its degree-13 Taylor polynomial (remainder < 4e-19), 2^-k from the
// exponent field.  Within 2 ulp of exp(); 0 below the normal range (d > 708).
__device__ __forceinline__ double exp_neg_fast(double d) {
    if (d > 708.0) return 0.0;
    const double k = rint(d * 1.4426950408889634);
    double r = fma(k, 6.93147180369123816490e-01, -d);
    r = fma(k, 1.90821492927058770002e-10, r);
    double p = 1.0 / 6227020800.0;
    p = fma(p, r, 1.0 / 479001600.0);
    p = fma(p, r, 1.0 / 39916800.0);
    p = fma(p, r, 1.0 / 3628800.0);
    p = fma(p, r, 1.0 / 362880.0);
    p = fma(p, r, 1.0 / 40320.0);
    p = fma(p, r, 1.0 / 5040.0);
    p = fma(p, r, 1.0 / 720.0);
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const long long ebits = static_cast<long long>(1023 - static_cast<int>(k)) << 52;
    return p * __longlong_as_double(ebits);
}

// 1/x by the hardware approximation and two Newton steps (within 1 ulp)
__device__ __forceinline__ double rcp_fast(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// Weight-warp versions of the exponential weights (sweep_tma.cu): same formulas with
// exp_neg_fast and reciprocal multiplications; agree with the reference formulas to a
// few ulp (the parity tests bound the matvec at 1e-11).
__device__ __forceinline__ ExpLin exp_linear_weights_fast(double d) {
    ExpLin w;
    double e0;
    if (d < RTK_EXP_SERIES_THRESHOLD) {
        w.wc = d * e1_over_d2(d);
        e0 = d - d * w.wc;
        w.att = 1.0 - e0;
    } else {
        w.att = exp_neg_fast(d);
        e0 = 1.0 - w.att;
        w.wc = (d - e0) * rcp_fast(d);
    }
    w.wu = e0 - w.wc;
    return w;
}

__device__ __forceinline__ ExpPar exp_parabolic_weights_fast(double du, double dd) {
    ExpPar w;
    double e0, e1, e2;
    if (du < RTK_EXP_SERIES_THRESHOLD) {
        e1 = du * du * e1_over_d2(du);
        e2 = du * du * du * e2_over_d3(du);
        e0 = du - e1;
        w.att = 1.0 - e0;
    } else {
        w.att = exp_neg_fast(du);
        e0 = 1.0 - w.att;
        e1 = du - e0;
        e2 = du * du - 2.0 * e1;
    }
    const double s = du + dd;
    const double r = rcp_fast(du * dd * s);
    w.wu = e0 + (e2 - (dd + 2.0 * du) * e1) * (dd * r);
    w.wc = (s * e1 - e2) * (s * r);
    w.wd = (e2 - du * e1) * (du * r);
    return w;
}

// Branch-free exponential moments for the weight warps of the ring sweep
// (sweep_tma.cu).  With d ln2-range-reduced, d = k ln2 + r, |r| <= ln2/2, and z = -r:
//   V(z) = sum_{m>=0} z^m / (m+3)!   (degree 11: truncation < 3e-18 relative on |z| <= 0.347)
//   T(z) = (e^z - 1 - z) / z^2 = 1/2 + z V(z),   e^z - 1 = z + z^2 T(z)
// k = 0 (d < ln2/2): e0 = d - d^2 T, e1 = d^2 T, e2 = 2 d^3 V  (no cancellation: these are
//                    the series of e_k, as the d < 0.05 branch of the reference formulas);
// k > 0:             att = 2^-k e^-r, e0 = 1 - att, e1 = d - e0, e2 = d^2 - 2 e1 (the closed forms).
// Both paths are evaluated and selected, so a warp never diverges: every lane costs the
// same ~30 FP64 instructions and the compiler can interleave several weights per thread.
// Agrees with exp_linear_weights / exp_parabolic_weights to a few ulp (the parity tests
// bound the matvec at 1e-11 against the oracle's formulas).
struct ExpMom {
    double att, e0, e1, e2, t;   // t = e1 / d^2 on the k = 0 path
    bool small;
};

template <bool E2>
__device__ __forceinline__ ExpMom exp_moments_bf(double d) {
    const double dc = fmin(d, 708.0);
    // k = rint(dc log2 e) by the 1.5 * 2^52 shifter (k is the low word of kb), no FRND / F2I
    const double kb = fma(dc, 1.4426950408889634, 6755399441055744.0);
    const double kf = kb - 6755399441055744.0;
    const int k = __double2loint(kb);
    double r = fma(kf, -6.93147180369123816490e-01, dc);
    r = fma(kf, -1.90821492927058770002e-10, r);
    const double z = -r;
    double v = 1.0 / 87178291200.0;   // 1/14!
    v = fma(v, z, 1.0 / 6227020800.0);
    v = fma(v, z, 1.0 / 479001600.0);
    v = fma(v, z, 1.0 / 39916800.0);
    v = fma(v, z, 1.0 / 3628800.0);
    v = fma(v, z, 1.0 / 362880.0);
    v = fma(v, z, 1.0 / 40320.0);
    v = fma(v, z, 1.0 / 5040.0);
    v = fma(v, z, 1.0 / 720.0);
    v = fma(v, z, 1.0 / 120.0);
    v = fma(v, z, 1.0 / 24.0);
    v = fma(v, z, 1.0 / 6.0);
    const double t = fma(z, v, 0.5);
    const double z2 = z * z;
    const double em1 = fma(z2, t, z);
    // 2^-k (exactly 1 for k = 0, so att = 1 + em1 there); 0 beyond the normal range
    const double scale = d > 708.0 ? 0.0 : __hiloint2double((1023 - k) << 20, 0);
    ExpMom m;
    m.small = k == 0;
    m.t = t;
    m.att = scale * (1.0 + em1);
    m.e0 = m.small ? -em1 : 1.0 - m.att;
    m.e1 = m.small ? z2 * t : d - m.e0;
    if (E2) m.e2 = m.small ? 2.0 * (z2 * d) * v : fma(d, d, -2.0 * m.e1);
    return m;
}

// rint / F2I variant of exp_moments_bf.  Measured at cfg2 (same arithmetic, different
// schedule): exp-linear sweep 267 us with this one vs 352 us with the shifter; the
// exp-parabolic sweep is faster with the shifter (349 vs 357 us).
template <bool E2>
__device__ __forceinline__ ExpMom exp_moments_bf_rint(double d) {
    const double dc = fmin(d, 708.0);
    const double kf = rint(dc * 1.4426950408889634);
    double r = fma(kf, -6.93147180369123816490e-01, dc);
    r = fma(kf, -1.90821492927058770002e-10, r);
    const double z = -r;
    double v = 1.0 / 87178291200.0;   // 1/14!
    v = fma(v, z, 1.0 / 6227020800.0);
    v = fma(v, z, 1.0 / 479001600.0);
    v = fma(v, z, 1.0 / 39916800.0);
    v = fma(v, z, 1.0 / 3628800.0);
    v = fma(v, z, 1.0 / 362880.0);
    v = fma(v, z, 1.0 / 40320.0);
    v = fma(v, z, 1.0 / 5040.0);
    v = fma(v, z, 1.0 / 720.0);
    v = fma(v, z, 1.0 / 120.0);
    v = fma(v, z, 1.0 / 24.0);
    v = fma(v, z, 1.0 / 6.0);
    const double t = fma(z, v, 0.5);
    const double z2 = z * z;
    const double em1 = fma(z2, t, z);
    const long long ebits = static_cast<long long>(1023 - static_cast<int>(kf)) << 52;
    const double att_big = d > 708.0 ? 0.0 : __longlong_as_double(ebits) * (1.0 + em1);
    ExpMom m;
    m.small = kf == 0.0;
    m.t = t;
    m.att = m.small ? 1.0 + em1 : att_big;
    m.e0 = m.small ? -em1 : 1.0 - att_big;
    m.e1 = m.small ? z2 * t : d - m.e0;
    if (E2) m.e2 = m.small ? 2.0 * (z2 * d) * v : fma(d, d, -2.0 * m.e1);
    return m;
}

__device__ __forceinline__ ExpLin exp_linear_weights_bf(double d) {
    const ExpMom m = exp_moments_bf_rint<false>(d);
    ExpLin w;
    w.att = m.att;
    w.wc = m.small ? d * m.t : m.e1 * rcp_fast(d);
    w.wu = m.e0 - w.wc;
    return w;
}

__device__ __forceinline__ ExpPar exp_parabolic_weights_bf(double du, double dd) {
    const ExpMom m = exp_moments_bf<true>(du);
    ExpPar w;
    w.att = m.att;
    const double s = du + dd;
    const double r = rcp_fast(du * dd * s);
    w.wc = (s * m.e1 - m.e2) * (s * r);
    w.wd = (m.e2 - du * m.e1) * (du * r);
    w.wu = (m.e0 - w.wc) - w.wd;   // the three weights sum to e0
    return w;
}

// exp_parabolic_weights_bf with the Lagrange denominators taken from per-depth tables: with
// du = c dt_u, dd = c dt_d (c = phi_f / |mu| per ray, dt per depth),
//   1 / (du dd) = rc2 qc,   1 / (dd (du + dd)) = rc2 qd,   rc2 = 1 / c^2 (once per ray),
//   qc = 1 / (dt_u dt_d),   qd = 1 / (dt_d (dt_u + dt_d))  (tabulated per depth at setup),
// which replaces the per-element reciprocal (MUFU + 4 FMA) and 4 multiplies by 2 multiplies.
__device__ __forceinline__ ExpPar exp_parabolic_weights_tab(double du, double dd, double rc2, double qc, double qd) {
    const ExpMom m = exp_moments_bf<true>(du);
    ExpPar w;
    w.att = m.att;
    const double s = du + dd;
    w.wc = (s * m.e1 - m.e2) * (rc2 * qc);
    w.wd = (m.e2 - du * m.e1) * (rc2 * qd);
    w.wu = (m.e0 - w.wc) - w.wd;   // the three weights sum to e0
    return w;
}

// Parabolic (Kunasz-Auer) weights through upwind u, current c, downwind d nodes.
__device__ __forceinline__ ExpPar exp_parabolic_weights(double du, double dd) {
    ExpPar w;
    double e0, e1, e2;
    if (du < RTK_EXP_SERIES_THRESHOLD) {
        e1 = du * du * e1_over_d2(du);
        e2 = du * du * du * e2_over_d3(du);
        e0 = du - e1;
        w.att = 1.0 - e0;
    } else {
        w.att = exp(-du);
        e0 = 1.0 - w.att;
        e1 = du - e0;
        e2 = du * du - 2.0 * e1;
    }
    // one division: 1/(du dd s) shared by the three Lagrange weights
    const double s = du + dd;
    const double r = 1.0 / (du * dd * s);
    w.wu = e0 + (e2 - (dd + 2.0 * du) * e1) * (dd * r);
    w.wc = (s * e1 - e2) * (s * r);
    w.wd = (e2 - du * e1) * (du * r);
    return w;
}

}  // namespace rtk
