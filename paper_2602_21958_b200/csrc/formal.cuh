// Formal-solver step weights shared by every sweep kernel.
//
// IE is the reference's implicit Euler (R/_kernels.py:70-88):
//     acc <- (acc + d S_c) / (1 + d)
// evaluated as acc * r + (d S_c) r with r = 1/(1+d), so the only operation on
// the loop-carried chain is one FMA (<= 1 ulp per step from the division form;
// the recursion is contractive, so it does not accumulate).
//
// EXP_LINEAR (Olson-Kunasz) and EXP_PARABOLIC (Kunasz-Auer) are EXTENSIONS
// with e_k = int_0^d t^k e^{-(d-t)} dt.  The small-d branch (Taylor series of
// e1 and e2 below EXP_SERIES_THRESHOLD, 12 terms) is the one the CPU oracle
// uses (oracle/rt_oracle.py: exp_weights) so both sides share it.
#pragma once

#define RTK_EXP_SERIES_THRESHOLD 0.05

namespace rtk {

__host__ __device__ __forceinline__ double e1_series(double d) {
    // sum_{n=2}^{13} (-1)^n d^n / n!  =  d^2 * (c2 + d (c3 + ... + d c13))
    const double c[12] = {1.0 / 2, -1.0 / 6, 1.0 / 24, -1.0 / 120, 1.0 / 720, -1.0 / 5040, 1.0 / 40320,
                          -1.0 / 362880, 1.0 / 3628800, -1.0 / 39916800, 1.0 / 479001600,
                          -1.0 / 6227020800.0};
    double acc = c[11];
#pragma unroll
    for (int k = 10; k >= 0; --k) acc = acc * d + c[k];
    return d * d * acc;
}

__host__ __device__ __forceinline__ double e2_series(double d) {
    // 2 sum_{n=3}^{14} (-1)^{n+1} d^n / n!
    const double c[12] = {2.0 / 6, -2.0 / 24, 2.0 / 120, -2.0 / 720, 2.0 / 5040, -2.0 / 40320,
                          2.0 / 362880, -2.0 / 3628800, 2.0 / 39916800, -2.0 / 479001600,
                          2.0 / 6227020800.0, -2.0 / 87178291200.0};
    double acc = c[11];
#pragma unroll
    for (int k = 10; k >= 0; --k) acc = acc * d + c[k];
    return d * d * d * acc;
}

struct ExpLin {
    double att, wu, wc;
};
struct ExpPar {
    double att, wu, wc, wd;
};

__device__ __forceinline__ ExpLin exp_linear_weights(double d) {
    ExpLin w;
    w.att = exp(-d);
    const double e0 = -expm1(-d);
    const double e1 = d < RTK_EXP_SERIES_THRESHOLD ? e1_series(d) : d - e0;
    w.wc = d > 0.0 ? e1 / d : 0.0;
    w.wu = e0 - w.wc;
    return w;
}

__device__ __forceinline__ ExpPar exp_parabolic_weights(double du, double dd) {
    ExpPar w;
    w.att = exp(-du);
    const double e0 = -expm1(-du);
    double e1, e2;
    if (du < RTK_EXP_SERIES_THRESHOLD) {
        e1 = e1_series(du);
        e2 = e2_series(du);
    } else {
        e1 = du - e0;
        e2 = du * du - 2.0 * e1;
    }
    const double s = du + dd;
    w.wu = e0 + (e2 - (dd + 2.0 * du) * e1) / (du * s);
    w.wc = (s * e1 - e2) / (du * dd);
    w.wd = (e2 - du * e1) / (dd * s);
    return w;
}

}  // namespace rtk
