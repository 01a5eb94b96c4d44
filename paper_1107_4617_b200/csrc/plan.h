// plan.h — host-side planner for the shiftable raised-cosine range kernel.
//
// Internal to libsf.so (not part of the C-ABI).  Everything here runs in
// fp64 / long double on the host; the device receives fp32 copies.
//
// Eq.(1) for phi(t) = cos(gamma t)^N, gamma = 1/(sigma_r sqrt N)
// (reading R1: q_N of PAPER.md:202 in the sigma_r scaling of Eq.(6),
// PAPER.md:244-247):
//     cos(gamma t)^N = sum_{n=0..N} C(N,n) 2^-N e^{j (2n-N) gamma t}.
// Conjugate pairing (exact): terms n=k and n=N-k have opposite frequencies and
// equal weights, so for t = f(y) - f(x)
//     c_k e^{j w_k t} + c_k e^{-j w_k t} = 2 c_k Re( conj(z_k(x)) z_k(y) ),
//     z_k(v) = e^{j w_k (v - c)},  w_k = (2k-N) gamma  (any centring constant c),
// which is how Algorithm 2 step 3 is evaluated in real
// arithmetic: pair k < N/2 gets weight 2 c_k; for even N the middle term
// k = N/2 (w = 0) gets weight c_{N/2}.
#pragma once

#include <cmath>
#include <vector>

namespace sf {

constexpr double kRangeT = 255.0;        // uint8 dynamic range half-width (R2)

inline int nmin(double sigma_r) {
    // N0 = ceil((2T/(pi sigma_r))^2): smallest N with T/(sigma_r sqrt N) <= pi/2,
    // i.e. a non-negative unimodal kernel on [-T,T] (R2).
    const double q = 2.0 * kRangeT / (M_PI * sigma_r);
    const double n = std::ceil(q * q - 1e-12);
    return n < 1.0 ? 1 : (int)n;
}

inline int pair_count(int N) { return N / 2 + 1; }

struct PairPlan {
    std::vector<double> omega;   // w_k = (2k - N) gamma, k = 0..floor(N/2)
    std::vector<double> weight;  // 2 c_k (k < N/2) or c_{N/2} (k = N/2)
};

inline PairPlan plan_pairs(int N, double sigma_r) {
    PairPlan p;
    const int K = pair_count(N);
    p.omega.resize(K);
    p.weight.resize(K);
    const long double gamma = 1.0L / ((long double)sigma_r * sqrtl((long double)N));
    const long double lgN = lgammal((long double)N + 1.0L) - (long double)N * logl(2.0L);
    for (int k = 0; k < K; ++k) {
        // c_k = C(N,k)/2^N via log-gamma in long double (no overflow up to N = 2048)
        const long double lc = lgN - lgammal((long double)k + 1.0L) - lgammal((long double)(N - k) + 1.0L);
        const long double ck = expl(lc);
        p.omega[k] = (double)((long double)(2 * k - N) * gamma);
        p.weight[k] = (double)((2 * k == N) ? ck : 2.0L * ck);
    }
    return p;
}

// Terms dropped at each end for the truncated expansion (sf_filter_truncated,
// PAPER.md:279-280): the smallest n0 with C(N,n0) >= eps * C(N, N/2).
inline int truncation_n0(int N, double eps) {
    if (N < 0 || !(eps >= 0.0) || !(eps < 1.0)) return -1;
    const long double lcmax = lgammal((long double)N + 1.0L) - lgammal((long double)(N / 2) + 1.0L) -
                              lgammal((long double)(N - N / 2) + 1.0L);
    const long double lthr = (eps > 0.0) ? logl((long double)eps) + lcmax : -1e300L;
    int n0 = 0;
    while (n0 < N / 2) {
        const long double lc = lgammal((long double)N + 1.0L) - lgammal((long double)n0 + 1.0L) -
                               lgammal((long double)(N - n0) + 1.0L);
        if (lc >= lthr - 1e-12L) break;
        ++n0;
    }
    return n0;
}

}  // namespace sf
