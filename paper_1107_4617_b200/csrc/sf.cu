// sf.cu — C-ABI entry points of libsf.so (see include/sf.h) and launch logic.
//
// The kernels live in box_kernel.cuh.  This file: argument validation (no
// enqueue on error), the fp64 planner call (plan.h), parameter packing and
// launches on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/sf.h"
#include "box_kernel.cuh"
#include "box_v4.cuh"
#include "box_v4r.cuh"
#include "box_small.cuh"
#include "v5_dispatch.h"
#include "v7_dispatch.h"
#include "v7q_dispatch.h"
#include "v7w_dispatch.h"
#include "nlm_kernel.cuh"
#include "nlm_dispatch.h"
#include "plan.h"
#include "poly_kernel.cuh"
#include "runtime.h"

namespace sf {

constexpr int kMaxBands = 8;                 // ranks of a fused term split (one NVLink domain)

struct BandTable {                           // by value; band o = rows [o*H/nband, (o+1)*H/nband)
    float* num[kMaxBands];
    float* den[kMaxBands];
    int nband;
};

// add the partial images into the band owners' buffers (atomics; peer memory
// for the fused term split).  Block row blockIdx.y = band.
__global__ void band_add_kernel(const float* __restrict__ pnum, const float* __restrict__ pden, int H, int W,
                                BandTable t) {
    const int o = blockIdx.y;
    const int b0 = (int)((long)o * H / t.nband), b1 = (int)((long)(o + 1) * H / t.nband);
    float* dn = t.num[o];
    float* dd = t.den[o];
    const size_t n = (size_t)(b1 - b0) * W, base = (size_t)b0 * W;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        atomicAdd(dn + i, pnum[base + i]);
        atomicAdd(dd + i, pden[base + i]);
    }
}

inline cudaError_t launch_band_add(const float* pnum, const float* pden, int H, int W, const BandTable& t,
                                   cudaStream_t s) {
    const size_t per = ((size_t)H * W / t.nband + 255) / 256;
    const unsigned bx = (unsigned)(per < 1 ? 1 : (per > 1184 ? 1184 : per));
    band_add_kernel<<<dim3(bx, t.nband), 256, 0, s>>>(pnum, pden, H, W, t);
    return cudaGetLastError();
}

// sf_finalize: out = c + P'/Q, the last line of Algorithm 2
__global__ void finalize_kernel(const float* __restrict__ num, const float* __restrict__ den,
                                const uint8_t* __restrict__ img, size_t n, float* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float q = den[i];
        out[i] = (q > 0.f && isfinite(q)) ? kCenter + num[i] / q : (float)img[i];
    }
}

inline cudaError_t launch_finalize(const float* num, const float* den, const uint8_t* img, size_t n,
                                   float* out, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t blocks = (n + 255) / 256;
    const size_t cap = (size_t)sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    finalize_kernel<<<(unsigned)blocks, 256, 0, s>>>(num, den, img, n, out);
    return cudaGetLastError();
}

}  // namespace sf

namespace {

thread_local int g_last_launches = 0;

bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
    const char* pa = static_cast<const char*>(a);
    const char* pb = static_cast<const char*>(b);
    return pa < pb + nb && pb < pa + na;
}

sf_status validate(const void* img, int H, int W, int radius, int kind, double sigma_r, int N) {
    if (!img) return SF_ERR_NULL;
    if (H < 1 || W < 1) return SF_ERR_SHAPE;
    if (sf::spatial_order(kind) < 0) return SF_ERR_KIND;
    if (!std::isfinite(sigma_r) || !(sigma_r > 0.0)) return SF_ERR_SIGMA;
    if (radius < 0 || radius > SF_MAX_RADIUS || radius > (H < W ? H : W) - 1) return SF_ERR_RADIUS;
    if (N > SF_MAX_ORDER || N < sf::nmin(sigma_r)) return SF_ERR_ORDER;
    return SF_OK;
}

double gamma_of(int N, double sigma_r) { return 1.0 / (sigma_r * std::sqrt((double)N)); }

sf::PairTable make_table(int N, double sigma_r, int pb, int pe) {
    const sf::PairPlan plan = sf::plan_pairs(N, sigma_r);
    sf::PairTable t;
    std::memset(&t, 0, sizeof(t));
    t.npairs = pe - pb;
    for (int k = pb; k < pe; ++k) {
        t.omega[k - pb] = (float)plan.omega[k];
        t.weight[k - pb] = (float)plan.weight[k];
    }
    return t;
}

// Kernel variant.  Default: the fastest for the case.  The
// environment variable SF_VARIANT = v1 | v4 | v4b | v5 | v5m | v7 | v7m | v7d pins one
// for A/B timing
// (tools/variants.py); every variant is a full CUDA implementation.
int variant() {
    static int v = [] {
        const char* e = std::getenv("SF_VARIANT");
        if (!e) return 0;
        if (!std::strcmp(e, "v1")) return 1;
        if (!std::strcmp(e, "v4")) return 4;
        if (!std::strcmp(e, "v5m")) return 6;
        if (!std::strcmp(e, "v5")) return 5;
        if (!std::strcmp(e, "v4b")) return 3;
        if (!std::strcmp(e, "v7")) return 11;
        if (!std::strcmp(e, "v7m")) return 12;
        if (!std::strcmp(e, "v7d")) return 13;
        if (!std::strcmp(e, "vs")) return 14;
        if (!std::strcmp(e, "v7w")) return 15;
        return 0;
    }();
    return v;
}

// v5 running-sum policy.  With the outgoing rows by rotation (om = false)
// the incoming (MUFU) and outgoing (rotated) stack values of a row differ by
// a few ulp, and the vertical running sums integrate the difference: the
// output error grows ~ kDriftCoef * rows * w_max^4 grey levels (measured on
// cfg4/cfg5, reading R15).  Segments are capped to keep it under
// kDriftBudget; when that cap would be short (< 256 rows: init-heavy), the
// outgoing rows are taken by MUFU as well (om = true), which makes them
// bit-identical to the incoming ones, so the sums do not drift at all.  On
// small images (< 1 Mpixel) the segments are short anyway and MUFU outgoing
// rows measured faster (cfg1 256^2: 0.037 vs 0.041 ms).
constexpr double kDriftCoef = 3.6e-5, kDriftBudget = 0.0125;

struct V5Choice {
    bool om;
    int maxseg;   // RB-row batches, 0 = unlimited
};

V5Choice v5_choice(int R, double pixels, const sf::PairTable& t, int v) {
    double wmax = 0.0;
    for (int k = 0; k < t.npairs; ++k) wmax = std::fmax(wmax, std::fabs((double)t.omega[k]));
    const double w4 = wmax * wmax * wmax * wmax;
    const double rows = w4 > 0.0 ? kDriftBudget / (kDriftCoef * w4) : 1e9;
    V5Choice c;
    c.om = v == 6 || v == 12 || (v != 5 && v != 11 && (R > 32 || rows < 256.0 || pixels < 1e6));
    c.maxseg = (c.om || rows >= 1e6) ? 0 : std::max(1, (int)(rows / 16.0));
    return c;
}

cudaError_t launch_v5(const sf::Params& p, const sf::PairTable& t, double gamma, cudaStream_t s, int v) {
    const V5Choice c = v5_choice(p.r, (double)p.out_rows * p.W, t, v);
    if ((v == 11 || v == 12 || v == 13) && p.r <= sf::kV7MaxR) return sf::launch_v7(p.r, c.om, c.maxseg, p, t, gamma, s);
    return sf::launch_v5(p.r, c.om, c.maxseg, false, p, t, gamma, s);
}

// Default per radius = the fastest measured on B200 for cfg5 (8192^2, N=118;
// profiles/r01_radius_sweep.jsonl): the single-consumer-warp ring kernel v4r
// for R = 4, 5 (short halo; and up to 8 on images of 1-8 Mpixel), the
// 8-consumer-warp v5 for every other radius 1..64, the runtime-radius v4b
// beyond (and for R = 0).
template <int R>
cudaError_t launch_ring(const sf::Params& p, const sf::PairTable& t, double gamma, cudaStream_t s) {
    int v = variant();
    // (R = 6..8: v4r on small images, where v5's per-CTA band-top init is a
    // larger share — cfg2 1080x1920 r=8: v4r 0.267 ms, v5 0.293 ms; below
    // 1 Mpixel v4r leaves most SMs idle and v5 wins — cfg1 256^2 r=5:
    // 0.037 vs 0.049 ms)
    const double pixels = (double)p.out_rows * p.W;
    if (v == 0 && pixels >= 1e6 && (R <= 5 || (R <= 8 && pixels < 8e6))) v = 4;
    if (v == 4) return sf::launch_box_v4r<R>(p, t, gamma, s);
    return launch_v5(p, t, gamma, s, v);
}

// q_M exponent of a spatial kind (0: box or unknown)
int spatial_m(int kind) {
    if (kind == SF_SPATIAL_RAISED_COS) return 2;
    return (kind > 100 && kind <= 108) ? kind - 100 : 0;
}

// outputs per v7q consumer lane (box_v7q.cuh: V7QG)
int v7q_g(int R, int F) {
    int g = (256 - 2 * R) / 16;
    g = g > 15 ? 15 : g;
    g -= (g % 2 == 0);
    return (F == 1 || g <= 9) ? g : 9;
}

// v7q modulation table for w1(u) = cos(beta u)^M = a_0 + sum_m a_m cos(nu_m u):
// binomial expansion of cos^M, nu_m = (M - 2m) beta,
// a_m = 2 C(M,m)/2^M (m < M/2), a_0 = C(M,M/2)/2^M for even M; fp64, cast once
sf::QModTab qmod_table(int R, int M, double beta, int G) {
    sf::QModTab q{};
    const int F = (M + 1) / 2, L = 2 * R + 1, RB = sf::kQRB;
    q.a0 = (M % 2 == 0) ? (float)sf::binom_over_2m(M, M / 2) : 0.f;
    for (int m = 0; m < F; ++m) {
        const double nu = (M - 2 * m) * beta, a = 2.0 * sf::binom_over_2m(M, m);
        // the running sums are kept pre-scaled by their weight a_m (the update
        // factors carry it), so the recombination at the centre is unscaled
        for (int i = 0; i < RB; ++i) {
            q.vic[m][i] = (float)(a * std::cos(nu * (i + R)));
            q.vis[m][i] = (float)(a * std::sin(nu * (i + R)));
            q.voc[m][i] = (float)(-a * std::cos(nu * (i - R - 1)));
            q.vos[m][i] = (float)(-a * std::sin(nu * (i - R - 1)));
            q.vac[m][i] = (float)std::cos(nu * i);
            q.vas[m][i] = (float)std::sin(nu * i);
        }
        q.rbc[m] = (float)std::cos(nu * RB);
        q.rbs[m] = (float)std::sin(nu * RB);
        for (int i = 0; i < L; ++i) {
            q.ic[m][i] = (float)(a * std::cos(nu * (i - R - 1)));
            q.is[m][i] = (float)(a * std::sin(nu * (i - R - 1)));
        }
        for (int j = 0; j < G; ++j) {
            q.hoc[m][j] = (float)(a * std::cos(nu * j));
            q.hos[m][j] = (float)(a * std::sin(nu * j));
            q.hic[m][j] = (float)(a * std::cos(nu * (j + L)));
            q.his[m][j] = (float)(a * std::sin(nu * (j + L)));
            q.hac[m][j] = (float)std::cos(nu * (j + R));
            q.has[m][j] = (float)std::sin(nu * (j + R));
        }
        q.rhc[m] = (float)std::cos(nu * G);
        q.rhs[m] = (float)std::sin(nu * G);
    }
    return q;
}

// small images (box_small.cuh): the small-image kernel while
// its tiles x pairs stay under ~40 pair steps per SM (measured crossover with
// v7's pair split: 256^2 with 16 pairs 20 vs 28 us, 384^2 34 vs 43 us; 256^2
// with 60 pairs and 512^2 with 16 pairs favour v7)
bool small_image(const sf::Params& p, const sf::PairTable& t) {
    const long tiles = (long)((p.W + sf::VsCfg<1>::TW - 1) / sf::VsCfg<1>::TW) *
                       ((p.out_rows + sf::VsCfg<1>::TH - 1) / sf::VsCfg<1>::TH);
    static const long cap = [] {
        const char* v = std::getenv("SF_VS_WORK");   // tools override of the crossover
        return v ? std::atol(v) : 0L;
    }();
    return tiles * t.npairs <= (cap > 0 ? cap : 40L * sf::current_device_info().sms);
}

sf_status launch(const sf::Params& p, const sf::PairTable& t, double gamma, cudaStream_t s) {
    cudaError_t e;
    sf::launch_counter() = 1;
    const bool box = p.kind == SF_SPATIAL_BOX;   // q_M: v7q (M <= 4, r <= 24), else v1
    // default box dispatch (profiles/r02_*): the small-image
    // kernel on images of a few pair steps per SM; v7 with the outgoing rows by
    // MUFU for r = 1..24, the wide v7 (v7w) for 25..64 (all with the
    // per-segment centre, reading R16), v4b for r = 0
    if (box && (variant() == 14 || (variant() == 0 && small_image(p, t))) && p.r >= 1 && p.r <= sf::kVsMaxR) {
        e = sf::launch_box_small(p, t, gamma, s);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return SF_ERR_CUDA;
        }
        g_last_launches = sf::launch_counter();
        return SF_OK;
    }
    if (box && variant() == 0 && p.r >= 1 && p.r <= sf::kV7MaxR) {
        e = launch_v5(p, t, gamma, s, 12);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return SF_ERR_CUDA;
        }
        g_last_launches = sf::launch_counter();
        return SF_OK;
    }
    // r = 25..64: the wide v7 (12 producer warps, 256-column strips, telescoping
    // start windows; cfg5 r = 64 12.4 -> 10.85 ms against v5), r = 9..24 with
    // SF_VARIANT=v7w (slower there than v7: 10.1 vs 8.9 ms at r = 16)
    if (box && (variant() == 15 || (variant() == 0 && p.r > sf::kV7MaxR)) && p.r >= sf::kV7WMinR &&
        p.r <= sf::kV7WMaxR) {
        e = sf::launch_v7w(p.r, p, t, gamma, s);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return SF_ERR_CUDA;
        }
        g_last_launches = sf::launch_counter();
        return SF_OK;
    }
    if (box && variant() == 0 && p.r > sf::kV7MaxR && p.r <= sf::kV5MaxR) {
        e = launch_v5(p, t, gamma, s, 6);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return SF_ERR_CUDA;
        }
        g_last_launches = sf::launch_counter();
        return SF_OK;
    }
    // separable q_M (M <= 4, r <= 24): the v7q band sweep (box_v7q.cuh)
    const int qm = spatial_m(p.kind);
    if (qm >= 1 && qm <= sf::kV7QMaxM && p.r >= 1 && p.r <= sf::kV7QMaxR && variant() == 0) {
        const double beta = p.beta > 0.f ? (double)p.beta : M_PI / (2.0 * (p.r + 1));
        const int F = (qm + 1) / 2;
        const sf::QModTab qt = qmod_table(p.r, qm, beta, v7q_g(p.r, F));
        e = sf::launch_v7q(p.r, F, p, t, qt, gamma, s);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return SF_ERR_CUDA;
        }
        g_last_launches = sf::launch_counter();
        return SF_OK;
    }
    if (!box || variant() == 1) e = sf::launch_box(p, t, s);   // q_M beyond v7q's range: tile kernel
    else if (p.r == 4) e = launch_ring<4>(p, t, gamma, s);
    else if (p.r == 5) e = launch_ring<5>(p, t, gamma, s);
    else if (p.r == 8) e = launch_ring<8>(p, t, gamma, s);
    else if (p.r == 10) e = launch_ring<10>(p, t, gamma, s);
    else if (p.r == 16) e = launch_ring<16>(p, t, gamma, s);
    else if (p.r >= 1 && p.r <= sf::kV5MaxR && variant() != 3) e = launch_v5(p, t, gamma, s, variant());
    else e = sf::launch_box_v4b(p, t, gamma, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return SF_ERR_CUDA;
    }
    g_last_launches = sf::launch_counter();
    return SF_OK;
}

// sf_accumulate: partials over a pair range, stored into num/den.
// sf_accumulate_add / sf_accumulate_scatter: the same partials computed into
// pool scratch, then one scatter-add pass (band_add_kernel) adds each row into
// its band owner's buffer (fp32 atomics, a peer GPU's memory over NVLink for
// the fused term split).  The add is a separate pass, not the filter's
// epilogue: an atomic epilogue in the hot kernels measured 3-13 % slower
// filters from register allocation alone.
sf_status accumulate_impl(const uint8_t* img, int H, int W, int radius, int kind, double sigma_r, int N,
                          int pair_begin, int pair_end, float* num, float* den, void* stream, int accum,
                          int nband = 0, float* const* band_num = nullptr, float* const* band_den = nullptr) {
    g_last_launches = 0;
    sf_status st = validate(img, H, W, radius, kind, sigma_r, N);
    if (st != SF_OK) return st;
    if (pair_begin < 0 || pair_end > sf::pair_count(N) || pair_begin > pair_end) return SF_ERR_RANGE;
    sf::BandTable bt{};
    if (accum == 2) {
        if (!band_num || !band_den) return SF_ERR_NULL;
        if (nband < 1 || nband > sf::kMaxBands || nband > H) return SF_ERR_RANGE;
        for (int o = 0; o < nband; ++o) {
            if (!band_num[o] || !band_den[o]) return SF_ERR_NULL;
            bt.num[o] = band_num[o];
            bt.den[o] = band_den[o];
        }
        bt.nband = nband;
    } else {
        if (!num || !den) return SF_ERR_NULL;
        const size_t nb = (size_t)H * W * sizeof(float);
        if (overlaps(img, (size_t)H * W, num, nb) || overlaps(img, (size_t)H * W, den, nb) ||
            overlaps(num, nb, den, nb))
            return SF_ERR_ALIAS;
        bt.num[0] = num;
        bt.den[0] = den;
        bt.nband = 1;
    }
    cudaStream_t s = (cudaStream_t)stream;
    float* part = nullptr;                            // [2][H][W] partials (add / scatter)
    if (accum && sf::scratch_alloc((void**)&part, (size_t)2 * H * W * sizeof(float), s) != cudaSuccess) {
        cudaGetLastError();
        return SF_ERR_CUDA;
    }
    sf::Params p{};
    p.img = img;
    p.img_row0 = 0;
    p.img_rows = H;
    p.H = H;
    p.W = W;
    p.r = radius;
    p.kind = kind;
    p.out_row0 = 0;
    p.out_rows = H;
    p.out = nullptr;
    p.num = accum ? part : num;
    p.den = accum ? part + (size_t)H * W : den;
    sf_status rs = launch(p, make_table(N, sigma_r, pair_begin, pair_end), gamma_of(N, sigma_r), s);
    if (accum) {
        if (rs == SF_OK) {
            const int launched = g_last_launches;
            if (sf::launch_band_add(part, part + (size_t)H * W, H, W, bt, s) != cudaSuccess) {
                cudaGetLastError();
                rs = SF_ERR_CUDA;
            }
            g_last_launches = rs == SF_OK ? launched + 1 : 0;
        }
        sf::scratch_free(part, s);
    }
    return rs;
}
}  // namespace

extern "C" {

int sf_pair_count(int N) { return N < 0 ? 0 : sf::pair_count(N); }

int sf_nmin(double sigma_r) {
    if (!std::isfinite(sigma_r) || !(sigma_r > 0.0)) return -1;
    return sf::nmin(sigma_r);
}

int sf_last_launch_count(void) { return g_last_launches; }

const char* sf_status_string(sf_status s) {
    switch (s) {
        case SF_OK: return "ok";
        case SF_ERR_NULL: return "null pointer";
        case SF_ERR_SHAPE: return "bad shape (H < 1 or W < 1)";
        case SF_ERR_RADIUS: return "bad radius (need 0 <= r <= min(H,W)-1 and r <= SF_MAX_RADIUS)";
        case SF_ERR_SIGMA: return "bad sigma_r (need finite > 0)";
        case SF_ERR_ORDER: return "bad order N (need sf_nmin(sigma_r) <= N <= SF_MAX_ORDER)";
        case SF_ERR_KIND: return "unknown spatial kind";
        case SF_ERR_RANGE: return "bad row or pair range";
        case SF_ERR_ALIAS: return "output overlaps input";
        case SF_ERR_CUDA: return "CUDA error";
    }
    return "unknown status";
}

sf_status sf_filter_rows(const uint8_t* img_band, int H, int W, int row_begin, int row_end,
                         int radius, int kind, double sigma_r, int N, float* out_band,
                         void* stream) {
    g_last_launches = 0;
    sf_status st = validate(img_band, H, W, radius, kind, sigma_r, N);
    if (st != SF_OK) return st;
    if (!out_band) return SF_ERR_NULL;
    if (row_begin < 0 || row_end > H || row_begin >= row_end) return SF_ERR_RANGE;
    const int in0 = row_begin - radius < 0 ? 0 : row_begin - radius;
    const int in1 = row_end + radius > H ? H : row_end + radius;
    if (overlaps(img_band, (size_t)(in1 - in0) * W, out_band,
                 (size_t)(row_end - row_begin) * W * sizeof(float)))
        return SF_ERR_ALIAS;
    sf::Params p{};
    p.img = img_band;
    p.img_row0 = in0;
    p.img_rows = in1 - in0;
    p.H = H;
    p.W = W;
    p.r = radius;
    p.kind = kind;
    p.out_row0 = row_begin;
    p.out_rows = row_end - row_begin;
    p.out = out_band;
    p.num = nullptr;
    p.den = nullptr;
    return launch(p, make_table(N, sigma_r, 0, sf::pair_count(N)), gamma_of(N, sigma_r), (cudaStream_t)stream);
}

sf_status sf_filter(const uint8_t* img, int H, int W, int radius, int kind, double sigma_r,
                    int N, float* out, void* stream) {
    g_last_launches = 0;
    sf_status st = validate(img, H, W, radius, kind, sigma_r, N);
    if (st != SF_OK) return st;
    if (!out) return SF_ERR_NULL;
    return sf_filter_rows(img, H, W, 0, H, radius, kind, sigma_r, N, out, stream);
}

// Shiftable NLM planner (nlm_kernel.cuh): gamma_k = sqrt(2 g(u_k)/(n h^2)),
// g(u) = exp(-|u|^2/(2 rho^2)); one representative per conjugate pair of
// multi-indices m in [0,n]^p, weight prod_k C(n,m_k)/2^n (x2 for a pair).
int nlm_pairs(int p, int n) {
    long total = 1;
    for (int k = 0; k < p; ++k) total *= (n + 1);
    return (int)((total + 1) / 2);
}

sf::NlmTable nlm_plan(int p, double h, double rho, int n) {
    sf::NlmTable t;
    std::memset(&t, 0, sizeof(t));
    t.p = p;
    double gam[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < p; ++k) {
        const double d2 = (k == 0) ? 0.0 : 1.0;             // |u_2|^2 = |u_3|^2 = 1
        const double g = (d2 == 0.0) ? 1.0 : (rho > 0.0 ? std::exp(-d2 / (2.0 * rho * rho)) : 0.0);
        gam[k] = std::sqrt(2.0 * g / ((double)n * h * h));
    }
    std::vector<long double> c(n + 1);
    const long double lgn = lgammal((long double)n + 1.0L) - (long double)n * logl(2.0L);
    for (int m = 0; m <= n; ++m)
        c[m] = expl(lgn - lgammal((long double)m + 1.0L) - lgammal((long double)(n - m) + 1.0L));
    long total = 1;
    for (int k = 0; k < p; ++k) total *= (n + 1);
    int np = 0;
    for (long idx = 0; idx < total; ++idx) {
        int mi[3] = {0, 0, 0};
        long rem = idx, cidx = 0, base = 1;
        for (int k = 0; k < p; ++k) {
            mi[k] = (int)(rem % (n + 1));
            rem /= (n + 1);
            cidx += (long)(n - mi[k]) * base;
            base *= (n + 1);
        }
        if (cidx < idx) continue;                          // the conjugate represents this pair
        long double w = 1.0L;
        for (int k = 0; k < p; ++k) {
            w *= c[mi[k]];
            t.om[k][np] = (float)((2.0 * mi[k] - n) * gam[k]);
        }
        t.weight[np] = (float)(cidx == idx ? w : 2.0L * w);
        ++np;
    }
    t.npairs = np;
    return t;
}

sf_status sf_nlm(const uint8_t* img, int H, int W, int radius, int p, double h, double rho, int n,
                 float* out, void* stream) {
    g_last_launches = 0;
    if (!img || !out) return SF_ERR_NULL;
    if (H < 1 || W < 1) return SF_ERR_SHAPE;
    if (radius < 0 || radius > SF_MAX_RADIUS || radius > (H < W ? H : W) - 1) return SF_ERR_RADIUS;
    if (p < 1 || p > 3) return SF_ERR_KIND;
    if (!std::isfinite(h) || !(h > 0.0) || !std::isfinite(rho) || !(rho >= 0.0)) return SF_ERR_SIGMA;
    if (n < sf::nmin(h / std::sqrt(2.0)) || nlm_pairs(p, n) > sf::kNlmMaxPairs) return SF_ERR_ORDER;
    if (overlaps(img, (size_t)H * W, out, (size_t)H * W * sizeof(float))) return SF_ERR_ALIAS;
    sf::Params pr{};
    pr.img = img;
    pr.img_row0 = 0;
    pr.img_rows = H;
    pr.H = H;
    pr.W = W;
    pr.r = radius;
    pr.kind = SF_SPATIAL_BOX;
    pr.out_row0 = 0;
    pr.out_rows = H;
    pr.out = out;
    // band sweep (box_nlm5.cuh) for the instantiated radii, else the tile kernel
    // (also SF_VARIANT=v1)
    const sf::NlmTable tab = nlm_plan(p, h, rho, n);
    cudaError_t e = cudaErrorInvalidValue;
    if (variant() != 1 && sf::nlm_v5n_has(radius) && 2 * radius + 1 < 8 * 16 && radius <= (W - 1))
        e = sf::launch_nlm_v5n(radius, p, pr, tab, (cudaStream_t)stream);
    else
        e = sf::launch_nlm(pr, tab, (cudaStream_t)stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return SF_ERR_CUDA;
    }
    g_last_launches = 1;
    return SF_OK;
}

int sf_nlm_pair_count(int p, int n) { return (p < 1 || p > 3 || n < 0) ? -1 : nlm_pairs(p, n); }

sf_status sf_spatial_filter(const uint8_t* img, int H, int W, int radius, int kind, float* out,
                            void* stream) {
    g_last_launches = 0;
    // order-0 range kernel: one term, omega = 0, weight 1 (Algorithm 1)
    sf_status st = validate(img, H, W, radius, kind, 1e30, 1);
    if (st != SF_OK) return st;
    if (!out) return SF_ERR_NULL;
    if (overlaps(img, (size_t)H * W, out, (size_t)H * W * sizeof(float))) return SF_ERR_ALIAS;
    sf::Params p{};
    p.img = img;
    p.img_row0 = 0;
    p.img_rows = H;
    p.H = H;
    p.W = W;
    p.r = radius;
    p.kind = kind;
    p.out_row0 = 0;
    p.out_rows = H;
    p.out = out;
    p.num = nullptr;
    p.den = nullptr;
    sf::PairTable t;
    std::memset(&t, 0, sizeof(t));
    t.npairs = 1;
    t.omega[0] = 0.f;
    t.weight[0] = 1.f;
    return launch(p, t, 0.0, (cudaStream_t)stream);
}

int sf_truncation_n0(int N, double eps) { return sf::truncation_n0(N, eps); }

sf_status sf_filter_truncated(const uint8_t* img, int H, int W, int radius, int kind, double sigma_r,
                              int N, double eps, float* out, void* stream) {
    g_last_launches = 0;
    sf_status st = validate(img, H, W, radius, kind, sigma_r, N);
    if (st != SF_OK) return st;
    if (!out) return SF_ERR_NULL;
    const int n0 = sf::truncation_n0(N, eps);
    if (n0 < 0) return SF_ERR_RANGE;
    if (overlaps(img, (size_t)H * W, out, (size_t)H * W * sizeof(float))) return SF_ERR_ALIAS;
    sf::Params p{};
    p.img = img;
    p.img_row0 = 0;
    p.img_rows = H;
    p.H = H;
    p.W = W;
    p.r = radius;
    p.kind = kind;
    p.out_row0 = 0;
    p.out_rows = H;
    p.out = out;
    p.num = nullptr;
    p.den = nullptr;
    return launch(p, make_table(N, sigma_r, n0, sf::pair_count(N)), gamma_of(N, sigma_r),
                  (cudaStream_t)stream);
}


sf_status sf_accumulate(const uint8_t* img, int H, int W, int radius, int kind, double sigma_r,
                        int N, int pair_begin, int pair_end, float* num, float* den,
                        void* stream) {
    return accumulate_impl(img, H, W, radius, kind, sigma_r, N, pair_begin, pair_end, num, den, stream, 0);
}

sf_status sf_accumulate_add(const uint8_t* img, int H, int W, int radius, int kind, double sigma_r,
                            int N, int pair_begin, int pair_end, float* num, float* den,
                            void* stream) {
    return accumulate_impl(img, H, W, radius, kind, sigma_r, N, pair_begin, pair_end, num, den, stream, 1);
}

sf_status sf_accumulate_scatter(const uint8_t* img, int H, int W, int radius, int kind, double sigma_r,
                                int N, int pair_begin, int pair_end, int nband, float* const* band_num,
                                float* const* band_den, void* stream) {
    return accumulate_impl(img, H, W, radius, kind, sigma_r, N, pair_begin, pair_end, nullptr, nullptr, stream, 2,
                           nband, band_num, band_den);
}

sf_status sf_finalize(const float* num, const float* den, const uint8_t* img, int H, int W,
                      float* out, void* stream) {
    g_last_launches = 0;
    if (!num || !den || !img || !out) return SF_ERR_NULL;
    if (H < 1 || W < 1) return SF_ERR_SHAPE;
    const size_t n = (size_t)H * W;
    if (overlaps(out, n * 4, num, n * 4) || overlaps(out, n * 4, den, n * 4) ||
        overlaps(out, n * 4, img, n))
        return SF_ERR_ALIAS;
    cudaError_t e = sf::launch_finalize(num, den, img, n, out, (cudaStream_t)stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return SF_ERR_CUDA;
    }
    g_last_launches = 1;
    return SF_OK;
}

// Host-buffer entry point.  Large bands are split into row chunks that are
// pipelined over two library streams: the H2D copy of chunk c+1 and the D2H
// copy of chunk c-1 overlap the kernel of chunk c (the copy engines and the
// SMs work at once).  Chunk c's kernel waits for the copies of chunks c-1..c+1,
// which cover its r-row halo; the input copies partition the band's rows.
sf_status sf_filter_rows_host(const uint8_t* img_host, int H, int W, int row_begin, int row_end,
                              int radius, int kind, double sigma_r, int N, float* out_host,
                              void* stream) {
    g_last_launches = 0;
    sf_status st = validate(img_host, H, W, radius, kind, sigma_r, N);
    if (st != SF_OK) return st;
    if (!out_host) return SF_ERR_NULL;
    if (row_begin < 0 || row_end > H || row_begin >= row_end) return SF_ERR_RANGE;
    cudaStream_t s = (cudaStream_t)stream;
    const int in0 = row_begin - radius < 0 ? 0 : row_begin - radius;
    const int in1 = row_end + radius > H ? H : row_end + radius;
    const size_t nin = (size_t)(in1 - in0) * W, nout = (size_t)(row_end - row_begin) * W;
    sf::DeviceInfo& di = sf::current_device_info();
    if (di.err != cudaSuccess) return SF_ERR_CUDA;
    uint8_t* d_img = nullptr;
    float* d_out = nullptr;
    if (sf::scratch_alloc((void**)&d_img, nin, s) != cudaSuccess ||
        sf::scratch_alloc((void**)&d_out, nout * sizeof(float), s) != cudaSuccess) {
        cudaGetLastError();
        sf::scratch_free(d_img, s);
        return SF_ERR_CUDA;
    }
    const int rows = row_end - row_begin;
    // up to 8 chunks of >= 512 rows, with a half-size first and last chunk:
    // the first H2D and the last D2H are the parts no kernel overlaps
    static const int chunks_env = [] { const char* e = std::getenv("SF_HOST_CHUNKS"); return e ? std::atoi(e) : 0; }();
    const int cmax = chunks_env > 0 && chunks_env <= 16 ? chunks_env : 8;   // tuning knob (tools/time_e2e.py)
    int nmid = rows / 512;
    nmid = nmid < 1 ? 1 : (nmid > cmax ? cmax : nmid);
    int nch = nmid > 1 ? nmid + 1 : 1;
    if (nch > 1 && radius * 2 > rows / (2 * nmid)) nch = 1;   // halo must stay within a neighbour chunk
    sf_status rs = SF_OK;
    int launches = 0;
    if (nch == 1) {
        if (cudaMemcpyAsync(d_img, img_host, nin, cudaMemcpyHostToDevice, s) != cudaSuccess) rs = SF_ERR_CUDA;
        if (rs == SF_OK)
            rs = sf_filter_rows(d_img, H, W, row_begin, row_end, radius, kind, sigma_r, N, d_out, stream);
        launches = g_last_launches;
        if (rs == SF_OK &&
            cudaMemcpyAsync(out_host, d_out, nout * sizeof(float), cudaMemcpyDeviceToHost, s) != cudaSuccess)
            rs = SF_ERR_CUDA;
    } else {
        int cb[18], cp[18];                                // chunk output rows / copied input rows
        // boundaries at (c - 1/2) / nmid of the rows: half, nmid - 1 full, half
        for (int c = 0; c <= nch; ++c)
            cb[c] = c == 0 ? row_begin : (c == nch ? row_end : row_begin + (int)((long)rows * (2 * c - 1) / (2 * nmid)));
        for (int c = 0; c <= nch; ++c) cp[c] = (c == 0) ? in0 : (c == nch ? in1 : cb[c]);
        cudaEvent_t ev0, evc[17], evd[2];
        cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
        for (int c = 0; c < nch; ++c) cudaEventCreateWithFlags(&evc[c], cudaEventDisableTiming);
        for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&evd[i], cudaEventDisableTiming);
        cudaEventRecord(ev0, s);                           // after the allocations and prior work on s
        for (int i = 0; i < 2; ++i) cudaStreamWaitEvent(di.aux[i], ev0, 0);
        auto copy_in = [&](int c) {
            cudaStream_t sc = di.aux[c & 1];
            if (cudaMemcpyAsync(d_img + (size_t)(cp[c] - in0) * W, img_host + (size_t)(cp[c] - in0) * W,
                                (size_t)(cp[c + 1] - cp[c]) * W, cudaMemcpyHostToDevice, sc) != cudaSuccess)
                rs = SF_ERR_CUDA;
            cudaEventRecord(evc[c], sc);
        };
        copy_in(0);
        if (nch > 1) copy_in(1);
        for (int c = 0; c < nch && rs == SF_OK; ++c) {
            if (c + 2 < nch) copy_in(c + 2);
            cudaStream_t sc = di.aux[c & 1];
            for (int d = c - 1; d <= c + 1; ++d)
                if (d >= 0 && d < nch) cudaStreamWaitEvent(sc, evc[d], 0);
            const int ia = cb[c] - radius < 0 ? 0 : cb[c] - radius;
            rs = sf_filter_rows(d_img + (size_t)(ia - in0) * W, H, W, cb[c], cb[c + 1], radius, kind, sigma_r,
                                N, d_out + (size_t)(cb[c] - row_begin) * W, (void*)sc);
            launches += g_last_launches;
            if (rs == SF_OK &&
                cudaMemcpyAsync(out_host + (size_t)(cb[c] - row_begin) * W, d_out + (size_t)(cb[c] - row_begin) * W,
                                (size_t)(cb[c + 1] - cb[c]) * W * sizeof(float), cudaMemcpyDeviceToHost,
                                sc) != cudaSuccess)
                rs = SF_ERR_CUDA;
        }
        for (int i = 0; i < 2; ++i) {
            cudaEventRecord(evd[i], di.aux[i]);
            cudaStreamWaitEvent(s, evd[i], 0);             // the caller's stream joins the pipeline
        }
        cudaStreamSynchronize(s);
        cudaEventDestroy(ev0);
        for (int c = 0; c < nch; ++c) cudaEventDestroy(evc[c]);
        for (int i = 0; i < 2; ++i) cudaEventDestroy(evd[i]);
    }
    sf::scratch_free(d_img, s);
    sf::scratch_free(d_out, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) rs = SF_ERR_CUDA;
    if (rs != SF_OK) cudaGetLastError();
    g_last_launches = rs == SF_OK ? launches : 0;
    return rs;
}

// f3 (poly_kernel.cuh): phi_p(t) = (1 - t^2/(2 N sigma_r^2))^N, valid on
// [-255, 255] for N >= ceil(255^2 / (2 sigma_r^2)) (reading R17)
int sf_nmin_poly(double sigma_r) {
    if (!std::isfinite(sigma_r) || !(sigma_r > 0.0)) return -1;
    const double q = 255.0 * 255.0 / (2.0 * sigma_r * sigma_r);
    const double n = std::ceil(q - 1e-12);
    return n < 1.0 ? 1 : (n > 1e9 ? 1000000000 : (int)n);
}

sf_status sf_filter_poly(const uint8_t* img, int H, int W, int radius, double sigma_r, int N, float* out,
                         void* stream) {
    g_last_launches = 0;
    if (!img || !out) return SF_ERR_NULL;
    if (H < 1 || W < 1) return SF_ERR_SHAPE;
    if (radius < 0 || radius > SF_MAX_POLY_RADIUS || radius > (H < W ? H : W) - 1) return SF_ERR_RADIUS;
    if (!std::isfinite(sigma_r) || !(sigma_r > 0.0)) return SF_ERR_SIGMA;
    if (N < sf_nmin_poly(sigma_r) || N > SF_MAX_POLY_ORDER) return SF_ERR_ORDER;
    if (overlaps(img, (size_t)H * W, out, (size_t)H * W * sizeof(float))) return SF_ERR_ALIAS;
    // Chebyshev coefficients of u -> phi_p(128 (u - v)) (degree D = 2N, exact
    // interpolation at the D+1 Chebyshev nodes, long double) for the 256
    // centre values, and the numerator's e_k (poly_kernel.cuh)
    const int D = 2 * N, M = D + 1, K = D + 2;
    const long double a = 128.0L * 128.0L / (2.0L * (long double)N * sigma_r * sigma_r);
    std::vector<long double> cs((size_t)(D + 1) * M), um(M);
    const long double PI = 3.141592653589793238462643383279502884L;
    for (int m = 0; m < M; ++m) {
        const long double th = PI * ((long double)m + 0.5L) / (long double)M;
        um[m] = cosl(th);
        for (int i = 0; i <= D; ++i) cs[(size_t)i * M + m] = cosl((long double)i * th);
    }
    std::vector<double> tab((size_t)256 * 2 * K);
    std::vector<long double> pm(M), c(D + 3);
    for (int v = 0; v < 256; ++v) {
        const long double vv = ((long double)v - 128.0L) / 128.0L;
        for (int m = 0; m < M; ++m) {
            const long double d = um[m] - vv;
            pm[m] = powl(1.0L - a * d * d, (long double)N);
        }
        for (int i = 0; i <= D; ++i) {
            long double sacc = 0.0L;
            for (int m = 0; m < M; ++m) sacc += pm[m] * cs[(size_t)i * M + m];
            c[i] = 2.0L * sacc / (long double)M;
        }
        c[0] *= 0.5L;
        c[D + 1] = c[D + 2] = 0.0L;
        double* cr = tab.data() + (size_t)v * 2 * K;
        for (int k = 0; k < K; ++k) {
            cr[k] = (double)(k <= D ? c[k] : 0.0L);
            const long double e = k == 0 ? 0.5L * c[1] : (k == 1 ? c[0] + 0.5L * c[2] : 0.5L * (c[k - 1] + c[k + 1]));
            cr[K + k] = (double)e;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    double* dtab = nullptr;
    if (sf::scratch_alloc((void**)&dtab, tab.size() * sizeof(double), s) != cudaSuccess ||
        cudaMemcpyAsync(dtab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, s) != cudaSuccess) {
        cudaGetLastError();
        if (dtab) sf::scratch_free(dtab, s);
        return SF_ERR_CUDA;
    }
    cudaStreamSynchronize(s);              // the pageable host table must outlive the copy
    sf::Params p{};
    p.img = img;
    p.img_row0 = 0;
    p.img_rows = H;
    p.H = H;
    p.W = W;
    p.r = radius;
    p.kind = SF_SPATIAL_BOX;
    p.out_row0 = 0;
    p.out_rows = H;
    p.out = out;
    cudaError_t e = sf::launch_poly(p, dtab, K, s);
    sf::scratch_free(dtab, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return SF_ERR_CUDA;
    }
    g_last_launches = 1;
    return SF_OK;
}

// f2: q_M spatial kernel fitted to a Gaussian of width sigma_s (Eq.(7),
// reading R18): w1(u) = cos(u / (sigma_s sqrt M))^M on |u| <= r, on the v1
// tile kernel's generic q_M walker with beta = 1/(sigma_s sqrt M)
int sf_spatial_mmin(int radius, double sigma_s) {
    if (radius < 0 || !std::isfinite(sigma_s) || !(sigma_s > 0.0)) return -1;
    const double q = 2.0 * radius / (M_PI * sigma_s);
    const double m = std::ceil(q * q - 1e-12);
    return m < 1.0 ? 1 : (m > 1e6 ? 1000000 : (int)m);
}

namespace {
sf_status spatial_sigma_impl(const uint8_t* img, int H, int W, int radius, double sigma_s, int M, double sigma_r,
                             int N, bool range, float* out, void* stream) {
    g_last_launches = 0;
    if (!img || !out) return SF_ERR_NULL;
    if (H < 1 || W < 1) return SF_ERR_SHAPE;
    if (M < 1 || M > 8) return SF_ERR_KIND;
    if (!std::isfinite(sigma_s) || !(sigma_s > 0.0)) return SF_ERR_SIGMA;
    sf_status st = validate(img, H, W, radius, SF_SPATIAL_QM(M), range ? sigma_r : 1e30, range ? N : 1);
    if (st != SF_OK) return st;
    if (M < sf_spatial_mmin(radius, sigma_s)) return SF_ERR_ORDER;
    if (overlaps(img, (size_t)H * W, out, (size_t)H * W * sizeof(float))) return SF_ERR_ALIAS;
    sf::Params p{};
    p.img = img;
    p.img_row0 = 0;
    p.img_rows = H;
    p.H = H;
    p.W = W;
    p.r = radius;
    p.kind = SF_SPATIAL_QM(M);
    p.out_row0 = 0;
    p.out_rows = H;
    p.out = out;
    p.beta = (float)(1.0 / (sigma_s * std::sqrt((double)M)));
    // the default dispatch: the v7q band sweep for M <= 4, r <= 24 (beta from
    // Params), the tile kernel's generic q_M walker otherwise
    if (range) return launch(p, make_table(N, sigma_r, 0, sf::pair_count(N)), gamma_of(N, sigma_r), (cudaStream_t)stream);
    sf::PairTable t;
    std::memset(&t, 0, sizeof(t));
    t.npairs = 1;
    t.weight[0] = 1.f;
    return launch(p, t, 0.0, (cudaStream_t)stream);
}
}  // namespace

sf_status sf_filter_spatial_sigma(const uint8_t* img, int H, int W, int radius, double sigma_s, int M,
                                  double sigma_r, int N, float* out, void* stream) {
    return spatial_sigma_impl(img, H, W, radius, sigma_s, M, sigma_r, N, true, out, stream);
}

sf_status sf_spatial_filter_sigma(const uint8_t* img, int H, int W, int radius, double sigma_s, int M, float* out,
                                  void* stream) {
    return spatial_sigma_impl(img, H, W, radius, sigma_s, M, 0.0, 0, false, out, stream);
}

sf_status sf_release_scratch(void) {
    sf::DeviceInfo& di = sf::current_device_info();
    if (di.err != cudaSuccess) return SF_ERR_CUDA;
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemPoolTrimTo(di.pool, 0) != cudaSuccess) {
        cudaGetLastError();
        return SF_ERR_CUDA;
    }
    return SF_OK;
}

// Host-buffer entry point without the synchronisation: the input copy runs
// on library stream aux[0], the filter on the caller's stream, the output
// copy on library stream aux[1] (one copy engine per direction), linked by
// events, so that successive calls pipeline: call s's output copy and call
// s+1's input copy overlap call s+1's / s's kernels.  The device buffers are
// stream-ordered pool allocations released after their last use on the
// stream of that use.  Completion: sf_host_sync().
sf_status sf_filter_rows_host_async(const uint8_t* img_host, int H, int W, int row_begin, int row_end,
                                    int radius, int kind, double sigma_r, int N, float* out_host,
                                    void* stream) {
    g_last_launches = 0;
    sf_status st = validate(img_host, H, W, radius, kind, sigma_r, N);
    if (st != SF_OK) return st;
    if (!out_host) return SF_ERR_NULL;
    if (row_begin < 0 || row_end > H || row_begin >= row_end) return SF_ERR_RANGE;
    cudaStream_t s = (cudaStream_t)stream;
    sf::DeviceInfo& di = sf::current_device_info();
    if (di.err != cudaSuccess) return SF_ERR_CUDA;
    const int in0 = row_begin - radius < 0 ? 0 : row_begin - radius;
    const int in1 = row_end + radius > H ? H : row_end + radius;
    const size_t nin = (size_t)(in1 - in0) * W, nout = (size_t)(row_end - row_begin) * W;
    uint8_t* d_img = nullptr;
    float* d_out = nullptr;
    cudaEvent_t ev[2];
    for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    sf_status rs = SF_OK;
    if (sf::scratch_alloc((void**)&d_img, nin, di.aux[0]) != cudaSuccess ||
        cudaMemcpyAsync(d_img, img_host, nin, cudaMemcpyHostToDevice, di.aux[0]) != cudaSuccess ||
        cudaEventRecord(ev[0], di.aux[0]) != cudaSuccess || cudaStreamWaitEvent(s, ev[0], 0) != cudaSuccess ||
        sf::scratch_alloc((void**)&d_out, nout * sizeof(float), s) != cudaSuccess)
        rs = SF_ERR_CUDA;
    int launches = 0;
    if (rs == SF_OK) {
        rs = sf_filter_rows(d_img, H, W, row_begin, row_end, radius, kind, sigma_r, N, d_out, stream);
        launches = g_last_launches;
    }
    if (d_img) sf::scratch_free(d_img, s);
    if (rs == SF_OK &&
        (cudaEventRecord(ev[1], s) != cudaSuccess || cudaStreamWaitEvent(di.aux[1], ev[1], 0) != cudaSuccess ||
         cudaMemcpyAsync(out_host, d_out, nout * sizeof(float), cudaMemcpyDeviceToHost, di.aux[1]) != cudaSuccess))
        rs = SF_ERR_CUDA;
    if (d_out) sf::scratch_free(d_out, rs == SF_OK ? di.aux[1] : s);
    for (int i = 0; i < 2; ++i) cudaEventDestroy(ev[i]);   // released once their work completes
    if (rs != SF_OK) cudaGetLastError();
    g_last_launches = rs == SF_OK ? launches : 0;
    return rs;
}

sf_status sf_host_sync(void) {
    sf::DeviceInfo& di = sf::current_device_info();
    if (di.err != cudaSuccess) return SF_ERR_CUDA;
    for (int i = 0; i < 2; ++i)
        if (cudaStreamSynchronize(di.aux[i]) != cudaSuccess) {
            cudaGetLastError();
            return SF_ERR_CUDA;
        }
    return SF_OK;
}

sf_status sf_filter_host(const uint8_t* img_host, int H, int W, int radius, int kind,
                         double sigma_r, int N, float* out_host, void* stream) {
    g_last_launches = 0;
    sf_status st = validate(img_host, H, W, radius, kind, sigma_r, N);
    if (st != SF_OK) return st;
    if (!out_host) return SF_ERR_NULL;
    return sf_filter_rows_host(img_host, H, W, 0, H, radius, kind, sigma_r, N, out_host, stream);
}

}  // extern "C"
