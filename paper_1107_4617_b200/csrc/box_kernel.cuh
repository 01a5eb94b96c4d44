// box_kernel.cuh — fused sm_100a tile kernel for Algorithm 2
// with the raised-cosine range kernel, box or q_2 spatial kernel.
//
// v1 design:
//   * one CTA = one TW x TH output tile; the uint8 tile + r-halo is staged
//     into shared memory once (reflect-101 by index math), centred (f - 128);
//   * loop over conjugate pairs k (PAPER.md:151 step 1 + plan.h pairing):
//       vertical pass   — one walker per input column: running moving sums
//                         ("recursion") of the 4 stack images
//                         cos, sin, (f-c)cos, (f-c)sin of w_k (f-c), generated
//                         on the fly with sincos, never materialised;
//       horizontal pass — one walker per (output row, column segment) runs the
//                         same recursion over the vertical sums (smem);
//       recombine       — P += w_k (C_x S[(f-c)C] + S_x S[(f-c)S]),
//                         Q += w_k (C_x S[C] + S_x S[S]),
//     P and Q stay in registers for all pairs;
//   * store f~ = c + P/Q once per pixel (or the partial P, Q for the term split).
// For the q_2 spatial kernel each pass runs three running sums per image
// (unmodulated, cos- and sin-modulated by the tile-local coordinate) and
// recombines them: w1(u-t) = 1/2 + 1/2(cos(a t)cos(a u) + sin(a t)sin(a u)),
// a = pi/(r+1) — the shiftable spatial expansion of Alg. 2.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sf {

constexpr int kMaxPairs = 1025;          // SF_MAX_ORDER/2 + 1
constexpr float kCenter = 128.0f;        // SF_CENTER
constexpr int kThreads = 256;

struct PairTable {                       // passed by value in the param block
    int npairs;
    float omega[kMaxPairs];
    float weight[kMaxPairs];
};

struct Params {
    const uint8_t* img;                  // first available input row (img_row0)
    int img_row0, img_rows;              // input rows [img_row0, img_row0+img_rows)
    int H, W, r, kind;
    int out_row0, out_rows;              // output rows [out_row0, out_row0+out_rows)
    float* out;                          // final ratio (rows relative to out_row0) or null
    float* num;                          // partial P' (centred at kCenter) or null
    float* den;                          // partial Q or null
    float beta;                          // q_M spatial frequency; 0 = pi/(2(r+1)) (T = r+1)
};

__device__ __forceinline__ int reflect101(int p, int L) {
    if (L == 1) return 0;
    while (p < 0 || p >= L) {
        p = p < 0 ? -p : p;
        p = p >= L ? 2 * (L - 1) - p : p;
    }
    return p;
}

// centred input value (f - c) at image row gy, column gx (reflect-101; rows
// outside the caller's band are never needed by a valid window and clamp)
__device__ __forceinline__ float ldf(const Params& p, int gy, int gx) {
    int ry = reflect101(gy, p.H) - p.img_row0;
    ry = ry < 0 ? 0 : (ry >= p.img_rows ? p.img_rows - 1 : ry);
    return (float)__ldg(p.img + (size_t)ry * p.W + gx) - kCenter;
}

__device__ __forceinline__ float4 gen4(float v, float om) {
    float s, c;
    __sincosf(om * v, &s, &c);
    return make_float4(c, s, v * c, v * s);
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float4 f4sub(float4 a, float4 b) { return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w); }
__device__ __forceinline__ float4 f4fma(float s, float4 a, float4 b) {
    return make_float4(fmaf(s, a.x, b.x), fmaf(s, a.y, b.y), fmaf(s, a.z, b.z), fmaf(s, a.w, b.w));
}
__device__ __forceinline__ float4 f4scale(float s, float4 a) { return make_float4(s * a.x, s * a.y, s * a.z, s * a.w); }

// Running moving-sum state of one walker over the 4 stack images.
// KIND 0: plain box sums.  KIND 1: box sums of the image and of its cos/sin
// modulations by the coordinate p (tables mc/ms in smem).
template <int KIND>
struct Walk;

template <>
struct Walk<0> {
    float4 s;
    __device__ void reset() { s = make_float4(0.f, 0.f, 0.f, 0.f); }
    __device__ void add(float4 g, int, const float*, const float*) { s = f4add(s, g); }
    __device__ void slide(float4 gin, int, float4 gout, int, const float*, const float*) {
        s = f4add(s, f4sub(gin, gout));
    }
    __device__ float4 value(int, const float*, const float*) const { return s; }
};

// q_M spatial kernel (M >= 1): q_M(u - t) = sum_m C(M,m)/2^M e^{j s_m beta (u - t)},
// s_m = 2m - M, beta = pi/(2(r+1)) (Eq.(1) applied to the spatial kernel,
// PAPER.md:47-54, 202).  Conjugate frequencies +-s pair up: NF nonzero |s|
// (s_f = 2f+1 for odd M, 2f+2 for even M) with weight 2 C(M,(M+s)/2)/2^M,
// plus for even M the zero frequency with weight C(M,M/2)/2^M.  A walker keeps
// per image one plain running sum and one cos- and one sin-modulated running
// sum per nonzero frequency (M+1 sums), modulated by the tile-local coordinate
// p (tables mc/ms: cos/sin(s_f beta p)), and recombines them at the centre.
__host__ __device__ constexpr double binom_over_2m(int M, int m) {
    double b = 1.0;
    for (int i = 0; i < m; ++i) b = b * (double)(M - i) / (double)(i + 1);
    for (int i = 0; i < M; ++i) b *= 0.5;
    return b;
}

template <int M>
struct WalkQ {
    static constexpr int NF = (M + 1) / 2;
    static constexpr bool ZERO = (M % 2) == 0;
    __host__ __device__ static constexpr int sf(int f) { return (M % 2) ? 2 * f + 1 : 2 * f + 2; }
    float4 s0, sc[NF], ss[NF];
    int lt;                                  // table stride (entries per frequency)
    __device__ void reset() {
        s0 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int f = 0; f < NF; ++f) sc[f] = ss[f] = s0;
    }
    __device__ void add(float4 g, int p, const float* mc, const float* ms) {
        if (ZERO) s0 = f4add(s0, g);
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            sc[f] = f4fma(mc[f * lt + p], g, sc[f]);
            ss[f] = f4fma(ms[f * lt + p], g, ss[f]);
        }
    }
    __device__ void slide(float4 gin, int pin, float4 gout, int pout, const float* mc, const float* ms) {
        if (ZERO) s0 = f4add(s0, f4sub(gin, gout));
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            sc[f] = f4fma(mc[f * lt + pin], gin, f4fma(-mc[f * lt + pout], gout, sc[f]));
            ss[f] = f4fma(ms[f * lt + pin], gin, f4fma(-ms[f * lt + pout], gout, ss[f]));
        }
    }
    // sum_u q_M(u - p_c) g(u) = w0 S0 + sum_f w_f (cos(s_f beta p_c) Sc_f + sin(s_f beta p_c) Ss_f)
    __device__ float4 value(int pc, const float* mc, const float* ms) const {
        float4 v = ZERO ? f4scale((float)binom_over_2m(M, M / 2), s0) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const float w = (float)(2.0 * binom_over_2m(M, (M + sf(f)) / 2));
            v = f4fma(w * mc[f * lt + pc], sc[f], f4fma(w * ms[f * lt + pc], ss[f], v));
        }
        return v;
    }
};

template <int KIND>
struct WalkSel {
    using type = WalkQ<KIND>;
};
template <>
struct WalkSel<0> {
    using type = Walk<0>;
};

// Output tile TW x TH; 256 threads; G = TW*TH/256 outputs per thread (one row segment).
template <int TW, int TH, int KIND>
__global__ void __launch_bounds__(kThreads)
bilateral_tile_v1(const Params p, const PairTable tab) {
    constexpr int NSEGH = kThreads / TH;          // horizontal segments per row
    constexpr int G = TW / NSEGH;                 // outputs per thread
    static_assert(NSEGH * TH == kThreads && G * NSEGH == TW, "tile shape");
    extern __shared__ float4 smem4[];

    const int r = p.r, W = p.W, H = p.H;
    const int TWI = TW + 2 * r, THI = TH + 2 * r;
    const int fstride = TWI | 1;                          // odd: conflict-free column reads
    const int vstride = ((TWI + 7) & ~7) + 1;             // float4 units, = 1 mod 8
    float4* vbuf = smem4;                                 // TH x vstride float4
    float* fin = reinterpret_cast<float*>(smem4 + TH * vstride);   // THI x fstride
    constexpr int NF = KIND > 0 ? (KIND + 1) / 2 : 0;     // nonzero spatial frequencies
    const int LT = THI > TWI ? THI : TWI;                 // table entries per frequency
    float* mc = fin + THI * fstride;                      // modulation tables (q_M)
    float* ms = mc + NF * LT;

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TW;                       // output tile origin (global)
    const int y0 = p.out_row0 + blockIdx.y * TH;

    // ---- stage the centred input tile + halo (reflect-101 by index math)
    for (int i = tid; i < THI * TWI; i += kThreads) {
        const int ty = i / TWI, tx = i - ty * TWI;
        int gy = reflect101(y0 - r + ty, H) - p.img_row0;
        gy = gy < 0 ? 0 : (gy >= p.img_rows ? p.img_rows - 1 : gy);   // rows never stored
        const int gx = reflect101(x0 - r + tx, W);
        fin[ty * fstride + tx] = (float)p.img[(size_t)gy * W + gx] - kCenter;
    }
    if (KIND > 0) {
        const float bp = p.beta > 0.f ? p.beta / 3.14159265358979f : 0.5f / (float)(r + 1);   // beta/pi
        for (int i = tid; i < NF * LT; i += kThreads) {
            const int f = i / LT, q = i - f * LT;
            const int sfreq = (KIND % 2) ? 2 * f + 1 : 2 * f + 2;
            float s, c;
            sincospif(bp * (float)(sfreq * q), &s, &c);
            mc[i] = c;
            ms[i] = s;
        }
    }
    __syncthreads();

    float P[G], Q[G];
#pragma unroll
    for (int j = 0; j < G; ++j) P[j] = Q[j] = 0.f;

    // vertical walkers: (column c, row segment)
    int nsegv = kThreads / TWI;
    nsegv = nsegv < 1 ? 1 : nsegv;
    while (TH % nsegv) --nsegv;
    const int segv = TH / nsegv;

    const int hy = tid % TH, hs = tid / TH, hx0 = hs * G;   // horizontal walker

    for (int k = 0; k < tab.npairs; ++k) {
        const float om = tab.omega[k], wk = tab.weight[k];
        for (int wv = tid; wv < TWI * nsegv; wv += kThreads) {
            const int c = wv % TWI, ys = (wv / TWI) * segv;
            typename WalkSel<KIND>::type acc;
            if constexpr (KIND > 0) acc.lt = LT;
            acc.reset();
            for (int i = 0; i <= 2 * r; ++i) acc.add(gen4(fin[(ys + i) * fstride + c], om), ys + i, mc, ms);
            for (int y = ys; y < ys + segv; ++y) {
                vbuf[y * vstride + c] = acc.value(y + r, mc, ms);
                if (y + 1 < ys + segv)
                    acc.slide(gen4(fin[(y + 2 * r + 1) * fstride + c], om), y + 2 * r + 1,
                              gen4(fin[y * fstride + c], om), y, mc, ms);
            }
        }
        __syncthreads();
        {
            const float4* vrow = vbuf + hy * vstride;
            const float* frow = fin + (hy + r) * fstride + r;
            typename WalkSel<KIND>::type acc;
            if constexpr (KIND > 0) acc.lt = LT;
            acc.reset();
            for (int i = 0; i <= 2 * r; ++i) acc.add(vrow[hx0 + i], hx0 + i, mc, ms);
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const int x = hx0 + j;
                const float4 h = acc.value(x + r, mc, ms);
                float sn, cs;
                __sincosf(om * frow[x], &sn, &cs);
                const float a = wk * cs, b = wk * sn;
                P[j] = fmaf(a, h.z, fmaf(b, h.w, P[j]));
                Q[j] = fmaf(a, h.x, fmaf(b, h.y, Q[j]));
                if (j + 1 < G) acc.slide(vrow[x + 2 * r + 1], x + 2 * r + 1, vrow[x], x, mc, ms);
            }
        }
        __syncthreads();
    }

    const int gy = y0 + hy;
    if (gy < p.out_row0 + p.out_rows) {
        const size_t rowoff = (size_t)(gy - p.out_row0) * W;
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int gx = x0 + hx0 + j;
            if (gx < W) {
                if (p.out) {
                    const float f = fin[(hy + r) * fstride + hx0 + j + r];
                    const float q = Q[j];
                    p.out[rowoff + gx] = (q > 0.f && isfinite(q)) ? kCenter + P[j] / q : kCenter + f;
                } else {
                    p.num[rowoff + gx] = P[j];
                    p.den[rowoff + gx] = Q[j];
                }
            }
        }
    }
}

template <int TW, int TH, int KIND>
inline cudaError_t launch_tile_v1(const Params& p, const PairTable& t, cudaStream_t s) {
    const int TWI = TW + 2 * p.r, THI = TH + 2 * p.r;
    const int vstride = ((TWI + 7) & ~7) + 1;
    constexpr int NF = KIND > 0 ? (KIND + 1) / 2 : 0;
    const int modl = 2 * NF * (THI > TWI ? THI : TWI);
    const size_t smem = (size_t)TH * vstride * 16 + (size_t)THI * (TWI | 1) * 4 + (size_t)modl * 4;
    cudaError_t e = cudaFuncSetAttribute(bilateral_tile_v1<TW, TH, KIND>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.W + TW - 1) / TW, (p.out_rows + TH - 1) / TH);
    bilateral_tile_v1<TW, TH, KIND><<<grid, kThreads, smem, s>>>(p, t);
    return cudaGetLastError();
}

// spatial order M of a spatial kind (include/sf.h): box 0, SF_SPATIAL_RAISED_COS
// (q_2) 2, SF_SPATIAL_QM(M) = 100 + M, M = 1..8; -1 if unknown
inline int spatial_order(int kind) {
    if (kind == 0) return 0;
    if (kind == 1) return 2;
    if (kind >= 101 && kind <= 108) return kind - 100;
    return -1;
}

template <int TW, int TH>
inline cudaError_t launch_tile_v1_m(const Params& p, const PairTable& t, cudaStream_t s) {
    switch (spatial_order(p.kind)) {
        case 0: return launch_tile_v1<TW, TH, 0>(p, t, s);
        case 1: return launch_tile_v1<TW, TH, 1>(p, t, s);
        case 2: return launch_tile_v1<TW, TH, 2>(p, t, s);
        case 3: return launch_tile_v1<TW, TH, 3>(p, t, s);
        case 4: return launch_tile_v1<TW, TH, 4>(p, t, s);
        case 5: return launch_tile_v1<TW, TH, 5>(p, t, s);
        case 6: return launch_tile_v1<TW, TH, 6>(p, t, s);
        case 7: return launch_tile_v1<TW, TH, 7>(p, t, s);
        case 8: return launch_tile_v1<TW, TH, 8>(p, t, s);
    }
    return cudaErrorInvalidValue;
}

inline cudaError_t launch_box(const Params& p, const PairTable& t, cudaStream_t s) {
    if (p.r <= 24) return launch_tile_v1_m<64, 64>(p, t, s);
    return launch_tile_v1_m<32, 32>(p, t, s);
}

}  // namespace sf
