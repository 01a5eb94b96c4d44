// nlm_kernel.cuh — shiftable non-local means with a tiny patch (SURVEY.md §8(f)
// f4, Eq.(approx_multivariate)), box outer window.
//
// The patch is p <= 3 pixels at offsets u_1 = (0,0), u_2 = (0,1), u_3 = (1,0)
// (reading R14).  The Gaussian patch weight is approximated by the separable
// shiftable kernel prod_k cos(gamma_k t_k)^n, whose expansion has (n+1)^p
// terms; conjugate multi-indices pair up as in the bilateral filter (plan:
// nlm_plan in sf.cu).  For a term with frequencies (w_1..w_p) the "stack"
// images are e^{j theta(z)} and f(z) e^{j theta(z)} with the phase field
//     theta(z) = sum_k w_k f(z + u_k),
// i.e. Algorithm 2's machinery with f inside the exponential replaced by a
// weighted sum of the patch values; the centre factor is e^{-j theta(x)}.
//
// Kernel: the tile design of v1 (box_kernel.cuh) — one CTA per 64 x 64 output
// tile with its r-halo (+1 row and column for the patch offsets) staged in
// shared memory, per term pair a vertical then a horizontal moving-sum pass
// (running sums), (Q, P') in registers across all terms.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"

namespace sf {

constexpr int kNlmMaxPairs = 512;

struct NlmTable {                        // passed by value (8 KB of the param block)
    int npairs, p;
    float om[3][kNlmMaxPairs];           // w_k of the pair's representative multi-index
    float weight[kNlmMaxPairs];          // prod_k C(n,m_k)/2^n, doubled for a conjugate pair
};

// phase-field stack (cos, sin, f cos, f sin) of theta = sum_k w_k f(z+u_k) at tile index i
__device__ __forceinline__ float4 nlm_gen(const float* fin, int i, int fstride, int p, float o0, float o1,
                                          float o2) {
    const float f = fin[i];
    float th = o0 * f;
    if (p > 1) th = fmaf(o1, fin[i + 1], th);
    if (p > 2) th = fmaf(o2, fin[i + fstride], th);
    float s, c;
    __sincosf(th, &s, &c);
    return make_float4(c, s, f * c, f * s);
}

template <int TW, int TH>
__global__ void __launch_bounds__(kThreads)
nlm_tile_kernel(const Params p, const NlmTable tab) {
    constexpr int NSEGH = kThreads / TH;
    constexpr int G = TW / NSEGH;
    static_assert(NSEGH * TH == kThreads && G * NSEGH == TW, "tile shape");
    extern __shared__ float4 smem4[];

    const int r = p.r, W = p.W, H = p.H;
    const int TWI = TW + 2 * r, THI = TH + 2 * r;
    const int fstride = (TWI + 1) | 1;                    // +1 column for u_2, odd stride
    const int vstride = ((TWI + 7) & ~7) + 1;
    float4* vbuf = smem4;                                 // TH x vstride float4
    float* fin = reinterpret_cast<float*>(smem4 + TH * vstride);   // (THI+1) x fstride

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TW;
    const int y0 = p.out_row0 + blockIdx.y * TH;
    for (int i = tid; i < (THI + 1) * (TWI + 1); i += kThreads) {
        const int ty = i / (TWI + 1), tx = i - ty * (TWI + 1);
        int gy = reflect101(y0 - r + ty, H) - p.img_row0;
        gy = gy < 0 ? 0 : (gy >= p.img_rows ? p.img_rows - 1 : gy);
        const int gx = reflect101(x0 - r + tx, W);
        fin[ty * fstride + tx] = (float)p.img[(size_t)gy * W + gx] - kCenter;
    }
    __syncthreads();

    float P[G], Q[G];
#pragma unroll
    for (int j = 0; j < G; ++j) P[j] = Q[j] = 0.f;
    int nsegv = kThreads / TWI;
    nsegv = nsegv < 1 ? 1 : nsegv;
    while (TH % nsegv) --nsegv;
    const int segv = TH / nsegv;
    const int hy = tid % TH, hs = tid / TH, hx0 = hs * G;
    const int pp = tab.p;

    for (int k = 0; k < tab.npairs; ++k) {
        const float o0 = tab.om[0][k], o1 = tab.om[1][k], o2 = tab.om[2][k], wk = tab.weight[k];
        for (int wv = tid; wv < TWI * nsegv; wv += kThreads) {
            const int c = wv % TWI, ys = (wv / TWI) * segv;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int i = 0; i <= 2 * r; ++i) acc = f4add(acc, nlm_gen(fin, (ys + i) * fstride + c, fstride, pp, o0, o1, o2));
            for (int y = ys; y < ys + segv; ++y) {
                vbuf[y * vstride + c] = acc;
                if (y + 1 < ys + segv)
                    acc = f4add(acc, f4sub(nlm_gen(fin, (y + 2 * r + 1) * fstride + c, fstride, pp, o0, o1, o2),
                                           nlm_gen(fin, y * fstride + c, fstride, pp, o0, o1, o2)));
            }
        }
        __syncthreads();
        {
            const float4* vrow = vbuf + hy * vstride;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int i = 0; i <= 2 * r; ++i) acc = f4add(acc, vrow[hx0 + i]);
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const int x = hx0 + j;
                // centre phase theta(x) at tile index (hy + r, x + r)
                const int ic = (hy + r) * fstride + x + r;
                float th = o0 * fin[ic];
                if (pp > 1) th = fmaf(o1, fin[ic + 1], th);
                if (pp > 2) th = fmaf(o2, fin[ic + fstride], th);
                float sn, cs;
                __sincosf(th, &sn, &cs);
                const float a = wk * cs, b = wk * sn;
                P[j] = fmaf(a, acc.z, fmaf(b, acc.w, P[j]));
                Q[j] = fmaf(a, acc.x, fmaf(b, acc.y, Q[j]));
                if (j + 1 < G) acc = f4add(acc, f4sub(vrow[x + 2 * r + 1], vrow[x]));
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
                const float f = fin[(hy + r) * fstride + hx0 + j + r];
                const float q = Q[j];
                p.out[rowoff + gx] = (q > 0.f && isfinite(q)) ? kCenter + P[j] / q : kCenter + f;
            }
        }
    }
}

inline cudaError_t launch_nlm(const Params& p, const NlmTable& t, cudaStream_t s) {
    auto go = [&](auto kern, int TW, int TH) -> cudaError_t {
        const int TWI = TW + 2 * p.r, THI = TH + 2 * p.r;
        const int vstride = ((TWI + 7) & ~7) + 1;
        const size_t smem = (size_t)TH * vstride * 16 + (size_t)(THI + 1) * ((TWI + 1) | 1) * 4;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        dim3 grid((p.W + TW - 1) / TW, (p.out_rows + TH - 1) / TH);
        kern<<<grid, kThreads, smem, s>>>(p, t);
        return cudaGetLastError();
    };
    if (p.r <= 24) return go(nlm_tile_kernel<64, 64>, 64, 64);
    return go(nlm_tile_kernel<32, 32>, 32, 32);
}

}  // namespace sf
