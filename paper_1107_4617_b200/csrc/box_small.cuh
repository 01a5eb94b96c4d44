// box_small.cuh — "vs": small-image kernel for Algorithm 2,
// box spatial kernel, compile-time radius R = 1..kVsMaxR.
//
// On an image with fewer (strip, 16-row batch) units than SMs (config 1,
// 256^2) the band-sweep kernels are bound by fixed cost, not arithmetic: a
// ~6 k-instruction kernel runs cold out of the instruction cache and every
// CTA pays a segment-top init.  This kernel is short and latency-oriented:
//
//   * CTA = one TH x TW output tile, NG = 4 independent groups of 256 threads;
//     group g runs the contiguous pair range [kb_g, ke_g) of the table, so a
//     CTA's critical path is npairs / 4 pair steps; the (Q, P') of the groups
//     are summed through shared memory at the end (no atomics, one launch).
//   * the centred tile + halo (d = f - c, c = the median of 5 pixels of the
//     tile's first output row, reading R16) is loaded once; the stack values
//     z_k(d) = e^{j w_k d} of every pixel advance across pairs by the rotation
//     z <- z e^{-j 2 gamma d} (w_{k-1} = w_k - 2 gamma, plan.h), seeded by one
//     sincos: no MUFU in the pair loop.
//   * per pair: (A) each thread writes the stack images (C, S) and (dC, dS)
//     of its pixels to shared memory (planar float2, Alg. 2 step 1); (B) one
//     thread per (input column, 4 output rows) runs the vertical moving sum
//     ("recursion") from 4 + 2R values held in registers;
//     (C) one thread per (output row, 2 outputs) the horizontal one, and
//     recombines at the centre, (Q, P') += w_k (C_x SC + S_x SS,
//     C_x SdC + S_x SdS) (Alg. 2 steps 2-3), the centre
//     values read from the stack images before the second barrier.
//   * output f~ = c + P'/Q (or the partials centred at kCenter, sf_accumulate).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"
#include "box_v4.cuh"
#include "box_v5.cuh"

namespace sf {

constexpr int kVsMaxR = 8;

template <int R>
struct VsCfg {
    static constexpr int TH = 16, TW = 32;         // output tile
    static constexpr int NG = 4, GT = 256;         // pair groups x threads per group
    static constexpr int NT = NG * GT;
    static constexpr int G = TW * TH / GT;         // outputs per phase-C thread (2)
    static constexpr int NSEG = TW / G;            // phase-C threads per row (16)
    static constexpr int L = 2 * R + 1;
    static constexpr int THI = TH + 2 * R, TWI = TW + 2 * R;
    static constexpr int NPIX = THI * TWI;
    static constexpr int NPX = (NPIX + GT - 1) / GT;    // pixels per phase-A thread
    static constexpr int SEGV = 4, NCH = TH / SEGV;     // phase B: 4 output rows per thread
    static constexpr int KB = SEGV + 2 * R, KC = G + 2 * R;   // values per B / C thread
    static_assert(TWI * NCH <= GT, "phase B: one thread per (column, chunk)");
    // per group (float2 planes): stack Scs, Sd [NPIX]; vertical sums Vcs, Vd [TH][TWI]
    static constexpr int GF2 = 2 * NPIX + 2 * TH * TWI;
    static constexpr int SMEM = NG * GF2 * 8;
};

__device__ __forceinline__ void vs_bar(int id) { asm volatile("bar.sync %0, 256;\n" ::"r"(id) : "memory"); }

// (f2add, f2sub: box_v4.cuh)

// windows of L consecutive values of v[0..K): w[j] = sum_{i<L} v[j+i], j < K - L + 1
// (first by a pairwise tree, then the running update w[j+1] = w[j] + v[j+L] - v[j])
template <int L, int K>
__device__ __forceinline__ void vs_windows(const float2 (&v)[K], float2 (&w)[K - L + 1]) {
    float2 t[L];
#pragma unroll
    for (int i = 0; i < L; ++i) t[i] = v[i];
#pragma unroll
    for (int s = 1; s < L; s *= 2) {
#pragma unroll
        for (int i = 0; i + s < L; i += 2 * s) t[i] = f2add(t[i], t[i + s]);
    }
    w[0] = t[0];
#pragma unroll
    for (int j = 1; j < K - L + 1; ++j) w[j] = f2add(w[j - 1], f2sub(v[j - 1 + L], v[j - 1]));
}

template <int R>
__global__ void __launch_bounds__(VsCfg<R>::NT, 1)
bilateral_box_small(const Params p, const PairTable tab, const float two_gamma) {
    using C = VsCfg<R>;
    constexpr int TH = C::TH, TW = C::TW, G = C::G, GT = C::GT, NPX = C::NPX, NPIX = C::NPIX;
    constexpr int TWI = C::TWI, L = C::L, KB = C::KB, KC = C::KC, SEGV = C::SEGV;
    extern __shared__ float2 smem2[];

    const int tiles_x = (p.W + TW - 1) / TW;
    const int x0 = (blockIdx.x % tiles_x) * TW;
    const int y0 = p.out_row0 + (blockIdx.x / tiles_x) * TH;
    const int g = threadIdx.x / GT, t = threadIdx.x % GT;
    float2* Scs = smem2 + (size_t)g * C::GF2;            // [THI][TWI]
    float2* Sd = Scs + NPIX;
    float2* Vcs = Sd + NPIX;                              // [TH][TWI]
    float2* Vd = Vcs + TH * TWI;
    const int kb = g * tab.npairs / C::NG, ke = (g + 1) * tab.npairs / C::NG;
    const float om0 = ke > kb ? tab.omega[ke - 1] : 0.f;  // |w| ascending: k = ke-1 .. kb
    const float dc = v5_dc(p, x0, min(y0, p.out_row0 + p.out_rows - 1), TW);   // 128 - c

    // phase-A pixels: d = f - c and the rotation factor e^{-j 2 gamma d}; z_k(d)
    // itself lives in the stack image Scs between pairs
    float2 ua[NPX];
    float da[NPX];
#pragma unroll
    for (int m = 0; m < NPX; ++m) {
        const int i = t + GT * m;
        const int iy = i / TWI, ix = i - iy * TWI;
        da[m] = (i < NPIX) ? ldf(p, y0 - R + iy, reflect101(x0 - R + ix, p.W)) + dc : 0.f;
        __sincosf(-two_gamma * da[m], &ua[m].y, &ua[m].x);
    }
    const int bc = t % TWI, bh = t / TWI;                 // phase B: column, chunk
    const int cy = t / C::NSEG, cx = (t % C::NSEG) * G;   // phase C: row, first output
    float2 QP[G];
#pragma unroll
    for (int j = 0; j < G; ++j) QP[j] = make_float2(0.f, 0.f);

    for (int k = ke - 1; k >= kb; --k) {
        const float wk = tab.weight[k];
        // (A) stack images of pair k: seeded by sincos, then z_k = z_{k+1} u
#pragma unroll
        for (int m = 0; m < NPX; ++m) {
            const int i = t + GT * m;
            if (i < NPIX) {
                float2 z;
                if (k == ke - 1) {
                    __sincosf(om0 * da[m], &z.y, &z.x);
                } else {
                    const float2 a = Scs[i];
                    z.x = fmaf(a.x, ua[m].x, -a.y * ua[m].y);
                    z.y = fmaf(a.x, ua[m].y, a.y * ua[m].x);
                }
                Scs[i] = z;
                Sd[i] = make_float2(da[m] * z.x, da[m] * z.y);
            }
        }
        vs_bar(1 + g);
        // centre values of this thread's phase-C outputs (read before the
        // second barrier: the next pair's phase A overwrites Scs after it)
        float2 zc[G];
#pragma unroll
        for (int j = 0; j < G; ++j) zc[j] = Scs[(cy + R) * TWI + cx + j + R];
        // (B) vertical moving sums, two channels at a time
        if (bh < C::NCH) {
            const int ys = bh * SEGV;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float2* col = (h ? Sd : Scs) + ys * TWI + bc;
                float2* dst = (h ? Vd : Vcs) + ys * TWI + bc;
                float2 v[KB], w[SEGV];
#pragma unroll
                for (int i = 0; i < KB; ++i) v[i] = col[i * TWI];
                vs_windows<L, KB>(v, w);
#pragma unroll
                for (int j = 0; j < SEGV; ++j) dst[j * TWI] = w[j];
            }
        }
        vs_bar(1 + g);
        // (C) horizontal moving sums and recombination at the centre
        {
            float2 wcs[G], wd[G];
            {
                const float2* row = Vcs + cy * TWI + cx;
                float2 v[KC];
#pragma unroll
                for (int i = 0; i < KC; ++i) v[i] = row[i];
                vs_windows<L, KC>(v, wcs);
            }
            {
                const float2* row = Vd + cy * TWI + cx;
                float2 v[KC];
#pragma unroll
                for (int i = 0; i < KC; ++i) v[i] = row[i];
                vs_windows<L, KC>(v, wd);
            }
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const float a = wk * zc[j].x, b = wk * zc[j].y;
                QP[j].x = fmaf(a, wcs[j].x, fmaf(b, wcs[j].y, QP[j].x));
                QP[j].y = fmaf(a, wd[j].x, fmaf(b, wd[j].y, QP[j].y));
            }
        }
    }

    // sum the groups' (Q, P') through shared memory (group g > 0 -> slot g - 1)
    __syncthreads();
    float2* red = smem2;                                  // [NG - 1][TH * TW]
    if (g > 0) {
#pragma unroll
        for (int j = 0; j < G; ++j) red[(g - 1) * TH * TW + cy * TW + cx + j] = QP[j];
    }
    __syncthreads();
    if (g > 0) return;
#pragma unroll
    for (int q = 1; q < C::NG; ++q) {
#pragma unroll
        for (int j = 0; j < G; ++j) QP[j] = f2add(QP[j], red[(q - 1) * TH * TW + cy * TW + cx + j]);
    }
    const int gy = y0 + cy;
    if (gy >= p.out_row0 + p.out_rows) return;
    const size_t rowoff = (size_t)(gy - p.out_row0) * p.W;
#pragma unroll
    for (int j = 0; j < G; ++j) {
        const int gx = x0 + cx + j;
        if (gx >= p.W) continue;
        const float q = QP[j].x, pp = QP[j].y;
        if (p.out) {
            p.out[rowoff + gx] = (q > 0.f && isfinite(q)) ? kCenter - dc + __fdividef(pp, q) : kCenter + ldf(p, gy, gx);
        } else {
            p.num[rowoff + gx] = fmaf(-dc, q, pp);   // centred at kCenter (ABI)
            p.den[rowoff + gx] = q;
        }
    }
}

template <int R>
inline cudaError_t launch_box_small_r(const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    using C = VsCfg<R>;
    cudaError_t e = cudaFuncSetAttribute(bilateral_box_small<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    const int tiles = ((p.W + C::TW - 1) / C::TW) * ((p.out_rows + C::TH - 1) / C::TH);
    bilateral_box_small<R><<<tiles, C::NT, C::SMEM, s>>>(p, t, (float)(2.0 * gamma));
    return cudaGetLastError();
}

inline cudaError_t launch_box_small(const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    switch (p.r) {
        case 1: return launch_box_small_r<1>(p, t, gamma, s);
        case 2: return launch_box_small_r<2>(p, t, gamma, s);
        case 3: return launch_box_small_r<3>(p, t, gamma, s);
        case 4: return launch_box_small_r<4>(p, t, gamma, s);
        case 5: return launch_box_small_r<5>(p, t, gamma, s);
        case 6: return launch_box_small_r<6>(p, t, gamma, s);
        case 7: return launch_box_small_r<7>(p, t, gamma, s);
        case 8: return launch_box_small_r<8>(p, t, gamma, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace sf
