// box_v2.cuh — band-sweep fused kernel for Algorithm 2 with
// the box spatial kernel and a compile-time radius R ("v2").
//
// Work unit (one CTA, 256 threads): a strip of TW = 8G output columns
// (TWI = TW + 2R input columns, one vertical walker per thread) by a band of
// rows, swept top to bottom in batches of RB = 16 rows.  For every batch and
// every conjugate pair k (plan.h):
//   vertical pass   — each column walker advances its moving sums of the four
//                     stack images cos, (f-c)cos, sin, (f-c)sin of w_k (f-c)
//                     by 16 rows ("recursion") and writes the
//                     16 vertical window sums to shared memory.  The running
//                     state lives in an L2-resident scratch between batches
//                     (32 B per column per pair), so there is no vertical
//                     halo except at the band top.  Exactness over long sweeps:
//                     block-reset sums — A (incoming rows of the current block
//                     of L = 2R+1 rows) and D (previous block minus outgoing
//                     rows), V = A + D, D := A every L rows — no difference of
//                     long sums is ever formed (precision rule P2/P3).
//   horizontal pass — 8 segments x 16 rows x 2 halves: the "cos" half sums
//                     (cos, (f-c)cos) and the "sin" half (sin, (f-c)sin) over
//                     the 2R+1 columns with a register ring (each vertical sum
//                     is read once from shared memory), then accumulates
//                     w_k cos(w_k f_x) (resp. sin) times its sums into its
//                     partial P', Q — registers, all pairs.
//   finalize        — the two halves add their partials (one shuffle) and
//                     write c + P'/Q (or the partial P', Q for the term split).
// Stack images are generated on the fly with MUFU sin/cos and never
// materialised.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"

namespace sf {

template <int R>
struct V2Cfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int NSEG = 8;
    static constexpr int G = (256 - 2 * R) / NSEG;     // outputs per horizontal walker
    static constexpr int TW = NSEG * G;                // output columns per strip
    static constexpr int TWI = TW + 2 * R;             // input columns (<= 256)
    static constexpr int RB = 16;                      // rows per batch
    static constexpr int PAD = (G % 2 == 0) ? 1 : 2;   // (G+PAD) odd: conflict-free segments
    static constexpr int NCOLP = TWI + (TWI / G + 1) * PAD;  // padded float4 per buffer row
    static constexpr int SMEM = RB * NCOLP * 16;
};

struct V2Extra {
    float4* scratch;    // [cta][pair][TWI][2] (A, D) running-sum state
    int band;           // rows per band (multiple of 16)
};

// (cos, v cos, sin, v sin) of om*v — the buffer layout (C, FC, S, FS)
__device__ __forceinline__ float4 gen4cs(float v, float om) {
    float s, c;
    __sincosf(om * v, &s, &c);
    return make_float4(c, v * c, s, v * s);
}

template <int R>
__global__ void __launch_bounds__(256, 1)
bilateral_box_v2(const Params p, const PairTable tab, const V2Extra ex) {
    using C = V2Cfg<R>;
    constexpr int L = C::L, G = C::G, RB = C::RB, PAD = C::PAD, NCOLP = C::NCOLP, TWI = C::TWI;
    extern __shared__ float4 vbuf[];                       // RB x NCOLP

    const int tid = threadIdx.x;
    const int npairs = tab.npairs;
    const int x0 = blockIdx.x * C::TW;
    const int yb0 = p.out_row0 + blockIdx.y * ex.band;
    const int yend = min(yb0 + ex.band, p.out_row0 + p.out_rows);

    // vertical walker (column c of the strip's input columns)
    const int c = tid;
    const bool vact = c < TWI;
    const int gxv = reflect101(x0 - R + (vact ? c : 0), p.W);
    const int cpad = c + (c / G) * PAD;
    float4* scr = ex.scratch + ((size_t)(blockIdx.y * gridDim.x + blockIdx.x) * npairs * TWI) * 2;

    // horizontal walker: row hry of the batch, segment hs, half hh (0: cos, 1: sin)
    const int hry = tid >> 4, hs = (tid >> 1) & 7, hh = tid & 1;
    const float hoff = hh ? 0.0f : 1.57079632679489662f;   // cos(t) = sin(t + pi/2)

    // ---- band top: D = sum of rows [yb0-R-1, yb0+R-1], A = 0, for every pair
    if (vact) {
        float fv[L];
#pragma unroll
        for (int i = 0; i < L; ++i) fv[i] = ldf(p, yb0 - R - 1 + i, gxv);
        for (int k = 0; k < npairs; ++k) {
            const float om = tab.omega[k];
            float4 D = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int i = 0; i < L; ++i) D = f4add(D, gen4cs(fv[i], om));
            scr[((size_t)k * TWI + c) * 2 + 0] = make_float4(0.f, 0.f, 0.f, 0.f);
            scr[((size_t)k * TWI + c) * 2 + 1] = D;
        }
    }

    for (int yb = yb0; yb < yend; yb += RB) {
        // inputs of this batch (pair-independent): incoming / outgoing rows of
        // the vertical walker, centre pixels of the horizontal walker
        float fin[RB], fout[RB];
        if (vact) {
#pragma unroll
            for (int i = 0; i < RB; ++i) {
                fin[i] = ldf(p, yb + i + R, gxv);
                fout[i] = ldf(p, yb + i - R - 1, gxv);
            }
        }
        float fpx[G], P[G], Q[G];
        {
            const int gy = yb + hry;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                fpx[j] = ldf(p, gy, reflect101(x0 + hs * G + j, p.W));
                P[j] = 0.f;
                Q[j] = 0.f;
            }
        }
        // block-reset phase of the first row of the batch
        const int ph0 = (yb - yb0) % L;

        for (int k = 0; k < npairs; ++k) {
            const float om = tab.omega[k], wk = tab.weight[k];
            // ---------------- vertical pass: 16 rows of moving sums
            if (vact) {
                float4* sp = scr + ((size_t)k * TWI + c) * 2;
                float4 A = sp[0], D = sp[1];
                int ph = ph0;
#pragma unroll
                for (int i = 0; i < RB; ++i) {
                    if (ph == 0 && (yb + i) > yb0) {          // block boundary: D := A
                        D = A;
                        A = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                    A = f4add(A, gen4cs(fin[i], om));
                    D = f4sub(D, gen4cs(fout[i], om));
                    vbuf[i * NCOLP + cpad] = f4add(A, D);
                    ph = (ph + 1 == L) ? 0 : ph + 1;
                }
                sp[0] = A;
                sp[1] = D;
            }
            __syncthreads();
            // ---------------- horizontal pass: ring of 2R+1 columns
            {
                const float2* vrow = reinterpret_cast<const float2*>(vbuf + hry * NCOLP + hs * (G + PAD)) + hh;
                float2 ring[L];
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < G + 2 * R; ++j) {
                    const float2 v = vrow[2 * (j + (j / G) * PAD)];
                    if (j >= L) {
                        acc.x -= ring[j % L].x;
                        acc.y -= ring[j % L].y;
                    }
                    acc.x += v.x;
                    acc.y += v.y;
                    ring[j % L] = v;
                    if (j >= 2 * R) {
                        const int o = j - 2 * R;
                        const float t = wk * __sinf(fmaf(om, fpx[o], hoff));
                        Q[o] = fmaf(t, acc.x, Q[o]);
                        P[o] = fmaf(t, acc.y, P[o]);
                    }
                }
            }
            __syncthreads();
        }

        // ---------------- combine the cos/sin halves and store
        const int gy = yb + hry;
        const bool rowok = gy < yend;
        const size_t rowoff = (size_t)(gy - p.out_row0) * p.W;
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const float pj = P[j] + __shfl_xor_sync(0xffffffffu, P[j], 1);
            const float qj = Q[j] + __shfl_xor_sync(0xffffffffu, Q[j], 1);
            const int gx = x0 + hs * G + j;
            if (rowok && gx < p.W && (j & 1) == hh) {
                if (p.out) {
                    p.out[rowoff + gx] = (qj > 0.f && isfinite(qj)) ? kCenter + pj / qj : kCenter + fpx[j];
                } else {
                    p.num[rowoff + gx] = pj;
                    p.den[rowoff + gx] = qj;
                }
            }
        }
    }
}

// Choose the band height: minimise waves x work with a band >= 4L rows.
inline int v2_band(int rows, int strips, int sms, int L) {
    int best = ((rows + 15) / 16) * 16;
    double best_cost = 1e30;
    const int minband = ((4 * L + 15) / 16) * 16 > 64 ? ((4 * L + 15) / 16) * 16 : 64;
    for (int nb = 1; nb <= 64; ++nb) {
        int band = ((rows + nb - 1) / nb + 15) / 16 * 16;
        if (band < minband && nb > 1) break;
        const int bands = (rows + band - 1) / band;
        const long units = (long)bands * strips;
        const long waves = (units + sms - 1) / sms;
        // time ~ waves x (band + band-top init of L rows)
        const double cost = (double)waves * (band + L);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = band;
        }
    }
    return best;
}

template <int R>
inline cudaError_t launch_box_v2(const Params& p, const PairTable& t, cudaStream_t s) {
    using C = V2Cfg<R>;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int strips = (p.W + C::TW - 1) / C::TW;
    V2Extra ex;
    ex.band = v2_band(p.out_rows, strips, sms, C::L);
    const int bands = (p.out_rows + ex.band - 1) / ex.band;
    const size_t scratch_bytes = (size_t)strips * bands * (t.npairs > 0 ? t.npairs : 1) * C::TWI * 32;
    cudaError_t e = cudaMallocAsync((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(bilateral_box_v2<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e == cudaSuccess) {
        bilateral_box_v2<R><<<dim3(strips, bands), 256, C::SMEM, s>>>(p, t, ex);
        e = cudaGetLastError();
    }
    cudaFreeAsync(ex.scratch, s);
    return e;
}

}  // namespace sf
