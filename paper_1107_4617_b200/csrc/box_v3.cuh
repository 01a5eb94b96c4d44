// box_v3.cuh — warp-specialised band-sweep kernel for Algorithm 2
// (PAPER.md:146-156), box spatial kernel, compile-time radius R.
//
// CTA = NV producer warps + 4 consumer warps, one output strip of TW = 4G
// columns x one band of rows, swept in batches of RB = 16 rows; for every
// (batch, conjugate pair) step the producers hand the consumers one 16-row
// slab of vertical moving sums through a double-buffered shared-memory ring
// (named barriers FULL/EMPTY), so generation + vertical sums overlap with the
// horizontal sums + recombination of the previous step.
//
//   producers (vertical, one input column per thread):
//     stack images cos, (f-c)cos, sin, (f-c)sin of w_k (f-c) (Alg. 2 step 1):
//       incoming row  — MUFU sin/cos;
//       outgoing row  — rotation recurrence across pairs (w_{k-1} = w_k - 2 gamma,
//                       z_{k-1} = z_k e^{-j 2 gamma (f-c)}), re-seeded with MUFU
//                       every kSeed pairs;
//     running vertical sums ("recursion"), state spilled to an
//     L2-resident scratch between batches (16 B per column per pair); bands
//     are <= 256 rows and start from an exact window sum, which bounds the
//     drift of the running sums (precision rule P3).
//   consumers (horizontal): walker = (row, segment, half); the cos half sums
//     (C, FC), the sin half (S, FS) over 2R+1 columns with a register ring
//     (each vertical sum read once, LDS.64), then adds w_k cos|sin(w_k f_x)
//     times its sums to its partial Q, P' (Alg. 2 step 3).
//     Partials stay in registers across all pairs; the two halves combine with
//     one shuffle and the band writes c + P'/Q (or P', Q for the term split).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"

namespace sf {

template <int R>
struct V3Cfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16;                                  // rows per step
    static constexpr int NSEG = 4;                                  // segments per row
    static constexpr int GREG = (210 - 2 * L) / 3;                  // register bound on G
    static constexpr int GCOL = (256 - 2 * R) / NSEG;               // <= 256 input columns
    static constexpr int G = GREG < GCOL ? GREG : GCOL;             // outputs per walker
    static constexpr int TW = NSEG * G;
    static constexpr int TWI = TW + 2 * R;
    static constexpr int NV = (TWI + 31) / 32;                      // producer warps
    static constexpr int NH = 4;                                    // consumer warps
    static constexpr int NT = 32 * (NV + NH);
    static constexpr int PAD = ((2 - G) % 8 + 8) % 8;               // (G + PAD) = 2 mod 8
    static constexpr int NSLOT = NSEG * (G + PAD) + 2 * R + 8;      // padded float4 per row
    static constexpr int NCOLP = NSLOT + ((1 - NSLOT) % 8 + 8) % 8;  // = 1 mod 8
    static constexpr int SMEM = 2 * RB * NCOLP * 16;                // double buffer
    static constexpr int kSeed = 8;                                 // rotation re-seed period
    static constexpr int MAXBAND = 256;
};

struct V3Extra {
    float4* scratch;     // [cta][pair][TWI] running vertical sums
    int band;            // rows per band (multiple of 16, <= 256)
    float two_gamma;     // w_{k} - w_{k-1}
};

__device__ __forceinline__ void nbar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int R>
__global__ void __launch_bounds__(V3Cfg<R>::NT, 1)
bilateral_box_v3(const Params p, const PairTable tab, const V3Extra ex) {
    using C = V3Cfg<R>;
    constexpr int L = C::L, G = C::G, RB = C::RB, PAD = C::PAD, NCOLP = C::NCOLP;
    constexpr int TWI = C::TWI, NT = C::NT;
    extern __shared__ float4 vbuf[];                     // [2][RB][NCOLP]

    const int tid = threadIdx.x;
    const int npairs = tab.npairs;
    const int x0 = blockIdx.x * C::TW;
    const int yb0 = p.out_row0 + blockIdx.y * ex.band;
    const int yend = min(yb0 + ex.band, p.out_row0 + p.out_rows);
    const int nbatch = (yend - yb0 + RB - 1) / RB;
    const int nsteps = nbatch * npairs;
    const int warp = tid >> 5;

    if (warp < C::NV) {
        // =========================== producers (vertical pass) =================
        asm volatile("setmaxnreg.dec.sync.aligned.u32 136;\n");
        const int c = tid;
        const bool act = c < TWI;
        const int gx = reflect101(x0 - R + (act ? c : 0), p.W);
        // padded slot of column c: segment s = floor((c - ?)...) -> columns are
        // laid out as [seg 0: G + PAD][seg 1]...; column c belongs to slot
        // c + PAD * min(c / G, NSEG) (the 2R tail columns follow the last segment)
        const int cseg = c / G < C::NSEG ? c / G : C::NSEG;
        const int cslot = c + PAD * cseg;
        float4* scr = ex.scratch + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * npairs * TWI;

        if (act) {                                       // band top: exact window sums
            float fv[L];
#pragma unroll
            for (int i = 0; i < L; ++i) fv[i] = ldf(p, yb0 - R - 1 + i, gx);
            for (int k = 0; k < npairs; ++k) {
                const float om = tab.omega[k];
                float4 V = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int i = 0; i < L; ++i) V = f4add(V, gen4cs(fv[i], om));
                scr[(size_t)k * TWI + c] = V;            // window of the row above the band
            }
        }
        int step = 0;
        for (int b = 0; b < nbatch; ++b) {
            const int yb = yb0 + b * RB;
            float fin[RB], fout[RB], uc[RB], us[RB], zc[RB], zs[RB];
#pragma unroll
            for (int i = 0; i < RB; ++i) {
                fin[i] = act ? ldf(p, yb + i + R, gx) : 0.f;
                fout[i] = act ? ldf(p, yb + i - R - 1, gx) : 0.f;
                __sincosf(-ex.two_gamma * fout[i], &us[i], &uc[i]);
            }
            for (int n = 0; n < npairs; ++n, ++step) {
                const int k = npairs - 1 - n;            // |w_k| ascending
                const float om = tab.omega[k];
                const int slot = step & 1;
                float4 V = act ? scr[(size_t)k * TWI + c] : make_float4(0.f, 0.f, 0.f, 0.f);
                if (n % C::kSeed == 0) {
#pragma unroll
                    for (int i = 0; i < RB; ++i) __sincosf(om * fout[i], &zs[i], &zc[i]);
                } else {
#pragma unroll
                    for (int i = 0; i < RB; ++i) {
                        const float a = zc[i], bb = zs[i];
                        zc[i] = fmaf(a, uc[i], -bb * us[i]);
                        zs[i] = fmaf(a, us[i], bb * uc[i]);
                    }
                }
                if (step >= 2) nbar_sync(3 + slot, NT);   // wait: slot consumed
                float4* dst = vbuf + slot * RB * NCOLP + cslot;
#pragma unroll
                for (int i = 0; i < RB; ++i) {
                    float s_, c_;
                    __sincosf(om * fin[i], &s_, &c_);
                    V.x += c_ - zc[i];
                    V.y += fmaf(fin[i], c_, -fout[i] * zc[i]);
                    V.z += s_ - zs[i];
                    V.w += fmaf(fin[i], s_, -fout[i] * zs[i]);
                    if (act) dst[i * NCOLP] = V;
                }
                nbar_arrive(1 + slot, NT);               // slot full
                if (act) scr[(size_t)k * TWI + c] = V;
            }
        }
    } else {
        // =========================== consumers (horizontal pass) ===============
        asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n");
        const int w = tid - 32 * C::NV;                  // 0..127
        const int hh = w & 1, hs = (w >> 1) & 3, hry = w >> 3;
        const float hoff = hh ? 0.0f : 1.57079632679489662f;
        int step = 0;
        for (int b = 0; b < nbatch; ++b) {
            const int yb = yb0 + b * RB;
            const int gy = yb + hry;
            float fpx[G], P[G], Q[G];
#pragma unroll
            for (int j = 0; j < G; ++j) {
                fpx[j] = ldf(p, gy, reflect101(x0 + hs * G + j, p.W));
                P[j] = 0.f;
                Q[j] = 0.f;
            }
            for (int n = 0; n < npairs; ++n, ++step) {
                const int k = npairs - 1 - n;
                const float om = tab.omega[k], wk = tab.weight[k];
                const int slot = step & 1;
                nbar_sync(1 + slot, NT);                  // wait: slot full
                const float2* vrow =
                    reinterpret_cast<const float2*>(vbuf + (slot * RB + hry) * NCOLP + hs * (G + PAD)) + hh;
                float2 ring[L];
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < G + 2 * R; ++j) {
                    // columns past this segment's G continue into the next segment
                    // (or the 2R tail), skipping its PAD slots
                    const int col = j + (j >= G ? PAD : 0);
                    const float2 v = vrow[2 * col];
                    if (j >= L) {
                        acc.x += v.x - ring[j % L].x;
                        acc.y += v.y - ring[j % L].y;
                    } else {
                        acc.x += v.x;
                        acc.y += v.y;
                    }
                    ring[j % L] = v;
                    if (j >= 2 * R) {
                        const int o = j - 2 * R;
                        const float t = wk * __sinf(fmaf(om, fpx[o], hoff));
                        Q[o] = fmaf(t, acc.x, Q[o]);
                        P[o] = fmaf(t, acc.y, P[o]);
                    }
                }
                if (step + 2 < nsteps) nbar_arrive(3 + slot, NT);   // slot empty
            }
            const bool rowok = gy < yend;
            const size_t rowoff = (size_t)(gy - p.out_row0) * p.W;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const float pj = P[j] + __shfl_xor_sync(0xffffffffu, P[j], 1);
                const float qj = Q[j] + __shfl_xor_sync(0xffffffffu, Q[j], 1);
                const int gxo = x0 + hs * G + j;
                if (rowok && gxo < p.W && (j & 1) == hh) {
                    if (p.out) {
                        p.out[rowoff + gxo] = (qj > 0.f && isfinite(qj)) ? kCenter + pj / qj : kCenter + fpx[j];
                    } else {
                        p.num[rowoff + gxo] = pj;
                        p.den[rowoff + gxo] = qj;
                    }
                }
            }
        }
    }
}

// band height: <= 256 rows, multiple of 16, minimising waves x (band + L)
inline int v3_band(int rows, int strips, int sms, int L, int maxband) {
    int best = 16;
    double best_cost = 1e30;
    for (int band = 16; band <= maxband; band += 16) {
        const long units = (long)strips * ((rows + band - 1) / band);
        const long waves = (units + sms - 1) / sms;
        const double cost = (double)waves * (band + L) + (band > rows ? 1e9 : 0.0);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = band;
        }
        if (band >= rows) break;
    }
    return best;
}

template <int R>
inline cudaError_t launch_box_v3(const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    using C = V3Cfg<R>;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int strips = (p.W + C::TW - 1) / C::TW;
    V3Extra ex;
    ex.band = v3_band(p.out_rows, strips, sms, C::L, C::MAXBAND);
    ex.two_gamma = (float)(2.0 * gamma);
    const int bands = (p.out_rows + ex.band - 1) / ex.band;
    const size_t scratch_bytes = (size_t)strips * bands * (t.npairs > 0 ? t.npairs : 1) * C::TWI * 16;
    cudaError_t e = cudaMallocAsync((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(bilateral_box_v3<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e == cudaSuccess) {
        bilateral_box_v3<R><<<dim3(strips, bands), C::NT, C::SMEM, s>>>(p, t, ex);
        e = cudaGetLastError();
    }
    cudaFreeAsync(ex.scratch, s);
    return e;
}

}  // namespace sf
