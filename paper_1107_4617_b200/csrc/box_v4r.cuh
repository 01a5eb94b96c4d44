// box_v4r.cuh — "v4r": warp-specialised band-sweep kernel for Algorithm 2
// (PAPER.md:146-156), box spatial kernel, compile-time radius R <= 16 with a
// register ring in the horizontal pass.
//
// CTA = 8 producer warps + 4 consumer warps; one output strip of TW = 4G
// columns (TWI = TW + 2R <= 256 input columns) x one band of rows, swept in
// batches of RB = 16 rows; per (batch, conjugate pair) step the producers hand
// the consumers a 16-row slab of vertical moving sums through a
// double-buffered shared-memory ring (named barriers FULL/EMPTY).
//
//   producers (vertical, one input column per thread):
//     stack images cos, (f-c)cos, sin, (f-c)sin of w_k (f-c) (Alg. 2 step 1):
//       incoming row  — MUFU sin/cos;
//       outgoing row  — rotation recurrence across pairs (w_{k-1} = w_k - 2 gamma,
//                       z_{k-1} = z_k e^{-j 2 gamma (f-c)}), re-seeded with MUFU
//                       every kSeed pairs;
//     running vertical sums ("recursion"), state spilled to an
//     L2-resident scratch between batches (16 B per column per pair; the next
//     pair's state is prefetched while the current one is processed); bands
//     start from an exact window sum (accumulated RB rows at a time with the
//     same rotation recurrence), which bounds the drift of the running sums.
//   consumers (horizontal): walker = (row, segment, half); the cos half sums
//     (C, FC), the sin half (S, FS) over 2R+1 columns with a register ring
//     (each vertical sum read once, LDS.64), then adds w_k cos|sin(w_k f_x)
//     times its sums to its partial (Q, P') (Alg. 2 step 3) —
//     packed f32x2 FADD2 / FFMA2.  Partials stay in registers across all
//     pairs; the centre values f_x are held as packed bf16 pairs (exact for
//     the integers -128..127) to make room for G up to 62 outputs per walker.
//     The two halves combine with one shuffle and the band writes c + P'/Q
//     (or P', Q for the term split).
//
// Registers (setmaxnreg): the register pool of a CTA is returned and granted
// per SM sub-partition, so every sub-partition must release at least what
// its consumer warp takes: 8 producer warps (two per sub-partition) at
// 168 -> 136 release 2*32*32 = 2048 = one consumer warp's 168 -> 232.  (With
// an odd producer-warp count one sub-partition starves and the CTA hangs.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"
#include "runtime.h"

namespace sf {

template <int R>
struct V4RCfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16;                                   // rows per step
    static constexpr int NSEG = 4;                                  // segments per row
    static constexpr int NV = 8;                                    // producer warps
    static constexpr int NH = 4;                                    // consumer warps
    static constexpr int NT = 32 * (NV + NH);                       // 384 threads
    // consumer registers: 2G (Q,P') + G/2 (bf16 f_x pairs) + 2L (ring) + ~32 <= 232
    // (the headroom keeps ptxas from spilling the centre values at R = 16)
    static constexpr int GREG = (2 * (200 - 2 * L)) / 5;
    static constexpr int GCOL = (32 * NV - 2 * R) / NSEG;           // TWI <= 256
    static constexpr int G0 = GREG < GCOL ? GREG : GCOL;
    static constexpr int G = G0 - (G0 & 1);                         // even: bf16 pairs
    static constexpr int TW = NSEG * G;
    static constexpr int TWI = TW + 2 * R;
    static constexpr int PAD = ((2 - G) % 8 + 8) % 8;               // (G + PAD) = 2 mod 8
    static constexpr int NSLOT = NSEG * (G + PAD) + 2 * R + 8;      // padded float4 per row
    static constexpr int NCOLP = NSLOT + ((1 - NSLOT) % 8 + 8) % 8;  // = 1 mod 8
    static constexpr int SMEM = 2 * RB * NCOLP * 16;                // double buffer
    static constexpr int kSeed = 8;                                 // rotation re-seed period
    static constexpr int MAXBAND = 256;
    static_assert(TWI <= 32 * NV && TWI > 32 * (NV - 1), "8 fully used producer warps");
    static_assert(2 * R <= G, "ring tail must stay within the next segment");
};

struct V4RExtra {
    float4* scratch;     // [slot][pair][TWI] running vertical sums
    int per_sm;          // unused (the slot is the CTA index; %smid is not stable)
    int band;            // rows per band (multiple of RB, <= MAXBAND)
    float two_gamma;     // w_k - w_{k-1}
};

__device__ __forceinline__ void v4r_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void v4r_bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// bf16 pair <-> two floats (exact for integer grey levels -128..127)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    return (__float_as_uint(lo) >> 16) | (__float_as_uint(hi) & 0xffff0000u);
}
__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

template <int R>
__global__ void __launch_bounds__(V4RCfg<R>::NT, 1)
bilateral_box_v4r(const Params p, const PairTable tab, const V4RExtra ex) {
    using C = V4RCfg<R>;
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
        // columns are laid out as [seg 0: G + PAD][seg 1]...[seg 3][2R tail]
        const int cseg = c / G < C::NSEG ? c / G : C::NSEG;
        const int cslot = c + PAD * cseg;
        const int slot_id = (int)(blockIdx.y * gridDim.x + blockIdx.x);   // one scratch slot per CTA
        float4* scr = ex.scratch + (size_t)slot_id * npairs * TWI;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);

        // band top: exact window sums of the row above the band, rows
        // [yb0-R-1, yb0+R-1], RB rows at a time, rotation across pairs
        if (act) {
            for (int i0 = 0; i0 < L; i0 += RB) {
                float fv[RB], zc[RB], zs[RB], uc[RB], us[RB];
#pragma unroll
                for (int i = 0; i < RB; ++i) {
                    fv[i] = (i0 + i < L) ? ldf(p, yb0 - R - 1 + i0 + i, gx) : 0.f;
                    __sincosf(-ex.two_gamma * fv[i], &us[i], &uc[i]);
                }
                float4 Vn = (i0 == 0 || npairs == 0) ? zero4 : scr[(size_t)(npairs - 1) * TWI + c];
                for (int n = 0; n < npairs; ++n) {
                    const int k = npairs - 1 - n;
                    const float om = tab.omega[k];
                    float4 V = Vn;
                    if (i0 > 0 && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWI + c];
#pragma unroll
                    for (int i = 0; i < RB; ++i) {
                        if (n % C::kSeed == 0) {
                            __sincosf(om * fv[i], &zs[i], &zc[i]);
                        } else {
                            const float a = zc[i], b = zs[i];
                            zc[i] = fmaf(a, uc[i], -b * us[i]);
                            zs[i] = fmaf(a, us[i], b * uc[i]);
                        }
                        if (i0 + i < L) {
                            V.x += zc[i];
                            V.y = fmaf(fv[i], zc[i], V.y);
                            V.z += zs[i];
                            V.w = fmaf(fv[i], zs[i], V.w);
                        }
                    }
                    scr[(size_t)k * TWI + c] = V;
                }
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
            float4 Vn = (act && npairs > 0) ? scr[(size_t)(npairs - 1) * TWI + c] : zero4;
            for (int n = 0; n < npairs; ++n, ++step) {
                const int k = npairs - 1 - n;            // |w_k| ascending
                const float om = tab.omega[k];
                const int slot = step & 1;
                float4 V = Vn;
                if (act && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWI + c];   // prefetch next pair
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
                if (step >= 2) v4r_bar_sync(3 + slot, NT);   // wait: slot consumed
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
                v4r_bar_arrive(1 + slot, NT);            // slot full
                if (act) scr[(size_t)k * TWI + c] = V;
            }
        }
        __threadfence();   // the next CTA on this SM reuses the scratch slot
    } else {
        // =========================== consumers (horizontal pass) ===============
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n");
        const int w = tid - 32 * C::NV;                  // 0..127
        const int hh = w & 1, hs = (w >> 1) & 3, hry = w >> 3;
        const float hoff = hh ? 0.0f : 1.57079632679489662f;
        int step = 0;
        for (int b = 0; b < nbatch; ++b) {
            const int yb = yb0 + b * RB;
            const int gy = yb + hry;
            uint32_t fpk[G / 2];                         // centre values, bf16 pairs
            float2 QP[G];                                // (Q, P') partials of this half
#pragma unroll
            for (int j = 0; j < G; j += 2) {
                fpk[j / 2] = pack_bf16x2(ldf(p, gy, reflect101(x0 + hs * G + j, p.W)),
                                         ldf(p, gy, reflect101(x0 + hs * G + j + 1, p.W)));
                QP[j] = make_float2(0.f, 0.f);
                QP[j + 1] = make_float2(0.f, 0.f);
            }
            for (int n = 0; n < npairs; ++n, ++step) {
                const int k = npairs - 1 - n;
                const float om = tab.omega[k], wk = tab.weight[k];
                const int slot = step & 1;
                v4r_bar_sync(1 + slot, NT);               // wait: slot full
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
                    acc = (j >= L) ? __fadd2_rn(acc, __fadd2_rn(v, make_float2(-ring[j % L].x, -ring[j % L].y)))
                                   : __fadd2_rn(acc, v);
                    ring[j % L] = v;
                    if (j >= 2 * R) {
                        const int o = j - 2 * R;
                        const float fx = (o & 1) ? bf16_hi(fpk[o / 2]) : bf16_lo(fpk[o / 2]);
                        const float t = wk * __sinf(fmaf(om, fx, hoff));
                        QP[o] = __ffma2_rn(make_float2(t, t), acc, QP[o]);
                    }
                }
                if (step + 2 < nsteps) v4r_bar_arrive(3 + slot, NT);   // slot empty
            }
            const bool rowok = gy < yend;
            const size_t rowoff = (size_t)(gy - p.out_row0) * p.W;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const float qj = QP[j].x + __shfl_xor_sync(0xffffffffu, QP[j].x, 1);
                const float pj = QP[j].y + __shfl_xor_sync(0xffffffffu, QP[j].y, 1);
                const int gxo = x0 + hs * G + j;
                if (rowok && gxo < p.W && (j & 1) == hh) {
                    if (p.out) {
                        const float fx = (j & 1) ? bf16_hi(fpk[j / 2]) : bf16_lo(fpk[j / 2]);
                        p.out[rowoff + gxo] = (qj > 0.f && isfinite(qj)) ? kCenter + pj / qj : kCenter + fx;
                    } else {
                        p.num[rowoff + gxo] = pj;
                        p.den[rowoff + gxo] = qj;
                    }
                }
            }
        }
    }
}

// Drift budget of the rotation recurrence for the outgoing rows (DESIGN.md
// reading R15): the running sums integrate the few-ulp difference between a
// row's incoming (MUFU) and outgoing (rotated) values, ~3.6e-5 rows w_max^4
// grey levels; the band (the running-sum segment) is capped to keep it under
// 0.0125 — the same budget as the v5 launcher (sf.cu v5_choice)
inline int drift_maxband(const PairTable& t, int maxband) {
    double wmax = 0.0;
    for (int k = 0; k < t.npairs; ++k) wmax = fmax(wmax, fabs((double)t.omega[k]));
    const double w4 = wmax * wmax * wmax * wmax;
    const double rows = w4 > 0.0 ? 0.0125 / (3.6e-5 * w4) : 1e9;
    int cap = (int)(rows / 16.0) * 16;
    cap = cap < 16 ? 16 : cap;
    return cap < maxband ? cap : maxband;
}

// band height: <= maxband rows, multiple of 16, minimising waves x (band + L/4)
// (the band-top init costs about a quarter of a full row per row of the window)
inline int v4r_band(int rows, int strips, int sms, int L, int maxband) {
    int best = 16;
    double best_cost = 1e30;
    for (int band = 16; band <= maxband; band += 16) {
        const long units = (long)strips * ((rows + band - 1) / band);
        const long waves = (units + sms - 1) / sms;
        const double cost = (double)waves * (band + 0.25 * L);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = band;
        }
        if (band >= rows) break;
    }
    return best;
}

template <int R>
inline cudaError_t launch_box_v4r(const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    using C = V4RCfg<R>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    const cudaError_t attr = cudaFuncSetAttribute(bilateral_box_v4r<R>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (attr != cudaSuccess) return attr;
    int per_sm_blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_blocks, bilateral_box_v4r<R>, C::NT, C::SMEM);
    const int strips = (p.W + C::TW - 1) / C::TW;
    V4RExtra ex;
    ex.band = v4r_band(p.out_rows, strips, di.sms, C::L, drift_maxband(t, C::MAXBAND));
    ex.two_gamma = (float)(2.0 * gamma);
    const int bands = (p.out_rows + ex.band - 1) / ex.band;
    ex.per_sm = 0;
    (void)per_sm_blocks;
    const size_t slots = (size_t)strips * bands;     // scratch slot = CTA index
    const size_t scratch_bytes = slots * (t.npairs > 0 ? t.npairs : 1) * C::TWI * 16;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    bilateral_box_v4r<R><<<dim3(strips, bands), C::NT, C::SMEM, s>>>(p, t, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
