// box_v5.cuh — "v5": warp-specialised band-sweep kernel for Algorithm 2
// (PAPER.md:146-156), box spatial kernel, compile-time radius R = 1..64
// (instantiated in v5_part.cu).  Two warps of each role per SM
// sub-partition, so that neither the vertical nor the horizontal pass is a
// single latency-bound warp (the v4r profile: its one consumer warp per
// sub-partition issued on 17% of its cycles while the producers waited at
// the barrier).
//
// CTA = NV producer warps + 8 consumer warps, one CTA per SM.  The work is
// the strip-major space of (output strip of TW = 8G columns, batch of RB = 16
// rows) units; each CTA takes one near-equal contiguous range of it (no wave
// quantisation), cut into segments at strip boundaries and at the drift cap
// (sf.cu, reading R15); each segment starts from an exact window
// sum.  Per (batch, conjugate pair) step the producers hand the consumers a
// 16-row slab of vertical moving sums through a double-buffered shared-memory
// ring (named barriers FULL/EMPTY per slot).
//
//   producers (vertical, one input column per thread): stack images
//     cos, (f-c)cos, sin, (f-c)sin of w_k (f-c) (Alg. 2 step 1) — incoming row
//     by MUFU sincos, outgoing row by the rotation recurrence across pairs
//     (re-seeded every kSeed pairs), or (OM = true) by MUFU sincos as well,
//     trading 4 FP32 + 4 registers per row for 2 MUFU; running vertical sums
//     ("recursion") with the state in a CTA-indexed,
//     L2-resident scratch (next pair prefetched).
//   consumers (horizontal, v4b's delta/scan walker): walker = (row, segment of
//     G outputs, half); the 8 segment walkers of a (row, half) are lanes of one
//     warp.  pass 1 reads the "in" and "out" vertical sums of each output
//     (no register ring, no halo re-read), keeps D_j = window(x_j) - S_s
//     implicitly by adding t_j D_j at once, and the segment's block total;
//     warp shuffles give every segment its start window S_s exactly (sums of
//     block totals + a telescoping scan); pass 2 adds t_j S_s.
//     t_j = cos|sin(w_k f_x) (Alg. 2 step 3), with w_k carried by
//     the deltas; (Q, P') stay in registers across all pairs; the halves
//     combine with one shuffle.
//
// Registers: R <= 32 — one uniform allocation of 128 (16 warps, no
// setmaxnreg); the producers hold their 2 x 16 row values as bf16 pairs and
// the consumers' segments are G = 24 outputs wide to fit.  R > 32 — 20 warps
// at 96 registers, producers 64 / consumers 144 via setmaxnreg (V5Cfg).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "box_kernel.cuh"
#include "runtime.h"

namespace sf {

template <int R>
struct V5Cfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16;                   // rows per step
    static constexpr int NSEG = 8;                  // segments per row (lanes of one warp)
    // outputs per walker: a consumer holds 3.5 G + ~25 registers and must fit
    // the uniform allocation of the CTA (no setmaxnreg)
    // (large R: G = 32, a 256-column strip, to cut the 2R-column producer halo)
    static constexpr int G = R > 32 ? 32 : 24;
    static constexpr int TW = NSEG * G;             // 192 (256) output columns per strip
    static constexpr int TWI = TW + 2 * R;
    static constexpr int NH = 8;                    // consumer warps
    // more than 16 warps (large R): registers per thread drop below 128, so the
    // producers (outgoing row by MUFU, no rotation state) shrink to PREG and
    // the consumers grow to CREG.  Then always 12 producer warps (the last
    // ones partly idle when TWI < 384): 20 warps compile to 96 registers, and
    // each sub-partition's 3 producer warps release 3*32*(96-64), exactly what
    // its 2 consumer warps take, 2*32*(144-96) (checked at launch, v5_pool_ok)
    static constexpr bool SMR = (TWI + 31) / 32 + NH > 16;
    static constexpr int NV = SMR ? 12 : (TWI + 31) / 32;   // producer warps
    static constexpr int NT = 32 * (NV + NH);
    static constexpr int PREG = 64, CREG = 144;
    static constexpr int PAD = ((1 - G) % 8 + 8) % 8;    // (G + PAD) = 1 mod 8: segments on disjoint banks
    // every producer lane computes a column (lanes past TWI repeat the last
    // input column into padding nobody reads): no per-lane predication, so
    // the pair step compiles to straight-line code for every R
    static constexpr int TWP = 32 * NV;
    static constexpr int NCOLP = TWP + PAD * (TWP / G) + 1;
    // slab ring depth: 3 when it fits in shared memory (absorbs step-time
    // jitter between the roles), else 2
    static constexpr int NBUF = 2;   // 3 measured no faster (profiles/r01_variants.jsonl)
    static constexpr int SMEM = NBUF * RB * NCOLP * 16;
    static constexpr int Q = L / G, PP = L % G;     // 2R+1 = Q G + PP
    static constexpr int CHMAX = SMR ? 8 : RB;       // init rows per chunk (register bound)
    static constexpr int NCH = (L + CHMAX - 1) / CHMAX;   // band-top init chunks
    static constexpr int CH = (L + NCH - 1) / NCH;  // rows per init chunk
    static constexpr int kSeed = 8;
    static_assert(TWI <= 384, "at most 12 producer warps");
    static_assert(!SMR || NV >= 8, "two producer warps per sub-partition");
    static_assert(Q < NSEG, "window must fit in the strip");
};

struct V5Extra {
    float4* scratch;     // [slot][pair][TWI] running vertical sums
    int diag;            // 0; 1 = consumers skip their arithmetic; 2 = producers skip theirs
                         // (SF_DIAG, tools: isolates each role's own step time)
    int bps;             // RB-row batches per strip (ceil(out_rows / RB))
    int total;           // strips * bps: the linear (strip, batch) work space
    int maxseg;          // batches per segment at most (running-sum restart)
    float two_gamma;     // w_k - w_{k-1}
    int psplit;          // v7 only: > 1 = pair split over a cluster of psplit CTAs per unit
};

__device__ __forceinline__ void v5_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void v5_bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// mbarriers for the slab ring (v5 / v7 MB kernels): FULL[slot] completes when every
// producer thread has stored its column of the slot (arrive has release.cta
// semantics), EMPTY[slot] when every consumer thread has read it;
// a waiting warp proceeds on its own phase, so consumer warps are not held in
// lockstep with each other as by a named barrier counting every thread
__device__ __forceinline__ uint32_t v7_smem_u32(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ void v7_mb_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(v7_smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void v7_mb_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(v7_smem_u32(b)) : "memory");
}
__device__ __forceinline__ void v7_mb_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "V7_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra V7_WAIT_%=;\n\t}\n" ::"r"(v7_smem_u32(b)), "r"(parity) : "memory");
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the phase
// completes (or the hint expires) instead of spinning on try_wait + branch.  Used
// by the wide kernel, whose consumers wait on the producers (ncu, v7w r = 64:
// SYNCS + BRA + MOV = 33 % of the consumer's instructions, issue slots taken from
// the role it waits for): r = 64 10.58 -> 10.47 ms; v7 is 0.4 % slower with it.
#ifndef SF_MB_SUSPEND_NS
#define SF_MB_SUSPEND_NS 20000u
#endif
__device__ __forceinline__ void v7_mb_wait_suspend(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "V7_WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra V7_WAITS_%=;\n\t}\n" ::"r"(v7_smem_u32(b)), "r"(parity), "r"(SF_MB_SUSPEND_NS) : "memory");
}

// bf16 pair <-> two floats (exact for integer grey levels -128..127)
__device__ __forceinline__ uint32_t v5_pack(float lo, float hi) {
    return (__float_as_uint(lo) >> 16) | (__float_as_uint(hi) & 0xffff0000u);
}
__device__ __forceinline__ float v5_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float v5_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// Per-segment centre for the OM kernels (reading R16): the median of 5 pixels
// of the segment's first output row across the strip.  Every pixel of every
// window a segment touches shares it, so f - c may replace f - 128 in the
// stack images and the phases (shiftability, SURVEY.md §8(d) "centering"); on
// flat backgrounds it keeps the window sums small.  Both roles compute it
// from the same pixels.  Returns 128 - c (an integer: f - c stays bf16-exact).
// (Measured free for the OM kernels; in the rotation kernels the extra live
// register cost 4 %, so those keep c = 128.)
__device__ __forceinline__ float v5_dc(const Params& p, int x0, int y, int tw) {
    float v[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] = ldf(p, y, min(x0 + k * (tw - 1) / 4, p.W - 1));
    auto cx = [](float& a, float& b) {               // median of 5: 7 compare-exchanges
        const float lo = fminf(a, b), hi = fmaxf(a, b);
        a = lo;
        b = hi;
    };
    cx(v[0], v[1]);
    cx(v[3], v[4]);
    cx(v[0], v[3]);
    cx(v[1], v[4]);
    cx(v[1], v[2]);
    cx(v[2], v[3]);
    cx(v[1], v[2]);
    return -v[2];                                    // -(c - 128)
}

// Balanced schedule: one CTA per SM; the (strip, batch) space, strip-major,
// is cut into gridDim.x near-equal contiguous ranges of RB-row batches, so
// every SM gets the same number of rows (no wave quantisation).  A range
// that crosses a strip boundary, or is longer than maxseg batches, becomes
// several segments, each with its own band-top window init.
struct V5Seg {
    int x0, yb0, yend, nbatch;
};
__device__ __forceinline__ V5Seg v5_seg(const Params& p, const V5Extra& ex, int tw, int rb, int u, int uend) {
    const int strip = u / ex.bps, b0 = u - strip * ex.bps;
    const int nb = min(min(ex.bps - b0, uend - u), ex.maxseg);
    V5Seg g;
    g.x0 = strip * tw;
    g.yb0 = p.out_row0 + b0 * rb;
    g.yend = min(g.yb0 + nb * rb, p.out_row0 + p.out_rows);
    g.nbatch = nb;
    return g;
}

#ifndef SF_V5_MB_DEFAULT
#define SF_V5_MB_DEFAULT 1   // measured: cfg5 r = 25 11.71 -> 11.18 ms, r = 48 12.72 -> 12.40, r = 64 12.55 -> 12.44
#endif

// MB: slab ring synchronised by mbarriers instead of named barriers (as v7)
template <int R, bool OM, bool MB = SF_V5_MB_DEFAULT>
__global__ void __launch_bounds__(V5Cfg<R>::NT, 1)
bilateral_box_v5(const Params p, const PairTable tab, const V5Extra ex) {
    using C = V5Cfg<R>;
    constexpr int L = C::L, G = C::G, RB = C::RB, PAD = C::PAD, NCOLP = C::NCOLP;
    constexpr int TWI = C::TWI, TWP = C::TWP, NT = C::NT, CH = C::CH;
    extern __shared__ float4 vbuf[];                     // [NBUF][RB][NCOLP]
    __shared__ uint64_t mbar[MB ? 2 * C::NBUF : 1];      // FULL[NBUF], EMPTY[NBUF]
    if constexpr (MB) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < C::NBUF; ++i) {
                v7_mb_init(&mbar[i], 32 * C::NV);
                v7_mb_init(&mbar[C::NBUF + i], 32 * C::NH);
            }
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
    }

    const int tid = threadIdx.x;
    const int npairs = tab.npairs;
    const int q = ex.total / gridDim.x, rem = ex.total % gridDim.x, bid = blockIdx.x;
    const int u_begin = bid * q + min(bid, rem);
    const int u_end = u_begin + q + (bid < rem ? 1 : 0);
    const int nsteps = (u_end - u_begin) * npairs;
    const int warp = tid >> 5;

    static_assert(!C::SMR || OM, "large-R configuration needs the register-light producer");
    if (warp < C::NV) {
        // =========================== producers (vertical pass) =================
        if constexpr (C::SMR) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n");
        const int c = tid;
        // large R (SMR, MUFU-bound producers): lanes past TWI stay idle;
        // otherwise every lane computes (see TWP)
        const bool act = !C::SMR || c < TWI;
        const int cs = c + PAD * (c / G);
        float4* scr = ex.scratch + (size_t)blockIdx.x * npairs * TWP;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, nbatch = sgm.nbatch;
            const int gx = reflect101(x0 - R + min(c, TWI - 1), p.W);
            const float dc = OM ? v5_dc(p, x0, yb0, C::TW) : 0.f;   // 128 - c
            auto fc = [&](float x) {                     // f - c from ldf's f - 128
                if constexpr (OM) return x + dc;
                else return x;
            };

            // band top: exact window sums of the row above the band, rows
            // [yb0-R-1, yb0+R-1], CH rows at a time, rotation across pairs
            if (act) {
                for (int i0 = 0; i0 < L; i0 += CH) {
                    float fv[CH], zc[CH], zs[CH], uc[CH], us[CH];
#pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        fv[i] = (i0 + i < L) ? fc(ldf(p, yb0 - R - 1 + i0 + i, gx)) : 0.f;
                        __sincosf(-ex.two_gamma * fv[i], &us[i], &uc[i]);
                    }
                    float4 Vn = (i0 == 0 || npairs == 0) ? zero4 : scr[(size_t)(npairs - 1) * TWP + c];
                    for (int n = 0; n < npairs; ++n) {
                        const int k = npairs - 1 - n;
                        const float om = tab.omega[k];
                        float4 V = Vn;
                        if (i0 > 0 && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWP + c];
#pragma unroll
                        for (int i = 0; i < CH; ++i) {
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
                        scr[(size_t)k * TWP + c] = V;
                    }
                }
            }
            // Main sweep.  Rows are handled in pairs (2i, 2i+1) in "planar" f32x2
            // registers — Zc = (zc_2i, zc_2i+1), Zs, Uc, Us — so the rotation
            // z <- z u is 4 packed instructions per row pair, in place, and the
            // per-row stack deltas are packed too; only the running sum V, which
            // is sequential in the row, stays scalar.
            constexpr int RP = RB / 2;
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                float2 Zc[OM ? 1 : RP], Zs[OM ? 1 : RP], Uc[OM ? 1 : RP], Us[OM ? 1 : RP];
                uint32_t fi2[RP], fo2[RP];                  // incoming / outgoing-row values, bf16 pairs
#pragma unroll
                for (int q = 0; q < RP; ++q) {
                    const int i = 2 * q;
                    fi2[q] = v5_pack(act ? fc(ldf(p, yb + i + R, gx)) : 0.f, act ? fc(ldf(p, yb + i + 1 + R, gx)) : 0.f);
                    const float fa = act ? fc(ldf(p, yb + i - R - 1, gx)) : 0.f;
                    const float fb = act ? fc(ldf(p, yb + i - R, gx)) : 0.f;
                    fo2[q] = v5_pack(fa, fb);
                    if constexpr (!OM) {
                        __sincosf(-ex.two_gamma * fa, &Us[q].x, &Uc[q].x);
                        __sincosf(-ex.two_gamma * fb, &Us[q].y, &Uc[q].y);
                    }
                }
                float4 Vn = (act && npairs > 0) ? scr[(size_t)(npairs - 1) * TWP + c] : zero4;
                // one pair step; `reseed` is a compile-time constant after the
                // unrolling below, so the rotation state needs no branch merges
                auto pair_step = [&](const int n, const bool reseed) {
                    const int k = npairs - 1 - n;            // |w_k| ascending
                    const float om = tab.omega[k];
                    const int slot = step % C::NBUF;
                    float4 V = Vn;
                    if (act && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWP + c];   // prefetch next pair
                    if constexpr (!OM) {
                        if (ex.diag == 2) {
                        } else if (reseed) {
#pragma unroll
                            for (int q = 0; q < RP; ++q) {
                                __sincosf(om * v5_lo(fo2[q]), &Zs[q].x, &Zc[q].x);
                                __sincosf(om * v5_hi(fo2[q]), &Zs[q].y, &Zc[q].y);
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < RP; ++q) {     // (zc + j zs)(uc + j us), planar
                                const float2 t = __fmul2_rn(Zc[q], Us[q]);
                                Zc[q] = __ffma2_rn(make_float2(-Zs[q].x, -Zs[q].y), Us[q], __fmul2_rn(Zc[q], Uc[q]));
                                Zs[q] = __ffma2_rn(Zs[q], Uc[q], t);
                            }
                        }
                    }
                    if (step >= C::NBUF) {                   // wait: slot consumed
                        if constexpr (MB) v7_mb_wait(&mbar[C::NBUF + slot], ((step / C::NBUF) - 1) & 1);
                        else v5_bar_sync(1 + C::NBUF + slot, NT);
                    }
                    float4* dst = vbuf + slot * RB * NCOLP + cs;
                    if (ex.diag != 2)
#pragma unroll
                    for (int q = 0; q < RP; ++q) {
                        const float2 Fi = make_float2(v5_lo(fi2[q]), v5_hi(fi2[q]));
                        const float2 Fo = make_float2(v5_lo(fo2[q]), v5_hi(fo2[q]));
                        const float2 arg = __fmul2_rn(make_float2(om, om), Fi);
                        float2 C2, S2, Co, So;
                        __sincosf(arg.x, &S2.x, &C2.x);
                        __sincosf(arg.y, &S2.y, &C2.y);
                        if constexpr (OM) {
                            const float2 ao = __fmul2_rn(make_float2(om, om), Fo);   // outgoing row: MUFU as well
                            __sincosf(ao.x, &So.x, &Co.x);
                            __sincosf(ao.y, &So.y, &Co.y);
                        } else {
                            Co = Zc[q];
                            So = Zs[q];
                        }
                        // stack deltas of both rows: (in - out) of cos, f cos, sin, f sin
                        const float2 Dc = __fadd2_rn(C2, make_float2(-Co.x, -Co.y));
                        const float2 Ds = __fadd2_rn(S2, make_float2(-So.x, -So.y));
                        const float2 Dfc = __ffma2_rn(Fi, C2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), Co));
                        const float2 Dfs = __ffma2_rn(Fi, S2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), So));
                        V.x += Dc.x;
                        V.y += Dfc.x;
                        V.z += Ds.x;
                        V.w += Dfs.x;
                        if (act) dst[(2 * q) * NCOLP] = V;
                        V.x += Dc.y;
                        V.y += Dfc.y;
                        V.z += Ds.y;
                        V.w += Dfs.y;
                        if (act) dst[(2 * q + 1) * NCOLP] = V;
                    }
                    if constexpr (MB) v7_mb_arrive(&mbar[slot]);   // slot full
                    else v5_bar_arrive(1 + slot, NT);
                    if (act) scr[(size_t)k * TWP + c] = V;
                    ++step;
                };
                for (int n0 = 0; n0 < npairs; n0 += C::kSeed) {
#pragma unroll
                    for (int m = 0; m < C::kSeed; ++m)
                        if (n0 + m < npairs) pair_step(n0 + m, m == 0);
                }
            }
        }   // segments
        __threadfence();   // the next CTA on this SM reuses the scratch slot
    } else {
        // =========================== consumers (horizontal pass) ===============
        static_assert(C::CREG == 144, "setmaxnreg immediate");
        if constexpr (C::SMR) asm volatile("setmaxnreg.inc.sync.aligned.u32 144;\n");
        const int w = tid - 32 * C::NV;                  // 0..255
        const int hh = w & 1, sg = (w >> 1) & 7, hry = w >> 4;
        const int lane = w & 31;
        const int rowbase = lane & 16;                   // lanes of this row: rowbase + 2*s + hh
        const float hoff = hh ? 0.0f : 1.57079632679489662f;
        const int xs = sg * G;                           // first output column (strip-relative)
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, yend = sgm.yend, nbatch = sgm.nbatch;
            const float dc = OM ? v5_dc(p, x0, yb0, C::TW) : 0.f;   // as the producers'
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                const int gy = yb + hry;
                float fxv[G];                                // centre values (f - c)
                float2 QP[G];
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    fxv[j] = ldf(p, gy, reflect101(x0 + xs + j, p.W));
                    if constexpr (OM) fxv[j] += dc;
                }
#pragma unroll
                for (int j = 0; j < G; ++j) QP[j] = make_float2(0.f, 0.f);
                for (int n = 0; n < npairs; ++n, ++step) {
                    const int k = npairs - 1 - n;
                    const float om = tab.omega[k], wk = tab.weight[k];
                    const int slot = step % C::NBUF;
                    if constexpr (MB) v7_mb_wait(&mbar[slot], (step / C::NBUF) & 1);   // wait: slot full
                    else v5_bar_sync(1 + slot, NT);
                    const float2* vrow = reinterpret_cast<const float2*>(vbuf + (slot * RB + hry) * NCOLP) + hh;
                    const float2* vo_row = vrow + 2 * (xs + PAD * sg);   // slot of column xs
                    if (ex.diag == 1) {
                        if (step + C::NBUF < nsteps) {
                        if constexpr (MB) v7_mb_arrive(&mbar[C::NBUF + slot]);
                        else v5_bar_arrive(1 + C::NBUF + slot, NT);
                    }
                        continue;
                    }
                    // pass 1
                    float T[G];
                    float2 dacc = make_float2(0.f, 0.f), bsum = make_float2(0.f, 0.f), bpre = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        // slot(c) = c + PAD*(c/G): out column xs+j is in segment sg;
                        // in column xs+j+L is (j+L)/G segments further (compile time)
                        const float2 vo = vo_row[2 * j];
                        const int ioff = (j + L) + PAD * ((j + L) / G);
                        const bool last = (j == G - 1);
                        const float2 vi = (!last || sg < C::NSEG - 1) ? vo_row[2 * ioff] : make_float2(0.f, 0.f);
                        if (j == C::PP) bpre = bsum;
                        bsum = __fadd2_rn(bsum, vo);
                        // w_k rides on the deltas (dacc = w_k D_j) instead of on T_j:
                        // one FFMA2 in place of an FADD2 + FMUL
                        T[j] = __sinf(fmaf(om, fxv[j], hoff));
                        QP[j] = __ffma2_rn(make_float2(T[j], T[j]), dacc, QP[j]);
                        dacc = __ffma2_rn(make_float2(wk, wk), __fadd2_rn(vi, make_float2(-vo.x, -vo.y)), dacc);
                    }
                    // S_0 = sum_{m<Q} B_m + prefix_Q(PP)
                    float2 S0 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int m = 0; m < C::Q; ++m) {
                        const int src = rowbase + 2 * m + hh;
                        S0.x += __shfl_sync(0xffffffffu, bsum.x, src);
                        S0.y += __shfl_sync(0xffffffffu, bsum.y, src);
                    }
                    {
                        const int src = rowbase + 2 * C::Q + hh;
                        S0.x += __shfl_sync(0xffffffffu, bpre.x, src);
                        S0.y += __shfl_sync(0xffffffffu, bpre.y, src);
                    }
                    // exclusive scan of the segment deltas over sg (stride 2 lanes)
                    float2 inc = dacc;
#pragma unroll
                    for (int d = 1; d < C::NSEG; d <<= 1) {
                        const float tx = __shfl_up_sync(0xffffffffu, inc.x, 2 * d);
                        const float ty = __shfl_up_sync(0xffffffffu, inc.y, 2 * d);
                        if (sg >= d) {
                            inc.x += tx;
                            inc.y += ty;
                        }
                    }
                    float2 exc;
                    exc.x = __shfl_up_sync(0xffffffffu, inc.x, 2);
                    exc.y = __shfl_up_sync(0xffffffffu, inc.y, 2);
                    if (sg == 0) exc = make_float2(0.f, 0.f);
                    const float2 Ss = __ffma2_rn(make_float2(wk, wk), S0, exc);   // w_k S_s
                    if (step + C::NBUF < nsteps) {
                        if constexpr (MB) v7_mb_arrive(&mbar[C::NBUF + slot]);
                        else v5_bar_arrive(1 + C::NBUF + slot, NT);
                    }   // slot empty
#pragma unroll
                    for (int j = 0; j < G; ++j) QP[j] = __ffma2_rn(make_float2(T[j], T[j]), Ss, QP[j]);
                }
                const bool rowok = gy < yend;
                const size_t rowoff = (size_t)(gy - p.out_row0) * p.W;
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const float qj = QP[j].x + __shfl_xor_sync(0xffffffffu, QP[j].x, 1);
                    const float pj = QP[j].y + __shfl_xor_sync(0xffffffffu, QP[j].y, 1);
                    const int gxo = x0 + xs + j;
                    if (rowok && gxo < p.W && (j & 1) == hh) {
                        if (p.out) {
                            const float fx = fxv[j];
                            const float cc = OM ? kCenter - dc : kCenter;
                            p.out[rowoff + gxo] = (qj > 0.f && isfinite(qj)) ? cc + pj / qj : cc + fx;
                        } else {
                            p.num[rowoff + gxo] = OM ? fmaf(-dc, qj, pj) : pj;   // centred at 128 (ABI)
                            p.den[rowoff + gxo] = qj;
                        }
                    }
                }
            }
        }   // segments
    }
}

// setmaxnreg moves registers within an SM sub-partition (warp w -> w % 4):
// each one's producers must free at least what its consumers claim, from the
// allocation the kernel was actually compiled to, else the CTA deadlocks.
inline bool v5_pool_ok(int regs, int nv, int nh, int preg, int creg) {
    for (int sp = 0; sp < 4; ++sp) {
        int np = 0, nc = 0;
        for (int w = 0; w < nv + nh; ++w)
            if (w % 4 == sp) (w < nv ? np : nc)++;
        if (np * (regs - preg) < nc * (creg - regs)) return false;
    }
    return regs * 32 * (nv + nh) <= 65536;
}

// maxseg: RB-row batches per running-sum segment (<= 0: unlimited); the
// SF_V5_MAXSEG environment variable overrides it (tools, A/B timing)
template <int R, bool OM = false>
inline cudaError_t launch_box_v5(const Params& p, const PairTable& t, double gamma, int maxseg, cudaStream_t s) {
    using C = V5Cfg<R>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    if constexpr (C::SMR) {
        static const bool pool_ok = [] {
            cudaFuncAttributes a{};
            return cudaFuncGetAttributes(&a, bilateral_box_v5<R, OM>) == cudaSuccess &&
                   v5_pool_ok(a.numRegs, C::NV, C::NH, C::PREG, C::CREG);
        }();
        if (!pool_ok) return cudaErrorLaunchOutOfResources;
    }
    const cudaError_t attr =
        cudaFuncSetAttribute(bilateral_box_v5<R, OM>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (attr != cudaSuccess) return attr;
    const int strips = (p.W + C::TW - 1) / C::TW;
    V5Extra ex;
    ex.bps = (p.out_rows + C::RB - 1) / C::RB;
    ex.total = strips * ex.bps;
    static const int maxseg_env = [] { const char* d = std::getenv("SF_V5_MAXSEG"); return d ? std::atoi(d) : 0; }();
    ex.maxseg = maxseg_env > 0 ? maxseg_env : (maxseg > 0 ? maxseg : ex.bps);
    ex.two_gamma = (float)(2.0 * gamma);
    const int grid = ex.total < di.sms ? ex.total : di.sms;   // one CTA per SM (__launch_bounds__(NT, 1), SMEM)
    static const int diag = [] { const char* d = std::getenv("SF_DIAG"); return d ? std::atoi(d) : 0; }();
    ex.diag = diag;

    const size_t scratch_bytes = (size_t)grid * (t.npairs > 0 ? t.npairs : 1) * C::TWP * 16;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    bilateral_box_v5<R, OM><<<grid, C::NT, C::SMEM, s>>>(p, t, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
