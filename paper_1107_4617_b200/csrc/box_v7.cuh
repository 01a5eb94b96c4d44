// box_v7.cuh — "v7": band-sweep kernel of Algorithm 2, box
// spatial kernel, compile-time radius R = 1..24 (instantiated in v7_part.cu;
// DESIGN.md §5).  One CTA per SM on v5's balanced schedule: 8 producer warps
// (vertical pass, one input column per lane) and 8 consumer warps (horizontal
// pass and recombination) hand a 16-row slab of vertical moving sums through
// a double-buffered shared-memory ring.  What differs from v5:
//
//  * a consumer lane owns G consecutive outputs of one row with all four
//    channels (C, FC, S, FS): one LDS.128 per "out" and per "in" column, and
//    (Q, P') of its outputs complete in its own registers (no cross-half
//    shuffle).  Its centre values z_j = e^{j w_n d_j} advance across pairs by
//    the rotation z <- z u, u = e^{-j 2 gamma d} (w_{n+1} = w_n - 2 gamma),
//    planar over output pairs (4 packed FP32 per 2 outputs), seeded by MUFU
//    once per batch: 6 G registers per lane (z, u, (Q, P')) against 10 G per
//    output pair of lanes in the half split, so registers are left for the
//    loads in flight.  Rotation without re-seeding is as accurate as a MUFU
//    sincos per pair (weighted by the pair weights).
//
//  * G = 15 (r <= 8), 14 (r = 9..16), 13 (r = 17..24), the largest with
//    TWI = 16 G + 2R <= 256 = the 8 producer warps (lanes past TWI compute a
//    clamped column and skip the slab store).  G odd, no slab padding:
//    consumer lanes of a quarter-warp (8 segments of one row) read slots
//    G s + j (distinct mod 8: bank-conflict free), producer lanes write
//    consecutive slots (conflict free).  G even: a quarter-warp is 4 segments
//    x 2 rows (lane bits s3 s2 row s1 s0) and the slab rows are skewed by one
//    slot (row stride 257), so it reads slots 14 t + j + row: again distinct
//    mod 8; the row-wise shuffles become indexed shuffles in segment space.
//    The producers' cost per strip step is fixed (256 lanes), so the wider
//    strip is fewer producer steps: cfg5 r = 16 8.86 -> 8.64 ms, r = 12
//    8.71 -> 8.23 (40 -> 37 strips on 8192 columns).
//
//  * per-segment centre (reading R16) and segment start windows from block
//    sums: with Q = L / G, X_s = bsum_s + X_{s+1} (Q shuffle rounds,
//    X = bpre to start) gives S_s = sum_{i<Q} bsum_{s+i} + bpre_{s+Q}; the last
//    Q segments of a row chain S_s = S_{s-1} + D_{s-1}.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "box_kernel.cuh"
#include "box_v5.cuh"
#include "runtime.h"

namespace sf {

// first byte of image row gy (reflect-101; rows outside the caller's band
// are never needed by a valid window and clamp), as ldf
__device__ __forceinline__ const uint8_t* v7_row(const Params& p, int gy) {
    int ry = reflect101(gy, p.H) - p.img_row0;
    ry = ry < 0 ? 0 : (ry >= p.img_rows ? p.img_rows - 1 : ry);
    return p.img + (size_t)ry * p.W;
}

// barrier over every thread of the cluster (release / acquire: shared-memory
// stores before it, local or remote, are visible after it)
__device__ __forceinline__ void cluster_arrive_wait() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// generic address of the same shared-memory location in cluster rank 0
template <class T>
__device__ __forceinline__ T* cluster_map_rank0(T* ptr) {
    uint64_t r;
    asm volatile("mapa.u64 %0, %1, 0;\n" : "=l"(r) : "l"(ptr));
    return reinterpret_cast<T*>(r);
}

#ifndef SF_V7_MB_DEFAULT
#define SF_V7_MB_DEFAULT 1   // measured: r = 4 7.93 -> 7.43 ms, r = 24 10.09 -> 9.60, r = 16 unchanged
#endif
#ifndef SF_V7_SREG
#define SF_V7_SREG 8         // registers moved from each producer to each consumer warp (setmaxnreg)
#endif
#ifndef SF_V7_UNR
#define SF_V7_UNR 8          // producer pair-loop unroll (outgoing rows by MUFU)
#endif
#ifndef SF_V7W_UNR
#define SF_V7W_UNR 8         // wide kernel: producer pair-loop unroll
#endif
#ifndef SF_V7_CHAIN2
#define SF_V7_CHAIN2 0       // end-of-row start windows without the broadcast round (A/B: r = 16 8.89, r = 24 9.13 ms; no gain at r = 16, not adopted)
#endif
#ifndef SF_V7_NB_DEFAULT
#define SF_V7_NB_DEFAULT 2   // slab ring depth
#endif
#ifndef SF_V7_EVENG
#define SF_V7_EVENG 1        // even G (r = 9..16: G = 14, 224-column strips) on the row-skewed slab
#endif

// outputs per consumer lane: the largest odd G <= 15 with 16 G + 2R <= the
// producer lanes (256, or 384 for the wide large-radius kernel)
template <int R, int NCOL = 256>
struct V7G {
    static constexpr int raw = (NCOL - 2 * R) / 16 > 15 ? 15 : (NCOL - 2 * R) / 16;
    static constexpr int value = (raw % 2) ? raw : raw - 1;
};

// v7 (not WIDE): even G allowed (SF_V7_EVENG).  G = 14 for r = 9..16 (strips of
// 224 instead of 208 columns).  An even G needs another slab layout to stay
// bank-conflict free: a quarter-warp of consumer lanes is 4 segments x 2 rows
// and the slab rows are skewed by one slot (row stride NCOLP + 1), so its
// LDS.128 reads slots 14 t + j + row (t = 0..3, row = 0, 1): distinct mod 8.
template <int R>
struct V7GE {
    static constexpr int raw = (256 - 2 * R) / 16 > 15 ? 15 : (256 - 2 * R) / 16;
    static constexpr int value = (SF_V7_EVENG || raw % 2) ? raw : raw - 1;
};

// v7w (WIDE, 384 producer lanes): G = 16 (SF_V7W_EVENG): 256-column strips,
// TWI = 256 + 2R <= 384 for every r <= 64 (odd build: G = 15, 240 columns)
#ifndef SF_V7W_EVENG
#define SF_V7W_EVENG 1
#endif
template <int R>
struct V7GW {
    static constexpr int value = SF_V7W_EVENG && (384 - 2 * R) / 16 >= 16 ? 16 : V7G<R, 384>::value;
};

// WIDE: the large-radius configuration (r = 25..64): 12 producer warps (384
// input columns, 3 per SMSP) at 64 registers and 8 consumer warps at 144
// (20 warps compiled at 96: per SMSP 3 x 64 + 2 x 144 = 5 x 96), G = 16 on
// the padded slab (V7GW)
template <int R, int NB = SF_V7_NB_DEFAULT, int SREG = SF_V7_SREG, bool WIDE = false>
struct V7Cfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16;                   // rows per step
    static constexpr int NSEG = 16;                 // segments (lanes) per row
    static constexpr int NV = WIDE ? 12 : 8, NH = 8;   // producer / consumer warps
    static constexpr int NCOLP = 32 * NV;           // slab row stride (float4 slots)
    static constexpr int G = WIDE ? V7GW<R>::value : V7GE<R>::value;   // outputs per lane
    // G = 14: 4 segments x 2 rows per quarter-warp, slab rows skewed by one slot.
    // G = 16: the odd-G lane order on a slab padded by one slot per 16 columns
    // (slot(c) = c + c / 16): a quarter-warp reads slots 17 s + const for its
    // "out" and its "in" columns alike (16 | G, so c / 16 steps with s).
    static constexpr bool PAD = G == 16;
    static constexpr bool EVEN = G % 2 == 0 && !PAD;
    static constexpr int SROW = NCOLP + (PAD ? NCOLP / 16 : EVEN ? 1 : 0);   // slab row stride (float4 slots)
    static_assert(G % 2 == 1 || PAD || G % 8 == 6 || G % 8 == 2, "bank-conflict-free slab layouts");
    static constexpr int J2 = (G + 1) / 2;          // planar output pairs
    static constexpr int TW = NSEG * G;
    static constexpr int TWI = TW + 2 * R;
    static constexpr int NT = 32 * (NV + NH);
    static constexpr int NBUF = NB;                 // slab ring depth (2, or 3: looser role coupling)
    static constexpr int SMEM = NBUF * RB * SROW * 16;
    // SREG: registers moved from the producers to the consumers by setmaxnreg
    // (per SMSP 2 producer + 2 consumer warps, so a balanced move).  8 measured
    // best (cfg5 r = 16: 11.0 -> 8.9 ms; 16-32 spill the producers)
    static constexpr int PREG = WIDE ? 64 : 128 - SREG, CREG = WIDE ? 144 : 128 + SREG;
    static constexpr int CREGS = WIDE ? 96 : 128;   // compiled registers per thread
    static constexpr int Q = L / G, PP = L % G;     // 2R+1 = Q G + PP
    // start windows: Q <= 3 by Q rounds of block sums (+ a chain for the last Q
    // segments); wider windows by the telescoping scan over the row
    static constexpr bool TELE = Q > 3;
    static constexpr int CHMAX = WIDE ? 6 : RB;     // (WIDE: the producers' 64 registers)
    static constexpr int NCH = (L + CHMAX - 1) / CHMAX;            // band-top init chunks
    static constexpr int CH = (L + NCH - 1) / NCH;                 // rows per init chunk
    static constexpr int kSeed = 8;                 // producer rotation re-seed interval
    static constexpr int UNR = WIDE ? SF_V7W_UNR : SF_V7_UNR;   // producer pair-loop unroll (OM)
    static_assert(TWI <= NCOLP, "strip within the producer lanes");
    static_assert(Q < NSEG, "the window fits in the row's segments");
};

// PS: the pair-split instantiation (cluster launch, ex.psplit > 1)
// MB: slab ring synchronised by mbarriers instead of named barriers
template <int R, bool OM, int NB = SF_V7_NB_DEFAULT, int SREG = SF_V7_SREG, bool PS = false, bool MB = SF_V7_MB_DEFAULT,
          bool WIDE = false>
__global__ void __launch_bounds__(V7Cfg<R, NB, SREG, WIDE>::NT, 1)
bilateral_box_v7(const Params p, const PairTable tab, const V5Extra ex) {
    using C = V7Cfg<R, NB, SREG, WIDE>;
    constexpr int L = C::L, G = C::G, J2 = C::J2, RB = C::RB, NCOLP = C::NCOLP;
    constexpr int TWI = C::TWI, NT = C::NT, CH = C::CH, SROW = C::SROW;
    extern __shared__ float4 vbuf[];                     // [NBUF][RB][SROW]
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
    // pair split (PS, small images): a cluster of ps CTAs shares one (strip,
    // batch) unit, CTA `prank` runs pairs [kb, kb + npairs) of the table, and
    // the partial (Q, P') are summed in rank 0's shared memory
    const int ps = PS ? ex.psplit : 1;
    const int prank = PS ? (int)(blockIdx.x % ps) : 0;
    const int kb = PS ? prank * tab.npairs / ps : 0;
    const int npairs = PS ? (prank + 1) * tab.npairs / ps - kb : tab.npairs;
    const int q = ex.total / gridDim.x, rem = ex.total % gridDim.x, bid = blockIdx.x;
    const int u_begin = PS ? bid / ps : bid * q + min(bid, rem);
    const int u_end = PS ? u_begin + 1 : u_begin + q + (bid < rem ? 1 : 0);
    const int nsteps = (u_end - u_begin) * npairs;
    const int warp = tid >> 5;

    if (warp < C::NV) {
        // =========================== producers (vertical pass) =================
        if constexpr (SREG > 0 || WIDE) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::PREG));
        const int c = tid;                               // slab slot = input column
        const bool act = c < TWI;                        // lanes past TWI compute a clamped column
        float4* scr = ex.scratch + (size_t)blockIdx.x * (PS ? tab.npairs : npairs) * NCOLP;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, nbatch = sgm.nbatch;
            const int gx = reflect101(x0 - R + min(c, TWI - 1), p.W);
            const float dc = v5_dc(p, x0, yb0, C::TW);   // 128 - c (reading R16)
            auto fc = [&](float x) { return x + dc; };   // f - c from ldf's f - 128

            if constexpr (PS) {
                // pair split (small images: the init is a large share): the same
                // window sums planar f32x2 over row pairs (rows past L seeded with
                // z = 0, which the rotation keeps at 0).  Only in this
                // instantiation: in the large-image kernel the change perturbed
                // the pair loop's code (cfg5 8.89 -> 9.16 ms)
                for (int i0 = 0; i0 < L; i0 += CH) {
                    constexpr int CP = (CH + 1) / 2;
                    float2 Fv[CP], Zc[CP], Zs[CP], Uc[CP], Us[CP];
                    auto valid = [&](int i) { return i < CH && i0 + i < L; };
#pragma unroll
                    for (int q = 0; q < CP; ++q) {
                        Fv[q].x = valid(2 * q) ? fc(ldf(p, yb0 - R - 1 + i0 + 2 * q, gx)) : 0.f;
                        Fv[q].y = valid(2 * q + 1) ? fc(ldf(p, yb0 - R + i0 + 2 * q, gx)) : 0.f;
                        __sincosf(-ex.two_gamma * Fv[q].x, &Us[q].x, &Uc[q].x);
                        __sincosf(-ex.two_gamma * Fv[q].y, &Us[q].y, &Uc[q].y);
                    }
                    float4 Vn = (i0 == 0 || npairs == 0) ? zero4 : scr[(size_t)(npairs - 1) * NCOLP + c];
                    for (int n = 0; n < npairs; ++n) {
                        const int k = npairs - 1 - n;
                        const float om = tab.omega[kb + k];
                        float4 V = Vn;
                        if (i0 > 0 && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * NCOLP + c];
                        if (n % C::kSeed == 0) {
#pragma unroll
                            for (int q = 0; q < CP; ++q) {
                                __sincosf(om * Fv[q].x, &Zs[q].x, &Zc[q].x);
                                __sincosf(om * Fv[q].y, &Zs[q].y, &Zc[q].y);
                                if (!valid(2 * q)) Zc[q].x = Zs[q].x = 0.f;
                                if (!valid(2 * q + 1)) Zc[q].y = Zs[q].y = 0.f;
                            }
                        } else {
#pragma unroll
                            for (int q = 0; q < CP; ++q) {       // (zc + j zs)(uc + j us), planar
                                const float2 t = __fmul2_rn(Zc[q], Us[q]);
                                Zc[q] = __ffma2_rn(make_float2(-Zs[q].x, -Zs[q].y), Us[q], __fmul2_rn(Zc[q], Uc[q]));
                                Zs[q] = __ffma2_rn(Zs[q], Uc[q], t);
                            }
                        }
                        float2 aC = make_float2(0.f, 0.f), aF = aC, aS = aC, aG = aC;
#pragma unroll
                        for (int q = 0; q < CP; ++q) {
                            aC = __fadd2_rn(aC, Zc[q]);
                            aF = __ffma2_rn(Fv[q], Zc[q], aF);
                            aS = __fadd2_rn(aS, Zs[q]);
                            aG = __ffma2_rn(Fv[q], Zs[q], aG);
                        }
                        V.x += aC.x + aC.y;
                        V.y += aF.x + aF.y;
                        V.z += aS.x + aS.y;
                        V.w += aG.x + aG.y;
                        scr[(size_t)k * NCOLP + c] = V;
                    }
                }
            } else {
                // segment top: exact window sums of the row above the segment,
                // rows [yb0-R-1, yb0+R-1], CH rows at a time, rotation across pairs
                for (int i0 = 0; i0 < L; i0 += CH) {
                    float fv[CH], zc[CH], zs[CH], uc[CH], us[CH];
    #pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        fv[i] = (i0 + i < L) ? fc(ldf(p, yb0 - R - 1 + i0 + i, gx)) : 0.f;
                        __sincosf(-ex.two_gamma * fv[i], &us[i], &uc[i]);
                    }
                    float4 Vn = (i0 == 0 || npairs == 0) ? zero4 : scr[(size_t)(npairs - 1) * NCOLP + c];
                    for (int n = 0; n < npairs; ++n) {
                        const int k = npairs - 1 - n;
                        const float om = tab.omega[kb + k];
                        float4 V = Vn;
                        if (i0 > 0 && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * NCOLP + c];
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
                        scr[(size_t)k * NCOLP + c] = V;
                    }
                }
            }
            // main sweep: rows in planar f32x2 pairs (2i, 2i+1), as in v5
            constexpr int RP = RB / 2;
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                float2 Zc[OM ? 1 : RP], Zs[OM ? 1 : RP], Uc[OM ? 1 : RP], Us[OM ? 1 : RP];
                uint32_t fi2[RP], fo2[RP];                  // incoming / outgoing-row values, bf16 pairs
#pragma unroll
                for (int q = 0; q < RP; ++q) {
                    const int i = 2 * q;
                    fi2[q] = v5_pack(fc(ldf(p, yb + i + R, gx)), fc(ldf(p, yb + i + 1 + R, gx)));
                    const float fa = fc(ldf(p, yb + i - R - 1, gx));
                    const float fb = fc(ldf(p, yb + i - R, gx));
                    fo2[q] = v5_pack(fa, fb);
                    if constexpr (!OM) {
                        __sincosf(-ex.two_gamma * fa, &Us[q].x, &Uc[q].x);
                        __sincosf(-ex.two_gamma * fb, &Us[q].y, &Uc[q].y);
                    }
                }
                float4 Vn = npairs > 0 ? scr[(size_t)(npairs - 1) * NCOLP + c] : zero4;
                auto pair_step = [&](const int n, const bool reseed) {
                    const int k = npairs - 1 - n;            // |w_k| ascending
                    const float om = tab.omega[kb + k];
                    const int slot = step % C::NBUF;
                    float4 V = Vn;
                    if (n + 1 < npairs) Vn = scr[(size_t)(k - 1) * NCOLP + c];   // prefetch next pair
                    if constexpr (!OM) {
                        if (reseed) {
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
                        if constexpr (MB && WIDE) v7_mb_wait_suspend(&mbar[C::NBUF + slot], ((step / C::NBUF) - 1) & 1);
                        else if constexpr (MB) v7_mb_wait(&mbar[C::NBUF + slot], ((step / C::NBUF) - 1) & 1);
                        else v5_bar_sync(1 + C::NBUF + slot, NT);
                    }
                    float4* dst = vbuf + slot * RB * SROW + (C::PAD ? c + (c >> 4) : c);
#pragma unroll
                    for (int q = 0; q < RP; ++q) {
                        const float2 Fi = make_float2(v5_lo(fi2[q]), v5_hi(fi2[q]));
                        const float2 Fo = make_float2(v5_lo(fo2[q]), v5_hi(fo2[q]));
                        const float2 arg = __fmul2_rn(make_float2(om, om), Fi);
                        float2 C2, S2, Co, So;
                        __sincosf(arg.x, &S2.x, &C2.x);
                        __sincosf(arg.y, &S2.y, &C2.y);
                        if constexpr (OM) {
                            const float2 ao = __fmul2_rn(make_float2(om, om), Fo);
                            __sincosf(ao.x, &So.x, &Co.x);
                            __sincosf(ao.y, &So.y, &Co.y);
                        } else {
                            Co = Zc[q];
                            So = Zs[q];
                        }
                        const float2 Dc = __fadd2_rn(C2, make_float2(-Co.x, -Co.y));
                        const float2 Ds = __fadd2_rn(S2, make_float2(-So.x, -So.y));
                        const float2 Dfc = __ffma2_rn(Fi, C2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), Co));
                        const float2 Dfs = __ffma2_rn(Fi, S2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), So));
                        V.x += Dc.x;
                        V.y += Dfc.x;
                        V.z += Ds.x;
                        V.w += Dfs.x;
                        if (act) dst[(2 * q) * SROW] = V;   // lanes past TWI: no slab traffic
                        V.x += Dc.y;
                        V.y += Dfc.y;
                        V.z += Ds.y;
                        V.w += Dfs.y;
                        if (act) dst[(2 * q + 1) * SROW] = V;
                    }
                    if constexpr (MB) {                      // slot full
                        v7_mb_arrive(&mbar[slot]);
                    } else {
                        v5_bar_arrive(1 + slot, NT);
                    }
                    scr[(size_t)k * NCOLP + c] = V;
                    ++step;
                };
                // unrolled kSeed pairs deep also for OM (a plain loop: 8.9 -> 9.6 ms)
                if constexpr (OM) {
                    for (int n0 = 0; n0 < npairs; n0 += C::UNR) {
#pragma unroll
                        for (int m = 0; m < C::UNR; ++m)
                            if (n0 + m < npairs) pair_step(n0 + m, m == 0);
                    }
                } else {
                    for (int n0 = 0; n0 < npairs; n0 += C::kSeed) {
#pragma unroll
                        for (int m = 0; m < C::kSeed; ++m)
                            if (n0 + m < npairs) pair_step(n0 + m, m == 0);
                    }
                }
            }
        }   // segments
        __threadfence();   // the next launch reuses the scratch slot
        if (PS) {          // the consumers' two cluster barriers (pair-split reduction)
            cluster_arrive_wait();
            cluster_arrive_wait();
        }
    } else {
        // =========================== consumers (horizontal pass) ===============
        if constexpr (SREG > 0 || WIDE) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::CREG));
        const int w = tid - 32 * C::NV;                  // 0..255
        // segment, row in the batch (even G: lane bits (s3 s2 row s1 s0))
        const int sg = C::EVEN ? (((w >> 3) & 3) << 2) | (w & 3) : w & 15;
        const int hry = C::EVEN ? ((w >> 5) << 1) | ((w >> 2) & 1) : w >> 4;
        // lane of segment s of this lane's row
        auto seg_lane = [&](int s) { return (C::EVEN ? ((s >> 2) << 3) | (w & 4) | (s & 3) : (w & 16) | s) & 31; };
        // value of the lane i segments further along / back along this lane's row.
        // Even G: the source lanes (i = 1..Q down, 1..Q up, segment s0) packed 5 bits
        // each in one register (shfl.idx reads bits 4:0 of its lane operand), opaque to
        // the compiler so that it is not recomputed from the lane id in the pair loop
        static_assert(!C::EVEN || C::Q <= 2, "2 Q + 1 lane indices in 32 bits");
        unsigned pk = 0;
        if constexpr (C::EVEN) {
#pragma unroll
            for (int i = 1; i <= C::Q; ++i) {
                pk |= (unsigned)seg_lane(sg + i) << (5 * (i - 1));
                pk |= (unsigned)seg_lane(sg - i) << (5 * (C::Q + i - 1));
            }
            pk |= (unsigned)seg_lane(C::NSEG - 1 - C::Q) << (10 * C::Q);
            asm volatile("" : "+r"(pk));
        }
        auto shdn = [&](float v, int i) {
            if constexpr (C::EVEN) return __shfl_sync(0xffffffffu, v, (int)(pk >> (5 * (i - 1))));
            else return __shfl_down_sync(0xffffffffu, v, i);
        };
        auto shup = [&](float v, int i) {
            if constexpr (C::EVEN) return __shfl_sync(0xffffffffu, v, (int)(pk >> (5 * (C::Q + i - 1))));
            else return __shfl_up_sync(0xffffffffu, v, i);
        };
        const int xs = sg * G;                           // first output column (strip-relative)
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, yend = sgm.yend, nbatch = sgm.nbatch;
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                const int gy = yb + hry;
                float2 Zc[J2], Zs[J2], Uc[J2], Us[J2];       // planar over outputs (2j, 2j+1)
                float2 QP[G];
                {
                    const float dc = v5_dc(p, x0, yb0, C::TW);
                    const float om0 = npairs > 0 ? tab.omega[kb + npairs - 1] : 0.f;
                    const uint8_t* rowp = v7_row(p, gy);
                    const int cx0 = x0 + xs;
                    const float bias = 8388608.0f + kCenter - dc;   // uint8 -> float by the exponent trick
                    float d[2 * J2];
                    if (cx0 + G <= p.W) {
#pragma unroll
                        for (int j = 0; j < G; ++j) d[j] = __uint_as_float(0x4B000000u | __ldg(rowp + cx0 + j)) - bias;
                    } else {
#pragma unroll
                        for (int j = 0; j < G; ++j)
                            d[j] = __uint_as_float(0x4B000000u | __ldg(rowp + reflect101(cx0 + j, p.W))) - bias;
                    }
                    if (G % 2) d[G] = 0.f;
#pragma unroll
                    for (int h = 0; h < J2; ++h) {
                        __sincosf(om0 * d[2 * h], &Zs[h].x, &Zc[h].x);
                        __sincosf(om0 * d[2 * h + 1], &Zs[h].y, &Zc[h].y);
                        __sincosf(-ex.two_gamma * d[2 * h], &Us[h].x, &Uc[h].x);
                        __sincosf(-ex.two_gamma * d[2 * h + 1], &Us[h].y, &Uc[h].y);
                    }
#pragma unroll
                    for (int j = 0; j < G; ++j) QP[j] = make_float2(0.f, 0.f);
                }
                for (int n = 0; n < npairs; ++n, ++step) {
                    const int k = npairs - 1 - n;
                    const float wk = tab.weight[kb + k];
                    const int slot = step % C::NBUF;
                    if constexpr (MB && WIDE) v7_mb_wait_suspend(&mbar[slot], (step / C::NBUF) & 1);   // wait: slot full
                    else if constexpr (MB) v7_mb_wait(&mbar[slot], (step / C::NBUF) & 1);
                    else v5_bar_sync(1 + slot, NT);
                    const float4* vrow = vbuf + (slot * RB + hry) * SROW + (C::PAD ? 17 * sg : xs);
                    // pass 1: window increments D_j = V(x_j + L) - V(x_j) (w-weighted,
                    // running), block sums of the "out" columns
                    float2 dcf = make_float2(0.f, 0.f), dsf = dcf;
                    float2 bcf = dcf, bsf = dcf, pcf = dcf, psf = dcf;
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        const float4 vo = vrow[j];
                        const bool last = (j == G - 1);
                        const float4 vi = (!last || sg < C::NSEG - 1) ? vrow[C::PAD ? j + L + ((j + L) >> 4) : j + L]
                                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                        if (j == C::PP) {
                            pcf = bcf;
                            psf = bsf;
                        }
                        bcf = __fadd2_rn(bcf, make_float2(vo.x, vo.y));
                        bsf = __fadd2_rn(bsf, make_float2(vo.z, vo.w));
                        const float zc = (j & 1) ? Zc[j / 2].y : Zc[j / 2].x;
                        const float zs = (j & 1) ? Zs[j / 2].y : Zs[j / 2].x;
                        QP[j] = __ffma2_rn(make_float2(zc, zc), dcf, QP[j]);
                        QP[j] = __ffma2_rn(make_float2(zs, zs), dsf, QP[j]);
                        dcf = __ffma2_rn(make_float2(wk, wk), __fadd2_rn(make_float2(vi.x, vi.y), make_float2(-vo.x, -vo.y)), dcf);
                        dsf = __ffma2_rn(make_float2(wk, wk), __fadd2_rn(make_float2(vi.z, vi.w), make_float2(-vo.z, -vo.w)), dsf);
                    }
                    if (step + C::NBUF < nsteps) {                                       // slot empty
                        if constexpr (MB) {
                            v7_mb_arrive(&mbar[C::NBUF + slot]);
                        } else {
                            v5_bar_arrive(1 + C::NBUF + slot, NT);
                        }
                    }
                    float2 scf, ssf;                          // w_k S_s
                    if constexpr (C::TELE) {
                        // telescoping: w S_s = w S_0 + sum_{s' < s} dacc_{s'} (exclusive
                        // scan of the lanes' window increments over the row), with
                        // S_0 = sum_{c < L} V(c) = sum_{s' < Q} bsum_{s'} + bpre_Q
                        // inclusive scan of the increments; S_0 by a butterfly sum over
                        // the row's 16 lanes of bsum (lanes < Q), bpre (lane Q), 0 (the
                        // rest): every lane ends with S_0, no broadcast round
                        float2 idc = dcf, ids = dsf;
                        const float2 zero2 = make_float2(0.f, 0.f);
                        float2 tc = sg < C::Q ? bcf : (sg == C::Q ? pcf : zero2);
                        float2 ts = sg < C::Q ? bsf : (sg == C::Q ? psf : zero2);
#pragma unroll
                        for (int o = 1; o < C::NSEG; o <<= 1) {
                            const int ox = C::EVEN ? (o < 4 ? o : 2 * o) : o;   // segment bit -> lane bit
                            const float t0 = shup(idc.x, o);
                            const float t1 = shup(idc.y, o);
                            const float t2 = shup(ids.x, o);
                            const float t3 = shup(ids.y, o);
                            const float t4 = __shfl_xor_sync(0xffffffffu, tc.x, ox);
                            const float t5 = __shfl_xor_sync(0xffffffffu, tc.y, ox);
                            const float t6 = __shfl_xor_sync(0xffffffffu, ts.x, ox);
                            const float t7 = __shfl_xor_sync(0xffffffffu, ts.y, ox);
                            if (sg >= o) {
                                idc = __fadd2_rn(idc, make_float2(t0, t1));
                                ids = __fadd2_rn(ids, make_float2(t2, t3));
                            }
                            tc = __fadd2_rn(tc, make_float2(t4, t5));
                            ts = __fadd2_rn(ts, make_float2(t6, t7));
                        }
                        scf = __ffma2_rn(make_float2(wk, wk), tc, __fadd2_rn(idc, make_float2(-dcf.x, -dcf.y)));
                        ssf = __ffma2_rn(make_float2(wk, wk), ts, __fadd2_rn(ids, make_float2(-dsf.x, -dsf.y)));
                    } else {
                    // start window S_s = sum_{i<Q} bsum_{s+i} + bpre_{s+Q}: Q independent
                    // shuffles (one round of latency, not Q chained ones)
                    float2 xcf, xsf;
                    if constexpr (C::Q == 0) {
                        xcf = pcf;
                        xsf = psf;
                    } else {
                        xcf = bcf;
                        xsf = bsf;
#pragma unroll
                        for (int i = 1; i < C::Q; ++i) {
                            xcf.x += shdn(bcf.x, i);
                            xcf.y += shdn(bcf.y, i);
                            xsf.x += shdn(bsf.x, i);
                            xsf.y += shdn(bsf.y, i);
                        }
                        xcf.x += shdn(pcf.x, C::Q);
                        xcf.y += shdn(pcf.y, C::Q);
                        xsf.x += shdn(psf.x, C::Q);
                        xsf.y += shdn(psf.y, C::Q);
                    }
                    scf = __fmul2_rn(make_float2(wk, wk), xcf);
                    ssf = __fmul2_rn(make_float2(wk, wk), xsf);
                    // the last Q segments of a row (their windows pass the strip's
                    // out-columns): w S_s = w S_{s0} + sum_{s0 <= s' < s} dacc_{s'},
                    // s0 = NSEG - 1 - Q, the increments by Q independent shuffles
                    if constexpr (C::Q > 0 && !SF_V7_CHAIN2) {
                        constexpr int s0 = C::NSEG - 1 - C::Q;
                        float2 ac = make_float2(0.f, 0.f), as = ac;
#pragma unroll
                        for (int i = 1; i <= C::Q; ++i) {
                            const float t0 = shup(dcf.x, i);
                            const float t1 = shup(dcf.y, i);
                            const float t2 = shup(dsf.x, i);
                            const float t3 = shup(dsf.y, i);
                            if (sg - s0 >= i) {
                                ac = __fadd2_rn(ac, make_float2(t0, t1));
                                as = __fadd2_rn(as, make_float2(t2, t3));
                            }
                        }
                        const int src = C::EVEN ? (int)(pk >> (10 * C::Q)) : seg_lane(s0);
                        const float2 bc = make_float2(__shfl_sync(0xffffffffu, scf.x, src), __shfl_sync(0xffffffffu, scf.y, src));
                        const float2 bs = make_float2(__shfl_sync(0xffffffffu, ssf.x, src), __shfl_sync(0xffffffffu, ssf.y, src));
                        if (sg > s0) {
                            scf = __fadd2_rn(bc, ac);
                            ssf = __fadd2_rn(bs, as);
                        }
                    }
                    // SF_V7_CHAIN2 (A/B): lane s' contributes Y_{s'} = dacc_{s'} (+ w S_{s0}
                    // in lane s0), lane s sums Y over s0 <= s - i, i = 1..Q, by Q
                    // independent shuffles (no broadcast round)
                    if constexpr (C::Q > 0 && SF_V7_CHAIN2) {
                        constexpr int s0 = C::NSEG - 1 - C::Q;
                        const float2 yc = sg == s0 ? __fadd2_rn(scf, dcf) : dcf;
                        const float2 ys = sg == s0 ? __fadd2_rn(ssf, dsf) : dsf;
                        float2 ac = make_float2(0.f, 0.f), as = ac;
#pragma unroll
                        for (int i = 1; i <= C::Q; ++i) {
                            const float t0 = shup(yc.x, i);
                            const float t1 = shup(yc.y, i);
                            const float t2 = shup(ys.x, i);
                            const float t3 = shup(ys.y, i);
                            if (sg - s0 >= i) {
                                ac = __fadd2_rn(ac, make_float2(t0, t1));
                                as = __fadd2_rn(as, make_float2(t2, t3));
                            }
                        }
                        if (sg > s0) {
                            scf = ac;
                            ssf = as;
                        }
                    }
                    }
                    // pass 2 (w_k S_s) and the rotation of the centre values to pair n+1
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        const float zc = (j & 1) ? Zc[j / 2].y : Zc[j / 2].x;
                        const float zs = (j & 1) ? Zs[j / 2].y : Zs[j / 2].x;
                        QP[j] = __ffma2_rn(make_float2(zc, zc), scf, QP[j]);
                        QP[j] = __ffma2_rn(make_float2(zs, zs), ssf, QP[j]);
                    }
#pragma unroll
                    for (int h = 0; h < J2; ++h) {               // (zc + j zs)(uc + j us), planar
                        const float2 t = __fmul2_rn(Zc[h], Us[h]);
                        Zc[h] = __ffma2_rn(make_float2(-Zs[h].x, -Zs[h].y), Us[h], __fmul2_rn(Zc[h], Uc[h]));
                        Zs[h] = __ffma2_rn(Zs[h], Uc[h], t);
                    }
                }
                if constexpr (PS) {
                    // every CTA of the cluster is past its slab traffic after the
                    // first barrier: ranks >= 1 store their (Q, P') into rank 0's
                    // slab memory (DSMEM), rank 0 adds them after the second
                    float2* stage = reinterpret_cast<float2*>(vbuf) + hry * C::TW + xs;
                    cluster_arrive_wait();
                    if (prank > 0) {
                        float2* dst = cluster_map_rank0(stage) + (size_t)(prank - 1) * RB * C::TW;
#pragma unroll
                        for (int j = 0; j < G; ++j) dst[j] = QP[j];
                    }
                    cluster_arrive_wait();
                    if (prank > 0) break;
                    for (int r = 1; r < ps; ++r) {
#pragma unroll
                        for (int j = 0; j < G; ++j) {
                            const float2 t = stage[(size_t)(r - 1) * RB * C::TW + j];
                            QP[j] = __fadd2_rn(QP[j], t);
                        }
                    }
                }
                const bool rowok = gy < yend;
                const size_t rowoff = (size_t)(gy - p.out_row0) * p.W;
                const float dc = v5_dc(p, x0, yb0, C::TW);
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const float qj = QP[j].x, pj = QP[j].y;
                    const int gxo = x0 + xs + j;
                    if (rowok && gxo < p.W) {
                        if (p.out) {
                            p.out[rowoff + gxo] = (qj > 0.f && isfinite(qj)) ? kCenter - dc + __fdividef(pj, qj)
                                                                             : kCenter + ldf(p, gy, gxo);
                        } else {
                            p.num[rowoff + gxo] = fmaf(-dc, qj, pj);   // centred at 128 (ABI)
                            p.den[rowoff + gxo] = qj;
                        }
                    }
                }
            }
        }   // segments
    }
}

// maxseg: RB-row batches per running-sum segment (<= 0: unlimited)
template <int R, bool OM, int NB = SF_V7_NB_DEFAULT, int SREG = SF_V7_SREG>
inline cudaError_t launch_box_v7(const Params& p, const PairTable& t, double gamma, int maxseg, cudaStream_t s) {
    using C = V7Cfg<R, NB, SREG>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    if constexpr (SREG > 0) {   // setmaxnreg needs the kernel compiled to exactly 128 registers
        static const bool regs_ok = [] {
            cudaFuncAttributes a{}, b{};
            return cudaFuncGetAttributes(&a, bilateral_box_v7<R, OM, NB, SREG, false>) == cudaSuccess &&
                   a.numRegs == 128 &&
                   (!OM || (cudaFuncGetAttributes(&b, bilateral_box_v7<R, OM, NB, SREG, OM>) == cudaSuccess &&
                            b.numRegs == 128));
        }();
        if (!regs_ok) return cudaErrorLaunchOutOfResources;
    }
    const int strips = (p.W + C::TW - 1) / C::TW;
    V5Extra ex;
    ex.diag = 0;
    ex.bps = (p.out_rows + C::RB - 1) / C::RB;
    ex.total = strips * ex.bps;
    ex.maxseg = maxseg > 0 ? maxseg : ex.bps;
    ex.two_gamma = (float)(2.0 * gamma);
    // pair split (OM kernels) for images of fewer units than SMs: ps CTAs (a
    // cluster) per unit, each over npairs / ps pairs (>= 5), partials reduced
    // over DSMEM in the slab memory (ps - 1 staging tiles of RB x TW float2)
    int ps = 1;
    if constexpr (OM) {
        while (ps < 4 && ex.total * (ps + 1) <= di.sms && t.npairs >= 5 * (ps + 1) &&
               (size_t)ps * C::RB * C::TW * 8 <= (size_t)C::SMEM)
            ++ps;
        static const int ps_env = [] {                // SF_V7_PS: tools override (1 = off)
            const char* v = getenv("SF_V7_PS");
            return v ? atoi(v) : 0;
        }();
        if (ps_env > 0 && ps_env <= 4 && t.npairs >= ps_env) ps = ps_env;
    }
    ex.psplit = ps;
    const int grid = ps > 1 ? ex.total * ps : (ex.total < di.sms ? ex.total : di.sms);
    const size_t scratch_bytes = (size_t)grid * (t.npairs > 0 ? t.npairs : 1) * C::NCOLP * 16;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    if (ps > 1) {
        if constexpr (OM) {
            e = cudaFuncSetAttribute(bilateral_box_v7<R, OM, NB, SREG, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
            if (e == cudaSuccess) {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(C::NT);
                cfg.dynamicSmemBytes = C::SMEM;
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = ps;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                e = cudaLaunchKernelEx(&cfg, bilateral_box_v7<R, OM, NB, SREG, true>, p, t, ex);
            }
            if (e == cudaSuccess) e = cudaGetLastError();
            if (e != cudaSuccess) {   // no room for the cluster (e.g. a partitioned GPU): unsplit
                cudaGetLastError();
                ps = 1;
            }
        }
    }
    if (ps == 1) {
        ex.psplit = 1;
        const int g1 = ex.total < di.sms ? ex.total : di.sms;   // <= grid: the scratch fits
        e = cudaFuncSetAttribute(bilateral_box_v7<R, OM, NB, SREG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM);
        if (e == cudaSuccess) {
            bilateral_box_v7<R, OM, NB, SREG, false><<<g1, C::NT, C::SMEM, s>>>(p, t, ex);
            e = cudaGetLastError();
        }
    }
    scratch_free(ex.scratch, s);
    return e;
}

// the wide large-radius kernel (r = 25..64; outgoing rows by MUFU, no pair
// split): one CTA per SM on the balanced schedule
template <int R>
inline cudaError_t launch_box_v7w(const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    using C = V7Cfg<R, SF_V7_NB_DEFAULT, 8, true>;
    auto kern = bilateral_box_v7<R, true, SF_V7_NB_DEFAULT, 8, false, SF_V7_MB_DEFAULT, true>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    static const bool regs_ok = [&] {   // setmaxnreg needs the kernel compiled to exactly CREGS registers
        cudaFuncAttributes a{};
        return cudaFuncGetAttributes(&a, kern) == cudaSuccess && a.numRegs == C::CREGS;
    }();
    if (!regs_ok) return cudaErrorLaunchOutOfResources;
    const int strips = (p.W + C::TW - 1) / C::TW;
    V5Extra ex;
    ex.diag = 0;
    ex.bps = (p.out_rows + C::RB - 1) / C::RB;
    ex.total = strips * ex.bps;
    ex.maxseg = ex.bps;
    ex.two_gamma = (float)(2.0 * gamma);
    ex.psplit = 1;
    const int grid = ex.total < di.sms ? ex.total : di.sms;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, (size_t)grid * (t.npairs > 0 ? t.npairs : 1) * C::NCOLP * 16, s);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e == cudaSuccess) {
        kern<<<grid, C::NT, C::SMEM, s>>>(p, t, ex);
        e = cudaGetLastError();
    }
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
