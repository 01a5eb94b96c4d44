// box_v7q.cuh — "v7q": the band-sweep kernel of Algorithm 2
// with a separable shiftable spatial kernel w(dx, dy) = w1(dx) w1(dy),
//     w1(u) = cos(beta u)^M = a_0 + sum_m a_m cos(nu_m u),
// nu_m = s_m beta for the F = ceil(M/2) nonzero frequencies s_m = M - 2k,
// a_m = 2 C(M,k) / 2^M, a_0 = C(M, M/2) / 2^M for even M (0 for odd M);
// beta = pi/(2(r+1)) (q_M with T = r+1) or the
// sigma_s fit of Eq. (7) (reading R18).  F = 1 serves
// M = 1, 2 (q_2 = config 3), F = 2 serves M = 3, 4.  Compile-time radius
// R = 1..24 (v7q_part.cu).
//
// Same CTA organisation as v7 (box_v7.cuh): one CTA per SM on the balanced
// schedule, 8 producer warps (vertical pass, one input column per lane) and
// 8 consumer warps (horizontal pass and recombination, a lane owns G
// consecutive outputs of one row), the double-buffered 16-row slab, the
// per-segment centre c (reading R16).  The spatial weight is applied per axis
// with the shiftability of w1 itself (Eq. (1) for the spatial kernel,
// PAPER.md:47-54, 134, 151): a window sum weighted by w1 centred at t is
//     sum_u w1(u - t) g(u) = a_0 A_0(t) + sum_m a_m Re[e^{-j nu_m (t - o)} A_m(t)],
//     A_m(t) = sum_{u in window(t)} e^{j nu_m (u - o)} g(u),
// for any origin o, with plain moving sums of the modulated images.
//
//  * producers: per column and pair the running sums A_0 and A_m (complex)
//    of the 4 stack images, origin = the current batch start yb (re-based by
//    e^{-j nu_m RB} from batch to batch), so every modulation factor is
//    indexed by the row offset inside the batch: a compile-time index into
//    the kernel's parameter table (uniform operands).  The sums are kept
//    pre-scaled by their weights a_0, a_m.  The slab holds the vertically
//    w1-weighted sum Vw in the channel order (C, S, (f-c)C, (f-c)S): the
//    halves (C, S) come as a pair from the MUFU sincos and ((f-c)C, (f-c)S)
//    from one FMUL2, so no register moves build the f32x2 operands.
//  * consumers: per lane the modulated running sums of Vw with the origin at
//    the lane's first slab column.  Pass 1: the window increments
//    D_m(j) (in column j+L, out column j) and the block sums B_m of the
//    "out" columns; Q, P' take z_j . demod_j(D(j)).  Start windows from the
//    block sums: X_s = B_s + e^{j nu G} X_{s+1} over Q shuffle rounds (X =
//    the first PP block terms to start), the last Q segments by the chain
//    S_s = e^{-j nu G} (S_{s-1} + D_{s-1}(G)).  Pass 2: z_j . demod_j(S).
//    The pair weight w_k is folded into the centre values
//    z_j = w_k (cos, sin)(w_k d_j) (MUFU, recomputed in each pass); Q and P'
//    accumulate per channel pair, (zc C, zs S) and (zc FC, zs FS), summed
//    at the end.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"
#include "box_v5.cuh"
#include "box_v7.cuh"
#include "runtime.h"
#include "v7q_dispatch.h"

namespace sf {

// outputs per consumer lane: F = 1 as v7; F = 2 (20 running values per lane) at most 9
template <int R, int F>
struct V7QG {
    static constexpr int v = V7G<R>::value;
    static constexpr int value = (F == 1 || v <= 9) ? v : 9;
};

#ifndef PREGF2
#define PREGF2 128
#endif
template <int R, int F>
struct V7QCfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = kQRB;
    static constexpr int NSEG = 16;
    static constexpr int G = V7QG<R, F>::value;
    static constexpr int TW = NSEG * G;
    static constexpr int TWI = TW + 2 * R;
    static constexpr int NV = 8, NH = 8;
    static constexpr int NT = 32 * (NV + NH);
    static constexpr int NCOLP = 32 * NV;
    static constexpr int NBUF = 2;
    static constexpr int SMEM = NBUF * RB * NCOLP * 16;
    // setmaxnreg per role (2 producer + 2 consumer warps per SMSP: a balanced
    // move); F = 1: the consumers hold (Q, P') split by channel (4 G), F = 2:
    // the producers hold 2 x 20 running-sum values (state + prefetch)
    static constexpr int PREG = F == 1 ? 104 : PREGF2, CREG = 256 - PREG;
    static constexpr int NSF = 1 + 2 * F;           // float4 state per column and pair
    static constexpr int Q = L / G, PP = L % G;
    static constexpr int NCH = (L + RB - 1) / RB;
    static constexpr int CH = (L + NCH - 1) / NCH;
    static constexpr int kSeed = 8;
    static_assert(G % 2 == 1 && G <= kQMaxG && TWI <= NCOLP, "odd G, strip within the producer lanes");
    static_assert(Q < NSEG && R <= kQMaxR && F >= 1 && F <= kQFMax, "v7q shape");
};

__device__ __forceinline__ float2 q_bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 q_lo(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 q_hi(const float4& v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float4 q_cat(const float2& a, const float2& b) { return make_float4(a.x, a.y, b.x, b.y); }
__device__ __forceinline__ float2 q_sub(const float2& a, const float2& b) {
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
}

__device__ __forceinline__ void q_sts128_if(bool pred, uint32_t addr, float2 a, float2 b) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t@p st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n\t}\n" ::"r"(addr),
                 "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "r"((int)pred)
                 : "memory");
}

template <int R, int F>
__global__ void __launch_bounds__(V7QCfg<R, F>::NT, 1)
bilateral_box_v7q(const Params p, const PairTable tab, const QModTab qt, const V5Extra ex) {
    using C = V7QCfg<R, F>;
    constexpr int L = C::L, G = C::G, RB = C::RB, NCOLP = C::NCOLP, NSF = C::NSF;
    constexpr int TWI = C::TWI, NT = C::NT, CH = C::CH;
    extern __shared__ float4 vbuf[];                     // [NBUF][RB][NCOLP]

    const int tid = threadIdx.x;
    const int npairs = tab.npairs;
    const int q = ex.total / gridDim.x, rem = ex.total % gridDim.x, bid = blockIdx.x;
    const int u_begin = bid * q + min(bid, rem);
    const int u_end = u_begin + q + (bid < rem ? 1 : 0);
    const int nsteps = (u_end - u_begin) * npairs;
    const int warp = tid >> 5;

    if (warp < C::NV) {
        // =========================== producers (vertical pass) =================
        if constexpr (C::PREG < 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::PREG));
        if constexpr (C::PREG > 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::PREG));
        const int c = tid;                               // slab slot = input column
        const bool act = c < TWI;
        float4* scr = ex.scratch + (size_t)blockIdx.x * npairs * NSF * NCOLP;
        const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(vbuf + c);
        auto sidx = [&](int k, int s) { return ((size_t)k * NSF + s) * NCOLP + c; };
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, nbatch = sgm.nbatch;
            const int gx = reflect101(x0 - R + min(c, TWI - 1), p.W);
            const float dc = v5_dc(p, x0, yb0, C::TW);   // 128 - c (reading R16)
            auto fc = [&](float x) { return x + dc; };

            // segment top: the modulated window sums of the row above the
            // segment, rows yb0-R-1+i (i < L), origin yb0, CH rows at a time
#pragma unroll
            for (int i0 = 0; i0 < L; i0 += CH) {
                float fv[CH], zc[CH], zs[CH], uc[CH], us[CH];
#pragma unroll
                for (int i = 0; i < CH; ++i) {
                    fv[i] = (i0 + i < L) ? fc(ldf(p, yb0 - R - 1 + i0 + i, gx)) : 0.f;
                    __sincosf(-ex.two_gamma * fv[i], &us[i], &uc[i]);
                }
                for (int n = 0; n < npairs; ++n) {
                    const int k = npairs - 1 - n;
                    const float om = tab.omega[k];
                    float4 E[NSF];
#pragma unroll
                    for (int s = 0; s < NSF; ++s) E[s] = i0 == 0 ? zero4 : scr[sidx(k, s)];
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
                            const float4 g = make_float4(zc[i], zs[i], fv[i] * zc[i], fv[i] * zs[i]);
                            E[0] = f4fma(qt.a0, g, E[0]);
#pragma unroll
                            for (int m = 0; m < F; ++m) {
                                E[1 + 2 * m] = f4fma(qt.ic[m][i0 + i], g, E[1 + 2 * m]);
                                E[2 + 2 * m] = f4fma(qt.is[m][i0 + i], g, E[2 + 2 * m]);
                            }
                        }
                    }
#pragma unroll
                    for (int s = 0; s < NSF; ++s) scr[sidx(k, s)] = E[s];
                }
            }
            // main sweep: rows in f32x2 pairs (2i, 2i+1) for the MUFU arguments
            constexpr int RP = RB / 2;
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                uint32_t fi2[RP], fo2[RP];                  // incoming / outgoing-row values, bf16 pairs
#pragma unroll
                for (int qq = 0; qq < RP; ++qq) {
                    const int i = 2 * qq;
                    fi2[qq] = v5_pack(fc(ldf(p, yb + i + R, gx)), fc(ldf(p, yb + i + 1 + R, gx)));
                    fo2[qq] = v5_pack(fc(ldf(p, yb + i - R - 1, gx)), fc(ldf(p, yb + i - R, gx)));
                }
                float4 En[NSF];
#pragma unroll
                for (int s = 0; s < NSF; ++s) En[s] = npairs > 0 ? scr[sidx(npairs - 1, s)] : zero4;
                for (int n = 0; n < npairs; ++n) {
                    const int k = npairs - 1 - n;            // |w_k| ascending
                    const float om = tab.omega[k];
                    const int slot = step % C::NBUF;
                    float2 E0a = q_lo(En[0]), E0b = q_hi(En[0]);
                    float2 Eca[F], Ecb[F], Esa[F], Esb[F];
#pragma unroll
                    for (int m = 0; m < F; ++m) {
                        Eca[m] = q_lo(En[1 + 2 * m]);
                        Ecb[m] = q_hi(En[1 + 2 * m]);
                        Esa[m] = q_lo(En[2 + 2 * m]);
                        Esb[m] = q_hi(En[2 + 2 * m]);
                    }
                    if (n + 1 < npairs) {                    // prefetch the next pair's state
#pragma unroll
                        for (int s = 0; s < NSF; ++s) En[s] = scr[sidx(k - 1, s)];
                    }
                    if (b > 0) {                             // re-base the origin from yb - RB to yb
#pragma unroll
                        for (int m = 0; m < F; ++m) {
                            const float cr = qt.rbc[m], sr = qt.rbs[m];
                            const float2 ca = Eca[m], cb = Ecb[m];
                            Eca[m] = __ffma2_rn(q_bc(cr), ca, __fmul2_rn(q_bc(sr), Esa[m]));
                            Ecb[m] = __ffma2_rn(q_bc(cr), cb, __fmul2_rn(q_bc(sr), Esb[m]));
                            Esa[m] = __ffma2_rn(q_bc(cr), Esa[m], __fmul2_rn(q_bc(-sr), ca));
                            Esb[m] = __ffma2_rn(q_bc(cr), Esb[m], __fmul2_rn(q_bc(-sr), cb));
                        }
                    }
                    if (step >= C::NBUF) v5_bar_sync(1 + C::NBUF + slot, NT);  // wait: slot consumed
                    const uint32_t dst = sbase + (uint32_t)(slot * RB * NCOLP) * 16u;
#pragma unroll
                    for (int qq = 0; qq < RP; ++qq) {
                        const float2 Fi = make_float2(v5_lo(fi2[qq]), v5_hi(fi2[qq]));
                        const float2 Fo = make_float2(v5_lo(fo2[qq]), v5_hi(fo2[qq]));
                        const float2 ai = __fmul2_rn(q_bc(om), Fi), ao = __fmul2_rn(q_bc(om), Fo);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int i = 2 * qq + h;
                            // slab layout (C, S, (f-c)C, (f-c)S): halves a = (C, S) straight
                            // from the MUFU pair, b = (f-c) a by one FMUL2 (no register moves)
                            float2 pi, po;
                            __sincosf(h ? ai.y : ai.x, &pi.y, &pi.x);
                            __sincosf(h ? ao.y : ao.x, &po.y, &po.x);
                            const float2 qi = __fmul2_rn(pi, q_bc(h ? Fi.y : Fi.x));
                            const float2 qo = __fmul2_rn(po, q_bc(h ? Fo.y : Fo.x));
                            // sums pre-scaled by their weights a_0, a_m (the tables carry them)
                            E0a = __ffma2_rn(q_bc(qt.a0), pi, __ffma2_rn(q_bc(-qt.a0), po, E0a));
                            E0b = __ffma2_rn(q_bc(qt.a0), qi, __ffma2_rn(q_bc(-qt.a0), qo, E0b));
                            float2 Va = E0a, Vb = E0b;
#pragma unroll
                            for (int m = 0; m < F; ++m) {
                                Eca[m] = __ffma2_rn(q_bc(qt.vic[m][i]), pi, __ffma2_rn(q_bc(qt.voc[m][i]), po, Eca[m]));
                                Ecb[m] = __ffma2_rn(q_bc(qt.vic[m][i]), qi, __ffma2_rn(q_bc(qt.voc[m][i]), qo, Ecb[m]));
                                Esa[m] = __ffma2_rn(q_bc(qt.vis[m][i]), pi, __ffma2_rn(q_bc(qt.vos[m][i]), po, Esa[m]));
                                Esb[m] = __ffma2_rn(q_bc(qt.vis[m][i]), qi, __ffma2_rn(q_bc(qt.vos[m][i]), qo, Esb[m]));
                                Va = __ffma2_rn(q_bc(qt.vac[m][i]), Eca[m], __ffma2_rn(q_bc(qt.vas[m][i]), Esa[m], Va));
                                Vb = __ffma2_rn(q_bc(qt.vac[m][i]), Ecb[m], __ffma2_rn(q_bc(qt.vas[m][i]), Esb[m], Vb));
                            }
                            // lanes past TWI: no slab traffic (predicated store, no branch)
                            q_sts128_if(act, dst + (uint32_t)(i * NCOLP) * 16u, Va, Vb);
                        }
                    }
                    v5_bar_arrive(1 + slot, NT);             // slot full
                    scr[sidx(k, 0)] = q_cat(E0a, E0b);
#pragma unroll
                    for (int m = 0; m < F; ++m) {
                        scr[sidx(k, 1 + 2 * m)] = q_cat(Eca[m], Ecb[m]);
                        scr[sidx(k, 2 + 2 * m)] = q_cat(Esa[m], Esb[m]);
                    }
                    ++step;
                }
            }
        }   // segments
        __threadfence();   // the next launch reuses the scratch slot
    } else {
        // =========================== consumers (horizontal pass) ===============
        if constexpr (C::CREG > 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::CREG));
        if constexpr (C::CREG < 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::CREG));
        const int w = tid - 32 * C::NV;                  // 0..255
        const int sg = w & 15, hry = w >> 4;             // segment, row in the batch
        const int xs = sg * G;                           // first output column (strip-relative)
        constexpr int NSS = 1 + 2 * F;                   // sums: DC, then (cos, sin) per frequency
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, yend = sgm.yend, nbatch = sgm.nbatch;
            const float dc = v5_dc(p, x0, yb0, C::TW);
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                const int gy = yb + hry;
                uint32_t dpk[(G + 1) / 2];                   // centre values f - c, bf16 pairs (exact)
                float2 Qv[G], Pv[G];                         // (sum zc.C, sum zs.S), (sum zc.FC, sum zs.FS)
                {
                    const uint8_t* rowp = v7_row(p, gy);
                    const int cx0 = x0 + xs;
                    float d[G + 1];
#pragma unroll
                    for (int j = 0; j < G; ++j)
                        d[j] = (float)__ldg(rowp + (cx0 + j < p.W ? cx0 + j : reflect101(cx0 + j, p.W))) - kCenter + dc;
                    d[G] = 0.f;
#pragma unroll
                    for (int h = 0; h < (G + 1) / 2; ++h) dpk[h] = v5_pack(d[2 * h], d[2 * h + 1]);
#pragma unroll
                    for (int j = 0; j < G; ++j) Qv[j] = Pv[j] = make_float2(0.f, 0.f);
                }
                for (int n = 0; n < npairs; ++n, ++step) {
                    const int k = npairs - 1 - n;
                    const float om = tab.omega[k], wk = tab.weight[k];
                    const int slot = step % C::NBUF;
                    // z_j = w_k (cos, sin)(w_k d_j): the pair weight folded into the
                    // centre values (MUFU, recomputed in each pass: no registers held)
                    auto zj = [&](int j) {
                        const float dj = (j & 1) ? v5_hi(dpk[j / 2]) : v5_lo(dpk[j / 2]);
                        float2 z;
                        __sincosf(om * dj, &z.y, &z.x);
                        return __fmul2_rn(z, q_bc(wk));
                    };
                    v5_bar_sync(1 + slot, NT);                // wait: slot full
                    const float4* vrow = vbuf + (slot * RB + hry) * NCOLP + xs;
                    // running increments D[s] and block sums B[s] (s: DC, cos_m, sin_m),
                    // all pre-scaled by a_0, a_m (tables); halves a = (C, S), b = (FC, FS);
                    // Bp = the first PP block terms
                    float2 Da[NSS], Db[NSS], Ba[NSS], Bb[NSS], Pa[NSS], Pb[NSS];
#pragma unroll
                    for (int s = 0; s < NSS; ++s) Da[s] = Db[s] = Ba[s] = Bb[s] = Pa[s] = Pb[s] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        const float4 vo = vrow[j];
                        const bool last = (j == G - 1);
                        const float4 vi = (!last || sg < C::NSEG - 1) ? vrow[j + L] : make_float4(0.f, 0.f, 0.f, 0.f);
                        if (j == C::PP) {
#pragma unroll
                            for (int s = 0; s < NSS; ++s) {
                                Pa[s] = Ba[s];
                                Pb[s] = Bb[s];
                            }
                        }
                        const float2 voa = q_lo(vo), vob = q_hi(vo), via = q_lo(vi), vib = q_hi(vi);
                        // Q, P' += z_j demod_j(D(j)), D before this column's increment
                        {
                            float2 Ta = Da[0], Tb = Db[0];
#pragma unroll
                            for (int m = 0; m < F; ++m) {
                                Ta = __ffma2_rn(q_bc(qt.hac[m][j]), Da[1 + 2 * m], __ffma2_rn(q_bc(qt.has[m][j]), Da[2 + 2 * m], Ta));
                                Tb = __ffma2_rn(q_bc(qt.hac[m][j]), Db[1 + 2 * m], __ffma2_rn(q_bc(qt.has[m][j]), Db[2 + 2 * m], Tb));
                            }
                            const float2 z = zj(j);
                            Qv[j] = __ffma2_rn(z, Ta, Qv[j]);
                            Pv[j] = __ffma2_rn(z, Tb, Pv[j]);
                        }
                        Ba[0] = __ffma2_rn(q_bc(qt.a0), voa, Ba[0]);
                        Bb[0] = __ffma2_rn(q_bc(qt.a0), vob, Bb[0]);
                        Da[0] = __ffma2_rn(q_bc(qt.a0), via, __ffma2_rn(q_bc(-qt.a0), voa, Da[0]));
                        Db[0] = __ffma2_rn(q_bc(qt.a0), vib, __ffma2_rn(q_bc(-qt.a0), vob, Db[0]));
#pragma unroll
                        for (int m = 0; m < F; ++m) {
                            const float oc = qt.hoc[m][j], os = qt.hos[m][j], ic = qt.hic[m][j], is = qt.his[m][j];
                            Ba[1 + 2 * m] = __ffma2_rn(q_bc(oc), voa, Ba[1 + 2 * m]);
                            Bb[1 + 2 * m] = __ffma2_rn(q_bc(oc), vob, Bb[1 + 2 * m]);
                            Ba[2 + 2 * m] = __ffma2_rn(q_bc(os), voa, Ba[2 + 2 * m]);
                            Bb[2 + 2 * m] = __ffma2_rn(q_bc(os), vob, Bb[2 + 2 * m]);
                            Da[1 + 2 * m] = __ffma2_rn(q_bc(ic), via, __ffma2_rn(q_bc(-oc), voa, Da[1 + 2 * m]));
                            Db[1 + 2 * m] = __ffma2_rn(q_bc(ic), vib, __ffma2_rn(q_bc(-oc), vob, Db[1 + 2 * m]));
                            Da[2 + 2 * m] = __ffma2_rn(q_bc(is), via, __ffma2_rn(q_bc(-os), voa, Da[2 + 2 * m]));
                            Db[2 + 2 * m] = __ffma2_rn(q_bc(is), vib, __ffma2_rn(q_bc(-os), vob, Db[2 + 2 * m]));
                        }
                    }
                    if (step + C::NBUF < nsteps) v5_bar_arrive(1 + C::NBUF + slot, NT);   // slot empty
                    // start windows X_s = B_s + e^{j nu G} X_{s+1}, X = Bp to start (Q rounds)
                    float2 Xa[NSS], Xb[NSS];
#pragma unroll
                    for (int s = 0; s < NSS; ++s) {
                        Xa[s] = Pa[s];
                        Xb[s] = Pb[s];
                    }
                    auto shd = [](float2 v) {
                        return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
                    };
                    auto shu = [](float2 v) {
                        return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
                    };
#pragma unroll
                    for (int i = 0; i < C::Q; ++i) {
                        Xa[0] = __fadd2_rn(Ba[0], shd(Xa[0]));
                        Xb[0] = __fadd2_rn(Bb[0], shd(Xb[0]));
#pragma unroll
                        for (int m = 0; m < F; ++m) {
                            const float rc = qt.rhc[m], rs = qt.rhs[m];
                            const float2 ca = shd(Xa[1 + 2 * m]), cb = shd(Xb[1 + 2 * m]);
                            const float2 sa = shd(Xa[2 + 2 * m]), sb = shd(Xb[2 + 2 * m]);
                            // (c + j s) e^{j nu G}
                            Xa[1 + 2 * m] = __fadd2_rn(Ba[1 + 2 * m], __ffma2_rn(q_bc(rc), ca, __fmul2_rn(q_bc(-rs), sa)));
                            Xb[1 + 2 * m] = __fadd2_rn(Bb[1 + 2 * m], __ffma2_rn(q_bc(rc), cb, __fmul2_rn(q_bc(-rs), sb)));
                            Xa[2 + 2 * m] = __fadd2_rn(Ba[2 + 2 * m], __ffma2_rn(q_bc(rs), ca, __fmul2_rn(q_bc(rc), sa)));
                            Xb[2 + 2 * m] = __fadd2_rn(Bb[2 + 2 * m], __ffma2_rn(q_bc(rs), cb, __fmul2_rn(q_bc(rc), sb)));
                        }
                    }
                    // the last Q segments of a row: S_s = e^{-j nu G} (S_{s-1} + D_{s-1}(G))
#pragma unroll
                    for (int t = 1; t <= C::Q; ++t) {
                        float2 Na[NSS], Nb[NSS];
                        Na[0] = shu(__fadd2_rn(Xa[0], Da[0]));
                        Nb[0] = shu(__fadd2_rn(Xb[0], Db[0]));
#pragma unroll
                        for (int m = 0; m < F; ++m) {
                            const float rc = qt.rhc[m], rs = qt.rhs[m];
                            const float2 ca = __fadd2_rn(Xa[1 + 2 * m], Da[1 + 2 * m]), cb = __fadd2_rn(Xb[1 + 2 * m], Db[1 + 2 * m]);
                            const float2 sa = __fadd2_rn(Xa[2 + 2 * m], Da[2 + 2 * m]), sb = __fadd2_rn(Xb[2 + 2 * m], Db[2 + 2 * m]);
                            // (c + j s) e^{-j nu G}
                            Na[1 + 2 * m] = shu(__ffma2_rn(q_bc(rc), ca, __fmul2_rn(q_bc(rs), sa)));
                            Nb[1 + 2 * m] = shu(__ffma2_rn(q_bc(rc), cb, __fmul2_rn(q_bc(rs), sb)));
                            Na[2 + 2 * m] = shu(__ffma2_rn(q_bc(rc), sa, __fmul2_rn(q_bc(-rs), ca)));
                            Nb[2 + 2 * m] = shu(__ffma2_rn(q_bc(rc), sb, __fmul2_rn(q_bc(-rs), cb)));
                        }
                        if (sg == C::NSEG - 1 - C::Q + t) {
#pragma unroll
                            for (int s = 0; s < NSS; ++s) {
                                Xa[s] = Na[s];
                                Xb[s] = Nb[s];
                            }
                        }
                    }
                    // pass 2: Q, P' += z_j demod_j(S)
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        float2 Ta = Xa[0], Tb = Xb[0];
#pragma unroll
                        for (int m = 0; m < F; ++m) {
                            Ta = __ffma2_rn(q_bc(qt.hac[m][j]), Xa[1 + 2 * m], __ffma2_rn(q_bc(qt.has[m][j]), Xa[2 + 2 * m], Ta));
                            Tb = __ffma2_rn(q_bc(qt.hac[m][j]), Xb[1 + 2 * m], __ffma2_rn(q_bc(qt.has[m][j]), Xb[2 + 2 * m], Tb));
                        }
                        const float2 z = zj(j);
                        Qv[j] = __ffma2_rn(z, Ta, Qv[j]);
                        Pv[j] = __ffma2_rn(z, Tb, Pv[j]);
                    }
                }
                const bool rowok = gy < yend;
                const size_t rowoff = (size_t)(gy - p.out_row0) * p.W;
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const float qj = Qv[j].x + Qv[j].y, pj = Pv[j].x + Pv[j].y;
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

template <int R, int F>
inline cudaError_t launch_box_v7q(const Params& p, const PairTable& t, const QModTab& qt, double gamma,
                                  cudaStream_t s) {
    using C = V7QCfg<R, F>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    static const bool regs_ok = [] {   // setmaxnreg needs the kernel compiled to exactly 128 registers
        cudaFuncAttributes a{};
        return cudaFuncGetAttributes(&a, bilateral_box_v7q<R, F>) == cudaSuccess && a.numRegs == 128;
    }();
    if (!regs_ok) return cudaErrorLaunchOutOfResources;
    cudaError_t e = cudaFuncSetAttribute(bilateral_box_v7q<R, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    const int strips = (p.W + C::TW - 1) / C::TW;
    V5Extra ex{};
    ex.bps = (p.out_rows + C::RB - 1) / C::RB;
    ex.total = strips * ex.bps;
    ex.maxseg = ex.bps;                                // outgoing rows by MUFU: no rotation drift
    ex.two_gamma = (float)(2.0 * gamma);
    ex.psplit = 1;
    const int grid = ex.total < di.sms ? ex.total : di.sms;
    const size_t scratch_bytes = (size_t)grid * (t.npairs > 0 ? t.npairs : 1) * C::NSF * C::NCOLP * 16;
    e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    bilateral_box_v7q<R, F><<<grid, C::NT, C::SMEM, s>>>(p, t, qt, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
