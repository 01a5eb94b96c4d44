// box_v6.cuh — "v6": the band-sweep kernel of Algorithm 2,
// box spatial kernel, compile-time radius R = 1..32 (instantiated in
// v6_part.cu).  Same CTA shape and schedule as v5 (one CTA per
// SM, NV producer warps for the vertical pass, 8 consumer warps for the
// horizontal pass and the recombination, a double-buffered shared-memory slab
// of vertical moving sums between them), with three changes:
//
//  * per-segment centre (reading R16): every segment of the balanced schedule
//    centres its stack images and phases at c = the median of 5 pixels of its
//    first output row (v5_dc), in both roles; partials convert to the ABI's
//    SF_CENTER with one FMA.  On flat backgrounds this keeps the f·cos / f·sin
//    window sums near zero instead of ~(2r+1)^2 · 127.
//
//  * consumer centre values by the Chebyshev recurrence across pairs
//    (Alg. 2 step 3): with the pairs in |w| order w_{n+1} =
//    w_n - 2 gamma, so for t = trig(w_n d + phi)
//        T_{n+1} = 2cos(2 gamma d) T_n - T_{n-1}
//    — one FFMA per output per pair instead of an FFMA, FMUL.RZ and a MUFU.
//    Seeds (T_0, T_{-1}) and 2cos(2 gamma d) come from MUFU once per batch.
//    Error: (m+1)·eps per injected rounding over m steps, weighted by the
//    binomial pair weights that fall off along the sequence; measured as
//    accurate as per-pair MUFU.
//
//  * segment start windows directly from block sums, not from a scan: with
//    Q = L / G, S_s = bsum_s + ... + bsum_{s+Q-1} + bpre_{s+Q} (own block
//    sums of the "out" columns and a prefix of the next block, gathered by
//    shuffles); the last Q segments of a row chain S_s = S_{s-1} + D_{s-1}.
//    4Q shuffles per pair instead of 12, and no long telescoping sum.  The
//    second pass QP_j += T_j w S_s of pair n is folded into pass 1 of pair
//    n+1 (T_n is the recurrence's "previous" value there), so the shuffles'
//    latency hides behind the next pair's work.
//
// Consumer registers: 5 G (T_n, T_{n-1}, 2cos, and (Q, P')) — G = 20..24.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"
#include "box_v5.cuh"
#include "runtime.h"

namespace sf {

template <int R, int GG>
struct V6Cfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16;                   // rows per step
    static constexpr int NSEG = 8;                  // segments per row (lanes of one warp)
    static constexpr int G = GG;                    // outputs per walker
    static constexpr int TW = NSEG * G;
    static constexpr int TWI = TW + 2 * R;
    static constexpr int NH = 8;                    // consumer warps (2 rows each)
    static constexpr int NV = (TWI + 31) / 32;      // producer warps (one column per lane)
    static constexpr int NT = 32 * (NV + NH);
    static constexpr int PAD = ((1 - G) % 8 + 8) % 8;    // (G + PAD) = 1 mod 8: segments on disjoint banks
    static constexpr int TWP = 32 * NV;
    static constexpr int NCOLP = TWP + PAD * (TWP / G) + 1;
    static constexpr int NBUF = 2;
    static constexpr int SMEM = NBUF * RB * NCOLP * 16;
    static constexpr int Q = L / G, PP = L % G;     // 2R+1 = Q G + PP
    static constexpr int CHMAX = RB;
    static constexpr int NCH = (L + CHMAX - 1) / CHMAX;
    static constexpr int CH = (L + NCH - 1) / NCH;
    static constexpr int kSeed = 8;
    static_assert(NV + NH <= 16, "uniform 128-register allocation");
    static_assert(Q < NSEG, "window must fit in the strip");
};

// outputs per consumer walker for radius R: the largest G whose 5 G
// registers fit the uniform 128-register allocation, with the window no
// wider than two segments where possible
template <int R>
struct V6G {
    static constexpr int value = 20;
};

// first byte of image row gy (reflect-101; rows outside the caller's band
// are never needed by a valid window and clamp), as ldf
__device__ __forceinline__ const uint8_t* v6_row(const Params& p, int gy) {
    int ry = reflect101(gy, p.H) - p.img_row0;
    ry = ry < 0 ? 0 : (ry >= p.img_rows ? p.img_rows - 1 : ry);
    return p.img + (size_t)ry * p.W;
}

template <int R, int GG, bool OM>
__global__ void __launch_bounds__(V6Cfg<R, GG>::NT, 1)
bilateral_box_v6(const Params p, const PairTable tab, const V5Extra ex) {
    using C = V6Cfg<R, GG>;
    constexpr int L = C::L, G = C::G, RB = C::RB, PAD = C::PAD, NCOLP = C::NCOLP;
    constexpr int TWI = C::TWI, TWP = C::TWP, NT = C::NT, CH = C::CH;
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
        const int c = tid;
        const int cs = c + PAD * (c / G);
        float4* scr = ex.scratch + (size_t)blockIdx.x * npairs * TWP;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, nbatch = sgm.nbatch;
            const int gx = reflect101(x0 - R + min(c, TWI - 1), p.W);
            const float dc = v5_dc(p, x0, yb0, C::TW);   // 128 - c (reading R16)
            auto fc = [&](float x) { return x + dc; };   // f - c from ldf's f - 128

            // segment top: exact window sums of the row above the segment,
            // rows [yb0-R-1, yb0+R-1], CH rows at a time, rotation across pairs
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
                float4 Vn = npairs > 0 ? scr[(size_t)(npairs - 1) * TWP + c] : zero4;
                auto pair_step = [&](const int n, const bool reseed) {
                    const int k = npairs - 1 - n;            // |w_k| ascending
                    const float om = tab.omega[k];
                    const int slot = step % C::NBUF;
                    float4 V = Vn;
                    if (n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWP + c];   // prefetch next pair
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
                    if (step >= C::NBUF) v5_bar_sync(1 + C::NBUF + slot, NT);  // wait: slot consumed
                    float4* dst = vbuf + slot * RB * NCOLP + cs;
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
                        dst[(2 * q) * NCOLP] = V;
                        V.x += Dc.y;
                        V.y += Dfc.y;
                        V.z += Ds.y;
                        V.w += Dfs.y;
                        dst[(2 * q + 1) * NCOLP] = V;
                    }
                    v5_bar_arrive(1 + slot, NT);             // slot full
                    scr[(size_t)k * TWP + c] = V;
                    ++step;
                };
                for (int n0 = 0; n0 < npairs; n0 += C::kSeed) {
#pragma unroll
                    for (int m = 0; m < C::kSeed; ++m)
                        if (n0 + m < npairs) pair_step(n0 + m, m == 0);
                }
            }
        }   // segments
        __threadfence();   // the next launch reuses the scratch slot
    } else {
        // =========================== consumers (horizontal pass) ===============
        const int w = tid - 32 * C::NV;                  // 0..255
        const int hh = w & 1, sg = (w >> 1) & 7, hry = w >> 4;
        const float hoff = hh ? 0.0f : 1.57079632679489662f;   // cos half: sin(x + pi/2)
        const int xs = sg * G;                           // first output column (strip-relative)
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, yend = sgm.yend, nbatch = sgm.nbatch;
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                const int gy = yb + hry;
                float Ta[G], Tb[G], c2[G];
                float2 QP[G];
                {
                    // seeds: T_0 = trig(w_{k0} d), T_{-1} = trig((w_{k0} + 2 gamma) d)
                    const float dc = v5_dc(p, x0, yb0, C::TW);
                    const float om0 = npairs > 0 ? tab.omega[npairs - 1] : 0.f;
                    const float om1 = om0 + ex.two_gamma;
                    const uint8_t* rowp = v6_row(p, gy);
                    const int cx0 = x0 + xs;
                    // uint8 -> float by the exponent trick (FMA pipe, no I2F):
                    // bits 0x4B000000 | b are the float 2^23 + b
                    const float bias = 8388608.0f + kCenter - dc;
                    float d[G];
                    if (cx0 + G <= p.W) {
#pragma unroll
                        for (int j = 0; j < G; ++j) d[j] = __uint_as_float(0x4B000000u | __ldg(rowp + cx0 + j)) - bias;
                    } else {
#pragma unroll
                        for (int j = 0; j < G; ++j)
                            d[j] = __uint_as_float(0x4B000000u | __ldg(rowp + reflect101(cx0 + j, p.W))) - bias;
                    }
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        c2[j] = 2.0f * __cosf(ex.two_gamma * d[j]);
                        Ta[j] = __sinf(fmaf(om0, d[j], hoff));
                        Tb[j] = __sinf(fmaf(om1, d[j], hoff));
                        QP[j] = make_float2(0.f, 0.f);
                    }
                }
                float2 wSs = make_float2(0.f, 0.f);          // w_{n-1} S_s of the previous pair
                auto pair_step = [&](const int n, float (&Tc)[G], float (&Tp)[G]) {
                    const int k = npairs - 1 - n;
                    const float wk = tab.weight[k];
                    const int slot = step % C::NBUF;
                    v5_bar_sync(1 + slot, NT);                // wait: slot full
                    const float2* vo_row =
                        reinterpret_cast<const float2*>(vbuf + (slot * RB + hry) * NCOLP) + hh + 2 * (xs + PAD * sg);
                    float2 dacc = make_float2(0.f, 0.f), bsum = make_float2(0.f, 0.f), bpre = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        const float2 vo = vo_row[2 * j];
                        const int ioff = (j + L) + PAD * ((j + L) / G);
                        const bool last = (j == G - 1);
                        const float2 vi = (!last || sg < C::NSEG - 1) ? vo_row[2 * ioff] : make_float2(0.f, 0.f);
                        if (j == C::PP) bpre = bsum;
                        bsum = __fadd2_rn(bsum, vo);
                        QP[j] = __ffma2_rn(make_float2(Tp[j], Tp[j]), wSs, QP[j]);   // pass 2 of pair n-1
                        QP[j] = __ffma2_rn(make_float2(Tc[j], Tc[j]), dacc, QP[j]);  // pass 1 of pair n
                        dacc = __ffma2_rn(make_float2(wk, wk), __fadd2_rn(vi, make_float2(-vo.x, -vo.y)), dacc);
                        Tp[j] = fmaf(c2[j], Tc[j], -Tp[j]);                           // T_{n+1}
                    }
                    if (step + C::NBUF < nsteps) v5_bar_arrive(1 + C::NBUF + slot, NT);   // slot empty
                    // start window of this segment: S_s = sum_{i<Q} bsum_{s+i} + bpre_{s+Q}
                    float2 S = C::Q == 0 ? bpre : bsum;
#pragma unroll
                    for (int i = 1; i <= C::Q; ++i) {
                        const float2 v = (i == C::Q) ? bpre : bsum;
                        S.x += __shfl_down_sync(0xffffffffu, v.x, 2 * i);
                        S.y += __shfl_down_sync(0xffffffffu, v.y, 2 * i);
                    }
                    float2 wS = __fmul2_rn(make_float2(wk, wk), S);
                    // the last Q segments of a row (their blocks run past the
                    // strip): w S_s = w S_{s-1} + dacc_{s-1}, dacc = w x the
                    // segment's window increment
#pragma unroll
                    for (int t = 1; t <= C::Q; ++t) {
                        const float2 nx = __fadd2_rn(wS, dacc);
                        const float ux = __shfl_up_sync(0xffffffffu, nx.x, 2);
                        const float uy = __shfl_up_sync(0xffffffffu, nx.y, 2);
                        if (sg == C::NSEG - 1 - C::Q + t) wS = make_float2(ux, uy);
                    }
                    wSs = wS;
                    ++step;
                };
                int n = 0;
                for (; n + 1 < npairs; n += 2) {
                    pair_step(n, Ta, Tb);
                    pair_step(n + 1, Tb, Ta);
                }
                if (n < npairs) {
                    pair_step(n, Ta, Tb);
#pragma unroll
                    for (int j = 0; j < G; ++j) QP[j] = __ffma2_rn(make_float2(Ta[j], Ta[j]), wSs, QP[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < G; ++j) QP[j] = __ffma2_rn(make_float2(Tb[j], Tb[j]), wSs, QP[j]);
                }
                const bool rowok = gy < yend;
                const size_t rowoff = (size_t)(gy - p.out_row0) * p.W;
                const float dc = v5_dc(p, x0, yb0, C::TW);
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const float qj = QP[j].x + __shfl_xor_sync(0xffffffffu, QP[j].x, 1);
                    const float pj = QP[j].y + __shfl_xor_sync(0xffffffffu, QP[j].y, 1);
                    const int gxo = x0 + xs + j;
                    if (rowok && gxo < p.W && (j & 1) == hh) {
                        if (p.out) {
                            const float cc = kCenter - dc;
                            p.out[rowoff + gxo] = (qj > 0.f && isfinite(qj)) ? cc + __fdividef(pj, qj)
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
template <int R, bool OM, int GG = V6G<R>::value>
inline cudaError_t launch_box_v6(const Params& p, const PairTable& t, double gamma, int maxseg, cudaStream_t s) {
    using C = V6Cfg<R, GG>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    const cudaError_t attr =
        cudaFuncSetAttribute(bilateral_box_v6<R, GG, OM>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (attr != cudaSuccess) return attr;
    const int strips = (p.W + C::TW - 1) / C::TW;
    V5Extra ex;
    ex.diag = 0;
    ex.bps = (p.out_rows + C::RB - 1) / C::RB;
    ex.total = strips * ex.bps;
    ex.maxseg = maxseg > 0 ? maxseg : ex.bps;
    ex.two_gamma = (float)(2.0 * gamma);
    const int grid = ex.total < di.sms ? ex.total : di.sms;
    const size_t scratch_bytes = (size_t)grid * (t.npairs > 0 ? t.npairs : 1) * C::TWP * 16;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    bilateral_box_v6<R, GG, OM><<<grid, C::NT, C::SMEM, s>>>(p, t, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
