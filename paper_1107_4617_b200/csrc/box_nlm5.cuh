// box_nlm5.cuh — "v5n": shiftable non-local means (
// PAPER.md:296-330) on the v5 band sweep (box_v5.cuh), compile-time outer
// radius R and patch size P = 1..3 (reading R14).
//
// Each conjugate pair of multi-indices (w_1..w_P) is one step of Algorithm
// 2 with f inside the exponential replaced by the phase field
//     theta(z) = w_1 f(z) + w_2 f(z + (0,1)) + w_3 f(z + (1,0)),
// so the stack images are cos, f cos, sin, f sin of theta and the centre
// factor is e^{-j theta(x)}.  Differences from v5:
//   * the outgoing rows are by MUFU (the multi-indices do not step by a
//     constant frequency, so there is no rotation recurrence across pairs),
//     which also makes the incoming and outgoing values of a row bit-identical
//     (no running-sum drift, unlimited segments);
//   * a producer thread keeps, per row of its column, f (bf16 pairs) and for
//     P >= 2 the right neighbour f(z + (0,1)); the lower neighbour of row i is
//     f of row i + 1, so one extra row per window covers it;
//   * consumer segments are G = 16 outputs (128-column strips: NLM windows
//     are small, and the consumer holds f, f right and f below per output).
// The schedule (one CTA per SM, balanced contiguous (strip, batch) ranges,
// segments), the slab handoff and the consumer's delta/scan walker are v5's.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"
#include "box_v5.cuh"
#include "nlm_kernel.cuh"
#include "runtime.h"

namespace sf {

template <int R>
struct V5NCfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16, NSEG = 8, G = 16;
    static constexpr int TW = NSEG * G;             // 128 output columns per strip
    static constexpr int TWI = TW + 2 * R;
    static constexpr int NV = (TWI + 31) / 32, NH = 8;
    static_assert(NV + NH <= 16, "uniform >= 128 registers");
    static constexpr int NT = 32 * (NV + NH);
    static constexpr int PAD = ((1 - G) % 8 + 8) % 8;
    static constexpr int TWP = 32 * NV;
    static constexpr int NCOLP = TWP + PAD * (TWP / G) + 1;
    static constexpr int NBUF = 2;
    static constexpr int SMEM = NBUF * RB * NCOLP * 16;
    static constexpr int Q = L / G, PP = L % G;
    static constexpr int CH = 8;                    // band-top init rows per chunk
    static_assert(Q < NSEG, "window must fit in the strip");
};

template <int R, int P>
__global__ void __launch_bounds__(V5NCfg<R>::NT, 1)
nlm_box_v5n(const Params p, const NlmTable tab, const V5Extra ex) {
    using C = V5NCfg<R>;
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
        const int c = tid;                               // lanes past TWI compute padding
        const int cs = c + PAD * (c / G);
        float4* scr = ex.scratch + (size_t)blockIdx.x * npairs * TWP;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int yb0 = sgm.yb0, nbatch = sgm.nbatch;
            const int gx = reflect101(sgm.x0 - R + min(c, TWI - 1), p.W);
            const int gxr = reflect101(sgm.x0 - R + min(c, TWI - 1) + 1, p.W);   // u_2 = (0, 1)

            // band top: exact window sums over rows [yb0-R-1, yb0+R-1]
            for (int i0 = 0; i0 < L; i0 += CH) {
                float fa[CH + 1], fb[CH];
#pragma unroll
                for (int i = 0; i <= CH; ++i) fa[i] = ldf(p, yb0 - R - 1 + i0 + i, gx);
#pragma unroll
                for (int i = 0; i < CH; ++i) fb[i] = P >= 2 ? ldf(p, yb0 - R - 1 + i0 + i, gxr) : 0.f;
                float4 Vn = (i0 == 0 || npairs == 0) ? zero4 : scr[(size_t)(npairs - 1) * TWP + c];
                for (int n = 0; n < npairs; ++n) {
                    const int k = npairs - 1 - n;
                    const float o0 = tab.om[0][k], o1 = tab.om[1][k], o2 = tab.om[2][k];
                    float4 V = Vn;
                    if (i0 > 0 && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWP + c];
#pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        float th = o0 * fa[i];
                        if (P >= 2) th = fmaf(o1, fb[i], th);
                        if (P >= 3) th = fmaf(o2, fa[i + 1], th);
                        float zs, zc;
                        __sincosf(th, &zs, &zc);
                        if (i0 + i < L) {
                            V.x += zc;
                            V.y = fmaf(fa[i], zc, V.y);
                            V.z += zs;
                            V.w = fmaf(fa[i], zs, V.w);
                        }
                    }
                    scr[(size_t)k * TWP + c] = V;
                }
            }
            constexpr int RP = RB / 2;
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                // rows 2q, 2q+1 of the incoming (yb+R+i) and outgoing (yb-R-1+i)
                // windows: f, f right, and f of the row below (= f of row i+1)
                uint32_t ai2[RP], ao2[RP], bi2[RP], bo2[RP];
                float ai16, ao16;                            // f of row 16 (below row 15)
#pragma unroll
                for (int qq = 0; qq < RP; ++qq) {
                    const int i = 2 * qq;
                    ai2[qq] = v5_pack(ldf(p, yb + i + R, gx), ldf(p, yb + i + 1 + R, gx));
                    ao2[qq] = v5_pack(ldf(p, yb + i - R - 1, gx), ldf(p, yb + i - R, gx));
                    if (P >= 2) {
                        bi2[qq] = v5_pack(ldf(p, yb + i + R, gxr), ldf(p, yb + i + 1 + R, gxr));
                        bo2[qq] = v5_pack(ldf(p, yb + i - R - 1, gxr), ldf(p, yb + i - R, gxr));
                    }
                }
                ai16 = P >= 3 ? ldf(p, yb + RB + R, gx) : 0.f;
                ao16 = P >= 3 ? ldf(p, yb + RB - R - 1, gx) : 0.f;
                float4 Vn = npairs > 0 ? scr[(size_t)(npairs - 1) * TWP + c] : zero4;
                for (int n = 0; n < npairs; ++n, ++step) {
                    const int k = npairs - 1 - n;
                    const float o0 = tab.om[0][k], o1 = tab.om[1][k], o2 = tab.om[2][k];
                    const int slot = step % C::NBUF;
                    float4 V = Vn;
                    if (n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWP + c];   // prefetch next pair
                    if (step >= C::NBUF) v5_bar_sync(1 + C::NBUF + slot, NT);  // wait: slot consumed
                    float4* dst = vbuf + slot * RB * NCOLP + cs;
#pragma unroll
                    for (int qq = 0; qq < RP; ++qq) {
                        const float2 Fi = make_float2(v5_lo(ai2[qq]), v5_hi(ai2[qq]));
                        const float2 Fo = make_float2(v5_lo(ao2[qq]), v5_hi(ao2[qq]));
                        float2 ti = __fmul2_rn(make_float2(o0, o0), Fi);
                        float2 to = __fmul2_rn(make_float2(o0, o0), Fo);
                        if (P >= 2) {
                            ti = __ffma2_rn(make_float2(o1, o1), make_float2(v5_lo(bi2[qq]), v5_hi(bi2[qq])), ti);
                            to = __ffma2_rn(make_float2(o1, o1), make_float2(v5_lo(bo2[qq]), v5_hi(bo2[qq])), to);
                        }
                        if (P >= 3) {
                            const float di = qq + 1 < RP ? v5_lo(ai2[qq + 1]) : ai16;
                            const float dout = qq + 1 < RP ? v5_lo(ao2[qq + 1]) : ao16;
                            ti = __ffma2_rn(make_float2(o2, o2), make_float2(Fi.y, di), ti);
                            to = __ffma2_rn(make_float2(o2, o2), make_float2(Fo.y, dout), to);
                        }
                        float2 C2, S2, Co, So;
                        __sincosf(ti.x, &S2.x, &C2.x);
                        __sincosf(ti.y, &S2.y, &C2.y);
                        __sincosf(to.x, &So.x, &Co.x);
                        __sincosf(to.y, &So.y, &Co.y);
                        const float2 Dc = __fadd2_rn(C2, make_float2(-Co.x, -Co.y));
                        const float2 Ds = __fadd2_rn(S2, make_float2(-So.x, -So.y));
                        const float2 Dfc = __ffma2_rn(Fi, C2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), Co));
                        const float2 Dfs = __ffma2_rn(Fi, S2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), So));
                        V.x += Dc.x;
                        V.y += Dfc.x;
                        V.z += Ds.x;
                        V.w += Dfs.x;
                        dst[(2 * qq) * NCOLP] = V;
                        V.x += Dc.y;
                        V.y += Dfc.y;
                        V.z += Ds.y;
                        V.w += Dfs.y;
                        dst[(2 * qq + 1) * NCOLP] = V;
                    }
                    v5_bar_arrive(1 + slot, NT);             // slot full
                    scr[(size_t)k * TWP + c] = V;
                }
            }
        }
    } else {
        // =========================== consumers (horizontal pass, v5's walker) ==
        const int w = tid - 32 * C::NV;                  // 0..255
        const int hh = w & 1, sg = (w >> 1) & 7, hry = w >> 4;
        const int lane = w & 31;
        const int rowbase = lane & 16;
        const float hoff = hh ? 0.0f : 1.57079632679489662f;
        const int xs = sg * G;
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, yend = sgm.yend, nbatch = sgm.nbatch;
            for (int b = 0; b < nbatch; ++b) {
                const int gy = yb0 + b * RB + hry;
                float fa[G], fb[G], fd[G];                   // centre patch: f, f right, f below
                float2 QP[G];
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const int gxo = reflect101(x0 + xs + j, p.W);
                    fa[j] = ldf(p, gy, gxo);
                    fb[j] = P >= 2 ? ldf(p, gy, reflect101(x0 + xs + j + 1, p.W)) : 0.f;
                    fd[j] = P >= 3 ? ldf(p, gy + 1, gxo) : 0.f;
                    QP[j] = make_float2(0.f, 0.f);
                }
                for (int n = 0; n < npairs; ++n, ++step) {
                    const int k = npairs - 1 - n;
                    const float o0 = tab.om[0][k], o1 = tab.om[1][k], o2 = tab.om[2][k], wk = tab.weight[k];
                    const int slot = step % C::NBUF;
                    v5_bar_sync(1 + slot, NT);                // wait: slot full
                    const float2* vrow = reinterpret_cast<const float2*>(vbuf + (slot * RB + hry) * NCOLP) + hh;
                    const float2* vo_row = vrow + 2 * (xs + PAD * sg);
                    float T[G];
                    float2 dacc = make_float2(0.f, 0.f), bsum = make_float2(0.f, 0.f),
                           bpre = make_float2(0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        const float2 vo = vo_row[2 * j];
                        const int ioff = (j + L) + PAD * ((j + L) / G);
                        const bool last = (j == G - 1);
                        const float2 vi = (!last || sg < C::NSEG - 1) ? vo_row[2 * ioff] : make_float2(0.f, 0.f);
                        if (j == C::PP) bpre = bsum;
                        bsum = __fadd2_rn(bsum, vo);
                        float th = fmaf(o0, fa[j], hoff);
                        if (P >= 2) th = fmaf(o1, fb[j], th);
                        if (P >= 3) th = fmaf(o2, fd[j], th);
                        T[j] = __sinf(th);
                        QP[j] = __ffma2_rn(make_float2(T[j], T[j]), dacc, QP[j]);
                        dacc = __ffma2_rn(make_float2(wk, wk), __fadd2_rn(vi, make_float2(-vo.x, -vo.y)), dacc);
                    }
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
                    if (step + C::NBUF < nsteps) v5_bar_arrive(1 + C::NBUF + slot, NT);   // slot empty
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
                    if (rowok && gxo < p.W && (j & 1) == hh)
                        p.out[rowoff + gxo] = (qj > 0.f && isfinite(qj)) ? kCenter + pj / qj : kCenter + fa[j];
                }
            }
        }
    }
}

template <int R, int P>
inline cudaError_t launch_nlm_v5n(const Params& p, const NlmTable& t, cudaStream_t s) {
    using C = V5NCfg<R>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    const cudaError_t attr =
        cudaFuncSetAttribute(nlm_box_v5n<R, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (attr != cudaSuccess) return attr;
    const int strips = (p.W + C::TW - 1) / C::TW;
    V5Extra ex{};
    ex.bps = (p.out_rows + C::RB - 1) / C::RB;
    ex.total = strips * ex.bps;
    ex.maxseg = ex.bps;                                  // MUFU in and out: no drift
    ex.two_gamma = 0.f;
    ex.diag = 0;
    const int grid = ex.total < di.sms ? ex.total : di.sms;
    const size_t scratch_bytes = (size_t)grid * (t.npairs > 0 ? t.npairs : 1) * C::TWP * 16;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    nlm_box_v5n<R, P><<<grid, C::NT, C::SMEM, s>>>(p, t, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
