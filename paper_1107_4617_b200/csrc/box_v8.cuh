// box_v8.cuh — "v8": band-sweep kernel of Algorithm 2, box
// spatial kernel, compile-time radius R = 1..24 (v8_part.cu).
// v7's consumer (full-output lanes, LDS.128, rotation centre values, odd G,
// no slab padding, per-segment centre, block-sum start windows) with a
// producer of 4 warps whose lanes own TWO input columns each (c and c + 128):
// one producer warp and two consumer warps per SM sub-partition, and the
// register file split by setmaxnreg as producers 232 / consumers 136.  The
// two columns are independent instruction streams, so the compiler can
// overlap one column's MUFU latency with the other's rotation and running
// sums, and the consumers have registers for loads in flight (v5-v7 were
// latency bound at ~50 % issue with 3.5 warps per sub-partition and no room
// to pipeline).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"
#include "box_v5.cuh"
#include "box_v6.cuh"
#include "box_v7.cuh"
#include "runtime.h"

namespace sf {

template <int R>
struct V8Cfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16;                   // rows per step
    static constexpr int NSEG = 16;                 // segments (lanes) per row
    static constexpr int G = V7G<R>::value;         // outputs per lane (odd, 16 G + 2R <= 256)
    static constexpr int J2 = (G + 1) / 2;          // planar output pairs
    static constexpr int TW = NSEG * G;
    static constexpr int TWI = TW + 2 * R;
    static constexpr int NV = 4, NH = 8;            // producer / consumer warps (1 + 2 per SMSP)
    static constexpr int NPC = 2;                   // input columns per producer lane
    static constexpr int NT = 32 * (NV + NH);
    static constexpr int NCOLP = 32 * NV * NPC;     // slab row stride (float4 slots)
    static constexpr int NBUF = 2;
    static constexpr int SMEM = NBUF * RB * NCOLP * 16;
    static constexpr int Q = L / G, PP = L % G;     // 2R+1 = Q G + PP
    static constexpr int NCH = (L + 7) / 8;          // band-top init chunks (8 rows x 2 columns)
    static constexpr int CH = (L + NCH - 1) / NCH;
    static constexpr int kSeed = 8;                 // producer rotation re-seed interval
    // register split (per SMSP: 1 producer + 2 consumer warps, 512 slots):
    // compiled at KREG = 168; producers grow by 64, consumers shrink by 32 each
    static constexpr int KREG = 168, PREG = 232, CREG = 136;
    static_assert(PREG - KREG == 2 * (KREG - CREG) && KREG * 3 <= 512, "balanced per sub-partition");
    static_assert(G % 2 == 1 && TWI <= NCOLP, "odd G, strip within the producer lanes");
    static_assert(Q <= 3, "window spans at most 4 segments");
};

template <int R, bool OM>
__global__ void __launch_bounds__(V8Cfg<R>::NT, 1)
bilateral_box_v8(const Params p, const PairTable tab, const V5Extra ex) {
    using C = V8Cfg<R>;
    constexpr int L = C::L, G = C::G, J2 = C::J2, RB = C::RB, NCOLP = C::NCOLP;
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
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::PREG));
        constexpr int NPC = C::NPC;
        int col[NPC];                                    // slab slots = input columns
#pragma unroll
        for (int e = 0; e < NPC; ++e) col[e] = tid + 32 * C::NV * e;
        float4* scr = ex.scratch + (size_t)blockIdx.x * npairs * NCOLP;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5Seg sgm = v5_seg(p, ex, C::TW, RB, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, nbatch = sgm.nbatch;
            int gx[NPC];
#pragma unroll
            for (int e = 0; e < NPC; ++e) gx[e] = reflect101(x0 - R + min(col[e], TWI - 1), p.W);
            const float dc = v5_dc(p, x0, yb0, C::TW);   // 128 - c (reading R16)
            auto fc = [&](float x) { return x + dc; };   // f - c from ldf's f - 128

            // segment top: exact window sums of the row above the segment,
            // rows [yb0-R-1, yb0+R-1], CH rows at a time, rotation across pairs
            for (int i0 = 0; i0 < L; i0 += CH) {
                float fv[NPC][CH], zc[NPC][CH], zs[NPC][CH], uc[NPC][CH], us[NPC][CH];
#pragma unroll
                for (int e = 0; e < NPC; ++e)
#pragma unroll
                    for (int i = 0; i < CH; ++i) {
                        fv[e][i] = (i0 + i < L) ? fc(ldf(p, yb0 - R - 1 + i0 + i, gx[e])) : 0.f;
                        __sincosf(-ex.two_gamma * fv[e][i], &us[e][i], &uc[e][i]);
                    }
                float4 Vn[NPC];
#pragma unroll
                for (int e = 0; e < NPC; ++e)
                    Vn[e] = (i0 == 0 || npairs == 0) ? zero4 : scr[(size_t)(npairs - 1) * NCOLP + col[e]];
                for (int n = 0; n < npairs; ++n) {
                    const int k = npairs - 1 - n;
                    const float om = tab.omega[k];
#pragma unroll
                    for (int e = 0; e < NPC; ++e) {
                        float4 V = Vn[e];
                        if (i0 > 0 && n + 1 < npairs) Vn[e] = scr[(size_t)(k - 1) * NCOLP + col[e]];
#pragma unroll
                        for (int i = 0; i < CH; ++i) {
                            if (n % C::kSeed == 0) {
                                __sincosf(om * fv[e][i], &zs[e][i], &zc[e][i]);
                            } else {
                                const float a = zc[e][i], b = zs[e][i];
                                zc[e][i] = fmaf(a, uc[e][i], -b * us[e][i]);
                                zs[e][i] = fmaf(a, us[e][i], b * uc[e][i]);
                            }
                            if (i0 + i < L) {
                                V.x += zc[e][i];
                                V.y = fmaf(fv[e][i], zc[e][i], V.y);
                                V.z += zs[e][i];
                                V.w = fmaf(fv[e][i], zs[e][i], V.w);
                            }
                        }
                        scr[(size_t)k * NCOLP + col[e]] = V;
                    }
                }
            }
            // main sweep: rows in planar f32x2 pairs (2i, 2i+1), as in v5, for
            // both columns of the lane
            constexpr int RP = RB / 2;
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                float2 Zc[NPC][OM ? 1 : RP], Zs[NPC][OM ? 1 : RP], Uc[NPC][OM ? 1 : RP], Us[NPC][OM ? 1 : RP];
                uint32_t fi2[NPC][RP], fo2[NPC][RP];        // incoming / outgoing-row values, bf16 pairs
#pragma unroll
                for (int e = 0; e < NPC; ++e)
#pragma unroll
                    for (int q = 0; q < RP; ++q) {
                        const int i = 2 * q;
                        fi2[e][q] = v5_pack(fc(ldf(p, yb + i + R, gx[e])), fc(ldf(p, yb + i + 1 + R, gx[e])));
                        const float fa = fc(ldf(p, yb + i - R - 1, gx[e]));
                        const float fb = fc(ldf(p, yb + i - R, gx[e]));
                        fo2[e][q] = v5_pack(fa, fb);
                        if constexpr (!OM) {
                            __sincosf(-ex.two_gamma * fa, &Us[e][q].x, &Uc[e][q].x);
                            __sincosf(-ex.two_gamma * fb, &Us[e][q].y, &Uc[e][q].y);
                        }
                    }
                float4 Vn[NPC];
#pragma unroll
                for (int e = 0; e < NPC; ++e) Vn[e] = npairs > 0 ? scr[(size_t)(npairs - 1) * NCOLP + col[e]] : zero4;
                auto pair_step = [&](const int n, const bool reseed) {
                    const int k = npairs - 1 - n;            // |w_k| ascending
                    const float om = tab.omega[k];
                    const int slot = step % C::NBUF;
                    float4 V[NPC];
#pragma unroll
                    for (int e = 0; e < NPC; ++e) {
                        V[e] = Vn[e];
                        if (n + 1 < npairs) Vn[e] = scr[(size_t)(k - 1) * NCOLP + col[e]];   // prefetch next pair
                    }
                    if constexpr (!OM) {
#pragma unroll
                        for (int e = 0; e < NPC; ++e) {
                            if (reseed) {
#pragma unroll
                                for (int q = 0; q < RP; ++q) {
                                    __sincosf(om * v5_lo(fo2[e][q]), &Zs[e][q].x, &Zc[e][q].x);
                                    __sincosf(om * v5_hi(fo2[e][q]), &Zs[e][q].y, &Zc[e][q].y);
                                }
                            } else {
#pragma unroll
                                for (int q = 0; q < RP; ++q) {     // (zc + j zs)(uc + j us), planar
                                    const float2 t = __fmul2_rn(Zc[e][q], Us[e][q]);
                                    Zc[e][q] = __ffma2_rn(make_float2(-Zs[e][q].x, -Zs[e][q].y), Us[e][q],
                                                          __fmul2_rn(Zc[e][q], Uc[e][q]));
                                    Zs[e][q] = __ffma2_rn(Zs[e][q], Uc[e][q], t);
                                }
                            }
                        }
                    }
                    if (step >= C::NBUF) v5_bar_sync(1 + C::NBUF + slot, NT);  // wait: slot consumed
                    float4* dst = vbuf + slot * RB * NCOLP;
#pragma unroll
                    for (int q = 0; q < RP; ++q)
#pragma unroll
                        for (int e = 0; e < NPC; ++e) {
                            const float2 Fi = make_float2(v5_lo(fi2[e][q]), v5_hi(fi2[e][q]));
                            const float2 Fo = make_float2(v5_lo(fo2[e][q]), v5_hi(fo2[e][q]));
                            const float2 arg = __fmul2_rn(make_float2(om, om), Fi);
                            float2 C2, S2, Co, So;
                            __sincosf(arg.x, &S2.x, &C2.x);
                            __sincosf(arg.y, &S2.y, &C2.y);
                            if constexpr (OM) {
                                const float2 ao = __fmul2_rn(make_float2(om, om), Fo);
                                __sincosf(ao.x, &So.x, &Co.x);
                                __sincosf(ao.y, &So.y, &Co.y);
                            } else {
                                Co = Zc[e][q];
                                So = Zs[e][q];
                            }
                            const float2 Dc = __fadd2_rn(C2, make_float2(-Co.x, -Co.y));
                            const float2 Ds = __fadd2_rn(S2, make_float2(-So.x, -So.y));
                            const float2 Dfc = __ffma2_rn(Fi, C2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), Co));
                            const float2 Dfs = __ffma2_rn(Fi, S2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), So));
                            V[e].x += Dc.x;
                            V[e].y += Dfc.x;
                            V[e].z += Ds.x;
                            V[e].w += Dfs.x;
                            dst[(2 * q) * NCOLP + col[e]] = V[e];
                            V[e].x += Dc.y;
                            V[e].y += Dfc.y;
                            V[e].z += Ds.y;
                            V[e].w += Dfs.y;
                            dst[(2 * q + 1) * NCOLP + col[e]] = V[e];
                        }
                    v5_bar_arrive(1 + slot, NT);             // slot full
#pragma unroll
                    for (int e = 0; e < NPC; ++e) scr[(size_t)k * NCOLP + col[e]] = V[e];
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
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::CREG));
        const int w = tid - 32 * C::NV;                  // 0..255
        const int sg = w & 15, hry = w >> 4;             // segment, row in the batch
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
                    const float om0 = npairs > 0 ? tab.omega[npairs - 1] : 0.f;
                    const uint8_t* rowp = v6_row(p, gy);
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
                    const float wk = tab.weight[k];
                    const int slot = step % C::NBUF;
                    v5_bar_sync(1 + slot, NT);                // wait: slot full
                    const float4* vrow = vbuf + (slot * RB + hry) * NCOLP + xs;
                    // pass 1: window increments D_j = V(x_j + L) - V(x_j) (w-weighted,
                    // running), block sums of the "out" columns
                    float2 dcf = make_float2(0.f, 0.f), dsf = dcf;
                    float2 bcf = dcf, bsf = dcf, pcf = dcf, psf = dcf;
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        const float4 vo = vrow[j];
                        const bool last = (j == G - 1);
                        const float4 vi = (!last || sg < C::NSEG - 1) ? vrow[j + L] : make_float4(0.f, 0.f, 0.f, 0.f);
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
                    if (step + C::NBUF < nsteps) v5_bar_arrive(1 + C::NBUF + slot, NT);   // slot empty
                    // start window S_s = sum_{i<Q} bsum_{s+i} + bpre_{s+Q}
                    float2 xcf = pcf, xsf = psf;
#pragma unroll
                    for (int i = 0; i < C::Q; ++i) {
                        xcf.x = bcf.x + __shfl_down_sync(0xffffffffu, xcf.x, 1);
                        xcf.y = bcf.y + __shfl_down_sync(0xffffffffu, xcf.y, 1);
                        xsf.x = bsf.x + __shfl_down_sync(0xffffffffu, xsf.x, 1);
                        xsf.y = bsf.y + __shfl_down_sync(0xffffffffu, xsf.y, 1);
                    }
                    float2 scf = __fmul2_rn(make_float2(wk, wk), xcf), ssf = __fmul2_rn(make_float2(wk, wk), xsf);
                    // the last Q segments of a row: w S_s = w S_{s-1} + dacc_{s-1}
#pragma unroll
                    for (int t = 1; t <= C::Q; ++t) {
                        const float2 ncf = __fadd2_rn(scf, dcf), nsf = __fadd2_rn(ssf, dsf);
                        const float a0 = __shfl_up_sync(0xffffffffu, ncf.x, 1);
                        const float a1 = __shfl_up_sync(0xffffffffu, ncf.y, 1);
                        const float a2 = __shfl_up_sync(0xffffffffu, nsf.x, 1);
                        const float a3 = __shfl_up_sync(0xffffffffu, nsf.y, 1);
                        if (sg == C::NSEG - 1 - C::Q + t) {
                            scf = make_float2(a0, a1);
                            ssf = make_float2(a2, a3);
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

// maxseg: RB-row batches per running-sum segment (<= 0: unlimited).  The
// register split assumes the kernel was compiled to exactly KREG registers
// (checked once: a mismatch would deadlock setmaxnreg, so it refuses).
template <int R, bool OM>
inline cudaError_t launch_box_v8(const Params& p, const PairTable& t, double gamma, int maxseg, cudaStream_t s) {
    using C = V8Cfg<R>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    static const bool regs_ok = [] {
        cudaFuncAttributes a{};
        return cudaFuncGetAttributes(&a, bilateral_box_v8<R, OM>) == cudaSuccess && a.numRegs == C::KREG;
    }();
    if (!regs_ok) return cudaErrorLaunchOutOfResources;
    const cudaError_t attr =
        cudaFuncSetAttribute(bilateral_box_v8<R, OM>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (attr != cudaSuccess) return attr;
    const int strips = (p.W + C::TW - 1) / C::TW;
    V5Extra ex;
    ex.diag = 0;
    ex.bps = (p.out_rows + C::RB - 1) / C::RB;
    ex.total = strips * ex.bps;
    ex.maxseg = maxseg > 0 ? maxseg : ex.bps;
    ex.two_gamma = (float)(2.0 * gamma);
    const int grid = ex.total < di.sms ? ex.total : di.sms;
    const size_t scratch_bytes = (size_t)grid * (t.npairs > 0 ? t.npairs : 1) * C::NCOLP * 16;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    bilateral_box_v8<R, OM><<<grid, C::NT, C::SMEM, s>>>(p, t, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
