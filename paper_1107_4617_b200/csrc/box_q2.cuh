// box_q2.cuh — "q2r": warp-specialised band-sweep kernel for Algorithm 2 with
// the separable raised-cosine spatial kernel q_2 (config 3; reading R5),
// compile-time radius R.  Same CTA organisation as v4r
// (box_v4r.cuh): 8 producer warps (vertical, one column per thread, 16-row
// batches, L2 scratch for the running state), 4 consumer warps (horizontal,
// register ring), double-buffered slabs, named barriers.
//
// q_2 per axis: w1(u) = (1 + cos(a u))/2, a = pi/(R+1), so
//   sum_u w1(u - t) g(u) = 1/2 A0(t) + 1/2 [cos(a t) Ac(t) + sin(a t) As(t)],
//   A0 = sum g(u), Ac = sum cos(a u) g(u), As = sum sin(a u) g(u) over the window,
// with any origin for u and t (shiftability).
//   producers: three running sums (A0, Ac, As) per stack image, modulated by the
//     row offset from the CURRENT BATCH START yb; at each batch the (Ac, As)
//     state is re-based to the new origin by one fixed rotation (a * RB).  All
//     per-row modulation factors are then compile-time constants.  The slab
//     holds the recombined weighted vertical sum Vw (C, FC, S, FS) — the same
//     slab format as the box kernels.
//   consumers: the horizontal weighted sum from a register ring of Vw with
//     three running sums per half, modulated by the column offset from the
//     walker's first column (walker-local origin: the walkers are independent),
//     so again every modulation factor is a compile-time constant.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"
#include "box_v4r.cuh"
#include "runtime.h"

namespace sf {

// constexpr cos/sin (Taylor series after reduction to [-pi, pi]) for the
// compile-time modulation factors
__host__ __device__ constexpr double q2_reduce(double x) {
    constexpr double tp = 6.283185307179586476925;
    while (x > 3.14159265358979323846) x -= tp;
    while (x < -3.14159265358979323846) x += tp;
    return x;
}
__host__ __device__ constexpr double q2_cos(double x) {
    x = q2_reduce(x);
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 30; ++k) {
        term *= -x * x / ((2.0 * k - 1.0) * (2.0 * k));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double q2_sin(double x) {
    x = q2_reduce(x);
    double term = x, sum = x;
    for (int k = 1; k < 30; ++k) {
        term *= -x * x / ((2.0 * k) * (2.0 * k + 1.0));
        sum += term;
    }
    return sum;
}

template <int R>
struct Q2Cfg {
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16;
    static constexpr int NSEG = 4;
    static constexpr int NV = 8, NH = 4;
    static constexpr int NT = 32 * (NV + NH);
    // consumer registers: 2G (Q,P') + G/2 (bf16 f_x) + 2L (ring) + 6 (sums) + ~32 <= 232
    static constexpr int GREG = (2 * (194 - 2 * L)) / 5;
    static constexpr int GCOL = (32 * NV - 2 * R) / NSEG;
    static constexpr int G0 = GREG < GCOL ? GREG : GCOL;
    static constexpr int G = G0 - (G0 & 1);
    static constexpr int TW = NSEG * G;
    static constexpr int TWI = TW + 2 * R;
    static constexpr int PAD = ((2 - G) % 8 + 8) % 8;
    static constexpr int NSLOT = NSEG * (G + PAD) + 2 * R + 8;
    static constexpr int NCOLP = NSLOT + ((1 - NSLOT) % 8 + 8) % 8;
    static constexpr int SMEM = 2 * RB * NCOLP * 16;
    static constexpr int kSeed = 8;
    static constexpr int MAXBAND = 256;
    static constexpr double A = 3.14159265358979323846 / (R + 1);
    static_assert(TWI <= 32 * NV && TWI > 32 * (NV - 1), "8 fully used producer warps");
    static_assert(2 * R <= G, "ring tail must stay within the next segment");
};

template <int R>
__global__ void __launch_bounds__(Q2Cfg<R>::NT, 1)
bilateral_q2_v4r(const Params p, const PairTable tab, const V4RExtra ex) {
    using C = Q2Cfg<R>;
    constexpr int L = C::L, G = C::G, RB = C::RB, PAD = C::PAD, NCOLP = C::NCOLP;
    constexpr int TWI = C::TWI, NT = C::NT;
    constexpr double A = C::A;
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
        const int cseg = c / G < C::NSEG ? c / G : C::NSEG;
        const int cslot = c + PAD * cseg;
        const int slot_id = (int)(blockIdx.y * gridDim.x + blockIdx.x);   // one scratch slot per CTA
        // state per pair: A0, Ac, As (3 float4), origin = the current batch start
        float4* scr = ex.scratch + (size_t)slot_id * npairs * TWI * 3;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        auto sidx = [&](int k, int w) { return ((size_t)k * TWI + c) * 3 + w; };

        // band top: window sums of the row above the band (rows yb0-R-1+i,
        // i < L), modulated by the offset (i - R - 1) from yb0; MUFU sincos
        if (act) {
            for (int k = 0; k < npairs; ++k) {
                const float om = tab.omega[k];
                float4 S0 = zero4, Sc = zero4, Ss = zero4;
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    const float f = ldf(p, yb0 - R - 1 + i, gx);
                    float s_, c_;
                    __sincosf(om * f, &s_, &c_);
                    const float4 g = make_float4(c_, f * c_, s_, f * s_);
                    const float cm = (float)q2_cos(A * (i - R - 1)), sm = (float)q2_sin(A * (i - R - 1));
                    S0 = f4add(S0, g);
                    Sc = f4fma(cm, g, Sc);
                    Ss = f4fma(sm, g, Ss);
                }
                scr[sidx(k, 0)] = S0;
                scr[sidx(k, 1)] = Sc;
                scr[sidx(k, 2)] = Ss;
            }
        }
        int step = 0;
        for (int b = 0; b < nbatch; ++b) {
            const int yb = yb0 + b * RB;
            float uc[RB], us[RB], zc[RB], zs[RB];
            uint32_t fi2[RB / 2], fo2[RB / 2];
#pragma unroll
            for (int i = 0; i < RB; i += 2) {
                fi2[i / 2] = pack_bf16x2(act ? ldf(p, yb + i + R, gx) : 0.f, act ? ldf(p, yb + i + 1 + R, gx) : 0.f);
                const float fa = act ? ldf(p, yb + i - R - 1, gx) : 0.f;
                const float fb = act ? ldf(p, yb + i - R, gx) : 0.f;
                fo2[i / 2] = pack_bf16x2(fa, fb);
                __sincosf(-ex.two_gamma * fa, &us[i], &uc[i]);
                __sincosf(-ex.two_gamma * fb, &us[i + 1], &uc[i + 1]);
            }
            for (int n = 0; n < npairs; ++n, ++step) {
                const int k = npairs - 1 - n;
                const float om = tab.omega[k];
                const int slot = step & 1;
                float4 S0 = act ? scr[sidx(k, 0)] : zero4;
                float4 Sc = act ? scr[sidx(k, 1)] : zero4;
                float4 Ss = act ? scr[sidx(k, 2)] : zero4;
                if (b > 0) {                                 // re-base (Sc, Ss) by a*RB rows
                    constexpr float cr = (float)q2_cos(A * RB), sr = (float)q2_sin(A * RB);
                    const float4 c0 = Sc;
                    Sc = f4fma(cr, c0, f4scale(sr, Ss));
                    Ss = f4fma(cr, Ss, f4scale(-sr, c0));
                }
                if (n % C::kSeed == 0) {
#pragma unroll
                    for (int i = 0; i < RB; ++i) {
                        const float fo = (i & 1) ? bf16_hi(fo2[i / 2]) : bf16_lo(fo2[i / 2]);
                        __sincosf(om * fo, &zs[i], &zc[i]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < RB; ++i) {
                        const float a = zc[i], bb = zs[i];
                        zc[i] = fmaf(a, uc[i], -bb * us[i]);
                        zs[i] = fmaf(a, us[i], bb * uc[i]);
                    }
                }
                if (step >= 2) v4r_bar_sync(3 + slot, NT);
                float4* dst = vbuf + slot * RB * NCOLP + cslot;
#pragma unroll
                for (int i = 0; i < RB; ++i) {
                    const float fo = (i & 1) ? bf16_hi(fo2[i / 2]) : bf16_lo(fo2[i / 2]);
                    const float fi = (i & 1) ? bf16_hi(fi2[i / 2]) : bf16_lo(fi2[i / 2]);
                    float s_, c_;
                    __sincosf(om * fi, &s_, &c_);
                    const float4 gi = make_float4(c_, fi * c_, s_, fi * s_);
                    const float4 go = make_float4(zc[i], fo * zc[i], zs[i], fo * zs[i]);
                    // modulation by the row offset from yb: in i+R, out i-R-1, centre i
                    const float ci = (float)q2_cos(A * (i + R)), si = (float)q2_sin(A * (i + R));
                    const float co = (float)q2_cos(A * (i - R - 1)), so = (float)q2_sin(A * (i - R - 1));
                    const float cc = (float)q2_cos(A * i), sc = (float)q2_sin(A * i);
                    S0 = f4add(S0, f4sub(gi, go));
                    Sc = f4fma(ci, gi, f4fma(-co, go, Sc));
                    Ss = f4fma(si, gi, f4fma(-so, go, Ss));
                    // weighted vertical sum at row yb+i: 1/2 S0 + 1/2 (cos Sc + sin Ss)
                    const float4 Vw = f4scale(0.5f, f4add(S0, f4fma(cc, Sc, f4scale(sc, Ss))));
                    if (act) dst[i * NCOLP] = Vw;
                }
                v4r_bar_arrive(1 + slot, NT);
                if (act) {
                    scr[sidx(k, 0)] = S0;
                    scr[sidx(k, 1)] = Sc;
                    scr[sidx(k, 2)] = Ss;
                }
            }
        }
        __threadfence();   // the next CTA on this SM reuses the scratch slot
    } else {
        // =========================== consumers (horizontal pass) ===============
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n");
        const int w = tid - 32 * C::NV;
        const int hh = w & 1, hs = (w >> 1) & 3, hry = w >> 3;
        const float hoff = hh ? 0.0f : 1.57079632679489662f;
        int step = 0;
        for (int b = 0; b < nbatch; ++b) {
            const int yb = yb0 + b * RB;
            const int gy = yb + hry;
            uint32_t fpk[G / 2];
            float2 QP[G];
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
                v4r_bar_sync(1 + slot, NT);
                const float2* vrow =
                    reinterpret_cast<const float2*>(vbuf + (slot * RB + hry) * NCOLP + hs * (G + PAD)) + hh;
                float2 ring[L];
                float2 a0 = make_float2(0.f, 0.f), ac = a0, as = a0;
#pragma unroll
                for (int j = 0; j < G + 2 * R; ++j) {
                    const int col = j + (j >= G ? PAD : 0);
                    const float2 v = vrow[2 * col];
                    // column j of the walker (walker-local origin): cos/sin(a j)
                    const float cj = (float)q2_cos(A * j), sj = (float)q2_sin(A * j);
                    if (j >= L) {
                        const float2 o = ring[j % L];
                        const float cl = (float)q2_cos(A * (j - L)), sl = (float)q2_sin(A * (j - L));
                        a0 = __fadd2_rn(a0, __fadd2_rn(v, make_float2(-o.x, -o.y)));
                        ac = __ffma2_rn(make_float2(cj, cj), v, __ffma2_rn(make_float2(-cl, -cl), o, ac));
                        as = __ffma2_rn(make_float2(sj, sj), v, __ffma2_rn(make_float2(-sl, -sl), o, as));
                    } else {
                        a0 = __fadd2_rn(a0, v);
                        ac = __ffma2_rn(make_float2(cj, cj), v, ac);
                        as = __ffma2_rn(make_float2(sj, sj), v, as);
                    }
                    ring[j % L] = v;
                    if (j >= 2 * R) {
                        const int o = j - 2 * R;                 // window centre at walker column o + R
                        const float ccn = (float)q2_cos(A * (o + R)), scn = (float)q2_sin(A * (o + R));
                        const float2 hw = __ffma2_rn(make_float2(ccn, ccn), ac, __ffma2_rn(make_float2(scn, scn), as, a0));
                        const float fx = (o & 1) ? bf16_hi(fpk[o / 2]) : bf16_lo(fpk[o / 2]);
                        const float t = 0.5f * wk * __sinf(fmaf(om, fx, hoff));
                        QP[o] = __ffma2_rn(make_float2(t, t), hw, QP[o]);
                    }
                }
                if (step + 2 < nsteps) v4r_bar_arrive(3 + slot, NT);
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

template <int R>
inline cudaError_t launch_q2_v4r(const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    using C = Q2Cfg<R>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    const cudaError_t attr = cudaFuncSetAttribute(bilateral_q2_v4r<R>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (attr != cudaSuccess) return attr;
    int per_sm_blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_blocks, bilateral_q2_v4r<R>, C::NT, C::SMEM);
    const int strips = (p.W + C::TW - 1) / C::TW;
    V4RExtra ex;
    ex.band = v4r_band(p.out_rows, strips, di.sms, 2 * C::L, drift_maxband(t, C::MAXBAND));
    ex.two_gamma = (float)(2.0 * gamma);
    const int bands = (p.out_rows + ex.band - 1) / ex.band;
    ex.per_sm = 0;
    (void)per_sm_blocks;
    const size_t slots = (size_t)strips * bands;     // scratch slot = CTA index
    const size_t scratch_bytes = slots * (t.npairs > 0 ? t.npairs : 1) * C::TWI * 16 * 3;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    bilateral_q2_v4r<R><<<dim3(strips, bands), C::NT, C::SMEM, s>>>(p, t, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
