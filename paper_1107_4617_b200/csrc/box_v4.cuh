// box_v4.cuh — "v4b": warp-specialised band-sweep kernel for Algorithm 2
// (PAPER.md:146-156), box spatial kernel, ANY radius 0 <= R <= 64 at run time
// (DESIGN.md §5).  The default only for r = 0 (and SF_VARIANT=v4b): every
// radius 1..64 has a compile-time band-sweep kernel (v7, v5).
//
// CTA = NV producer warps (one input column per thread, TWI = 256 + 2R
// columns) + 4 consumer warps; one output strip of TW = 256 columns x one
// band of rows, swept in batches of RB = 8 rows; per (batch, conjugate pair)
// step the producers hand the consumers an 8-row slab of vertical moving sums
// through a double-buffered shared-memory ring (named barriers FULL/EMPTY).
//
//   producers (vertical pass, as v3): stack images cos, (f-c)cos, sin,
//     (f-c)sin of w_k (f-c) (Alg. 2 step 1) — incoming row with MUFU sincos,
//     outgoing row by the rotation recurrence across pairs (re-seeded every
//     kSeed pairs); running vertical sums ("recursion") with the
//     state in an L2-resident scratch between batches; the next pair's state
//     is prefetched while the current pair is processed.
//   consumers (horizontal pass, no register ring, no halo re-read):
//     walker = (row, segment of G = 32 outputs, half); the 8 segment walkers
//     of one (row, half) are lanes of one warp.
//       pass 1: D_j = sum_{i<=j} (V[x_j + 2R + 1] - V[x_j])  (in - out, two
//               reads per output) kept in registers, plus the walker's block
//               total B_s = sum of its 32 "out" columns and the prefix of its
//               out columns at p = (2R+1) mod 32;
//       scan:   the window sum at the segment start
//                 S_0 = B_0 + ... + B_{q-1} + prefix_q(p),   2R+1 = 32q + p,
//                 S_{s+1} = S_s + D^{(s)}_{G-1}              (telescoping)
//               by warp shuffles (exact sums of the same values, no long
//               prefix differences);
//       pass 2: window(x_j) = S_s + D_j, so Q, P' += t_j (S_s + D_j) with
//               t_j = w_k cos|sin(w_k f_x) (Alg. 2 step 3): the
//               t_j D_j part is added in pass 1, t_j S_s here (packed FFMA2).
//     Partials stay in registers across all pairs; the halves combine with one
//     shuffle and the band writes c + P'/Q (or P', Q for the term split).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"
#include "runtime.h"

namespace sf {

struct V4BCfg {
    static constexpr int RB = 8;                 // rows per step
    static constexpr int NSEG = 8;               // segments per row (lanes of one warp)
    static constexpr int G = 32;                 // outputs per walker
    static constexpr int TW = NSEG * G;          // 256 output columns per strip
    static constexpr int NH = 4;                 // consumer warps (RB x NSEG x 2 = 128)
    static constexpr int MAXR = 64;
    static constexpr int NVMAX = (TW + 2 * MAXR + 31) / 32;     // 12 producer warps
    static constexpr int NTMAX = 32 * (NVMAX + NH);              // 512 threads
    static constexpr int kSeed = 8;              // rotation re-seed period (pairs)
    static constexpr int MAXBAND = 1024;       // long bands amortise the L-row band-top init
    // slot(c) = c + c/32: one pad float4 per 32 columns -> the 8 segments x 2
    // halves of a row hit disjoint banks; producer warps store 512 B runs.
    static constexpr int NCOLP = 400;            // >= slot(TW + 2*MAXR - 1) + 1 = 396
    static constexpr int SMEM = 2 * RB * NCOLP * 16;
    // setmaxnreg (CTA register pool = NT x 128 at launch): producers release
    // NV*32*(128-104) >= 8*32*24 = 6144 >= consumers' need 128*(152-128) = 3072
    static constexpr int PREG = 104, CREG = 152;
};

struct V4Extra {
    float4* scratch;     // [slot][pair][TWI] running vertical sums
    int per_sm;          // unused (the slot is the CTA index; %smid is not stable)
    int band;            // rows per band (multiple of RB, <= MAXBAND)
    float two_gamma;     // w_k - w_{k-1}
};

__device__ __forceinline__ int v4_slot(int c) { return c + (c >> 5); }

__device__ __forceinline__ void v4_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void v4_bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }

__global__ void __launch_bounds__(V4BCfg::NTMAX, 1)
bilateral_box_v4b(const Params p, const PairTable tab, const V4Extra ex) {
    using C = V4BCfg;
    constexpr int RB = C::RB, G = C::G, NCOLP = C::NCOLP;
    extern __shared__ float4 vbuf[];                     // [2][RB][NCOLP]

    const int R = p.r, L = 2 * R + 1;
    const int TWI = C::TW + 2 * R;
    const int NV = (TWI + 31) >> 5;
    const int NT = 32 * (NV + C::NH);
    const int tid = threadIdx.x;
    const int npairs = tab.npairs;
    const int x0 = blockIdx.x * C::TW;
    const int yb0 = p.out_row0 + blockIdx.y * ex.band;
    const int yend = min(yb0 + ex.band, p.out_row0 + p.out_rows);
    const int nbatch = (yend - yb0 + RB - 1) / RB;
    const int nsteps = nbatch * npairs;
    const int warp = tid >> 5;

    if (warp < NV) {
        // =========================== producers (vertical pass) =================
        asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n");
        const int c = tid;
        const bool act = c < TWI;
        const int gx = reflect101(x0 - R + (act ? c : 0), p.W);
        const int cs = v4_slot(c);
        const int slot_id = (int)(blockIdx.y * gridDim.x + blockIdx.x);   // one scratch slot per CTA
        float4* scr = ex.scratch + (size_t)slot_id * npairs * TWI;

        // band top: exact window sums of the row above the band, rows
        // [yb0-R-1, yb0+R-1], accumulated RB rows at a time with the rotation
        // recurrence across pairs (seeded by MUFU every kSeed pairs).
        if (act) {
            for (int i0 = 0; i0 < L; i0 += RB) {
                float fv[RB], zc[RB], zs[RB], uc[RB], us[RB];
#pragma unroll
                for (int i = 0; i < RB; ++i) {
                    const bool in = i0 + i < L;
                    fv[i] = in ? ldf(p, yb0 - R - 1 + i0 + i, gx) : 0.f;
                    __sincosf(-ex.two_gamma * fv[i], &us[i], &uc[i]);
                }
                const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
                float4 Vn = (i0 == 0 || npairs == 0) ? zero4 : scr[(size_t)(npairs - 1) * TWI + c];
                for (int n = 0; n < npairs; ++n) {
                    const int k = npairs - 1 - n;
                    const float om = tab.omega[k];
                    float4 V = Vn;
                    if (i0 > 0 && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWI + c];   // prefetch
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
            float4 Vn = (act && npairs > 0) ? scr[(size_t)(npairs - 1) * TWI + c] : make_float4(0.f, 0.f, 0.f, 0.f);
            for (int n = 0; n < npairs; ++n, ++step) {
                const int k = npairs - 1 - n;            // |w_k| ascending
                const float om = tab.omega[k];
                const int slot = step & 1;
                float4 V = Vn;
                if (act && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWI + c];   // prefetch
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
                if (step >= 2) v4_bar_sync(3 + slot, NT);  // wait: slot consumed
                float4* dst = vbuf + slot * RB * NCOLP + cs;
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
                v4_bar_arrive(1 + slot, NT);             // slot full
                if (act) scr[(size_t)k * TWI + c] = V;
            }
        }
        __threadfence();   // the next CTA on this SM reuses the scratch slot
    } else {
        // =========================== consumers (horizontal pass) ===============
        asm volatile("setmaxnreg.inc.sync.aligned.u32 152;\n");
        const int w = tid - 32 * NV;                     // 0..127
        const int hh = w & 1, sg = (w >> 1) & 7, hry = w >> 4;
        const int lane = w & 31;
        const float hoff = hh ? 0.0f : 1.57079632679489662f;
        const int q = L >> 5, pp = L & 31;               // 2R+1 = 32 q + pp
        const int xs = sg * G;                           // first output column (strip-relative)
        int step = 0;
        for (int b = 0; b < nbatch; ++b) {
            const int yb = yb0 + b * RB;
            const int gy = yb + hry;
            float fpx[G];
            float2 QP[G];
#pragma unroll
            for (int j = 0; j < G; ++j) {
                fpx[j] = ldf(p, gy, reflect101(x0 + xs + j, p.W));
                QP[j] = make_float2(0.f, 0.f);
            }
            for (int n = 0; n < npairs; ++n, ++step) {
                const int k = npairs - 1 - n;
                const float om = tab.omega[k], wk = tab.weight[k];
                const int slot = step & 1;
                v4_bar_sync(1 + slot, NT);                // wait: slot full
                const float2* vrow = reinterpret_cast<const float2*>(vbuf + (slot * RB + hry) * NCOLP) + hh;
                // pass 1: running (in - out) deltas D_j (window(x_j) = S_s + D_j),
                // block total, out-prefix at pp.  The D_j part of the output is
                // accumulated at once (Q, P' += t_j D_j) and t_j kept for pass 2.
                float T[G];
                float2 dacc = make_float2(0.f, 0.f), bsum = make_float2(0.f, 0.f), bpre = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const int co = xs + j, ci = co + L;
                    const float2 vo = vrow[2 * v4_slot(co)];
                    // the last segment's final "in" column (ci = TWI) is past the
                    // strip; its delta feeds no later segment, so read zero
                    const float2 vi = (j < G - 1 || ci < TWI) ? vrow[2 * v4_slot(ci)] : make_float2(0.f, 0.f);
                    if (j == pp) bpre = bsum;
                    bsum = f2add(bsum, vo);
                    T[j] = wk * __sinf(fmaf(om, fpx[j], hoff));
                    QP[j] = __ffma2_rn(make_float2(T[j], T[j]), dacc, QP[j]);
                    dacc = f2add(dacc, f2sub(vi, vo));
                }
                // S_0 = sum_{m<q} B_m + prefix_q(pp); segments are lanes 2*sg+hh (+16 rows)
                const int rowbase = lane & 16;            // lanes of this row: rowbase + 2*s + hh
                float2 S0 = make_float2(0.f, 0.f);
                for (int m = 0; m < q && m < 8; ++m) {
                    const int src = rowbase + 2 * m + hh;
                    S0.x += __shfl_sync(0xffffffffu, bsum.x, src);
                    S0.y += __shfl_sync(0xffffffffu, bsum.y, src);
                }
                if (q < 8) {
                    const int src = rowbase + 2 * q + hh;
                    S0.x += __shfl_sync(0xffffffffu, bpre.x, src);
                    S0.y += __shfl_sync(0xffffffffu, bpre.y, src);
                } else {
                    // 2R+1 >= 256: the window passes the strip's 8 blocks (R >= 128, never)
                }
                // inclusive scan of the segment totals dacc over sg (3 steps, stride
                // 2 lanes), then shifted by one segment -> exclusive
                float2 ex_ = dacc;
#pragma unroll
                for (int d = 1; d < 8; d <<= 1) {
                    const float tx = __shfl_up_sync(0xffffffffu, ex_.x, 2 * d);
                    const float ty = __shfl_up_sync(0xffffffffu, ex_.y, 2 * d);
                    if (sg >= d) {
                        ex_.x += tx;
                        ex_.y += ty;
                    }
                }
                float2 exc;
                exc.x = __shfl_up_sync(0xffffffffu, ex_.x, 2);
                exc.y = __shfl_up_sync(0xffffffffu, ex_.y, 2);
                if (sg == 0) exc = make_float2(0.f, 0.f);
                const float2 Ss = f2add(S0, exc);                // S_0 + sum_{s'<s} dacc_{s'}
                if (step + 2 < nsteps) v4_bar_arrive(3 + slot, NT);   // slot empty (data in registers)
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

// band height: <= maxband rows, multiple of rb, minimising waves x (band + L)
inline int v4_band(int rows, int strips, int sms, int L, int maxband, int rb) {
    int best = rb;
    double best_cost = 1e30;
    for (int band = rb; band <= maxband; band += rb) {
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

inline cudaError_t launch_box_v4b(const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    using C = V4BCfg;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    const cudaError_t attr = cudaFuncSetAttribute(bilateral_box_v4b, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   C::SMEM);
    if (attr != cudaSuccess) return attr;
    const int TWI = C::TW + 2 * p.r;
    const int NV = (TWI + 31) / 32;
    const int NT = 32 * (NV + C::NH);
    int per_sm_blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_blocks, bilateral_box_v4b, NT, C::SMEM);
    const int strips = (p.W + C::TW - 1) / C::TW;
    V4Extra ex;
    ex.band = v4_band(p.out_rows, strips, di.sms, 2 * p.r + 1, C::MAXBAND, C::RB);
    ex.two_gamma = (float)(2.0 * gamma);
    const int bands = (p.out_rows + ex.band - 1) / ex.band;
    ex.per_sm = 0;
    (void)per_sm_blocks;
    const size_t slots = (size_t)strips * bands;     // scratch slot = CTA index
    const size_t scratch_bytes = slots * (t.npairs > 0 ? t.npairs : 1) * TWI * 16;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    bilateral_box_v4b<<<dim3(strips, bands), NT, C::SMEM, s>>>(p, t, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
