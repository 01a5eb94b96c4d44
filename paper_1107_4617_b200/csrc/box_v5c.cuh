// box_v5c.cuh — "v5c": the large-radius v5 (box kernel, R = 33..64) on
// clusters of two CTAs that share their halo columns through distributed
// shared memory.
//
// v5 at large R gives every 256-column output strip its own 256 + 2R input
// columns of vertical moving sums: 1.5x the producer work at R = 64, and the
// producers (outgoing rows by MUFU) are the bottleneck.  Here two CTAs of a
// cluster own two adjacent strips; together they need 512 + 2R input columns,
// and each computes one half, 256 + R of them.  The R columns a CTA computes
// for its partner are also stored straight into the partner's slab with
// st.async (DSMEM), which completes transaction bytes on the partner's FULL
// mbarrier.  So the consumers read only local shared memory, exactly as in
// v5, and the producers do 1.25x instead of 1.5x the columns of a strip.
//
// Handoff: per slab slot two mbarriers in each CTA —
//   full[s]:  one arrival by producer thread 0 after a named barrier over
//             the producer warps (which drains their shared-memory stores),
//             + R x 16 x 16 bytes of partner st.async transactions
//             (expect_tx with that arrival);
//   empty[s]: 8 local + 8 partner consumer-warp arrivals (the partner's
//             producers write into this slot too, so they wait for both).
// Everything else — the one-CTA-per-SM balanced schedule over (strip pair,
// batch) units, segments, scratch, the consumer's delta/scan walkers, the
// register split 64/144 by setmaxnreg — is v5's (box_v5.cuh).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "box_kernel.cuh"
#include "box_v5.cuh"
#include "runtime.h"

namespace sf {

template <int R>
struct V5CCfg {
    static_assert(R > 32 && R <= 64, "v5c covers the large radii");
    static constexpr int L = 2 * R + 1;
    static constexpr int RB = 16, NSEG = 8, G = 32;
    static constexpr int TW = NSEG * G;             // 256 output columns per strip
    static constexpr int TWI = TW + 2 * R;          // input columns a strip's consumers read
    static constexpr int HALF = TW + R;             // input columns each CTA of the pair computes
    static constexpr int NV = 10, NH = 8;           // producer / consumer warps
    static_assert(HALF <= 32 * NV, "one column per producer lane");
    // + 2 idle warps: 20 warps compile to 96 registers (18 would too), and
    // then every sub-partition needs 3 warps releasing 96 - 64 for its 2
    // consumer warps' 144 - 96 (v5_pool_ok); the idle warps only release
    static constexpr int NVW = 12;                  // warps before the consumers
    static constexpr int NT = 32 * (NVW + NH);      // 640 threads
    static constexpr int PREG = 64, CREG = 144;
    static constexpr int TWP = 32 * NV;             // scratch columns per pair
    static constexpr int PAD = ((1 - G) % 8 + 8) % 8;
    static constexpr int NCOLP = TWI + PAD * (TWI / G) + 1;
    static constexpr int NBUF = 2;
    static constexpr int SMEM = NBUF * RB * NCOLP * 16;
    static constexpr int Q = L / G, PP = L % G;
    static constexpr int CH = 8;                    // band-top init rows per chunk
    static constexpr int kRemoteBytes = R * RB * 16;   // partner bytes per slot per step
    static_assert(Q < NSEG, "window must fit in the strip");
};

struct V5CExtra {
    float4* scratch;     // [cta][pair][TWP] running vertical sums
    int bps;             // RB-row batches per strip
    int total;           // strip pairs * bps
    int maxseg;          // batches per segment at most
    int strips;          // output strips (the last pair may have a strip past W)
    int diag;            // SF_DIAG = 3: no partner stores (timing of the DSMEM share; wrong output)
};

__device__ __forceinline__ uint32_t v5c_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t v5c_mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void v5c_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n"
            " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void v5c_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void v5c_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void v5c_arrive_remote(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void v5c_st_async(uint32_t cluster_addr, float4 v, uint32_t cluster_bar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
            cluster_addr),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(cluster_bar)
        : "memory");
}
__device__ __forceinline__ void v5c_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

struct V5CSeg {
    int x0, yb0, yend, nbatch;
};
__device__ __forceinline__ V5CSeg v5c_seg(const Params& p, const V5CExtra& ex, int tw, int rb, int rank, int u,
                                          int uend) {
    const int sp = u / ex.bps, b0 = u - sp * ex.bps;
    const int nb = min(min(ex.bps - b0, uend - u), ex.maxseg);
    V5CSeg g;
    g.x0 = (2 * sp + rank) * tw;
    g.yb0 = p.out_row0 + b0 * rb;
    g.yend = min(g.yb0 + nb * rb, p.out_row0 + p.out_rows);
    g.nbatch = nb;
    return g;
}

template <int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(V5CCfg<R>::NT, 1)
bilateral_box_v5c(const Params p, const PairTable tab, const V5CExtra ex) {
    using C = V5CCfg<R>;
    constexpr int L = C::L, G = C::G, RB = C::RB, PAD = C::PAD, NCOLP = C::NCOLP;
    constexpr int TW = C::TW, HALF = C::HALF, TWP = C::TWP, NBUF = C::NBUF, CH = C::CH;
    extern __shared__ float4 vbuf[];                     // [NBUF][RB][NCOLP]
    __shared__ __align__(8) uint64_t full_bar[NBUF], empty_bar[NBUF];

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t partner = rank ^ 1u;
    const int npairs = tab.npairs;
    const int ncl = gridDim.x >> 1, cid = blockIdx.x >> 1;
    const int q = ex.total / ncl, rem = ex.total % ncl;
    const int u_begin = cid * q + min(cid, rem);
    const int u_end = u_begin + q + (cid < rem ? 1 : 0);
    const int nsteps = (u_end - u_begin) * npairs;

    if (tid == 0) {
        for (int s = 0; s < NBUF; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(v5c_smem(&full_bar[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(v5c_smem(&empty_bar[s])), "r"(2 * C::NH));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    v5c_cluster_sync();

    if (warp >= C::NV && warp < C::NVW) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n");   // idle: registers for the consumers
    } else if (warp < C::NV) {
        // =========================== producers (vertical pass) =================
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n");
        const int t = tid;
        const bool act = t < HALF;
        const int c = rank == 0 ? t : R + t;              // strip-relative input column
        const int cs = c + PAD * (c / G);
        // the partner reads this column too: store it into its slab as well
        const bool remote = act && (rank == 0 ? c >= TW : c < 2 * R);
        const int cp = rank == 0 ? c - TW : c + TW;       // the column in the partner's strip
        const uint32_t rdst = v5c_mapa(v5c_smem(vbuf + (remote ? cp + PAD * (cp / G) : 0)), partner);
        float4* scr = ex.scratch + (size_t)blockIdx.x * npairs * TWP;
        const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5CSeg sgm = v5c_seg(p, ex, TW, RB, rank, u, u_end);
            u += sgm.nbatch;
            const int yb0 = sgm.yb0, nbatch = sgm.nbatch;
            const int gx = reflect101(sgm.x0 - R + min(c, C::TWI - 1), p.W);

            // band top: exact window sums of the row above the segment (as v5,
            // all by MUFU: the init is ~7 % of the work at these radii)
            if (act) {
                for (int i0 = 0; i0 < L; i0 += CH) {
                    float fv[CH], zc[CH], zs[CH];
#pragma unroll
                    for (int i = 0; i < CH; ++i) fv[i] = (i0 + i < L) ? ldf(p, yb0 - R - 1 + i0 + i, gx) : 0.f;
                    float4 Vn = (i0 == 0 || npairs == 0) ? zero4 : scr[(size_t)(npairs - 1) * TWP + t];
                    for (int n = 0; n < npairs; ++n) {
                        const int k = npairs - 1 - n;
                        const float om = tab.omega[k];
                        float4 V = Vn;
                        if (i0 > 0 && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWP + t];
#pragma unroll
                        for (int i = 0; i < CH; ++i) {
                            __sincosf(om * fv[i], &zs[i], &zc[i]);
                            if (i0 + i < L) {
                                V.x += zc[i];
                                V.y = fmaf(fv[i], zc[i], V.y);
                                V.z += zs[i];
                                V.w = fmaf(fv[i], zs[i], V.w);
                            }
                        }
                        scr[(size_t)k * TWP + t] = V;
                    }
                }
            }
            constexpr int RP = RB / 2;
            for (int b = 0; b < nbatch; ++b) {
                const int yb = yb0 + b * RB;
                uint32_t fi2[RP], fo2[RP];                // incoming / outgoing-row values, bf16 pairs
#pragma unroll
                for (int qq = 0; qq < RP; ++qq) {
                    const int i = 2 * qq;
                    fi2[qq] = v5_pack(act ? ldf(p, yb + i + R, gx) : 0.f, act ? ldf(p, yb + i + 1 + R, gx) : 0.f);
                    fo2[qq] = v5_pack(act ? ldf(p, yb + i - R - 1, gx) : 0.f, act ? ldf(p, yb + i - R, gx) : 0.f);
                }
                float4 Vn = (act && npairs > 0) ? scr[(size_t)(npairs - 1) * TWP + t] : zero4;
                for (int n = 0; n < npairs; ++n, ++step) {
                    const int k = npairs - 1 - n;
                    const float om = tab.omega[k];
                    const int slot = step % NBUF;
                    float4 V = Vn;
                    if (act && n + 1 < npairs) Vn = scr[(size_t)(k - 1) * TWP + t];   // prefetch next pair
                    if (step >= NBUF) v5c_wait(v5c_smem(&empty_bar[slot]), ((step / NBUF) - 1) & 1);
                    float4* dst = vbuf + slot * RB * NCOLP + cs;
                    const uint32_t rslot = rdst + (uint32_t)(slot * RB * NCOLP * 16);
                    const uint32_t rfull = v5c_mapa(v5c_smem(&full_bar[slot]), partner);
#pragma unroll
                    for (int qq = 0; qq < RP; ++qq) {
                        const float2 Fi = make_float2(v5_lo(fi2[qq]), v5_hi(fi2[qq]));
                        const float2 Fo = make_float2(v5_lo(fo2[qq]), v5_hi(fo2[qq]));
                        const float2 arg = __fmul2_rn(make_float2(om, om), Fi);
                        const float2 ao = __fmul2_rn(make_float2(om, om), Fo);
                        float2 C2, S2, Co, So;
                        __sincosf(arg.x, &S2.x, &C2.x);
                        __sincosf(arg.y, &S2.y, &C2.y);
                        __sincosf(ao.x, &So.x, &Co.x);
                        __sincosf(ao.y, &So.y, &Co.y);
                        const float2 Dc = __fadd2_rn(C2, make_float2(-Co.x, -Co.y));
                        const float2 Ds = __fadd2_rn(S2, make_float2(-So.x, -So.y));
                        const float2 Dfc = __ffma2_rn(Fi, C2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), Co));
                        const float2 Dfs = __ffma2_rn(Fi, S2, __fmul2_rn(make_float2(-Fo.x, -Fo.y), So));
                        V.x += Dc.x;
                        V.y += Dfc.x;
                        V.z += Ds.x;
                        V.w += Dfs.x;
                        if (act) dst[(2 * qq) * NCOLP] = V;
                        if (remote && ex.diag != 3) v5c_st_async(rslot + (uint32_t)((2 * qq) * NCOLP * 16), V, rfull);
                        V.x += Dc.y;
                        V.y += Dfc.y;
                        V.z += Ds.y;
                        V.w += Dfs.y;
                        if (act) dst[(2 * qq + 1) * NCOLP] = V;
                        if (remote && ex.diag != 3) v5c_st_async(rslot + (uint32_t)((2 * qq + 1) * NCOLP * 16), V, rfull);
                    }
                    asm volatile("bar.sync 1, %0;" ::"r"(32 * C::NV) : "memory");
                    if (tid == 0) v5c_arrive_tx(v5c_smem(&full_bar[slot]), ex.diag == 3 ? 0 : C::kRemoteBytes);
                    if (act) scr[(size_t)k * TWP + t] = V;
                }
            }
        }
    } else {
        // =========================== consumers (horizontal pass, v5's) =========
        asm volatile("setmaxnreg.inc.sync.aligned.u32 144;\n");
        const int w = tid - 32 * C::NVW;                 // 0..255
        const int hh = w & 1, sg = (w >> 1) & 7, hry = w >> 4;
        const int lane = w & 31;
        const int rowbase = lane & 16;
        const float hoff = hh ? 0.0f : 1.57079632679489662f;
        const int xs = sg * G;
        int step = 0;
        for (int u = u_begin; u < u_end;) {
            const V5CSeg sgm = v5c_seg(p, ex, TW, RB, rank, u, u_end);
            u += sgm.nbatch;
            const int x0 = sgm.x0, yb0 = sgm.yb0, yend = sgm.yend, nbatch = sgm.nbatch;
            for (int b = 0; b < nbatch; ++b) {
                const int gy = yb0 + b * RB + hry;
                float fxv[G];
                float2 QP[G];
#pragma unroll
                for (int j = 0; j < G; ++j) fxv[j] = ldf(p, gy, reflect101(x0 + xs + j, p.W));
#pragma unroll
                for (int j = 0; j < G; ++j) QP[j] = make_float2(0.f, 0.f);
                for (int n = 0; n < npairs; ++n, ++step) {
                    const int k = npairs - 1 - n;
                    const float om = tab.omega[k], wk = tab.weight[k];
                    const int slot = step % NBUF;
                    v5c_wait(v5c_smem(&full_bar[slot]), (step / NBUF) & 1);
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
                        T[j] = wk * __sinf(fmaf(om, fxv[j], hoff));
                        QP[j] = __ffma2_rn(make_float2(T[j], T[j]), dacc, QP[j]);
                        dacc = __fadd2_rn(dacc, __fadd2_rn(vi, make_float2(-vo.x, -vo.y)));
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
                    const float2 Ss = __fadd2_rn(S0, exc);
                    if (step + NBUF < nsteps) {               // slot empty: local and partner producers
                        __syncwarp();
                        if (lane == 0) {
                            const uint32_t e = v5c_smem(&empty_bar[slot]);
                            v5c_arrive(e);
                            v5c_arrive_remote(v5c_mapa(e, partner));
                        }
                    }
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
                            p.out[rowoff + gxo] = (qj > 0.f && isfinite(qj)) ? kCenter + pj / qj : kCenter + fxv[j];
                        } else {
                            p.num[rowoff + gxo] = pj;
                            p.den[rowoff + gxo] = qj;
                        }
                    }
                }
            }
        }
    }
    __threadfence();
    v5c_cluster_sync();   // no CTA leaves while its partner may still touch its shared memory
}

template <int R>
inline cudaError_t launch_box_v5c(const Params& p, const PairTable& t, int maxseg, cudaStream_t s) {
    using C = V5CCfg<R>;
    DeviceInfo& di = current_device_info();
    if (di.err != cudaSuccess) return di.err;
    static const bool pool_ok = [] {
        cudaFuncAttributes a{};
        return cudaFuncGetAttributes(&a, bilateral_box_v5c<R>) == cudaSuccess &&
               v5_pool_ok(a.numRegs, C::NVW, C::NH, C::PREG, C::CREG);
    }();
    if (!pool_ok) return cudaErrorLaunchOutOfResources;
    const cudaError_t attr =
        cudaFuncSetAttribute(bilateral_box_v5c<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (attr != cudaSuccess) return attr;
    V5CExtra ex;
    ex.strips = (p.W + C::TW - 1) / C::TW;
    ex.bps = (p.out_rows + C::RB - 1) / C::RB;
    ex.total = ((ex.strips + 1) / 2) * ex.bps;
    static const int maxseg_env = [] { const char* d = std::getenv("SF_V5_MAXSEG"); return d ? std::atoi(d) : 0; }();
    ex.maxseg = maxseg_env > 0 ? maxseg_env : (maxseg > 0 ? maxseg : ex.bps);
    static const int diag = [] { const char* d = std::getenv("SF_DIAG"); return d ? std::atoi(d) : 0; }();
    ex.diag = diag;
    const int ncl = ex.total < di.sms / 2 ? ex.total : di.sms / 2;   // one CTA per SM, pairs
    const size_t scratch_bytes = (size_t)2 * ncl * (t.npairs > 0 ? t.npairs : 1) * C::TWP * 16;
    cudaError_t e = scratch_alloc((void**)&ex.scratch, scratch_bytes, s);
    if (e != cudaSuccess) return e;
    bilateral_box_v5c<R><<<2 * ncl, C::NT, C::SMEM, s>>>(p, t, ex);
    e = cudaGetLastError();
    scratch_free(ex.scratch, s);
    return e;
}

}  // namespace sf
