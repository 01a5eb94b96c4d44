/*
 * sf.h — C-ABI of the B200 (sm_100a) constant-time bilateral filter with a
 * shiftable raised-cosine range kernel (Chaudhury, "Constant-time filtering
 * using shiftable kernels", arxiv 1107.4617).
 *
 * Library: paper_1107_4617_b200/libsf.so.  Plain C types only; no torch or
 * CUDA types in the signatures (`stream` is a cudaStream_t passed as void*,
 * NULL = the legacy default stream).
 *
 * What every entry point computes (Eq.(3), evaluated by
 * Algorithm 2):
 *
 *   out[y,x] = sum_{|dy|,|dx|<=r} w(dy,dx) phi(f(y+dy,x+dx) - f(y,x)) f(y+dy,x+dx)
 *              ------------------------------------------------------------------
 *              sum_{|dy|,|dx|<=r} w(dy,dx) phi(f(y+dy,x+dx) - f(y,x))
 *
 *   phi(t) = cos(t / (sigma_r sqrt N))^N   — q_N of PAPER.md:202 in the sigma_r
 *            scaling of Eq.(6), expanded per Eq.(1) into the
 *            N+1 exponentials e^{j (2n-N) t/(sigma_r sqrt N)} with weights
 *            C(N,n)/2^N (computed in fp64 on the host, used in fp32);
 *   w      = 1 (SF_SPATIAL_BOX) or w1(dy) w1(dx), w1(u) = (1+cos(pi u/(r+1)))/2
 *            (SF_SPATIAL_RAISED_COS, q_2 with T = r+1);
 *   f      = the uint8 image extended by whole-sample symmetric reflection
 *            ("reflect-101": -i -> i, (L-1)+i -> (L-1)-i), reading R3.
 *
 * Layout: images are row-major and tightly packed: uint8 input pitch = W
 * bytes, fp32 output pitch = W floats.  Row index y in [0,H), column x in [0,W).
 * Ownership: every pointer argument is caller-owned.  Internally the library
 * takes scratch from a private stream-ordered device memory pool (per
 * device): the running-sum state of the band-sweep kernels (~16 B per strip
 * column per conjugate pair per SM, e.g. 20-32 MB for config 5), the fp32
 * partials of sf_accumulate_add / _scatter (8 B per pixel) and the staging
 * buffers of the *_host entry points (5 B per pixel).  Scratch is returned to
 * the pool on the call's stream before the call returns, and the pool KEEPS
 * it for the next call (re-mapping 10-300 MB costs milliseconds); call
 * sf_release_scratch() to hand the unused part back to the device (e.g.
 * before a large allocation by another library).
 * Errors: arguments are validated synchronously and NOTHING is enqueued on
 * error.  On success the device-pointer entry points are asynchronous on
 * `stream`; launch failures return SF_ERR_CUDA; asynchronous faults surface
 * at the caller's next synchronisation.  No global mutable state: calls on
 * distinct streams are thread-safe.  No CPU fallback exists: without a CUDA
 * device every compute entry point returns SF_ERR_CUDA.
 */
#ifndef SF_H
#define SF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SF_SPATIAL_BOX = 0,          /* w = 1 on [-r,r]^2 (configs 1,2,4,5)            */
    SF_SPATIAL_RAISED_COS = 1    /* w = q_2 (x) q_2, T = r+1 (config 3)             */
} sf_spatial_kind;

/* General separable shiftable spatial kernels: spatial
 * kind SF_SPATIAL_QM(M), M = 1..8, is w = q_M (x) q_M with
 * q_M(u) = cos(pi u / (2(r+1)))^M on |u| <= r (PAPER.md:202 with T = r+1, so
 * the kernel is positive on the window); its order of shiftability is M+1 per
 * axis, (M+1)^2 spatial terms in Algorithm 2.  SF_SPATIAL_QM(2) equals
 * SF_SPATIAL_RAISED_COS. */
#define SF_SPATIAL_QM(M) (100 + (M))

typedef enum {
    SF_OK = 0,
    SF_ERR_NULL = 1,        /* a required pointer is NULL                          */
    SF_ERR_SHAPE = 2,       /* H < 1 or W < 1                                      */
    SF_ERR_RADIUS = 3,      /* radius < 0 or radius > min(H,W)-1 (reflect-101), or
                               radius > SF_MAX_RADIUS                              */
    SF_ERR_SIGMA = 4,       /* sigma_r not finite or <= 0                          */
    SF_ERR_ORDER = 5,       /* N < sf_nmin(sigma_r) (kernel not a valid kernel,
                               PAPER.md:276-279) or N > SF_MAX_ORDER               */
    SF_ERR_KIND = 6,        /* unknown spatial_kind (not BOX, RAISED_COS, QM(1..8)) */
    SF_ERR_RANGE = 7,       /* bad row range or pair range                         */
    SF_ERR_ALIAS = 8,       /* an output buffer overlaps an input buffer           */
    SF_ERR_CUDA = 9         /* CUDA error (no device, launch failure, copy failure)*/
} sf_status;

#define SF_CENTER 128.0f      /* centring constant of the partial numerators      */
#define SF_MAX_ORDER 2048     /* largest N accepted                                */
#define SF_MAX_RADIUS 64      /* largest spatial radius accepted.  The run time of
                                 the band-sweep kernels is independent of r
                                  but their strip holds
                                 TW + 2r input columns in one CTA's shared
                                 memory and producer warps;
                                 r = 64 keeps the halo at <= 1/2 of a 256-column
                                 strip.  Larger radii return SF_ERR_RADIUS.    */

/* Whole-image filter.  img: device, H*W uint8.  out: device, H*W float
 * (unrounded grey levels).  N >= sf_nmin(sigma_r).  Asynchronous on stream. */
sf_status sf_filter(const uint8_t *img, int H, int W, int radius, int spatial_kind,
                    double sigma_r, int N, float *out, void *stream);

/* Row band of the same filter (multi-GPU row-band sharding).
 * Output rows [row_begin,row_end) of the H x W image are written to out_band
 * ((row_end-row_begin) x W floats, device).  img_band (device) holds the input
 * rows [max(0,row_begin-radius), min(H,row_end+radius)) of the full image,
 * first of them at img_band.  Output is identical to the corresponding rows
 * of sf_filter.  Requires 0 <= row_begin < row_end <= H. */
sf_status sf_filter_rows(const uint8_t *img_band, int H, int W, int row_begin, int row_end,
                         int radius, int spatial_kind, double sigma_r, int N,
                         float *out_band, void *stream);

/* Term split: partial numerator and denominator of
 * Algorithm 2 step 3 over conjugate pairs [pair_begin,pair_end) of
 * 0..sf_pair_count(N)-1 (pair k joins terms n=k and n=N-k; for even N the last
 * pair is the single middle term n=N/2).  num/den: device, H*W floats,
 * OVERWRITTEN (not accumulated):
 *   num = sum_{pairs} sum_y w phi_k (f(x-y) - SF_CENTER),  den = sum_{pairs} sum_y w phi_k
 * where phi_k is the pair's share of phi.  Summing num/den over a partition
 * of the pairs and calling sf_finalize gives sf_filter's result. */
sf_status sf_accumulate(const uint8_t *img, int H, int W, int radius, int spatial_kind,
                        double sigma_r, int N, int pair_begin, int pair_end,
                        float *num, float *den, void *stream);

/* As sf_accumulate, but the partials are ADDED into num/den (fp32 atomic adds,
 * in no fixed order, by a scatter-add pass after the filter kernel — 2
 * launches; the partials live in library scratch meanwhile) instead of
 * overwriting them.
 * num/den may be another GPU's buffers mapped into this process (CUDA IPC;
 * NVLink / NVSwitch peer memory): the term split with a one-sided reduction
 * — each rank adds the partial sums of its pair range
 * straight into the root's two H x W images, with no collective library.
 * The caller zeroes num/den before the first add and orders all adds before
 * sf_finalize (stream / host barrier).  Errors as sf_accumulate. */
sf_status sf_accumulate_add(const uint8_t *img, int H, int W, int radius, int spatial_kind,
                            double sigma_r, int N, int pair_begin, int pair_end,
                            float *num, float *den, void *stream);

/* As sf_accumulate_add, with the output rows split into nband (1..8) bands
 * [o*H/nband, (o+1)*H/nband) and band o's partials added into band_num[o] /
 * band_den[o] (each (rows of band o) x W, typically rank o's buffer mapped
 * into this process): the reduce-scatter form — every rank receives only its
 * band's partials, so no single GPU's NVLink ingress
 * carries everything.  SF_ERR_NULL for a null band pointer, SF_ERR_RANGE for
 * nband outside 1..min(8, H); otherwise as sf_accumulate. */
sf_status sf_accumulate_scatter(const uint8_t *img, int H, int W, int radius, int spatial_kind,
                                double sigma_r, int N, int pair_begin, int pair_end, int nband,
                                float *const *band_num, float *const *band_den, void *stream);

/* The last line of Algorithm 2: f~ = P/Q, here with the
 * partials centred at SF_CENTER, out = SF_CENTER + num/den; where den <= 0 or
 * is not finite, out = img (never expected for N >= N0: den >= 1, reading R9).
 * All device pointers, H*W each; out must not overlap num, den or img
 * (SF_ERR_ALIAS).  Asynchronous on stream. */
sf_status sf_finalize(const float *num, const float *den, const uint8_t *img, int H, int W,
                      float *out, void *stream);

/* Constant-time spatial filtering, Algorithm 1:
 *   out[y,x] = sum_{|dy|,|dx|<=r} w(dy,dx) f(y+dy,x+dx) / sum w(dy,dx)
 * with the spatial_kind weight (box = moving average, or q_M) and reflect-101
 * f — the filter of sf_filter with the range kernel replaced by 1 (order 0).
 * Arguments, layout and errors as sf_filter (no sigma_r / N). */
sf_status sf_spatial_filter(const uint8_t *img, int H, int W, int radius, int spatial_kind,
                            float *out, void *stream);

/* Shiftable non-local means with a tiny patch (
 * Eq.(NL) and Eq.(approx_multivariate)):
 *   out[y,x] = sum_{|dy|,|dx|<=r} f(z) phi(t) / sum phi(t),   z = (y-dy, x-dx),
 *   t_k = f(x+u_k) - f(z+u_k) over the patch offsets u_1 = (0,0), u_2 = (0,1),
 *   u_3 = (1,0) (p = 1, 2 or 3 of them, reading R14),
 *   phi(t) = prod_k cos(gamma_k t_k)^n ~ exp(-h^-2 sum_k g(u_k) t_k^2),
 *   gamma_k = sqrt(2 g(u_k) / (n h^2)), g(u) = exp(-|u|^2 / (2 rho^2))
 * (rho = 0: only the centre pixel, g = [u = 0]), reflect-101 f.  The order
 * of the separable shiftable kernel is (n+1)^p; its
 * conjugate pairs, sf_nlm_pair_count(p, n), must be <= 512.  n must be
 * >= sf_nmin(h / sqrt 2) (every factor a valid kernel).  Errors:
 * SF_ERR_KIND for p outside 1..3, SF_ERR_SIGMA for h <= 0 or rho < 0 or
 * non-finite, SF_ERR_ORDER for n out of range; otherwise as sf_filter.
 * p = 1 is the bilateral filter of sf_filter with sigma_r = h / sqrt 2, N = n. */
sf_status sf_nlm(const uint8_t *img, int H, int W, int radius, int p, double h, double rho, int n,
                 float *out, void *stream);

/* Conjugate pairs of the order-(n+1)^p NLM expansion; -1 for invalid p, n. */
int sf_nlm_pair_count(int p, int n);

/* Truncated expansion: "discarding the less significant
 * basis functions" of Eq.(1).  The terms n with
 * C(N,n)/2^N < eps * max_n C(N,n)/2^N are dropped — n0 = sf_truncation_n0(N,
 * eps) at each end — and the filter of sf_filter is evaluated with the kept
 * terms n0..N-n0 (conjugate pairs n0..floor(N/2)), i.e. with the kernel
 * phi_eps(t) = sum_{n=n0}^{N-n0} C(N,n) 2^-N cos((2n-N) t/(sigma_r sqrt N)).
 * The work is the kept terms; |phi_eps - phi| <= the dropped weight.
 * eps in [0, 1) (0 = sf_filter exactly); otherwise SF_ERR_RANGE.  Arguments,
 * layout and errors otherwise as sf_filter. */
sf_status sf_filter_truncated(const uint8_t *img, int H, int W, int radius, int spatial_kind,
                              double sigma_r, int N, double eps, float *out, void *stream);

/* Terms dropped at each end of the order-N expansion for threshold eps (see
 * sf_filter_truncated); -1 for invalid arguments. */
int sf_truncation_n0(int N, double eps);

/* End-to-end convenience: HOST img (H*W uint8) -> HOST out (H*W float).
 * Copies host->device, runs sf_filter, copies device->host on `stream`, and
 * synchronises the stream before returning.  Pinned host memory is fastest. */
sf_status sf_filter_host(const uint8_t *img_host, int H, int W, int radius, int spatial_kind,
                         double sigma_r, int N, float *out_host, void *stream);

/* Row-band variant of sf_filter_host (HOST img_band as in sf_filter_rows,
 * HOST out_band of (row_end-row_begin) x W floats). */
sf_status sf_filter_rows_host(const uint8_t *img_band_host, int H, int W, int row_begin,
                              int row_end, int radius, int spatial_kind, double sigma_r, int N,
                              float *out_band_host, void *stream);

/* Asynchronous form of sf_filter_rows_host for pipelined end-to-end use:
 * enqueues the host->device copy of img_band_host on a library copy stream,
 * the filter on `stream` (after that copy), and the device->host copy into
 * out_band_host on a second library copy stream (after the filter), and
 * returns without waiting.  Successive calls therefore overlap one call's
 * output copy and the next call's input copy with the kernels.  Both host
 * buffers must be page-locked and stay valid until sf_host_sync() returns;
 * out_band_host is complete only then.  Arguments and errors as
 * sf_filter_rows_host. */
sf_status sf_filter_rows_host_async(const uint8_t *img_band_host, int H, int W, int row_begin,
                                    int row_end, int radius, int spatial_kind, double sigma_r, int N,
                                    float *out_band_host, void *stream);

/* Wait for every copy enqueued by sf_filter_rows_host_async on this device. */
sf_status sf_host_sync(void);

/* Return the unused memory of this device's scratch pool (see Ownership)
 * to the device: cudaMemPoolTrimTo(pool, 0) after synchronising the device.
 * SF_ERR_CUDA without a device or on failure. */
sf_status sf_release_scratch(void);

/* Gaussian-fitted separable spatial kernel: the filter
 * of sf_filter with the spatial weight w(dy,dx) = w1(dy) w1(dx),
 *   w1(u) = q_M(u / sqrt M) = cos(u / (sigma_s sqrt M))^M  on |u| <= radius,
 * i.e. q_M of PAPER.md:202 with T = pi sigma_s / 2, whose Eq.(7) limit
 * (exponent pi^2, reading R10) is exp(-u^2/(2 sigma_s^2)):
 * a spatial Gaussian of width sigma_s, independent of the window radius
 * (reading R18).  Order M+1 per axis, (M+1)^2 spatial terms in Algorithm 2.
 * M = 1..8 (SF_ERR_KIND) and M >= sf_spatial_mmin(radius, sigma_s), the
 * order at which w1 >= 0 on the window (SF_ERR_ORDER); sigma_s finite > 0
 * (SF_ERR_SIGMA).  Other arguments and errors as sf_filter. */
sf_status sf_filter_spatial_sigma(const uint8_t *img, int H, int W, int radius, double sigma_s, int M,
                                  double sigma_r, int N, float *out, void *stream);

/* Algorithm 1 with the same Gaussian-fitted spatial
 * kernel: out = sum w f / sum w.  Arguments as sf_filter_spatial_sigma. */
sf_status sf_spatial_filter_sigma(const uint8_t *img, int H, int W, int radius, double sigma_s, int M,
                                  float *out, void *stream);

/* Smallest M with cos(u/(sigma_s sqrt M)) >= 0 for |u| <= radius:
 * ceil((2 radius/(pi sigma_s))^2); -1 for invalid arguments. */
int sf_spatial_mmin(int radius, double sigma_s);

/* The polynomial range kernel: the filter of sf_filter
 * with box spatial kernel and phi replaced by
 *   phi_p(t) = (1 - t^2 / (2 N sigma_r^2))^N,
 * p_N(t) = (1 - t^2/T^2)^N of PAPER.md:202 (order of shiftability 2N+1,
 * PAPER.md:204-205) in the Eq.(5) scaling p_N(t/sqrt N) -> exp(-t^2/T^2)
 * with T = sqrt(2) sigma_r (reading R17: the same Gaussian
 * limit exp(-t^2/(2 sigma_r^2)) as sf_filter's kernel).  Evaluated by
 * Algorithm 2 in fp64 with a Chebyshev basis of the 2N+1-dimensional shift
 * space (the monomial basis of the paper cancels catastrophically; DESIGN.md
 * §8).  Requires N >= sf_nmin_poly(sigma_r) (phi_p >= 0 on [-255, 255]) and
 * N <= SF_MAX_POLY_ORDER (SF_ERR_ORDER), radius <= SF_MAX_POLY_RADIUS
 * (SF_ERR_RADIUS).  img/out: device, H*W.  Synchronises `stream` once (to
 * upload its coefficient table), then runs asynchronously on it. */
#define SF_MAX_POLY_ORDER 512
#define SF_MAX_POLY_RADIUS 32
sf_status sf_filter_poly(const uint8_t *img, int H, int W, int radius, double sigma_r, int N,
                         float *out, void *stream);

/* Smallest valid order of phi_p: ceil(255^2 / (2 sigma_r^2)); -1 for invalid sigma_r. */
int sf_nmin_poly(double sigma_r);

/* Number of conjugate pairs, floor(N/2)+1. */
int sf_pair_count(int N);

/* Smallest valid order N0 = ceil((2*255/(pi sigma_r))^2) (reading R2). */
int sf_nmin(double sigma_r);

/* Number of kernel launches the last successful call on this thread enqueued
 * (for bench accounting). */
int sf_last_launch_count(void);   /* thread-local */

const char *sf_status_string(sf_status s);

#ifdef __cplusplus
}
#endif

#endif /* SF_H */
