/*
 * oracle/sf_oracle.c — fp64 CPU oracle for the constant-time bilateral filter
 * with shiftable kernels (Chaudhury, arxiv 1107.4617).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * in paper_1107_4617_b200/ (and never includes anything from there).
 *
 * Citations are PAPER.md line numbers ("PAPER.md:L") in /root/reference, with
 * the equation/algorithm they fall in.  Readings of silent/garbled passages
 * are the numbered readings R1.. of DESIGN.md §3.
 *
 *   Range kernel (R1): phi(t) = cos(gamma t)^N, gamma = 1/(sigma_r sqrt N)
 *     = q_N(t/sqrt N) of PAPER.md:202 rescaled so that the Eq.(6) limit
 *      is exp(-t^2/(2 sigma_r^2)).
 *   Shiftable expansion, Eq.(1):
 *     cos(gamma t)^N = ((e^{j gamma t}+e^{-j gamma t})/2)^N
 *                    = sum_{n=0..N} c_n e^{j omega_n t},
 *     c_n = C(N,n)/2^N, omega_n = (2n-N) gamma          (order N+1)
 *   so phi(t - tau) = sum_n d_n(tau) phi_n(t) with
 *     d_n(tau) = c_n e^{-j omega_n tau}, phi_n(t) = e^{j omega_n t}.
 *   Spatial kernel: box (M=1, c_1=1, phi_1=1) or (R5) the separable raised
 *     cosine w(y)=w1(y1)w1(y2), w1(u) = (1+cos(alpha u))/2 = q_2(u) with
 *     T=r+1, alpha = pi/(r+1); per axis
 *     w1(u - tau) = sum_{s in {0,+1,-1}} b_s e^{-j s alpha tau} e^{j s alpha u},
 *     b_0 = 1/2, b_{+-1} = 1/4  (order 3 per axis, M = 3^2 as PAPER.md:168).
 *   Boundary (R3): f is extended by whole-sample symmetric reflection
 *     ("reflect-101": -i -> i, (L-1)+i -> (L-1)-i); requires r <= min(H,W)-1.
 *   Window (R4): the moving sum Sum(F,x,T) of PAPER.md:98-103 over the
 *     inclusive square [-r,r]^2 (T = r).
 *
 * Two implementations:
 *   oracle_bilateral_direct    — Eq.(3) as a literal
 *                                double loop (O1, brute force).
 *   oracle_bilateral_shiftable — Algorithm 2 step by step:
 *                                step 1 the images a_{m,n}, g_{m,n}, h_{m,n};
 *                                step 2 their moving sums "using recursion"
 *                                (running sums); step 3 the ratio.
 *                                All N+1 complex terms, no pairing, no truncation.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_T 255.0            /* range half-width for uint8 data (R2) */
#define ORACLE_PI 3.14159265358979323846

enum { OR_OK = 0, OR_ERR_ARG = 1, OR_ERR_NOMEM = 2 };

/* ---------------------------------------------------------------- kernels */

/* Eq.(1) coefficients of the raised-cosine range kernel (see header).
 * c_n by the exact product recursion c_0 = 2^-N, c_{n+1} = c_n (N-n)/(n+1)
 * in long double (exact binomials, no overflow for large N). */
int oracle_expansion(int N, double sigma_r, double *omega, double *c)
{
    if (N < 0 || !(sigma_r > 0.0) || !omega || !c) return OR_ERR_ARG;
    double gamma = (N > 0) ? 1.0 / (sigma_r * sqrt((double)N)) : 0.0;
    long double cn = ldexpl(1.0L, -N);
    for (int n = 0; n <= N; ++n) {
        omega[n] = (double)(2 * n - N) * gamma;
        c[n] = (double)cn;
        cn = cn * (long double)(N - n) / (long double)(n + 1);
    }
    return OR_OK;
}

/* phi(t) = cos(t/(sigma_r sqrt N))^N  (R1; q_N of PAPER.md:202 rescaled). */
double oracle_range_kernel(double t, double sigma_r, int N)
{
    if (N == 0) return 1.0;
    return pow(cos(t / (sigma_r * sqrt((double)N))), (double)N);
}

/* Truncated expansion: "discarding the less significant
 * basis functions in (def)".  The n0 smallest-weight terms
 * at each end of Eq.(1) are dropped; the kept set n0..N-n0 is symmetric, so
 *   phi_eps(t) = sum_{n=n0}^{N-n0} c_n e^{j omega_n t} = sum_{n=n0}^{N-n0} c_n cos(omega_n t)
 * (written out term by term, fp64). */
double oracle_range_kernel_truncated(double t, double sigma_r, int N, int n0)
{
    if (N == 0) return 1.0;
    const double gamma = 1.0 / (sigma_r * sqrt((double)N));
    long double cn = ldexpl(1.0L, -N);
    double s = 0.0;
    for (int n = 0; n <= N; ++n) {
        if (n >= n0 && n <= N - n0) s += (double)cn * cos((double)(2 * n - N) * gamma * t);
        cn = cn * (long double)(N - n) / (long double)(n + 1);
    }
    return s;
}

/* Terms dropped per end for threshold eps (reading R12): the smallest n0 with
 * c_{n0} >= eps * max_n c_n (c_n = C(N,n)/2^N is unimodal and symmetric). */
int oracle_truncation_n0(int N, double eps)
{
    if (N < 0 || !(eps >= 0.0)) return -1;
    long double cmax = 1.0L, c = 1.0L;            /* ratios to c_0: C(N,n) */
    for (int n = 0; n < N / 2; ++n) cmax = cmax * (long double)(N - n) / (long double)(n + 1);
    int n0 = 0;
    while (n0 < N / 2 && c < (long double)eps * cmax) {
        c = c * (long double)(N - n0) / (long double)(n0 + 1);
        ++n0;
    }
    return n0;
}

/* f3, the polynomial range kernel: p_N(t) = (1 -
 * t^2/T^2)^N of PAPER.md:202, order of shiftability 2N+1,
 * in the scaling of Eq.(5), p_N(t/sqrt N) -> exp(-t^2/T^2);
 * reading R17 takes T = sqrt(2) sigma_r, so that the limit is the same
 * Gaussian exp(-t^2/(2 sigma_r^2)) as the raised cosine's (R1):
 *   phi_p(t) = (1 - t^2/(2 N sigma_r^2))^N. */
double oracle_range_kernel_poly(double t, double sigma_r, int N)
{
    if (N == 0) return 1.0;
    return pow(1.0 - t * t / (2.0 * (double)N * sigma_r * sigma_r), (double)N);
}

/* Smallest N for which phi_p is a valid kernel on [-T, T], T = 255 (R2, R17):
 * 1 - t^2/(2 N sigma_r^2) >= 0 for |t| <= 255, N >= 255^2/(2 sigma_r^2). */
int oracle_nmin_poly(double sigma_r)
{
    double q = ORACLE_T * ORACLE_T / (2.0 * sigma_r * sigma_r);
    int n = (int)ceil(q - 1e-12);
    return n < 1 ? 1 : n;
}

/* Gaussian target of Eq.(6) in the sigma_r scaling (R1). */
double oracle_gaussian_kernel(double t, double sigma_r)
{
    return exp(-t * t / (2.0 * sigma_r * sigma_r));
}

/* Smallest valid order (R2): cos argument within [-pi/2, pi/2] on [-T, T],
 * N0 = ceil((2T/(pi sigma_r))^2), "of the order O(T^2/sigma^2)" PAPER.md:278. */
int oracle_nmin(double sigma_r)
{
    double q = 2.0 * ORACLE_T / (ORACLE_PI * sigma_r);
    int n = (int)ceil(q * q - 1e-12);
    return n < 1 ? 1 : n;
}

/* Order of the raised-cosine spatial kernel for a spatial kind: kind 1 is q_2
 * (reading R5); kind 100+M is q_M, M = 1..16 (the general
 * separable shiftable kernels of PAPER.md:202, 210-212); box (kind 0) -> 0. */
static int spatial_order(int kind)
{
    if (kind == 1) return 2;
    if (kind >= 101 && kind <= 116) return kind - 100;
    return 0;
}

/* One-axis spatial weight w1(u) for |u| <= r: box 1; q_M(u) = cos(pi u/(2T))^M
 * with T = r+1, so that the kernel is positive on [-r, r]
 * (kind 1: q_2 = (1 + cos(pi u/(r+1)))/2, reading R5). */
double oracle_spatial_weight(int u, int radius, int kind)
{
    if (u < -radius || u > radius) return 0.0;
    if (kind == 0) return 1.0;
    if (kind == 1) return 0.5 * (1.0 + cos(ORACLE_PI * (double)u / (double)(radius + 1)));
    return pow(cos(ORACLE_PI * (double)u / (2.0 * (double)(radius + 1))), (double)spatial_order(kind));
}

/* The same family with the frequency beta given (f2, Gaussian-fitted spatial
 * kernel): w1(u) = cos(beta u)^M on |u| <= r, M = spatial_order(kind).  Eq.(7)
 * (exponent pi^2 by reading R10): q_M(u/sqrt M) with
 * T = pi sigma_s / 2 tends to exp(-u^2/(2 sigma_s^2)), i.e. beta =
 * pi/(2 T sqrt M) = 1/(sigma_s sqrt M) (reading R18).  beta <= 0: the
 * default T = r + 1 (beta = pi/(2(r+1))). */
double oracle_spatial_weight_beta(int u, int radius, int kind, double beta)
{
    if (beta <= 0.0) return oracle_spatial_weight(u, radius, kind);
    if (u < -radius || u > radius) return 0.0;
    if (kind == 0) return 1.0;
    return pow(cos(beta * (double)u), (double)spatial_order(kind));
}

/* Smallest spatial order M with cos(u/(sigma_s sqrt M)) >= 0 on |u| <= r
 * (R18): r/(sigma_s sqrt M) <= pi/2, M >= (2r/(pi sigma_s))^2. */
int oracle_spatial_mmin(int radius, double sigma_s)
{
    double q = 2.0 * (double)radius / (ORACLE_PI * sigma_s);
    int m = (int)ceil(q * q - 1e-12);
    return m < 1 ? 1 : m;
}

/* whole-sample symmetric reflection (R3) */
static int reflect101(int p, int L)
{
    if (L == 1) return 0;
    while (p < 0 || p >= L) {
        if (p < 0) p = -p;
        if (p >= L) p = 2 * (L - 1) - p;
    }
    return p;
}

static int check_args(const uint8_t *img, int H, int W, int radius, int kind)
{
    if (!img || H < 1 || W < 1 || radius < 0) return OR_ERR_ARG;
    if (radius > (H < W ? H : W) - 1) return OR_ERR_ARG;
    if (kind != 0 && kind != 1 && spatial_order(kind) == 0) return OR_ERR_ARG;
    return OR_OK;
}

/* ------------------------------------------------------ moving sum (real) */

/* Sum(F, x, T) of PAPER.md:98-103 on the reflect-101-extended F, computed by
 * recursion (running sums, "using recursion" PAPER.md:103): a horizontal pass
 * then a vertical pass, each re-initialised per row / column. */
int oracle_moving_sum(const double *F, int H, int W, int radius, double *out)
{
    if (!F || !out || H < 1 || W < 1 || radius < 0) return OR_ERR_ARG;
    if (radius > (H < W ? H : W) - 1) return OR_ERR_ARG;
    const int R = radius, L = 2 * R + 1;
    double *hs = (double *)malloc(sizeof(double) * (size_t)H * W);
    double *line = (double *)malloc(sizeof(double) * (size_t)((H > W ? H : W) + 2 * R));
    if (!hs || !line) { free(hs); free(line); return OR_ERR_NOMEM; }
    for (int y = 0; y < H; ++y) {                     /* horizontal */
        for (int p = -R; p < W + R; ++p) line[p + R] = F[(size_t)y * W + reflect101(p, W)];
        double s = 0.0;
        for (int i = 0; i < L; ++i) s += line[i];
        hs[(size_t)y * W] = s;
        for (int x = 1; x < W; ++x) { s += line[x + 2 * R] - line[x - 1]; hs[(size_t)y * W + x] = s; }
    }
    for (int x = 0; x < W; ++x) {                     /* vertical */
        for (int p = -R; p < H + R; ++p) line[p + R] = hs[(size_t)reflect101(p, H) * W + x];
        double s = 0.0;
        for (int i = 0; i < L; ++i) s += line[i];
        out[x] = s;
        for (int y = 1; y < H; ++y) { s += line[y + 2 * R] - line[y - 1]; out[(size_t)y * W + x] = s; }
    }
    free(hs); free(line);
    return OR_OK;
}

/* ----------------------------------------------------- O1: brute force Eq.(3) */

/* Eq.(3), literally:
 *   f~(x) = sum_y w(y) phi(f(x-y)-f(x)) f(x-y) / sum_y w(y) phi(f(x-y)-f(x))
 * over y in [-r,r]^2 with reflect-101 f.  range_kind 0: raised cosine
 * (sigma_r, N); range_kind 2: its expansion truncated to terms n0..N-n0;
 * range_kind 1: Gaussian exp(-t^2/2sigma_r^2) (for the Eq.(6)
 * convergence pin); range_kind 3: the polynomial kernel phi_p (f3).  idx: flat pixel indices y*W+x to evaluate (n_idx of
 * them), or NULL for every pixel in row-major order.  num/den may be NULL. */
int oracle_bilateral_direct_ex3(const uint8_t *img, int H, int W, int radius, int kind,
                                double sigma_r, int N, int range_kind, int n0,
                                const int64_t *idx, int64_t n_idx,
                                double *out, double *num, double *den, int nthreads, double beta);

int oracle_bilateral_direct_ex2(const uint8_t *img, int H, int W, int radius, int kind,
                                double sigma_r, int N, int range_kind, int n0,
                                const int64_t *idx, int64_t n_idx,
                                double *out, double *num, double *den, int nthreads)
{
    return oracle_bilateral_direct_ex3(img, H, W, radius, kind, sigma_r, N, range_kind, n0, idx, n_idx,
                                       out, num, den, nthreads, 0.0);
}

/* ex3: with the spatial frequency beta of oracle_spatial_weight_beta */
int oracle_bilateral_direct_ex3(const uint8_t *img, int H, int W, int radius, int kind,
                                double sigma_r, int N, int range_kind, int n0,
                                const int64_t *idx, int64_t n_idx,
                                double *out, double *num, double *den, int nthreads, double beta)
{
    int e = check_args(img, H, W, radius, kind);
    if (e) return e;
    if (!out || !(sigma_r > 0.0) || N < 0) return OR_ERR_ARG;
    const int R = radius;
    int64_t count = idx ? n_idx : (int64_t)H * W;
    double *w1 = (double *)malloc(sizeof(double) * (2 * R + 1));
    double phi_tab[511];
    if (!w1) return OR_ERR_NOMEM;
    for (int u = -R; u <= R; ++u) w1[u + R] = oracle_spatial_weight_beta(u, R, kind, beta);
    for (int t = -255; t <= 255; ++t)      /* phi at the 511 possible differences */
        phi_tab[t + 255] = range_kind == 0 ? oracle_range_kernel((double)t, sigma_r, N)
                         : range_kind == 1 ? oracle_gaussian_kernel((double)t, sigma_r)
                         : range_kind == 3 ? oracle_range_kernel_poly((double)t, sigma_r, N)
                                           : oracle_range_kernel_truncated((double)t, sigma_r, N, n0);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
    for (int64_t i = 0; i < count; ++i) {
        int64_t p = idx ? idx[i] : i;
        int y = (int)(p / W), x = (int)(p % W);
        double fx = img[p];
        double sn = 0.0, sd = 0.0;
        for (int dy = -R; dy <= R; ++dy) {
            const uint8_t *row = img + (size_t)reflect101(y - dy, H) * W;
            for (int dx = -R; dx <= R; ++dx) {
                double fy = row[reflect101(x - dx, W)];
                double wgt = w1[dy + R] * w1[dx + R] * phi_tab[(int)(fy - fx) + 255];
                sn += wgt * fy;
                sd += wgt;
            }
        }
        out[i] = sn / sd;
        if (num) num[i] = sn;
        if (den) den[i] = sd;
    }
    free(w1);
    return OR_OK;
}

int oracle_bilateral_direct_ex(const uint8_t *img, int H, int W, int radius, int kind,
                               double sigma_r, int N, int range_kind,
                               const int64_t *idx, int64_t n_idx,
                               double *out, double *num, double *den, int nthreads)
{
    return oracle_bilateral_direct_ex2(img, H, W, radius, kind, sigma_r, N, range_kind, 0, idx, n_idx,
                                       out, num, den, nthreads);
}

int oracle_bilateral_direct(const uint8_t *img, int H, int W, int radius, int kind,
                            double sigma_r, int N, const int64_t *idx, int64_t n_idx,
                            double *out, int nthreads)
{
    return oracle_bilateral_direct_ex(img, H, W, radius, kind, sigma_r, N, 0, idx, n_idx,
                                      out, NULL, NULL, nthreads);
}

/* ------------------------------------------- O2: Algorithm 2, step by step */

/* Algorithm 2 for output rows [row_begin,row_end) and
 * range terms n in [n_begin,n_end) of 0..N, all spatial terms m.
 *   step 1: a_{m,n}(x) = c_m(x) d_n(f(x)),
 *           g_{m,n}(x) = phi_m(x) phi_n(f(x)) f(x),  h_{m,n}(x) = phi_m(x) phi_n(f(x))
 *   step 2: Sum(g_{m,n},x,T), Sum(h_{m,n},x,T) by recursion (running sums)
 *   step 3: num = sum_{m,n} a Sum(g), den = sum_{m,n} a Sum(h), f~ = num/den.
 * Images are complex fp64; the moving sums run on the padded (reflect-101)
 * band so that every window has (2r+1)^2 samples.  Coordinates of phi_m are
 * absolute pixel indices (row, col) — the origin is arbitrary by shiftability.
 * Outputs (row-major, (row_end-row_begin) x W): num/den = real parts of the
 * partial sums over the term range (may be NULL), out = num/den (may be NULL).
 * Work is split over row bands (OpenMP); the arithmetic per pixel is the
 * same whatever the thread count. */
int oracle_bilateral_shiftable_ex(const uint8_t *img, int H, int W, int radius, int kind,
                                  double sigma_r, int N, int n_begin, int n_end,
                                  int row_begin, int row_end,
                                  double *num, double *den, double *out, int nthreads, double beta);

int oracle_bilateral_shiftable(const uint8_t *img, int H, int W, int radius, int kind,
                               double sigma_r, int N, int n_begin, int n_end,
                               int row_begin, int row_end,
                               double *num, double *den, double *out, int nthreads)
{
    return oracle_bilateral_shiftable_ex(img, H, W, radius, kind, sigma_r, N, n_begin, n_end, row_begin, row_end,
                                         num, den, out, nthreads, 0.0);
}

/* _ex: with the spatial frequency beta of oracle_spatial_weight_beta (the
 * spatial expansion's frequencies s_m beta, same weights C(M,m)/2^M) */
int oracle_bilateral_shiftable_ex(const uint8_t *img, int H, int W, int radius, int kind,
                                  double sigma_r, int N, int n_begin, int n_end,
                                  int row_begin, int row_end,
                                  double *num, double *den, double *out, int nthreads, double beta)
{
    int e = check_args(img, H, W, radius, kind);
    if (e) return e;
    if (!(sigma_r > 0.0) || N < 0) return OR_ERR_ARG;
    if (n_begin < 0 || n_end > N + 1 || n_begin > n_end) return OR_ERR_ARG;
    if (row_begin < 0 || row_end > H || row_begin > row_end) return OR_ERR_ARG;
    const int R = radius, rows = row_end - row_begin;
    if (rows == 0) return OR_OK;

    double *omega = (double *)malloc(sizeof(double) * (N + 1));
    double *cn = (double *)malloc(sizeof(double) * (N + 1));
    if (!omega || !cn) { free(omega); free(cn); return OR_ERR_NOMEM; }
    oracle_expansion(N, sigma_r, omega, cn);

    /* spatial expansion per axis (Eq.(1) applied to q_M):
     *   q_M(u - tau) = sum_{m=0}^{M} C(M,m)/2^M e^{-j s_m beta tau} e^{j s_m beta u},
     *   s_m = 2m - M, beta = pi/(2(r+1));  box: one term s = 0, b = 1.
     * (q_2: s in {-2,0,2} beta = {-1,0,1} pi/(r+1), b = {1/4,1/2,1/4}, reading R5.) */
    const int MO = spatial_order(kind);
    const int M1 = (kind == 0) ? 1 : MO + 1;
    double s_m[17], b_m[17];
    for (int m = 0; m < M1; ++m) {
        s_m[m] = (kind == 0) ? 0.0 : (double)(2 * m - MO);
        long double b = ldexpl(1.0L, -MO);
        for (int i = 0; i < m; ++i) b = b * (long double)(MO - i) / (long double)(i + 1);
        b_m[m] = (kind == 0) ? 1.0 : (double)b;
    }
    const double alpha = beta > 0.0 ? beta : ORACLE_PI / (2.0 * (double)(R + 1));   /* beta */

    const int BAND = 32;
    const int nbands = (rows + BAND - 1) / BAND;
    int status = OR_OK;

#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        const int PW = W + 2 * R;                 /* padded width            */
        const int PH = BAND + 2 * R;              /* padded band height      */
        double complex *g = malloc(sizeof(double complex) * (size_t)PH * PW);
        double complex *h = malloc(sizeof(double complex) * (size_t)PH * PW);
        double complex *gs = malloc(sizeof(double complex) * (size_t)PH * W);  /* horiz sums */
        double complex *hs = malloc(sizeof(double complex) * (size_t)PH * W);
        double complex *Sg = malloc(sizeof(double complex) * (size_t)BAND * W); /* Sum(g) */
        double complex *Sh = malloc(sizeof(double complex) * (size_t)BAND * W); /* Sum(h) */
        double complex *an = malloc(sizeof(double complex) * (size_t)BAND * W); /* num acc */
        double complex *ad = malloc(sizeof(double complex) * (size_t)BAND * W); /* den acc */
        double *fpad = malloc(sizeof(double) * (size_t)PH * PW);
        double complex lut[256];
        double complex *ecol = malloc(sizeof(double complex) * (size_t)PW);  /* phi_m column factor */
        double complex *ccol = malloc(sizeof(double complex) * (size_t)W);   /* c_m column factor   */
        int ok = g && h && gs && hs && Sg && Sh && an && ad && fpad && ecol && ccol;
        if (!ok) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            status = OR_ERR_NOMEM;
        }
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int b = 0; b < nbands; ++b) {
            if (!ok) continue;
            const int y0 = row_begin + b * BAND;
            const int nb = (y0 + BAND <= row_end) ? BAND : row_end - y0;
            const int ph = nb + 2 * R;
            /* f on the padded band: padded (i,j) <-> absolute (y0-R+i, j-R) */
            for (int i = 0; i < ph; ++i) {
                const uint8_t *row = img + (size_t)reflect101(y0 - R + i, H) * W;
                for (int j = 0; j < PW; ++j) fpad[(size_t)i * PW + j] = row[reflect101(j - R, W)];
            }
            for (size_t q = 0; q < (size_t)nb * W; ++q) an[q] = ad[q] = 0.0;

            for (int m1 = 0; m1 < M1; ++m1)          /* spatial term, row axis    */
            for (int m2 = 0; m2 < M1; ++m2)          /* spatial term, column axis */
            for (int n = n_begin; n < n_end; ++n) {  /* range term                */
                /* memoised per-axis factors of phi_m and c_m (same values as
                   evaluating e^{j s alpha p} at each pixel) */
                for (int j = 0; j < PW; ++j) ecol[j] = cexp(I * s_m[m2] * alpha * (double)(j - R));
                for (int x = 0; x < W; ++x) ccol[x] = b_m[m2] * cexp(-I * s_m[m2] * alpha * (double)x);
                /* phi_n(v) = e^{j omega_n v} for the 256 possible values v */
                for (int v = 0; v < 256; ++v) lut[v] = cexp(I * omega[n] * (double)v);
                /* step 1: g_{m,n}, h_{m,n} on the padded band */
                for (int i = 0; i < ph; ++i) {
                    const double prow = (double)(y0 - R + i);
                    const double complex er = cexp(I * s_m[m1] * alpha * prow);
                    for (int j = 0; j < PW; ++j) {
                        const double complex phim = er * ecol[j];
                        const double fv = fpad[(size_t)i * PW + j];
                        const double complex hv = phim * lut[(int)fv];
                        h[(size_t)i * PW + j] = hv;
                        g[(size_t)i * PW + j] = hv * fv;
                    }
                }
                /* step 2: moving sums by recursion — horizontal then vertical */
                for (int i = 0; i < ph; ++i) {
                    const double complex *gr = g + (size_t)i * PW, *hr = h + (size_t)i * PW;
                    double complex sg = 0.0, sh = 0.0;
                    for (int k = 0; k < 2 * R + 1; ++k) { sg += gr[k]; sh += hr[k]; }
                    gs[(size_t)i * W] = sg; hs[(size_t)i * W] = sh;
                    for (int x = 1; x < W; ++x) {
                        sg += gr[x + 2 * R] - gr[x - 1];
                        sh += hr[x + 2 * R] - hr[x - 1];
                        gs[(size_t)i * W + x] = sg; hs[(size_t)i * W + x] = sh;
                    }
                }
                for (int x = 0; x < W; ++x) {
                    double complex sg = 0.0, sh = 0.0;
                    for (int k = 0; k < 2 * R + 1; ++k) { sg += gs[(size_t)k * W + x]; sh += hs[(size_t)k * W + x]; }
                    Sg[x] = sg; Sh[x] = sh;
                    for (int yy = 1; yy < nb; ++yy) {
                        sg += gs[(size_t)(yy + 2 * R) * W + x] - gs[(size_t)(yy - 1) * W + x];
                        sh += hs[(size_t)(yy + 2 * R) * W + x] - hs[(size_t)(yy - 1) * W + x];
                        Sg[(size_t)yy * W + x] = sg; Sh[(size_t)yy * W + x] = sh;
                    }
                }
                /* step 3 (accumulation): a_{m,n}(x) = c_m(x) d_n(f(x)) */
                for (int yy = 0; yy < nb; ++yy) {
                    const double xr = (double)(y0 + yy);
                    const double complex cr = b_m[m1] * cexp(-I * s_m[m1] * alpha * xr);
                    for (int x = 0; x < W; ++x) {
                        const double complex cm = cr * ccol[x];
                        const double fx = fpad[(size_t)(yy + R) * PW + (x + R)];
                        /* d_n(f(x)) = c_n e^{-j omega_n f(x)} = c_n conj(phi_n(f(x))) */
                        const double complex a = cm * cn[n] * conj(lut[(int)fx]);
                        an[(size_t)yy * W + x] += a * Sg[(size_t)yy * W + x];
                        ad[(size_t)yy * W + x] += a * Sh[(size_t)yy * W + x];
                    }
                }
            }
            /* step 3 (ratio) */
            for (int yy = 0; yy < nb; ++yy)
                for (int x = 0; x < W; ++x) {
                    size_t q = (size_t)yy * W + x, o = (size_t)(y0 - row_begin + yy) * W + x;
                    double nv = creal(an[q]), dv = creal(ad[q]);
                    if (num) num[o] = nv;
                    if (den) den[o] = dv;
                    if (out) out[o] = nv / dv;
                }
        }
        free(g); free(h); free(gs); free(hs); free(Sg); free(Sh); free(an); free(ad); free(fpad);
        free(ecol); free(ccol);
    }
    free(omega); free(cn);
    return status;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------ f4: shiftable non-local means, tiny p */

/* Non-local means (Eq.(NL)) with the inner patch sum over p
 * offsets u_1 = (0,0), u_2 = (0,1), u_3 = (1,0) (reading R14) and the outer
 * integral over the square [-r, r]^2 (Eq.(approx_multivariate)):
 *   f^(x) = sum_y f(x-y) phi(t_1..t_p) / sum_y phi(t_1..t_p),
 *   t_k = f(x+u_k) - f(x-y+u_k),
 *   phi(t) = prod_k psi_k(t_k) ~ exp(-h^-2 sum_k g(u_k) t_k^2),
 *   g(u) = exp(-|u|^2 / (2 rho^2)) (rho = 0: g(u) = [u = 0]),
 *   psi_k(t) = cos(gamma_k t)^n, gamma_k = sqrt(2 g(u_k) / (n h^2))
 * — the separable shiftable approximation "of order n^p"
 * built from the raised cosine of the range kernel (reading R1: cos(t/(s sqrt n))^n
 * with s_k = h / sqrt(2 g(u_k))).  f is reflect-101 extended. */
static void nlm_offsets(int k, int *dy, int *dx)
{
    *dy = (k == 2) ? 1 : 0;
    *dx = (k == 1) ? 1 : 0;
}

static double nlm_gamma(int k, double h, double rho, int n)
{
    int dy, dx;
    nlm_offsets(k, &dy, &dx);
    double d2 = (double)(dy * dy + dx * dx);
    double g = (d2 == 0.0) ? 1.0 : (rho > 0.0 ? exp(-d2 / (2.0 * rho * rho)) : 0.0);
    return sqrt(2.0 * g / ((double)n * h * h));
}

static int nlm_check(const uint8_t *img, int H, int W, int radius, int p, double h, double rho, int n)
{
    if (!img || H < 1 || W < 1 || radius < 0) return OR_ERR_ARG;
    if (radius > H - 1 || radius > W - 1) return OR_ERR_ARG;
    if (p < 1 || p > 3 || !(h > 0.0) || !(rho >= 0.0) || n < 1) return OR_ERR_ARG;
    return OR_OK;
}

/* O1: the definition, a literal double loop (brute force). */
int oracle_nlm_direct(const uint8_t *img, int H, int W, int radius, int p, double h, double rho,
                      int n, double *out, int nthreads)
{
    int e = nlm_check(img, H, W, radius, p, h, rho, n);
    if (e) return e;
    if (!out) return OR_ERR_ARG;
    double gam[3];
    for (int k = 0; k < p; ++k) gam[k] = nlm_gamma(k, h, rho, n);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (int64_t q = 0; q < (int64_t)H * W; ++q) {
        const int y = (int)(q / W), x = (int)(q % W);
        double sn = 0.0, sd = 0.0;
        for (int dy = -radius; dy <= radius; ++dy)
            for (int dx = -radius; dx <= radius; ++dx) {
                const int zy = y - dy, zx = x - dx;          /* neighbour x - y */
                double wgt = 1.0;
                for (int k = 0; k < p; ++k) {
                    int uy, ux;
                    nlm_offsets(k, &uy, &ux);
                    const double fc = img[(size_t)reflect101(y + uy, H) * W + reflect101(x + ux, W)];
                    const double fz = img[(size_t)reflect101(zy + uy, H) * W + reflect101(zx + ux, W)];
                    wgt *= pow(cos(gam[k] * (fc - fz)), (double)n);
                }
                const double fv = img[(size_t)reflect101(zy, H) * W + reflect101(zx, W)];
                sn += wgt * fv;
                sd += wgt;
            }
        out[q] = sn / sd;
    }
    return OR_OK;
}

/* O2: the paper's moving-sum algorithm, step by step, for
 * all (n+1)^p multi-indices m (no pairing):
 *   H_m(z) = prod_k e^{-j w_{k,m_k} f(z+u_k)},  G_m(z) = f(z) H_m(z),
 *   c_m(x) = prod_k C(n,m_k) 2^-n e^{+j w_{k,m_k} f(x+u_k)},  w_{k,m} = (2m-n) gamma_k,
 *   num(x) = sum_m c_m(x) Sum(G_m, x, r),  den(x) = sum_m c_m(x) Sum(H_m, x, r),
 * Sum = the moving sum over [-r,r]^2 (running sums, horizontal then vertical,
 * on the reflect-101 padded image); out = num / den. */
int oracle_nlm_shiftable(const uint8_t *img, int H, int W, int radius, int p, double h, double rho,
                         int n, double *out)
{
    int e = nlm_check(img, H, W, radius, p, h, rho, n);
    if (e) return e;
    if (!out) return OR_ERR_ARG;
    const int R = radius, PW = W + 2 * R, PH = H + 2 * R;
    double gam[3];
    for (int k = 0; k < p; ++k) gam[k] = nlm_gamma(k, h, rho, n);
    double *cn = malloc(sizeof(double) * (n + 1));
    double *fp = malloc(sizeof(double) * (size_t)PH * PW);
    double complex *Hm = malloc(sizeof(double complex) * (size_t)PH * PW);
    double complex *Gm = malloc(sizeof(double complex) * (size_t)PH * PW);
    double complex *hsH = malloc(sizeof(double complex) * (size_t)PH * W);
    double complex *hsG = malloc(sizeof(double complex) * (size_t)PH * W);
    double complex *num = malloc(sizeof(double complex) * (size_t)H * W);
    double complex *den = malloc(sizeof(double complex) * (size_t)H * W);
    if (!cn || !fp || !Hm || !Gm || !hsH || !hsG || !num || !den) {
        free(cn); free(fp); free(Hm); free(Gm); free(hsH); free(hsG); free(num); free(den);
        return OR_ERR_NOMEM;
    }
    long double c = ldexpl(1.0L, -n);
    for (int m = 0; m <= n; ++m) {
        cn[m] = (double)c;
        c = c * (long double)(n - m) / (long double)(m + 1);
    }
    /* padded image: padded (i,j) <-> absolute (i-R, j-R) */
    for (int i = 0; i < PH; ++i)
        for (int j = 0; j < PW; ++j)
            fp[(size_t)i * PW + j] = img[(size_t)reflect101(i - R, H) * W + reflect101(j - R, W)];
    for (size_t q = 0; q < (size_t)H * W; ++q) num[q] = den[q] = 0.0;
    int mi[3] = {0, 0, 0};
    int total = 1;
    for (int k = 0; k < p; ++k) total *= (n + 1);
    for (int t = 0; t < total; ++t) {
        int rem = t;
        for (int k = 0; k < p; ++k) { mi[k] = rem % (n + 1); rem /= (n + 1); }
        double wm[3];
        double cm = 1.0;
        for (int k = 0; k < p; ++k) { wm[k] = (2.0 * mi[k] - n) * gam[k]; cm *= cn[mi[k]]; }
        /* H_m, G_m on the padded image (neighbour values f(z+u_k), reflect-101) */
        for (int i = 0; i < PH; ++i)
            for (int j = 0; j < PW; ++j) {
                double ph = 0.0;
                for (int k = 0; k < p; ++k) {
                    int uy, ux;
                    nlm_offsets(k, &uy, &ux);
                    ph += wm[k] * (double)img[(size_t)reflect101(i - R + uy, H) * W + reflect101(j - R + ux, W)];
                }
                const double complex hz = cexp(-I * ph);
                Hm[(size_t)i * PW + j] = hz;
                Gm[(size_t)i * PW + j] = hz * fp[(size_t)i * PW + j];
            }
        /* moving sums by recursion: horizontal then vertical */
        for (int i = 0; i < PH; ++i) {
            double complex sh = 0.0, sg = 0.0;
            for (int j = 0; j < 2 * R + 1; ++j) { sh += Hm[(size_t)i * PW + j]; sg += Gm[(size_t)i * PW + j]; }
            hsH[(size_t)i * W] = sh; hsG[(size_t)i * W] = sg;
            for (int x = 1; x < W; ++x) {
                sh += Hm[(size_t)i * PW + x + 2 * R] - Hm[(size_t)i * PW + x - 1];
                sg += Gm[(size_t)i * PW + x + 2 * R] - Gm[(size_t)i * PW + x - 1];
                hsH[(size_t)i * W + x] = sh; hsG[(size_t)i * W + x] = sg;
            }
        }
        for (int x = 0; x < W; ++x) {
            double complex sh = 0.0, sg = 0.0;
            for (int i = 0; i < 2 * R + 1; ++i) { sh += hsH[(size_t)i * W + x]; sg += hsG[(size_t)i * W + x]; }
            for (int y = 0; y < H; ++y) {
                if (y > 0) {
                    sh += hsH[(size_t)(y + 2 * R) * W + x] - hsH[(size_t)(y - 1) * W + x];
                    sg += hsG[(size_t)(y + 2 * R) * W + x] - hsG[(size_t)(y - 1) * W + x];
                }
                /* c_m(x) = prod_k c_{m_k} e^{+j w_k f(x+u_k)} */
                double ph = 0.0;
                for (int k = 0; k < p; ++k) {
                    int uy, ux;
                    nlm_offsets(k, &uy, &ux);
                    ph += wm[k] * (double)img[(size_t)reflect101(y + uy, H) * W + reflect101(x + ux, W)];
                }
                const double complex a = cm * cexp(I * ph);
                num[(size_t)y * W + x] += a * sg;
                den[(size_t)y * W + x] += a * sh;
            }
        }
    }
    for (size_t q = 0; q < (size_t)H * W; ++q) out[q] = creal(num[q]) / creal(den[q]);
    free(cn); free(fp); free(Hm); free(Gm); free(hsH); free(hsG); free(num); free(den);
    return OR_OK;
}

/* ------------------------------ f3: Algorithm 2 with the polynomial kernel */

/* Coefficients of Eq.(1) for phi_p (R17) in the normalised variable
 * u = (f - 128)/128 (the paper's basis functions t^i of a polynomial kernel,
 * order 2N+1): with a = 128^2/(2 N sigma_r^2),
 *   phi_p(f_y - f_x) = (1 - a (u_y - u_x)^2)^N = sum_{i=0}^{2N} d_i(u_x) u_y^i,
 *   d_i(v) = sum_{j=ceil(i/2)}^{N} C(N,j) (-a)^j C(2j,i) (-v)^{2j-i}
 * (the binomial theorem twice), in long double. */
int oracle_poly_coeffs(int N, double sigma_r, double v, double *d)
{
    if (N < 0 || N > 2048 || !(sigma_r > 0.0) || !d) return OR_ERR_ARG;
    const long double a = N > 0 ? 128.0L * 128.0L / (2.0L * (long double)N * sigma_r * sigma_r) : 0.0L;
    long double acc[2 * 2048 + 1];
    for (int i = 0; i <= 2 * N; ++i) acc[i] = 0.0L;
    long double cnj = 1.0L;                          /* C(N, j)  */
    long double aj = 1.0L;                           /* (-a)^j   */
    for (int j = 0; j <= N; ++j) {
        long double c2ji = 1.0L;                     /* C(2j, i) */
        for (int i = 0; i <= 2 * j; ++i) {
            acc[i] += cnj * aj * c2ji * powl(-(long double)v, (long double)(2 * j - i));
            c2ji = c2ji * (long double)(2 * j - i) / (long double)(i + 1);
        }
        cnj = cnj * (long double)(N - j) / (long double)(j + 1);
        aj = -aj * a;
    }
    for (int i = 0; i <= 2 * N; ++i) d[i] = (double)acc[i];
    return OR_OK;
}

/* Algorithm 2 with phi_p and the box spatial kernel, step
 * by step: step 1 the images h_i = u^i and g_i = u^i f, i = 0..2N; step 2
 * their moving sums by recursion (oracle_moving_sum); step 3 num = sum_i
 * d_i(u_x) Sum(g_i), den = sum_i d_i(u_x) Sum(h_i), out = num/den.  fp64.
 * The terms d_i Sum(h_i) alternate in sign and grow like (1 + 4a)^N while
 * their sum is O(1): in fp64 the result is exact to ~1e-9 for small N and
 * degrades for large N (tests/test_oracle_pins.py pins both). */
int oracle_bilateral_poly_shiftable(const uint8_t *img, int H, int W, int radius, double sigma_r, int N,
                                    double *out)
{
    int e = check_args(img, H, W, radius, 0);
    if (e) return e;
    if (!out || !(sigma_r > 0.0) || N < 0 || N > 2048) return OR_ERR_ARG;
    const size_t n = (size_t)H * W;
    const int K = 2 * N + 1;
    double *dtab = (double *)malloc(sizeof(double) * 256 * (size_t)K);
    double *hi = (double *)malloc(sizeof(double) * n), *gi = (double *)malloc(sizeof(double) * n);
    double *sh = (double *)malloc(sizeof(double) * n), *sg = (double *)malloc(sizeof(double) * n);
    double *num = (double *)calloc(n, sizeof(double)), *den = (double *)calloc(n, sizeof(double));
    if (!dtab || !hi || !gi || !sh || !sg || !num || !den) {
        free(dtab); free(hi); free(gi); free(sh); free(sg); free(num); free(den);
        return OR_ERR_NOMEM;
    }
    for (int v = 0; v < 256; ++v) oracle_poly_coeffs(N, sigma_r, ((double)v - 128.0) / 128.0, dtab + (size_t)v * K);
    for (size_t q = 0; q < n; ++q) hi[q] = 1.0;                 /* u^0 */
    for (int i = 0; i < K && e == OR_OK; ++i) {
        for (size_t q = 0; q < n; ++q) gi[q] = hi[q] * (double)img[q];
        e = oracle_moving_sum(hi, H, W, radius, sh);
        if (e == OR_OK) e = oracle_moving_sum(gi, H, W, radius, sg);
        for (size_t q = 0; q < n && e == OR_OK; ++q) {
            const double di = dtab[(size_t)img[q] * K + i];
            num[q] += di * sg[q];
            den[q] += di * sh[q];
        }
        for (size_t q = 0; q < n; ++q) hi[q] *= ((double)img[q] - 128.0) / 128.0;   /* u^{i+1} */
    }
    for (size_t q = 0; q < n && e == OR_OK; ++q) out[q] = num[q] / den[q];
    free(dtab); free(hi); free(gi); free(sh); free(sg); free(num); free(den);
    return e;
}
