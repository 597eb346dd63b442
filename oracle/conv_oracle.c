/*
 * CPU restatement of the reference's convolution semantics -- TEST
 * INFRASTRUCTURE (the checker and the timed CPU baseline), never a product
 * code path.  See oracle/conv_oracle.py for the numpy twin and the citations:
 *
 *   direct:   left-deep sum in (c, ky, kx) order over a zero-padded input
 *             (reference pkg/src/convio/dag.py:270-284, model.py:65-70)
 *   winograd: P = B^T d B, J = G g G^T per channel (step 1), P.J (step 2),
 *             left-deep channel sum (step 3), A^T Pi A (step 4)
 *             (dag.py:343-401); ragged outputs computed on the e-padded
 *             domain and cropped (dag.py:291-299)
 *
 * Inputs are fp32 (what the GPU path consumes); products and sums are fp64.
 * Threads: OpenMP over (image, output channel) pairs -- every output is
 * still accumulated by one thread in the fixed (c, ky, kx) order, so the
 * result is independent of the thread count.
 */
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 0;

int oracle_set_threads(int n) {
    g_threads = n;
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* x: [n, c, h, w] fp32; wt: [k, c, kh, kw] fp32; y: [n, k, p, q] fp64
 *
 * Register-blocked: a task owns OB output channels x one output row; for each
 * XB-wide column block the OB x XB accumulators stay in registers while the
 * (c, ky, kx) terms stream in that fixed order, every output's sum still
 * left-deep in the DAG order.  The input is copied once, zero-padded, so the
 * padding taps are real "+ 0 * w" terms as in the DAG over the padded input
 * (fp64 products of fp32 values are exact, so the result is bit-identical to
 * a scalar (c, ky, kx) loop and independent of the blocking and thread count).
 */
#define OB 6
#define XB 8
typedef double v4d __attribute__((vector_size(32)));

/* one XB-wide block of OB output rows; S = stride (1 and 2 compile-time) */
static inline __attribute__((always_inline)) void dc_block(const float *xc0, const double *wk, int c, int taps,
                                                          int kw, size_t plane, int wp, int S,
                                                          v4d acc[OB][XB / 4]) {
    for (int o = 0; o < OB; ++o)
        for (int j = 0; j < XB / 4; ++j) acc[o][j] = (v4d){0.0, 0.0, 0.0, 0.0};
    for (int ci = 0; ci < c; ++ci) {
        const float *xc = xc0 + (size_t)ci * plane;
        const double *wc = wk + (size_t)ci * taps * OB;
        for (int t = 0; t < taps; ++t) {
            const int ky = t / kw, kx = t - ky * kw;
            const float *xr = xc + (size_t)ky * wp + kx;
            v4d xv[XB / 4];
            for (int j = 0; j < XB / 4; ++j)
                xv[j] = (v4d){(double)xr[(4 * j) * S], (double)xr[(4 * j + 1) * S], (double)xr[(4 * j + 2) * S],
                              (double)xr[(4 * j + 3) * S]};
            for (int o = 0; o < OB; ++o) {
                const double wv = wc[t * OB + o];
                const v4d wb = {wv, wv, wv, wv};
                for (int j = 0; j < XB / 4; ++j) acc[o][j] += xv[j] * wb;
            }
        }
    }
}

int oracle_direct_conv_f32in(const float *x, const float *wt, double *y,
                             int n, int c, int h, int w, int k, int kh, int kw,
                             int stride, int pad, int reserved) {
    (void)reserved;
    if (n < 0 || c < 1 || h < 1 || w < 1 || k < 1 || kh < 1 || kw < 1 || stride < 1 || pad < 0)
        return 2;
    const int hp = h + 2 * pad, wp = w + 2 * pad;
    if (kh > hp || kw > wp) return 3;
    const int p = (hp - kh) / stride + 1, q = (wp - kw) / stride + 1;
    if (n == 0) return 0;
    /* zero-padded copy; XB*stride floats of slack past the end for the last
       column block's don't-care reads */
    const size_t plane = (size_t)hp * wp;
    float *xp = (float *)calloc((size_t)n * c * plane + (size_t)XB * stride + 64, sizeof(float));
    if (!xp) return 4;
#pragma omp parallel for schedule(static)
    for (long bc = 0; bc < (long)n * c; ++bc)
        for (int iy = 0; iy < h; ++iy)
            memcpy(xp + bc * plane + (size_t)(iy + pad) * wp + pad, x + (bc * h + iy) * (long)w,
                   sizeof(float) * (size_t)w);
    const int kbl = (k + OB - 1) / OB;
    const long tasks = (long)n * kbl * p;
    const int taps = kh * kw;
    /* filters as fp64 [k block][c][tap][OB] (missing channels of a ragged block: 0) */
    double *wk = (double *)calloc((size_t)kbl * c * taps * OB, sizeof(double));
    if (!wk) {
        free(xp);
        return 4;
    }
#pragma omp parallel for schedule(static)
    for (int oc = 0; oc < k; ++oc)
        for (int ci = 0; ci < c; ++ci)
            for (int t = 0; t < taps; ++t)
                wk[(((size_t)(oc / OB) * c + ci) * taps + t) * OB + oc % OB] =
                    (double)wt[((size_t)oc * c + ci) * taps + t];
#pragma omp parallel for schedule(dynamic, 4)
    for (long tk = 0; tk < tasks; ++tk) {
        const int oy = (int)(tk % p);
        const int kb = (int)((tk / p) % kbl);
        const int b = (int)(tk / ((long)p * kbl));
        const int oc0 = kb * OB;
        const int nob = k - oc0 < OB ? k - oc0 : OB;
        const float *xb = xp + (size_t)b * c * plane + (size_t)oy * stride * wp;
        for (int ox0 = 0; ox0 < q; ox0 += XB) {
            v4d acc[OB][XB / 4];
            const float *xc0 = xb + (size_t)ox0 * stride;
            const double *wb = wk + (size_t)kb * c * taps * OB;
            if (stride == 1) dc_block(xc0, wb, c, taps, kw, plane, wp, 1, acc);
            else if (stride == 2) dc_block(xc0, wb, c, taps, kw, plane, wp, 2, acc);
            else dc_block(xc0, wb, c, taps, kw, plane, wp, stride, acc);
            const int nx = q - ox0 < XB ? q - ox0 : XB;
            for (int o = 0; o < nob; ++o) {
                double *yr = y + (((size_t)b * k + oc0 + o) * p + oy) * q + ox0;
                for (int j = 0; j < nx; ++j) yr[j] = acc[o][j / 4][j % 4];
            }
        }
    }
    free(wk);
    free(xp);
    return 0;
}
#undef OB
#undef XB

/* matrices row-major: at [e x m], g [m x r], bt [m x m] */
int oracle_winograd_conv_f32in(const float *x, const float *wt, double *y,
                               int n, int c, int h, int w, int k, int r, int e, int pad,
                               const double *at, const double *g, const double *bt) {
    if (n < 0 || c < 1 || h < 1 || w < 1 || k < 1 || r < 1 || e < 1 || pad < 0) return 2;
    const int m = e + r - 1;
    const int hp = h + 2 * pad, wp = w + 2 * pad;
    if (r > hp || r > wp) return 3;
    const int p = hp - r + 1, q = wp - r + 1;
    const int ty = (p + e - 1) / e, tx = (q + e - 1) / e;
    const int mm = m * m;
    /* kernel transforms U[oc][ci][m*m] (shared across tiles: a value-level
       reuse that does not change any product) */
    double *u = (double *)malloc(sizeof(double) * (size_t)k * c * mm);
    if (!u) return 4;
#pragma omp parallel for schedule(static)
    for (long kc = 0; kc < (long)k * c; ++kc) {
        const float *gk = wt + kc * r * r;
        double tmp[64 * 16];
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < r; ++j) {
                double s = 0.0;
                for (int t = 0; t < r; ++t) s += g[i * r + t] * (double)gk[t * r + j];
                tmp[i * r + j] = s;
            }
        for (int i = 0; i < m; ++i)
            for (int l = 0; l < m; ++l) {
                double s = 0.0;
                for (int j = 0; j < r; ++j) s += tmp[i * r + j] * g[l * r + j];
                u[kc * mm + i * m + l] = s;
            }
    }
    const long pairs = (long)n * k;
#pragma omp parallel for schedule(dynamic, 1)
    for (long bk = 0; bk < pairs; ++bk) {
        const int b = (int)(bk / k), oc = (int)(bk % k);
        const float *xb = x + (long)b * c * h * w;
        double *yo = y + bk * (long)p * q;
        double d[16 * 16], t1[16 * 16], v[16 * 16], acc[16 * 16], o1[16 * 16];
        for (int tyi = 0; tyi < ty; ++tyi) {
            for (int txi = 0; txi < tx; ++txi) {
                memset(acc, 0, sizeof(double) * mm);
                for (int ci = 0; ci < c; ++ci) {
                    const float *xc = xb + (long)ci * h * w;
                    for (int i = 0; i < m; ++i)
                        for (int j = 0; j < m; ++j) {
                            const int iy = tyi * e + i - pad, ix = txi * e + j - pad;
                            d[i * m + j] = (iy >= 0 && iy < h && ix >= 0 && ix < w)
                                               ? (double)xc[(long)iy * w + ix] : 0.0;
                        }
                    for (int i = 0; i < m; ++i)          /* B^T d */
                        for (int j = 0; j < m; ++j) {
                            double s = 0.0;
                            for (int t = 0; t < m; ++t) s += bt[i * m + t] * d[t * m + j];
                            t1[i * m + j] = s;
                        }
                    for (int i = 0; i < m; ++i)          /* (B^T d) B */
                        for (int l = 0; l < m; ++l) {
                            double s = 0.0;
                            for (int t = 0; t < m; ++t) s += t1[i * m + t] * bt[l * m + t];
                            v[i * m + l] = s;
                        }
                    const double *uk = u + ((long)oc * c + ci) * mm;
                    for (int i = 0; i < mm; ++i) acc[i] += uk[i] * v[i];
                }
                for (int i = 0; i < e; ++i)              /* A^T Pi */
                    for (int l = 0; l < m; ++l) {
                        double s = 0.0;
                        for (int t = 0; t < m; ++t) s += at[i * m + t] * acc[t * m + l];
                        o1[i * m + l] = s;
                    }
                for (int i = 0; i < e; ++i)              /* (A^T Pi) A, cropped */
                    for (int j = 0; j < e; ++j) {
                        const int oy = tyi * e + i, ox = txi * e + j;
                        if (oy >= p || ox >= q) continue;
                        double s = 0.0;
                        for (int t = 0; t < m; ++t) s += o1[i * m + t] * at[j * m + t];
                        yo[(long)oy * q + ox] = s;
                    }
            }
        }
    }
    free(u);
    return 0;
}
