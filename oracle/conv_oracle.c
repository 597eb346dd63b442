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

/* x: [n, c, h, w] fp32; wt: [k, c, kh, kw] fp32; y: [n, k, p, q] fp64 */
int oracle_direct_conv_f32in(const float *x, const float *wt, double *y,
                             int n, int c, int h, int w, int k, int kh, int kw,
                             int stride, int pad, int reserved) {
    (void)reserved;
    if (n < 0 || c < 1 || h < 1 || w < 1 || k < 1 || kh < 1 || kw < 1 || stride < 1 || pad < 0)
        return 2;
    const int hp = h + 2 * pad, wp = w + 2 * pad;
    if (kh > hp || kw > wp) return 3;
    const int p = (hp - kh) / stride + 1, q = (wp - kw) / stride + 1;
    const long pairs = (long)n * k;
#pragma omp parallel for schedule(dynamic, 1)
    for (long bk = 0; bk < pairs; ++bk) {
        const int b = (int)(bk / k), oc = (int)(bk % k);
        double *acc = y + bk * (long)p * q;
        memset(acc, 0, sizeof(double) * (size_t)p * q);
        const float *xb = x + (long)b * c * h * w;
        const float *wk = wt + (long)oc * c * kh * kw;
        for (int ci = 0; ci < c; ++ci) {
            const float *xc = xb + (long)ci * h * w;
            for (int ky = 0; ky < kh; ++ky) {
                for (int kx = 0; kx < kw; ++kx) {
                    const double wv = (double)wk[(ci * kh + ky) * kw + kx];
                    /* valid output columns for this tap: 0 <= ox*stride + kx - pad < w */
                    int ox_lo = 0, ox_hi = q;
                    while (ox_lo < q && ox_lo * stride + kx - pad < 0) ++ox_lo;
                    while (ox_hi > ox_lo && (ox_hi - 1) * stride + kx - pad >= w) --ox_hi;
                    for (int oy = 0; oy < p; ++oy) {
                        const int iy = oy * stride + ky - pad;
                        if (iy < 0 || iy >= h) continue;        /* zero padding */
                        const float *xr = xc + (long)iy * w + kx - pad;
                        double *ar = acc + (long)oy * q;
                        if (stride == 1) {
                            for (int ox = ox_lo; ox < ox_hi; ++ox) ar[ox] += (double)xr[ox] * wv;
                        } else {
                            for (int ox = ox_lo; ox < ox_hi; ++ox)
                                ar[ox] += (double)xr[ox * stride] * wv;
                        }
                    }
                }
            }
        }
    }
    return 0;
}

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
