// K8: channels-last FP32 direct convolution for input layers with few channels
// (C <= 4: RGB(A) / grey images -- VGG-16 conv1_1 is C = 3, K = 64, 224 x 224).
// The stacked-pixel kernel (direct_nhwc.cuh) and the tensor-core GEMMs stage
// 32-channel (128-B) K blocks and cannot take C = 3; the register micro-tile
// kernel (direct_fp32.cuh) runs this layer at ~35 % of the FFMA peak.
//
// The same output-stationary dataflow as plan_direct_dataflow
// (reference src/dataflow.py:219-250) with the whole input-channel range in one
// stage: a CTA owns a 16 x 16 output block; it stages the block's
// (16*stride + 2)^2 x C input footprint (zero halo) once and walks the output
// channels in chunks of 32 (a 9 C x 32 filter slice each); each thread accumulates 2 pixels x 32
// channels in registers in the DAG's (c, ky, kx) order (dag.py:247-285), and the
// 256 x 32 output block leaves through a shared-memory transpose so 8 lanes write
// each pixel's 128 contiguous bytes.  Roofline: FFMA (2 LDS + 8 broadcast
// LDS.128 per 64 FFMA) against the output write (K / C times the input bytes).
//
// Tile convention (convio_query / convio_conv_direct_f32): layout HWC, x = y = 16,
// z = 32, n_xt = n_yt = n_zt = 1, with C <= 4, 3 x 3 kernel, stride 1 or 2.
#include <stdarg.h>
#include <algorithm>

#include "common.cuh"

namespace convio {

struct SmallCParams {
    const float *x;    // NHWC
    const float *wp;   // packed [C][R*S][K] (convio_pack_filter_direct)
    const float *bias;
    float *y;          // NHWC
    int n, c, h, w, k, p, q, pad;
    int tiles_x, tiles_y;
    int relu;
};

constexpr int SC_BX = 16, SC_BY = 16, SC_BK = 32, SC_THREADS = 128;
static_assert(SC_BK % 4 == 0, "float4 filter rows");

template <int CI, int ST>
struct SmallCSmem {
    static constexpr int FW = SC_BX * ST + 2, FH = SC_BY * ST + 2;
    static constexpr int IN = FH * FW * CI;                    // input footprint
    static constexpr int W = 9 * CI * SC_BK;                   // filter slice per 32 channels
    static constexpr int OUT = SC_BX * SC_BY * (SC_BK + 4);    // transpose (+4 pad, 16-B rows)
};

template <int CI, int ST>
__global__ void __launch_bounds__(SC_THREADS, 5) direct_smallc_kernel(const SmallCParams P) {
    using L = SmallCSmem<CI, ST>;
    extern __shared__ __align__(16) float sm[];
    float *s_w = sm;                 // [c][tap][32] of the current chunk, 16-B aligned
    float *s_in = s_w + L::W;        // [fy][fx][c]
    float *s_out = s_in + ((L::IN + 3) & ~3);   // [pixel][36], 16-B aligned
    pdl_wait();
    const int tid = threadIdx.x;
    int b = blockIdx.x;
    const int tx = b % P.tiles_x;
    b /= P.tiles_x;
    const int ty = b % P.tiles_y;
    const int img = b / P.tiles_y;
    const int ox0 = tx * SC_BX, oy0 = ty * SC_BY;
    const int ix0 = ox0 * ST - P.pad, iy0 = oy0 * ST - P.pad;

    // input footprint, zero halo; consecutive threads read consecutive floats of a row
    const float *xi = P.x + (int64_t)img * P.h * P.w * CI;
    for (int i = tid; i < L::IN; i += SC_THREADS) {
        const int fy = i / (L::FW * CI);
        const int rem = i - fy * (L::FW * CI);
        const int fx = rem / CI, c = rem - fx * CI;
        const int iy = iy0 + fy, ix = ix0 + fx;
        s_in[i] = (iy >= 0 && iy < P.h && ix >= 0 && ix < P.w)
                      ? __ldg(xi + ((int64_t)iy * P.w + ix) * CI + c) : 0.0f;
    }
    const int px = tid % SC_BX, py = (tid / SC_BX) * 2;   // 2 output rows per thread
    // the footprint stays staged while the block walks the K / 32 output-channel chunks
    for (int k0 = 0; k0 < P.k; k0 += SC_BK) {
    // filter slice: s_w[(c * 9 + tap) * 32 + kk] = wp[(c * 9 + tap) * K + k0 + kk]
    // (staging all K filters once measured slower: 0.204 vs 0.191 ms on conv1_1)
    for (int i = tid; i < L::W / 4; i += SC_THREADS) {
        const int ct = i / (SC_BK / 4), k4 = i - ct * (SC_BK / 4);
        reinterpret_cast<float4 *>(s_w)[i] =
            __ldg(reinterpret_cast<const float4 *>(P.wp + (int64_t)ct * P.k + k0) + k4);
    }
    __syncthreads();
    const float *s_wk = s_w;
    float acc[2][SC_BK];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < SC_BK; ++j) acc[r][j] = 0.0f;
#pragma unroll
    for (int c = 0; c < CI; ++c) {
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
#pragma unroll
            for (int kx = 0; kx < 3; ++kx) {
                const float a0 = s_in[((py * ST + ky) * L::FW + px * ST + kx) * CI + c];
                const float a1 = s_in[(((py + 1) * ST + ky) * L::FW + px * ST + kx) * CI + c];
                const float4 *wv = reinterpret_cast<const float4 *>(s_wk + (c * 9 + ky * 3 + kx) * SC_BK);
#pragma unroll
                for (int j = 0; j < SC_BK / 4; ++j) {
                    const float4 wj = wv[j];
                    acc[0][4 * j] = fmaf(a0, wj.x, acc[0][4 * j]);
                    acc[0][4 * j + 1] = fmaf(a0, wj.y, acc[0][4 * j + 1]);
                    acc[0][4 * j + 2] = fmaf(a0, wj.z, acc[0][4 * j + 2]);
                    acc[0][4 * j + 3] = fmaf(a0, wj.w, acc[0][4 * j + 3]);
                    acc[1][4 * j] = fmaf(a1, wj.x, acc[1][4 * j]);
                    acc[1][4 * j + 1] = fmaf(a1, wj.y, acc[1][4 * j + 1]);
                    acc[1][4 * j + 2] = fmaf(a1, wj.z, acc[1][4 * j + 2]);
                    acc[1][4 * j + 3] = fmaf(a1, wj.w, acc[1][4 * j + 3]);
                }
            }
        }
    }
    // transpose through shared memory: pixel-major rows of 32 (+4 pad) floats
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int pix = (py + r) * SC_BX + px;
#pragma unroll
        for (int j = 0; j < SC_BK; j += 4)
            *reinterpret_cast<float4 *>(s_out + pix * (SC_BK + 4) + j) =
                make_float4(acc[r][j], acc[r][j + 1], acc[r][j + 2], acc[r][j + 3]);
    }
    __syncthreads();
    const int lane8 = tid & 7;                   // 8 lanes x float4 = one pixel's 32 channels
    const float4 bv = P.bias ? __ldg(reinterpret_cast<const float4 *>(P.bias + k0) + lane8)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int pix = tid >> 3; pix < SC_BX * SC_BY; pix += SC_THREADS / 8) {
        const int oy = oy0 + pix / SC_BX, ox = ox0 + pix % SC_BX;
        if (oy >= P.p || ox >= P.q) continue;
        float4 o = *reinterpret_cast<const float4 *>(s_out + pix * (SC_BK + 4) + 4 * lane8);
        o.x += bv.x; o.y += bv.y; o.z += bv.z; o.w += bv.w;
        if (P.relu) {
            o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f);
            o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
        }
        reinterpret_cast<float4 *>(P.y + (((int64_t)img * P.p + oy) * P.q + ox) * P.k + k0)[lane8] = o;
    }
    __syncthreads();   // s_w / s_out reused by the next chunk
    }
}

using SmallCFn = void (*)(const SmallCParams);

template <int ST>
static SmallCFn smallc_fn(int c) {
    switch (c) {
        case 1: return &direct_smallc_kernel<1, ST>;
        case 2: return &direct_smallc_kernel<2, ST>;
        case 3: return &direct_smallc_kernel<3, ST>;
        case 4: return &direct_smallc_kernel<4, ST>;
        default: return nullptr;
    }
}

static size_t smallc_smem(int c, int st) {
    const int fw = SC_BX * st + 2, fh = SC_BY * st + 2;
    return sizeof(float) * ((((size_t)fh * fw * c + 3) & ~size_t(3)) + 9 * c * SC_BK +
                            SC_BX * SC_BY * (SC_BK + 4)) + 16;
}

bool smallc_tile(const convio_conv_desc *d, const convio_tile *t) {
    return d && t && d->layout == CONVIO_LAYOUT_HWC && t->layout == CONVIO_LAYOUT_HWC && d->c <= 4 &&
           t->x == SC_BX && t->y == SC_BY && t->z == SC_BK && t->n_xt == 1 && t->n_yt == 1 &&
           t->n_zt == 1;
}

static int smallc_plan(const convio_conv_desc *d, const convio_tile *t, SmallCParams *P, SmallCFn *fn,
                       dim3 *grid, size_t *smem, char *reason, size_t rlen) {
    auto fail = [&](int code, const char *fmt, ...) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(reason, rlen, fmt, ap);
        va_end(ap);
        set_error("%s", reason);
        return code;
    };
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->k < 1 || d->pad < 0)
        return fail(CONVIO_EINVAL, "descriptor fields must be >= 1 (pad >= 0)");
    if (d->r != 3 || d->s != 3) return fail(CONVIO_EINFEASIBLE, "small-C kernel: 3x3 filters only");
    if (d->stride != 1 && d->stride != 2)
        return fail(CONVIO_EINFEASIBLE, "small-C kernel: stride 1 or 2");
    if (d->k % SC_BK) return fail(CONVIO_EINFEASIBLE, "small-C kernel: K=%d not a multiple of 32", d->k);
    const int hp = d->h + 2 * d->pad, wp = d->w + 2 * d->pad;
    if (hp < 3 || wp < 3) return fail(geometry_error(), "kernel larger than padded input");
    const int p = (hp - 3) / d->stride + 1, q = (wp - 3) / d->stride + 1;
    // the model's legality rule on the block (reference dataflow.py:228-233):
    // resident x*y*z outputs + footprint + kw*z filter words <= s_b
    const int fw = SC_BX * d->stride + 2, fh = SC_BY * d->stride + 2;
    const int64_t resident = (int64_t)SC_BX * SC_BY * SC_BK + (int64_t)fw * fh + 3 * SC_BK;
    if (resident > t->s_b)
        return fail(schedule_error(), "stage 0 resident set %lld words exceeds s_b=%d",
                    (long long)resident, t->s_b);
    *fn = d->stride == 1 ? smallc_fn<1>(d->c) : smallc_fn<2>(d->c);
    if (!*fn) return fail(CONVIO_EINFEASIBLE, "small-C kernel: C=%d > 4", d->c);
    P->n = d->n; P->c = d->c; P->h = d->h; P->w = d->w; P->k = d->k; P->p = p; P->q = q;
    P->pad = d->pad;
    P->tiles_x = (q + SC_BX - 1) / SC_BX;
    P->tiles_y = (p + SC_BY - 1) / SC_BY;
    const int64_t blocks = (int64_t)P->tiles_x * P->tiles_y * d->n;
    if (blocks >= ((int64_t)1 << 31)) return fail(CONVIO_EINFEASIBLE, "grid exceeds launch limits");
    *grid = dim3((unsigned)blocks, 1, 1);
    *smem = smallc_smem(d->c, d->stride);
    return CONVIO_OK;
}

int direct_smallc_query(const convio_conv_desc *d, const convio_tile *t, convio_launch_info *out) {
    SmallCParams P;
    SmallCFn fn;
    dim3 grid;
    size_t smem;
    int rc = smallc_plan(d, t, &P, &fn, &grid, &smem, out->reason, sizeof(out->reason));
    if (rc) return rc;
    int regs = 0;
    if (launch_fit((const void *)fn, SC_THREADS, smem, &regs) < 1) {
        snprintf(out->reason, sizeof(out->reason), "small-C block does not fit an SM");
        return CONVIO_EINFEASIBLE;
    }
    out->legal = 1;
    out->grid_x = grid.x; out->grid_y = grid.y; out->grid_z = 1;
    out->block_threads = SC_THREADS;
    out->smem_bytes = (int)smem;
    out->regs_per_thread = regs;
    out->channel_chunk = d->c;
    out->stages = 1;
    out->p = P.p; out->q = P.q;
    out->flops = 2LL * d->n * d->k * P.p * P.q * (int64_t)d->c * 9;
    out->workspace_bytes = 4LL * d->k * d->c * 9;
    snprintf(out->reason, sizeof(out->reason),
             "channels-last small-C FFMA: 16x16 px x 32 ch per block, C=%d staged whole", d->c);
    return CONVIO_OK;
}

int direct_smallc_run(const convio_conv_desc *d, const convio_tile *t, const float *x, const float *wp,
                      const float *bias, int relu, float *y, cudaStream_t stream) {
    SmallCParams P;
    SmallCFn fn;
    dim3 grid;
    size_t smem;
    char why[160];
    int rc = smallc_plan(d, t, &P, &fn, &grid, &smem, why, sizeof(why));
    if (rc) return rc;
    if ((reinterpret_cast<uintptr_t>(y) & 15) || (reinterpret_cast<uintptr_t>(wp) & 15) ||
        (bias && (reinterpret_cast<uintptr_t>(bias) & 15))) {
        set_error("small-C kernel needs 16-byte aligned output, packed filter and bias");
        return CONVIO_EINFEASIBLE;
    }
    int regs = 0;
    if (launch_fit((const void *)fn, SC_THREADS, smem, &regs) < 1) {
        set_error("small-C block does not fit an SM");
        return CONVIO_EINFEASIBLE;
    }
    P.x = x; P.wp = wp; P.bias = bias; P.y = y; P.relu = relu;
    CONVIO_CUDA_TRY(launch_pdl(fn, grid, dim3(SC_THREADS), smem, stream, P));
    note_launch();
    return CONVIO_OK;
}

}  // namespace convio
