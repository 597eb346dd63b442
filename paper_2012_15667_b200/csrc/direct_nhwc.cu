// Host side of the channels-last FP32 direct kernel (direct_nhwc.cuh): device
// projection of a TileConfig, TMA descriptors, launch.  Reached through
// convio_query / convio_conv_direct_f32 when the tile asks for it.
#include <stdarg.h>
#include <algorithm>

#include "direct_nhwc.cuh"

namespace convio {

using NhwcFn = void (*)(const NhwcParams, const CUtensorMap, const CUtensorMap);

// A HWC tile with z in {64, 128} and either 16 x 16 threads (n_xt * n_yt = 16
// pixel groups, n_zt = 16 channel groups) or n_xt = n_yt = n_zt = 1 ("library
// thread layout", needed where no 16-way split divides x, y -- e.g. 7 x 7
// maps) is realised by the stacked-pixel kernel.  (The register micro-tile
// kernels never compile x*y*z-output threads, so (1,1,1) is otherwise illegal.)
bool nhwc_tile(const convio_conv_desc *d, const convio_tile *t) {
    if (!d || !t || d->layout != CONVIO_LAYOUT_HWC || t->layout != CONVIO_LAYOUT_HWC) return false;
    if (t->z != 64 && t->z != 128) return false;
    return (t->n_zt == 16 && t->n_xt * t->n_yt == 16) ||
           (t->n_xt == 1 && t->n_yt == 1 && t->n_zt == 1);
}

struct NhwcPlan {
    NhwcParams P;
    NhwcFn fn = nullptr;
    dim3 grid;
    size_t smem = 0;
    int regs = 0;
    int bn = 0;
};

static int plan_nhwc(const convio_conv_desc *d, const convio_tile *t, NhwcPlan *pl, char *reason,
                     size_t rlen) {
    auto fail = [&](int code, const char *fmt, ...) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(reason, rlen, fmt, ap);
        va_end(ap);
        set_error("%s", reason);
        return code;
    };
    const int hp = d->h + 2 * d->pad, wp = d->w + 2 * d->pad;
    if (d->r > hp || d->s > wp) return fail(geometry_error(), "kernel larger than padded input");
    const int p = (hp - d->r) / d->stride + 1, q = (wp - d->s) / d->stride + 1;
    if (d->r != d->s) return fail(CONVIO_EINFEASIBLE, "square kernels only");
    if (d->stride > 2) return fail(CONVIO_EINFEASIBLE, "channels-last direct kernel: stride 1 or 2");
    if (d->c % 32) return fail(CONVIO_EINFEASIBLE, "C=%d is not a multiple of 32 (one 128-B stage row)", d->c);
    if (d->k % 4) return fail(CONVIO_EINFEASIBLE, "K must be a multiple of 4");
    if (q % t->x || p % t->y || d->k % t->z)
        return fail(schedule_error(), "tile %dx%dx%d does not divide output %dx%dx%d", t->x, t->y,
                    t->z, q, p, d->k);
    const int tile_w = d->stride * (t->x - 1) + d->s, tile_h = d->stride * (t->y - 1) + d->r;
    const int64_t resident = (int64_t)t->x * t->y * t->z + (int64_t)tile_w * tile_h + (int64_t)d->r * d->s * t->z;
    if (resident > t->s_b)
        return fail(schedule_error(), "stage 0 resident set %lld words exceeds s_b=%d",
                    (long long)resident, t->s_b);
    const int px = t->x * t->y;
    if (px > 128) return fail(CONVIO_EINFEASIBLE, "x*y=%d pixels exceed the 128-row register tile", px);
    if (t->x * d->stride > 256 || t->y * d->stride > 256)
        return fail(CONVIO_EINFEASIBLE, "TMA box dims > 256");
    const int bn = t->z;
    NhwcFn fn = bn == 128 ? &direct_nhwc_f32_kernel<128> : &direct_nhwc_f32_kernel<64>;
    const size_t stage = 128 * 128 + 32 * (size_t)bn * 4;
    const size_t ring = std::min<size_t>((size_t)8 * t->s_b, 227 * 1024 - 2048);
    int stages = (int)std::min<size_t>(6, ring / stage);
    stages = std::max(stages, 2);
    const size_t smem = stages * stage + 1024 + 256;
    if (smem > 227 * 1024) return fail(CONVIO_EINFEASIBLE, "ring needs %zu B smem", smem);
    NhwcParams &P = pl->P;
    memset(&P, 0, sizeof(P));
    const int imgs = std::max(1, std::min(128 / px, d->n));
    P.n = d->n; P.c = d->c; P.h = d->h; P.w = d->w; P.k = d->k; P.p = p; P.q = q;
    P.pad = d->pad; P.stride = d->stride; P.ks = d->r;
    P.bx = t->x; P.by = t->y; P.imgs = imgs;
    P.tiles_x = q / t->x; P.tiles_y = p / t->y; P.img_groups = (d->n + imgs - 1) / imgs;
    P.cblocks = d->c / 32; P.kblocks = d->r * d->s * P.cblocks;
    P.stages = stages;
    pl->grid = dim3(d->k / bn, P.tiles_x * P.tiles_y * P.img_groups, 1);
    if (pl->grid.y > 65535) return fail(CONVIO_EINFEASIBLE, "grid exceeds launch limits");
    pl->fn = fn;
    pl->smem = smem;
    pl->bn = bn;
    if (launch_fit((const void *)fn, 288, smem, &pl->regs) < 1)
        return fail(CONVIO_EINFEASIBLE, "block (288 threads, %zu B smem) does not fit", smem);
    return CONVIO_OK;
}

// M[xi][t][k] = sum_c V[xi][t][c] * U[xi][c][k] on the FFMA kernel: the
// Winograd element-wise GEMMs of the channels-last FP32 Winograd path
// (winograd_tc.cu, precision CONVIO_PREC_FP32).  One launch for all xi.
int direct_nhwc_batched_run(int bn, int s_b, int xi, int t_count, int c, int k, const float *v,
                            const float *u, float *m, cudaStream_t stream) {
    if (bn != 64 && bn != 128) {
        set_error("FFMA batched GEMM needs z in {64, 128}, got %d", bn);
        return CONVIO_EINFEASIBLE;
    }
    if (c % 32 || k % bn) {
        set_error("FFMA batched GEMM needs C %% 32 == 0 and z | K (C=%d, K=%d, z=%d)", c, k, bn);
        return CONVIO_EINFEASIBLE;
    }
    NhwcPlan pl;
    NhwcParams &P = pl.P;
    memset(&P, 0, sizeof(P));
    NhwcFn fn = bn == 128 ? &direct_nhwc_f32_kernel<128> : &direct_nhwc_f32_kernel<64>;
    const size_t stage = 128 * 128 + 32 * (size_t)bn * 4;
    const size_t ring = std::min<size_t>((size_t)8 * s_b, 227 * 1024 - 2048);
    const int stages = std::max(2, (int)std::min<size_t>(6, ring / stage));
    const size_t smem = stages * stage + 1024 + 256;
    P.n = xi; P.c = c; P.h = 1; P.w = t_count; P.k = k; P.p = 1; P.q = t_count;
    P.pad = 0; P.stride = 1; P.ks = 1;
    P.bx = 128; P.by = 1; P.imgs = 1;
    P.tiles_x = (t_count + 127) / 128; P.tiles_y = 1; P.img_groups = xi;
    P.cblocks = c / 32; P.kblocks = P.cblocks;
    P.stages = stages;
    P.batched = 1;
    int regs = 0;
    if (launch_fit((const void *)fn, 288, smem, &regs) < 1) {
        set_error("FFMA batched GEMM block does not fit");
        return CONVIO_EINFEASIBLE;
    }
    const dim3 grid(k / bn, P.tiles_x * xi, 1);
    if (grid.y > 65535) {
        set_error("grid exceeds launch limits");
        return CONVIO_EINFEASIBLE;
    }
    CUtensorMap tx, tw;
    cuuint64_t xd[4] = {(cuuint64_t)c, (cuuint64_t)t_count, 1, (cuuint64_t)xi};
    cuuint64_t xs[3] = {(cuuint64_t)c * 4, (cuuint64_t)t_count * c * 4, (cuuint64_t)t_count * c * 4};
    cuuint32_t xb[4] = {32, 128, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint64_t wd[3] = {(cuuint64_t)k, (cuuint64_t)c, (cuuint64_t)xi};
    cuuint64_t ws[2] = {(cuuint64_t)k * 4, (cuuint64_t)c * k * 4};
    cuuint32_t wb[3] = {(cuuint32_t)bn, 32, 1};
    if (!encode_tensor_map_tiled_ex(&tx, 4, const_cast<float *>(v), xd, xs, xb, es, true) ||
        !encode_tensor_map_tiled_ex(&tw, 3, const_cast<float *>(u), wd, ws, wb, es, false)) {
        set_error("TMA descriptors cannot describe the Winograd operands");
        return CONVIO_EINFEASIBLE;
    }
    P.bias = nullptr;
    P.y = m;
    P.relu = 0;
    fn<<<grid, 288, smem, stream>>>(P, tx, tw);
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

int direct_nhwc_query(const convio_conv_desc *d, const convio_tile *t, convio_launch_info *out) {
    NhwcPlan pl;
    int rc = plan_nhwc(d, t, &pl, out->reason, sizeof(out->reason));
    if (rc) return rc;
    out->legal = 1;
    out->grid_x = pl.grid.x; out->grid_y = pl.grid.y; out->grid_z = pl.grid.z;
    out->block_threads = 288;
    out->smem_bytes = (int)pl.smem;
    out->regs_per_thread = pl.regs;
    out->channel_chunk = 32;
    out->stages = pl.P.stages;
    out->p = pl.P.p; out->q = pl.P.q;
    out->flops = 2LL * d->n * d->k * pl.P.p * pl.P.q * (int64_t)d->c * d->r * d->s;
    out->workspace_bytes = 4LL * d->k * d->c * d->r * d->s;
    snprintf(out->reason, sizeof(out->reason),
             "channels-last FFMA: %d px x %d img x %d ch per block, tma ring %d stages", pl.P.bx * pl.P.by,
             pl.P.imgs, pl.bn, pl.P.stages);
    return CONVIO_OK;
}

// wp: filters packed C R S K (convio_pack_filter_direct)
int direct_nhwc_run(const convio_conv_desc *d, const convio_tile *t, const float *x, const float *wp,
                    const float *bias, int relu, float *y, cudaStream_t stream) {
    NhwcPlan pl;
    char why[160];
    int rc = plan_nhwc(d, t, &pl, why, sizeof(why));
    if (rc) return rc;
    const NhwcParams &P = pl.P;
    if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(wp) & 15)) {
        set_error("channels-last direct kernel needs 16-byte aligned x and filter");
        return CONVIO_EINFEASIBLE;
    }
    CUtensorMap tx, tw;
    cuuint64_t xd[4] = {(cuuint64_t)P.c, (cuuint64_t)P.w, (cuuint64_t)P.h, (cuuint64_t)P.n};
    cuuint64_t xs[3] = {(cuuint64_t)P.c * 4, (cuuint64_t)P.w * P.c * 4, (cuuint64_t)P.h * P.w * P.c * 4};
    cuuint32_t xb[4] = {32, (cuuint32_t)(P.bx * P.stride), (cuuint32_t)(P.by * P.stride), (cuuint32_t)P.imgs};
    cuuint32_t xes[4] = {1, (cuuint32_t)P.stride, (cuuint32_t)P.stride, 1};
    const int rs = P.ks * P.ks;
    cuuint64_t wd[3] = {(cuuint64_t)P.k, (cuuint64_t)rs, (cuuint64_t)P.c};
    cuuint64_t ws[2] = {(cuuint64_t)P.k * 4, (cuuint64_t)rs * P.k * 4};
    cuuint32_t wb[3] = {(cuuint32_t)pl.bn, 1, 32};
    cuuint32_t es[3] = {1, 1, 1};
    if (!encode_tensor_map_tiled_ex(&tx, 4, const_cast<float *>(x), xd, xs, xb, xes, true) ||
        !encode_tensor_map_tiled_ex(&tw, 3, const_cast<float *>(wp), wd, ws, wb, es, false)) {
        set_error("TMA descriptors cannot describe these tensors");
        return CONVIO_EINFEASIBLE;
    }
    pl.P.bias = bias;
    pl.P.y = y;
    pl.P.relu = relu;
    pl.fn<<<pl.grid, 288, pl.smem, stream>>>(pl.P, tx, tw);
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

}  // namespace convio
