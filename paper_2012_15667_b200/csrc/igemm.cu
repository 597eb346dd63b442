// Host side of the tcgen05 implicit-GEMM convolution (TF32 in, FP32 accumulate):
// device projection of a TileConfig, filter packing, TMA descriptors, launch.
#include <stdarg.h>
#include <algorithm>

#include "igemm_tcgen05.cuh"

namespace convio {

using IgemmFn = void (*)(const IgemmParams, const CUtensorMap, const CUtensorMap);

static IgemmFn igemm_kernel(int bn, bool split) {
    if (split) {
        switch (bn) {
            case 64: return &igemm_tf32_tcgen05_kernel<64, true>;
            case 128: return &igemm_tf32_tcgen05_kernel<128, true>;
            case 256: return &igemm_tf32_tcgen05_kernel<256, true>;
            default: return nullptr;
        }
    }
    switch (bn) {
        case 64: return &igemm_tf32_tcgen05_kernel<64, false>;
        case 128: return &igemm_tf32_tcgen05_kernel<128, false>;
        case 256: return &igemm_tf32_tcgen05_kernel<256, false>;
        default: return nullptr;
    }
}

// KCRS -> [R*S][K][C]
__global__ void pack_filter_igemm_kernel(const float *w, float *wq, int k, int c, int rs) {
    const int64_t total = (int64_t)k * c * rs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int cc = i % c;
        const int kk = (i / c) % k;
        const int tap = i / ((int64_t)c * k);
        wq[i] = w[((int64_t)kk * c + cc) * rs + tap];
    }
}

struct IgemmPlan {
    IgemmParams P;
    IgemmFn fn = nullptr;
    dim3 grid;
    size_t smem = 0;
    int regs = 0;
    int bn = 0;
    int threads = 128;
    bool split = false;
};

static int plan_igemm(const convio_conv_desc *d, const convio_tile *t, IgemmPlan *pl, char *reason,
                      size_t rlen, bool split) {
    auto fail = [&](int code, const char *fmt, ...) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(reason, rlen, fmt, ap);
        va_end(ap);
        set_error("%s", reason);
        return code;
    };
    if (!d || !t) return fail(CONVIO_EINVAL, "null descriptor or tile");
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->k < 1 || d->r < 1 || d->s < 1 ||
        d->stride < 1 || d->pad < 0)
        return fail(CONVIO_EINVAL, "descriptor fields must be >= 1 (pad >= 0)");
    const int hp = d->h + 2 * d->pad, wp = d->w + 2 * d->pad;
    if (d->r > hp || d->s > wp) return fail(CONVIO_EINFEASIBLE, "kernel larger than padded input");
    const int p = (hp - d->r) / d->stride + 1, q = (wp - d->s) / d->stride + 1;
    if (d->layout != CONVIO_LAYOUT_HWC)
        return fail(CONVIO_EINFEASIBLE, "tcgen05 implicit GEMM needs the HWC (NHWC) layout");
    if (t->layout != d->layout) return fail(CONVIO_EINVAL, "tile layout differs from tensor layout");
    if (d->stride > 2) return fail(CONVIO_EINFEASIBLE, "tcgen05 implicit GEMM supports stride 1 and 2");
    if (d->r != d->s) return fail(CONVIO_EINFEASIBLE, "square kernels only");
    if (d->c % 32) return fail(CONVIO_EINFEASIBLE, "C=%d is not a multiple of 32 (one 128-B K block)", d->c);
    if (t->x < 1 || t->y < 1 || t->z < 1 || t->s_b < 1)
        return fail(CONVIO_EINFEASIBLE, "tile fields must be >= 1");
    if (q % t->x || p % t->y || d->k % t->z)
        return fail(CONVIO_EINFEASIBLE, "tile %dx%dx%d does not divide output %dx%dx%d", t->x, t->y,
                    t->z, q, p, d->k);
    const int tile_w = d->stride * (t->x - 1) + d->s, tile_h = d->stride * (t->y - 1) + d->r;
    const int64_t resident = (int64_t)t->x * t->y * t->z + (int64_t)tile_w * tile_h + (int64_t)d->r * d->s * t->z;
    if (resident > t->s_b)
        return fail(CONVIO_EINFEASIBLE, "stage 0 resident set %lld words exceeds s_b=%d",
                    (long long)resident, t->s_b);
    const int bn = t->z;
    IgemmFn fn = igemm_kernel(bn, split);
    if (!fn)
        return fail(CONVIO_EINFEASIBLE, "tcgen05 tiles need z in {64, 128, 256}, got %d", bn);
    const int px = t->x * t->y;
    if (px > 128) return fail(CONVIO_EINFEASIBLE, "x*y=%d pixels exceed the M=128 MMA tile", px);
    if (t->x * d->stride > 256 || t->y * d->stride > 256)
        return fail(CONVIO_EINFEASIBLE, "TMA box dims > 256");
    const int imgs = std::max(1, std::min(128 / px, d->n));
    // ring depth: the outputs live in TMEM, so s_b only sizes the TMA ring:
    // ring bytes <= 6 * s_b (s_b = 16384 words -> 96 KB, two CTAs per SM;
    // 32768 -> 192 KB, one deep-ring CTA per SM), 2..6 stages
    const int stage_words = (128 * 32 + bn * 32) * (split ? 2 : 1);
    const size_t stage_bytes = (size_t)4 * stage_words;
    const size_t ring_cap = std::min<size_t>((size_t)6 * t->s_b, 227 * 1024 - 2048);
    int stages = (int)std::min<size_t>(6, ring_cap / stage_bytes);
    if (stages < 2) stages = 2;
    while (stages > 2 && stages * stage_bytes + 2048 > 227 * 1024) --stages;
    const size_t smem = stages * stage_bytes + 1024 + 512;
    if (smem > 227 * 1024) return fail(CONVIO_EINFEASIBLE, "tcgen05 ring needs %zu B smem", smem);
    IgemmParams &P = pl->P;
    memset(&P, 0, sizeof(P));
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
    pl->split = split;
    pl->threads = split ? 256 : 128;
    if (launch_fit((const void *)fn, pl->threads, smem, &pl->regs) < 1)
        return fail(CONVIO_EINFEASIBLE, "tcgen05 block (%d threads, %zu B smem) does not fit",
                    pl->threads, smem);
    return CONVIO_OK;
}

static bool make_igemm_maps(const IgemmPlan &pl, const float *x, const float *wq, CUtensorMap *tx,
                            CUtensorMap *tw) {
    const IgemmParams &P = pl.P;
    if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(wq) & 15)) return false;
    cuuint64_t xd[4] = {(cuuint64_t)P.c, (cuuint64_t)P.w, (cuuint64_t)P.h, (cuuint64_t)P.n};
    cuuint64_t xs[3] = {(cuuint64_t)P.c * 4, (cuuint64_t)P.w * P.c * 4, (cuuint64_t)P.h * P.w * P.c * 4};
    // stride: box spans stride*(pixels) input positions, traversal stride picks every stride-th
    cuuint32_t xb[4] = {32, (cuuint32_t)(P.bx * P.stride), (cuuint32_t)(P.by * P.stride),
                        (cuuint32_t)P.imgs};
    cuuint32_t xes[4] = {1, (cuuint32_t)P.stride, (cuuint32_t)P.stride, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (!encode_tensor_map_tiled_ex(tx, 4, const_cast<float *>(x), xd, xs, xb, xes, true)) return false;
    const int rs = P.ks * P.ks;
    cuuint64_t wd[3] = {(cuuint64_t)P.c, (cuuint64_t)P.k, (cuuint64_t)rs};
    cuuint64_t ws[2] = {(cuuint64_t)P.c * 4, (cuuint64_t)P.k * P.c * 4};
    cuuint32_t wb[3] = {32, (cuuint32_t)pl.bn, 1};
    return encode_tensor_map_tiled_ex(tw, 3, const_cast<float *>(wq), wd, ws, wb, es, true);
}

int igemm_query(const convio_conv_desc *d, const convio_tile *t, convio_launch_info *out, bool split) {
    IgemmPlan pl;
    int rc = plan_igemm(d, t, &pl, out->reason, sizeof(out->reason), split);
    if (rc) return rc;
    out->legal = 1;
    out->grid_x = pl.grid.x; out->grid_y = pl.grid.y; out->grid_z = pl.grid.z;
    out->block_threads = pl.threads;
    out->smem_bytes = (int)pl.smem;
    out->regs_per_thread = pl.regs;
    out->channel_chunk = 32;
    out->stages = pl.P.stages;
    out->p = pl.P.p; out->q = pl.P.q;
    out->flops = 2LL * d->n * d->k * pl.P.p * pl.P.q * (int64_t)d->c * d->r * d->s;
    out->workspace_bytes = 4LL * d->k * d->c * d->r * d->s;
    snprintf(out->reason, sizeof(out->reason), "tcgen05 %s: M=128 (%d px x %d img), N=%d, %d stages",
             split ? "3xtf32" : "tf32", pl.P.bx * pl.P.by, pl.P.imgs, pl.bn, pl.P.stages);
    return CONVIO_OK;
}

}  // namespace convio

using namespace convio;

extern "C" {

int convio_pack_filter_igemm(const convio_conv_desc *desc, const float *w, float *wq, void *stream) {
    clear_error();
    if (!desc || !w || !wq) {
        set_error("null argument");
        return CONVIO_EINVAL;
    }
    const int64_t total = (int64_t)desc->k * desc->c * desc->r * desc->s;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
    pack_filter_igemm_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(w, wq, desc->k, desc->c,
                                                                      desc->r * desc->s);
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

static int conv_igemm(const convio_conv_desc *desc, const convio_tile *tile, const float *x,
                      const float *w, int32_t w_is_packed, const float *bias, int32_t relu, float *y,
                      void *workspace, size_t workspace_bytes, void *stream, bool split) {
    clear_error();
    reset_launches();
    if (!x || !w || !y || !tile) {
        set_error("null tensor pointer or tile");
        return CONVIO_EINVAL;
    }
    IgemmPlan pl;
    char why[160];
    int rc = plan_igemm(desc, tile, &pl, why, sizeof(why), split);
    if (rc) return rc;
    const float *wq = w;
    if (!w_is_packed) {
        const size_t need = 4ULL * desc->k * desc->c * desc->r * desc->s;
        if (!workspace || workspace_bytes < need) {
            set_error("workspace of %zu bytes needed for the packed filter", need);
            return CONVIO_EINVAL;
        }
        rc = convio_pack_filter_igemm(desc, w, (float *)workspace, stream);
        if (rc) return rc;
        wq = (const float *)workspace;
        reset_launches();
        note_launch();
    }
    CUtensorMap tx, tw;
    if (!make_igemm_maps(pl, x, wq, &tx, &tw)) {
        set_error("TMA descriptors cannot describe these tensors (alignment)");
        return CONVIO_EINFEASIBLE;
    }
    pl.P.bias = bias;
    pl.P.y = y;
    pl.P.relu = relu;
    pl.fn<<<pl.grid, pl.threads, pl.smem, (cudaStream_t)stream>>>(pl.P, tx, tw);
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

int convio_conv_igemm_tf32(const convio_conv_desc *desc, const convio_tile *tile, const float *x,
                           const float *w, int32_t w_is_packed, const float *bias, int32_t relu,
                           float *y, void *workspace, size_t workspace_bytes, void *stream) {
    return conv_igemm(desc, tile, x, w, w_is_packed, bias, relu, y, workspace, workspace_bytes,
                      stream, false);
}

int convio_conv_igemm_3xtf32(const convio_conv_desc *desc, const convio_tile *tile, const float *x,
                             const float *w, int32_t w_is_packed, const float *bias, int32_t relu,
                             float *y, void *workspace, size_t workspace_bytes, void *stream) {
    return conv_igemm(desc, tile, x, w, w_is_packed, bias, relu, y, workspace, workspace_bytes,
                      stream, true);
}

}  // extern "C"
