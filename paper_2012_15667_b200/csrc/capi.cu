// C-ABI of libconvio_b200.so: argument checking, the device projection of a
// TileConfig (legality + launch shape), and the launches.  See
// include/convio_b200.h for the contract and the reference interfaces each
// entry point replaces.
#include <stdarg.h>
#include <algorithm>
#include <atomic>
#include <mutex>

#include "direct_fp32.cuh"
#include "winograd_fp32.cuh"

namespace convio {

static thread_local char t_err[512];
static thread_local int t_launches = 0;

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(t_err, sizeof(t_err), fmt, ap);
    va_end(ap);
}
void clear_error() { t_err[0] = 0; }
void note_launch() { ++t_launches; }
void reset_launches() { t_launches = 0; }

int direct_instance_count();

// ---------------------------------------------------------------------------
// device properties (cached once per process, per device)
// ---------------------------------------------------------------------------
struct DevInfo {
    bool ok = false;
    int max_smem_optin = 0;
    int sms = 0;
};

static DevInfo query_device() {
    DevInfo d;
    int dev = 0, count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return d;
    }
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return d;
    }
    cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    d.ok = true;
    return d;
}

static const DevInfo &dev_info() {
    static DevInfo info = query_device();
    return info;
}

static constexpr int kSmemCapBytes = 227 * 1024;

// ---------------------------------------------------------------------------
// descriptor checks
// ---------------------------------------------------------------------------
static int check_desc(const convio_conv_desc *d, int *p, int *q) {
    if (!d) {
        set_error("null descriptor");
        return CONVIO_EINVAL;
    }
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->k < 1 || d->r < 1 || d->s < 1 ||
        d->stride < 1 || d->pad < 0) {
        set_error("descriptor fields must be >= 1 (pad >= 0)");
        return CONVIO_EINVAL;
    }
    if (d->layout < CONVIO_LAYOUT_CHW || d->layout > CONVIO_LAYOUT_HWC) {
        set_error("layout must be CHW(0), CWH(1) or HWC(2)");
        return CONVIO_EINVAL;
    }
    const int hp = d->h + 2 * d->pad, wp = d->w + 2 * d->pad;
    if (d->r > hp || d->s > wp) {
        set_error("kernel %dx%d larger than padded input %dx%d", d->s, d->r, wp, hp);
        return CONVIO_EINFEASIBLE;
    }
    *p = (hp - d->r) / d->stride + 1;
    *q = (wp - d->s) / d->stride + 1;
    int64_t elems = (int64_t)d->n * d->c * d->h * d->w;
    int64_t oelems = (int64_t)d->n * d->k * (*p) * (*q);
    if (elems >= (int64_t)1 << 31 || oelems >= (int64_t)1 << 31 ||
        (int64_t)d->k * d->c * d->r * d->s >= (int64_t)1 << 31) {
        set_error("tensor too large for 32-bit in-kernel indexing");
        return CONVIO_EINFEASIBLE;
    }
    return CONVIO_OK;
}

// ---------------------------------------------------------------------------
// shared-memory pitch: smallest pitch >= width minimising bank conflicts of
// the row reads (each lane reads base + t_y*ystep*pitch + t_x*xstep)
// ---------------------------------------------------------------------------
static int choose_pitch(int width, int nxt, int nyt, int nthreads, int xstep, int ystep) {
    int best_pitch = width, best_conf = 1 << 30;
    for (int pitch = width; pitch < width + 32; ++pitch) {
        int worst = 0;
        for (int w0 = 0; w0 < nthreads; w0 += 32) {
            int addr[32], na = 0;
            for (int l = 0; l < 32 && w0 + l < nthreads; ++l) {
                const int tid = w0 + l;
                const int tx = tid % nxt, ty = (tid / nxt) % nyt;
                const int a = ty * ystep * pitch + tx * xstep;
                bool seen = false;
                for (int i = 0; i < na; ++i) seen |= addr[i] == a;
                if (!seen) addr[na++] = a;
            }
            int bank[32] = {0};
            for (int i = 0; i < na; ++i) worst = std::max(worst, ++bank[addr[i] & 31]);
        }
        if (worst < best_conf) {
            best_conf = worst;
            best_pitch = pitch;
        }
        if (best_conf == 1) break;
    }
    return best_pitch;
}

// ---------------------------------------------------------------------------
// direct: device projection of a TileConfig
// ---------------------------------------------------------------------------
struct DirectPlan {
    DirectParams P;
    DirectKernelFn fn = nullptr;
    bool generic = false;
    dim3 grid;
    int threads = 0;
    size_t smem = 0;
    int regs = 0;
};

static int plan_direct(const convio_conv_desc *d, const convio_tile *t, DirectPlan *pl,
                       char *reason, size_t rlen) {
    int p = 0, q = 0;
    int rc = check_desc(d, &p, &q);
    if (rc) {
        snprintf(reason, rlen, "%s", t_err);
        return rc;
    }
    DirectParams &P = pl->P;
    memset(&P, 0, sizeof(P));
    P.n = d->n; P.c = d->c; P.h = d->h; P.w = d->w; P.k = d->k; P.p = p; P.q = q;
    P.ks = d->r; P.stride = d->stride; P.pad = d->pad; P.layout = d->layout;
    P.xs = act_strides(d->layout, d->c, d->h, d->w);
    P.ys = act_strides(d->layout, d->k, p, q);
    auto fail = [&](int code, const char *fmt, ...) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(reason, rlen, fmt, ap);
        va_end(ap);
        set_error("%s", reason);
        return code;
    };
    if (!t) return fail(CONVIO_EINVAL, "null tile");
    if (t->x < 1 || t->y < 1 || t->z < 1 || t->s_b < 1 || t->n_xt < 1 || t->n_yt < 1 || t->n_zt < 1)
        return fail(CONVIO_EINFEASIBLE, "tile fields must be >= 1");
    if (t->layout != d->layout)
        return fail(CONVIO_EINVAL, "tile layout %d differs from tensor layout %d", t->layout, d->layout);
    if (t->x % t->n_xt || t->y % t->n_yt || t->z % t->n_zt)
        return fail(CONVIO_EINFEASIBLE, "thread counts must divide the tile dims");
    if (q % t->x || p % t->y || d->k % t->z)
        return fail(CONVIO_EINFEASIBLE, "tile %dx%dx%d does not divide output %dx%dx%d", t->x, t->y,
                    t->z, q, p, d->k);
    const int tile_w = d->stride * (t->x - 1) + d->s;
    const int tile_h = d->stride * (t->y - 1) + d->r;
    const int64_t vol = (int64_t)t->x * t->y * t->z;
    const int64_t resident = vol + (int64_t)tile_w * tile_h + (int64_t)d->r * d->s * t->z;
    if (resident > t->s_b)
        return fail(CONVIO_EINFEASIBLE, "stage 0 resident set %lld words exceeds s_b=%d",
                    (long long)resident, t->s_b);
    const int threads = t->n_xt * t->n_yt * t->n_zt;
    if (threads > 1024) return fail(CONVIO_EINFEASIBLE, "%d threads per block > 1024", threads);
    const int TX = t->x / t->n_xt, TY = t->y / t->n_yt, TZ = t->z / t->n_zt;
    DirectKernelFn fn = nullptr;
    if (d->r == d->s) fn = find_direct_kernel(d->r, d->stride, TX, TY, TZ);
    if (!fn)
        return fail(CONVIO_EINFEASIBLE,
                    "no compiled micro-tile TX=%d TY=%d TZ=%d for %dx%d stride %d", TX, TY, TZ,
                    d->s, d->r, d->stride);
    // staging: registers hold the xyz outputs; s_b - xyz words stage inputs
    // and filters, `ck` channels per stage, double-buffered when it fits.
    const int pitch = choose_pitch(tile_w, t->n_xt, t->n_yt, threads, TX * d->stride,
                                   TY * d->stride);
    const int64_t per_ch = (int64_t)tile_h * pitch + (int64_t)d->r * d->s * t->z;
    const int64_t budget = (int64_t)t->s_b - vol;
    int stages = budget >= 2 * per_ch ? 2 : 1;
    int64_t ck = budget / (stages * per_ch);
    ck = std::max<int64_t>(1, std::min<int64_t>(ck, 16));
    ck = std::min<int64_t>(ck, d->c);
    auto stage_bytes = [&](int64_t cks) {
        int64_t in_stage = (cks * tile_h * pitch + 3) & ~3LL;
        int64_t w_stage = cks * d->r * d->s * t->z;
        return 4 * (in_stage + w_stage);
    };
    while (ck > 1 && stages * stage_bytes(ck) > kSmemCapBytes) --ck;
    if (stages * stage_bytes(ck) > kSmemCapBytes && stages == 2) stages = 1;
    if (stages * stage_bytes(ck) > kSmemCapBytes)
        return fail(CONVIO_EINFEASIBLE, "staging needs %lld B of shared memory > 227 KB",
                    (long long)(stages * stage_bytes(ck)));
    P.bx = t->x; P.by = t->y; P.bz = t->z;
    P.nxt = t->n_xt; P.nyt = t->n_yt; P.nzt = t->n_zt;
    P.ck = (int)ck; P.stages = stages;
    P.tile_w = tile_w; P.tile_h = tile_h; P.pitch = pitch;
    P.in_stage = (int)((ck * tile_h * pitch + 3) & ~3LL);
    P.w_stage = (int)(ck * d->r * d->s * t->z);
    P.tiles_x = q / t->x; P.tiles_y = p / t->y;
    pl->grid = dim3(d->k / t->z, P.tiles_x * P.tiles_y, d->n);
    if (pl->grid.y > 65535 || pl->grid.z > 65535)
        return fail(CONVIO_EINFEASIBLE, "grid %u x %u x %u exceeds launch limits", pl->grid.x,
                    pl->grid.y, pl->grid.z);
    pl->fn = fn;
    pl->threads = threads;
    pl->smem = (size_t)stages * stage_bytes(ck);
    const DevInfo &dev = dev_info();
    if (dev.ok) {
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, (const void *)fn) == cudaSuccess) pl->regs = fa.numRegs;
        if ((int)pl->smem > dev.max_smem_optin)
            return fail(CONVIO_EINFEASIBLE, "smem %zu > device opt-in max %d", pl->smem,
                        dev.max_smem_optin);
        if (pl->smem > 48 * 1024)
            cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pl->smem);
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, (const void *)fn, threads,
                                                          pl->smem) != cudaSuccess ||
            blocks < 1) {
            cudaGetLastError();
            return fail(CONVIO_EINFEASIBLE,
                        "block of %d threads x %d regs + %zu B smem does not fit an SM", threads,
                        pl->regs, pl->smem);
        }
    }
    return CONVIO_OK;
}

// Default device tile when the caller passes none: the largest register
// micro-tile family that divides the output, ~128-256 threads per block.
static int default_direct_tile(const convio_conv_desc *d, convio_tile *out) {
    int p = 0, q = 0;
    int rc = check_desc(d, &p, &q);
    if (rc) return rc;
    static const int txs[] = {8, 7, 4, 2, 1};
    static const int tzs[] = {8, 4, 16, 2, 1};
    static const int tys[] = {1, 2};
    double best_score = -1;
    convio_tile best{};
    for (int TX : txs)
        for (int TZ : tzs)
            for (int TY : tys) {
                if (q % TX || p % TY || d->k % TZ) continue;
                for (int nxt = 1; nxt <= 32; ++nxt) {
                    if (q % (nxt * TX)) continue;
                    for (int nzt = 1; nzt <= 16; ++nzt) {
                        if (d->k % (nzt * TZ)) continue;
                        for (int nyt = 1; nyt <= 64; ++nyt) {
                            if (p % (nyt * TY)) continue;
                            const int threads = nxt * nyt * nzt;
                            if (threads < 32 || threads > 512) continue;
                            convio_tile t{nxt * TX, nyt * TY, nzt * TZ, 0, nxt, nyt, nzt, d->layout, 0};
                            const int tile_w = d->stride * (t.x - 1) + d->s;
                            const int tile_h = d->stride * (t.y - 1) + d->r;
                            const int64_t vol = (int64_t)t.x * t.y * t.z;
                            const int64_t per_ch = (int64_t)tile_h * (tile_w + 1) + d->r * d->s * t.z;
                            t.s_b = (int)std::min<int64_t>(vol + 2 * 8 * per_ch + 64, 1 << 30);
                            DirectPlan pl;
                            char why[160];
                            if (plan_direct(d, &t, &pl, why, sizeof(why)) != CONVIO_OK) continue;
                            const double per_thread = (double)TX * TY * TZ;
                            const double blocks = (double)pl.grid.x * pl.grid.y * pl.grid.z;
                            const int sms = dev_info().ok ? dev_info().sms : 148;
                            const double waves = blocks / (2.0 * sms);
                            double score = std::min(per_thread, 64.0) * 4 +
                                           std::min((double)threads, 256.0) / 64.0 -
                                           (waves < 1.0 ? 40.0 * (1.0 - waves) : 0.0) +
                                           std::min((double)t.z, 64.0) / 16.0;
                            if (score > best_score) {
                                best_score = score;
                                best = t;
                            }
                        }
                    }
                }
            }
    if (best_score < 0) {
        set_error("no compiled tile fits this layer");
        return CONVIO_EINFEASIBLE;
    }
    *out = best;
    return CONVIO_OK;
}

// generic fallback + filter packing kernels
__global__ void direct_conv_f32_generic_kernel(const DirectParams P, int kh, int kw) {
    const int64_t total = (int64_t)P.n * P.k * P.p * P.q;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int ox = idx % P.q;
        const int oy = (idx / P.q) % P.p;
        const int kk = (idx / ((int64_t)P.q * P.p)) % P.k;
        const int b = idx / ((int64_t)P.q * P.p * P.k);
        const float *xb = P.x + b * P.xs.n;
        float acc = 0.0f;
        for (int c = 0; c < P.c; ++c)
            for (int ky = 0; ky < kh; ++ky) {
                const int iy = oy * P.stride + ky - P.pad;
                for (int kx = 0; kx < kw; ++kx) {
                    const int ix = ox * P.stride + kx - P.pad;
                    const float xv = (iy >= 0 && iy < P.h && ix >= 0 && ix < P.w)
                                         ? __ldg(xb + c * P.xs.c + iy * P.xs.y + ix * P.xs.x)
                                         : 0.0f;
                    acc = fmaf(xv, __ldg(P.wp + ((int64_t)(c * kh + ky) * kw + kx) * P.k + kk), acc);
                }
            }
        if (P.bias) acc += P.bias[kk];
        if (P.relu) acc = fmaxf(acc, 0.0f);
        P.y[b * P.ys.n + kk * P.ys.c + oy * P.ys.y + ox * P.ys.x] = acc;
    }
}

__global__ void pack_filter_direct_kernel(const float *w, float *wp, int k, int c, int rs) {
    const int64_t total = (int64_t)k * c * rs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        // i indexes the destination [c][rs][k] so the stores are coalesced
        const int kk = i % k;
        const int tap = (i / k) % rs;
        const int cc = i / ((int64_t)k * rs);
        wp[i] = w[((int64_t)kk * c + cc) * rs + tap];
    }
}

// ---------------------------------------------------------------------------
// FP32 FFMA peak probe
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) ffma_peak_kernel(float *sink, int iters) {
    float a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 1e-7f + j;
    const float b = 0.9999f + threadIdx.x * 1e-9f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], b, a[(j + 1) & 15]);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j];
    if (s == 1234.5f) sink[blockIdx.x] = s;
}

}  // namespace convio

using namespace convio;

extern "C" {

int convio_version(void) { return 100; }

const char *convio_last_error(void) { return t_err; }

int convio_last_launch_count(void) { return t_launches; }

static void fill_info_direct(const DirectPlan &pl, convio_launch_info *out,
                             const convio_conv_desc *d) {
    out->legal = 1;
    out->grid_x = pl.grid.x; out->grid_y = pl.grid.y; out->grid_z = pl.grid.z;
    out->block_threads = pl.threads;
    out->smem_bytes = (int)pl.smem;
    out->regs_per_thread = pl.regs;
    out->channel_chunk = pl.P.ck;
    out->stages = pl.P.stages;
    out->smem_pitch = pl.P.pitch;
    out->p = pl.P.p; out->q = pl.P.q;
    out->flops = 2LL * d->n * d->k * pl.P.p * pl.P.q * (int64_t)d->c * d->r * d->s;
    out->workspace_bytes = 4LL * d->k * d->c * d->r * d->s;
    out->reason[0] = 0;
}

int convio_query(const convio_conv_desc *desc, const convio_tile *tile, int32_t algorithm,
                 convio_launch_info *out) {
    clear_error();
    if (!out) {
        set_error("null output");
        return CONVIO_EINVAL;
    }
    memset(out, 0, sizeof(*out));
    if (algorithm == CONVIO_ALG_DIRECT) {
        DirectPlan pl;
        int rc = plan_direct(desc, tile, &pl, out->reason, sizeof(out->reason));
        if (rc == CONVIO_OK) fill_info_direct(pl, out, desc);
        return rc;
    }
    if (algorithm == CONVIO_ALG_WINOGRAD) return winograd_query(desc, tile, out);
    set_error("unknown algorithm %d", algorithm);
    return CONVIO_EINVAL;
}

int64_t convio_workspace_bytes(const convio_conv_desc *desc, const convio_tile *tile,
                               int32_t algorithm) {
    (void)tile;
    if (!desc) return -1;
    if (algorithm == CONVIO_ALG_DIRECT) return 4LL * desc->k * desc->c * desc->r * desc->s;
    if (algorithm == CONVIO_ALG_WINOGRAD) return winograd_workspace_bytes(desc, tile);
    return -1;
}

int convio_pack_filter_direct(const convio_conv_desc *desc, const float *w, float *w_packed,
                              void *stream) {
    clear_error();
    int p, q;
    int rc = check_desc(desc, &p, &q);
    if (rc) return rc;
    if (!w || !w_packed) {
        set_error("null filter pointer");
        return CONVIO_EINVAL;
    }
    const int64_t total = (int64_t)desc->k * desc->c * desc->r * desc->s;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
    pack_filter_direct_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(w, w_packed, desc->k, desc->c,
                                                                        desc->r * desc->s);
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

int convio_conv_direct_f32(const convio_conv_desc *desc, const convio_tile *tile, const float *x,
                           const float *w, int32_t w_is_packed, const float *bias, int32_t relu,
                           float *y, void *workspace, size_t workspace_bytes, void *stream) {
    clear_error();
    reset_launches();
    int p, q;
    int rc = check_desc(desc, &p, &q);
    if (rc) return rc;
    if (!x || !w || !y) {
        set_error("null tensor pointer");
        return CONVIO_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    convio_tile chosen;
    DirectPlan pl;
    char why[160];
    bool generic = false;
    if (!tile) {
        if (default_direct_tile(desc, &chosen) == CONVIO_OK) {
            tile = &chosen;
        } else {
            generic = true;
        }
    }
    if (!generic) {
        rc = plan_direct(desc, tile, &pl, why, sizeof(why));
        if (rc) return rc;
    } else {
        memset(&pl.P, 0, sizeof(pl.P));
        pl.P.n = desc->n; pl.P.c = desc->c; pl.P.h = desc->h; pl.P.w = desc->w;
        pl.P.k = desc->k; pl.P.p = p; pl.P.q = q; pl.P.ks = desc->r;
        pl.P.stride = desc->stride; pl.P.pad = desc->pad; pl.P.layout = desc->layout;
        pl.P.xs = act_strides(desc->layout, desc->c, desc->h, desc->w);
        pl.P.ys = act_strides(desc->layout, desc->k, p, q);
    }
    const float *wp = w;
    if (!w_is_packed) {
        const size_t need = 4ULL * desc->k * desc->c * desc->r * desc->s;
        if (!workspace || workspace_bytes < need) {
            set_error("workspace of %zu bytes needed for the packed filter", need);
            return CONVIO_EINVAL;
        }
        rc = convio_pack_filter_direct(desc, w, (float *)workspace, stream);
        if (rc) return rc;
        wp = (const float *)workspace;
    }
    pl.P.x = x; pl.P.wp = wp; pl.P.bias = bias; pl.P.y = y; pl.P.relu = relu;
    if (generic) {
        const int64_t total = (int64_t)desc->n * desc->k * p * q;
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
        direct_conv_f32_generic_kernel<<<blocks, 256, 0, st>>>(pl.P, desc->r, desc->s);
    } else {
        pl.fn<<<pl.grid, pl.threads, pl.smem, st>>>(pl.P);
    }
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

int convio_ffma_peak(float *sink, int32_t blocks, int32_t iters, int64_t *flops, void *stream) {
    clear_error();
    if (!sink || blocks < 1 || iters < 1) {
        set_error("bad ffma probe arguments");
        return CONVIO_EINVAL;
    }
    ffma_peak_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(sink, iters);
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    if (flops) *flops = 2LL * blocks * 256 * (int64_t)iters * 8 * 16;
    return CONVIO_OK;
}

}  // extern "C"
