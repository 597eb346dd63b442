// Winograd F(e x e, 3 x 3) host side: filter transform, the device
// projection of a TileConfig, and the C entry points.
#include <stdarg.h>
#include <algorithm>
#include <array>
#include <map>
#include <mutex>

#include "winograd_fp32.cuh"

namespace convio {

// ---- compiled instances: (E, TZ, TP, UPT) -----------------------------------
#define CONVIO_WI(E, TZ, TP, U) {E, TZ, TP, U, &winograd_f32_kernel<E, TZ, TP, U>}
#define CONVIO_WI_U4(E, TZ, TP) \
    CONVIO_WI(E, TZ, TP, 1), CONVIO_WI(E, TZ, TP, 2), CONVIO_WI(E, TZ, TP, 3), CONVIO_WI(E, TZ, TP, 4)
#define CONVIO_WI_FAMILY(E)                                                                  \
    CONVIO_WI_U4(E, 4, 2), CONVIO_WI_U4(E, 4, 4), CONVIO_WI_U4(E, 4, 8), CONVIO_WI_U4(E, 8, 2), \
        CONVIO_WI_U4(E, 8, 4), CONVIO_WI(E, 8, 8, 1), CONVIO_WI(E, 8, 8, 2),                   \
        CONVIO_WI_U4(E, 4, 1), CONVIO_WI_U4(E, 8, 1), CONVIO_WI_U4(E, 16, 1),                  \
        CONVIO_WI(E, 2, 2, 1), CONVIO_WI(E, 2, 2, 2), CONVIO_WI(E, 2, 1, 1), CONVIO_WI(E, 1, 1, 1), \
        CONVIO_WI(E, 1, 2, 1)

struct WinoEntry {
    int e, tz, tp, upt;
    WinoKernelFn fn;
};

static const WinoEntry kWinoEntries[] = {CONVIO_WI_FAMILY(2), CONVIO_WI_FAMILY(4)};

WinoKernelFn find_winograd_kernel(int e, int tz, int tp, int upt) {
    for (const WinoEntry &en : kWinoEntries)
        if (en.e == e && en.tz == tz && en.tp == tp && en.upt == upt) return en.fn;
    return nullptr;
}

// ---- transform matrices (Lavin & Gray), row-major ---------------------------
static const float kG2[4 * 3] = {1, 0, 0, 0.5f, 0.5f, 0.5f, 0.5f, -0.5f, 0.5f, 0, 0, 1};
static const float kBT2[4 * 4] = {1, 0, -1, 0, 0, 1, 1, 0, 0, -1, 1, 0, 0, 1, 0, -1};
static const float kAT2[2 * 4] = {1, 1, 1, 0, 0, 1, -1, -1};
static const float kG4[6 * 3] = {1.0f / 4,  0,          0,         -1.0f / 6, -1.0f / 6, -1.0f / 6,
                                 -1.0f / 6, 1.0f / 6,   -1.0f / 6, 1.0f / 24, 1.0f / 12, 1.0f / 6,
                                 1.0f / 24, -1.0f / 12, 1.0f / 6,  0,         0,         1};
static const float kBT4[6 * 6] = {4, 0, -5, 0,  1, 0, 0, -4, -4, 1,  1, 0, 0, 4, -4, -1, 1, 0,
                                  0, -2, -1, 2, 1, 0, 0, 2,  -1, -2, 1, 0, 0, 4, 0,  -5, 0, 1};
static const float kAT4[4 * 6] = {1, 1, 1, 1, 1, 0, 0, 1, -1, 2, -2, 0,
                                  0, 1, 1, 4, 4, 0, 0, 1, -1, 8, -8, 1};

struct GMat {
    float g[6 * 3];
};

// U[xi][c][k] = (G g G^T)[xi], one thread per (k, c) pair
template <int M>
__global__ void winograd_filter_transform_kernel(const float *w, float *u, int k, int c, GMat G) {
    const int64_t pairs = (int64_t)k * c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pairs;
         i += (int64_t)gridDim.x * blockDim.x) {
        // i = cc * k + kk so the stores of U rows are coalesced over kk
        const int kk = i % k;
        const int cc = i / k;
        const float *g = w + ((int64_t)kk * c + cc) * 9;
        float t[M][3];
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                float s = 0.0f;
#pragma unroll
                for (int b = 0; b < 3; ++b) s = fmaf(G.g[a * 3 + b], g[b * 3 + j], s);
                t[a][j] = s;
            }
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int l = 0; l < M; ++l) {
                float s = 0.0f;
#pragma unroll
                for (int j = 0; j < 3; ++j) s = fmaf(t[a][j], G.g[l * 3 + j], s);
                u[((int64_t)(a * M + l) * c + cc) * k + kk] = s;
            }
    }
}

// ---- device projection ------------------------------------------------------
struct WinoPlan {
    WinoParams P;
    WinoKernelFn fn = nullptr;
    dim3 grid;
    int threads = 0;
    size_t smem = 0;
    int regs = 0;
    int e = 0;
};

static int wino_check_desc(const convio_conv_desc *d, int e, int *p, int *q, char *reason,
                           size_t rlen) {
    if (!d) {
        snprintf(reason, rlen, "null descriptor");
        return CONVIO_EINVAL;
    }
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->k < 1 || d->r < 1 || d->s < 1 ||
        d->stride < 1 || d->pad < 0 || d->layout < 0 || d->layout > 2) {
        snprintf(reason, rlen, "invalid descriptor");
        return CONVIO_EINVAL;
    }
    if (d->stride != 1) {
        snprintf(reason, rlen, "Winograd requires unit stride");
        return geometry_error();
    }
    if (d->r != 3 || d->s != 3) {
        snprintf(reason, rlen, "Winograd kernels are compiled for 3x3 filters, got %dx%d", d->s, d->r);
        return CONVIO_EINFEASIBLE;
    }
    if (e != 2 && e != 4) {
        snprintf(reason, rlen, "compiled Winograd tiles are F(2,3) and F(4,3), got e=%d", e);
        return CONVIO_EINFEASIBLE;
    }
    const int hp = d->h + 2 * d->pad, wp = d->w + 2 * d->pad;
    if (hp < 3 || wp < 3) {
        snprintf(reason, rlen, "kernel larger than padded input");
        return geometry_error();
    }
    *p = hp - 2;
    *q = wp - 2;
    return CONVIO_OK;
}

static int plan_winograd(const convio_conv_desc *d, const convio_tile *t, int e, WinoPlan *pl,
                         char *reason, size_t rlen) {
    int p = 0, q = 0;
    int rc = wino_check_desc(d, e, &p, &q, reason, rlen);
    auto fail = [&](int code, const char *fmt, ...) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(reason, rlen, fmt, ap);
        va_end(ap);
        set_error("%s", reason);
        return code;
    };
    if (rc) {
        set_error("%s", reason);
        return rc;
    }
    if (!t) return fail(CONVIO_EINVAL, "null tile");
    if (t->x < 1 || t->y < 1 || t->z < 1 || t->s_b < 1 || t->n_xt < 1 || t->n_yt < 1 || t->n_zt < 1)
        return fail(CONVIO_EINFEASIBLE, "tile fields must be >= 1");
    if (t->layout != d->layout)
        return fail(CONVIO_EINVAL, "tile layout %d differs from tensor layout %d", t->layout, d->layout);
    if (t->x % t->n_xt || t->y % t->n_yt || t->z % t->n_zt)
        return fail(CONVIO_EINFEASIBLE, "thread counts must divide the tile dims");
    if (q % t->x || p % t->y || d->k % t->z)
        return fail(schedule_error(), "tile %dx%dx%d does not divide output %dx%dx%d", t->x, t->y,
                    t->z, q, p, d->k);
    if (t->x % e || t->y % e)
        return fail(schedule_error(), "tile dims %dx%d not divisible by e=%d", t->x, t->y, e);
    const int m = e + 2, mm = m * m;
    const int npos = (t->x / e) * (t->y / e);
    // the model's shared-kernel-transform schedule must fit s_b
    // (pkg/src/convio/dataflow.py:268-280 with shared_kernel_transform=True)
    const int64_t resident = 2LL * mm * npos * t->z + (int64_t)npos * mm + 9LL * t->z;
    if (resident > t->s_b)
        return fail(schedule_error(), "stage 0 resident set %lld words exceeds s_b=%d",
                    (long long)resident, t->s_b);
    const int threads = t->n_xt * t->n_yt * t->n_zt;
    if (threads > 1024) return fail(CONVIO_EINFEASIBLE, "%d threads per block > 1024", threads);
    // GEMM decomposition: (xi, TP positions, TZ channels) units dealt
    // round-robin to the `threads` threads; pick the compiled micro-tile with
    // the best FMA-per-shared-load ratio times load balance.
    const WinoEntry *best = nullptr;
    double best_score = -1;
    int best_units = 0;
    for (const WinoEntry &en : kWinoEntries) {
        if (en.e != e || t->z % en.tz || npos % en.tp) continue;
        const int units = mm * (npos / en.tp) * (t->z / en.tz);
        if ((units + threads - 1) / threads != en.upt) continue;
        const double eff = (double)units / ((double)en.upt * threads);
        const double ratio = (double)en.tz * en.tp / (en.tz + en.tp);
        const double score = eff * ratio;
        if (score > best_score) {
            best_score = score;
            best = &en;
            best_units = units;
        }
    }
    if (!best)
        return fail(CONVIO_EINFEASIBLE,
                    "no compiled Winograd micro-tile splits %d units of z=%d x %d positions over %d threads",
                    mm * npos * t->z, t->z, npos, threads);
    const int TP = best->tp, TZ = best->tz;
    WinoKernelFn fn = best->fn;
    WinoParams &P = pl->P;
    memset(&P, 0, sizeof(P));
    P.n = d->n; P.c = d->c; P.h = d->h; P.w = d->w; P.k = d->k; P.p = p; P.q = q;
    P.pad = d->pad; P.layout = d->layout;
    P.xs = act_strides(d->layout, d->c, d->h, d->w);
    P.ys = act_strides(d->layout, d->k, p, q);
    P.bx = t->x; P.by = t->y; P.bz = t->z;
    P.px = t->x / e; P.npos = npos; P.npg = npos / TP; P.nzg = t->z / TZ;
    P.units = best_units;
    P.tile_w = t->x + 2; P.tile_h = t->y + 2;
    bool tma = d->layout == CONVIO_LAYOUT_CHW && d->w % 4 == 0 && ((int64_t)d->h * d->w) % 4 == 0 &&
               d->k % 4 == 0 && t->z % 4 == 0 && t->z <= 256 && P.tile_h <= 256 &&
               ((P.tile_w + 6) & ~3) <= 256;
    // staged rows start at a 16-byte-aligned column: up to 3 leading extras
    P.pitch = ((P.tile_w + 3 + 3) & ~3) | (tma ? 0 : 1);
    if (tma) P.pitch = (P.tile_w + 3 + 3) & ~3;
    P.u_pitch = t->z;                      // U slice is the dense [xi][cc][z] box
    P.v_pitch = (npos + 3) & ~3;
    if (P.v_pitch % 32 == 0) P.v_pitch += 4;
    P.o_pitch = npos | 1;
    auto round32 = [](int64_t v) { return (v + 31) & ~31LL; };
    const int64_t per_ch = (int64_t)P.tile_h * P.pitch + (int64_t)mm * t->z;
    const int64_t budget = (int64_t)t->s_b - (int64_t)mm * npos * t->z;
    auto bytes = [&](int64_t cks, int st) {
        const int64_t ring = st * (round32(cks * P.tile_h * P.pitch) + round32(cks * mm * t->z));
        const int64_t v = 2 * round32(cks * mm * P.v_pitch);
        const int64_t exch = (int64_t)mm * t->z * P.o_pitch;
        return 4 * (round32(std::max(ring + v, exch)) + 4 * st);
    };
    // occupancy first (12 warps/SM), then a pipelined ring, then channels per stage
    int regs_guess = kernel_regs((const void *)fn);
    if (regs_guess <= 0) regs_guess = 128;
    const int warps_per_block = (threads + 31) / 32;
    const int regs_per_warp = ((regs_guess * 32 + 255) / 256) * 256;
    const int by_regs = 65536 / std::max(1, regs_per_warp * warps_per_block);
    const int by_threads = 2048 / threads;
    int stages = 1;
    int64_t ck = 1;
    double ring_score = -1;
    for (int st = 1; st <= 3; ++st) {
        for (int64_t cks = 1; cks <= std::min<int64_t>(16, d->c); cks *= 2) {
            if (st * cks * per_ch > budget && !(st == 1 && cks == 1)) continue;
            const int64_t by = bytes(cks, st);
            if (by > 227 * 1024) continue;
            const int by_smem = (int)((228 * 1024) / (by + 1024));
            const int blocks = std::min(std::min(by_regs, by_threads), std::min(by_smem, 32));
            if (blocks < 1) continue;
            const double score = std::min(blocks * warps_per_block, 12) * 1000.0 +
                                 (st >= 2 ? 500.0 : 0.0) + (st == 3 ? 100.0 : 0.0) +
                                 std::min<int64_t>(cks * (st > 1 ? st - 1 : 1), 16) * 10.0;
            if (score > ring_score) {
                ring_score = score;
                stages = st;
                ck = cks;
            }
        }
    }
    if (bytes(ck, stages) > 227 * 1024)
        return fail(CONVIO_EINFEASIBLE, "Winograd staging needs %lld B of shared memory > 227 KB",
                    (long long)bytes(ck, stages));
    if (tma && stages < 2) tma = false;
    P.ck = (int)ck;
    P.stages = stages;
    P.in_stage = (int)round32(ck * P.tile_h * P.pitch);
    P.u_stage = (int)round32(ck * mm * t->z);
    P.v_floats = (int)round32(ck * mm * P.v_pitch);
    P.use_tma = tma ? 1 : 0;
    P.in_box_bytes = (int)(4 * ck * P.tile_h * P.pitch);
    P.u_box_bytes = (int)(4 * ck * mm * t->z);
    P.bar_off = (int)round32(std::max<int64_t>(stages * (P.in_stage + P.u_stage) + 2LL * P.v_floats,
                                               (int64_t)mm * t->z * P.o_pitch));
    P.tiles_x = q / t->x; P.tiles_y = p / t->y;
    pl->grid = dim3(d->k / t->z, P.tiles_x * P.tiles_y, d->n);
    if (pl->grid.y > 65535 || pl->grid.z > 65535)
        return fail(CONVIO_EINFEASIBLE, "grid exceeds launch limits");
    pl->fn = fn;
    pl->threads = threads;
    pl->smem = (size_t)bytes(ck, stages);
    pl->e = e;
    if (launch_fit((const void *)fn, threads, pl->smem, &pl->regs) < 1)
        return fail(CONVIO_EINFEASIBLE, "block of %d threads x %d regs + %zu B smem does not fit an SM",
                    threads, pl->regs, pl->smem);
    return CONVIO_OK;
}

int winograd_default_tile(const convio_conv_desc *d, int e, convio_tile *out);

static bool make_winograd_tensor_maps(const WinoParams &P, int e, CUtensorMap *tm_in, CUtensorMap *tm_u) {
    // the input box exactly as the direct kernel's (same 16-byte-aligned start rule)
    DirectParams D;
    memset(&D, 0, sizeof(D));
    D.x = P.x; D.wp = P.u; D.n = P.n; D.c = P.c; D.h = P.h; D.w = P.w; D.k = P.k;
    D.pitch = P.pitch; D.tile_h = P.tile_h; D.ck = P.ck; D.ks = 1; D.bz = P.bz;
    CUtensorMap dummy;
    if (!make_direct_tensor_maps(D, tm_in, &dummy)) return false;
    const int mm = (e + 2) * (e + 2);
    if (reinterpret_cast<uintptr_t>(P.u) & 15) return false;
    cuuint64_t dim[3] = {(cuuint64_t)P.k, (cuuint64_t)P.c, (cuuint64_t)mm};
    cuuint64_t str[2] = {(cuuint64_t)P.k * 4, (cuuint64_t)P.c * P.k * 4};
    cuuint32_t box[3] = {(cuuint32_t)P.bz, (cuuint32_t)P.ck, (cuuint32_t)mm};
    cuuint32_t es[3] = {1, 1, 1};
    return encode_tensor_map_tiled(tm_u, 3, const_cast<float *>(P.u), dim, str, box, es);
}

static int default_winograd_tile(const convio_conv_desc *d, int e, convio_tile *out) {
    int p = 0, q = 0;
    char why[160];
    int rc = wino_check_desc(d, e, &p, &q, why, sizeof(why));
    if (rc) {
        set_error("%s", why);
        return rc;
    }
    const int m = e + 2, mm = m * m;
    double best = -1;
    convio_tile bt{};
    for (int x = e; x <= std::min(q, 64); x += e) {
        if (q % x) continue;
        for (int y = e; y <= std::min(p, 64); y += e) {
            if (p % y) continue;
            const int npos = (x / e) * (y / e);
            if (npos > 64) continue;
            for (int z = 4; z <= std::min(d->k, 128); z *= 2) {
                if (d->k % z) continue;
                for (int threads = 64; threads <= 512; threads *= 2) {
                    // split threads over the tile axes: n_zt | z, n_xt | x, n_yt | y
                    int nxt = -1, nyt = -1, nzt = -1;
                    for (int a = 1; a <= x && nxt < 0; ++a) {
                        if (x % a) continue;
                        for (int b = 1; b <= y && nxt < 0; ++b) {
                            if (y % b || threads % (a * b)) continue;
                            const int c = threads / (a * b);
                            if (z % c == 0) { nxt = a; nyt = b; nzt = c; }
                        }
                    }
                    if (nxt < 0) continue;
                    convio_tile t{x, y, z, 0, nxt, nyt, nzt, d->layout, e};
                    const int64_t res = 2LL * mm * npos * z + (int64_t)npos * mm + 9LL * z;
                    const int64_t stage = (int64_t)(y + 2) * ((x + 2) | 1) + mm * (z + 4) + mm * (npos + 4);
                    t.s_b = (int)std::max<int64_t>(res, (int64_t)mm * npos * z + 2 * 8 * stage);
                    WinoPlan pl;
                    if (plan_winograd(d, &t, e, &pl, why, sizeof(why)) != CONVIO_OK) continue;
                    const double blocks = (double)pl.grid.x * pl.grid.y * pl.grid.z;
                    const double waves = blocks / 296.0;
                    const double per_thread = (double)mm * npos * z / threads;
                    const double reuse = (double)z * npos / (z + npos);
                    double score = std::min(per_thread, 64.0) * 2 + reuse -
                                   (waves < 1.0 ? 60.0 * (1.0 - waves) : 0.0) -
                                   (per_thread > 128 ? 1000.0 : 0.0);
                    if (score > best) {
                        best = score;
                        bt = t;
                    }
                }
            }
        }
    }
    if (best < 0) {
        set_error("no compiled Winograd tile fits this layer");
        return CONVIO_EINFEASIBLE;
    }
    *out = bt;
    return CONVIO_OK;
}

int winograd_default_tile(const convio_conv_desc *d, int e, convio_tile *out) {
    static std::mutex mu;
    static std::map<std::array<int, 11>, convio_tile> cache;
    std::array<int, 11> key{d->n, d->c, d->h, d->w, d->k, d->r, d->s, d->stride, d->pad, d->layout, e};
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *out = it->second;
            return CONVIO_OK;
        }
    }
    int rc = default_winograd_tile(d, e, out);
    if (rc == CONVIO_OK) {
        std::lock_guard<std::mutex> lock(mu);
        cache[key] = *out;
    }
    return rc;
}

int winograd_query(const convio_conv_desc *d, const convio_tile *t, convio_launch_info *out) {
    const int e = t ? (t->e ? t->e : 2) : 2;
    WinoPlan pl;
    int rc = plan_winograd(d, t, e, &pl, out->reason, sizeof(out->reason));
    if (rc) return rc;
    out->legal = 1;
    out->grid_x = pl.grid.x; out->grid_y = pl.grid.y; out->grid_z = pl.grid.z;
    out->block_threads = pl.threads;
    out->smem_bytes = (int)pl.smem;
    out->regs_per_thread = pl.regs;
    out->channel_chunk = pl.P.ck;
    out->stages = pl.P.stages;
    out->smem_pitch = pl.P.pitch;
    out->p = pl.P.p; out->q = pl.P.q;
    const int m = e + 2;
    const int64_t tiles = (int64_t)d->n * ((pl.P.p + e - 1) / e) * ((pl.P.q + e - 1) / e);
    out->flops = 2LL * m * m * tiles * d->k * d->c;   // element-wise GEMM flops
    out->workspace_bytes = winograd_workspace_bytes(d, t);
    return CONVIO_OK;
}

int64_t winograd_workspace_bytes(const convio_conv_desc *d, const convio_tile *t) {
    const int e = t && t->e ? t->e : 4;
    const int m = std::max(e, 4) + 2;
    return 4LL * m * m * d->c * d->k;
}

}  // namespace convio

using namespace convio;

extern "C" {

int convio_winograd_matrices(int32_t e, int32_t r, float *at, float *g, float *bt) {
    clear_error();
    if (r != 3 || (e != 2 && e != 4)) {
        set_error("compiled Winograd transforms exist for F(2,3) and F(4,3) only");
        return CONVIO_EINFEASIBLE;
    }
    const int m = e + 2;
    if (at) memcpy(at, e == 2 ? kAT2 : kAT4, sizeof(float) * e * m);
    if (g) memcpy(g, e == 2 ? kG2 : kG4, sizeof(float) * m * 3);
    if (bt) memcpy(bt, e == 2 ? kBT2 : kBT4, sizeof(float) * m * m);
    return CONVIO_OK;
}

int convio_winograd_filter_transform(const convio_conv_desc *desc, int32_t e, const float *w,
                                     float *u, void *stream) {
    clear_error();
    int p, q;
    char why[160];
    int rc = wino_check_desc(desc, e, &p, &q, why, sizeof(why));
    if (rc) {
        set_error("%s", why);
        return rc;
    }
    if (!w || !u) {
        set_error("null filter pointer");
        return CONVIO_EINVAL;
    }
    GMat G;
    memset(&G, 0, sizeof(G));
    memcpy(G.g, e == 2 ? kG2 : kG4, sizeof(float) * (e + 2) * 3);
    const int64_t pairs = (int64_t)desc->k * desc->c;
    const int blocks = (int)std::min<int64_t>((pairs + 127) / 128, 4096);
    if (e == 2)
        winograd_filter_transform_kernel<4><<<blocks, 128, 0, (cudaStream_t)stream>>>(w, u, desc->k, desc->c, G);
    else
        winograd_filter_transform_kernel<6><<<blocks, 128, 0, (cudaStream_t)stream>>>(w, u, desc->k, desc->c, G);
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

int convio_conv_winograd_f32(const convio_conv_desc *desc, const convio_tile *tile, int32_t e,
                             const float *x, const float *w, int32_t w_is_transformed,
                             const float *bias, int32_t relu, float *y, void *workspace,
                             size_t workspace_bytes, void *stream) {
    clear_error();
    reset_launches();
    if (!x || !w || !y) {
        set_error("null tensor pointer");
        return CONVIO_EINVAL;
    }
    convio_tile chosen;
    if (!tile) {
        int rc = winograd_default_tile(desc, e, &chosen);
        if (rc) return rc;
        tile = &chosen;
    }
    if (tile->e && tile->e != e) {
        set_error("tile e=%d differs from requested e=%d", tile->e, e);
        return CONVIO_EINVAL;
    }
    WinoPlan pl;
    char why[160];
    int rc = plan_winograd(desc, tile, e, &pl, why, sizeof(why));
    if (rc) return rc;
    const float *u = w;
    if (!w_is_transformed) {
        const size_t need = 4ULL * (e + 2) * (e + 2) * desc->c * desc->k;
        if (!workspace || workspace_bytes < need) {
            set_error("workspace of %zu bytes needed for the transformed filter", need);
            return CONVIO_EINVAL;
        }
        rc = convio_winograd_filter_transform(desc, e, w, (float *)workspace, stream);
        if (rc) return rc;
        u = (const float *)workspace;
        reset_launches();
        note_launch();
    }
    pl.P.x = x; pl.P.u = u; pl.P.bias = bias; pl.P.y = y; pl.P.relu = relu;
    CUtensorMap tm_in, tm_u;
    memset(&tm_in, 0, sizeof(tm_in));
    memset(&tm_u, 0, sizeof(tm_u));
    if (pl.P.use_tma && !make_winograd_tensor_maps(pl.P, e, &tm_in, &tm_u)) pl.P.use_tma = 0;
    pl.fn<<<pl.grid, pl.threads, pl.smem, (cudaStream_t)stream>>>(pl.P, tm_in, tm_u);
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

}  // extern "C"
