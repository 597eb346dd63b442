// Direct convolution, FP32 on CUDA cores: the paper's output-stationary
// dataflow (reference pkg/src/convio/dataflow.py:219-250) on sm_100a.
//
// Block  = one x*y*z output sub-block (TileConfig x, y, z), resident in
//          registers for the whole channel loop (output-stationary).
// Thread = an x/n_xt * y/n_yt * z/n_zt register micro-tile (TX, TY, TZ):
//          TX consecutive output columns of TY consecutive rows for TZ
//          consecutive output channels.
// Stage  = `ck` input channels (the paper's alpha; reference alpha = 1): the
//          x' * y' input footprint and the ck*R*S*z filter slice.  The
//          footprint's halo is zero-filled by the copy engine, so padding is
//          never materialised.
// Pipe   = an NS-deep ring of stages in shared memory.
//          TMA path (NCHW, 16-byte-aligned strides): one elected thread
//          issues cp.async.bulk.tensor (4-D input box, 2-D filter box) that
//          completes on a per-stage mbarrier; consumer warps wait on the
//          "full" barrier and release the slot through an "empty" barrier --
//          no block-wide barrier in the main loop.
//          cp.async path (other layouts / unaligned strides): LDGSTS
//          multistage ring, one __syncthreads per stage.
// Inner  = per (channel, ky): KS*TZ weights to registers, then per output
//          row a register row segment of ST*(TX-1)+KS inputs reused across
//          the KS taps ("shift" reuse) -> KS*TX*TZ FFMA per row segment.
// Every output accumulates in (c, ky, kx) order, the reference DAG's
// left-deep summation order (pkg/src/convio/dag.py:274-284), in fp32 FMA.
#pragma once

#include <cudaTypedefs.h>

#include <type_traits>

#include "common.cuh"

namespace convio {

struct DirectParams {
    const float *x;
    const float *wp;      // packed filters [c][ky][kx][k]
    const float *bias;    // [k] or nullptr
    float *y;
    int n, c, h, w, k, p, q;
    int ks, stride, pad, layout;
    ActStrides xs, ys;
    int bx, by, bz;           // block output tile
    int nxt, nyt, nzt;        // threads per axis
    int ck;                   // channels per stage
    int stages;               // ring depth NS (1..4)
    int tile_w, tile_h;       // input footprint x', y'
    int pitch;                // smem row pitch (floats)
    int in_stage;             // floats per input stage (128-B multiple)
    int w_stage;              // floats per weight stage (128-B multiple)
    int tiles_x, tiles_y;
    int relu;
    int use_tma;              // 1: TMA + mbarrier ring, 0: cp.async ring
    int in_box_bytes, w_box_bytes;
    int w_row_shift;          // log2(bz/4) if a power of two, else -1
};

// ---- mbarrier / TMA primitives (PTX) ------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: a pipeline bug (byte count, parity) traps after ~2^28 polls
// (seconds) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0, polls = 0;
    while (true) {
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if (++polls > (1u << 28)) asm volatile("trap;");
    }
}
// `map` is the generic address of a __grid_constant__ kernel parameter; it
// must be taken at kernel scope (a by-reference lambda capture would copy
// the descriptor to local memory, which TMA cannot read).
__device__ __forceinline__ void tma_load_4d(void *dst, uint64_t map, int c0, int c1, int c2,
                                            int c3, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, uint64_t map, int c0, int c1, int c2,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, uint64_t map, int c0, int c1,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// v[t] = src[SH + t] for t < N: the widest aligned load at each position
// (LDS.128 / .64 / .32 on a 16-byte-aligned `src`; the host guarantees
// pitch % 4 == 0 and a 4-aligned thread column offset), exactly N registers.
template <int N, int SH, int P = SH>
__device__ __forceinline__ void load_row_exact(float (&v)[N], const float *src) {
    if constexpr (P < SH + N) {
        if constexpr (P % 4 == 0 && P + 4 <= SH + N) {
            const float4 f = *reinterpret_cast<const float4 *>(src + P);
            v[P - SH] = f.x; v[P - SH + 1] = f.y; v[P - SH + 2] = f.z; v[P - SH + 3] = f.w;
            load_row_exact<N, SH, P + 4>(v, src);
        } else if constexpr (P % 2 == 0 && P + 2 <= SH + N) {
            const float2 f = *reinterpret_cast<const float2 *>(src + P);
            v[P - SH] = f.x; v[P - SH + 1] = f.y;
            load_row_exact<N, SH, P + 2>(v, src);
        } else {
            v[P - SH] = src[P];
            load_row_exact<N, SH, P + 1>(v, src);
        }
    }
}

template <int V>
using IntC = std::integral_constant<int, V>;

template <int KS, int ST, int TX, int TY, int TZ>
__global__ void direct_conv_f32_kernel(const __grid_constant__ DirectParams P,
                                       const __grid_constant__ CUtensorMap tm_in,
                                       const __grid_constant__ CUtensorMap tm_w) {
    extern __shared__ __align__(128) float smem[];
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int t_x = tid % P.nxt;
    const int t_rest = tid / P.nxt;
    const int t_y = t_rest % P.nyt;
    const int t_z = t_rest / P.nyt;

    const int k0 = blockIdx.x * P.bz;
    const int xt = blockIdx.y % P.tiles_x;
    const int yt = blockIdx.y / P.tiles_x;
    const int img = blockIdx.z;
    const int ox0 = xt * P.bx, oy0 = yt * P.by;
    const int iy0 = oy0 * ST - P.pad;
    // the staged footprint starts at a 16-byte-aligned column (TMA requires
    // the innermost box coordinate to be a multiple of 4 floats); `shift`
    // is the offset of the true footprint start inside the staged row
    const int ix0 = ox0 * ST - P.pad;
    const int shift = ((ix0 % 4) + 4) % 4;
    const int ix0a = ix0 - shift;
    const int stage_w = P.tile_w + shift;

    const int NS = P.stages;
    float *in_s = smem;
    float *w_s = smem + NS * P.in_stage;
    uint64_t *full = reinterpret_cast<uint64_t *>(w_s + NS * P.w_stage);
    uint64_t *empty = full + NS;
    const int nwarps = (nthr + 31) >> 5;
    const float *xb = P.x + (int64_t)img * P.xs.n;
    const int nchunks = (P.c + P.ck - 1) / P.ck;

    // ---- producers ---------------------------------------------------------
    const uint64_t map_in = reinterpret_cast<uint64_t>(&tm_in);
    const uint64_t map_w = reinterpret_cast<uint64_t>(&tm_w);
    auto tma_issue = [&](int chunk, int slot) {   // one thread
        uint64_t *bar = full + slot;
        mbar_arrive_expect_tx(bar, P.in_box_bytes + P.w_box_bytes);
        tma_load_4d(in_s + slot * P.in_stage, map_in, ix0a, iy0, chunk * P.ck, img, bar);
        tma_load_2d(w_s + slot * P.w_stage, map_w, k0, chunk * P.ck * KS * KS, bar);
    };
    auto cp_issue = [&](int chunk, int slot) {    // all threads
        const int c0 = chunk * P.ck;
        float *din = in_s + slot * P.in_stage;
        if (P.layout == CONVIO_LAYOUT_CHW && nthr >= 32) {
            // warp-per-row(s): lanes run along the contiguous columns, one
            // uniform division per row instead of three per element
            const int lane = tid & 31, warp = tid >> 5, nfull = nthr >> 5;
            const int lpr = stage_w <= 8 ? 8 : (stage_w <= 16 ? 16 : 32);   // lanes per row
            const int rpi = 32 / lpr;                                      // rows per warp pass
            const int segs = (stage_w + 31) >> 5;
            const int rows = P.ck * P.tile_h;
            const int sub = lane / lpr, lcol = lane - sub * lpr;
            if (warp < nfull) {
                for (int it = warp; it * rpi < rows * segs; it += nfull) {
                    const int rs = it * rpi + sub;
                    if (rs >= rows * segs) break;
                    const int row = segs == 1 ? rs : rs / segs;
                    const int col = (segs == 1 ? 0 : (rs - row * segs) * 32) + lcol;
                    if (col >= stage_w) continue;
                    const int cc = row / P.tile_h, r = row - cc * P.tile_h;
                    const int gc = c0 + cc, gy = iy0 + r, gx = ix0a + col;
                    const bool v = gc < P.c && gy >= 0 && gy < P.h && gx >= 0 && gx < P.w;
                    const float *src = v ? xb + gc * P.xs.c + gy * P.xs.y + gx : P.x;
                    cp_async4(din + (cc * P.tile_h + r) * P.pitch + col, src, v);
                }
            }
        } else {
            const int total = P.ck * P.tile_h * stage_w;
            for (int i = tid; i < total; i += nthr) {
                int cc, r, col;
                if (P.layout == CONVIO_LAYOUT_HWC) {          // channels contiguous
                    cc = i % P.ck;
                    const int t = i / P.ck;
                    col = t % stage_w;
                    r = t / stage_w;
                } else if (P.layout == CONVIO_LAYOUT_CWH) {   // rows contiguous
                    r = i % P.tile_h;
                    const int t = i / P.tile_h;
                    col = t % stage_w;
                    cc = t / stage_w;
                } else {                                      // columns contiguous
                    col = i % stage_w;
                    const int t = i / stage_w;
                    r = t % P.tile_h;
                    cc = t / P.tile_h;
                }
                const int gc = c0 + cc, gy = iy0 + r, gx = ix0a + col;
                const bool v = gc < P.c && gy >= 0 && gy < P.h && gx >= 0 && gx < P.w;
                const float *src = v ? xb + gc * P.xs.c + gy * P.xs.y + gx * P.xs.x : P.x;
                cp_async4(din + (cc * P.tile_h + r) * P.pitch + col, src, v);
            }
        }
        float *dw = w_s + slot * P.w_stage;
        const int rows = P.ck * KS * KS;   // (cc, tap) rows of bz filters
        if ((P.bz & 3) == 0 && (P.k & 3) == 0) {
            const int per_row = P.bz >> 2;
            const int tot = rows * per_row;
            const int sh = P.w_row_shift;   // log2(per_row) when a power of two, else -1
            for (int i = tid; i < tot; i += nthr) {
                const int row = sh >= 0 ? (i >> sh) : i / per_row;
                const int j = (i - row * per_row) << 2;
                const int gc = c0 + row / (KS * KS);
                const bool v = gc < P.c;
                const float *src = v ? P.wp + ((int64_t)c0 * KS * KS + row) * P.k + k0 + j : P.wp;
                cp_async16(dw + row * P.bz + j, src, v);
            }
        } else {
            const int tot = rows * P.bz;
            for (int i = tid; i < tot; i += nthr) {
                const int row = i / P.bz, j = i - row * P.bz;
                const int gc = c0 + row / (KS * KS);
                const bool v = gc < P.c;
                const float *src = v ? P.wp + ((int64_t)c0 * KS * KS + row) * P.k + k0 + j : P.wp;
                cp_async4(dw + row * P.bz + j, src, v);
            }
        }
    };

    // ---- consumers ---------------------------------------------------------
    float acc[TY][TZ][TX];
#pragma unroll
    for (int i = 0; i < TY; ++i)
#pragma unroll
        for (int zz = 0; zz < TZ; ++zz)
#pragma unroll
            for (int xx = 0; xx < TX; ++xx) acc[i][zz][xx] = 0.0f;

    constexpr int SEG = ST * (TX - 1) + KS;
    constexpr bool VEC_IN = ((TX * ST) % 4) == 0;
    const int in_off = (t_y * TY * ST) * P.pitch + t_x * TX * ST;
    const int w_off = t_z * TZ;

    // SH = the block's staged-row shift (compile-time inside, dispatched once
    // per chunk so the register row loads stay exact-width vector loads)
    auto compute_chunk_sh = [&](int slot, auto sh_tag) {
        constexpr int SH = decltype(sh_tag)::value;
        (void)SH;
        const float *ins = in_s + slot * P.in_stage + in_off;
        const float *wss = w_s + slot * P.w_stage + w_off;
        const int ch_stride = P.tile_h * P.pitch;
#pragma unroll 1
        for (int cc = 0; cc < P.ck; ++cc) {
            const float *in_c = ins + cc * ch_stride;
            const float *w_c = wss + cc * (KS * KS) * P.bz;
#pragma unroll
            for (int ky = 0; ky < KS; ++ky) {
                float wr[KS][TZ];
#pragma unroll
                for (int kx = 0; kx < KS; ++kx) {
                    const float *wrow = w_c + (ky * KS + kx) * P.bz;
                    if constexpr (TZ % 4 == 0) {
#pragma unroll
                        for (int j = 0; j < TZ; j += 4) {
                            const float4 v = *reinterpret_cast<const float4 *>(wrow + j);
                            wr[kx][j] = v.x; wr[kx][j + 1] = v.y;
                            wr[kx][j + 2] = v.z; wr[kx][j + 3] = v.w;
                        }
                    } else if constexpr (TZ % 2 == 0) {
#pragma unroll
                        for (int j = 0; j < TZ; j += 2) {
                            const float2 v = *reinterpret_cast<const float2 *>(wrow + j);
                            wr[kx][j] = v.x; wr[kx][j + 1] = v.y;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < TZ; ++j) wr[kx][j] = wrow[j];
                    }
                }
#pragma unroll
                for (int i = 0; i < TY; ++i) {
                    const float *row = in_c + (i * ST + ky) * P.pitch;
                    float xr[SEG];
                    if constexpr (VEC_IN) {
                        load_row_exact<SEG, SH>(xr, row);
                    } else {
#pragma unroll
                        for (int t = 0; t < SEG; ++t) xr[t] = row[shift + t];
                    }
#pragma unroll
                    for (int kx = 0; kx < KS; ++kx)
#pragma unroll
                        for (int zz = 0; zz < TZ; ++zz)
#pragma unroll
                            for (int xx = 0; xx < TX; ++xx)
                                acc[i][zz][xx] = fmaf(xr[xx * ST + kx], wr[kx][zz], acc[i][zz][xx]);
                }
            }
        }
    };
    auto compute_chunk = [&](int slot) {
        if constexpr (VEC_IN) {
            switch (shift) {   // block-uniform
                case 0: compute_chunk_sh(slot, IntC<0>{}); break;
                case 1: compute_chunk_sh(slot, IntC<1>{}); break;
                case 2: compute_chunk_sh(slot, IntC<2>{}); break;
                default: compute_chunk_sh(slot, IntC<3>{}); break;
            }
        } else {
            compute_chunk_sh(slot, IntC<0>{});
        }
    };

    if (P.use_tma) {
        if (tid == 0) {
            for (int s = 0; s < NS; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, nwarps);
            }
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_in));
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_w));
            for (int s = 0; s < NS - 1 && s < nchunks; ++s) tma_issue(s, s);
        }
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            const int slot = chunk % NS;
            mbar_wait(full + slot, (chunk / NS) & 1);
            compute_chunk(slot);
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(empty + slot);
            // refill the slot consumed one iteration ago with chunk + NS - 1
            const int next = chunk + NS - 1;
            if (tid == 0 && next < nchunks) {
                const int nslot = next % NS;
                if (next >= NS) mbar_wait(empty + nslot, ((next / NS) - 1) & 1);
                tma_issue(next, nslot);
            }
        }
    } else {
        const int pre = NS > 1 ? NS - 1 : 1;
        for (int s = 0; s < pre; ++s) {
            if (s < nchunks) cp_issue(s, s);
            cp_async_commit();
        }
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            // the group of `chunk` is complete once at most NS-2 newer groups pend
            if (NS >= 4) cp_async_wait<2>();
            else if (NS == 3) cp_async_wait<1>();
            else cp_async_wait<0>();
            __syncthreads();   // chunk visible to all; slot (chunk-1)%NS free
            if (NS >= 2) {
                const int next = chunk + NS - 1;
                if (next < nchunks) cp_issue(next, next % NS);
                cp_async_commit();
            }
            compute_chunk(chunk % NS);
            if (NS == 1) {
                __syncthreads();
                if (chunk + 1 < nchunks) cp_issue(chunk + 1, 0);
                cp_async_commit();
            }
        }
    }

    // epilogue: optional bias + ReLU, store the register micro-tile
    float *yb = P.y + (int64_t)img * P.ys.n;
    const int oxt = ox0 + t_x * TX;
    const bool vec4 = (TX % 4 == 0) && P.layout == CONVIO_LAYOUT_CHW && (P.q % 4 == 0);
#pragma unroll
    for (int i = 0; i < TY; ++i) {
        const int oy = oy0 + t_y * TY + i;
#pragma unroll
        for (int zz = 0; zz < TZ; ++zz) {
            const int kk = k0 + t_z * TZ + zz;
            const float b = P.bias ? __ldg(P.bias + kk) : 0.0f;
            float *dst = yb + kk * P.ys.c + oy * P.ys.y + oxt * P.ys.x;
            float v[TX];
#pragma unroll
            for (int xx = 0; xx < TX; ++xx) {
                float t = acc[i][zz][xx] + b;
                v[xx] = P.relu ? fmaxf(t, 0.0f) : t;
            }
            if (vec4) {
#pragma unroll
                for (int xx = 0; xx < TX; xx += 4)
                    *reinterpret_cast<float4 *>(dst + xx) = make_float4(v[xx], v[xx + 1], v[xx + 2], v[xx + 3]);
            } else {
#pragma unroll
                for (int xx = 0; xx < TX; ++xx) dst[xx * P.ys.x] = v[xx];
            }
        }
    }
}

// Fallback for shapes without a compiled micro-tile (non-square kernels,
// unusual strides): one thread per output, same (c, ky, kx) order, reads
// through L1.  Never used by the tuner (its tiles are illegal there).
__global__ void direct_conv_f32_generic_kernel(const DirectParams P, int kh, int kw);

// Repack KCRS -> C R S K.
__global__ void pack_filter_direct_kernel(const float *w, float *wp, int k, int c, int rs);

using DirectKernelFn = void (*)(const DirectParams, const CUtensorMap, const CUtensorMap);

// Lookup of the compiled instances: nullptr if (KS, ST, TX, TY, TZ) absent.
DirectKernelFn find_direct_kernel(int ks, int st, int tx, int ty, int tz);

// Build the TMA descriptors of a plan (host); false if TMA cannot describe it.
bool make_direct_tensor_maps(const DirectParams &P, CUtensorMap *tm_in, CUtensorMap *tm_w);
bool encode_tensor_map_tiled(CUtensorMap *map, int rank, void *base, const cuuint64_t *dim,
                             const cuuint64_t *strides, const cuuint32_t *box, const cuuint32_t *es);
bool encode_tensor_map_tiled_ex(CUtensorMap *map, int rank, void *base, const cuuint64_t *dim,
                                const cuuint64_t *strides, const cuuint32_t *box, const cuuint32_t *es,
                                bool swizzle128);
bool encode_tensor_map_bf16_sw128(CUtensorMap *map, int rank, void *base, const cuuint64_t *dim,
                                  const cuuint64_t *strides, const cuuint32_t *box,
                                  const cuuint32_t *es);

}  // namespace convio
