// Direct convolution, FP32 on CUDA cores: the paper's output-stationary
// dataflow (reference pkg/src/convio/dataflow.py:219-250) on sm_100a.
//
// Block  = one x*y*z output sub-block (TileConfig x, y, z), resident in
//          registers for the whole channel loop (output-stationary).
// Thread = an x/n_xt * y/n_yt * z/n_zt register micro-tile (TX, TY, TZ):
//          TX consecutive output columns of TY consecutive rows for TZ
//          consecutive output channels.
// Stage  = `ck` input channels (the paper's alpha, reference alpha = 1): the
//          x' * y' input footprint (halo zero-filled -> padding is never
//          materialised) and the ck*R*S*z filter slice, streamed global ->
//          shared with cp.async (LDGSTS) into a 1- or 2-deep ring.
// Inner  = per (channel, ky): KS*TZ weights to registers, then per output
//          row a register row segment of ST*(TX-1)+KS inputs reused across
//          the KS taps ("shift" reuse) -> KS*TX*TZ FFMA per row segment.
// Every output accumulates in (c, ky, kx) order, the reference DAG's
// left-deep summation order (pkg/src/convio/dag.py:274-284), in fp32 FMA.
#pragma once

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
    int stages;               // 1 or 2
    int tile_w, tile_h;       // input footprint x', y'
    int pitch;                // smem row pitch (floats)
    int in_stage;             // floats per input stage
    int w_stage;              // floats per weight stage
    int tiles_x, tiles_y;
    int relu;
};

template <int KS, int ST, int TX, int TY, int TZ>
__global__ void direct_conv_f32_kernel(const DirectParams P) {
    extern __shared__ __align__(16) float smem[];
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
    const int ix0 = ox0 * ST - P.pad, iy0 = oy0 * ST - P.pad;

    float *in_s = smem;
    float *w_s = smem + P.stages * P.in_stage;
    const float *xb = P.x + (int64_t)img * P.xs.n;
    const int taps_z = KS * KS * P.bz;
    const int nchunks = (P.c + P.ck - 1) / P.ck;

    auto load_chunk = [&](int chunk, int buf) {
        const int c0 = chunk * P.ck;
        float *din = in_s + buf * P.in_stage;
        const int total = P.ck * P.tile_h * P.tile_w;
        for (int i = tid; i < total; i += nthr) {
            int cc, r, col;
            if (P.layout == CONVIO_LAYOUT_HWC) {          // channels contiguous
                cc = i % P.ck;
                const int t = i / P.ck;
                col = t % P.tile_w;
                r = t / P.tile_w;
            } else if (P.layout == CONVIO_LAYOUT_CWH) {   // rows contiguous
                r = i % P.tile_h;
                const int t = i / P.tile_h;
                col = t % P.tile_w;
                cc = t / P.tile_w;
            } else {                                      // columns contiguous
                col = i % P.tile_w;
                const int t = i / P.tile_w;
                r = t % P.tile_h;
                cc = t / P.tile_h;
            }
            const int gc = c0 + cc, gy = iy0 + r, gx = ix0 + col;
            const bool v = gc < P.c && gy >= 0 && gy < P.h && gx >= 0 && gx < P.w;
            const float *src = v ? xb + gc * P.xs.c + gy * P.xs.y + gx * P.xs.x : P.x;
            cp_async4(din + (cc * P.tile_h + r) * P.pitch + col, src, v);
        }
        float *dw = w_s + buf * P.w_stage;
        const int rows = P.ck * KS * KS;   // (cc, tap) rows of bz filters
        if ((P.bz & 3) == 0 && (P.k & 3) == 0) {
            const int per_row = P.bz >> 2;
            const int tot = rows * per_row;
            for (int i = tid; i < tot; i += nthr) {
                const int row = i / per_row, j = (i - row * per_row) << 2;
                const int cc = row / (KS * KS), tap = row - cc * (KS * KS);
                const int gc = c0 + cc;
                const bool v = gc < P.c;
                const float *src = v ? P.wp + ((int64_t)gc * KS * KS + tap) * P.k + k0 + j : P.wp;
                cp_async16(dw + row * P.bz + j, src, v);
            }
        } else {
            const int tot = rows * P.bz;
            for (int i = tid; i < tot; i += nthr) {
                const int row = i / P.bz, j = i - row * P.bz;
                const int cc = row / (KS * KS), tap = row - cc * (KS * KS);
                const int gc = c0 + cc;
                const bool v = gc < P.c;
                const float *src = v ? P.wp + ((int64_t)gc * KS * KS + tap) * P.k + k0 + j : P.wp;
                cp_async4(dw + row * P.bz + j, src, v);
            }
        }
        (void)taps_z;
    };

    float acc[TY][TZ][TX];
#pragma unroll
    for (int i = 0; i < TY; ++i)
#pragma unroll
        for (int zz = 0; zz < TZ; ++zz)
#pragma unroll
            for (int xx = 0; xx < TX; ++xx) acc[i][zz][xx] = 0.0f;

    constexpr int SEG = ST * (TX - 1) + KS;
    const int in_off = (t_y * TY * ST) * P.pitch + t_x * TX * ST;
    const int w_off = t_z * TZ;

    auto compute_chunk = [&](int buf) {
        const float *ins = in_s + buf * P.in_stage + in_off;
        const float *wss = w_s + buf * P.w_stage + w_off;
        const int ch_stride = P.tile_h * P.pitch;
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
#pragma unroll
                    for (int t = 0; t < SEG; ++t) xr[t] = row[t];
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

    if (P.stages >= 2) {
        load_chunk(0, 0);
        cp_async_commit();
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            if (chunk + 1 < nchunks) {
                load_chunk(chunk + 1, (chunk + 1) & 1);
                cp_async_commit();
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            compute_chunk(chunk & 1);
            __syncthreads();
        }
    } else {
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            load_chunk(chunk, 0);
            cp_async_commit();
            cp_async_wait<0>();
            __syncthreads();
            compute_chunk(0);
            __syncthreads();
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

using DirectKernelFn = void (*)(const DirectParams);

// Lookup of the compiled instances: nullptr if (KS, ST, TX, TY, TZ) absent.
DirectKernelFn find_direct_kernel(int ks, int st, int tx, int ty, int tz);

}  // namespace convio
