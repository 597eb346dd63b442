// Winograd F(e x e, 3 x 3) with the element-wise batched GEMM on the tensor
// cores (tcgen05) -- the north star's "TF32/BF16 tcgen05 variant for ...
// Winograd's batched GEMM".  The four steps of the reference DAG
// (pkg/src/convio/dag.py:302-403; schedule dataflow.py:253-310):
//
//   1. input transform   V[xi][t][c] = (B^T d_{t,c} B)[xi]      (winograd_input_tc_kernel)
//   2. kernel transform  U[xi][k][c] = (G g_{k,c} G^T)[xi]      (winograd_filter_tc_kernel,
//                                                                 once per filter: shared)
//   3. products + sum    M[xi][t][k] = sum_c V[xi][t][c] U[xi][k][c]
//                        -> m^2 GEMMs of T x K x C in ONE tcgen05 launch
//                           (igemm_tcgen05_kernel, batched mode)
//   4. output transform  y_{t,k} = A^T M_{t,k} A (+ bias, ReLU)  (winograd_output_tc_kernel)
//
// t = (image, tile row, tile col) with e x e output tiles; NHWC activations.
// The batch is processed in chunks of images whose V and M (the transformed
// tiles) fit a tuned budget (chunk_l2_bytes below); small budgets keep them
// in the 126 MB L2 between the three launches, large ones (measured faster)
// run the whole batch in three launches.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdarg.h>
#include <algorithm>

#include "igemm_tcgen05.cuh"

namespace convio {

// The same Lavin & Gray matrices as winograd.cu / oracle/winograd_mats.py,
// written out so the zero coefficients cost nothing.
template <int E>
struct WinoTf;

template <>
struct WinoTf<2> {   // F(2x2, 3x3), m = 4
    static constexpr int M = 4;
    static constexpr float GMAX = 4.0f;     // (max row abs-sum of B^T = 2)^2
    static constexpr float GROW = 2.0f;     // max row abs-sum of B^T
    template <typename T>
    __device__ __forceinline__ static void bt(const T (&d)[4], T (&o)[4]) {
        o[0] = d[0] - d[2];
        o[1] = d[1] + d[2];
        o[2] = d[2] - d[1];
        o[3] = d[1] - d[3];
    }
    __device__ __forceinline__ static void at(const float (&m)[4], float (&y)[2]) {
        y[0] = m[0] + m[1] + m[2];
        y[1] = m[1] - m[2] - m[3];
    }
    __device__ __forceinline__ static void g(const float (&w)[3], float (&o)[4]) {
        o[0] = w[0];
        o[1] = 0.5f * (w[0] + w[1] + w[2]);
        o[2] = 0.5f * (w[0] - w[1] + w[2]);
        o[3] = w[2];
    }
};

template <>
struct WinoTf<4> {   // F(4x4, 3x3), m = 6
    static constexpr int M = 6;
    static constexpr float GMAX = 100.0f;   // (max row abs-sum of B^T = 10)^2
    static constexpr float GROW = 10.0f;    // max row abs-sum of B^T
    template <typename T>
    __device__ __forceinline__ static void bt(const T (&d)[6], T (&o)[6]) {
        o[0] = fmaf(4.0f, d[0], fmaf(-5.0f, d[2], d[4]));
        o[1] = fmaf(-4.0f, d[1] + d[2], d[3] + d[4]);
        o[2] = fmaf(4.0f, d[1] - d[2], d[4] - d[3]);
        o[3] = fmaf(2.0f, d[3] - d[1], d[4] - d[2]);
        o[4] = fmaf(2.0f, d[1] - d[3], d[4] - d[2]);
        o[5] = fmaf(4.0f, d[1], fmaf(-5.0f, d[3], d[5]));
    }
    __device__ __forceinline__ static void at(const float (&m)[6], float (&y)[4]) {
        const float a = m[1] + m[2], b = m[1] - m[2], c = m[3] + m[4], d = m[3] - m[4];
        y[0] = m[0] + a + c;
        y[1] = fmaf(2.0f, d, b);
        y[2] = fmaf(4.0f, c, a);
        y[3] = fmaf(8.0f, d, b) + m[5];
    }
    __device__ __forceinline__ static void g(const float (&w)[3], float (&o)[6]) {
        o[0] = 0.25f * w[0];
        o[1] = (-1.0f / 6.0f) * (w[0] + w[1] + w[2]);
        o[2] = (-1.0f / 6.0f) * (w[0] - w[1] + w[2]);
        o[3] = (1.0f / 24.0f) * w[0] + (1.0f / 12.0f) * w[1] + (1.0f / 6.0f) * w[2];
        o[4] = (1.0f / 24.0f) * w[0] - (1.0f / 12.0f) * w[1] + (1.0f / 6.0f) * w[2];
        o[5] = w[2];
    }
};

template <typename T>
__device__ __forceinline__ void store_elem(T *p, float v) {
    if constexpr (sizeof(T) == 2)
        *p = __float2bfloat16_rn(v);
    else
        *p = v;
}

struct WinoTcGeom {
    int n, c, h, w, k, pad;
    int p, q;            // output
    int tiles_y, tiles_x;
    int img0, imgs;      // chunk
};

// per-component application of a 1-D transform to 4 channels at once
template <int N, int NO, typename F>
__device__ __forceinline__ void apply4(const float4 (&d)[N], float4 (&o)[NO], F f) {
    float a[N], r[NO];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int i = 0; i < N; ++i) a[i] = reinterpret_cast<const float *>(&d[i])[q];
        f(a, r);
#pragma unroll
        for (int i = 0; i < NO; ++i) reinterpret_cast<float *>(&o[i])[q] = r[i];
    }
}

template <typename T>
__device__ __forceinline__ void store4(T *p, float4 v) {
    if constexpr (sizeof(T) == 2) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t *>(&lo);
        u.y = *reinterpret_cast<uint32_t *>(&hi);
        *reinterpret_cast<uint2 *>(p) = u;
    } else {
        *reinterpret_cast<float4 *>(p) = v;
    }
}

// Step 1: one thread per (tile, 4 channels); channels fastest so every LDG.128
// and every V store is a coalesced warp access (C % 32 == 0 by the plan); each
// channel sees the scalar B^T d B of the one-channel form.
// (The first version -- one thread per channel, 64-bit index math -- was
// instruction-issue bound at ~990 instructions per warp-element.)
template <int E, typename T>
__global__ void __launch_bounds__(128, 3) winograd_input_tc_kernel(const float *__restrict__ x,
                                                                T *__restrict__ v, WinoTcGeom g) {
    pdl_wait();
    constexpr int M = WinoTf<E>::M;
    const int c4n = g.c >> 2;
    const int tpi = g.tiles_y * g.tiles_x;
    const int t_count = tpi * g.imgs;
    const int total = t_count * c4n;
    const int64_t xi_stride = (int64_t)t_count * g.c;
    const int row4 = g.w * c4n;   // float4 per input row
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int t = i / c4n;
        const int c4 = i - t * c4n;
        const int img = t / tpi;
        const int rem = t - img * tpi;
        const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
        const int iy0 = ty * E - g.pad, ix0 = tx * E - g.pad;
        const float4 *xb = reinterpret_cast<const float4 *>(x + (int64_t)(g.img0 + img) * g.h * g.w * g.c) + c4;
        float4 d[M][M];
#pragma unroll
        for (int a = 0; a < M; ++a) {
            const int iy = iy0 + a;
            const bool rok = iy >= 0 && iy < g.h;
#pragma unroll
            for (int b = 0; b < M; ++b) {
                const int ix = ix0 + b;
                d[a][b] = (rok && ix >= 0 && ix < g.w) ? __ldg(xb + iy * row4 + ix * c4n)
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        float4 tmp[M][M];   // tmp[a][j] = (B^T d)[a][j]
#pragma unroll
        for (int j = 0; j < M; ++j) {
            float4 col[M], o[M];
#pragma unroll
            for (int a = 0; a < M; ++a) col[a] = d[a][j];
            apply4<M, M>(col, o, [](const float (&in)[M], float (&out)[M]) { WinoTf<E>::bt(in, out); });
#pragma unroll
            for (int a = 0; a < M; ++a) tmp[a][j] = o[a];
        }
        T *vp = v + (int64_t)t * g.c + 4 * c4;
#pragma unroll
        for (int a = 0; a < M; ++a) {
            float4 o[M];
            apply4<M, M>(tmp[a], o, [](const float (&in)[M], float (&out)[M]) { WinoTf<E>::bt(in, out); });
#pragma unroll
            for (int b = 0; b < M; ++b) store4(vp + (a * M + b) * xi_stride, o[b]);
        }
    }
}

__device__ __forceinline__ void split_f16(float v, float scale, __half &hi, __half &lo) {
    const float s = v * scale;
    hi = __float2half_rn(s);
    lo = __float2half_rn(s - __half2float(hi));
}

// Step 1, 3xF16 form: V = B^T d B as above, then per tile a power-of-two scale
// from the footprint's largest |d| over all C channels (the tile's threads are
// consecutive: c4 fastest) and fp16 hi / lo planes V16[plane][xi][t][c] +
// row_exp[xi][t] for the GEMM epilogue.
// The loop is block-uniform (C / 4 threads of a tile never straddle a block: 128
// is a multiple of C / 4 for C in {64, 128, 256, 512}).
template <int E>
__global__ void __launch_bounds__(128, 3) winograd_input_f16x3_kernel(const float *__restrict__ x,
                                                                   __half *__restrict__ v,
                                                                   int *__restrict__ row_exp,
                                                                   WinoTcGeom g) {
    pdl_wait();
    constexpr int M = WinoTf<E>::M;
    __shared__ float red[4][1];
    const int c4n = g.c >> 2;
    const int tpi = g.tiles_y * g.tiles_x;
    const int t_count = tpi * g.imgs;
    const int total = t_count * c4n;
    const int64_t xi_stride = (int64_t)t_count * g.c;
    const int row4 = g.w * c4n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = blockIdx.x * blockDim.x; base < total; base += gridDim.x * blockDim.x) {
        const int i = base + threadIdx.x;
        const bool active = i < total;
        const int ii = active ? i : total - 1;
        const int t = ii / c4n;
        const int c4 = ii - t * c4n;
        const int img = t / tpi;
        const int rem = t - img * tpi;
        const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
        const int iy0 = ty * E - g.pad, ix0 = tx * E - g.pad;
        const float4 *xb = reinterpret_cast<const float4 *>(x + (int64_t)(g.img0 + img) * g.h * g.w * g.c) + c4;
        float4 d[M][M];
#pragma unroll
        for (int a = 0; a < M; ++a) {
            const int iy = iy0 + a;
            const bool rok = active && iy >= 0 && iy < g.h;
#pragma unroll
            for (int b = 0; b < M; ++b) {
                const int ix = ix0 + b;
                d[a][b] = (rok && ix >= 0 && ix < g.w) ? __ldg(xb + iy * row4 + ix * c4n)
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        float4 tmp[M][M];
#pragma unroll
        for (int j = 0; j < M; ++j) {
            float4 col[M], o[M];
#pragma unroll
            for (int a = 0; a < M; ++a) col[a] = d[a][j];
            apply4<M, M>(col, o, [](const float (&in)[M], float (&out)[M]) { WinoTf<E>::bt(in, out); });
#pragma unroll
            for (int a = 0; a < M; ++a) tmp[a][j] = o[a];
        }
        // one scale per tile: |V| <= GROW * max|B^T d| over the tile's (B^T d) values and
        // channels (GROW = the largest row abs-sum of B^T), so every xi row of the tile fits
        // (-2^15, 2^15); fp16 being floating point, rows below the bound keep their 11 bits.
        // (Taken from B^T d, not d, so the footprint registers are dead across the barrier.)
        float fm = 0.0f;
#pragma unroll
        for (int a = 0; a < M; ++a)
#pragma unroll
            for (int b = 0; b < M; ++b)
                fm = fmaxf(fm, fmaxf(fmaxf(fabsf(tmp[a][b].x), fabsf(tmp[a][b].y)),
                                     fmaxf(fabsf(tmp[a][b].z), fabsf(tmp[a][b].w))));
        const int grp = c4n < 32 ? c4n : 32;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
            if (off < grp) fm = fmaxf(fm, __shfl_xor_sync(0xffffffffu, fm, off));
        if (c4n > 32) {   // the tile spans c4n / 32 warps of this block
            if (lane == 0) red[warp][0] = fm;
            __syncthreads();
            const int w0 = warp & ~(c4n / 32 - 1);
            for (int w = 0; w < c4n / 32; ++w) fm = fmaxf(fm, red[w0 + w][0]);
            __syncthreads();
        }
        const int e = f16_row_exp(fm * WinoTf<E>::GROW);
        const float sc = pow2f(e);
        // pass 2: scaled hi / lo planes (all lanes: the lane-pair exchange below is
        // a full-warp shuffle; inactive lanes skip only the stores)
        {
            __half *vp = v + (int64_t)t * g.c + 4 * c4;
            const int64_t plane = (int64_t)M * M * xi_stride;
#pragma unroll
            for (int a = 0; a < M; ++a) {
                float4 o[M];
                apply4<M, M>(tmp[a], o, [](const float (&in)[M], float (&out)[M]) { WinoTf<E>::bt(in, out); });
#pragma unroll
                for (int b = 0; b < M; ++b) {
                    __half h[4], l[4];
                    split_f16(o[b].x, sc, h[0], l[0]);
                    split_f16(o[b].y, sc, h[1], l[1]);
                    split_f16(o[b].z, sc, h[2], l[2]);
                    split_f16(o[b].w, sc, h[3], l[3]);
                    // lane pairs (c4, c4 + 1) trade halves so each lane stores 16 B of one
                    // plane: even lanes the 8 channels' hi, odd lanes their lo
                    __half *dst = vp + (a * M + b) * xi_stride;
                    const uint2 hv = *reinterpret_cast<const uint2 *>(h);
                    const uint2 lv = *reinterpret_cast<const uint2 *>(l);
                    // every lane of the warp runs the exchange (inactive lanes trade
                    // don't-care halves) so the full-mask shuffle is well defined
                    const bool odd = c4 & 1;
                    const uint2 send = odd ? hv : lv;
                    const uint32_t gx = __shfl_xor_sync(0xffffffffu, send.x, 1),
                                   gy = __shfl_xor_sync(0xffffffffu, send.y, 1);
                    if (!active) continue;
                    if (!odd)
                        *reinterpret_cast<uint4 *>(dst) = make_uint4(hv.x, hv.y, gx, gy);
                    else
                        *reinterpret_cast<uint4 *>(dst - 4 + plane) = make_uint4(gx, gy, lv.x, lv.y);
                    if (c4 == 0) row_exp[(int64_t)(a * M + b) * t_count + t] = e;
                }
            }
        }
    }
}

// 3xF16 kernel operand: U (fp32, [xi][k][c]) -> power-of-two scale per (xi, k) row
// over c, fp16 hi / lo planes U16[plane][xi][k][c] and col_exp[xi][k].  One warp
// per row.
__global__ void __launch_bounds__(256) winograd_u_split_f16x3_kernel(const float *__restrict__ u,
                                                                     __half *__restrict__ u16,
                                                                     int *__restrict__ col_exp,
                                                                     int rows, int c) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t plane = (int64_t)rows * c;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += (gridDim.x * blockDim.x) >> 5) {
        const float *ur = u + (int64_t)r * c;
        float mx = 0.0f;
        for (int j = lane; j < c; j += 32) mx = fmaxf(mx, fabsf(ur[j]));
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        const int e = f16_row_exp(mx);
        const float sc = pow2f(e);
        for (int j = lane; j < c; j += 32) {
            __half h, l;
            split_f16(ur[j], sc, h, l);
            u16[(int64_t)r * c + j] = h;
            u16[plane + (int64_t)r * c + j] = l;
        }
        if (lane == 0) col_exp[r] = e;
    }
}

// Step 2: U[xi][k][c] = (G g G^T)[xi] (K-major B operand of the tensor-core
// GEMM) or, CK = true, U[xi][c][k] (the FFMA GEMM's [channel][n] rows); one
// thread per (k, c), c fastest.
template <int E, typename T, bool CK = false>
__global__ void winograd_filter_tc_kernel(const float *__restrict__ w, T *__restrict__ u, int k,
                                          int c) {
    pdl_wait();
    constexpr int M = WinoTf<E>::M;
    const int64_t pairs = (int64_t)k * c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pairs;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float *g = w + i * 9;   // KCRS: (k, c) pairs are contiguous 3x3 filters
        float t[M][3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            float col[3] = {g[j], g[3 + j], g[6 + j]}, o[M];
            WinoTf<E>::g(col, o);
#pragma unroll
            for (int a = 0; a < M; ++a) t[a][j] = o[a];
        }
#pragma unroll
        for (int a = 0; a < M; ++a) {
            float o[M];
            WinoTf<E>::g(t[a], o);
#pragma unroll
            for (int b = 0; b < M; ++b) {
                const int64_t j = CK ? (i % c) * (int64_t)k + i / c : i;
                store_elem(u + (int64_t)(a * M + b) * pairs + j, o[b]);
            }
        }
    }
}

// Batched step 2 (a step's filter prep in one launch): jobs of one e and a float U,
// thread index over the concatenated (k, c) pairs of all jobs
constexpr int kWinoJobs = 32;
struct WinoFilterBatch {
    int n;
    int64_t cum[kWinoJobs + 1];   // pair (or, for the split, row) prefix sums
    const float *w[kWinoJobs];
    float *u[kWinoJobs];
    int k[kWinoJobs], c[kWinoJobs];
};
template <int E>
__global__ void winograd_filter_tc_batched_kernel(const __grid_constant__ WinoFilterBatch B) {
    pdl_wait();
    constexpr int M = WinoTf<E>::M;
    for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < B.cum[B.n];
         gi += (int64_t)gridDim.x * blockDim.x) {
        int j = 0;
        while (B.cum[j + 1] <= gi) ++j;
        const int64_t i = gi - B.cum[j], pairs = B.cum[j + 1] - B.cum[j];
        const float *g = B.w[j] + i * 9;
        float t[M][3];
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
            float col[3] = {g[jj], g[3 + jj], g[6 + jj]}, o[M];
            WinoTf<E>::g(col, o);
#pragma unroll
            for (int a = 0; a < M; ++a) t[a][jj] = o[a];
        }
#pragma unroll
        for (int a = 0; a < M; ++a) {
            float o[M];
            WinoTf<E>::g(t[a], o);
#pragma unroll
            for (int b = 0; b < M; ++b) B.u[j][(int64_t)(a * M + b) * pairs + i] = o[b];
        }
    }
}
// batched 3xF16 split of U (one warp per (job, xi * k) row, rows concatenated)
__global__ void __launch_bounds__(256) winograd_u_split_f16x3_batched_kernel(const __grid_constant__ WinoFilterBatch B) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int64_t gr = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; gr < B.cum[B.n];
         gr += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int j = 0;
        while (B.cum[j + 1] <= gr) ++j;
        const int64_t r = gr - B.cum[j], rows = B.cum[j + 1] - B.cum[j];
        const int c = B.c[j];
        const float *ur = B.u[j] + r * c;
        __half *u16 = reinterpret_cast<__half *>(B.u[j] + rows * c);
        int *col_exp = reinterpret_cast<int *>(B.u[j] + 2 * rows * c);
        float mx = 0.0f;
        for (int i = lane; i < c; i += 32) mx = fmaxf(mx, fabsf(ur[i]));
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        const int e = f16_row_exp(mx);
        const float sc = pow2f(e);
        for (int i = lane; i < c; i += 32) {
            __half h, l;
            split_f16(ur[i], sc, h, l);
            u16[r * c + i] = h;
            u16[rows * c + r * c + i] = l;
        }
        if (lane == 0) col_exp[r] = e;
    }
}

// U = G g G^T of one 3x3 filter g (9 contiguous floats), o[a * M + b]: the same
// arithmetic as winograd_filter_tc_kernel, so both give identical bits
template <int E>
__device__ __forceinline__ void wino_filter_u(const float *__restrict__ g, float (&o)[WinoTf<E>::M * WinoTf<E>::M]) {
    constexpr int M = WinoTf<E>::M;
    float t[M][3];
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) {
        float col[3] = {g[jj], g[3 + jj], g[6 + jj]}, oc[M];
        WinoTf<E>::g(col, oc);
#pragma unroll
        for (int a = 0; a < M; ++a) t[a][jj] = oc[a];
    }
#pragma unroll
    for (int a = 0; a < M; ++a) {
        float orow[M];
        WinoTf<E>::g(t[a], orow);
#pragma unroll
        for (int b = 0; b < M; ++b) o[a * M + b] = orow[b];
    }
}

// Batched 3xF16 U in ONE pass (no fp32 U round trip through HBM, one launch instead
// of transform + split): one block per (job, output channel k); pass 1 recomputes U
// over the C channels for the per-xi max |U| (-> the row exponents), pass 2 recomputes
// it and writes the hi / lo planes, a channel pair per thread (half2 stores).  B.cum
// here is the prefix sum of K.  Bit-identical to winograd_filter_tc_batched_kernel +
// winograd_u_split_f16x3_batched_kernel (same arithmetic, same split).
template <int E>
__global__ void __launch_bounds__(256) winograd_filter_f16x3_batched_kernel(const __grid_constant__ WinoFilterBatch B) {
    pdl_wait();
    constexpr int M = WinoTf<E>::M, MM = M * M;
    __shared__ float red[8][MM];
    __shared__ float scs[MM];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t gr = blockIdx.x; gr < B.cum[B.n]; gr += gridDim.x) {
        int j = 0;
        while (B.cum[j + 1] <= gr) ++j;
        const int kk = (int)(gr - B.cum[j]), k = B.k[j], c = B.c[j];
        const float *wk = B.w[j] + (int64_t)kk * c * 9;
        const int64_t rows = (int64_t)MM * k;
        __half *u16 = reinterpret_cast<__half *>(B.u[j] + rows * c);
        int *col_exp = reinterpret_cast<int *>(B.u[j] + 2 * rows * c);
        float mx[MM];
#pragma unroll
        for (int q = 0; q < MM; ++q) mx[q] = 0.0f;
        for (int cc = threadIdx.x; cc < c; cc += blockDim.x) {
            const float *g = wk + (int64_t)cc * 9;
            float t[M][3];
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) {
                float col[3] = {g[jj], g[3 + jj], g[6 + jj]}, oc[M];
                WinoTf<E>::g(col, oc);
#pragma unroll
                for (int a = 0; a < M; ++a) t[a][jj] = oc[a];
            }
#pragma unroll
            for (int a = 0; a < M; ++a) {
                float r[M];
                WinoTf<E>::g(t[a], r);
#pragma unroll
                for (int b = 0; b < M; ++b) mx[a * M + b] = fmaxf(mx[a * M + b], fabsf(r[b]));
            }
        }
#pragma unroll
        for (int q = 0; q < MM; ++q) {
            float v = mx[q];
            for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
            if (lane == 0) red[warp][q] = v;
        }
        __syncthreads();
        if (threadIdx.x < MM) {
            float v = red[0][threadIdx.x];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = fmaxf(v, red[w][threadIdx.x]);
            const int e = f16_row_exp(v);
            scs[threadIdx.x] = pow2f(e);
            col_exp[(int64_t)threadIdx.x * k + kk] = e;
        }
        __syncthreads();
        volatile float *vscs = scs;
        const int64_t kc = (int64_t)k * c, lo_off = rows * c;
        for (int p = threadIdx.x; 2 * p < c; p += blockDim.x) {
            // G g (the column pass) for both channels, then one row of U at a time
            float t0[M][3], t1[M][3];
            const float *g0 = wk + (int64_t)(2 * p) * 9, *g1 = g0 + 9;
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) {
                float col0[3] = {g0[jj], g0[3 + jj], g0[6 + jj]}, col1[3] = {g1[jj], g1[3 + jj], g1[6 + jj]};
                float oc0[M], oc1[M];
                WinoTf<E>::g(col0, oc0);
                WinoTf<E>::g(col1, oc1);
#pragma unroll
                for (int a = 0; a < M; ++a) {
                    t0[a][jj] = oc0[a];
                    t1[a][jj] = oc1[a];
                }
            }
            __half *ph = u16 + (int64_t)kk * c + 2 * p;
#pragma unroll
            for (int a = 0; a < M; ++a) {
                float r0[M], r1[M];
                WinoTf<E>::g(t0[a], r0);
                WinoTf<E>::g(t1[a], r1);
#pragma unroll
                for (int b = 0; b < M; ++b) {
                    const int q = a * M + b;
                    __half h0, l0, h1, l1;
                    const float sc = vscs[q];   // re-read per use: keeps 36 scales out of registers
                    split_f16(r0[b], sc, h0, l0);
                    split_f16(r1[b], sc, h1, l1);
                    *reinterpret_cast<__half2 *>(ph) = __halves2half2(h0, h1);
                    *reinterpret_cast<__half2 *>(ph + lo_off) = __halves2half2(l0, l1);
                    ph += kc;   // next xi row: a pointer walk, not 36 hoisted offsets
                }
            }
        }
        __syncthreads();   // red / scs are reused by the next row
    }
}

// Step 4: one thread per (tile, output channel), k fastest (coalesced M
// loads and NHWC stores); bias + ReLU fused; ragged tiles masked.
template <int E>
__global__ void __launch_bounds__(128, 4) winograd_output_tc_kernel(const float *__restrict__ mm,
                                                                 const float *__restrict__ bias,
                                                                 float *__restrict__ y, WinoTcGeom g,
                                                                 int relu) {
    // one thread per (tile, 4 output channels), LDG.128 / STG.128, 32-bit index math
    pdl_wait();
    constexpr int M = WinoTf<E>::M;
    const int k4n = g.k >> 2;
    const int tpi = g.tiles_y * g.tiles_x;
    const int t_count = tpi * g.imgs;
    const int total = t_count * k4n;
    const int64_t xi_stride = (int64_t)t_count * g.k;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int t = i / k4n;
        const int k4 = i - t * k4n;
        const int img = t / tpi;
        const int rem = t - img * tpi;
        const int ty = rem / g.tiles_x, tx = rem - ty * g.tiles_x;
        const float *mp = mm + (int64_t)t * g.k + 4 * k4;
        float4 tmp[E][M];
#pragma unroll
        for (int b = 0; b < M; ++b) {
            float4 col[M], o[E];
#pragma unroll
            for (int a = 0; a < M; ++a) col[a] = __ldg(reinterpret_cast<const float4 *>(mp + (a * M + b) * xi_stride));
            apply4<M, E>(col, o, [](const float (&in)[M], float (&out)[E]) { WinoTf<E>::at(in, out); });
#pragma unroll
            for (int a = 0; a < E; ++a) tmp[a][b] = o[a];
        }
        const float4 bv = bias ? __ldg(reinterpret_cast<const float4 *>(bias) + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 *yb = reinterpret_cast<float4 *>(y + (int64_t)(g.img0 + img) * g.p * g.q * g.k) + k4;
#pragma unroll
        for (int a = 0; a < E; ++a) {
            float4 o[E];
            apply4<M, E>(tmp[a], o, [](const float (&in)[M], float (&out)[E]) { WinoTf<E>::at(in, out); });
            const int oy = ty * E + a;
#pragma unroll
            for (int b = 0; b < E; ++b) {
                const int ox = tx * E + b;
                if (oy < g.p && ox < g.q) {
                    float4 rv = make_float4(o[b].x + bv.x, o[b].y + bv.y, o[b].z + bv.z, o[b].w + bv.w);
                    if (relu) {
                        rv.x = fmaxf(rv.x, 0.f); rv.y = fmaxf(rv.y, 0.f);
                        rv.z = fmaxf(rv.z, 0.f); rv.w = fmaxf(rv.w, 0.f);
                    }
                    yb[(oy * g.q + ox) * k4n] = rv;
                }
            }
        }
    }
}

// KIND_FFMA: the element-wise GEMMs on the CUDA cores (direct_nhwc_f32_kernel
// in batched mode) -- the paper-faithful FP32 path in the same pipeline
constexpr int KIND_FFMA = 3;

static int kind_of_prec(int32_t precision) {
    switch (precision) {
        case CONVIO_PREC_TF32: return KIND_TF32;
        case CONVIO_PREC_3XTF32: return KIND_3XTF32;
        case CONVIO_PREC_BF16: return KIND_BF16;
        case CONVIO_PREC_FP32: return KIND_FFMA;
        case CONVIO_PREC_3XF16: return KIND_3XF16;
        default: return -1;
    }
}

int direct_nhwc_batched_run(int bn, int s_b, int xi, int t_count, int c, int k, const float *v,
                            const float *u, float *m, cudaStream_t stream);

static inline size_t al256(size_t b) { return (b + 255) & ~size_t(255); }

// Budget for one chunk's transformed tiles (V + M) = 16 KB x tile.s_b: s_b =
// 2048 -> 32 MB (L2-resident chunks), 8192 (the default) -> 128 MB, 32768 ->
// 512 MB (the whole ResNet-50 batch at once).  Measured (scripts/
// probe_wtc_chunk.py, 3xTF32 F(4,3), batch 256): the L2-resident chunks lose --
// every chunk pays three launch ramps and wave tails, and the dirty V / M lines
// are written back to HBM anyway -- res3 0.311 ms at 64 MB vs 0.206 ms unchunked,
// res4 0.237 vs 0.161, res5 0.180 vs 0.120; the tuner picks s_b per layer.
static size_t chunk_l2_bytes(int s_b) { return (size_t)16384 * (size_t)std::max(s_b, 64); }

struct WinoTcPlan {
    WinoTcGeom g;
    int e, m, kind, bn, s_b;
    bool pair, tsa;   // CTA pair (n_zt 2 or 4); 3xTF32 A operand in TMEM (n_zt 4)
    int chunk_imgs;
    size_t u_bytes, v_bytes, m_bytes;   // per chunk for V and M
};

static int plan_wino_tc(const convio_conv_desc *d, const convio_tile *t, int e, int32_t precision,
                        WinoTcPlan *pl, char *reason, size_t rlen) {
    auto fail = [&](int code, const char *fmt, ...) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(reason, rlen, fmt, ap);
        va_end(ap);
        set_error("%s", reason);
        return code;
    };
    if (!d) return fail(CONVIO_EINVAL, "null descriptor");
    const int kind = kind_of_prec(precision);
    if (kind < 0) return fail(CONVIO_EINVAL, "unknown precision %d", precision);
    if (e != 2 && e != 4) return fail(CONVIO_EINFEASIBLE, "Winograd e must be 2 or 4 (got %d)", e);
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->k < 1 || d->pad < 0)
        return fail(CONVIO_EINVAL, "descriptor fields must be >= 1 (pad >= 0)");
    if (d->r != 3 || d->s != 3) return fail(CONVIO_EINFEASIBLE, "Winograd needs a 3x3 kernel");
    if (d->stride != 1)
        return fail(geometry_error(), "Winograd requires stride 1 (reference WinogradParams.check_shape)");
    if (d->layout != CONVIO_LAYOUT_HWC)
        return fail(CONVIO_EINFEASIBLE, "tensor-core Winograd needs the HWC (NHWC) layout");
    const int p = d->h + 2 * d->pad - 2, q = d->w + 2 * d->pad - 2;
    if (p < 1 || q < 1) return fail(geometry_error(), "kernel larger than padded input");
    const int cb = (kind == KIND_BF16 || kind == KIND_3XF16) ? 64 : 32;
    if (d->c % cb) return fail(CONVIO_EINFEASIBLE, "C=%d is not a multiple of %d", d->c, cb);
    int bn = t ? t->z : (d->k % 256 == 0 ? 256 : (d->k % 128 == 0 ? 128 : 64));
    int s_b = t ? t->s_b : 8192;
    const bool pair = kind != KIND_FFMA && (t ? (t->n_zt == 2 || t->n_zt == 4) : true);
    const bool tsa = t && t->n_zt == 4;
    if (kind == KIND_3XF16 && (!pair || tsa))
        return fail(CONVIO_EINFEASIBLE, "3xF16 Winograd GEMMs run on the CTA pair (n_zt = 2)");
    if (kind == KIND_3XF16 && (d->c > 512 || (d->c & (d->c - 1))))
        return fail(CONVIO_EINFEASIBLE, "3xF16 input transform: C a power of two in [64, 512]");
    if (tsa && (kind != KIND_3XTF32 || (t->z != 64 && t->z != 128)))
        return fail(CONVIO_EINFEASIBLE, "A-in-TMEM (n_zt = 4) Winograd GEMMs need 3xTF32 and z <= 128");
    if (kind == KIND_FFMA && !t) bn = d->k % 128 == 0 ? 128 : 64;
    if (t && (t->n_xt != 1 || t->n_yt != 1 || (t->n_zt != 1 && t->n_zt != 2 && t->n_zt != 4) ||
              (kind == KIND_FFMA && t->n_zt != 1)))
        return fail(CONVIO_EINFEASIBLE,
                    "Winograd tiles take n_xt = n_yt = 1 and n_zt in {1, 2 (tcgen05 CTA pair), "
                    "4 (pair, A in TMEM)}");
    if (kind == KIND_FFMA && bn != 64 && bn != 128)
        return fail(CONVIO_EINFEASIBLE, "FFMA Winograd GEMM needs z in {64, 128}, got %d", bn);
    if (t && t->layout != d->layout) return fail(CONVIO_EINVAL, "tile layout differs from tensor layout");
    if (t && t->e != e) return fail(CONVIO_EINVAL, "tile e=%d differs from e=%d", t->e, e);
    if (bn != 64 && bn != 128 && bn != 256)
        return fail(CONVIO_EINFEASIBLE, "tcgen05 Winograd needs z in {64, 128, 256}, got %d", bn);
    if (d->k % bn) return fail(CONVIO_EINFEASIBLE, "z=%d does not divide K=%d", bn, d->k);
    const int m = e + 2;
    const size_t es = kind == KIND_BF16 ? 2 : 4;
    WinoTcGeom &g = pl->g;
    g.n = d->n; g.c = d->c; g.h = d->h; g.w = d->w; g.k = d->k; g.pad = d->pad;
    g.p = p; g.q = q;
    g.tiles_y = (p + e - 1) / e; g.tiles_x = (q + e - 1) / e;
    const size_t tpi = (size_t)g.tiles_y * g.tiles_x;
    const size_t per_img = tpi * m * m * ((size_t)d->c * es + (size_t)d->k * 4);
    int chunk = (int)std::max<size_t>(1, chunk_l2_bytes(s_b) / per_img);
    chunk = std::min(chunk, d->n);
    // keep the GEMM's T axis within the TMA box-coordinate / grid limits
    while (chunk > 1 && (size_t)chunk * tpi > (size_t)1 << 24) chunk /= 2;
    if ((size_t)chunk * tpi >= ((size_t)1 << 31)) return fail(CONVIO_EINFEASIBLE, "too many tiles");
    // the transform kernels index a chunk's tiles x channels and an image's
    // pixels x channels in 32-bit arithmetic
    if ((size_t)chunk * tpi * (size_t)std::max(d->c, d->k) >= ((size_t)1 << 31) ||
        (size_t)std::max<int64_t>((int64_t)d->h * d->w, (int64_t)p * q) * (size_t)std::max(d->c, d->k) >=
            ((size_t)1 << 31))
        return fail(CONVIO_EINFEASIBLE, "chunk or image too large for 32-bit transform indexing");
    pl->e = e; pl->m = m; pl->kind = kind; pl->bn = bn; pl->s_b = s_b; pl->pair = pair;
    pl->tsa = tsa;
    pl->chunk_imgs = chunk;
    // 3xF16: U = [fp32 U | fp16 hi plane | fp16 lo plane | col_exp], V = [hi | lo | row_exp]
    const bool f16 = kind == KIND_3XF16;
    pl->u_bytes = al256((size_t)m * m * d->k * d->c * es * (f16 ? 2 : 1) + (f16 ? (size_t)m * m * d->k * 4 : 0));
    pl->v_bytes = al256((size_t)m * m * chunk * tpi * d->c * es + (f16 ? (size_t)m * m * chunk * tpi * 4 : 0));
    pl->m_bytes = al256((size_t)m * m * chunk * tpi * d->k * 4);
    return CONVIO_OK;
}

static int launch_filter_tc(const WinoTcPlan &pl, const float *w, void *u, cudaStream_t st) {
    const int64_t pairs = (int64_t)pl.g.k * pl.g.c;
    const int blocks = (int)std::min<int64_t>((pairs + 255) / 256, 148 * 8);
    const bool bf = pl.kind == KIND_BF16;
    if (pl.kind == KIND_FFMA) {   // U[xi][c][k]: the FFMA GEMM reads [channel][n] rows
        if (pl.e == 2) CONVIO_CUDA_TRY(launch_pdl(winograd_filter_tc_kernel<2, float, true>, dim3(blocks), dim3(256), 0, st, w, (float *)u, pl.g.k, pl.g.c));
        else CONVIO_CUDA_TRY(launch_pdl(winograd_filter_tc_kernel<4, float, true>, dim3(blocks), dim3(256), 0, st, w, (float *)u, pl.g.k, pl.g.c));
    } else if (pl.e == 2) {
        if (bf) CONVIO_CUDA_TRY(launch_pdl(winograd_filter_tc_kernel<2, __nv_bfloat16>, dim3(blocks), dim3(256), 0, st, w, (__nv_bfloat16 *)u, pl.g.k, pl.g.c));
        else CONVIO_CUDA_TRY(launch_pdl(winograd_filter_tc_kernel<2, float>, dim3(blocks), dim3(256), 0, st, w, (float *)u, pl.g.k, pl.g.c));
    } else {
        if (bf) CONVIO_CUDA_TRY(launch_pdl(winograd_filter_tc_kernel<4, __nv_bfloat16>, dim3(blocks), dim3(256), 0, st, w, (__nv_bfloat16 *)u, pl.g.k, pl.g.c));
        else CONVIO_CUDA_TRY(launch_pdl(winograd_filter_tc_kernel<4, float>, dim3(blocks), dim3(256), 0, st, w, (float *)u, pl.g.k, pl.g.c));
    }
    if (pl.kind == KIND_3XF16) {   // fp32 U -> scaled fp16 hi / lo planes + col_exp
        note_launch();
        const int rows = pl.m * pl.m * pl.g.k;
        const size_t ub = (size_t)rows * pl.g.c * 4;
        CONVIO_CUDA_TRY(launch_pdl(winograd_u_split_f16x3_kernel, dim3((unsigned)std::min(rows / 8 + 1, 148 * 16)),
                                   dim3(256), 0, st, (const float *)u, (__half *)((uint8_t *)u + ub),
                                   (int *)((uint8_t *)u + 2 * ub), rows, pl.g.c));
    }
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

static int grid_for(int64_t work, int threads = 256) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads, 148 * 16));
}

int wino_tc_query(const convio_conv_desc *d, const convio_tile *t, int32_t precision,
                  convio_launch_info *out) {
    WinoTcPlan pl;
    const int e = t ? t->e : 0;
    int rc = plan_wino_tc(d, t, e, precision, &pl, out->reason, sizeof(out->reason));
    if (rc) return rc;
    IgemmPlan gp;
    const int tc = pl.chunk_imgs * pl.g.tiles_y * pl.g.tiles_x;
    if (pl.kind != KIND_FFMA) {
        rc = plan_igemm_batched(pl.kind, pl.bn, pl.s_b, pl.pair, pl.tsa, pl.m * pl.m, tc, d->c, d->k, &gp,
                                out->reason, sizeof(out->reason));
        if (rc) return rc;
        out->grid_x = gp.grid.x; out->grid_y = gp.grid.y; out->grid_z = gp.grid.z;
        out->block_threads = gp.threads;
        out->smem_bytes = (int)gp.smem;
        out->regs_per_thread = gp.regs;
        out->stages = gp.P.stages;
    } else {
        out->grid_x = d->k / pl.bn; out->grid_y = ((tc + 127) / 128) * pl.m * pl.m; out->grid_z = 1;
        out->block_threads = 288;
    }
    out->legal = 1;
    out->channel_chunk = pl.kind == KIND_BF16 ? 64 : 32;
    out->p = pl.g.p; out->q = pl.g.q;
    const int64_t tiles = (int64_t)d->n * pl.g.tiles_y * pl.g.tiles_x;
    out->flops = 2LL * pl.m * pl.m * tiles * d->k * d->c;   // element-wise GEMM flops
    out->workspace_bytes = (int64_t)(pl.u_bytes + pl.v_bytes + pl.m_bytes);
    snprintf(out->reason, sizeof(out->reason),
             "tcgen05 Winograd F(%d,3) %s: %d GEMMs of T=%d (chunk %d img) x K=%d x C=%d, N=%d",
             pl.e, pl.kind == KIND_FFMA ? "fp32 FFMA" : pl.kind == KIND_BF16 ? "bf16" : (pl.kind == KIND_3XTF32 ? "3xtf32" : "tf32"),
             pl.m * pl.m, tc, pl.chunk_imgs, d->k, d->c, pl.bn);
    return CONVIO_OK;
}

int64_t wino_tc_workspace_bytes(const convio_conv_desc *d, const convio_tile *t, int32_t precision) {
    WinoTcPlan pl;
    char why[160];
    if (!t) {   // no tile: enough for the library default of either e
        int64_t best = -1;
        for (int e : {2, 4})
            if (!plan_wino_tc(d, nullptr, e, precision, &pl, why, sizeof(why)))
                best = std::max<int64_t>(best, (int64_t)(pl.u_bytes + pl.v_bytes + pl.m_bytes));
        return best;
    }
    if (plan_wino_tc(d, t, t->e, precision, &pl, why, sizeof(why))) return -1;
    return (int64_t)(pl.u_bytes + pl.v_bytes + pl.m_bytes);
}

}  // namespace convio

using namespace convio;

extern "C" {

int convio_winograd_filter_transform_tc(const convio_conv_desc *desc, int32_t e, int32_t precision,
                                        const float *w, void *u, void *stream) {
    clear_error();
    reset_launches();
    WinoTcPlan pl;
    char why[160];
    int rc = plan_wino_tc(desc, nullptr, e, precision, &pl, why, sizeof(why));
    if (rc) return rc;
    if (!w || !u) {
        set_error("null filter pointer");
        return CONVIO_EINVAL;
    }
    return launch_filter_tc(pl, w, u, (cudaStream_t)stream);
}

int convio_winograd_filter_transform_tc_batched(int32_t count, const convio_conv_desc *descs, int32_t e,
                                                int32_t precision, const float *const *w, void *const *u,
                                                void *stream) {
    clear_error();
    reset_launches();
    if (count < 0 || count > kWinoJobs || (count && (!descs || !w || !u))) {
        set_error("count must be in [0, %d] with non-null arrays", kWinoJobs);
        return CONVIO_EINVAL;
    }
    if (!count) return CONVIO_OK;
    WinoFilterBatch B, S;
    memset(&B, 0, sizeof(B));
    memset(&S, 0, sizeof(S));
    B.n = S.n = count;
    int kind = -1;
    for (int i = 0; i < count; ++i) {
        WinoTcPlan pl;
        char why[160];
        int rc = plan_wino_tc(descs + i, nullptr, e, precision, &pl, why, sizeof(why));
        if (rc) return rc;
        if (pl.kind == KIND_FFMA || pl.kind == KIND_BF16) {
            set_error("batched Winograd filter transform: fp32 U only (TF32 / 3xTF32 / 3xF16)");
            return CONVIO_EINVAL;
        }
        if (!w[i] || !u[i]) {
            set_error("job %d: null filter pointer", i);
            return CONVIO_EINVAL;
        }
        kind = pl.kind;
        B.w[i] = S.w[i] = w[i];
        B.u[i] = S.u[i] = (float *)u[i];
        B.k[i] = S.k[i] = pl.g.k;
        B.c[i] = S.c[i] = pl.g.c;
        B.cum[i + 1] = B.cum[i] + (int64_t)pl.g.k * pl.g.c;
        S.cum[i + 1] = S.cum[i] + (int64_t)pl.m * pl.m * pl.g.k;
    }
    bool even_c = true;
    for (int i = 0; i < count; ++i) even_c = even_c && (B.c[i] % 2 == 0);
    if (kind == KIND_3XF16 && even_c) {   // fused transform + split, one launch
        WinoFilterBatch F = B;
        for (int i = 0; i < count; ++i) F.cum[i + 1] = F.cum[i] + F.k[i];
        const int fblocks = (int)std::min<int64_t>(F.cum[count], 148 * 8);
        if (e == 2) CONVIO_CUDA_TRY(launch_pdl(winograd_filter_f16x3_batched_kernel<2>, dim3(fblocks), dim3(256), 0, (cudaStream_t)stream, F));
        else CONVIO_CUDA_TRY(launch_pdl(winograd_filter_f16x3_batched_kernel<4>, dim3(fblocks), dim3(256), 0, (cudaStream_t)stream, F));
        note_launch();
        CONVIO_CUDA_TRY(cudaGetLastError());
        return CONVIO_OK;
    }
    const int blocks = (int)std::min<int64_t>((B.cum[count] + 255) / 256, 148 * 8);
    if (e == 2) CONVIO_CUDA_TRY(launch_pdl(winograd_filter_tc_batched_kernel<2>, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, B));
    else CONVIO_CUDA_TRY(launch_pdl(winograd_filter_tc_batched_kernel<4>, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, B));
    note_launch();
    if (kind == KIND_3XF16) {
        const int sblocks = (int)std::min<int64_t>(S.cum[count] / 8 + 1, 148 * 16);
        CONVIO_CUDA_TRY(launch_pdl(winograd_u_split_f16x3_batched_kernel, dim3(sblocks), dim3(256), 0, (cudaStream_t)stream, S));
        note_launch();
    }
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

int convio_winograd_bgemm(const convio_conv_desc *desc, const convio_tile *tile, int32_t e,
                          int32_t precision, const float *x, const void *w, int32_t w_is_transformed,
                          const float *bias, int32_t relu, float *y, void *workspace,
                          size_t workspace_bytes, void *stream) {
    clear_error();
    reset_launches();
    WinoTcPlan pl;
    char why[160];
    int rc = plan_wino_tc(desc, tile, e, precision, &pl, why, sizeof(why));
    if (rc) return rc;
    if (!x || !w || !y) {
        set_error("null tensor pointer");
        return CONVIO_EINVAL;
    }
    const size_t need = pl.u_bytes + pl.v_bytes + pl.m_bytes;
    if (!workspace || workspace_bytes < need) {
        set_error("workspace of %zu bytes needed (U + chunk V + chunk M)", need);
        return CONVIO_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *ws = (uint8_t *)workspace;
    const void *u = w;
    if (!w_is_transformed) {
        rc = launch_filter_tc(pl, (const float *)w, ws, st);
        if (rc) return rc;
        u = ws;
    }
    void *v = ws + pl.u_bytes;
    float *mm = (float *)(ws + pl.u_bytes + pl.v_bytes);
    const int tpi = pl.g.tiles_y * pl.g.tiles_x;
    const bool bf = pl.kind == KIND_BF16;
    for (int img0 = 0; img0 < desc->n; img0 += pl.chunk_imgs) {
        WinoTcGeom g = pl.g;
        g.img0 = img0;
        g.imgs = std::min(pl.chunk_imgs, desc->n - img0);
        const int tc = g.imgs * tpi;
        const int gin = grid_for((int64_t)tc * (g.c / 4), 128), gout = grid_for((int64_t)tc * (g.k / 4), 128);
        const size_t vb = (size_t)pl.m * pl.m * tc * g.c * 4;   // 3xF16: hi + lo planes
        if (pl.kind == KIND_3XF16) {
            if (pl.e == 2)
                CONVIO_CUDA_TRY(launch_pdl(winograd_input_f16x3_kernel<2>, dim3(gin), dim3(128), 0, st, x,
                                           (__half *)v, (int *)((uint8_t *)v + vb), g));
            else
                CONVIO_CUDA_TRY(launch_pdl(winograd_input_f16x3_kernel<4>, dim3(gin), dim3(128), 0, st, x,
                                           (__half *)v, (int *)((uint8_t *)v + vb), g));
        } else if (pl.e == 2) {
            if (bf) CONVIO_CUDA_TRY(launch_pdl(winograd_input_tc_kernel<2, __nv_bfloat16>, dim3(gin), dim3(128), 0, st, x, (__nv_bfloat16 *)v, g));
            else CONVIO_CUDA_TRY(launch_pdl(winograd_input_tc_kernel<2, float>, dim3(gin), dim3(128), 0, st, x, (float *)v, g));
        } else {
            if (bf) CONVIO_CUDA_TRY(launch_pdl(winograd_input_tc_kernel<4, __nv_bfloat16>, dim3(gin), dim3(128), 0, st, x, (__nv_bfloat16 *)v, g));
            else CONVIO_CUDA_TRY(launch_pdl(winograd_input_tc_kernel<4, float>, dim3(gin), dim3(128), 0, st, x, (float *)v, g));
        }
        note_launch();
        CONVIO_CUDA_TRY(cudaGetLastError());
        if (pl.kind == KIND_FFMA) {
            rc = direct_nhwc_batched_run(pl.bn, 32768, pl.m * pl.m, tc, g.c, g.k, (const float *)v,
                                         (const float *)u, mm, st);
        } else {
            IgemmPlan gp;
            rc = plan_igemm_batched(pl.kind, pl.bn, pl.s_b, pl.pair, pl.tsa, pl.m * pl.m, tc, g.c, g.k, &gp, why,
                                    sizeof(why));
            if (rc) return rc;
            const void *ua = u;
            if (pl.kind == KIND_3XF16) {
                const size_t ub = (size_t)pl.m * pl.m * g.k * g.c * 4;
                ua = (const uint8_t *)u + ub;
                gp.P.row_exp = (const int *)((const uint8_t *)v + vb);
                gp.P.col_exp = (const int *)((const uint8_t *)u + 2 * ub);
            }
            rc = igemm_launch(gp, v, ua, nullptr, 0, mm, st);
        }
        if (rc) return rc;
        if (pl.e == 2)
            CONVIO_CUDA_TRY(launch_pdl(winograd_output_tc_kernel<2>, dim3(gout), dim3(128), 0, st, (const float *)mm, bias, y, g, relu));
        else
            CONVIO_CUDA_TRY(launch_pdl(winograd_output_tc_kernel<4>, dim3(gout), dim3(128), 0, st, (const float *)mm, bias, y, g, relu));
        note_launch();
        CONVIO_CUDA_TRY(cudaGetLastError());
    }
    return CONVIO_OK;
}

}  // extern "C"
