// Direct convolution, FP32 on CUDA cores, channels-last (the reference's HWC
// layout, pkg/src/convio/dataflow.py:23): the output-stationary dataflow of
// plan_direct_dataflow (dataflow.py:219-250) with the block's pixels stacked
// into a 128-row register tile, so the FFMA work per staged word does not
// shrink with the feature map (14x14 / 7x7 maps keep the same reuse as 56x56).
//
// Block   = x*y pixels of ceil(128/(x*y)) images (the GEMM M axis, <= 128 rows)
//           x z output channels (z = BN in {64, 128}), resident in registers.
// Stage   = one (tap, 32-channel) slice: a TMA box [imgs][y][x][32 ch] of the
//           input shifted by the tap (halo zero-filled = padding, stride via
//           TMA traversal strides; SWIZZLE_128B so the row reads below are
//           bank-conflict free) and a [32 ch][BN] box of the C R S K packed
//           filter (convio_pack_filter_direct).  NS-deep ring, one producer
//           thread, mbarrier full/empty -- no block-wide barrier in the loop.
// Threads = 256 consumers as 16 pixel groups x 16 channel groups: thread
//           (mg, ng) owns rows mg + 16 i (i < 8) and channels
//           h*64 + 4 ng + u (u < 4, h < BN/64): per 4 channels 8 + BN/32
//           LDS.128 feed 32 * BN/16 FFMA (256 at BN = 128).
// Every output accumulates its R*S*C products in (tap, channel) order in
// fp32 FMA (tolerance as the NCHW kernel: SURVEY.md §8(d)).
#pragma once

#include "direct_fp32.cuh"

namespace convio {

struct NhwcParams {
    const float *bias;
    float *y;
    int n, c, h, w, k, p, q, pad, stride, ks;
    int bx, by, imgs;
    int tiles_x, tiles_y, img_groups;
    int kblocks, cblocks;
    int stages;
    int relu;
    int batched;      // Winograd element-wise GEMMs: "image" = xi, pixels = tiles, filter = U[xi][C][K]
};

__device__ __forceinline__ float4 lds128_f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

template <int BN>
__global__ void __launch_bounds__(288, 1)
    direct_nhwc_f32_kernel(const __grid_constant__ NhwcParams P, const __grid_constant__ CUtensorMap tm_x,
                           const __grid_constant__ CUtensorMap tm_w) {
    constexpr int A_BYTES = 128 * 128;        // 128 pixel rows x 32 fp32 (SW128)
    constexpr int B_BYTES = 32 * BN * 4;      // 32 channels x BN fp32
    constexpr int STAGE = A_BYTES + B_BYTES;
    constexpr int TN = BN / 16;               // output channels per thread
    constexpr int H = BN / 64;                // 64-channel halves
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int NS = P.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NS * STAGE);
    uint64_t *empty = full + NS;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int k0 = blockIdx.x * BN;
    const int xt = blockIdx.y % P.tiles_x;
    const int rest = blockIdx.y / P.tiles_x;
    const int yt = rest % P.tiles_y;
    const int ig = rest / P.tiles_y;
    const int ox0 = xt * P.bx, oy0 = yt * P.by, img0 = ig * P.imgs;
    const uint64_t map_x = reinterpret_cast<uint64_t>(&tm_x);
    const uint64_t map_w = reinterpret_cast<uint64_t>(&tm_w);

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_x));
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_w));
    }
    __syncthreads();

    if (warp == 8) {
        if (lane == 0) {
            // ---- TMA producer ---------------------------------------------------------
            const uint32_t bytes = (uint32_t)(P.bx * P.by * P.imgs * 128 + B_BYTES);
            int s = 0, tap = 0, cb = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < P.kblocks; ++kb) {
                if (kb >= NS) mbar_wait(empty + s, ph ^ 1);
                const int r = tap / P.ks, sx = tap - r * P.ks;
                uint8_t *a = smem + s * STAGE;
                mbar_arrive_expect_tx(full + s, bytes);
                tma_load_4d(a, map_x, cb * 32, ox0 * P.stride + sx - P.pad, oy0 * P.stride + r - P.pad,
                            img0, full + s);
                if (P.batched) tma_load_3d(a + A_BYTES, map_w, k0, cb * 32, img0, full + s);
                else tma_load_3d(a + A_BYTES, map_w, k0, tap, cb * 32, full + s);
                if (++cb == P.cblocks) {
                    cb = 0;
                    ++tap;
                }
                if (++s == NS) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
        return;
    }

    // ---- consumers: 16 pixel groups x 16 channel groups --------------------------
    // in a warp: 4 pixel groups x 8 channel groups (conflict-free row reads)
    const int mg = (warp & 3) * 4 + (lane >> 3);     // 0..15
    const int ng = (warp >> 2) * 8 + (lane & 7);     // 0..15
    const uint32_t a_row = (uint32_t)mg * 128;
    const uint32_t swz = (uint32_t)(mg & 7);
    float acc[8][TN];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

    int s = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < P.kblocks; ++kb) {
        mbar_wait(full + s, ph);
        const uint32_t a_base = smem_u32(smem + s * STAGE) + a_row;
        const uint32_t b_base = smem_u32(smem + s * STAGE + A_BYTES) + (uint32_t)ng * 16;
#pragma unroll 2
        for (int cq = 0; cq < 8; ++cq) {
            float4 a[8];
            const uint32_t chunk = ((uint32_t)cq ^ swz) << 4;
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = lds128_f(a_base + i * 16 * 128 + chunk);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float b[TN];
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const float4 v = lds128_f(b_base + (uint32_t)((cq * 4 + u) * BN * 4 + h * 256));
                    b[h * 4] = v.x; b[h * 4 + 1] = v.y; b[h * 4 + 2] = v.z; b[h * 4 + 3] = v.w;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float av = u == 0 ? a[i].x : u == 1 ? a[i].y : u == 2 ? a[i].z : a[i].w;
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av, b[j], acc[i][j]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
        if (++s == NS) {
            s = 0;
            ph ^= 1;
        }
    }

    // ---- epilogue: bias + ReLU, NHWC float4 stores ----------------------------------
    const int per_img = P.bx * P.by;
    float bv[TN];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int u = 0; u < 4; ++u)
            bv[h * 4 + u] = P.bias ? __ldg(P.bias + k0 + h * 64 + ng * 4 + u) : 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = mg + 16 * i;
        const int im = m / per_img, pix = m - im * per_img;
        const int py = pix / P.bx, px = pix - py * P.bx;
        const int img = img0 + im, oy = oy0 + py, ox = ox0 + px;
        if (m >= per_img * P.imgs || img >= P.n || oy >= P.p || ox >= P.q) continue;
        float *dst = P.y + (((int64_t)img * P.p + oy) * P.q + ox) * P.k + k0 + ng * 4;
#pragma unroll
        for (int h = 0; h < H; ++h) {
            float4 o;
            o.x = acc[i][h * 4] + bv[h * 4];
            o.y = acc[i][h * 4 + 1] + bv[h * 4 + 1];
            o.z = acc[i][h * 4 + 2] + bv[h * 4 + 2];
            o.w = acc[i][h * 4 + 3] + bv[h * 4 + 3];
            if (P.relu) {
                o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f);
                o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
            }
            *reinterpret_cast<float4 *>(dst + h * 64) = o;
        }
    }
}

}  // namespace convio
