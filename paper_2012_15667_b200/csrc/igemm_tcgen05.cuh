// Direct convolution as an implicit GEMM on the 5th-generation tensor cores
// (tcgen05, FP32 accumulate in TMEM) -- the "TF32/BF16 tcgen05 variant for
// the dense contraction stage" of the north star, same output-stationary
// block (x*y pixels x z channels per CTA) as the FP32 dataflow
// (reference pkg/src/convio/dataflow.py:219-250).
//
//   GEMM view  D[m][n] += A[m][kk] * B[n][kk]
//     m  = pixel of the block (x*y pixels of up to `imgs` stacked images),
//     n  = output channel (z = BN per CTA),
//     kk = (tap r,s ; input-channel c), walked as R*S taps x C/CB blocks
//          (CB = 32 fp32 or 64 bf16 channels = one 128-B row).
//   A    = NHWC input box [imgs][y][x][CB ch] for tap (r,s): one TMA 4-D load
//          per k-block, zero-filled halo (= padding), SWIZZLE_128B, i.e. the
//          canonical K-major UMMA layout (128-B rows, 1024-B swizzle atoms).
//   B    = packed filters [RS][K][C] box [BN][CB ch], same layout.
//   MMA  = one elected thread issues 4 x tcgen05.mma (M=128, N=BN, K=32 B)
//          per k-block; tcgen05.commit releases the smem stage to the TMA thread.
//   D    = 128 lanes x BN fp32 columns in TMEM; 4 warps tcgen05.ld their 32
//          lanes and store NHWC rows (+ bias / ReLU).
// Rows of the A tile beyond x*y*imgs are don't-care (never stored).
//
// Batched mode (P.batched, Winograd's element-wise GEMMs, dataflow.py:253-310
// step 3): the "image" axis is the Winograd element xi, the pixel axis the
// tile index t, R = S = 1, and the filter box's third coordinate is xi, so
// one launch computes M[xi][t][k] = sum_c V[xi][t][c] * U[xi][k][c] for all xi.
#pragma once

#include "direct_fp32.cuh"

namespace convio {

struct IgemmParams {
    const float *bias;
    float *y;
    int n, c, h, w, k, p, q, pad, stride;
    int bx, by, imgs;          // block: bx * by pixels of `imgs` images (<= 128 rows)
    int tiles_x, tiles_y, img_groups;
    int kblocks;               // 9 * C / 32 (R*S taps x channel blocks)
    int cblocks;               // C / 32
    int ks;                    // kernel edge
    int stages;
    int relu;
    int batched;               // 1: Winograd element-wise GEMMs (see header)
    int splits;                // split-K factor (blockIdx.z = split; > 1 only without ReLU)
    // KIND_3XF16 (batched only): power-of-two exponents the operands were scaled by;
    // the epilogue multiplies D[t][k] by 2^-(row_exp[g][t] + col_exp[g][k])
    // KIND_3XF16C (conv): col_exp[k] = the packed filter's per-output-channel exponents
    const int *row_exp;
    const int *col_exp;
    int nred;
    // grouped conv (3xF16C pair kernels): G independent layers of one shape and plan in
    // one launch -- inputs / outputs stacked along N (layer_imgs images each), filters
    // as G packed slices (filter map gains a layer dimension), bias G x K, the packed
    // slice's exponents col_stride ints apart.  layer_imgs = 0: one layer
    int layer_imgs;
    int col_stride;
};

// operand kinds of the tcgen05 contraction
//   KIND_3XF16  batched Winograd GEMMs: operands pre-split into fp16 hi / lo planes
//   KIND_3XF16C direct conv: fp32 activations TMA-staged and split in shared
//               memory by converter warps (one power-of-two scale per tensor),
//               filters pre-split into fp16 planes (scale per output channel)
enum IgemmKind : int { KIND_TF32 = 0, KIND_3XTF32 = 1, KIND_BF16 = 2, KIND_3XF16 = 4, KIND_3XF16C = 5 };

// Power-of-two scale exponent for a row (or tensor) whose largest magnitude is
// `mx`: the scaled values lie in (-2^15, 2^15), so their fp16 hi parts are
// normal down to 2^-24 of the maximum and nothing overflows.  Clamped to
// pow2f's range [-126, 127], so the exponent an epilogue undoes is always the
// one that was applied.
__device__ __forceinline__ int f16_row_exp(float mx) {
    if (!(mx >= 1.17549435e-38f)) return 0;   // zero / subnormal: unscaled
    const int ex = ((__float_as_int(mx) >> 23) & 0xff) - 126;   // mx = f * 2^ex, f in [0.5, 1)
    return min(127, max(-126, 15 - ex));
}

// the activation exponent of KIND_3XF16C: max over the nred partial maxima
// (non-negative float bits compare as ints), one warp, all lanes get it
__device__ __forceinline__ int f16c_act_exp(const int *partials, int nred, int lane) {
    int m = 0;
    for (int i = lane; i < nred; i += 32) m = max(m, __ldg(partials + i));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
    return f16_row_exp(__int_as_float(m));
}

// 2^e as a float for e in [-126, 127] (exponent bits; a multiply by it is exact
// wherever the product stays normal) -- ldexpf costs ~20 instructions
__device__ __forceinline__ float pow2f(int e) {
    e = max(-126, min(127, e));
    return __int_as_float((e + 127) << 23);
}

// ---- tcgen05 / UMMA primitives ----------------------------------------------------
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    // K-major, SWIZZLE_128B: 128-B rows, 8-row (1024-B) atoms -> SBO = 1024 B.
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);        // start address
    d |= (uint64_t)1 << 16;                             // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                   // SBO
    d |= (uint64_t)1 << 46;                             // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                             // layout: SWIZZLE_128B
    return d;
}

template <int BN, int KIND>
__device__ __forceinline__ constexpr uint32_t idesc_m128() {
    // kind::tf32: A/B format 2 (TF32); kind::f16: A/B format 1 (BF16)
    return (1u << 4)          // D format F32
           | ((KIND == KIND_BF16 ? 1u : 2u) << 7)
           | ((KIND == KIND_BF16 ? 1u : 2u) << 10)
           | ((uint32_t)(BN >> 3) << 17)
           | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

// store v rounded to TF32 (cvt.rna), explicit shared window
__device__ __forceinline__ void sts128_tf32(uint32_t addr, float4 v) {
    uint32_t a, b, c, d;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(a) : "f"(v.x));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(v.y));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(c) : "f"(v.z));
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(d) : "f"(v.w));
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_ld_32x32b(uint32_t taddr, float (&v)[N]);

template <>
__device__ __forceinline__ void tmem_ld_32x32b<32>(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
        "%30, %31}, [%32];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// KIND_3XTF32: each operand is split into hi = tf32(v) (the raw operand,
// read by the tensor core with the low mantissa bits dropped) and
// lo = rna_tf32(v - hi) written by 4 converter warps; every k-step issues
// A_hi*B_lo + A_lo*B_hi + A_hi*B_hi -- FP32-level accuracy on the tensor cores.
// KIND_BF16: operands are bf16 in HBM (64 channels per 128-B row), kind::f16.
// 3xTF32 converter warps of the single-CTA kernel: 4 keeps 256 threads so two
// CTAs share an SM at s_b = 16384 (measured: 8 warps cost res2 0.518 -> 0.674 ms
// by losing that second CTA); the pair kernel uses 8 below BN = 256.
template <int BN>
constexpr int conv_warps() { return 4; }

template <int BN, int KIND>
constexpr int igemm_threads() { return KIND == KIND_3XTF32 ? 128 + 32 * conv_warps<BN>() : 128; }

template <int BN, int KIND>
__global__ void __launch_bounds__(igemm_threads<BN, KIND>(), 1)
    igemm_tcgen05_kernel(const __grid_constant__ IgemmParams P,
                              const __grid_constant__ CUtensorMap tm_x,
                              const __grid_constant__ CUtensorMap tm_w) {
    constexpr bool SPLIT = KIND == KIND_3XTF32;
    constexpr int A_BYTES = 128 * 128;       // 128 rows x 128 B (32 fp32 / 64 bf16)
    constexpr int B_BYTES = BN * 128;        // BN rows x 128 B
    constexpr int CB = KIND == KIND_BF16 ? 64 : 32;   // channels per k-block
    // stage: [A | B] (TMA; hi after conversion) then, when split, [A_lo | B_lo]
    constexpr int STAGE = (A_BYTES + B_BYTES) * (SPLIT ? 2 : 1);
    constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B atoms
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int NS = P.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NS * STAGE);
    uint64_t *empty = full + NS;
    uint64_t *done = empty + NS;
    uint64_t *conv = done + 1;                        // split: converted[NS]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(conv + NS);

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
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        if (SPLIT)
            for (int s = 0; s < NS; ++s) mbar_init(conv + s, conv_warps<BN>());
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_x));
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_w));
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    pdl_wait();

    // split-K (small grids): this CTA reduces k-blocks [kb_lo, kb_hi) and adds its
    // partial tile into the zeroed output
    const int kb_lo = (int)(((int64_t)P.kblocks * blockIdx.z) / P.splits);
    const int kb_hi = (int)(((int64_t)P.kblocks * (blockIdx.z + 1)) / P.splits);
    const int nkb = kb_hi - kb_lo;
    if (tid == 0) {
        // ---- TMA producer ---------------------------------------------------------
        int s = 0, tap = kb_lo / P.cblocks, cb = kb_lo - tap * P.cblocks;
        uint32_t ph = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            if (kb >= NS) mbar_wait(empty + s, ph ^ 1);
            const int r = tap / P.ks, sx = tap - r * P.ks;
            uint8_t *a = smem + s * STAGE;
            uint8_t *b = a + A_BYTES;
            mbar_arrive_expect_tx(full + s, (uint32_t)(P.bx * P.by * P.imgs * 128 + B_BYTES));
            // stride > 1: the map's traversal strides pick every stride-th pixel
            tma_load_4d(a, map_x, cb * CB, ox0 * P.stride + sx - P.pad, oy0 * P.stride + r - P.pad,
                        img0, full + s);
            tma_load_3d(b, map_w, cb * CB, k0, P.batched ? img0 : tap, full + s);
            if (++cb == P.cblocks) {
                cb = 0;
                ++tap;
            }
            if (++s == NS) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (tid == 32) {
        // ---- MMA issuer (single thread) -------------------------------------------
        constexpr uint32_t idesc = idesc_m128<BN, KIND>();
        int s = 0;
        uint32_t ph = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(SPLIT ? conv + s : full + s, ph);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t a = smem_u32(smem + s * STAGE);
            const uint32_t b = a + A_BYTES;
            const uint64_t ad = umma_desc_sw128(a), bd = umma_desc_sw128(b);
            if constexpr (SPLIT) {
                const uint64_t adl = umma_desc_sw128(a + A_BYTES + B_BYTES);
                const uint64_t bdl = umma_desc_sw128(b + A_BYTES + B_BYTES);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t o = (uint64_t)(kk * 2);
                    umma_tf32(tmem, ad + o, bdl + o, idesc, (kb | kk) != 0);   // small terms first
                    umma_tf32(tmem, adl + o, bd + o, idesc, 1);
                    umma_tf32(tmem, ad + o, bd + o, idesc, 1);
                }
            } else if constexpr (KIND == KIND_BF16) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)   // K = 16 bf16 = 32 B per MMA
                    umma_bf16(tmem, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc,
                              (kb | kk) != 0);
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)   // K = 8 tf32 = 32 B per MMA
                    umma_tf32(tmem, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc,
                              (kb | kk) != 0);
            }
            umma_commit(empty + s);
            if (++s == NS) {
                s = 0;
                ph ^= 1;
            }
        }
        umma_commit(done);
    } else if (SPLIT && warp >= 4) {
        // ---- converter warps: lo = v - tf32(v) alongside the raw operand --------------
        // The tensor core reads the raw fp32 operand as TF32 by dropping the low
        // 13 mantissa bits, so hi = v & ~0x1fff needs no store: only lo is
        // written (itself rounded to TF32), halving the conversion's smem traffic.
        constexpr int NT = 32 * conv_warps<BN>();
        const int ct = tid - 128;                    // 0 .. NT-1
        constexpr int PER = (A_BYTES + B_BYTES) / 16 / NT;    // float4 per converter thread
        int s = 0;
        uint32_t ph = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(full + s, ph);
            // explicit shared-window addressing (LDS/STS, not generic LD/ST);
            // all loads first so their latencies overlap
            const uint32_t hi_s = smem_u32(smem + s * STAGE) + ct * 16;
            const uint32_t lo_s = hi_s + A_BYTES + B_BYTES;
            float4 v[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) v[j] = lds128(hi_s + j * NT * 16);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                float4 l;
                l.x = v[j].x - __uint_as_float(__float_as_uint(v[j].x) & 0xffffe000u);
                l.y = v[j].y - __uint_as_float(__float_as_uint(v[j].y) & 0xffffe000u);
                l.z = v[j].z - __uint_as_float(__float_as_uint(v[j].z) & 0xffffe000u);
                l.w = v[j].w - __uint_as_float(__float_as_uint(v[j].w) & 0xffffe000u);
                sts128_tf32(lo_s + j * NT * 16, l);
            }
            // generic-proxy stores -> visible to the tensor core's async proxy
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(conv + s);
            if (++s == NS) {
                s = 0;
                ph ^= 1;
            }
        }
    }
    // ---- epilogue: TMEM -> registers -> NHWC global ---------------------------------
    if (SPLIT && warp >= 4) {        // converters have no TMEM lanes to drain
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();
        return;
    }
    mbar_wait(done, 0);
    __syncwarp();   // the producer / MMA lanes rejoin their warps before .sync.aligned loads
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int m = warp * 32 + lane;                 // D row = TMEM lane = pixel
    const int per_img = P.bx * P.by;
    const int im = m / per_img, pix = m - im * per_img;
    const int py = pix / P.bx, px = pix - py * P.bx;
    const int img = img0 + im, oy = oy0 + py, ox = ox0 + px;
    const bool valid = m < per_img * P.imgs && img < P.n && oy < P.p && ox < P.q;
    float *dst = P.y + (((int64_t)img * P.p + oy) * P.q + ox) * P.k + k0;
    const bool add_bias = P.bias && blockIdx.z == 0;
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld_32x32b<32>(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
        if (valid) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                float4 o;
                o.x = v[j] + (add_bias ? __ldg(P.bias + k0 + c0 + j) : 0.0f);
                o.y = v[j + 1] + (add_bias ? __ldg(P.bias + k0 + c0 + j + 1) : 0.0f);
                o.z = v[j + 2] + (add_bias ? __ldg(P.bias + k0 + c0 + j + 2) : 0.0f);
                o.w = v[j + 3] + (add_bias ? __ldg(P.bias + k0 + c0 + j + 3) : 0.0f);
                if (P.splits > 1) {   // partial sums of the K range: fp32 vector atomics
                    atomicAdd(reinterpret_cast<float4 *>(dst + c0 + j), o);
                    continue;
                }
                if (P.relu) {
                    o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f);
                    o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
                }
                *reinterpret_cast<float4 *>(dst + c0 + j) = o;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
}

// ---- host-side plan (igemm.cu) -------------------------------------------------
using IgemmFn = void (*)(const IgemmParams, const CUtensorMap, const CUtensorMap);

struct PairParams;   // igemm_pair.cuh
using PairFn = void (*)(const PairParams, const CUtensorMap, const CUtensorMap, const CUtensorMap);

struct IgemmPlan {
    IgemmParams P;
    IgemmFn fn = nullptr;
    bool pair = false;       // persistent CTA-pair kernel (igemm_pair.cuh)
    bool halo = false;       // footprint staging (pair kernel, stride 1)
    bool tsa = false;        // 3xTF32 pair kernel with the A operand in TMEM
    bool fold = false;       // halo + the S horizontal taps in one MMA of N = S * K
    int resb_slots = 0;      // halo TSA: filter slice resident in smem (one slot per k-block)
    int64_t tail_start = 0;  // pair kernel: tile items from here on are split-K (P.splits)
    int *scale_state = nullptr;   // 3xF16C: speculative activation scale state (workspace)
    bool no_resb = false;    // planning option: never keep the filter resident
    int layers = 1;          // grouped conv: layers stacked along N (filter map gains a dim)
    size_t layer_bytes = 0;  // grouped conv: bytes between consecutive packed filter slices
    PairFn pfn = nullptr;
    int groups = 1, blocks_per_group = 0;
    int fpr = 0, fp_bytes = 0, a_slot = 0, na = 0;
    bool gather = false;     // halo TSA with exact x * y * imgs blocks (converters gather taps)
    int fw = 0, fh = 0;      // gather: footprint width / height per image
    dim3 grid;
    size_t smem = 0;
    int regs = 0;
    int bn = 0;
    int threads = 128;
    int kind = KIND_TF32;
};

// M[xi][t][k] = sum_c V[xi][t][c] * U[xi][k][c] (Winograd step 3) in one launch
int plan_igemm_batched(int kind, int bn, int s_b, bool pair, bool tsa, int xi, int t_count, int c, int k,
                       IgemmPlan *pl, char *reason, size_t rlen);
int igemm_launch(IgemmPlan &pl, const void *x, const void *wq, const float *bias, int relu, float *y,
                 cudaStream_t stream);

}  // namespace convio
