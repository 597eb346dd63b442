// Host side of the tcgen05 implicit-GEMM convolution (TF32 / 3xTF32 / BF16 in,
// FP32 accumulate): device projection of a TileConfig, filter packing, TMA
// descriptors, launch; plus the batched launcher the tensor-core Winograd
// path uses for its element-wise GEMMs (winograd_tc.cu).
#include <cuda_bf16.h>
#include <stdarg.h>
#include <algorithm>

#include <stdlib.h>

#include "igemm_pair.cuh"

namespace convio {

#ifdef CONVIO_TRACE
unsigned long long *g_trace_ptr = nullptr;   // dev builds: the pair kernel's pipeline trace
#endif

template <int KIND>
static IgemmFn igemm_kernel_kind(int bn) {
    switch (bn) {
        case 64: return &igemm_tcgen05_kernel<64, KIND>;
        case 128: return &igemm_tcgen05_kernel<128, KIND>;
        case 256: return &igemm_tcgen05_kernel<256, KIND>;
        default: return nullptr;
    }
}

static IgemmFn igemm_kernel(int bn, int kind) {
    if (kind == KIND_3XTF32) return igemm_kernel_kind<KIND_3XTF32>(bn);
    if (kind == KIND_BF16) return igemm_kernel_kind<KIND_BF16>(bn);
    return igemm_kernel_kind<KIND_TF32>(bn);
}

template <int KIND, bool HALO>
static PairFn pair_kernel_kind(int bn) {
    switch (bn) {
        case 64: return &igemm_pair_kernel<64, KIND, HALO, false>;
        case 128: return &igemm_pair_kernel<128, KIND, HALO, false>;
        case 256: return &igemm_pair_kernel<256, KIND, HALO, false>;
        default: return nullptr;
    }
}

template <bool HALO>
static PairFn pair_kernel_h(int bn, int kind) {
    if (kind == KIND_3XTF32) return pair_kernel_kind<KIND_3XTF32, HALO>(bn);
    if (kind == KIND_BF16) return pair_kernel_kind<KIND_BF16, HALO>(bn);
    return pair_kernel_kind<KIND_TF32, HALO>(bn);
}

// fold: halo + S taps per MMA, N = 3 K (K = 64 -> N = 192); 3xF16C may take the
// A operand in TMEM (tsa, the converters apply the row shift) with the filter
// resident in shared memory (resb)
static PairFn pair_kernel_fold(int n, int kind, bool tsa = false, bool resb = false) {
    if (n != 192) return nullptr;
    if (tsa) {
        if (kind != KIND_3XF16C) return nullptr;
        return resb ? &igemm_pair_kernel<192, KIND_3XF16C, true, true, true, true>
                    : &igemm_pair_kernel<192, KIND_3XF16C, true, true, true, false>;
    }
    if (resb) return nullptr;
    if (kind == KIND_3XF16C) return &igemm_pair_kernel<192, KIND_3XF16C, true, false, true>;
    if (kind == KIND_3XTF32) return &igemm_pair_kernel<192, KIND_3XTF32, true, false, true>;
    if (kind == KIND_BF16) return &igemm_pair_kernel<192, KIND_BF16, true, false, true>;
    return &igemm_pair_kernel<192, KIND_TF32, true, false, true>;
}

// tsa: 3xTF32 with the A operand in tensor memory (BN <= 128, no halo)
static PairFn pair_kernel(int bn, int kind, bool halo, bool tsa) {
    if (tsa && kind == KIND_3XF16C && halo) {   // halo footprint, converters shift rows into TMEM
        if (bn == 64) return &igemm_pair_kernel<64, KIND_3XF16C, true, true>;
        if (bn == 128) return &igemm_pair_kernel<128, KIND_3XF16C, true, true>;
        if (bn == 256) return &igemm_pair_kernel<256, KIND_3XF16C, true, true>;
        return nullptr;
    }
    if (tsa && kind == KIND_3XF16C) {   // 3xF16C, A in TMEM (BN = 256: one accumulator)
        if (bn == 64) return &igemm_pair_kernel<64, KIND_3XF16C, false, true>;
        if (bn == 128) return &igemm_pair_kernel<128, KIND_3XF16C, false, true>;
        if (bn == 256) return &igemm_pair_kernel<256, KIND_3XF16C, false, true>;
        return nullptr;
    }
    if (tsa) {
        if (kind != KIND_3XTF32 || halo) return nullptr;
        if (bn == 64) return &igemm_pair_kernel<64, KIND_3XTF32, false, true>;
        if (bn == 128) return &igemm_pair_kernel<128, KIND_3XTF32, false, true>;
        return nullptr;
    }
    if (kind == KIND_3XF16) {   // scaled fp16 hi / lo planes (batched Winograd GEMMs)
        if (halo) return nullptr;
        return pair_kernel_kind<KIND_3XF16, false>(bn);
    }
    if (kind == KIND_3XF16C)    // direct conv, activations split in shared memory
        return halo ? pair_kernel_kind<KIND_3XF16C, true>(bn) : pair_kernel_kind<KIND_3XF16C, false>(bn);
    return halo ? pair_kernel_h<true>(bn, kind) : pair_kernel_h<false>(bn, kind);
}

static const char *kind_name(int kind) {
    return kind == KIND_3XTF32 ? "3xtf32" : (kind == KIND_BF16 ? "bf16" : (kind == KIND_3XF16C ? "3xf16" : "tf32"));
}

// channels per k-block: one 128-B operand row (32 fp32, 64 bf16 / fp16)
static int kblock_channels(int kind) {
    return (kind == KIND_BF16 || kind == KIND_3XF16 || kind == KIND_3XF16C) ? 64 : 32;
}

// 3xF16C filter operand: KCRS -> fp16 hi / lo planes [2][R*S][K][C] with one
// power-of-two scale per output channel k over its C*R*S weights (col_exp[k],
// undone by the GEMM epilogue).  One block per output channel: the row's max by a
// block reduction, then tap-major passes where each thread writes __half2 pairs of
// channels (coalesced plane rows; the strided KCRS re-reads hit L1).
__global__ void __launch_bounds__(256) pack_filter_f16x3_kernel(const float *__restrict__ w,
                                                                __half *__restrict__ wq,
                                                                int *__restrict__ col_exp, int k, int c,
                                                                int rs) {
    pdl_wait();
    __shared__ float red[8];
    const int crs = c * rs;
    const int64_t plane = (int64_t)rs * k * c;
    for (int kk = blockIdx.x; kk < k; kk += gridDim.x) {
        const float *wr = w + (int64_t)kk * crs;
        float mx = 0.0f;
        for (int j = threadIdx.x; j < crs; j += blockDim.x) mx = fmaxf(mx, fabsf(wr[j]));
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        mx = red[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, red[i]);
        const int e = f16_row_exp(mx);
        const float sc = pow2f(e);
        const int pairs = (c + 1) / 2;
        for (int t = threadIdx.x; t < rs * pairs; t += blockDim.x) {
            const int tap = t / pairs, cc = 2 * (t - tap * pairs);
            __half *hrow = wq + ((int64_t)tap * k + kk) * c;
            const float v0 = wr[cc * rs + tap] * sc;
            const float v1 = cc + 1 < c ? wr[(cc + 1) * rs + tap] * sc : 0.0f;
            const __half2 hi = __floats2half2_rn(v0, v1);
            const float2 hf = __half22float2(hi);
            const __half2 lo = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
            if (cc + 1 < c) {
                *reinterpret_cast<__half2 *>(hrow + cc) = hi;
                *reinterpret_cast<__half2 *>(hrow + plane + cc) = lo;
            } else {
                hrow[cc] = __low2half(hi);
                hrow[plane + cc] = __low2half(lo);
            }
        }
        if (threadIdx.x == 0) col_exp[kk] = e;
        __syncthreads();   // red[] is reused by the next row
    }
}

// Batched form: every filter of a step in one launch (block b -> job, output channel
// through the kcum prefix sums): the per-layer launches each filled only K blocks
constexpr int kPackJobs = 32;
struct PackJob {
    const float *w;
    __half *wq;
    int *col_exp;
    int k, c, rs;
};
struct PackBatch {
    int n;
    int kcum[kPackJobs + 1];
    PackJob job[kPackJobs];
};
// STAGED: the row's C*R*S weights come in once with 16-B coalesced loads into shared
// memory (max |w| on the way), and the tap-major plane writes read them from there
// (rows up to kPackStageFloats; larger filters read the strided KCRS row from global)
constexpr int kPackStageFloats = 12288;   // 48 KB: C*R*S <= 12288 (C <= 1365 at 3x3)
template <bool STAGED>
__global__ void __launch_bounds__(256) pack_filters_f16x3_batched_kernel(const __grid_constant__ PackBatch B) {
    pdl_wait();
    __shared__ float red[8];
    extern __shared__ float4 stage4[];
    float *stage = reinterpret_cast<float *>(stage4);
    const int total = B.kcum[B.n];
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
        int j = 0;
        while (B.kcum[j + 1] <= g) ++j;
        const PackJob &J = B.job[j];
        const int kk = g - B.kcum[j], c = J.c, rs = J.rs, k = J.k;
        const int crs = c * rs;
        const int64_t plane = (int64_t)rs * k * c;
        const float *wr = J.w + (int64_t)kk * crs;
        float mx = 0.0f;
        if (STAGED) {
            if (((reinterpret_cast<uintptr_t>(wr) & 15) == 0) && (crs & 3) == 0) {
                const float4 *w4 = reinterpret_cast<const float4 *>(wr);
                for (int i = threadIdx.x; i < (crs >> 2); i += blockDim.x) {
                    const float4 v = __ldg(w4 + i);
                    stage4[i] = v;
                    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
                }
            } else {
                for (int i = threadIdx.x; i < crs; i += blockDim.x) {
                    const float v = wr[i];
                    stage[i] = v;
                    mx = fmaxf(mx, fabsf(v));
                }
            }
        } else {
            for (int i = threadIdx.x; i < crs; i += blockDim.x) mx = fmaxf(mx, fabsf(wr[i]));
        }
        for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        mx = red[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, red[i]);
        const int e = f16_row_exp(mx);
        const float sc = pow2f(e);
        const float *src = STAGED ? stage : wr;
        const int pairs = (c + 1) / 2;
        // (tap, pair) of t walked incrementally: one division per row, not one per pair
        // (the per-pair division made this kernel issue-bound: 71 % issue slots busy)
        const int dtap = (int)blockDim.x / pairs, dp = (int)blockDim.x - dtap * pairs;
        int tap = (int)threadIdx.x / pairs, pp = (int)threadIdx.x - tap * pairs;
        for (int t = threadIdx.x; t < rs * pairs; t += blockDim.x) {
            const int cc = 2 * pp;
            __half *hrow = J.wq + ((int64_t)tap * k + kk) * c;
            const float v0 = src[cc * rs + tap] * sc;
            const float v1 = cc + 1 < c ? src[(cc + 1) * rs + tap] * sc : 0.0f;
            const __half2 hi = __floats2half2_rn(v0, v1);
            const float2 hf = __half22float2(hi);
            const __half2 lo = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
            if (cc + 1 < c) {
                *reinterpret_cast<__half2 *>(hrow + cc) = hi;
                *reinterpret_cast<__half2 *>(hrow + plane + cc) = lo;
            } else {
                hrow[cc] = __low2half(hi);
                hrow[plane + cc] = __low2half(lo);
            }
            tap += dtap;
            pp += dp;
            if (pp >= pairs) {
                pp -= pairs;
                ++tap;
            }
        }
        if (threadIdx.x == 0) J.col_exp[kk] = e;
        __syncthreads();   // red[] and the stage are reused by the next row
    }
}

// 3xF16C activation scale: per-block max |x| (float bits) into partials[blockIdx.x];
// the GEMM reduces the nred partials into one exponent (f16c_act_exp).
// The grid walks x from its END to its start, so the most recently read ~L2-size
// tail of the walk is the START of x -- where the GEMM's first work items (low
// images first) read: for inputs larger than L2 about one L2's worth of the
// GEMM's activation reads hit L2 instead of HBM.
constexpr int kAbsmaxBlocks = 296;
__global__ void __launch_bounds__(256) absmax_partials_kernel(const float *__restrict__ x, int64_t n,
                                                              int *__restrict__ partials) {
    pdl_wait();
    __shared__ float red[8];
    float m = 0.0f;
    const int64_t n4 = n >> 2;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    for (int64_t j = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += step)
        m = fmaxf(m, fabsf(x[j]));
    int64_t i = n4 - 1 - (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    for (; i - 3 * step >= 0; i -= 4 * step) {
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = __ldg(x4 + i - j * step);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
    }
    for (; i >= 0; i -= step) {
        const float4 v = __ldg(x4 + i);
        m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
        partials[blockIdx.x] = __float_as_int(m);
    }
}

// KCRS -> [R*S][K][C] (fp32 or bf16, round-to-nearest-even)
template <typename T>
__global__ void pack_filter_igemm_kernel(const float *w, T *wq, int k, int c, int rs) {
    pdl_wait();
    const int64_t total = (int64_t)k * c * rs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int cc = i % c;
        const int kk = (i / c) % k;
        const int tap = i / ((int64_t)c * k);
        const float v = w[((int64_t)kk * c + cc) * rs + tap];
        if constexpr (sizeof(T) == 2)
            wq[i] = __float2bfloat16_rn(v);
        else
            wq[i] = v;
    }
}

// fp32 -> bf16 (RNE), 8 elements per thread-step when aligned
__global__ void convert_bf16_kernel(const float *__restrict__ src, __nv_bfloat16 *__restrict__ dst,
                                    int64_t n) {
    pdl_wait();
    const int64_t n8 = n / 8;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += step) {
        const float4 a = reinterpret_cast<const float4 *>(src)[2 * i];
        const float4 b = reinterpret_cast<const float4 *>(src)[2 * i + 1];
        __nv_bfloat162 o[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                               __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
        reinterpret_cast<uint4 *>(dst)[i] = *reinterpret_cast<uint4 *>(o);
    }
    for (int64_t i = n8 * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += step)
        dst[i] = __float2bfloat16_rn(src[i]);
}

static int vfail(char *reason, size_t rlen, int code, const char *fmt, va_list ap) {
    vsnprintf(reason, rlen, fmt, ap);
    set_error("%s", reason);
    return code;
}

static int pfail(char *reason, size_t rlen, int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    int rc = vfail(reason, rlen, code, fmt, ap);
    va_end(ap);
    return rc;
}

// Ring depth, smem and occupancy shared by the conv and batched plans.  The
// outputs live in TMEM, so s_b only sizes the TMA ring: ring bytes <= 6*s_b
// (s_b = 16384 words -> 96 KB, two CTAs per SM; 32768 -> 192 KB, one deep-ring
// CTA per SM), 2..12 stages.
// pair = true: the persistent CTA-pair kernel (igemm_pair.cuh), selected by a
// tile with n_zt == 2 (two CTAs share the z = BN output channels of one MMA);
// n_zt == 1: one 128-row tile per CTA (igemm_tcgen05.cuh).
static int plan_ring(IgemmPlan *pl, int bn, int kind, int s_b, bool pair, char *reason, size_t rlen) {
    if (pair) {
        // persistent pair: one CTA per SM, the whole shared memory is the ring
        // (halo: two footprint slots first, the filter stages in the rest)
        PairFn pfn = pl->fold ? pair_kernel_fold(bn, kind, pl->tsa, pl->resb_slots > 0)
                              : pair_kernel(bn, kind, pl->halo, pl->tsa);
        if (!pfn)
            return pfail(reason, rlen, CONVIO_EINFEASIBLE,
                         pl->tsa ? "A-in-TMEM tiles need 3xTF32 (z in {64, 128}, no halo) or 3xF16"
                                 : "tcgen05 tiles need z in {64, 128, 256}, got %d", bn);
        const int mult = (kind == KIND_3XTF32 || kind == KIND_3XF16 || kind == KIND_3XF16C) ? 2 : 1;
        // non-halo 3xTF32 without TSA: hi-only TMA stages + 2 decoupled lo slots
        const bool loslot = kind == KIND_3XTF32 && !pl->halo && !pl->tsa && bn == 256;
        // 3xF16C with A in TMEM, no halo: the fp32 activation boxes in their own ring of
        // na [A0 | A1] slots (released by the converters), the stages hold the filter planes
        const bool aring = pl->tsa && kind == KIND_3XF16C && !pl->halo;
        if (aring) pl->na = bn >= 256 ? 3 : (bn >= 128 ? 4 : 5);
        if (const char *na = getenv("CONVIO_DEV_NA"))   // dev knob: A-ring depth sensitivity
            if (aring) pl->na = std::max(2, std::min(6, atoi(na)));
        const size_t stage_bytes = (pl->tsa && kind == KIND_3XTF32) ? (size_t)(128 * 128 + 2 * (bn / 2) * 128)
                                           : (size_t)((pl->halo || aring ? 0 : 128 * 128) + (bn / 2) * 128) *
                                                 (loslot ? 1 : mult);
        const size_t a_ring = pl->halo ? (size_t)pl->na * pl->a_slot * mult
                                       : (aring ? (size_t)pl->na * 2 * 128 * 128 : (loslot ? 2 * stage_bytes : 0));
        const size_t budget = 227 * 1024 - 1024 - 1024 - pair_epi_bytes(pl->fold) - pair_epi_const_bytes(pl->P.k);
        if (a_ring + 2 * stage_bytes > budget)
            return pfail(reason, rlen, CONVIO_EINFEASIBLE, "tcgen05 pair footprint ring does not fit");
        // small stages (narrow BN, no lo copy) need many in flight to cover the
        // TMA latency (~1 us) at a few hundred MMA cycles per stage
        int stages = (int)std::min<size_t>(16, (budget - a_ring) / stage_bytes);
        if (const char *cap = getenv("CONVIO_DEV_MAX_STAGES"))   // dev knob: ring-depth sensitivity
            stages = std::max(2, std::min(stages, atoi(cap)));
        if (pl->resb_slots > 0) {   // resident filter: exactly one slot per k-block
            if (a_ring + (size_t)pl->resb_slots * stage_bytes > budget)
                return pfail(reason, rlen, CONVIO_EINFEASIBLE, "resident filter slice does not fit");
            stages = pl->resb_slots;
        }
        if (stages < 2)
            return pfail(reason, rlen, CONVIO_EINFEASIBLE, "tcgen05 pair ring does not fit");
        pl->P.stages = stages;
        pl->pair = true;
        pl->pfn = pfn;
        pl->fn = nullptr;
        pl->smem = a_ring + stages * stage_bytes + 1024 + 1024 + pair_epi_bytes(pl->fold) +
                   pair_epi_const_bytes(pl->P.k);
        pl->bn = bn;
        pl->kind = kind;
        pl->threads = kind == KIND_3XF16C ? 512 : (kind == KIND_3XTF32 ? ((bn >= 256 || pl->tsa) ? 384 : 512) : 256);
        if (launch_fit_cluster((const void *)pfn, pl->threads, pl->smem, &pl->regs) < 1)
            return pfail(reason, rlen, CONVIO_EINFEASIBLE,
                         "tcgen05 pair block (%d threads, %zu B smem) does not fit", pl->threads,
                         pl->smem);
        return CONVIO_OK;
    }
    if (kind == KIND_3XF16C)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "3xF16 implicit GEMMs run on the CTA pair (n_zt = 2)");
    IgemmFn fn = igemm_kernel(bn, kind);
    if (!fn)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "tcgen05 tiles need z in {64, 128, 256}, got %d",
                     bn);
    const size_t stage_bytes = (size_t)(128 * 128 + bn * 128) * (kind == KIND_3XTF32 ? 2 : 1);
    const size_t ring_cap = std::min<size_t>((size_t)6 * s_b, 227 * 1024 - 2048);
    int stages = (int)std::min<size_t>(12, ring_cap / stage_bytes);
    if (stages < 2) stages = 2;
    while (stages > 2 && stages * stage_bytes + 2048 > 227 * 1024) --stages;
    const size_t smem = stages * stage_bytes + 1024 + 512;
    if (smem > 227 * 1024)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "tcgen05 ring needs %zu B smem", smem);
    pl->P.stages = stages;
    pl->fn = fn;
    pl->smem = smem;
    pl->bn = bn;
    pl->kind = kind;
    pl->threads = kind == KIND_3XTF32 ? 256 : 128;
    if (launch_fit((const void *)fn, pl->threads, smem, &pl->regs) < 1)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "tcgen05 block (%d threads, %zu B smem) does not fit",
                     pl->threads, smem);
    return CONVIO_OK;
}

// persistent grid: one CTA pair per TPC (fewer if there are fewer work items).
// Tail split-K (non-halo conv tiles): when the last round of tile items would leave
// pairs idle -- ResNet-50 res4 at batch 256: 196 items on 74 pairs, 3 rounds for
// 2.65 rounds of work -- the last T tile items are split into S K ranges so the
// partial tiles fill the final round; the epilogue reduce-adds them (TMA .add) into
// the output zeroed from the tail's first image on (bias by the first split; never
// with ReLU, see igemm_launch).  (T, S) minimise the modelled rounds of k-blocks,
// and are kept only if they save >= 5 %.
static int finish_pair_grid(IgemmPlan *pl) {
    const int pairs = (pl->blocks_per_group + 1) / 2;
    const int64_t base = (int64_t)pl->groups * pairs * (pl->fold ? 1 : pl->P.k / pl->bn);
    const int64_t nclus = std::max(1, device_sms() / 2);
    pl->P.splits = 1;
    pl->tail_start = base;
    static const bool no_tail = getenv("CONVIO_DEV_NO_TAIL") != nullptr;   // dev knob: A/B timing
    if (!pl->halo && !pl->P.batched && base % nclus && !no_tail) {
        const int64_t kb = pl->P.kblocks;
        const double whole = (double)((base + nclus - 1) / nclus) * kb;
        double best = whole * 0.95;
        for (int64_t T = base % nclus; T <= base; T += nclus) {
            for (int sp = 2; sp <= 8; ++sp) {
                if (kb / sp < 6) break;
                const double t = (double)((base - T) / nclus) * kb +
                                 (double)((T * sp + nclus - 1) / nclus) * (double)((kb + sp - 1) / sp);
                if (t < best) {
                    best = t;
                    pl->P.splits = sp;
                    pl->tail_start = base - T;
                }
            }
            if (T >= 2 * nclus) break;   // the tail is at most the last two rounds
        }
    }
    const int64_t items = pl->tail_start + (base - pl->tail_start) * pl->P.splits;
    if (items >= ((int64_t)1 << 31)) {
        set_error("too many work items");
        return CONVIO_EINFEASIBLE;
    }
    const int64_t clusters = std::max<int64_t>(1, std::min<int64_t>(items, device_sms() / 2));
    pl->grid = dim3((unsigned)(2 * clusters), 1, 1);
    return CONVIO_OK;
}

// Halo staging (tile n_xt = 2, CTA pair n_zt = 2, stride 1): a block is y rows
// x fpr = x + S - 1 footprint columns (fpr % 8 == 0, fpr * y = 128 MMA rows,
// x valid outputs per row); the (y + R - 1) x fpr footprint is staged once per
// channel block and the taps are row offsets into it.  Ragged edges (Q % x,
// P % y) are zero-filled by TMA and masked in the epilogue.
static int plan_igemm_halo(const convio_conv_desc *d, const convio_tile *t, IgemmPlan *pl, char *reason,
                           size_t rlen, int kind, int p, int q) {
    if (t->n_yt != 1 || (t->n_zt != 2 && !(t->n_zt == 4 && kind == KIND_3XF16C)))
        return pfail(reason, rlen, CONVIO_EINFEASIBLE,
                     "halo-staged tcgen05 tiles take n_xt = 2, n_yt = 1, n_zt = 2 (CTA pair; "
                     "3xF16 also n_zt = 4: A operand in TMEM)");
    if (d->stride != 1)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "halo staging needs stride 1");
    const int fpr = t->x + d->s - 1;
    if (fpr % 8 || fpr * t->y != 128)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE,
                     "halo tile: (x + S - 1) = %d must be a multiple of 8 with (x + S - 1) * y = 128", fpr);
    if (d->k % t->z)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "z=%d does not divide K=%d", t->z, d->k);
    if (t->x > q + d->s - 1 || t->y > p + d->r - 1 || fpr > 256 || t->y + d->r - 1 > 256)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "halo tile larger than the output");
    const int cb = kblock_channels(kind);
    IgemmParams &P = pl->P;
    memset(&P, 0, sizeof(P));
    pl->halo = true;
    // fold the S horizontal taps into one MMA when N = S * z fits (z = K, 3x3)
    pl->fold = t->z == d->k && d->s == 3 && d->s * t->z == 192;
    pl->fpr = fpr;
    const int fp_rows = (t->y + d->r - 1) * fpr;
    pl->fp_bytes = fp_rows * 128;
    pl->a_slot = ((fp_rows + d->s - 1) * 128 + 1023) & ~1023;
    pl->tsa = t->n_zt == 4;
    // footprint slots: 3 when the ring keeps >= 3 filter stages (short items -- fold tiles,
    // 3 k-blocks -- need the next footprints in flight across a whole item: its TMA
    // latency under load is ~1.5 us); halo TSA fold with one n-block: the CTA's whole
    // filter slice stays resident when it fits next to the footprint slots (ResNet-50
    // res2 / VGG conv1_2: 3 x 24 KB)
    {
        const int mult = (kind == KIND_3XTF32 || kind == KIND_3XF16C) ? 2 : 1;
        const size_t budget = 227 * 1024 - 1024 - 1024 - pair_epi_bytes(pl->fold) - pair_epi_const_bytes(d->k);
        const size_t stage = (size_t)((pl->fold ? d->s * t->z : t->z) / 2) * 128 * mult;
        const size_t slot = (size_t)pl->a_slot * mult;
        const int kblocks = (pl->fold ? d->r : d->r * d->s) * (d->c / kblock_channels(kind));
        const size_t slice = (size_t)kblocks * stage;
        pl->na = 3 * slot + 3 * stage <= budget ? 3 : 2;
        if (pl->tsa && pl->fold && !pl->no_resb) {
            if (3 * slot + slice <= budget) pl->na = 3;
            if ((size_t)pl->na * slot + slice <= budget) pl->resb_slots = kblocks;
        }
    }
    P.k = d->k;   // (plan_ring sizes the epilogue's per-channel constants by K)
    int rc = plan_ring(pl, pl->fold ? d->s * t->z : t->z, kind, t->s_b, true, reason, rlen);
    if (rc) return rc;
    P.n = d->n; P.c = d->c; P.h = d->h; P.w = d->w; P.k = d->k; P.p = p; P.q = q;
    P.pad = d->pad; P.stride = 1; P.ks = d->r;
    P.bx = t->x; P.by = t->y; P.imgs = 1;
    P.tiles_x = (q + t->x - 1) / t->x; P.tiles_y = (p + t->y - 1) / t->y; P.img_groups = d->n;
    P.cblocks = d->c / cb; P.kblocks = (pl->fold ? d->r : d->r * d->s) * P.cblocks;
    pl->groups = 1;
    pl->blocks_per_group = P.tiles_x * P.tiles_y * P.img_groups;
    return finish_pair_grid(pl);
}

// Gather halo (3xF16C, tile threads (1, 1, 8)): exact x * y pixel blocks of
// imgs = 128 / (x * y) stacked images (x | Q, y | P: no wrap-around columns, no ragged
// edges); the [imgs][fh][fw] input footprint (fw = (x - 1) * stride + S) is staged once
// per channel block and the converters gather each tap's rows from it into TMEM.
static int plan_igemm_gather(const convio_conv_desc *d, const convio_tile *t, IgemmPlan *pl, char *reason,
                             size_t rlen, int kind, int p, int q) {
    if (kind != KIND_3XF16C)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "gathered-footprint tiles (n_zt = 8) take 3xF16");
    if (q % t->x || p % t->y || d->k % t->z)
        return pfail(reason, rlen, schedule_error(), "tile %dx%dx%d does not divide output %dx%dx%d", t->x,
                     t->y, t->z, q, p, d->k);
    const int px = t->x * t->y;
    if (px > 128) return pfail(reason, rlen, CONVIO_EINFEASIBLE, "x*y=%d pixels exceed the M=128 MMA tile", px);
    const int imgs = std::max(1, std::min(128 / px, d->n));
    const int fw = (t->x - 1) * d->stride + d->s, fh = (t->y - 1) * d->stride + d->r;
    if (fw > 256 || fh > 256 || imgs > 256)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "footprint box dims > 256");
    const int cb = kblock_channels(kind);
    IgemmParams &P = pl->P;
    memset(&P, 0, sizeof(P));
    pl->halo = true;
    pl->gather = true;
    pl->tsa = true;
    pl->fw = fw;
    pl->fh = fh;
    pl->fpr = fw;
    const int fp_rows = fw * fh * imgs;
    pl->fp_bytes = fp_rows * 128;
    pl->a_slot = (fp_rows * 128 + 1023) & ~1023;
    pl->na = 2;
    {
        const size_t budget = 227 * 1024 - 1024 - 1024 - pair_epi_bytes(false) - pair_epi_const_bytes(d->k);
        const size_t stage = (size_t)(t->z / 2) * 128 * 2;
        if (3 * (size_t)pl->a_slot * 2 + 3 * stage <= budget) pl->na = 3;
    }
    P.k = d->k;
    int rc = plan_ring(pl, t->z, kind, t->s_b, true, reason, rlen);
    if (rc) return rc;
    P.n = d->n; P.c = d->c; P.h = d->h; P.w = d->w; P.k = d->k; P.p = p; P.q = q;
    P.pad = d->pad; P.stride = d->stride; P.ks = d->r;
    P.bx = t->x; P.by = t->y; P.imgs = imgs;
    P.tiles_x = q / t->x; P.tiles_y = p / t->y; P.img_groups = (d->n + imgs - 1) / imgs;
    P.cblocks = d->c / cb; P.kblocks = d->r * d->s * P.cblocks;
    pl->groups = 1;
    pl->blocks_per_group = P.tiles_x * P.tiles_y * P.img_groups;
    return finish_pair_grid(pl);
}

static int plan_igemm(const convio_conv_desc *d, const convio_tile *t, IgemmPlan *pl, char *reason,
                      size_t rlen, int kind) {
    auto fail = [&](int code, const char *fmt, ...) {
        va_list ap;
        va_start(ap, fmt);
        int rc = vfail(reason, rlen, code, fmt, ap);
        va_end(ap);
        return rc;
    };
    if (!d || !t) return fail(CONVIO_EINVAL, "null descriptor or tile");
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->k < 1 || d->r < 1 || d->s < 1 ||
        d->stride < 1 || d->pad < 0)
        return fail(CONVIO_EINVAL, "descriptor fields must be >= 1 (pad >= 0)");
    const int hp = d->h + 2 * d->pad, wp = d->w + 2 * d->pad;
    if (d->r > hp || d->s > wp) return fail(geometry_error(), "kernel larger than padded input");
    const int p = (hp - d->r) / d->stride + 1, q = (wp - d->s) / d->stride + 1;
    if (d->layout != CONVIO_LAYOUT_HWC)
        return fail(CONVIO_EINFEASIBLE, "tcgen05 implicit GEMM needs the HWC (NHWC) layout");
    if (t->layout != d->layout) return fail(CONVIO_EINVAL, "tile layout differs from tensor layout");
    if (d->stride > 2) return fail(CONVIO_EINFEASIBLE, "tcgen05 implicit GEMM supports stride 1 and 2");
    if (d->r != d->s) return fail(CONVIO_EINFEASIBLE, "square kernels only");
    const int cb = kblock_channels(kind);
    if (d->c % cb)
        return fail(CONVIO_EINFEASIBLE, "C=%d is not a multiple of %d (one 128-B K block)", d->c, cb);
    if (t->x < 1 || t->y < 1 || t->z < 1 || t->s_b < 1)
        return fail(CONVIO_EINFEASIBLE, "tile fields must be >= 1");
    if (t->n_xt == 1 && t->n_yt == 1 && t->n_zt == 8) return plan_igemm_gather(d, t, pl, reason, rlen, kind, p, q);
    if (t->n_xt == 2) return plan_igemm_halo(d, t, pl, reason, rlen, kind, p, q);
    if (q % t->x || p % t->y || d->k % t->z)
        return fail(schedule_error(), "tile %dx%dx%d does not divide output %dx%dx%d", t->x, t->y,
                    t->z, q, p, d->k);
    const int tile_w = d->stride * (t->x - 1) + d->s, tile_h = d->stride * (t->y - 1) + d->r;
    const int64_t resident = (int64_t)t->x * t->y * t->z + (int64_t)tile_w * tile_h + (int64_t)d->r * d->s * t->z;
    if (resident > t->s_b)
        return fail(schedule_error(), "stage 0 resident set %lld words exceeds s_b=%d",
                    (long long)resident, t->s_b);
    const int px = t->x * t->y;
    if (px > 128) return fail(CONVIO_EINFEASIBLE, "x*y=%d pixels exceed the M=128 MMA tile", px);
    if (t->x * d->stride > 256 || t->y * d->stride > 256)
        return fail(CONVIO_EINFEASIBLE, "TMA box dims > 256");
    IgemmParams &P = pl->P;
    memset(&P, 0, sizeof(P));
    if (t->n_xt != 1 || t->n_yt != 1 || (t->n_zt != 1 && t->n_zt != 2 && t->n_zt != 4))
        return fail(CONVIO_EINFEASIBLE,
                    "tcgen05 tiles take n_xt = n_yt = 1 and n_zt in {1 (one CTA), 2 (CTA pair), "
                    "4 (CTA pair, 3xTF32 / 3xF16 A operand in TMEM)}");
    pl->tsa = t->n_zt == 4;
    P.k = d->k;   // (plan_ring sizes the epilogue's per-channel constants by K)
    int rc = plan_ring(pl, t->z, kind, t->s_b, t->n_zt >= 2, reason, rlen);
    if (rc) return rc;
    const int imgs = std::max(1, std::min(128 / px, d->n));
    P.n = d->n; P.c = d->c; P.h = d->h; P.w = d->w; P.k = d->k; P.p = p; P.q = q;
    P.pad = d->pad; P.stride = d->stride; P.ks = d->r;
    P.bx = t->x; P.by = t->y; P.imgs = imgs;
    P.tiles_x = q / t->x; P.tiles_y = p / t->y; P.img_groups = (d->n + imgs - 1) / imgs;
    P.cblocks = d->c / cb; P.kblocks = d->r * d->s * P.cblocks;
    pl->groups = 1;
    pl->blocks_per_group = P.tiles_x * P.tiles_y * P.img_groups;
    if (pl->pair) return finish_pair_grid(pl);
    pl->grid = dim3(d->k / pl->bn, P.tiles_x * P.tiles_y * P.img_groups, 1);
    if (pl->grid.y > 65535) return fail(CONVIO_EINFEASIBLE, "grid exceeds launch limits");
    // split-K when the output tiles cannot fill the GPU (small batches, e.g. a
    // rank's shard of a sharded batch): up to two CTAs per SM, >= 4 k-blocks each;
    // partial tiles are added with fp32 atomics into the zeroed output (no ReLU)
    const int64_t ctas = (int64_t)pl->grid.x * pl->grid.y;
    const int target = 2 * device_sms();
    P.splits = 1;
    if (ctas < target && P.kblocks >= 8)
        P.splits = (int)std::max<int64_t>(1, std::min<int64_t>({8, (target + ctas - 1) / ctas, P.kblocks / 4}));
    pl->grid.z = P.splits;
    return CONVIO_OK;
}

// M[xi][t][k] = sum_c V[xi][t][c] * U[xi][k][c]: V is an "image" per xi of
// 1 x T pixels, U the filter of tap xi.
int plan_igemm_batched(int kind, int bn, int s_b, bool pair, bool tsa, int xi, int t_count, int c, int k,
                       IgemmPlan *pl, char *reason, size_t rlen) {
    const int cb = (kind == KIND_BF16 || kind == KIND_3XF16) ? 64 : 32;
    if (kind == KIND_3XF16 && (!pair || tsa))
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "3xF16 GEMMs run on the CTA pair (n_zt = 2)");
    if (c % cb)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "C=%d is not a multiple of %d", c, cb);
    if (k % bn)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "K=%d is not a multiple of z=%d", k, bn);
    IgemmParams &P = pl->P;
    memset(&P, 0, sizeof(P));
    pl->tsa = pair && tsa;
    P.k = k;   // (plan_ring sizes the epilogue's per-channel constants by K)
    int rc = plan_ring(pl, bn, kind, s_b, pair, reason, rlen);
    if (rc) return rc;
    P.n = xi; P.c = c; P.h = 1; P.w = t_count; P.k = k; P.p = 1; P.q = t_count;
    P.pad = 0; P.stride = 1; P.ks = 1;
    P.bx = 128; P.by = 1; P.imgs = 1;
    P.tiles_x = (t_count + 127) / 128; P.tiles_y = 1; P.img_groups = xi;
    P.cblocks = c / cb; P.kblocks = P.cblocks;
    P.batched = 1;
    P.splits = 1;
    pl->groups = xi;
    pl->blocks_per_group = P.tiles_x;
    if (pl->pair) return finish_pair_grid(pl);
    pl->grid = dim3(k / bn, P.tiles_x * xi, 1);
    if (pl->grid.y > 65535)
        return pfail(reason, rlen, CONVIO_EINFEASIBLE, "grid exceeds launch limits");
    return CONVIO_OK;
}

// the pair kernel's output map: fp32 NHWC [K][Q][P][N] (batched: [K][T][1][xi]), box =
// one 32-channel slice of a CTA's block (halo: its x valid columns), 128-B swizzle
static bool make_output_map(const IgemmPlan &pl, float *y, CUtensorMap *ty) {
    const IgemmParams &P = pl.P;
    if (reinterpret_cast<uintptr_t>(y) & 15) return false;
    cuuint64_t yd[4] = {(cuuint64_t)P.k, (cuuint64_t)P.q, (cuuint64_t)P.p, (cuuint64_t)P.n};
    cuuint64_t ys[3] = {(cuuint64_t)P.k * 4, (cuuint64_t)P.q * P.k * 4, (cuuint64_t)P.p * P.q * P.k * 4};
    cuuint32_t yb[4] = {32, (cuuint32_t)P.bx, (cuuint32_t)P.by, (cuuint32_t)P.imgs};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return encode_tensor_map_tiled_ex(ty, 4, y, yd, ys, yb, es, true);
}

static bool make_igemm_maps(const IgemmPlan &pl, const void *x, const void *wq, CUtensorMap *tx,
                            CUtensorMap *tw) {
    const IgemmParams &P = pl.P;
    if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(wq) & 15)) return false;
    // 2-byte operands (bf16, or the 3xF16 fp16 planes: TMA copies bytes, the type
    // only sets the element size)
    // 3xF16C: fp32 activations (32-channel boxes, split in smem), fp16 filter planes
    const bool bf = pl.kind == KIND_BF16 || pl.kind == KIND_3XF16;
    const bool wbf = bf || pl.kind == KIND_3XF16C;
    const int planes = pl.kind == KIND_3XF16 ? 2 : 1;   // hi, lo planes along images / taps
    const int wplanes = (pl.kind == KIND_3XF16 || pl.kind == KIND_3XF16C) ? 2 : 1;
    const cuuint64_t es_b = bf ? 2 : 4;
    const cuuint64_t wes_b = wbf ? 2 : 4;
    const cuuint32_t cb = bf ? 64 : 32;
    const cuuint32_t wcb = wbf ? 64 : 32;
    cuuint64_t xd[4] = {(cuuint64_t)P.c, (cuuint64_t)P.w, (cuuint64_t)P.h, (cuuint64_t)P.n * planes};
    cuuint64_t xs[3] = {(cuuint64_t)P.c * es_b, (cuuint64_t)P.w * P.c * es_b,
                        (cuuint64_t)P.h * P.w * P.c * es_b};
    // stride: box spans stride*(pixels) input positions, traversal stride picks every stride-th
    cuuint32_t xb[4] = {cb, (cuuint32_t)(P.bx * P.stride), (cuuint32_t)(P.by * P.stride),
                        (cuuint32_t)P.imgs};
    if (pl.gather) {   // [imgs][fh][fw] pixels, every one (no traversal stride)
        xb[1] = (cuuint32_t)pl.fw;
        xb[2] = (cuuint32_t)pl.fh;
        xb[3] = (cuuint32_t)P.imgs;
    } else if (pl.halo) {   // the block's whole input footprint: y + R - 1 rows of fpr pixels
        xb[1] = (cuuint32_t)pl.fpr;
        xb[2] = (cuuint32_t)(P.by + P.ks - 1);
        xb[3] = 1;
    }
    cuuint32_t xes[4] = {1, (cuuint32_t)(pl.gather ? 1 : P.stride), (cuuint32_t)(pl.gather ? 1 : P.stride), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const int taps = P.batched ? P.n : P.ks * P.ks;
    cuuint64_t wd[3] = {(cuuint64_t)P.c, (cuuint64_t)P.k, (cuuint64_t)taps * wplanes};
    cuuint64_t ws[2] = {(cuuint64_t)P.c * wes_b, (cuuint64_t)P.k * P.c * wes_b};
    cuuint32_t wb[3] = {wcb, (cuuint32_t)(pl.pair ? pl.bn / 2 : pl.bn), 1};
    const bool xok = bf ? encode_tensor_map_bf16_sw128(tx, 4, const_cast<void *>(x), xd, xs, xb, xes)
                        : encode_tensor_map_tiled_ex(tx, 4, const_cast<void *>(x), xd, xs, xb, xes, true);
    if (!xok) return false;
    if (pl.layers > 1) {   // grouped conv: G packed slices, layer_bytes apart
        if (pl.layer_bytes & 15) return false;
        if (pl.fold) {
            cuuint64_t fd[3] = {(cuuint64_t)P.c, (cuuint64_t)taps * P.k * wplanes, (cuuint64_t)pl.layers};
            cuuint64_t fs[2] = {(cuuint64_t)P.c * wes_b, (cuuint64_t)pl.layer_bytes};
            cuuint32_t fb[3] = {wcb, (cuuint32_t)(pl.bn / 2), 1};
            return encode_tensor_map_bf16_sw128(tw, 3, const_cast<void *>(wq), fd, fs, fb, es);
        }
        cuuint64_t gd[4] = {(cuuint64_t)P.c, (cuuint64_t)P.k, (cuuint64_t)taps * wplanes, (cuuint64_t)pl.layers};
        cuuint64_t gs[3] = {(cuuint64_t)P.c * wes_b, (cuuint64_t)P.k * P.c * wes_b, (cuuint64_t)pl.layer_bytes};
        cuuint32_t gb[4] = {wcb, (cuuint32_t)(pl.pair ? pl.bn / 2 : pl.bn), 1, 1};
        return encode_tensor_map_bf16_sw128(tw, 4, const_cast<void *>(wq), gd, gs, gb, es);
    }
    if (pl.fold) {   // packed filter as [R*S*K rows][C]: a kernel row's S*K rows are contiguous
        cuuint64_t fd[2] = {(cuuint64_t)P.c, (cuuint64_t)taps * P.k * wplanes};
        cuuint64_t fs[1] = {(cuuint64_t)P.c * wes_b};
        cuuint32_t fb[2] = {wcb, (cuuint32_t)(pl.bn / 2)};
        if (wbf) return encode_tensor_map_bf16_sw128(tw, 2, const_cast<void *>(wq), fd, fs, fb, es);
        return encode_tensor_map_tiled_ex(tw, 2, const_cast<void *>(wq), fd, fs, fb, es, true);
    }
    if (wbf) return encode_tensor_map_bf16_sw128(tw, 3, const_cast<void *>(wq), wd, ws, wb, es);
    return encode_tensor_map_tiled_ex(tw, 3, const_cast<void *>(wq), wd, ws, wb, es, true);
}

int igemm_launch(IgemmPlan &pl, const void *x, const void *wq, const float *bias, int relu, float *y,
                 cudaStream_t stream) {
    CUtensorMap tx, tw, ty;
    if (!make_igemm_maps(pl, x, wq, &tx, &tw) || (pl.pair && !make_output_map(pl, y, &ty))) {
        set_error("TMA descriptors cannot describe these tensors (alignment)");
        return CONVIO_EINFEASIBLE;
    }
    pl.P.bias = bias;
    pl.P.y = y;
    pl.P.relu = relu;
    if (pl.pair) {
        PairParams PP{};   // value-initialised: every field not set below is 0
        PP.g = pl.P;
        PP.groups = pl.groups;
        PP.blocks_per_group = pl.blocks_per_group;
        PP.pairs_per_group = (pl.blocks_per_group + 1) / 2;
        PP.nblocks = pl.fold ? 1 : pl.P.k / pl.bn;
        PP.base_items = PP.groups * PP.pairs_per_group * PP.nblocks;
        PP.tail_start = (int)pl.tail_start;
        if (PP.g.splits < 1 || relu) {   // ReLU does not commute with the split sum
            PP.g.splits = 1;
            PP.tail_start = PP.base_items;
        }
        PP.items = PP.tail_start + (PP.base_items - PP.tail_start) * PP.g.splits;
        if (PP.g.splits > 1) {
            // zero the output from the image group of the tail's first block on (whole
            // tiles before it overwrite their part of that range with plain stores)
            const int first_pair = PP.tail_start / PP.nblocks;
            const int first_block = 2 * (first_pair % PP.pairs_per_group);
            const int64_t img_lo = (int64_t)(first_block / (PP.g.tiles_x * PP.g.tiles_y)) * PP.g.imgs +
                                   (PP.g.layer_imgs ? (int64_t)(first_pair / PP.pairs_per_group) * PP.g.layer_imgs : 0);
            const size_t per_img = (size_t)PP.g.p * PP.g.q * PP.g.k;
            if (img_lo < PP.g.n)
                CONVIO_CUDA_TRY(cudaMemsetAsync(y + img_lo * per_img, 0,
                                                (size_t)(PP.g.n - img_lo) * per_img * sizeof(float), stream));
        }
        PP.fpr = pl.fpr;
        PP.fp_bytes = pl.fp_bytes;
        PP.a_slot = pl.a_slot;
        PP.na = pl.na;
        PP.scale_state = pl.scale_state;
        PP.gather = pl.gather ? 1 : 0;
        PP.fw = pl.fw;
        PP.fh = pl.fh;
        PP.fallback = 0;
        PP.spec_ctas = 0;
        PP.trace = nullptr;
#ifdef CONVIO_TRACE
        static unsigned long long *d_trace = nullptr;
        if (!d_trace) CONVIO_CUDA_TRY(cudaMalloc(&d_trace, 24 * 1024 * sizeof(unsigned long long)));
        CONVIO_CUDA_TRY(cudaMemsetAsync(d_trace, 0, 24 * 1024 * sizeof(unsigned long long), stream));
        PP.trace = d_trace;
        g_trace_ptr = d_trace;
#endif
        if (PP.g.splits > 1)   // after a memset node: a plain stream dependency
            pl.pfn<<<pl.grid, pl.threads, pl.smem, stream>>>(PP, tx, tw, ty);
        else
            CONVIO_CUDA_TRY(launch_pdl(pl.pfn, pl.grid, dim3(pl.threads), pl.smem, stream, PP, tx, tw, ty));
        note_launch();
        CONVIO_CUDA_TRY(cudaGetLastError());
        static const bool skip_check = getenv("CONVIO_DEV_SKIP_CHECK") != nullptr;   // dev: timing A/B only
        if (pl.kind == KIND_3XF16C && !skip_check) {
            // the checking launch: exits at once when the speculative scale held, else redoes
            // the whole conv with the exact scale (whole tiles, plain stores over the output)
            PairParams PF = PP;
            PF.fallback = 1;
            PF.g.splits = 1;
            PF.tail_start = PF.base_items;
            PF.items = PF.base_items;
            PF.spec_ctas = (int)pl.grid.x;
            const unsigned clus = (unsigned)std::max(1, std::min(PF.items, device_sms() / 2));
            CONVIO_CUDA_TRY(launch_pdl(pl.pfn, dim3(2 * clus), dim3(pl.threads), pl.smem, stream, PF, tx, tw, ty));
            note_launch();
            CONVIO_CUDA_TRY(cudaGetLastError());
        }
        return CONVIO_OK;
    }
    if (pl.P.splits > 1 && relu) {   // ReLU does not commute with the split sum
        pl.P.splits = 1;
        pl.grid.z = 1;
    }
    if (pl.P.splits > 1)
        CONVIO_CUDA_TRY(cudaMemsetAsync(y, 0, (size_t)pl.P.n * pl.P.p * pl.P.q * pl.P.k * sizeof(float), stream));
    if (pl.P.splits > 1)   // after a memset node: a plain stream dependency
        pl.fn<<<pl.grid, pl.threads, pl.smem, stream>>>(pl.P, tx, tw);
    else
        CONVIO_CUDA_TRY(launch_pdl(pl.fn, pl.grid, dim3(pl.threads), pl.smem, stream, pl.P, tx, tw));
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

int launch_convert_bf16(const float *src, void *dst, int64_t n, cudaStream_t stream) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n / 8 + 255) / 256, 148 * 16));
    CONVIO_CUDA_TRY(launch_pdl(convert_bf16_kernel, dim3(blocks), dim3(256), 0, stream, src,
                               (__nv_bfloat16 *)dst, n));
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

static inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// 3xF16C packed filter: [fp16 hi plane | fp16 lo plane] (align256) then col_exp[K]
static size_t f16c_filter_bytes(const convio_conv_desc *d) {
    return align256((size_t)4 * d->k * d->c * d->r * d->s) + align256((size_t)4 * d->k);
}
// 3xF16C workspace: [absmax partials (align256) | packed filter]
static size_t f16c_partials_bytes() { return align256((size_t)4 * kAbsmaxBlocks); }

int64_t igemm_workspace_bytes(const convio_conv_desc *d, int kind) {
    if (kind == KIND_3XF16C) return (int64_t)(f16c_partials_bytes() + f16c_filter_bytes(d));
    const int64_t wbytes = (int64_t)d->k * d->c * d->r * d->s * (kind == KIND_BF16 ? 2 : 4);
    if (kind != KIND_BF16) return wbytes;
    return (int64_t)align256(wbytes) + 2LL * d->n * d->c * d->h * d->w;
}

int igemm_query(const convio_conv_desc *d, const convio_tile *t, convio_launch_info *out, int kind) {
    IgemmPlan pl;
    int rc = plan_igemm(d, t, &pl, out->reason, sizeof(out->reason), kind);
    if (rc) return rc;
    out->legal = 1;
    out->grid_x = pl.grid.x; out->grid_y = pl.grid.y; out->grid_z = pl.grid.z;
    out->block_threads = pl.threads;
    out->smem_bytes = (int)pl.smem;
    out->regs_per_thread = pl.regs;
    out->channel_chunk = kblock_channels(kind);
    out->stages = pl.P.stages;
    out->p = pl.P.p; out->q = pl.P.q;
    out->flops = 2LL * d->n * d->k * pl.P.p * pl.P.q * (int64_t)d->c * d->r * d->s;
    out->workspace_bytes = igemm_workspace_bytes(d, kind);
    out->grid_z = pl.grid.z;
    snprintf(out->reason, sizeof(out->reason), "tcgen05 %s%s: M=%d (%d px x %d img per CTA), N=%d, %d stages%s",
             kind_name(kind), pl.fold ? (pl.tsa ? (pl.resb_slots ? " CTA pair (persistent, halo footprint shifted into TMEM, 3 taps per MMA, resident filter)" : " CTA pair (persistent, halo footprint shifted into TMEM, 3 taps per MMA)") : " CTA pair (persistent, halo footprint, 3 taps per MMA)") : pl.gather ? " CTA pair (persistent, footprint gathered into TMEM)" : pl.halo ? (pl.tsa ? " CTA pair (persistent, halo footprint shifted into TMEM)" : " CTA pair (persistent, halo-staged footprint)") : (pl.tsa ? " CTA pair (persistent, A in TMEM)" : (pl.pair ? " CTA pair (persistent)" : "")), pl.pair ? 256 : 128,
             pl.P.bx * pl.P.by, pl.P.imgs, pl.bn, pl.P.stages,
             pl.P.splits > 1 ? ", split-K" : "");
    return CONVIO_OK;
}

int launch_pack_filter_f16x3(const convio_conv_desc *desc, const float *w, void *packed, cudaStream_t stream) {
    const int blocks = std::max(1, std::min(desc->k, 148 * 8));
    __half *planes = (__half *)packed;
    int *col_exp = (int *)((uint8_t *)packed + align256((size_t)4 * desc->k * desc->c * desc->r * desc->s));
    CONVIO_CUDA_TRY(launch_pdl(pack_filter_f16x3_kernel, dim3(blocks), dim3(256), 0, stream, w, planes, col_exp,
                               desc->k, desc->c, desc->r * desc->s));
    note_launch();
    return CONVIO_OK;
}

int launch_absmax_partials(const float *x, int64_t n, int *partials, int *nred, cudaStream_t stream) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(kAbsmaxBlocks, (n / 4 + 2047) / 2048));
    CONVIO_CUDA_TRY(launch_pdl(absmax_partials_kernel, dim3(blocks), dim3(256), 0, stream, x, n, partials));
    note_launch();
    *nred = blocks;
    return CONVIO_OK;
}

int launch_pack_filter_igemm(const convio_conv_desc *desc, const float *w, void *wq, int bf16,
                             cudaStream_t stream) {
    const int64_t total = (int64_t)desc->k * desc->c * desc->r * desc->s;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
    if (bf16)
        CONVIO_CUDA_TRY(launch_pdl(pack_filter_igemm_kernel<__nv_bfloat16>, dim3(blocks), dim3(256), 0,
                                   stream, w, (__nv_bfloat16 *)wq, desc->k, desc->c, desc->r * desc->s));
    else
        CONVIO_CUDA_TRY(launch_pdl(pack_filter_igemm_kernel<float>, dim3(blocks), dim3(256), 0, stream,
                                   w, (float *)wq, desc->k, desc->c, desc->r * desc->s));
    note_launch();
    return CONVIO_OK;
}

}  // namespace convio

using namespace convio;

static int prec_kind(int32_t precision) {
    switch (precision) {
        case CONVIO_PREC_TF32: return KIND_TF32;
        case CONVIO_PREC_3XTF32: return KIND_3XTF32;
        case CONVIO_PREC_BF16: return KIND_BF16;
        case CONVIO_PREC_3XF16: return KIND_3XF16C;
        default: return -1;
    }
}

extern "C" {

int convio_pack_filter_igemm(const convio_conv_desc *desc, const float *w, float *wq, void *stream) {
    clear_error();
    if (!desc || !w || !wq) {
        set_error("null argument");
        return CONVIO_EINVAL;
    }
    return launch_pack_filter_igemm(desc, w, wq, 0, (cudaStream_t)stream);
}

int convio_pack_filter_igemm_bf16(const convio_conv_desc *desc, const float *w, void *wq,
                                  void *stream) {
    clear_error();
    if (!desc || !w || !wq) {
        set_error("null argument");
        return CONVIO_EINVAL;
    }
    return launch_pack_filter_igemm(desc, w, wq, 1, (cudaStream_t)stream);
}

int convio_pack_filter_igemm_f16x3(const convio_conv_desc *desc, const float *w, void *w_packed,
                                   void *stream) {
    clear_error();
    if (!desc || !w || !w_packed) {
        set_error("null argument");
        return CONVIO_EINVAL;
    }
    if (reinterpret_cast<uintptr_t>(w_packed) & 255) {
        set_error("convio_pack_filter_igemm_f16x3 needs a 256-byte aligned buffer");
        return CONVIO_EINVAL;
    }
    return launch_pack_filter_f16x3(desc, w, w_packed, (cudaStream_t)stream);
}

int convio_conv_igemm_grouped(const convio_conv_desc *desc, const convio_tile *tile, int32_t precision,
                              int32_t layers, const float *x, const void *w_packed, size_t layer_bytes,
                              const float *bias, int32_t relu, float *y, void *workspace, size_t workspace_bytes,
                              void *stream) {
    clear_error();
    reset_launches();
    const int kind = prec_kind(precision);
    if (kind != KIND_3XF16C) {
        set_error("grouped implicit GEMMs: 3xF16 only");
        return CONVIO_EINVAL;
    }
    if (!x || !w_packed || !y || !tile || !desc || layers < 1 || desc->n < 1) {
        set_error("null tensor pointer / descriptor / tile, or layers < 1");
        return CONVIO_EINVAL;
    }
    if ((reinterpret_cast<uintptr_t>(w_packed) & 255) || (layer_bytes & 255) ||
        layer_bytes < f16c_filter_bytes(desc) || (reinterpret_cast<uintptr_t>(workspace) & 255) ||
        !workspace || workspace_bytes < f16c_partials_bytes()) {
        set_error("grouped 3xF16: 256-byte aligned packed slices of >= %zu bytes and a %zu-byte workspace",
                  f16c_filter_bytes(desc), f16c_partials_bytes());
        return CONVIO_EINVAL;
    }
    if ((int64_t)desc->n * layers > INT32_MAX || layer_bytes / 4 > (size_t)INT32_MAX) {
        set_error("grouped 3xF16: layers * n (%lld) or the slice size overflows", (long long)desc->n * layers);
        return CONVIO_EINVAL;
    }
    convio_conv_desc dg = *desc;
    dg.n = desc->n * layers;   // the stacked batch
    IgemmPlan pl;
    char why[160];
    int rc = plan_igemm(&dg, tile, &pl, why, sizeof(why), kind);
    if (rc) return rc;
    if (!pl.pair || desc->n % pl.P.imgs) {
        set_error("grouped 3xF16 needs CTA-pair tiles whose image stack (%d) divides the per-layer batch %d",
                  pl.P.imgs, desc->n);
        return CONVIO_EINFEASIBLE;
    }
    pl.layers = layers;
    pl.layer_bytes = layer_bytes;
    pl.P.layer_imgs = layers > 1 ? desc->n : 0;
    if (layers > 1) {   // one group per layer: a pair never spans two layers' blocks
        pl.P.img_groups = (desc->n + pl.P.imgs - 1) / pl.P.imgs;
        pl.groups = layers;
        pl.blocks_per_group = pl.P.tiles_x * pl.P.tiles_y * pl.P.img_groups;
        rc = finish_pair_grid(&pl);
        if (rc) return rc;
    }
    pl.P.col_stride = (int)(layer_bytes / 4);
    pl.scale_state = (int *)workspace;
    pl.P.col_exp = (const int *)((const uint8_t *)w_packed +
                                 align256((size_t)4 * desc->k * desc->c * desc->r * desc->s));
    return igemm_launch(pl, x, w_packed, bias, relu, y, (cudaStream_t)stream);
}

int convio_pack_filters_igemm_f16x3_batched(int32_t count, const convio_conv_desc *descs, const float *const *w,
                                            void *const *w_packed, void *stream) {
    clear_error();
    if (count < 0 || count > kPackJobs || (count && (!descs || !w || !w_packed))) {
        set_error("count must be in [0, %d] with non-null arrays", kPackJobs);
        return CONVIO_EINVAL;
    }
    if (!count) return CONVIO_OK;
    PackBatch B;
    memset(&B, 0, sizeof(B));
    B.n = count;
    for (int i = 0; i < count; ++i) {
        const convio_conv_desc *d = descs + i;
        if (!w[i] || !w_packed[i] || (reinterpret_cast<uintptr_t>(w_packed[i]) & 255) || d->k < 1 || d->c < 1 ||
            d->r < 1 || d->s < 1) {
            set_error("job %d: null / unaligned buffer or empty filter", i);
            return CONVIO_EINVAL;
        }
        B.job[i].w = w[i];
        B.job[i].wq = (__half *)w_packed[i];
        B.job[i].col_exp = (int *)((uint8_t *)w_packed[i] + align256((size_t)4 * d->k * d->c * d->r * d->s));
        B.job[i].k = d->k;
        B.job[i].c = d->c;
        B.job[i].rs = d->r * d->s;
        B.kcum[i + 1] = B.kcum[i] + d->k;
    }
    int max_crs = 0;
    for (int i = 0; i < count; ++i) max_crs = std::max(max_crs, B.job[i].c * B.job[i].rs);
    const int blocks = std::max(1, std::min(B.kcum[count], 148 * 8));
    if (max_crs <= kPackStageFloats) {
        const size_t smem = (size_t)((max_crs + 3) & ~3) * 4;
        // (a per-device function attribute: set on every call, not cached per process)
        CONVIO_CUDA_TRY(cudaFuncSetAttribute(pack_filters_f16x3_batched_kernel<true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kPackStageFloats * 4));
        CONVIO_CUDA_TRY(launch_pdl(pack_filters_f16x3_batched_kernel<true>, dim3(blocks), dim3(256), smem,
                                   (cudaStream_t)stream, B));
    } else {
        CONVIO_CUDA_TRY(launch_pdl(pack_filters_f16x3_batched_kernel<false>, dim3(blocks), dim3(256), 0,
                                   (cudaStream_t)stream, B));
    }
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

#ifdef CONVIO_TRACE
// dev builds only: copy the last pair-kernel pipeline trace (8 x 1024 clock64 stamps)
int convio_dev_trace(unsigned long long *host) {
    if (!g_trace_ptr) return CONVIO_EINVAL;
    return cudaMemcpy(host, g_trace_ptr, 24 * 1024 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
                   cudaSuccess
               ? CONVIO_OK
               : CONVIO_EINTERNAL;
}
#endif

int64_t convio_pack_filter_igemm_f16x3_bytes(const convio_conv_desc *desc) {
    if (!desc) return -1;
    return (int64_t)f16c_filter_bytes(desc);
}

int convio_convert_bf16(const float *src, void *dst, int64_t n, void *stream) {
    clear_error();
    if (!src || !dst || n < 0) {
        set_error("null argument or negative count");
        return CONVIO_EINVAL;
    }
    if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15)) {
        set_error("convio_convert_bf16 needs 16-byte aligned buffers");
        return CONVIO_EINVAL;
    }
    if (n == 0) return CONVIO_OK;
    return launch_convert_bf16(src, dst, n, (cudaStream_t)stream);
}

int convio_conv_igemm(const convio_conv_desc *desc, const convio_tile *tile, int32_t precision,
                      const float *x, const void *w, int32_t w_is_packed, const float *bias,
                      int32_t relu, float *y, void *workspace, size_t workspace_bytes, void *stream) {
    clear_error();
    reset_launches();
    const int kind = prec_kind(precision);
    if (kind < 0) {
        set_error("unknown precision %d", precision);
        return CONVIO_EINVAL;
    }
    if (!x || !w || !y || !tile || !desc) {
        set_error("null tensor pointer, descriptor or tile");
        return CONVIO_EINVAL;
    }
    IgemmPlan pl;
    char why[160];
    int rc = plan_igemm(desc, tile, &pl, why, sizeof(why), kind);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (kind == KIND_3XF16C) {
        // workspace [absmax partials | packed fp16 filter planes + col_exp]; a packed
        // filter (convio_pack_filter_igemm_f16x3) leaves only the partials here
        const size_t need_here = w_is_packed ? f16c_partials_bytes() : (size_t)igemm_workspace_bytes(desc, kind);
        if (!workspace || workspace_bytes < need_here || (reinterpret_cast<uintptr_t>(workspace) & 255)) {
            set_error("workspace of %zu bytes (256-byte aligned) needed (activation scale state%s)", need_here,
                      w_is_packed ? "" : " + packed fp16 filter");
            return CONVIO_EINVAL;
        }
        if (reinterpret_cast<uintptr_t>(w) & 255) {
            set_error("3xF16 filter operand must be 256-byte aligned");
            return CONVIO_EINVAL;
        }
        const void *wq = w;
        if (!w_is_packed) {
            wq = (uint8_t *)workspace + f16c_partials_bytes();
            rc = launch_pack_filter_f16x3(desc, (const float *)w, const_cast<void *>(wq), st);
            if (rc) return rc;
        }
        // speculative activation scale: the state lives in the workspace's first 16 bytes
        // (zeroed by the caller before a workspace's first use: no speculation yet)
        pl.scale_state = (int *)workspace;
        pl.P.col_exp = (const int *)((const uint8_t *)wq + align256((size_t)4 * desc->k * desc->c * desc->r * desc->s));
        return igemm_launch(pl, x, wq, bias, relu, y, st);
    }
    const bool bf = kind == KIND_BF16;
    const size_t wbytes = (size_t)desc->k * desc->c * desc->r * desc->s * (bf ? 2 : 4);
    const size_t need = (size_t)igemm_workspace_bytes(desc, kind);
    const size_t need_here = bf ? need : (w_is_packed ? 0 : need);
    if (need_here && (!workspace || workspace_bytes < need_here)) {
        set_error("workspace of %zu bytes needed (%s)", need_here,
                  bf ? "bf16 filter + bf16 activations" : "packed filter");
        return CONVIO_EINVAL;
    }
    const void *wq = w;
    if (!w_is_packed) {
        rc = launch_pack_filter_igemm(desc, (const float *)w, workspace, bf, st);
        if (rc) return rc;
        wq = workspace;
    }
    const void *xa = x;
    if (bf) {
        void *xb = (uint8_t *)workspace + align256(wbytes);
        rc = launch_convert_bf16(x, xb, (int64_t)desc->n * desc->c * desc->h * desc->w, st);
        if (rc) return rc;
        xa = xb;
    }
    return igemm_launch(pl, xa, wq, bias, relu, y, st);
}

int convio_conv_igemm_tf32(const convio_conv_desc *desc, const convio_tile *tile, const float *x,
                           const float *w, int32_t w_is_packed, const float *bias, int32_t relu,
                           float *y, void *workspace, size_t workspace_bytes, void *stream) {
    return convio_conv_igemm(desc, tile, CONVIO_PREC_TF32, x, w, w_is_packed, bias, relu, y,
                             workspace, workspace_bytes, stream);
}

int convio_conv_igemm_3xtf32(const convio_conv_desc *desc, const convio_tile *tile, const float *x,
                             const float *w, int32_t w_is_packed, const float *bias, int32_t relu,
                             float *y, void *workspace, size_t workspace_bytes, void *stream) {
    return convio_conv_igemm(desc, tile, CONVIO_PREC_3XTF32, x, w, w_is_packed, bias, relu, y,
                             workspace, workspace_bytes, stream);
}

}  // extern "C"
