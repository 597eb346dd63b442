// Persistent CTA-pair implicit GEMM on tcgen05 (cta_group::2, M = 256).
//
// Same GEMM view as igemm_tcgen05.cuh (D[m][n] += A[m][kk] * B[n][kk], m =
// pixels, n = output channels, kk = taps x channel blocks), re-organised for
// the B200 tensor-core / L2 balance:
//
//  * A cluster of two CTAs on one TPC shares one M = 256 x N = BN MMA: each
//    CTA stages its own 128-pixel A block and HALF of the BN filter rows; the
//    leader's single thread issues tcgen05.mma.cta_group::2, which reads both
//    CTAs' shared memory.  Per-SM operand traffic (TMA from L2 and smem reads
//    by the tensor core) drops from (128 + BN) to (128 + BN/2) rows per k-block.
//  * Persistent: one pair per TPC walks the (pixel-pair, n-block) work list
//    (n fastest, so the pair re-reads its A block from L2 while it is hot).
//  * The TMEM accumulator is double-buffered (2 x BN columns): the epilogue
//    warps drain tile i while the MMA issuer accumulates tile i+1.
//
// HALO variant (stride 1, tile n_xt = 2): instead of one tap-shifted A box per
// (tap, channel block), the block's input footprint is staged once per channel
// block in its own ring and the R*S taps are descriptor offsets into it (an
// SW128 K-major operand may start at any 128-B row: the swizzle phase follows
// the absolute smem address, see scripts/dev/umma_shift_selftest.cu), cutting
// the A operand's L2 traffic by ~R*S / (1 + halo).  Each footprint row holds
// fpr pixels of which fpr - S + 1 are valid outputs (the rest are wrap-around
// rows, computed and never stored).
//
// Warp roles (per CTA):  warp 0 = TMA producer, warp 1 = MMA issuer (leader
// CTA) + TMEM allocator, warps 4..7 = epilogue (TMEM lane quadrants 0..3),
// warps 8.. = 3xTF32 converters (KIND_3XTF32 only; 4 at BN = 256, 8 below).
//
// Synchronisation (s = ring stage, a = accumulator buffer):
//   full[s]   leader: TMA bytes of BOTH CTAs (non-split; .cta_group::2 TMA
//             signals the leader's barrier) / own bytes (split)
//   conv[s]   leader, count 8: the 4 converter warps of each CTA (split)
//   empty[s]  each CTA, via tcgen05.commit multicast to both CTAs
//   tfull[a]  each CTA, via tcgen05.commit multicast (accumulator ready)
//   tempty[a] leader, count 8: the 4 epilogue warps of each CTA
#pragma once

#include <cuda_fp16.h>

#include "igemm_tcgen05.cuh"

namespace convio {

// epilogue staging box after the ring + barriers: 128 rows x 32 fp32 channels (one TMA store);
// FOLD tiles (3-k-block items: the drain paces the MMAs) double-buffer it
constexpr size_t kPairEpiBytes = 128 * 32 * sizeof(float);
constexpr size_t pair_epi_bytes(bool fold) { return fold ? 2 * kPairEpiBytes : kPairEpiBytes; }
// after the staging box(es): the epilogue's per-channel constants in shared memory --
// bias[K] and the 3xF16 column scales 2^-e[k] as floats (K <= kEpiConstK; larger K
// reads them from global memory).  Per-lane __ldg's of 32 biases + 32 exponents per
// chunk (~2k cycles of dependent L1/L2 latency) had made the drain the pacer of short
// items (fold tiles: 3 k-blocks)
constexpr int kEpiConstK = 1024;
inline size_t pair_epi_const_bytes(int k) { return k <= kEpiConstK ? (size_t)8 * k : 0; }

struct PairParams {
    IgemmParams g;          // geometry as in the single-CTA kernel
    int groups;             // 1 (conv) or xi (batched Winograd GEMMs)
    int blocks_per_group;   // pixel blocks per group
    int pairs_per_group;    // ceil(blocks_per_group / 2)
    int nblocks;            // K / BN
    int items;              // tail_start + (base_items - tail_start) * splits
    int base_items;         // groups * pairs_per_group * nblocks (one K range each)
    int tail_start;         // tile items from here on are split into g.splits K ranges
    // 3xF16C speculative activation scale (see f16c_spec_ok): scale_state[0] = the max |x|
    // (float bits) to speculate with, [1] = [0] ^ kScaleTag, [2] = the value the speculative
    // launch used, [4 + cta] = each speculative CTA's observed max |x|.  fallback = 1: the
    // checking launch -- exits at once if the speculation held, else redoes the conv with
    // the observed (exact) max
    int *scale_state;
    int fallback;
    int spec_ctas;          // the speculative launch's CTA count (its partial maxima)
    // gather halo (HALO + TSA, gather = 1): A row m = output pixel (img, py, px) of an
    // exact x * y * imgs block (no wrap-around columns); the footprint box is
    // [imgs][fh][fw] pixels, fw = (x - 1) * stride + S, and the converters read tap (r, s)
    // of row m at footprint pixel (img, py * stride + r, px * stride + s)
    int gather;
    int fw, fh;
    // halo staging (HALO kernels): the (y + R - 1) x fpr input footprint of a
    // 128-row block is staged ONCE per channel block; tap (r, s) is the view
    // starting (r * fpr + s) rows into it (rows = y x fpr pixels, x = fpr - S + 1
    // of each footprint row valid).  fp_bytes = footprint box bytes per CTA,
    // a_slot = its smem slot (rounded to 1 KB, + S - 1 overrun rows).
    int fpr;
    int fp_bytes;
    int a_slot;
    int na;                 // footprint slots
    unsigned long long *trace;   // CONVIO_TRACE builds: per-role clock64 stamps of cluster 0
};

// Pipeline trace (dev builds with -DCONVIO_TRACE): the leader CTA of cluster 0
// stamps clock64() at each role's hand-off points into trace[row][i] (row: 0
// producer may issue k-block i, 1 converter saw its data, 2 converter done, 3 MMA
// issuer saw it converted, 4 MMAs issued, 5 epilogue saw accumulator i, 6 drained)
#ifdef CONVIO_TRACE
#define PAIR_TRACE(row, i)                                                                      \
    do {                                                                                        \
        if (PP.trace && blockIdx.x < 2 && (i) < 1024) PP.trace[((row) + 8 * blockIdx.x) * 1024 + (i)] = clock64(); \
    } while (0)
// fine epilogue stamps (leader CTA of cluster 0, warp 4 lane 0): rows 18..23
#define EPI_TRACE(row, i)                                                                       \
    do {                                                                                        \
        if (PP.trace && blockIdx.x == 0 && (i) < 1024) PP.trace[(row) * 1024 + (i)] = clock64(); \
    } while (0)
#else
#define PAIR_TRACE(row, i) \
    do {                   \
    } while (0)
#define EPI_TRACE(row, i) \
    do {                  \
    } while (0)
#endif

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// shared::cluster address of the same variable in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

// Arrive on a barrier of the pair (shared::cluster address from mapa) with the
// default .release.cta semantics -- the form CUTLASS's 2-SM transform pipeline
// uses (cutlass/arch/barrier.h umma_arrive_2x1SM_sm0).  The .release.cluster
// form compiles to MEMBAR.ALL.GPU + ERRBAR per arrive, which measured as the
// 3xTF32 converters' dominant stall (ncu, res2 pair BN=64).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

// wait on a barrier that the peer CTA also arrives on (default acquire, as the
// CUTLASS 2-SM consumer waits)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) { mbar_wait(bar, parity); }

// TMA store of a staged output box (shared::cta -> global, bulk-group completion)
__device__ __forceinline__ void tma_store_4d(uint64_t map, uint32_t src, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(map),
        "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
// the same with an fp32 add into global (partial tiles of the split-K tail)
__device__ __forceinline__ void tma_reduce_add_4d(uint64_t map, uint32_t src, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(map),
        "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }
// tcgen05.ld without the wait: several loads in flight, one tcgen05.wait::ld
__device__ __forceinline__ void tmem_ld_x32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
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
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// named barrier among the 4 epilogue warps (id 1; id 0 is __syncthreads)
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// one lane of the (converged) warp: tcgen05.mma / commit are issued once per warp
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n.reg .pred P;\n"
        "elect.sync _|P, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

// Non-blocking probe of a barrier phase.  The MMA issuer probes the NEXT k-block's
// barrier while the current k-block's MMAs drain: a blocking wait between
// k-blocks costs ~130-230 issue cycles even on a completed phase, long enough to
// empty the tensor core's short MMA queue at N = 128 (64 -> 83 cycles per MMA,
// scripts/dev/umma_contention_probe.cu).
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}

// TMA load whose completion is signalled on the LEADER CTA's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_4d_pair(void *dst, uint64_t map, int c0, int c1, int c2, int c3,
                                                 uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void *dst, uint64_t map, int c0, int c1, int c2,
                                                 uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d_pair(void *dst, uint64_t map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}

template <int BN, int KIND>
__device__ __forceinline__ constexpr uint32_t idesc_m256() {
    // A/B format: 0 F16 (kind::f16), 1 BF16 (kind::f16), 2 TF32 (kind::tf32)
    constexpr uint32_t F = KIND == KIND_BF16 ? 1u : ((KIND == KIND_3XF16 || KIND == KIND_3XF16C) ? 0u : 2u);
    return (1u << 4) | (F << 7) | (F << 10) |
           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

template <int KIND>
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
    if constexpr (KIND == KIND_BF16 || KIND == KIND_3XF16 || KIND == KIND_3XF16C) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
            "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
    }
}

__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

// Pixel-block origin of block `blk` of group `grp` (conv: group 0, blocks
// enumerate (img group, tile row, tile col); batched: group = xi, blocks are
// 128-tile runs of the T axis).  Out-of-range blocks land beyond the tensor,
// so TMA fills zeros and the epilogue masks every row.
__device__ __forceinline__ void pair_block_origin(const IgemmParams &P, int grp, int blk, int &ox0,
                                                  int &oy0, int &img0) {
    if (P.batched) {
        ox0 = blk * P.bx;
        oy0 = 0;
        img0 = grp;
    } else {
        const int xt = blk % P.tiles_x;
        const int rest = blk / P.tiles_x;
        const int yt = rest % P.tiles_y;
        const int ig = rest / P.tiles_y;
        ox0 = xt * P.bx;
        oy0 = yt * P.by;
        img0 = ig * P.imgs + (P.layer_imgs ? grp * P.layer_imgs : 0);   // grouped conv: group = layer
    }
}

// 3xTF32 converter warps per CTA: the A block's conversion cost does not shrink
// with BN while the MMA work does, so narrow tiles get twice the converters.
// 3xF16C: 8 always (two threads per A row, see convert_f16_rows; the f16 MMAs
// take half the 3xTF32 time per channel, so the split must keep up at any BN)
template <int BN, bool TSA = false, int KIND = KIND_3XTF32>
constexpr int pair_conv_warps() { return KIND == KIND_3XF16C ? 8 : ((BN >= 256 || TSA) ? 4 : 8); }

template <int BN, int KIND, bool TSA = false>
constexpr int pair_threads() {
    return (KIND == KIND_3XTF32 || KIND == KIND_3XF16C) ? 256 + 32 * pair_conv_warps<BN, TSA, KIND>() : 256;
}

// 3xF16C split of staged activation rows, in place: rows [0, nrows) of two SW128
// fp32 tiles b0 (channels 0..31) and b1 (channels 32..63) become the fp16 hi
// plane (b0, 64 channels per 128-B row) and lo plane (b1) of the same rows:
// hi = rn(v * 2^e), lo = rn(v * 2^e - hi), e the tensor's exponent (f16_row_exp).
// Two threads per row (thread h reads tile b_h: the pair sits in one warp, so
// a __syncwarp between the read and write phases makes the in-place rewrite
// safe); per 8-thread LDS/STS phase 4 rows x 2 halves hit 8 distinct 16-B
// chunks (the h = 1 thread walks its chunks rotated by half a row).
// fp32 pair -> scaled fp16 hi / lo pairs with packed fp32x2 arithmetic (FMUL2 / FADD2):
// 7 instructions per 2 values instead of 10
__device__ __forceinline__ void split_f16x2(float a, float b, float2 sc2, uint32_t &hi, uint32_t &lo) {
    const float2 s2 = __fmul2_rn(make_float2(a, b), sc2);
    const __half2 h = __floats2half2_rn(s2.x, s2.y);
    const float2 hf = __half22float2(h);
    const float2 d = __fadd2_rn(s2, make_float2(-hf.x, -hf.y));
    const __half2 l = __floats2half2_rn(d.x, d.y);
    hi = *reinterpret_cast<const uint32_t *>(&h);
    lo = *reinterpret_cast<const uint32_t *>(&l);
}

template <int NT>
__device__ __forceinline__ void convert_f16_rows(uint32_t b0, uint32_t b1, int nrows, int ct, float sc,
                                                 float &amax) {
    const int h = ct & 1;
    for (int base = 0; base < nrows; base += NT / 2) {
        const int m = base + (ct >> 1);
        const bool act = m < nrows;
        const int sw = m & 7;
        const uint32_t src = (h ? b1 : b0) + (uint32_t)m * 128;
        float4 v[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int ip = (i + 2 * h) & 3;
            if (act) {
                v[2 * i] = lds128(src + (uint32_t)(((2 * ip) ^ sw) << 4));
                v[2 * i + 1] = lds128(src + (uint32_t)(((2 * ip + 1) ^ sw) << 4));
            }
        }
        __syncwarp();
        if (act) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int ip = (i + 2 * h) & 3;
                const int q = 4 * h + ip;   // fp16 chunk: channels 8q .. 8q + 7
                amax = fmaxf(amax, fmaxf(fmaxf(fmaxf(fabsf(v[2 * i].x), fabsf(v[2 * i].y)),
                                               fmaxf(fabsf(v[2 * i].z), fabsf(v[2 * i].w))),
                                         fmaxf(fmaxf(fabsf(v[2 * i + 1].x), fabsf(v[2 * i + 1].y)),
                                               fmaxf(fabsf(v[2 * i + 1].z), fabsf(v[2 * i + 1].w)))));
                uint32_t hw[4], lw[4];
                const float2 sc2 = make_float2(sc, sc);
                split_f16x2(v[2 * i].x, v[2 * i].y, sc2, hw[0], lw[0]);
                split_f16x2(v[2 * i].z, v[2 * i].w, sc2, hw[1], lw[1]);
                split_f16x2(v[2 * i + 1].x, v[2 * i + 1].y, sc2, hw[2], lw[2]);
                split_f16x2(v[2 * i + 1].z, v[2 * i + 1].w, sc2, hw[3], lw[3]);
                const uint32_t off = (uint32_t)m * 128 + (uint32_t)((q ^ sw) << 4);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(b0 + off), "r"(hw[0]),
                             "r"(hw[1]), "r"(hw[2]), "r"(hw[3])
                             : "memory");
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(b1 + off), "r"(lw[0]),
                             "r"(lw[1]), "r"(lw[2]), "r"(lw[3])
                             : "memory");
            }
        }
        __syncwarp();
    }
}

// ---- 3xF16C speculative activation scale --------------------------------------------
// The speculative launch scales x by 2^e, e = f16_row_exp(spec), spec = the max |x| the
// previous call on this workspace observed (state[0], valid iff state[1] = state[0] ^
// kScaleTag: a fresh or foreign workspace means no speculation), records spec in state[2]
// and stores each CTA's observed max |x| in state[4 + cta] -- plain stores, nothing to
// reset between calls.  The speculation held iff the observed max, scaled, neither
// overflows fp16 nor sits more than 2 binades below the exact scale's [2^14, 2^15) (so
// the split keeps its 22 significant bits for everything within 2^-16 of the max).
// Otherwise the fallback launch redoes the conv with e = f16_row_exp(observed max) -- the
// exact per-tensor scale; either way it leaves the observed max as the next speculation.
constexpr int kScaleTag = 0x5ca1ab1e;
__device__ __forceinline__ bool f16c_spec_ok(int spec, int obs) {
    if (spec <= 0 || obs <= 0) return false;
    const float top = __int_as_float(obs) * pow2f(f16_row_exp(__int_as_float(spec)));
    return top < 65504.f && top >= 4096.f;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// the max |x| a speculative launch scales with (0: none)
__device__ __forceinline__ int f16c_spec_value(const int *state) {
    const int s0 = ld_relaxed_gpu(state), s1 = ld_relaxed_gpu(state + 1);
    return (s0 ^ kScaleTag) == s1 ? s0 : 0;
}
// speculative launch: the converter warps' max |x| -> this CTA's slot
__device__ __forceinline__ void f16c_publish_max(const PairParams &PP, float amax, int *cta_max, int nconv) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    if (PP.fallback) return;
    if ((threadIdx.x & 31) == 0) atomicMax(cta_max, __float_as_int(amax));
    asm volatile("bar.sync 2, %0;\n" ::"r"(32 * nconv) : "memory");   // the converter warps only
    if (threadIdx.x == 256) PP.scale_state[4 + blockIdx.x] = *cta_max;
}

// A operand from tensor memory (TSA): tcgen05.mma [d], [a_tmem], b_desc -- the
// tensor core then reads only B from shared memory
__device__ __forceinline__ void umma_pair_ts_tf32(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                                  uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

// 3xF16C with A in TMEM: tcgen05.mma kind::f16 [d], [a_tmem], b_desc
__device__ __forceinline__ void umma_pair_ts_f16(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                                 uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
        "%30, %31, %32};\n" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
        "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// lo = v - tf32(v) (rounded to TF32) of n16 16-byte vectors by NT threads,
// explicit shared-window addressing; loads batched so their latencies overlap
template <int NT>
__device__ __forceinline__ void convert_lo_range(uint32_t hi, uint32_t lo, int n16, int ct) {
    int i = ct;
    for (; i + 3 * NT < n16; i += 4 * NT) {
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = lds128(hi + (uint32_t)(i + j * NT) * 16);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float4 l;
            l.x = v[j].x - __uint_as_float(__float_as_uint(v[j].x) & 0xffffe000u);
            l.y = v[j].y - __uint_as_float(__float_as_uint(v[j].y) & 0xffffe000u);
            l.z = v[j].z - __uint_as_float(__float_as_uint(v[j].z) & 0xffffe000u);
            l.w = v[j].w - __uint_as_float(__float_as_uint(v[j].w) & 0xffffe000u);
            sts128_tf32(lo + (uint32_t)(i + j * NT) * 16, l);
        }
    }
    for (; i < n16; i += NT) {
        const float4 v = lds128(hi + (uint32_t)i * 16);
        float4 l;
        l.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
        l.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
        l.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
        l.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
        sts128_tf32(lo + (uint32_t)i * 16, l);
    }
}

// K-major SW128 descriptor of an operand starting at any 128-B row of a
// 1 KB-aligned TMA-written tile.  The tensor core applies the 128-B swizzle on
// absolute smem address bits (as TMA does when writing), so the plain
// descriptor of the row address is correct and the base-offset field must stay
// 0 -- measured: scripts/dev/umma_shift_selftest.cu (base_offset = 0 exact for
// every row shift; base_offset = (addr >> 7) & 7 wrong unless the shift is a
// multiple of 8 rows).
__device__ __forceinline__ uint64_t umma_desc_sw128_row(uint32_t addr) { return umma_desc_sw128(addr); }

// FOLD (halo tiles with S * K <= 256, K = z): the S horizontal taps of a kernel
// row share one MMA of N = S * K -- B = [W(r,0); W(r,1); W(r,2)] rows, A = the
// footprint view of row r -- and the epilogue adds the S column groups shifted
// by s rows (warp shuffles: the s-shift stays inside a footprint row).  R MMAs
// of N = 192 per channel block instead of R*S of N = 64 (48 cycles each on the
// tensor core: 67 % of its rate at N = 64).
// HALO + TSA (3xF16C): the converter warps apply the tap shift themselves -- lane m
// of tap (r, s) reads footprint row m + r * fpr + s from the fp32 footprint slot,
// splits it and tcgen05.st's the hi / lo pair into an A slot of TMEM -- so the
// footprint crosses L2 once per channel block (halo) while the tensor core reads
// only the filter from shared memory (TSA).  RESB (halo TSA fold, one n-block): the
// CTA's whole filter slice is staged ONCE (the ring holds kblocks filter slots) and
// only footprints stream per work item; a grouped launch reloads it when the CTA's
// items move on to the next layer, after the MMAs on the old slice have completed.
template <int BN, int KIND, bool HALO, bool TSA, bool FOLD = false, bool RESB = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair_threads<BN, KIND, TSA>(), 1)
    igemm_pair_kernel(const __grid_constant__ PairParams PP, const __grid_constant__ CUtensorMap tm_x,
                      const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_y) {
    // KIND_3XF16C (direct conv): the activation k-block (64 channels) arrives as two
    // fp32 TMA boxes (channels 0..31 where the hi operand goes, 32..63 where the lo
    // operand goes) and the converter warps rewrite them in place into the fp16
    // hi / lo planes; the filter's fp16 hi / lo planes come by TMA (lo plane R*S
    // taps further on).  Same stage layout, barriers and 3-MMA issue as 3xTF32.
    constexpr bool F16C = KIND == KIND_3XF16C;
    constexpr bool SPLIT = KIND == KIND_3XTF32 || F16C;   // converter warps
    // KIND_3XF16 (batched Winograd GEMMs): operands pre-split by the transforms into
    // scaled fp16 hi / lo planes (the lo plane xi-count images / taps further on);
    // TMA brings all four, the MMA issues hi*lo + lo*hi + hi*hi like 3xTF32 -- no
    // converters -- and the epilogue undoes the power-of-two row / column scales
    constexpr bool F16X3 = KIND == KIND_3XF16;
    static_assert(!F16X3 || (!HALO && !TSA && !FOLD), "3xF16: plain pair tiles");
    static_assert(!(TSA && HALO) || F16C, "halo tiles with A in TMEM: 3xF16C only");
    static_assert(!RESB || (TSA && HALO && FOLD), "resident filter: fold halo tiles with A in TMEM");
    constexpr int HB = BN / 2;                        // filter rows staged per CTA
    constexpr int A_BYTES = 128 * 128;
    constexpr int B_BYTES = HB * 128;
    constexpr int MULT = (SPLIT || F16X3) ? 2 : 1;    // hi (raw) + lo copies
    constexpr int CB = (KIND == KIND_BF16 || F16X3 || F16C) ? 64 : 32;   // channels per k-block
    // TSA (3xTF32, BN <= 128): A_hi / A_lo live in TMEM columns after the two
    // accumulators, NTA k-block slots of 64 columns (32 hi + 32 lo)
    static_assert(!TSA || (SPLIT && (!HALO || F16C) && (BN <= 128 || F16C)), "TSA: 3xTF32 / 3xF16C");
    // accumulator buffers: 2 (the epilogue drains one while the MMAs fill the other),
    // 1 for 3xF16C TSA at BN = 256 (its 256 columns + 4 A slots fill the 512)
    // (FOLD's N = 192 keeps two: 384 columns + 2 A slots)
    constexpr int NACC = (TSA && BN > 128 && !FOLD) ? 1 : 2;
    // (power-of-two allocation; FOLD's 2 x 192 columns take 512)
    constexpr uint32_t TMEM_COLS = (TSA || 2 * BN > 256) ? 512 : (2 * BN < 32 ? 32 : 2 * BN);
    constexpr uint32_t A_COL0 = NACC * BN;
    // TSA A slots of 64 columns: 3xTF32 32 hi + 32 lo fp32 channels; 3xF16C the same 64
    // channels as fp16 pairs (32 hi + 32 lo columns)
    constexpr int NTA = TSA ? (512 - NACC * BN) / 64 : 1;
    constexpr int NCW = pair_conv_warps<BN, TSA, KIND>();   // converter warps (3xTF32 / 3xF16C)
    const IgemmParams &P = PP.g;
    // stage layout: non-halo [A | B]; TSA [A | B | B_lo]; halo: A footprint slots,
    // then B stages [B | B_lo].  Non-halo 3xTF32 (LOSLOT): the lo copies live in
    // NL = 2 slots after the TMA ring, decoupled from it, so the ring holds more
    // k-blocks in flight (N = 256: 4 TMA stages instead of 3 whole [hi | lo]
    // stages) -- the MMA issuer of the short-K Winograd GEMMs was waiting on
    // converters that were waiting on TMA data.
    // (N = 256 only: measured 1-2 % faster there, 7-8 % slower at N = 128, where
    // two lo slots let the converters run only two k-blocks ahead of the MMAs)
    constexpr bool LOSLOT = KIND == KIND_3XTF32 && !HALO && !TSA && BN == 256;
    constexpr int NL = 2;
    constexpr int LO_SLOT = A_BYTES + B_BYTES;
    // ARING (3xF16C, A in TMEM, no halo): the fp32 activation boxes get their own ring
    // of NA slots [A0 | A1], released by the converters as soon as the rows are in TMEM;
    // the filter planes stay in the stage ring [B_hi | B_lo] until the MMAs complete --
    // an A box then lives ~TMA latency + split instead of until its MMAs retire
    constexpr bool ARING = TSA && F16C && !HALO;
    const int STAGE = (HALO || ARING) ? B_BYTES * MULT
                           : ((TSA && !F16C) ? A_BYTES + 2 * B_BYTES : (A_BYTES + B_BYTES) * (LOSLOT ? 1 : MULT));
    const int ASLOT = HALO ? PP.a_slot * MULT : (ARING ? 2 * A_BYTES : 0);
    const int NA = (HALO || ARING) ? PP.na : 0;

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int NS = P.stages;
    uint8_t *aring = smem;                            // halo footprint slots
    uint8_t *bring = smem + NA * ASLOT;               // stages
    uint8_t *loring = bring + NS * STAGE;             // LOSLOT: lo copies
    uint8_t *ring_end = loring + (LOSLOT ? NL * LO_SLOT : 0);
    uint64_t *full = reinterpret_cast<uint64_t *>(ring_end);
    uint64_t *empty = full + NS;
    uint64_t *conv = empty + NS;
    uint64_t *tfull = conv + NS;
    uint64_t *tempty = tfull + 2;
    uint64_t *afull = tempty + 2;                     // halo: footprint slot barriers (ARING: A slots)
    uint64_t *aempty = afull + 6;
    uint64_t *aconv = aempty + 6;
    uint64_t *tconv = aconv + 6;                      // TSA: A slot in TMEM converted
    uint64_t *tfree = tconv + 6;                      // TSA: A slot in TMEM consumed
    uint64_t *lofree = tfree + 6;                     // LOSLOT: lo slot consumed by the MMAs
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(lofree + NL);
    int &f16c_scale_max = reinterpret_cast<int *>(tmem_slot)[1];   // 3xF16C: the max |x| scaled with
    int &f16c_cta_max = reinterpret_cast<int *>(tmem_slot)[2];     // 3xF16C: this CTA's observed max
    // 3xF16C: the max |x| this launch scales with (speculative: the previous call's
    // observation; fallback: this call's), and the per-CTA max its converters reduce into
    if constexpr (F16C) {
        if (threadIdx.x == 0) f16c_cta_max = 0;
        if (PP.fallback) {   // the checking launch: reduce the speculative launch's per-CTA maxima
            pdl_wait();
            int obs = threadIdx.x < PP.spec_ctas ? ld_relaxed_gpu(PP.scale_state + 4 + threadIdx.x) : 0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) obs = max(obs, __shfl_xor_sync(0xffffffffu, obs, off));
            if (threadIdx.x == 0) f16c_scale_max = 0;
            __syncthreads();
            if ((threadIdx.x & 31) == 0 && obs > 0) atomicMax(&f16c_scale_max, obs);
            __syncthreads();
            if (threadIdx.x == 0) {
                const int o = f16c_scale_max;
                const int spec = ld_relaxed_gpu(PP.scale_state + 2);
                if (blockIdx.x == 0) {   // the next call speculates with this call's max
                    PP.scale_state[0] = o;
                    PP.scale_state[1] = o ^ kScaleTag;
                }
                if (f16c_spec_ok(spec, o)) f16c_scale_max = -1;   // the speculation held
            }
        }
        __syncthreads();
        if (PP.fallback && f16c_scale_max < 0) return;   // every thread of the pair: nothing to redo
    }

    const int tid = threadIdx.x;
    // warp index through a shuffle: the compiler then knows it is warp-uniform
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int cluster_id = blockIdx.x >> 1;
    const int nclusters = gridDim.x >> 1;
    const uint64_t map_x = reinterpret_cast<uint64_t>(&tm_x);
    const uint64_t map_w = reinterpret_cast<uint64_t>(&tm_w);
    const uint64_t map_y = reinterpret_cast<uint64_t>(&tm_y);

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
            mbar_init(conv + s, 2 * NCW);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 8);
        }
        for (int a = 0; a < 6; ++a) {
            mbar_init(aconv + a, 2 * NCW);
            mbar_init(afull + a, 1);
            mbar_init(aempty + a, TSA ? NCW : 1);   // A in TMEM: the converters read the slot
        }
        for (int l = 0; l < NL && LOSLOT; ++l) mbar_init(lofree + l, 1);
        for (int a = 0; a < NTA && TSA; ++a) {
            mbar_init(tconv + a, 2 * NCW);
            mbar_init(tfree + a, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_x));
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(map_w));
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    pdl_wait();   // the prologue above overlapped the previous kernel's tail
    if constexpr (F16C) {   // the speculation (state written by the previous call's fallback launch)
        if (!PP.fallback) {
            if (tid == 0) {
                f16c_scale_max = f16c_spec_value(PP.scale_state);
                if (blockIdx.x == 0) PP.scale_state[2] = f16c_scale_max;
            }
            __syncthreads();
        }
    }
#ifdef CONVIO_TRACE   // per-CTA start / end (globaltimer ns): rows 16 / 17
    if (PP.trace && tid == 0 && blockIdx.x < 1024) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        PP.trace[16 * 1024 + blockIdx.x] = g;
    }
#endif

    // work item -> (group, pair, n-block); n fastest
    // tail split-K (non-halo): tile items [0, tail_start) keep their whole K range; each
    // later tile item is split into P.splits K ranges (work items tail_start + j, j =
    // tile * splits + split), so the last round of the persistent grid is filled with
    // partial tiles that the epilogue reduce-adds into the zeroed output
    auto krange = [&](int item, int &kb_lo, int &kb_hi) {
        if constexpr (HALO) {   // halo tiles never split (compile-time: no cost)
            kb_lo = 0;
            kb_hi = P.kblocks;
            return -1;
        }
        if (item < PP.tail_start) {
            kb_lo = 0;
            kb_hi = P.kblocks;
            return -1;   // a whole tile
        }
        const int spl = (item - PP.tail_start) % P.splits;
        kb_lo = (int)(((int64_t)P.kblocks * spl) / P.splits);
        kb_hi = (int)(((int64_t)P.kblocks * (spl + 1)) / P.splits);
        return spl;
    };
    auto decode = [&](int item, int &grp, int &pair, int &nb) {
        if constexpr (!HALO) {
            if (item >= PP.tail_start) item = PP.tail_start + (item - PP.tail_start) / P.splits;
        }
        nb = item % PP.nblocks;
        const int rest = item / PP.nblocks;
        pair = rest % PP.pairs_per_group;
        grp = rest / PP.pairs_per_group;
    };
    const int taps = FOLD ? P.ks : P.ks * P.ks;       // k-groups per channel block
    constexpr int KOUT = FOLD ? BN / 3 : BN;          // output channels per work item
    static_assert(!FOLD || (HALO && BN % 3 == 0), "FOLD: halo tiles, N = 3 * K");

    if (warp == 0) {
        if (lane == 0) {
            // ---- TMA producer (both CTAs) -------------------------------------------
            const uint32_t a_rows_bytes = (uint32_t)(P.bx * P.by * P.imgs * 128);
            // 3xF16C: two activation boxes and two filter planes per k-block
            const uint32_t cta_bytes = ((HALO || ARING) ? (uint32_t)B_BYTES : a_rows_bytes + B_BYTES) * (F16C ? 2u : 1u);
            const int lo_tap = P.ks * P.ks;                   // 3xF16C: filter lo plane offset (taps)
            int s = 0, sa = 0;
            uint32_t ph = 0, pha = 0;
            int it = 0, ita = 0;
            // RESB: the CTA's filter slice stays resident (slot cb * taps + tap, halo order),
            // loaded once -- per layer when grouped: before a reload the producer waits for
            // the MMAs on the old slice (the issuer commits `empty`, unused by the ring here)
            int resident = -1;
            uint32_t rph = 0;
            for (int item = cluster_id; item < PP.items; item += nclusters) {
                int grp, pair, nb;
                decode(item, grp, pair, nb);
                if constexpr (RESB) {
                    const int layer = P.layer_imgs ? grp : 0;
                    if (layer != resident) {
                        if (resident >= 0) {
                            mbar_wait(empty, rph);
                            rph ^= 1;
                        }
                        mbar_arrive_expect_tx(full, (uint32_t)(P.kblocks * STAGE));
                        for (int cb = 0, slot = 0; cb < P.cblocks; ++cb)
                            for (int tap = 0; tap < taps; ++tap, ++slot) {
                                uint8_t *b = bring + slot * STAGE;
                                const int frow = tap * P.ks * P.k + (int)rank * HB;
                                if (P.layer_imgs) {
                                    tma_load_3d(b, map_w, cb * CB, frow, layer, full);
                                    tma_load_3d(b + B_BYTES, map_w, cb * CB, frow + lo_tap * P.k, layer, full);
                                } else {
                                    tma_load_2d(b, map_w, cb * CB, frow, full);
                                    tma_load_2d(b + B_BYTES, map_w, cb * CB, frow + lo_tap * P.k, full);
                                }
                            }
                        resident = layer;
                    }
                }
                int ox0, oy0, img0;
                pair_block_origin(P, grp, pair * 2 + (int)rank, ox0, oy0, img0);
                const int n0 = nb * BN + (int)rank * HB;
                int kb_lo, kb_hi;
                krange(item, kb_lo, kb_hi);
                int tap = HALO ? 0 : kb_lo / P.cblocks, cb = HALO ? 0 : kb_lo - tap * P.cblocks;
                for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
                    // FOLD: the filter rows of kernel row `tap` (S taps x K channels) of
                    // the packed [R*S*K][C] view; this CTA stages its HB of them
                    const int frow = tap * P.ks * P.k + (int)rank * HB;
                    if (HALO && tap == 0) {
                        // the block's input footprint for channel block cb, once
                        if (ita >= NA) mbar_wait(aempty + sa, pha ^ 1);
                        uint8_t *fa = aring + sa * ASLOT;
                        const int xc = ox0 * P.stride - P.pad, yc = oy0 * P.stride - P.pad;
                        if constexpr (F16C) {   // channels 0..31 -> hi slot, 32..63 -> lo slot
                            mbar_arrive_expect_tx(afull + sa, 2u * (uint32_t)PP.fp_bytes);
                            tma_load_4d(fa, map_x, cb * CB, xc, yc, img0, afull + sa);
                            tma_load_4d(fa + PP.a_slot, map_x, cb * CB + 32, xc, yc, img0, afull + sa);
                        } else if constexpr (SPLIT) {
                            mbar_arrive_expect_tx(afull + sa, (uint32_t)PP.fp_bytes);
                            tma_load_4d(fa, map_x, cb * CB, xc, yc, img0, afull + sa);
                        } else {
                            if (leader) mbar_arrive_expect_tx(afull + sa, 2u * (uint32_t)PP.fp_bytes);
                            tma_load_4d_pair(fa, map_x, cb * CB, xc, yc, img0, afull + sa);
                        }
                        ++ita;
                        if (++sa == NA) {
                            sa = 0;
                            pha ^= 1;
                        }
                    }
                    if constexpr (!RESB) {
                    if (!ARING && it >= NS) mbar_wait(empty + s, ph ^ 1);
                    PAIR_TRACE(0, it);
                    const int r = tap / P.ks, sx = tap - r * P.ks;
                    uint8_t *a = bring + s * STAGE;
                    uint8_t *b = HALO ? a : a + A_BYTES;
                    const int xc = ox0 * P.stride + sx - P.pad, yc = oy0 * P.stride + r - P.pad;
                    const int wc = P.batched ? img0 : tap;
                    if constexpr (F16C) {    // own barrier, as 3xTF32; [A0 | B_hi | A1 | B_lo]
                        if constexpr (ARING) {   // A slot [A0 | A1]; stage [B_hi | B_lo]
                            if (ita >= NA) mbar_wait(aempty + sa, pha ^ 1);
                            uint8_t *as = aring + sa * ASLOT;
                            mbar_arrive_expect_tx(afull + sa, 2u * a_rows_bytes);
                            tma_load_4d(as, map_x, cb * CB, xc, yc, img0, afull + sa);
                            tma_load_4d(as + A_BYTES, map_x, cb * CB + 32, xc, yc, img0, afull + sa);
                            ++ita;
                            if (++sa == NA) {
                                sa = 0;
                                pha ^= 1;
                            }
                        } else {
                        mbar_arrive_expect_tx(full + s, cta_bytes);
                        uint8_t *blo = (HALO || ARING) ? b + B_BYTES : b + A_BYTES + B_BYTES;
                        if (!HALO && !ARING) {
                            tma_load_4d(a, map_x, cb * CB, xc, yc, img0, full + s);
                            tma_load_4d(a + A_BYTES + B_BYTES, map_x, cb * CB + 32, xc, yc, img0, full + s);
                        }
                        if (P.layer_imgs) {   // grouped: the item's layer (its group) -- both CTAs
                            const int layer = grp;   // of a pair use ITS filter, spare blocks included
                            if (FOLD) {
                                tma_load_3d(b, map_w, cb * CB, frow, layer, full + s);
                                tma_load_3d(blo, map_w, cb * CB, frow + lo_tap * P.k, layer, full + s);
                            } else {
                                tma_load_4d(b, map_w, cb * CB, n0, wc, layer, full + s);
                                tma_load_4d(blo, map_w, cb * CB, n0, wc + lo_tap, layer, full + s);
                            }
                        } else if (FOLD) {
                            tma_load_2d(b, map_w, cb * CB, frow, full + s);
                            tma_load_2d(blo, map_w, cb * CB, frow + lo_tap * P.k, full + s);
                        } else {
                            tma_load_3d(b, map_w, cb * CB, n0, wc, full + s);
                            tma_load_3d(blo, map_w, cb * CB, n0, wc + lo_tap, full + s);
                        }
                        }   // !ARING (its filter planes come from warp 2)
                    } else if constexpr (SPLIT) {   // own barrier: the converters need a local signal
                        mbar_arrive_expect_tx(full + s, cta_bytes);
                        if (!HALO) tma_load_4d(a, map_x, cb * CB, xc, yc, img0, full + s);
                        if (FOLD) tma_load_2d(b, map_w, cb * CB, frow, full + s);
                        else tma_load_3d(b, map_w, cb * CB, n0, wc, full + s);
                    } else {                 // both CTAs' bytes complete on the leader's barrier
                        if (leader) mbar_arrive_expect_tx(full + s, 2 * MULT * cta_bytes);
                        if (!HALO) tma_load_4d_pair(a, map_x, cb * CB, xc, yc, img0, full + s);
                        if (FOLD) tma_load_2d_pair(b, map_w, cb * CB, frow, full + s);
                        else tma_load_3d_pair(b, map_w, cb * CB, n0, wc, full + s);
                        if constexpr (F16X3) {   // lo planes: P.n (= xi) images / taps further on
                            tma_load_4d_pair(a + A_BYTES + B_BYTES, map_x, cb * CB, xc, yc, img0 + P.n, full + s);
                            tma_load_3d_pair(b + A_BYTES + B_BYTES, map_w, cb * CB, n0, wc + P.n, full + s);
                        }
                    }
                    if (!ARING && ++s == NS) {
                        s = 0;
                        ph ^= 1;
                    }
                    }   // !RESB
                    // halo: channel block outer, taps inner (footprint reused by all taps)
                    if (HALO) {
                        if (++tap == taps) {
                            tap = 0;
                            ++cb;
                        }
                    } else if (++cb == P.cblocks) {
                        cb = 0;
                        ++tap;
                    }
                }
            }
        }
    } else if (ARING && warp == 2) {
        if (lane == 0) {
            // ---- ARING filter producer: the [B_hi | B_lo] stages run on their own ring, so a
            // stage still held by in-flight MMAs never blocks the activation loads of warp 0 ----
            const int lo_tap = P.ks * P.ks;
            int s = 0, it = 0;
            uint32_t ph = 0;
            for (int item = cluster_id; item < PP.items; item += nclusters) {
                int grp, pair, nb;
                decode(item, grp, pair, nb);
                const int n0 = nb * BN + (int)rank * HB;
                int kb_lo, kb_hi;
                krange(item, kb_lo, kb_hi);
                int tap = kb_lo / P.cblocks, cb = kb_lo - tap * P.cblocks;
                for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
                    if (it >= NS) mbar_wait(empty + s, ph ^ 1);
                    uint8_t *b = bring + s * STAGE;
                    // both CTAs' planes complete on the LEADER's barrier: the MMA issuer waits on
                    // it directly, the converters never wait for filter data
                    if (leader) mbar_arrive_expect_tx(full + s, 4u * (uint32_t)B_BYTES);
                    if (P.layer_imgs) {   // grouped: the item's layer (its group)
                        const int layer = grp;
                        tma_load_4d_pair(b, map_w, cb * CB, n0, tap, layer, full + s);
                        tma_load_4d_pair(b + B_BYTES, map_w, cb * CB, n0, tap + lo_tap, layer, full + s);
                    } else {
                        tma_load_3d_pair(b, map_w, cb * CB, n0, tap, full + s);
                        tma_load_3d_pair(b + B_BYTES, map_w, cb * CB, n0, tap + lo_tap, full + s);
                    }
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
        }
    } else if (warp == 1) {
        if (leader) {
            // ---- MMA issuer (leader CTA): the whole warp runs the loop, so descriptors and
            // counters stay warp-uniform (uniform registers); one elected lane issues.  A
            // single-lane issuer made the compiler wrap every tcgen05.mma in an ELECT +
            // 4 x R2UR.BROADCAST loop, ~90 issue cycles per MMA: slower than an N = 128 MMA
            // (64 cycles), so the tensor core starved ----------------------------------
            constexpr uint32_t idesc = idesc_m256<BN, KIND>();
            int s = 0, sa = 0, ta = 0, l = 0, kbc = 0;
            uint32_t ph = 0, pha = 0, pht = 0;
            int t = 0;
            for (int item = cluster_id; item < PP.items; item += nclusters, ++t) {
                const int acc = NACC == 2 ? (t & 1) : 0;
                if (t >= NACC) mbar_wait_cluster(tempty + acc, ((t / NACC) - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                int tap = 0;
                uint32_t fa = 0;
                int kb_lo, kb_hi;
                krange(item, kb_lo, kb_hi);
                int cur_layer = 0, next_layer = -1;   // RESB grouped: the slice's layer changes
                if (RESB && P.layer_imgs) {
                    int g_, p_, n_;
                    decode(item, g_, p_, n_);
                    cur_layer = g_;
                    if (item + nclusters < PP.items) {
                        decode(item + nclusters, g_, p_, n_);
                        next_layer = g_;
                    }
                }
                for (int kb = kb_lo; kb < kb_hi; ++kb) {
                    if constexpr (TSA) {
                        mbar_wait_cluster(tconv + ta, pht);
                        if constexpr (ARING) mbar_wait(full + s, ph);   // both CTAs' filter planes
                        PAIR_TRACE(3, kbc);
                        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                        // 3xTF32 stage [A | B | B_lo]; 3xF16C [A0 | B_hi | A1 | B_lo]; halo [B_hi | B_lo]
                        // (RESB: filter slot kb of the resident slice)
                        const uint32_t b = smem_u32(bring + (RESB ? kb : s) * STAGE) + ((HALO || ARING) ? 0 : A_BYTES);
                        const uint64_t bd = umma_desc_sw128(b),
                                       bdl = umma_desc_sw128(b + ((F16C && !HALO && !ARING) ? A_BYTES + B_BYTES : B_BYTES));
                        const uint32_t ahi = tmem + A_COL0 + (uint32_t)(ta * 64);
                        const bool first = kb == kb_lo;
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint64_t o = (uint64_t)(kk * 2);
                                const uint32_t ak = ahi + (uint32_t)(kk * 8);
#ifdef CONVIO_ABL_1MMA   // ablation (timing only, wrong numerics): hi*hi alone
                                umma_pair_ts_f16(d, ak, bd + o, idesc, !(first && kk == 0));
                                continue;
#endif
                                if constexpr (F16C) {
                                    umma_pair_ts_f16(d, ak, bdl + o, idesc, !(first && kk == 0));
                                    umma_pair_ts_f16(d, ak + 32, bd + o, idesc, 1);
                                    umma_pair_ts_f16(d, ak, bd + o, idesc, 1);
                                } else {
                                    umma_pair_ts_tf32(d, ak, bdl + o, idesc, !(first && kk == 0));
                                    umma_pair_ts_tf32(d, ak + 32, bd + o, idesc, 1);
                                    umma_pair_ts_tf32(d, ak, bd + o, idesc, 1);
                                }
                            }
                            if constexpr (!RESB) umma_commit_pair(empty + s);
                            else if (kb + 1 == kb_hi && next_layer >= 0 && next_layer != cur_layer)
                                umma_commit_pair(empty);   // the resident slice may be reloaded
                            umma_commit_pair(tfree + ta);
                        }
                        __syncwarp();
                        PAIR_TRACE(4, kbc);
                        ++kbc;
                        if (++ta == NTA) {
                            ta = 0;
                            pht ^= 1;
                        }
                        if (!RESB && ++s == NS) {
                            s = 0;
                            ph ^= 1;
                        }
                        continue;
                    }
                    if (HALO && tap == 0) {
                        if constexpr (SPLIT) mbar_wait_cluster(aconv + sa, pha);
                        else mbar_wait(afull + sa, pha);
                        fa = smem_u32(aring + sa * ASLOT);
                    }
                    if constexpr (SPLIT) mbar_wait_cluster(conv + s, ph);
                    else mbar_wait(full + s, ph);   // F16X3: all four planes by TMA
                    PAIR_TRACE(3, kbc);
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    const uint32_t st = smem_u32(bring + s * STAGE);
                    uint32_t a, b;
                    if (HALO) {
                        const int r = FOLD ? tap : tap / P.ks, sx = FOLD ? 0 : tap - r * P.ks;
                        a = fa + (uint32_t)((r * PP.fpr + sx) * 128);
                        b = st;
                    } else {
                        a = st;
                        b = st + A_BYTES;
                    }
                    const uint64_t ad = HALO ? umma_desc_sw128_row(a) : umma_desc_sw128(a);
                    const uint64_t bd = umma_desc_sw128(b);
                    const bool first = kb == kb_lo;
                    const uint32_t lo = smem_u32(loring + l * LO_SLOT);
                    const uint32_t alo = HALO ? a + (uint32_t)PP.a_slot : (LOSLOT ? lo : a + A_BYTES + B_BYTES);
                    const uint32_t blo = HALO ? b + (uint32_t)B_BYTES : (LOSLOT ? lo + A_BYTES : b + A_BYTES + B_BYTES);
                    const uint64_t adl = HALO ? umma_desc_sw128_row(alo) : umma_desc_sw128(alo);
                    const uint64_t bdl = umma_desc_sw128(blo);
                    if (elect_one()) {
#ifdef CONVIO_ABL_1MMA   // ablation (timing only, wrong numerics): hi*hi alone
                        if constexpr (F16C) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                umma_pair<KIND>(d, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc,
                                                !(first && kk == 0));
                        } else
#endif
                        if constexpr (SPLIT || F16X3) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint64_t o = (uint64_t)(kk * 2);
                                umma_pair<KIND>(d, ad + o, bdl + o, idesc, !(first && kk == 0));
                                umma_pair<KIND>(d, adl + o, bd + o, idesc, 1);
                                umma_pair<KIND>(d, ad + o, bd + o, idesc, 1);
                            }
                        } else {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                umma_pair<KIND>(d, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc,
                                                !(first && kk == 0));
                        }
                        umma_commit_pair(empty + s);
                        if constexpr (LOSLOT) umma_commit_pair(lofree + l);   // lo slot consumed
                        if (HALO && tap + 1 == taps)
                            umma_commit_pair(aempty + sa);   // footprint consumed by all taps
                    }
                    __syncwarp();
                    PAIR_TRACE(4, kbc);
                    ++kbc;
                    if constexpr (LOSLOT) {
                        if (++l == NL) l = 0;
                    }
                    if (HALO && ++tap == taps) {
                        tap = 0;
                        if (++sa == NA) {
                            sa = 0;
                            pha ^= 1;
                        }
                    }
                    if (++s == NS) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (elect_one()) umma_commit_pair(tfull + acc);
                __syncwarp();
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---- epilogue (one K range per item): TMEM -> registers (unscale, bias, ReLU) ->
        // a 128-B-swizzled staging box in shared memory -> ONE TMA store per 32 channels.
        // Each lane owns an accumulator row (no transposes, no per-lane global stores),
        // and the accumulator is released to the MMA issuer as soon as its last
        // columns are in registers ----
        const int q = warp - 4;                       // TMEM lane quadrant
        const int m = q * 32 + lane;                  // pixel row of this CTA's A block
        const uint32_t tempty_leader = mapa_shared(smem_u32(tempty), 0);
        const uint32_t stg = smem_u32(ring_end + 1024);
        // per-channel epilogue constants (not for the batched Winograd GEMMs: their column
        // exponents differ per xi) staged by the 4 epilogue warps -- once, or per layer
        // of a grouped launch when the CTA's items reach the next layer
        const bool cs_smem = !F16X3 && P.k <= kEpiConstK;
        float *ebias = reinterpret_cast<float *>(ring_end + 1024 + pair_epi_bytes(FOLD));
        float *escale = ebias + P.k;
        const int act_exp = F16C ? f16_row_exp(__int_as_float(f16c_scale_max)) : 0;   // one per tensor
        // 3xF16C: one FFMA per output, y = acc * 2^-(e_act + e_k) + b_k, when every channel's
        // exponent sum is a normal power of two (always, but for operands near 2^-60); else
        // the two exact multiplies
        bool fused_scale = false;
        int staged = -1;   // the layer whose constants are in shared memory
        auto stage_consts = [&](int layer) {
            const float *bias = P.bias ? P.bias + (int64_t)layer * P.k : nullptr;
            const int *cexp = F16C ? P.col_exp + (int64_t)layer * P.col_stride : nullptr;
            bool ok = true;
            for (int k = m; k < P.k; k += 128) {
                ebias[k] = bias ? __ldg(bias + k) : 0.f;
                if constexpr (F16C) {
                    const int ek = __ldg(cexp + k), e = act_exp + ek;
                    ok = ok && e >= -126 && e <= 127;
                    escale[k] = pow2f(-ek);
                } else {
                    escale[k] = 1.f;
                }
            }
            uint32_t all;
            asm volatile("{\n.reg .pred p, q;\nsetp.ne.u32 q, %1, 0;\nbar.red.and.pred p, 1, 128, q;\n"
                         "selp.u32 %0, 1, 0, p;\n}\n" : "=r"(all) : "r"((uint32_t)ok) : "memory");
            fused_scale = F16C && all;
            if (fused_scale)   // fold the tensor scale into the column scales
                for (int k = m; k < P.k; k += 128) escale[k] = pow2f(-(act_exp + __ldg(cexp + k)));
            epi_bar();
            staged = layer;
        };
        if (cs_smem) stage_consts(0);
        // staging row = position in the store box [img][y][x] (halo: the x valid columns)
        int srow;
        bool inbox;
        if (HALO && !PP.gather) {
            const int py = m / PP.fpr, px = m - py * PP.fpr;
            srow = py * P.bx + px;
            inbox = px < P.bx;
        } else {
            srow = m;
            inbox = m < P.bx * P.by * P.imgs;
        }
        const bool issuer = q == 0 && lane == 0;
        int nbox = 0;
        int t = 0;
        for (int item = cluster_id; item < PP.items; item += nclusters, ++t) {
            int grp, pair, nb;
            decode(item, grp, pair, nb);
            int kb_lo, kb_hi;
            const int spl = krange(item, kb_lo, kb_hi);   // -1: a whole tile
            const bool with_bias = P.bias != nullptr && spl <= 0;
            const int acc = NACC == 2 ? (t & 1) : 0;
            // the item's geometry (integer divisions) before the wait, not after it
            const int blk = pair * 2 + (int)rank;
            int ox0, oy0, img0;
            pair_block_origin(P, grp, blk, ox0, oy0, img0);
            const int k0 = nb * KOUT;
            const int layer = P.layer_imgs ? grp : 0;   // grouped conv: group = layer
            // (the previous item's last epi_bar: every lane is done with the old constants)
            if (cs_smem && layer != staged) stage_consts(layer);
            float rs = 1.f;   // the row's operand scale (3xF16 families; 1 when folded into escale)
            if constexpr (F16X3) {
                const int per_img = P.bx * P.by;
                const int im = m / per_img, pix = m - im * per_img;
                const int py = pix / P.bx, px = pix - py * P.bx;
                const int img = img0 + im, ox = ox0 + px;
                const bool ok = inbox && img < P.n && oy0 + py < P.p && ox < P.q;
                rs = pow2f(-(ok ? __ldg(P.row_exp + (int64_t)img * P.q + ox) : 0));
            } else if constexpr (F16C) {
                rs = fused_scale ? 1.f : pow2f(-act_exp);
            }
            mbar_wait(tfull + acc, (t / NACC) & 1);
            if (q == 0 && lane == 0) PAIR_TRACE(5, t);
            __syncwarp();
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (q == 0 && lane == 0) EPI_TRACE(18, t);
#pragma unroll 1
            for (int c0 = 0; c0 < KOUT; c0 += 32) {
                float v[32];
                if constexpr (FOLD) {
                    // y[p] = E[p][0:K] + E[p+1][K:2K] + E[p+2][2K:3K]: rows p+1, p+2 are
                    // lanes +1, +2 of this warp (valid columns never cross a footprint row);
                    // the three loads in flight together, one wait
                    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0);
                    uint32_t r0[32], r1[32], r2[32];
                    tmem_ld_x32_nowait(ta, r0);
                    tmem_ld_x32_nowait(ta + (uint32_t)KOUT, r1);
                    tmem_ld_x32_nowait(ta + (uint32_t)(2 * KOUT), r2);
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                    if (c0 == 0 && q == 0 && lane == 0) EPI_TRACE(19, t);
#ifdef CONVIO_ABL_NOSHFL   // ablation (timing only, wrong numerics): no row shift
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        v[j] = __uint_as_float(r0[j]) + __uint_as_float(r1[j]) + __uint_as_float(r2[j]);
#else
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        v[j] = __uint_as_float(r0[j]) +
                               __shfl_down_sync(0xffffffffu, __uint_as_float(r1[j]), 1) +
                               __shfl_down_sync(0xffffffffu, __uint_as_float(r2[j]), 2);
#endif
                } else {
                    tmem_ld_32x32b<32>(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0), v);
                    if (c0 == 0 && q == 0 && lane == 0) EPI_TRACE(19, t);
                }
                if (c0 == 0 && q == 0 && lane == 0) EPI_TRACE(20, t);
                if (c0 + 32 >= KOUT) {   // accumulator fully read: hand it back to the MMA issuer
                    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_leader + (uint32_t)(acc * 8));
                    if (q == 0 && lane == 0) PAIR_TRACE(6, t);
                }
                // unscale (exact powers of two, two multiplies: the exponent sum may pass
                // pow2f's range), bias, ReLU
                const int kc = k0 + c0;
#ifdef CONVIO_ABL_NOUNSCALE   // ablation (timing only, wrong numerics): no unscale / bias
                if (0)
#endif
                if (cs_smem) {
                    // the chunk's 32 channel scales and biases: 16 broadcast LDS.128 from the
                    // shared-memory constants, issued together (explicit shared-space loads:
                    // generic loads of these addresses, one dependent pair per 4 channels,
                    // cost the fold epilogue ~14 % of res2's time)
                    const uint32_t es = smem_u32(escale + kc), eb = smem_u32(ebias + kc);
                    float4 c4v[8], b4v[8];
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        c4v[j4] = lds128(es + 16u * (uint32_t)j4);
                        b4v[j4] = lds128(eb + 16u * (uint32_t)j4);
                    }
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        const float cs[4] = {c4v[j4].x, c4v[j4].y, c4v[j4].z, c4v[j4].w};
                        const float b4[4] = {with_bias ? b4v[j4].x : 0.f, with_bias ? b4v[j4].y : 0.f,
                                             with_bias ? b4v[j4].z : 0.f, with_bias ? b4v[j4].w : 0.f};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            float o = v[4 * j4 + u];
                            // (rs = 1 when the tensor scale is folded into cs: o * rs is exact)
                            if constexpr (F16X3 || F16C) o = fmaf(o * rs, cs[u], b4[u]);
                            else o += b4[u];
                            v[4 * j4 + u] = P.relu ? fmaxf(o, 0.f) : o;
                        }
                    }
                } else {
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) {
                    float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
                    float cs[4] = {1.f, 1.f, 1.f, 1.f};
                    if (with_bias) bv = __ldg(reinterpret_cast<const float4 *>(P.bias + (int64_t)layer * P.k + kc) + j4);
                    if constexpr (F16X3 || F16C) {
                        const int4 ce = __ldg(reinterpret_cast<const int4 *>(
                            P.col_exp + (P.batched ? (int64_t)grp * P.k : (int64_t)layer * P.col_stride) + kc) + j4);
                        cs[0] = pow2f(-ce.x); cs[1] = pow2f(-ce.y); cs[2] = pow2f(-ce.z); cs[3] = pow2f(-ce.w);
                    }
                    const float b4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float o = v[4 * j4 + u];
                        if constexpr (F16X3 || F16C) o = fmaf(fused_scale ? o : o * rs, cs[u], b4[u]);
                        else o += b4[u];
                        v[4 * j4 + u] = P.relu ? fmaxf(o, 0.f) : o;
                    }
                }
                }
                if (c0 == 0 && q == 0 && lane == 0) PAIR_TRACE(7, t);   // chunk 0 in registers
                // staging box: FOLD alternates two (the store of chunk i-1 may still be reading)
                const uint32_t box = FOLD ? stg + (uint32_t)((nbox++ & 1) * kPairEpiBytes) : stg;
                if (issuer) {
                    if constexpr (FOLD) bulk_wait_read1();
                    else bulk_wait_read0();   // the previous chunk's store has read the box
                }
                epi_bar();
                if (inbox) {
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4)
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                                         box + (uint32_t)srow * 128 + (uint32_t)((j4 ^ (srow & 7)) << 4)),
                                     "f"(v[4 * j4]), "f"(v[4 * j4 + 1]), "f"(v[4 * j4 + 2]), "f"(v[4 * j4 + 3])
                                     : "memory");
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                epi_bar();
                if (RESB && c0 == 0 && q == 0 && lane == 0) PAIR_TRACE(0, t);   // chunk 0 staged
                if (issuer && blk < PP.blocks_per_group) {   // (a pair's spare block stores nothing)
                    if (spl >= 0) tma_reduce_add_4d(map_y, box, kc, ox0, oy0, img0);
                    else tma_store_4d(map_y, box, kc, ox0, oy0, img0);
                    bulk_commit();
                }
            }
        }
        if (issuer) bulk_wait0();
    } else if (TSA && F16C && warp >= 8) {
        // ---- 3xF16C TSA converters: warp (q, h) owns TMEM lanes 32q..32q+31 = A rows and
        // channel half h (fp32 tile h of the stage / footprint); each thread splits its row's
        // 32 channels into scaled fp16 hi / lo pairs and tcgen05.st's them to the A slot.
        // Halo: the row is footprint row m + r * fpr + s of tap (r, s) ----
        const int q = warp & 3, h = (warp >> 2) & 1;
        const int m = q * 32 + lane;
        const uint32_t tconv_leader = mapa_shared(smem_u32(tconv), 0);
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + A_COL0 + (uint32_t)(16 * h);
        const float sc = pow2f(f16_row_exp(__int_as_float(f16c_scale_max)));
        const int a_rows = P.bx * P.by * P.imgs;      // rows the TMA boxes fill (no halo; gather: real rows)
        const int fp_rows = PP.fp_bytes / 128;        // footprint rows (halo)
        // gather halo: this row's footprint pixel for tap (0, 0)
        int g_base = 0;
        if (HALO && PP.gather) {
            const int per_img = P.bx * P.by;
            const int im = m / per_img, pix = m - im * per_img;
            const int py = pix / P.bx, px = pix - py * P.bx;
            g_base = (im * PP.fh + py * P.stride) * PP.fw + px * P.stride;
        }
        float amax = 0.f;                             // max |x| over the real (loaded) rows
        int s = 0, ta = 0, it = 0, sa = 0;
        uint32_t ph = 0, pht = 0, pha = 0;
        uint32_t fa = 0;
        int resident = -1;   // RESB: the layer whose filter slice has landed
        uint32_t rph = 0;
        for (int item = cluster_id; item < PP.items; item += nclusters) {
            if constexpr (RESB) {
                int g_, p_, n_;
                decode(item, g_, p_, n_);
                const int layer = P.layer_imgs ? g_ : 0;
                if (layer != resident) {
                    mbar_wait(full, rph);
                    rph ^= 1;
                    resident = layer;
                }
            }
            int kb_lo, kb_hi;
            krange(item, kb_lo, kb_hi);
            int tap = 0;
            for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
                uint32_t row;
                int sw;
                bool real;   // a TMA-loaded row (not a wrap-around / beyond-the-box row)
                if constexpr (HALO) {
                    if (tap == 0) {
                        mbar_wait(afull + sa, pha);
                        fa = smem_u32(aring + sa * ASLOT);
                    }
                    // B of this tap landed (the MMA issuer learns it through tconv)
                    if constexpr (!RESB) mbar_wait(full + s, ph);
                    const int r = FOLD ? tap : tap / P.ks, sx = FOLD ? 0 : tap - r * P.ks;
                    const int fr = PP.gather ? g_base + r * PP.fw + sx : m + r * PP.fpr + sx;
                    row = fa + (h ? (uint32_t)PP.a_slot : 0u) + (uint32_t)fr * 128;
                    sw = fr & 7;
                    real = PP.gather ? m < a_rows : fr < fp_rows;
                } else {   // ARING: the A slot (the filter planes are the MMA issuer's to wait for)
                    mbar_wait(afull + sa, pha);
                    if (warp == 8 && lane == 0) EPI_TRACE(21, it);   // (trace builds) A data here
                    row = smem_u32(aring + sa * ASLOT) + (h ? (uint32_t)A_BYTES : 0u) + (uint32_t)m * 128;
                    sw = m & 7;
                    real = m < a_rows;
                }
                if (it >= NTA) mbar_wait(tfree + ta, pht ^ 1);
                if (warp == 8 && lane == 0) PAIR_TRACE(1, it);
                uint32_t hw[16], lw[16];
#ifdef CONVIO_ABL_NOCONV   // ablation (timing only, wrong numerics): no smem reads / split
#pragma unroll
                for (int c = 0; c < 16; ++c) hw[c] = lw[c] = row + c;
                if (0)
#endif
#pragma unroll
                for (int c = 0; c < 8; ++c) {   // fp32 chunk c: channels 32h + 4c .. 4c + 3
                    const float4 v = lds128(row + (uint32_t)((c ^ sw) << 4));
                    if (real) amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
                    const float2 sc2 = make_float2(sc, sc);
                    split_f16x2(v.x, v.y, sc2, hw[2 * c], lw[2 * c]);
                    split_f16x2(v.z, v.w, sc2, hw[2 * c + 1], lw[2 * c + 1]);
                }
                const uint32_t ta_col = (uint32_t)(ta * 64);
                tmem_st_32x32b_x16(lane_base + ta_col, hw);
                tmem_st_32x32b_x16(lane_base + ta_col + 32, lw);
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                if (warp == 8 && lane == 0) PAIR_TRACE(2, it);
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tconv_leader + (uint32_t)(ta * 8));
                if (warp == 8 && lane == 0) EPI_TRACE(22, it);   // (trace builds) signalled
                if (++ta == NTA) {
                    ta = 0;
                    pht ^= 1;
                }
                if constexpr (HALO) {
                    if (++tap == taps) {   // this warp is done reading the footprint
                        tap = 0;
                        if (lane == 0) mbar_arrive(aempty + sa);
                        if (++sa == NA) {
                            sa = 0;
                            pha ^= 1;
                        }
                    }
                } else {   // ARING: the A slot is in TMEM now
                    if (lane == 0) mbar_arrive(aempty + sa);
                    if (++sa == NA) {
                        sa = 0;
                        pha ^= 1;
                    }
                }
                if (!RESB && ++s == NS) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
        f16c_publish_max(PP, amax, &f16c_cta_max, NCW);
    } else if (TSA && warp >= 8) {
        // ---- TSA converters: warp q owns TMEM lanes 32q..32q+31 = A rows; each
        // thread reads its row's 32 channels from the SW128 stage, writes the
        // hi (truncated) / lo (rna) halves to TMEM with tcgen05.st, and converts
        // its share of the B rows to B_lo in shared memory.
        const int q = warp & 3;
        const int m = q * 32 + lane;
        const int ct = tid - 256;                    // 0..127
        const uint32_t tconv_leader = mapa_shared(smem_u32(tconv), 0);
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + A_COL0;
        int s = 0, ta = 0, it = 0;
        uint32_t ph = 0, pht = 0;
        for (int item = cluster_id; item < PP.items; item += nclusters) {
            int kb_lo, kb_hi;
            krange(item, kb_lo, kb_hi);
            for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
                mbar_wait(full + s, ph);
                if (it >= NTA) mbar_wait(tfree + ta, pht ^ 1);
                const uint32_t st = smem_u32(bring + s * STAGE);
                const uint32_t row = st + (uint32_t)m * 128;
                uint32_t hi[32], lo[32];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float4 v = lds128(row + (uint32_t)((c ^ (m & 7)) << 4));
                    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t h = __float_as_uint(e[j]) & 0xffffe000u;
                        hi[c * 4 + j] = h;
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo[c * 4 + j]) : "f"(e[j] - __uint_as_float(h)));
                    }
                }
                const uint32_t ta_col = (uint32_t)(ta * 64);
                tmem_st_32x32b_x32(lane_base + ta_col, hi);
                tmem_st_32x32b_x32(lane_base + ta_col + 32, lo);
                convert_lo_range<128>(st + A_BYTES, st + A_BYTES + B_BYTES, B_BYTES / 16, ct);
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(tconv_leader + (uint32_t)(ta * 8));
                if (++ta == NTA) {
                    ta = 0;
                    pht ^= 1;
                }
                if (++s == NS) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (F16C && warp >= 8) {
        // ---- 3xF16C converters: activation rows -> scaled fp16 hi / lo planes, in place;
        // the filter planes arrive pre-split, so a filter stage is only passed on ----
        const int ct = tid - 256;                    // 0 .. 255
        const uint32_t conv_leader = mapa_shared(smem_u32(conv), 0);
        const uint32_t aconv_leader = mapa_shared(smem_u32(aconv), 0);
        const float sc = pow2f(f16_row_exp(__int_as_float(f16c_scale_max)));
        const int a_rows = P.bx * P.by * P.imgs;
        const int fp_rows = PP.fp_bytes / 128;
        float amax = 0.f;
        int s = 0, sa = 0, kbc = 0;
        uint32_t ph = 0, pha = 0;
        for (int item = cluster_id; item < PP.items; item += nclusters) {
            int tap = 0;
            int kb_lo, kb_hi;
            krange(item, kb_lo, kb_hi);
            for (int kb = kb_lo; kb < kb_hi; ++kb) {
                if (HALO && tap == 0) {
                    mbar_wait(afull + sa, pha);
                    const uint32_t f0 = smem_u32(aring + sa * ASLOT);
#ifndef CONVIO_ABL_NOCONV
                    convert_f16_rows<32 * NCW>(f0, f0 + (uint32_t)PP.a_slot, fp_rows, ct, sc, amax);
#endif
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(aconv_leader + (uint32_t)(sa * 8));
                    if (++sa == NA) {
                        sa = 0;
                        pha ^= 1;
                    }
                }
                mbar_wait(full + s, ph);
                if (warp == 8 && lane == 0) PAIR_TRACE(1, kbc);
                if constexpr (!HALO) {
                    const uint32_t st = smem_u32(bring + s * STAGE);
#ifndef CONVIO_ABL_NOCONV
                    convert_f16_rows<32 * NCW>(st, st + A_BYTES + B_BYTES, a_rows, ct, sc, amax);
#endif
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                }
                __syncwarp();
                if (warp == 8 && lane == 0) PAIR_TRACE(2, kbc);
                ++kbc;
                if (lane == 0) mbar_arrive_cluster(conv_leader + (uint32_t)(s * 8));
                if (HALO && ++tap == taps) tap = 0;
                if (++s == NS) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
        f16c_publish_max(PP, amax, &f16c_cta_max, NCW);
    } else if (SPLIT && !TSA && warp >= 8) {
        // ---- converters: lo = v - tf32(v) of this CTA's staged operands (3xTF32) ----
        const int ct = tid - 256;                    // 0 .. 32*NCW-1
        const uint32_t conv_leader = mapa_shared(smem_u32(conv), 0);
        const uint32_t aconv_leader = mapa_shared(smem_u32(aconv), 0);
        int s = 0, sa = 0, l = 0, itl = 0;
        uint32_t ph = 0, pha = 0, phl = 0;
        for (int item = cluster_id; item < PP.items; item += nclusters) {
            int tap = 0;
            int kb_lo, kb_hi;
            krange(item, kb_lo, kb_hi);
            for (int kb = kb_lo; kb < kb_hi; ++kb) {
                if (HALO && tap == 0) {
                    mbar_wait(afull + sa, pha);
                    const uint32_t hi = smem_u32(aring + sa * ASLOT);
                    convert_lo_range<32 * NCW>(hi, hi + (uint32_t)PP.a_slot, PP.fp_bytes / 16, ct);
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(aconv_leader + (uint32_t)(sa * 8));
                    if (++sa == NA) {
                        sa = 0;
                        pha ^= 1;
                    }
                }
                mbar_wait(full + s, ph);
                const uint32_t hi = smem_u32(bring + s * STAGE);
                if constexpr (HALO) {
                    convert_lo_range<32 * NCW>(hi, hi + B_BYTES, B_BYTES / 16, ct);
                } else if constexpr (!LOSLOT) {
                    convert_lo_range<32 * NCW>(hi, hi + A_BYTES + B_BYTES, (A_BYTES + B_BYTES) / 16, ct);
                } else {
                    if (itl >= NL) mbar_wait(lofree + l, phl ^ 1);   // slot's previous MMAs done
                    convert_lo_range<32 * NCW>(hi, smem_u32(loring + l * LO_SLOT), (A_BYTES + B_BYTES) / 16, ct);
                    ++itl;
                    if (++l == NL) {
                        l = 0;
                        phl ^= 1;
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(conv_leader + (uint32_t)(s * 8));
                if (HALO && ++tap == taps) tap = 0;
                if (++s == NS) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    }
    // ---- teardown ---------------------------------------------------------------------
#ifdef CONVIO_TRACE
    if (PP.trace && warp == 4 && lane == 0 && blockIdx.x < 1024) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        PP.trace[17 * 1024 + blockIdx.x] = g;
    }
#endif
    __syncwarp();   // role lanes rejoin their warps before the .aligned cluster barrier
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cluster_sync_all();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
}

}  // namespace convio
