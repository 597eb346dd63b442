// Standalone probe: tcgen05.mma rate of one CTA pair (cta_group::2, M = 256, kind::f16,
// 3-product pattern) while 8 other warps per CTA load the SM with
//   BG = 0: nothing, 1: tcgen05.st (32 KB per round into TMEM columns the MMA does not
//   use), 2: LDS.128 sweeps of shared memory, 3: both -- the converter-warp traffic of
// the 3xF16 conv kernels.  Cycles per MMA (K = 32 B).  Timing only (stale operands).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -o umma_contention_probe umma_contention_probe.cu -lcuda
#include <cstdio>

#include "../../paper_2012_15667_b200/csrc/igemm_pair.cuh"

using namespace convio;

template <int NN, bool TS, int BG, int NC = 0>
__global__ void __cluster_dims__(2, 1, 1) k_cont(long long *cycles, int iters, const uint8_t *gsrc) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t *a = sm;
    uint8_t *b = sm + 2 * 128 * 128;
    uint8_t *junk = b + 2 * 128 * 128;     // 64 KB swept by the LDS warps
    uint64_t *done = reinterpret_cast<uint64_t *>(junk + 65536);
    uint64_t *bulk = done + 2;
    uint32_t *slot = reinterpret_cast<uint32_t *>(done + 1);
    volatile uint32_t *stop = slot + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    // operands: non-trivial bit patterns (fp16 values in [-1, 1)), so the tensor core does real work
    for (int i = threadIdx.x; i < 4 * 128 * 128 / 4; i += blockDim.x) {
        const uint32_t h = (uint32_t)(i * 2654435761u + blockIdx.x * 97u);
        reinterpret_cast<uint32_t *>(a)[i] = (h & 0x3bff3bffu) | 0x30003000u;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_init(done, 1);
        mbar_init(bulk, 1);
        mbar_init(bulk + 1, 1);
        mbar_init(bulk + 2, 1);
        mbar_init(bulk + 3, 1);
        mbar_arrive(bulk + 3);   // phase 0 complete: waits on parity 0 return at once
        *stop = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *slot;
    if (warp == 0) {
        if (rank == 0 && lane == 0) {
            const uint64_t ad = umma_desc_sw128(smem_u32(a)), bd = umma_desc_sw128(smem_u32(b));
            const uint64_t adl = umma_desc_sw128(smem_u32(a) + 128 * 128), bdl = umma_desc_sw128(smem_u32(b) + 128 * 128);
            constexpr uint32_t idesc = idesc_m256<NN, KIND_3XF16C>();
            const uint32_t ta = tmem + 256;
            const long long t0 = clock64();
            for (int it = 0; it < iters; ++it)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    if (NC >= 3 && kk == 0) {   // the conv kernels' per-k-block barrier wait (already complete)
                        if (NC != 4) mbar_wait(bulk + 3, 0);
                        if (NC != 5) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    }
                    if constexpr (TS) {
                        umma_pair_ts_f16(tmem, ta + kk * 8, bdl + kk * 2, idesc, 1);
                        umma_pair_ts_f16(tmem, ta + 32 + kk * 8, bd + kk * 2, idesc, 1);
                        umma_pair_ts_f16(tmem, ta + kk * 8, bd + kk * 2, idesc, 1);
                    } else {
                        umma_pair<KIND_3XF16C>(tmem, ad + kk * 2, bdl + kk * 2, idesc, 1);
                        umma_pair<KIND_3XF16C>(tmem, adl + kk * 2, bd + kk * 2, idesc, 1);
                        umma_pair<KIND_3XF16C>(tmem, ad + kk * 2, bd + kk * 2, idesc, 1);
                    }
                    if (kk == 3) {   // NC commits per k-block (the conv kernels: stage + A slot release)
                        if (NC >= 1 && NC <= 3) umma_commit_pair(bulk + 1);
                        if (NC >= 2 && NC <= 3) umma_commit_pair(bulk + 2);
                    }
                }
            umma_commit_pair(done);
            mbar_wait(done, 0);
            *cycles = (clock64() - t0) / (12LL * iters);
            *stop = 1;
        } else if (rank == 1 && lane == 0) {
            mbar_wait(done, 0);
            *stop = 1;
        }
    } else if (warp >= 4 && (BG & 7)) {
        const int q = warp & 3;
        uint32_t r[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = lane + i;
        float acc = 0.f;
        while (!*stop) {
            if (BG & 1) {   // 2 x 16 columns per warp per round: the converters' A-slot stores
                const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + 384 + (uint32_t)(16 * ((warp >> 2) & 1));
                tmem_st_32x32b_x16(base, r);
                tmem_st_32x32b_x16(base + 32, r);
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            }
            if (BG & 4) {   // epilogue-like TMEM reads: 32 columns per warp per round
                float v[32];
                const long long t0 = clock64();
                tmem_ld_32x32b<32>(tmem + ((uint32_t)(q * 32) << 16) + 384, v);
                const long long t1 = clock64();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc += v[j];
                if (warp == 4 && lane == 0 && rank == 0) { cycles[1] += t1 - t0; cycles[2] += 1; }
            }
            if (BG & 2) {   // 8 x LDS.128 per thread per round
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float4 v = lds128(smem_u32(junk) + (uint32_t)((((warp - 4) * 32 + lane) * 128 + (c << 4)) & 65535));
                    acc += v.x + v.y + v.z + v.w;
                }
            }
        }
        if (acc == 12345.f) *cycles = 0;
    } else if ((BG & 8) && warp == 3 && lane == 0) {   // bulk copies global -> smem (TMA-like writes)
        uint32_t phase = 0;
        for (int rep = 0; !*stop; rep = (rep + 1) & 63) {
            mbar_arrive_expect_tx(bulk, 65536);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                         ::"r"(smem_u32(junk)), "l"(gsrc + (size_t)rep * 65536), "r"(65536), "r"(smem_u32(bulk)) : "memory");
            mbar_wait(bulk, phase);
            phase ^= 1;
        }
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int NN, bool TS, int BG, int NC = 0>
static void run(long long *dcyc, int ctas = 2) {
    const size_t smem = 1024 + 4 * 128 * 128 + 65536 + 64;
    cudaFuncSetAttribute(k_cont<NN, TS, BG, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long cyc = 0;
    static uint8_t *g = nullptr;
    if (!g) cudaMalloc(&g, 64 << 20);
    cudaMemset(dcyc, 0, 24);
    k_cont<NN, TS, BG, NC><<<ctas, 384, smem>>>(dcyc, ctas > 2 ? 65536 : 2048, g);
    cudaError_t e = cudaDeviceSynchronize();
    long long all[3] = {0, 0, 0};
    cudaMemcpy(all, dcyc, 24, cudaMemcpyDeviceToHost);
    cyc = all[0];
    if (all[2]) printf("   tcgen05.ld x32 + wait under MMA load: %lld cycles avg over %lld\n", all[1] / all[2], all[2]);
    static const char *bg[] = {"idle", "tcgen05.st", "LDS.128", "tcgen05.st + LDS.128", "tcgen05.ld", "", "", "",
                               "bulk copy", "", "", "", "tcgen05.ld + bulk", "", "", "all"};
    printf("%d commits/k-block %3d CTAs: pair M256 N%3d f16 3-product %s, 8 background warps: %-20s %lld cycles per MMA %s\n", NC, ctas, NN,
           TS ? "A in TMEM" : "A in smem", bg[BG], cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    long long *dcyc;
    cudaMalloc(&dcyc, 24);
    run<256, false, 4>(dcyc); run<128, true, 4>(dcyc); run<256, false, 4>(dcyc, 148);
    return 0;
    run<128, true, 0, 3>(dcyc); run<128, true, 0, 4>(dcyc); run<128, true, 0, 5>(dcyc);
    run<128, false, 0, 3>(dcyc); run<128, false, 0, 4>(dcyc); run<128, false, 0, 5>(dcyc);
    run<256, false, 0, 3>(dcyc);
    run<128, true, 0, 1>(dcyc); run<128, true, 0, 2>(dcyc); run<256, false, 0, 2>(dcyc); run<128, false, 0, 2>(dcyc);
    run<128, true, 0>(dcyc, 148); run<256, false, 0>(dcyc, 148); run<128, true, 15>(dcyc, 148);
    run<128, true, 0>(dcyc); run<128, true, 1>(dcyc); run<128, true, 2>(dcyc); run<128, true, 3>(dcyc);
    run<128, true, 4>(dcyc); run<128, true, 8>(dcyc); run<128, true, 12>(dcyc); run<128, true, 15>(dcyc);
    run<256, false, 4>(dcyc); run<256, false, 8>(dcyc); run<256, false, 14>(dcyc);
    run<128, false, 0>(dcyc); run<128, false, 2>(dcyc);
    run<256, false, 0>(dcyc); run<256, false, 2>(dcyc);
    run<256, true, 0>(dcyc); run<256, true, 1>(dcyc); run<256, true, 3>(dcyc);
    return 0;
}
