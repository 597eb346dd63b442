// Standalone probe: tcgen05.mma issue rate of one CTA pair (cta_group::2, M = 256)
// per operand kind (tf32 / f16) and N, with A from shared memory (SS) or from
// tensor memory (TS).  One elected thread issues 4 K-steps x iters MMAs into
// one accumulator; cycles per MMA (K = 32 B) are printed.  Timing only (stale
// operands).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o umma_rate_probe umma_rate_probe.cu -lcuda
#include <cstdio>

#include "../../paper_2012_15667_b200/csrc/igemm_pair.cuh"

using namespace convio;

// PAT = 0: one operand pair; PAT = 1: the 3-product split pattern of the conv kernels
// (hi*lo, lo*hi, hi*hi with distinct A / B planes per product)
template <int NN, int KIND, bool TS, int PAT = 0>
__global__ void __cluster_dims__(2, 1, 1) k_rate(long long *cycles, int iters) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t *a = sm;                       // 2 planes x 128 x 128 B
    uint8_t *b = sm + 2 * 128 * 128;       // 2 planes x 128 x 128 B (NN/2 rows used)
    uint64_t *done = reinterpret_cast<uint64_t *>(b + 2 * 128 * 128);
    uint32_t *slot = reinterpret_cast<uint32_t *>(done + 1);
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        mbar_init(done, 1);
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
    if (rank == 0 && threadIdx.x == 0) {
        const uint64_t ad = umma_desc_sw128(smem_u32(a)), bd = umma_desc_sw128(smem_u32(b));
        const uint64_t adl = umma_desc_sw128(smem_u32(a) + 128 * 128), bdl = umma_desc_sw128(smem_u32(b) + 128 * 128);
        constexpr uint32_t idesc = idesc_m256<NN, KIND>();
        const uint32_t ta = tmem + 256;    // A operand columns (TS)
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if constexpr (PAT == 1) {
                    if constexpr (TS) {
                        umma_pair_ts_f16(tmem, ta + kk * 8, bdl + kk * 2, idesc, 1);
                        umma_pair_ts_f16(tmem, ta + 32 + kk * 8, bd + kk * 2, idesc, 1);
                        umma_pair_ts_f16(tmem, ta + kk * 8, bd + kk * 2, idesc, 1);
                    } else {
                        umma_pair<KIND>(tmem, ad + kk * 2, bdl + kk * 2, idesc, 1);
                        umma_pair<KIND>(tmem, adl + kk * 2, bd + kk * 2, idesc, 1);
                        umma_pair<KIND>(tmem, ad + kk * 2, bd + kk * 2, idesc, 1);
                    }
                } else if constexpr (TS) {
                    if constexpr (KIND == KIND_3XF16C) umma_pair_ts_f16(tmem, ta + kk * 8, bd + kk * 2, idesc, 1);
                    else umma_pair_ts_tf32(tmem, ta + kk * 8, bd + kk * 2, idesc, 1);
                } else {
                    umma_pair<KIND>(tmem, ad + kk * 2, bd + kk * 2, idesc, 1);
                }
            }
        umma_commit_pair(done);
        mbar_wait(done, 0);
        *cycles = (clock64() - t0) / ((PAT ? 12LL : 4LL) * iters);
    } else if (rank == 1 && threadIdx.x == 0) {
        mbar_wait(done, 0);
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int NN, int KIND, bool TS, int PAT = 0>
static void rate(long long *dcyc) {
    const size_t smem = 1024 + 4 * 128 * 128 + 64;
    cudaFuncSetAttribute(k_rate<NN, KIND, TS, PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long cyc = 0;
    k_rate<NN, KIND, TS, PAT><<<2, 128, smem>>>(dcyc, 4096);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    printf("pair M256 N%3d %s %s%s: %lld cycles per MMA (K = 32 B) %s\n", NN,
           KIND == KIND_3XF16C ? "f16 " : "tf32", TS ? "A in TMEM" : "A in smem",
           PAT ? " 3-product split pattern" : "", cyc,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long *dcyc;
    cudaMalloc(&dcyc, 8);
    rate<64, KIND_TF32, false>(dcyc);
    rate<128, KIND_TF32, false>(dcyc);
    rate<256, KIND_TF32, false>(dcyc);
    rate<64, KIND_3XF16C, false>(dcyc);
    rate<128, KIND_3XF16C, false>(dcyc);
    rate<192, KIND_3XF16C, false>(dcyc);
    rate<256, KIND_3XF16C, false>(dcyc);
    rate<64, KIND_3XF16C, true>(dcyc);
    rate<128, KIND_3XF16C, true>(dcyc);
    rate<256, KIND_3XF16C, true>(dcyc);
    rate<128, KIND_TF32, true>(dcyc);
    rate<64, KIND_3XF16C, false, 1>(dcyc);
    rate<128, KIND_3XF16C, false, 1>(dcyc);
    rate<192, KIND_3XF16C, false, 1>(dcyc);
    rate<256, KIND_3XF16C, false, 1>(dcyc);
    rate<64, KIND_3XF16C, true, 1>(dcyc);
    rate<192, KIND_3XF16C, true, 1>(dcyc);
    rate<128, KIND_3XF16C, true, 1>(dcyc);
    rate<256, KIND_3XF16C, true, 1>(dcyc);
    return 0;
}
