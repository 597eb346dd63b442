// Standalone probe: can a tcgen05.mma K-major SWIZZLE_128B operand descriptor
// start at an arbitrary 128-B row inside a TMA-written (1024-B aligned) tile?
// The A tile is a 192-row "footprint" written by TMA; the MMA reads the 128
// rows starting at row `shift` (the tap offset of the halo-staged implicit
// GEMM).  Two descriptor variants: base_offset = 0, and base_offset =
// (start >> 7) & 7.  Prints the max error of each against a host reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o umma_shift_selftest \
//        umma_shift_selftest.cu -lcuda
#include <cmath>
#include <cstdio>
#include <vector>

#include "../../paper_2012_15667_b200/csrc/igemm_tcgen05.cuh"

using namespace convio;

constexpr int ROWS = 192, N = 64;

__global__ void k_shift(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                        float *out, int shift, int use_base) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t *a = sm;                       // ROWS x 128 B
    uint8_t *b = sm + ROWS * 128;          // N x 128 B
    uint64_t *bar = reinterpret_cast<uint64_t *>(b + N * 128);
    uint64_t *done = bar + 1;
    uint32_t *slot = reinterpret_cast<uint32_t *>(done + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, ROWS * 128 + N * 128);
        tma_load_2d(a, reinterpret_cast<uint64_t>(&tma), 0, 0, bar);
        tma_load_2d(b, reinterpret_cast<uint64_t>(&tmb), 0, 0, bar);
        mbar_wait(bar, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t start = smem_u32(a) + shift * 128;
        uint64_t ad = umma_desc_sw128(start);
        if (use_base) ad |= (uint64_t)((start >> 7) & 7) << 49;
        const uint64_t bd = umma_desc_sw128(smem_u32(b));
        constexpr uint32_t idesc = idesc_m128<N, KIND_TF32>();
        for (int kk = 0; kk < 4; ++kk)
            umma_tf32(tmem, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc, kk != 0);
        umma_commit(done);
    }
    mbar_wait(done, 0);
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    for (int c0 = 0; c0 < N; c0 += 32) {
        float v[32];
        tmem_ld_32x32b<32>(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * N + c0 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(64));
}

// Throughput probe: one thread issues `iters` x 4 MMAs (M=128, N=64, K=8 tf32)
// reading the A operand at row offset `shift`; returns cycles per MMA.
template <int NN, bool BF16, int ND = 1>
__global__ void k_rate(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
                       long long *cycles, int shift, int iters) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t *a = sm;
    uint8_t *b = sm + ROWS * 128;
    uint64_t *bar = reinterpret_cast<uint64_t *>(b + 256 * 128);
    uint64_t *done = bar + 1;
    uint32_t *slot = reinterpret_cast<uint32_t *>(done + 1);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, ROWS * 128 + N * 128);
        tma_load_2d(a, reinterpret_cast<uint64_t>(&tma), 0, 0, bar);
        tma_load_2d(b, reinterpret_cast<uint64_t>(&tmb), 0, 0, bar);
        mbar_wait(bar, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint64_t ad = umma_desc_sw128(smem_u32(a) + shift * 128);
        const uint64_t bd = umma_desc_sw128(smem_u32(b));   // rows >= N are stale: timing only
        constexpr uint32_t idesc = idesc_m128<NN, BF16 ? KIND_BF16 : KIND_TF32>();
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
            for (int kk = 0; kk < 4; ++kk) {
                // ND independent accumulators (D columns kk % ND * NN): does the tensor
                // core overlap MMAs that do not chain on one accumulator?
                const uint32_t dcol = tmem + (uint32_t)((kk % ND) * NN);
                if constexpr (BF16) umma_bf16(dcol, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc, 1);
                else umma_tf32(dcol, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc, 1);
            }
        umma_commit(done);
        mbar_wait(done, 0);
        *cycles = (clock64() - t0) / (4LL * iters);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
}

template <int NN, bool BF16, int ND = 1>
static void rate(const CUtensorMap &ma, const CUtensorMap &mb, long long *dcyc, int s) {
    const size_t smem = 1024 + ROWS * 128 + 256 * 128 + 64;
    cudaFuncSetAttribute(k_rate<NN, BF16, ND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long cyc = 0;
    k_rate<NN, BF16, ND><<<1, 128, smem>>>(ma, mb, dcyc, s, 4096);
    cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    printf("rate: %s M128 N%3d shift=%2d accumulators=%d: %lld cycles per MMA (K = 32 B)\n",
           BF16 ? "bf16" : "tf32", NN, s, ND, cyc);
}

int main() {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    std::vector<float> ha(ROWS * 32), hb(N * 32);
    for (size_t i = 0; i < ha.size(); ++i) ha[i] = (float)((i * 37 % 101) - 50) / 64.0f;   // tf32-exact
    for (size_t i = 0; i < hb.size(); ++i) hb[i] = (float)((i * 53 % 97) - 48) / 32.0f;
    float *da, *db, *dout;
    cudaMalloc(&da, ha.size() * 4);
    cudaMalloc(&db, hb.size() * 4);
    cudaMalloc(&dout, 128 * N * 4);
    cudaMemcpy(da, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap ma, mb;
    cuuint64_t dA[2] = {32, ROWS}, sA[1] = {128}, dB[2] = {32, N}, sB[1] = {128};
    cuuint32_t bA[2] = {32, ROWS}, bB[2] = {32, N}, es[2] = {1, 1};
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, da, dA, sA, bA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, db, dB, sB, bB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = 1024 + ROWS * 128 + N * 128 + 64;
    cudaFuncSetAttribute(k_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    std::vector<float> out(128 * N);
    const int shifts[] = {0, 1, 2, 3, 7, 8, 9, 16, 17, 18, 34, 50, 64};
    for (int use_base = 0; use_base < 2; ++use_base) {
        for (int s : shifts) {
            cudaMemset(dout, 0, 128 * N * 4);
            k_shift<<<1, 128, smem>>>(ma, mb, dout, s, use_base);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("base=%d shift=%d: CUDA error %s\n", use_base, s, cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < N; ++n) {
                    double ref = 0;
                    for (int k = 0; k < 32; ++k) ref += (double)ha[(m + s) * 32 + k] * hb[n * 32 + k];
                    maxerr = fmax(maxerr, fabs(ref - out[m * N + n]));
                }
            printf("base_offset=%s shift=%2d: max abs err %.3g\n", use_base ? "(start>>7)&7" : "0", s, maxerr);
        }
    }
    long long *dcyc;
    cudaMalloc(&dcyc, 8);
    for (int s : {0, 1, 17}) rate<64, false>(ma, mb, dcyc, s);
    rate<128, false>(ma, mb, dcyc, 0);
    rate<256, false>(ma, mb, dcyc, 0);
    rate<256, false>(ma, mb, dcyc, 17);
    rate<64, true>(ma, mb, dcyc, 0);
    rate<128, true>(ma, mb, dcyc, 0);
    rate<256, true>(ma, mb, dcyc, 0);
    rate<64, false, 2>(ma, mb, dcyc, 0);
    rate<64, false, 4>(ma, mb, dcyc, 0);
    rate<128, false, 2>(ma, mb, dcyc, 0);
    return 0;
}

// ---- CTA-pair (cta_group::2) MMA rate: M = 256 over two CTAs, N = NN --------------
#include "../../paper_2012_15667_b200/csrc/igemm_pair.cuh"

template <int NN>
__global__ void __cluster_dims__(2, 1, 1) k_rate_pair(long long *cycles, int iters) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t *a = sm;                       // 128 x 128 B (stale data: timing only)
    uint8_t *b = sm + 128 * 128;           // NN/2 x 128 B
    uint64_t *done = reinterpret_cast<uint64_t *>(b + 128 * 128);
    uint32_t *slot = reinterpret_cast<uint32_t *>(done + 1);
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *slot;
    if (rank == 0 && threadIdx.x == 0) {
        const uint64_t ad = umma_desc_sw128(smem_u32(a)), bd = umma_desc_sw128(smem_u32(b));
        constexpr uint32_t idesc = idesc_m256<NN, KIND_TF32>();
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
            for (int kk = 0; kk < 4; ++kk) umma_pair<KIND_TF32>(tmem, ad + kk * 2, bd + kk * 2, idesc, 1);
        umma_commit_pair(done);
        mbar_wait(done, 0);
        *cycles = (clock64() - t0) / (4LL * iters);
    } else if (rank == 1 && threadIdx.x == 0) {
        mbar_wait(done, 0);
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
}

template <int NN>
static void rate_pair(long long *dcyc) {
    const size_t smem = 1024 + 2 * 128 * 128 + 64;
    cudaFuncSetAttribute(k_rate_pair<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long cyc = 0;
    k_rate_pair<NN><<<2, 128, smem>>>(dcyc, 4096);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    printf("rate: tf32 pair M256 N%3d: %lld cycles per MMA (K = 32 B) %s\n", NN, cyc,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int pair_rates() {
    long long *dcyc;
    cudaMalloc(&dcyc, 8);
    rate_pair<64>(dcyc);
    rate_pair<128>(dcyc);
    rate_pair<192>(dcyc);
    rate_pair<256>(dcyc);
    return 0;
}
static int pair_rates_done = (pair_rates(), 0);
