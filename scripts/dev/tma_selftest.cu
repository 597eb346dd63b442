// Standalone TMA probe: 4-D tiled box loads with OOB zero fill, variants of box width.
#include <cstdio>
#include <vector>
#include "../../paper_2012_15667_b200/csrc/direct_fp32.cuh"

using namespace convio;

__global__ void k_tma(const __grid_constant__ CUtensorMap tm, float *out, int bw, int bh, int bc,
                      int x0, int y0, int c0) {
    extern __shared__ __align__(128) float sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + bw * bh * bc + 32);
    const uint64_t map = reinterpret_cast<uint64_t>(&tm);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, bw * bh * bc * 4);
        tma_load_4d(sm, map, x0, y0, c0, 0, bar);
    }
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < bw * bh * bc; i += blockDim.x) out[i] = sm[i];
}

int main() {
    auto enc = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    const int W = 56, H = 56, C = 8, N = 1;
    std::vector<float> h(W * H * C);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 1 << 20);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    struct V { int bw, bh, bc, x0, y0, c0; } vs[] = {
        {16, 4, 2, 0, 0, 0}, {16, 4, 2, 48, 54, 7}, {64, 4, 2, 0, 0, 0}, {16, 4, 2, 0, -1, 0},
        {16, 4, 2, -4, 0, 0}, {16, 4, 2, -1, 0, 0}, {16, 4, 2, -1, -1, 0}};
    for (auto v : vs) {
        CUtensorMap tm;
        cuuint64_t gdim[4] = {W, H, C, N};
        cuuint64_t gstr[3] = {W * 4ull, W * H * 4ull, W * H * C * 4ull};
        cuuint32_t box[4] = {(cuuint32_t)v.bw, (cuuint32_t)v.bh, (cuuint32_t)v.bc, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, gdim, gstr, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        size_t smem = v.bw * v.bh * v.bc * 4 + 256;
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
        k_tma<<<1, 128, smem>>>(tm, o, v.bw, v.bh, v.bc, v.x0, v.y0, v.c0);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> got(v.bw * v.bh * v.bc);
        int bad = -1;
        if (e == cudaSuccess) {
            cudaMemcpy(got.data(), o, got.size() * 4, cudaMemcpyDeviceToHost);
            for (int c = 0; c < v.bc && bad < 0; ++c)
                for (int y = 0; y < v.bh && bad < 0; ++y)
                    for (int x = 0; x < v.bw; ++x) {
                        int gx = v.x0 + x, gy = v.y0 + y, gc = v.c0 + c;
                        float want = (gx >= 0 && gx < W && gy >= 0 && gy < H && gc < C) ? h[(gc * H + gy) * W + gx] : 0.f;
                        if (got[(c * v.bh + y) * v.bw + x] != want) { bad = (c * v.bh + y) * v.bw + x; break; }
                    }
        }
        printf("box %dx%dx%d at (%d,%d,%d): encode=%d launch=%s mismatch_at=%d\n", v.bw, v.bh, v.bc,
               v.x0, v.y0, v.c0, (int)r, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 1 << 20);
            cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice); }
    }
    return 0;
}
