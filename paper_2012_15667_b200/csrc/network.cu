// The steps either side of the conv path in a chained network forward (SURVEY.md
// §8(f) items 2-3): NCHW <-> NHWC layout staging (the reference's layout axis,
// pkg/src/convio/dataflow.py:23, made a counted device kernel instead of a host /
// framework copy) and 2x2 / stride-2 max pooling of channels-last activations,
// which VGG-style networks put between conv blocks.  All HBM-streaming: one read
// and one write of every element, coalesced on both sides.
#include <algorithm>

#include "common.cuh"

namespace convio {

// [n][c][hw] <-> [n][hw][c] through 32 x 33 shared-memory tiles (coalesced reads and
// writes; the +1 column keeps the transposed read conflict-free).  TO_NHWC picks the
// direction: rows of the source tile are channels (NCHW -> NHWC) or pixels.
template <bool TO_NHWC>
__global__ void __launch_bounds__(256) transpose_chw_kernel(const float *__restrict__ x, float *__restrict__ y,
                                                            int c, int hw) {
    pdl_wait();
    __shared__ float t[32][33];
    const int64_t img = blockIdx.z;
    const int rows = TO_NHWC ? c : hw, cols = TO_NHWC ? hw : c;
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    const float *src = x + img * (int64_t)c * hw;
    float *dst = y + img * (int64_t)c * hw;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, cc = c0 + threadIdx.x;
        if (r < rows && cc < cols) t[i][threadIdx.x] = __ldg(src + (int64_t)r * cols + cc);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int cc = c0 + i, r = r0 + threadIdx.x;
        if (cc < cols && r < rows) dst[(int64_t)cc * rows + r] = t[threadIdx.x][i];
    }
}

// few channels (C <= 4, e.g. the RGB input of a network): one thread per pixel,
// channel planes read coalesced, the pixel's C values written contiguously
__global__ void __launch_bounds__(256) nchw_to_nhwc_smallc_kernel(const float *__restrict__ x,
                                                                  float *__restrict__ y, int c, int64_t hw,
                                                                  int64_t total) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t img = i / hw, p = i - img * hw;
        const float *src = x + img * c * hw + p;
        float *dst = y + i * c;
        for (int cc = 0; cc < c; ++cc) dst[cc] = __ldg(src + cc * hw);
    }
}

// y[n][oy][ox][c] = max over the 2 x 2 window (NHWC, C % 4 == 0, float4 over
// channels; odd H / W drop the last row / column as floor pooling does)
__global__ void __launch_bounds__(256) maxpool2x2_nhwc_kernel(const float *__restrict__ x, float *__restrict__ y,
                                                              int h, int w, int c, int64_t total4) {
    pdl_wait();
    const int oh = h / 2, ow = w / 2, c4 = c / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ch = (int)(i % c4);
        int64_t rest = i / c4;
        const int ox = (int)(rest % ow);
        rest /= ow;
        const int oy = (int)(rest % oh);
        const int64_t img = rest / oh;
        const float4 *p = reinterpret_cast<const float4 *>(x + ((img * h + 2 * oy) * w + 2 * ox) * (int64_t)c) + ch;
        const int64_t row = (int64_t)w * c4;
        const float4 a = __ldg(p), b = __ldg(p + c4), d = __ldg(p + row), e = __ldg(p + row + c4);
        float4 o;
        o.x = fmaxf(fmaxf(a.x, b.x), fmaxf(d.x, e.x));
        o.y = fmaxf(fmaxf(a.y, b.y), fmaxf(d.y, e.y));
        o.z = fmaxf(fmaxf(a.z, b.z), fmaxf(d.z, e.z));
        o.w = fmaxf(fmaxf(a.w, b.w), fmaxf(d.w, e.w));
        reinterpret_cast<float4 *>(y)[i] = o;
    }
}

static int grid_for(int64_t total) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
}

static int launch_transpose(const float *x, float *y, int n, int c, int hw, bool to_nhwc, cudaStream_t st) {
    if (to_nhwc && c <= 4) {
        const int64_t total = (int64_t)n * hw;
        CONVIO_CUDA_TRY(launch_pdl(nchw_to_nhwc_smallc_kernel, dim3(grid_for(total)), dim3(256), 0, st, x, y, c,
                                   (int64_t)hw, total));
    } else {
        const int rows = to_nhwc ? c : hw, cols = to_nhwc ? hw : c;
        const dim3 grid((cols + 31) / 32, (rows + 31) / 32, n);
        if (grid.y > 65535 || grid.z > 65535) {
            set_error("layout transpose grid exceeds launch limits");
            return CONVIO_EINFEASIBLE;
        }
        if (to_nhwc)
            CONVIO_CUDA_TRY(launch_pdl(transpose_chw_kernel<true>, grid, dim3(32, 8), 0, st, x, y, c, hw));
        else
            CONVIO_CUDA_TRY(launch_pdl(transpose_chw_kernel<false>, grid, dim3(32, 8), 0, st, x, y, c, hw));
    }
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

}  // namespace convio

using namespace convio;

extern "C" {

int convio_nchw_to_nhwc(const float *x, float *y, int32_t n, int32_t c, int32_t h, int32_t w, void *stream) {
    clear_error();
    reset_launches();
    if (!x || !y || n < 1 || c < 1 || h < 1 || w < 1) {
        set_error("null tensor or non-positive extent");
        return CONVIO_EINVAL;
    }
    return launch_transpose(x, y, n, c, h * w, true, (cudaStream_t)stream);
}

int convio_nhwc_to_nchw(const float *x, float *y, int32_t n, int32_t c, int32_t h, int32_t w, void *stream) {
    clear_error();
    reset_launches();
    if (!x || !y || n < 1 || c < 1 || h < 1 || w < 1) {
        set_error("null tensor or non-positive extent");
        return CONVIO_EINVAL;
    }
    return launch_transpose(x, y, n, c, h * w, false, (cudaStream_t)stream);
}

int convio_maxpool2x2_nhwc(const float *x, float *y, int32_t n, int32_t h, int32_t w, int32_t c, void *stream) {
    clear_error();
    reset_launches();
    if (!x || !y || n < 1 || h < 2 || w < 2 || c < 4 || c % 4) {
        set_error("maxpool2x2_nhwc needs C %% 4 == 0 and H, W >= 2");
        return CONVIO_EINVAL;
    }
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) {
        set_error("maxpool2x2_nhwc needs 16-byte aligned tensors");
        return CONVIO_EINVAL;
    }
    const int64_t total4 = (int64_t)n * (h / 2) * (w / 2) * (c / 4);
    CONVIO_CUDA_TRY(launch_pdl(maxpool2x2_nhwc_kernel, dim3(grid_for(total4)), dim3(256), 0, (cudaStream_t)stream,
                               x, y, (int)h, (int)w, (int)c, total4));
    note_launch();
    CONVIO_CUDA_TRY(cudaGetLastError());
    return CONVIO_OK;
}

}  // extern "C"
