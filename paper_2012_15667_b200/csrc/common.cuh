// Shared device/host helpers for the convio_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/convio_b200.h"

namespace convio {

// ---- error plumbing (thread-local message, codes from convio_b200.h) -------
void set_error(const char *fmt, ...);
void clear_error();   // also resets the error kind to CONVIO_EKIND_NONE
// rc CONVIO_EINFEASIBLE with the reference exception class recorded explicitly
// (convio_last_error_kind): the reference's ScheduleError (dataflow.py:30,
// raised by the planners for a tile that does not divide the output or a
// resident set above s_b, dataflow.py:222-233,263-279) and GeometryError
// (model.py:14: kernel larger than the padded input, non-unit Winograd stride)
int schedule_error();
int geometry_error();
void note_launch();
void reset_launches();

// Blocks of `fn` that fit one SM with this launch shape (cached per
// (fn, threads, smem)); sets *regs.  Returns 1 without checking when no
// device is present (CPU-only legality queries).
int launch_fit(const void *fn, int threads, size_t smem, int *regs);
// Same for a cluster (CTA-pair) kernel: 1 if one block fits an SM.
int launch_fit_cluster(const void *fn, int threads, size_t smem, int *regs);
// SMs of the current device (148 without a device).
int device_sms();
// Registers per thread of a kernel (cached); 0 without a device.
int kernel_regs(const void *fn);

struct Status {
    int code;
};

#define CONVIO_CUDA_TRY(expr)                                                     \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) {                                                  \
            ::convio::set_error("%s failed: %s", #expr, cudaGetErrorString(_e)); \
            return CONVIO_EINTERNAL;                                              \
        }                                                                         \
    } while (0)

// ---- programmatic dependent launch --------------------------------------------
// Kernels launched through launch_pdl() may be launched while the previous kernel
// on the stream drains its last blocks, so block launch and the prologue (barrier
// init, TMEM allocation, descriptor prefetch) overlap that tail.  Every such
// kernel calls pdl_wait() before its first global-memory access:
// griddepcontrol.wait returns when the preceding grid has completed and its
// writes are visible.  Measured (bench.py, CONVIO_PDL=0/1): batch 32 step 0.695
// -> 0.676 ms, batch 256 unchanged.  An explicit griddepcontrol.launch_dependents
// at kernel entry (dependents launch once all blocks run) made batch 256 5 %
// slower (3.23 -> 3.40 ms): the waiting blocks of the next kernel sit on SMs the
// current kernel's tail could use.  CONVIO_PDL=0 launches them plainly.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---- layouts ------------------------------------------------------------------
// Element strides of an activation tensor [n][c][h][w] stored in `layout`.
struct ActStrides {
    int64_t n, c, y, x;
};

__host__ __device__ inline ActStrides act_strides(int layout, int c, int h, int w) {
    ActStrides s;
    s.n = (int64_t)c * h * w;
    if (layout == CONVIO_LAYOUT_HWC) {        // n h w c
        s.c = 1; s.x = c; s.y = (int64_t)w * c;
    } else if (layout == CONVIO_LAYOUT_CWH) { // n c w h
        s.y = 1; s.x = h; s.c = (int64_t)h * w;
    } else {                                  // n c h w
        s.x = 1; s.y = w; s.c = (int64_t)h * w;
    }
    return s;
}

// ---- cp.async (LDGSTS) helpers ------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 4-byte async copy; src_bytes = 0 zero-fills (halo / channel tail).
__device__ __forceinline__ void cp_async4(void *dst, const void *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(valid ? 4 : 0));
}

// 16-byte async copy (bypasses L1); src_bytes = 0 zero-fills.
__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(valid ? 16 : 0));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

}  // namespace convio
