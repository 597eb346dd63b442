/*
 * convio_b200 -- C-ABI of the B200 (sm_100a) convolution dataflow kernels.
 *
 * The reference package (arxiv 2012.15667 "convio", pure Python) has no FFI:
 * its "execution" of a dataflow is the word-counting simulator.  This ABI is
 * the device boundary *below* the reference's Python API:
 *
 *   reference interface replaced                      entry point here
 *   ----------------------------------------------------------------------
 *   dataflow.simulate(plan_direct_dataflow(...))      convio_conv_direct_f32
 *     pkg/src/convio/dataflow.py:219-250, 316-338       (executes the schedule)
 *   dataflow.simulate(plan_winograd_dataflow(...))    convio_conv_winograd_f32
 *     pkg/src/convio/dataflow.py:253-310, 316-338
 *   shared_kernel_transform=True (J_k shared)         convio_winograd_filter_transform
 *     pkg/src/convio/dataflow.py:273, dag.py:353-383
 *   autotune.measure -> legality of a TileConfig      convio_query
 *     pkg/src/convio/autotune.py:173-190 (ScheduleError/InfeasibleTileError)
 *
 * Conventions
 *   - Plain pointers and sizes only.  All device buffers (x, w, y, workspace)
 *     are allocated by the caller; the library never allocates in the hot path
 *     and keeps no pointer after return.  `stream` is a cudaStream_t (NULL =
 *     legacy default stream); all work is ordered on it.  Calls are reentrant.
 *   - Activations are fp32 in the layout named by `layout`:
 *       CONVIO_LAYOUT_CHW = NCHW, CONVIO_LAYOUT_CWH = N C W H (x outer, y inner),
 *       CONVIO_LAYOUT_HWC = NHWC (the reference's LAYOUTS axis,
 *       pkg/src/convio/dataflow.py:23).  Output uses the same layout.
 *   - Filters are fp32 KCRS (reference index map wt[oc, c, ky, kx],
 *     pkg/src/convio/dag.py:262-267).
 *   - Padding is zero-filled in the kernel (no padded copy is made).
 *   - Return codes mirror the reference CLI's exit classes
 *     (pkg/src/convio/cli.py:472-485):
 *       0 OK, 2 invalid argument, 3 geometry / infeasible tile / capacity,
 *       4 CUDA or internal error.  convio_last_error() gives the message
 *       (thread-local, valid until the next call on the same thread).
 */
#ifndef CONVIO_B200_H
#define CONVIO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CONVIO_OK 0
#define CONVIO_EINVAL 2
#define CONVIO_EINFEASIBLE 3
#define CONVIO_EINTERNAL 4

/* Reference exception class of the last rc-3 failure (convio_last_error_kind):
 * the Python binding raises exactly this class, never guessing from the text. */
#define CONVIO_EKIND_NONE 0
#define CONVIO_EKIND_SCHEDULE 1    /* dataflow.ScheduleError (pkg/src/convio/dataflow.py:30) */
#define CONVIO_EKIND_INFEASIBLE 2  /* dataflow.InfeasibleTileError (pkg/src/convio/dataflow.py:26) */
#define CONVIO_EKIND_GEOMETRY 3    /* model.GeometryError (pkg/src/convio/model.py:14) */

#define CONVIO_LAYOUT_CHW 0
#define CONVIO_LAYOUT_CWH 1
#define CONVIO_LAYOUT_HWC 2

#define CONVIO_ALG_DIRECT 0
#define CONVIO_ALG_WINOGRAD 1
#define CONVIO_ALG_IGEMM_TF32 2   /* tcgen05 implicit GEMM, TF32 in / FP32 accumulate */
#define CONVIO_ALG_IGEMM_3XTF32 3 /* tcgen05 implicit GEMM, 3xTF32 split: FP32-level accuracy */
#define CONVIO_ALG_IGEMM_BF16 4   /* tcgen05 implicit GEMM, BF16 operands / FP32 accumulate */
#define CONVIO_ALG_WINOGRAD_TC_TF32 5   /* Winograd, element-wise GEMMs on tcgen05 (TF32) */
#define CONVIO_ALG_WINOGRAD_TC_3XTF32 6 /* ... 3xTF32 (FP32-level GEMM accuracy) */
#define CONVIO_ALG_WINOGRAD_TC_BF16 7   /* ... BF16 transformed operands */
#define CONVIO_ALG_WINOGRAD_NHWC 8      /* same pipeline, element-wise GEMMs as a batched FP32 FFMA GEMM */
#define CONVIO_ALG_WINOGRAD_TC_3XF16 9  /* ... scaled fp16 hi / lo planes, 3 f16 MMAs (FP32-level) */
#define CONVIO_ALG_IGEMM_3XF16 10       /* tcgen05 implicit GEMM, 3xF16 split (FP32-level, f16 rate) */

/* Operand precision of the tcgen05 contractions (FP32 accumulate always). */
#define CONVIO_PREC_TF32 0
#define CONVIO_PREC_3XTF32 1
#define CONVIO_PREC_BF16 2
#define CONVIO_PREC_FP32 3   /* convio_winograd_bgemm only: FP32 FFMA GEMMs on the CUDA cores */
#define CONVIO_PREC_3XF16 4  /* operands split into power-of-two-scaled fp16 hi / lo planes
                                (22-bit, like 3xTF32), 3 MMAs at the f16 rate; C % 64 == 0,
                                CTA pair tiles.  convio_winograd_bgemm: split by the transforms
                                (one scale per tile row / filter row); convio_conv_igemm: the
                                activations split in shared memory with one scale per tensor
                                (an |x| max pass first), the filter per output channel */

/* One convolution layer (valid geometry after zero padding `pad`). */
typedef struct convio_conv_desc {
    int32_t n, c, h, w;   /* batch, input channels, input height, width (unpadded) */
    int32_t k, r, s;      /* output channels, kernel height, kernel width */
    int32_t stride, pad;
    int32_t layout;       /* CONVIO_LAYOUT_* */
} convio_conv_desc;

/* Mirrors TileConfig (pkg/src/convio/dataflow.py:34-76); e = 0 for None. */
typedef struct convio_tile {
    int32_t x, y, z, s_b;
    int32_t n_xt, n_yt, n_zt;
    int32_t layout;
    int32_t e;
} convio_tile;

/* Device projection of a tile: what convio_conv_* would launch. */
typedef struct convio_launch_info {
    int32_t legal;              /* 1 if launchable, else reason[] says why */
    int32_t grid_x, grid_y, grid_z;
    int32_t block_threads;
    int32_t smem_bytes;         /* dynamic shared memory per block */
    int32_t regs_per_thread;    /* from cudaFuncGetAttributes (0 if unknown) */
    int32_t channel_chunk;      /* input channels per pipeline stage (paper alpha) */
    int32_t stages;             /* pipeline depth */
    int32_t smem_pitch;         /* padded row pitch of the staged input tile */
    int32_t p, q;               /* output height, width */
    int64_t flops;              /* algorithmic flops of the launch */
    int64_t workspace_bytes;    /* workspace the call needs */
    char reason[160];
} convio_launch_info;

int convio_version(void);
const char *convio_last_error(void);
/* CONVIO_EKIND_* of the last failure on this thread (valid with convio_last_error). */
int convio_last_error_kind(void);

/* Legality + launch shape of (desc, tile, algorithm); never launches. */
int convio_query(const convio_conv_desc *desc, const convio_tile *tile, int32_t algorithm,
                 convio_launch_info *out);

/* The tile convio_conv_* uses when called with tile == NULL. */
int convio_default_tile(const convio_conv_desc *desc, int32_t algorithm, int32_t e,
                        convio_tile *out);

/* Workspace bytes for convio_conv_* with this tile (packed / transformed filters). */
int64_t convio_workspace_bytes(const convio_conv_desc *desc, const convio_tile *tile,
                               int32_t algorithm);

/* Repack KCRS filters to the direct kernel's C R S K layout (ws >= K*C*R*S floats). */
int convio_pack_filter_direct(const convio_conv_desc *desc, const float *w, float *w_packed,
                              void *stream);

/* Direct convolution y = conv(x, w), the output-stationary dataflow
 * (x*y*z outputs per block resident in registers, channel stages through
 * shared memory).  tile == NULL picks the default device tile.  If
 * `w_is_packed` the filter is already in convio_pack_filter_direct layout. */
int convio_conv_direct_f32(const convio_conv_desc *desc, const convio_tile *tile,
                           const float *x, const float *w, int32_t w_is_packed,
                           const float *bias, int32_t relu, float *y,
                           void *workspace, size_t workspace_bytes, void *stream);

/* Winograd filter transform U[xi][c][k] = (G g G^T)[xi] for F(e x e, r x r). */
int convio_winograd_filter_transform(const convio_conv_desc *desc, int32_t e, const float *w,
                                     float *u, void *stream);

/* Fused Winograd F(e x e, 3 x 3): input transform, element-wise batched GEMM
 * over channels, output transform in one kernel, transformed tiles on chip.
 * If `w_is_transformed`, w holds U from convio_winograd_filter_transform. */
int convio_conv_winograd_f32(const convio_conv_desc *desc, const convio_tile *tile, int32_t e,
                             const float *x, const float *w, int32_t w_is_transformed,
                             const float *bias, int32_t relu, float *y,
                             void *workspace, size_t workspace_bytes, void *stream);

/* Repack KCRS filters to [R*S][K][C] for the tcgen05 implicit GEMM. */
int convio_pack_filter_igemm(const convio_conv_desc *desc, const float *w, float *w_packed,
                             void *stream);

/* Direct convolution as an implicit GEMM on the 5th-gen tensor cores
 * (tcgen05.mma kind::tf32, accumulators in TMEM, TMA SWIZZLE_128B operand
 * staging).  NHWC (CONVIO_LAYOUT_HWC) activations, C % 32 == 0, stride 1,
 * tile z in {64,128,256}, x*y <= 128 (ceil(128/(x*y)) images stacked per MMA
 * tile).  tile->n_zt selects the kernel: 1 = one 128-row tile per CTA,
 * 2 = persistent CTA pair (cta_group::2, M = 256, each CTA stages z/2 filter
 * rows, double-buffered TMEM accumulators), 4 = the pair with the 3xTF32 A
 * operand split into TMEM (z <= 128); n_xt = 2 (with n_zt = 2, stride 1):
 * halo-staged input footprint; otherwise n_xt = n_yt = 1.  Inputs are consumed at TF32 precision, accumulation is FP32.
 * Replaces the same schedule as convio_conv_direct_f32 (dataflow.py:219-250). */
int convio_conv_igemm_tf32(const convio_conv_desc *desc, const convio_tile *tile, const float *x,
                           const float *w, int32_t w_is_packed, const float *bias, int32_t relu,
                           float *y, void *workspace, size_t workspace_bytes, void *stream);

/* Same implicit GEMM with each operand split into hi = rna_tf32(v) and
 * lo = v - hi (3 MMAs per k-step: hi*lo + lo*hi + hi*hi): FP32-level
 * accuracy on the tensor cores.  z in {64, 128}. */
int convio_conv_igemm_3xtf32(const convio_conv_desc *desc, const convio_tile *tile, const float *x,
                             const float *w, int32_t w_is_packed, const float *bias, int32_t relu,
                             float *y, void *workspace, size_t workspace_bytes, void *stream);

/* Generic form of the two calls above plus BF16 and 3xF16 (CONVIO_PREC_*).  For
 * BF16 the fp32 activations are converted to bf16 NHWC in the workspace first
 * (C % 64 == 0), filters packed to bf16 [R*S][K][C] unless `w_is_packed`
 * (then w holds convio_pack_filter_igemm_bf16 output).  For 3xF16 (CTA pair
 * tiles, C % 64 == 0) the workspace (256-byte aligned) starts with the
 * activation-scale state and, unless `w_is_packed` (convio_pack_filter_igemm_f16x3
 * output), holds the packed filter; the activations stay fp32 in HBM and are split
 * on chip with one power-of-two scale per tensor.  That scale is speculated from the
 * max |x| the previous call on the SAME workspace observed; every call checks it on
 * the device (a second launch) and redoes the conv with the exact scale when it
 * would overflow fp16 or lose precision, so results never depend on the state --
 * reusing a layer's workspace across calls only makes them faster (any bytes,
 * e.g. a fresh or foreign workspace, mean "no speculation").  Two launches per
 * call; not reentrant on one workspace.  Replaces the same schedule as
 * convio_conv_direct_f32 (dataflow.py:219-250). */
int convio_conv_igemm(const convio_conv_desc *desc, const convio_tile *tile, int32_t precision,
                      const float *x, const void *w, int32_t w_is_packed, const float *bias,
                      int32_t relu, float *y, void *workspace, size_t workspace_bytes, void *stream);

/* KCRS fp32 -> the 3xF16 filter operand of convio_conv_igemm (CONVIO_PREC_3XF16):
 * fp16 hi / lo planes [2][R*S][K][C] scaled by 2^e[k] per output channel, then
 * e[K] (int32) at byte offset align256(4*K*C*R*S); w_packed 256-byte aligned and
 * convio_pack_filter_igemm_f16x3_bytes(desc) long.  Replaces the filter side of
 * the same schedule (dataflow.py:219-250). */
int convio_pack_filter_igemm_f16x3(const convio_conv_desc *desc, const float *w, void *w_packed,
                                   void *stream);
/* The same for `count` <= 32 filters in ONE launch (a step's filter prep: the
 * per-filter launches each occupied only K blocks of the GPU).  Arrays of
 * descriptors, KCRS filters and 256-byte aligned outputs; same layout per job. */
/* `layers` independent 3xF16 convolutions of ONE shape and tile (desc->n images each)
 * in one persistent launch: x / y stacked along N (layers * n images), the packed
 * filters (convio_pack_filter_igemm_f16x3) as 256-byte aligned slices `layer_bytes`
 * apart, bias layers x K (or null), one activation-scale state for the group.  The
 * tile's image stack must divide n; the same schedule per layer as convio_conv_igemm
 * (dataflow.py:219-250), grouped like a grouped GEMM. */
int convio_conv_igemm_grouped(const convio_conv_desc *desc, const convio_tile *tile, int32_t precision,
                              int32_t layers, const float *x, const void *w_packed, size_t layer_bytes,
                              const float *bias, int32_t relu, float *y, void *workspace, size_t workspace_bytes,
                              void *stream);
/* The tensor-core Winograd filter transform (convio_winograd_filter_transform_tc) of
 * `count` <= 32 filters of one e and one precision in one launch; fp32-U precisions
 * (TF32, 3xTF32, 3xF16).  3xF16 (even C) writes the fp16 hi / lo planes and exponents
 * in one pass -- bit-identical to the per-filter transform + split -- and leaves the
 * fp32 U region of the buffer unwritten (the GEMM never reads it). */
int convio_winograd_filter_transform_tc_batched(int32_t count, const convio_conv_desc *descs, int32_t e,
                                                int32_t precision, const float *const *w, void *const *u,
                                                void *stream);
int convio_pack_filters_igemm_f16x3_batched(int32_t count, const convio_conv_desc *descs, const float *const *w,
                                            void *const *w_packed, void *stream);
int64_t convio_pack_filter_igemm_f16x3_bytes(const convio_conv_desc *desc);

/* KCRS fp32 -> [R*S][K][C] bf16 (round to nearest even). */
int convio_pack_filter_igemm_bf16(const convio_conv_desc *desc, const float *w, void *w_packed,
                                  void *stream);

/* dst[i] = bf16_rne(src[i]), both 16-byte aligned. */
int convio_convert_bf16(const float *src, void *dst, int64_t n, void *stream);

/* Tensor-core Winograd filter transform U[xi][k][c] = (G g G^T)[xi]
 * (fp32 for TF32/3xTF32, bf16 for BF16) -- the shared kernel transform
 * (dataflow.py:273 shared_kernel_transform=True, dag.py:353-383). */
int convio_winograd_filter_transform_tc(const convio_conv_desc *desc, int32_t e, int32_t precision,
                                        const float *w, void *u, void *stream);

/* Winograd F(e x e, 3 x 3), e in {2, 4}, with step 3 (the element-wise
 * products summed over channels, dag.py:384-401) as (e+2)^2 batched GEMMs
 * M[xi][t][k] = sum_c V[xi][t][c] U[xi][k][c] on tcgen05 in one launch, and
 * the input/output transforms as HBM-streaming kernels; the batch is run in
 * chunks of V + M <= 16 KB x tile->s_b bytes.  NHWC, stride 1, C % 32 (% 64 for
 * BF16) == 0; precision CONVIO_PREC_FP32 runs the element-wise GEMMs on the
 * CUDA cores (the channels-last FFMA kernel in batched mode, z in {64, 128},
 * U laid out [xi][c][k] as convio_winograd_filter_transform writes it);
 * tile->z in {64,128,256} is the GEMM's N tile, tile->s_b sizes
 * the chunk, tile->n_zt in {1, 2, 4} picks the single-CTA / CTA-pair /
 * CTA-pair-with-A-in-TMEM (3xTF32, z <= 128) GEMM kernel, tile->e must equal
 * e (tile == NULL: defaults).
 * Replaces plan_winograd_dataflow + simulate (dataflow.py:253-338). */
int convio_winograd_bgemm(const convio_conv_desc *desc, const convio_tile *tile, int32_t e,
                          int32_t precision, const float *x, const void *w, int32_t w_is_transformed,
                          const float *bias, int32_t relu, float *y, void *workspace,
                          size_t workspace_bytes, void *stream);

/* The transform matrices the kernels use (row-major AT e*m, G m*r, BT m*m). */
int convio_winograd_matrices(int32_t e, int32_t r, float *at, float *g, float *bt);

/* FP32 FFMA throughput probe (the CUDA-core roofline denominator):
 * runs `iters` FMA chains on every SM; returns flops executed in *flops. */
int convio_ffma_peak(float *sink, int32_t blocks, int32_t iters, int64_t *flops, void *stream);

/* Number of kernel launches the last convio_conv_* call on this thread issued. */
int convio_last_launch_count(void);

/* ---- steps either side of the conv path in a chained network forward ----------
 * (the reference's layout axis CHW / HWC,
 * pkg/src/convio/dataflow.py:23, staged on the device as a counted kernel) */

/* y[n][h][w][c] = x[n][c][h][w] (both fp32, contiguous). */
int convio_nchw_to_nhwc(const float *x, float *y, int32_t n, int32_t c, int32_t h, int32_t w, void *stream);

/* y[n][c][h][w] = x[n][h][w][c]. */
int convio_nhwc_to_nchw(const float *x, float *y, int32_t n, int32_t c, int32_t h, int32_t w, void *stream);

/* 2x2 / stride-2 max pooling of NHWC activations (C % 4 == 0, 16-byte aligned;
 * floor for odd H / W): y is n x h/2 x w/2 x c. */
int convio_maxpool2x2_nhwc(const float *x, float *y, int32_t n, int32_t h, int32_t w, int32_t c, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CONVIO_B200_H */
