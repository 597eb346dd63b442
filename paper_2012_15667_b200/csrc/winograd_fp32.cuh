// Fused Winograd F(e x e, 3 x 3), FP32 on CUDA cores: the paper's Winograd
// dataflow (reference pkg/src/convio/dataflow.py:253-310, DAG steps
// dag.py:358-401) with the transformed tiles kept on chip.
//
// Block  = an x*y*z output sub-block: NPOS = (x/e)(y/e) tile positions.
// Stage  = ck input channels: (x+2)(y+2) input footprint (zero-filled halo)
//          and the m^2*ck*z transformed-filter slice U in an NS-deep smem
//          ring: TMA (4-D input box + 3-D U box, mbarrier complete_tx) when
//          the strides allow, else a cp.async ring.
// Step 1 = input transform V = B^T d B of every (channel, position) into a
//          double-buffered smem V (the kernel transform is shared: U from
//          convio_winograd_filter_transform, i.e. shared_kernel_transform);
//          one block barrier per stage.
// Step 2+3 = m^2 independent GEMMs accumulated over channels in registers:
//          the (xi, position group of TP, z group of TZ) units are dealt
//          round-robin to the block's threads (UPT units each), so any thread
//          count projects -- the accumulators are the "first temporary array"
//          of the paper's schedule.
// Step 4 = after the last channel the accumulators go through smem and each
//          (z, position) gets A^T Pi A, + bias/ReLU, stored to HBM.
#pragma once

#include "direct_fp32.cuh"   // mbarrier / TMA primitives

namespace convio {

struct WinoParams {
    const float *x;
    const float *u;       // [m*m][c][k]
    const float *bias;
    float *y;
    int n, c, h, w, k, p, q, pad, layout;
    ActStrides xs, ys;
    int bx, by, bz;       // block output tile
    int px, npos;         // positions per row, positions per block
    int npg;              // position groups (npos / TP)
    int nzg;              // z groups (bz / TZ)
    int units;            // m^2 * npg * nzg GEMM units, round-robin over threads
    int ck, stages;
    int tile_w, tile_h, pitch;
    int in_stage, u_stage;   // floats per stage
    int u_pitch;             // floats per (cc, xi) row of U in smem (>= bz)
    int v_pitch;             // floats per (cc, xi) row of V in smem (>= npos)
    int v_floats;            // ck * m*m * v_pitch
    int o_pitch;             // floats per (xi, z) row of the exchange buffer
    int tiles_x, tiles_y;
    int relu;
    int use_tma;
    int in_box_bytes, u_box_bytes;
    int bar_off;             // float offset of the mbarriers in smem
};

template <int E>
struct WinoMats;

// Lavin & Gray F(2x2, 3x3)
template <>
struct WinoMats<2> {
    static constexpr int M = 4;
    __device__ static void input(const float d[4][4], float v[4][4]) {
        float t[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            t[0][j] = d[0][j] - d[2][j];
            t[1][j] = d[1][j] + d[2][j];
            t[2][j] = d[2][j] - d[1][j];
            t[3][j] = d[1][j] - d[3][j];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[i][0] = t[i][0] - t[i][2];
            v[i][1] = t[i][1] + t[i][2];
            v[i][2] = t[i][2] - t[i][1];
            v[i][3] = t[i][1] - t[i][3];
        }
    }
    __device__ static void output(const float m[4][4], float y[2][2]) {
        float t[2][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            t[0][j] = m[0][j] + m[1][j] + m[2][j];
            t[1][j] = m[1][j] - m[2][j] - m[3][j];
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            y[i][0] = t[i][0] + t[i][1] + t[i][2];
            y[i][1] = t[i][1] - t[i][2] - t[i][3];
        }
    }
};

// Lavin & Gray F(4x4, 3x3)
template <>
struct WinoMats<4> {
    static constexpr int M = 6;
    __device__ static void bt_col(const float *d, int s, float *o, int so) {
        // o = B^T d along one axis; B^T rows:
        // [4 0 -5 0 1 0] [0 -4 -4 1 1 0] [0 4 -4 -1 1 0] [0 -2 -1 2 1 0] [0 2 -1 -2 1 0] [0 4 0 -5 0 1]
        const float d0 = d[0], d1 = d[s], d2 = d[2 * s], d3 = d[3 * s], d4 = d[4 * s], d5 = d[5 * s];
        o[0] = fmaf(4.0f, d0, fmaf(-5.0f, d2, d4));
        o[so] = fmaf(-4.0f, d1 + d2, d3 + d4);
        o[2 * so] = fmaf(4.0f, d1 - d2, d4 - d3);
        o[3 * so] = fmaf(2.0f, d3 - d1, d4 - d2);
        o[4 * so] = fmaf(2.0f, d1 - d3, d4 - d2);
        o[5 * so] = fmaf(4.0f, d1, fmaf(-5.0f, d3, d5));
    }
    __device__ static void input(const float d[6][6], float v[6][6]) {
        float t[6][6];
#pragma unroll
        for (int j = 0; j < 6; ++j) bt_col(&d[0][j], 6, &t[0][j], 6);
#pragma unroll
        for (int i = 0; i < 6; ++i) bt_col(&t[i][0], 1, &v[i][0], 1);
    }
    __device__ static void at_col(const float *m, int s, float *o, int so) {
        // A^T rows: [1 1 1 1 1 0] [0 1 -1 2 -2 0] [0 1 1 4 4 0] [0 1 -1 8 -8 1]
        const float m0 = m[0], m1 = m[s], m2 = m[2 * s], m3 = m[3 * s], m4 = m[4 * s], m5 = m[5 * s];
        const float a = m1 + m2, b = m1 - m2, c = m3 + m4, dd = m3 - m4;
        o[0] = m0 + a + c;
        o[so] = fmaf(2.0f, dd, b);
        o[2 * so] = fmaf(4.0f, c, a);
        o[3 * so] = fmaf(8.0f, dd, b) + m5;
    }
    __device__ static void output(const float m[6][6], float y[4][4]) {
        float t[4][6];
#pragma unroll
        for (int j = 0; j < 6; ++j) at_col(&m[0][j], 6, &t[0][j], 6);
#pragma unroll
        for (int i = 0; i < 4; ++i) at_col(&t[i][0], 1, &y[i][0], 1);
    }
};

template <int E, int TZ, int TP, int UPT>
__global__ void winograd_f32_kernel(const __grid_constant__ WinoParams P,
                                    const __grid_constant__ CUtensorMap tm_in,
                                    const __grid_constant__ CUtensorMap tm_u) {
    constexpr int M = E + 2;
    constexpr int MM = M * M;
    extern __shared__ __align__(128) float smem[];
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;

    const int k0 = blockIdx.x * P.bz;
    const int xt = blockIdx.y % P.tiles_x;
    const int yt = blockIdx.y / P.tiles_x;
    const int img = blockIdx.z;
    const int ox0 = xt * P.bx, oy0 = yt * P.by;
    const int iy0 = oy0 - P.pad;
    const int ix0 = ox0 - P.pad;
    const int shift = ((ix0 % 4) + 4) % 4;   // staged rows start 16-byte aligned
    const int ix0a = ix0 - shift;
    const int stage_w = P.tile_w + shift;

    const int NS = P.stages;
    float *in_s = smem;
    float *u_s = in_s + NS * P.in_stage;
    float *v_s = u_s + NS * P.u_stage;          // 2 buffers of v_floats
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + P.bar_off);
    uint64_t *empty = full + NS;
    const int nwarps = (nthr + 31) >> 5;
    const float *xb = P.x + (int64_t)img * P.xs.n;
    const int nchunks = (P.c + P.ck - 1) / P.ck;
    const uint64_t map_in = reinterpret_cast<uint64_t>(&tm_in);
    const uint64_t map_u = reinterpret_cast<uint64_t>(&tm_u);

    auto tma_issue = [&](int chunk, int slot) {   // one thread
        uint64_t *bar = full + slot;
        mbar_arrive_expect_tx(bar, P.in_box_bytes + P.u_box_bytes);
        tma_load_4d(in_s + slot * P.in_stage, map_in, ix0a, iy0, chunk * P.ck, img, bar);
        tma_load_3d(u_s + slot * P.u_stage, map_u, k0, chunk * P.ck, 0, bar);
    };
    auto cp_issue = [&](int chunk, int slot) {    // all threads
        const int c0 = chunk * P.ck;
        float *din = in_s + slot * P.in_stage;
        const int total = P.ck * P.tile_h * stage_w;
        for (int i = tid; i < total; i += nthr) {
            int cc, r, col;
            if (P.layout == CONVIO_LAYOUT_HWC) {
                cc = i % P.ck;
                const int t = i / P.ck;
                col = t % stage_w;
                r = t / stage_w;
            } else if (P.layout == CONVIO_LAYOUT_CWH) {
                r = i % P.tile_h;
                const int t = i / P.tile_h;
                col = t % stage_w;
                cc = t / stage_w;
            } else {
                col = i % stage_w;
                const int t = i / stage_w;
                r = t % P.tile_h;
                cc = t / P.tile_h;
            }
            const int gc = c0 + cc, gy = iy0 + r, gx = ix0a + col;
            const bool v = gc < P.c && gy >= 0 && gy < P.h && gx >= 0 && gx < P.w;
            const float *src = v ? xb + gc * P.xs.c + gy * P.xs.y + gx * P.xs.x : P.x;
            cp_async4(din + (cc * P.tile_h + r) * P.pitch + col, src, v);
        }
        // U slice -> [xi][cc][z] (the TMA box layout)
        float *du = u_s + slot * P.u_stage;
        const int rows = MM * P.ck;
        if ((P.bz & 3) == 0 && (P.k & 3) == 0) {
            const int per_row = P.bz >> 2;
            const int tot = rows * per_row;
            for (int i = tid; i < tot; i += nthr) {
                const int row = i / per_row, j = (i - row * per_row) << 2;
                const int xi = row / P.ck, cc = row - xi * P.ck;
                const int gc = c0 + cc;
                const bool v = gc < P.c;
                const float *src = v ? P.u + ((int64_t)xi * P.c + gc) * P.k + k0 + j : P.u;
                cp_async16(du + row * P.bz + j, src, v);
            }
        } else {
            const int tot = rows * P.bz;
            for (int i = tid; i < tot; i += nthr) {
                const int row = i / P.bz, j = i - row * P.bz;
                const int xi = row / P.ck, cc = row - xi * P.ck;
                const int gc = c0 + cc;
                const bool v = gc < P.c;
                const float *src = v ? P.u + ((int64_t)xi * P.c + gc) * P.k + k0 + j : P.u;
                cp_async4(du + row * P.bz + j, src, v);
            }
        }
    };

    // step 1: V[cc][xi][pos] = (B^T d B)[xi] for every (channel, position)
    auto transform_inputs = [&](int slot, float *vbuf) {
        const float *din = in_s + slot * P.in_stage + shift;
        const int tasks = P.ck * P.npos;
        for (int t = tid; t < tasks; t += nthr) {
            const int cc = t / P.npos, pos = t - cc * P.npos;
            const int py = pos / P.px, pxx = pos - py * P.px;
            const float *src = din + (cc * P.tile_h + py * E) * P.pitch + pxx * E;
            float d[M][M], v[M][M];
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
                for (int j = 0; j < M; ++j) d[i][j] = src[i * P.pitch + j];
            WinoMats<E>::input(d, v);
            float *dst = vbuf + cc * MM * P.v_pitch + pos;
#pragma unroll
            for (int i = 0; i < M; ++i)
#pragma unroll
                for (int j = 0; j < M; ++j) dst[(i * M + j) * P.v_pitch] = v[i][j];
        }
    };

    // GEMM units: u = zg + nzg * (pg + npg * xi); thread t owns u = t + j*nthr
    int u_xi[UPT], u_z[UPT], u_p[UPT];
    bool u_ok[UPT];
#pragma unroll
    for (int j = 0; j < UPT; ++j) {
        const int u = tid + j * nthr;
        u_ok[j] = u < P.units;
        const int uu = u_ok[j] ? u : 0;
        const int zg = uu % P.nzg;
        const int rest = uu / P.nzg;
        u_z[j] = zg * TZ;
        u_p[j] = (rest % P.npg) * TP;
        u_xi[j] = rest / P.npg;
    }

    float acc[UPT][TZ][TP];
#pragma unroll
    for (int j = 0; j < UPT; ++j)
#pragma unroll
        for (int a = 0; a < TZ; ++a)
#pragma unroll
            for (int b = 0; b < TP; ++b) acc[j][a][b] = 0.0f;

    // steps 2+3: acc[z][pos] += U[xi][cc][z] * V[cc][xi][pos]
    auto gemm = [&](int slot, const float *vbuf) {
        const float *ub = u_s + slot * P.u_stage;
        const int vstep = MM * P.v_pitch;
#pragma unroll
        for (int j = 0; j < UPT; ++j) {
            if (!u_ok[j]) continue;
            const float *us = ub + u_xi[j] * P.ck * P.bz + u_z[j];
            const float *vs = vbuf + u_xi[j] * P.v_pitch + u_p[j];
#pragma unroll 4
            for (int cc = 0; cc < P.ck; ++cc) {
                float ur[TZ], vr[TP];
                if constexpr (TZ % 4 == 0) {
#pragma unroll
                    for (int q = 0; q < TZ; q += 4) {
                        const float4 t = *reinterpret_cast<const float4 *>(us + cc * P.bz + q);
                        ur[q] = t.x; ur[q + 1] = t.y; ur[q + 2] = t.z; ur[q + 3] = t.w;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < TZ; ++q) ur[q] = us[cc * P.bz + q];
                }
                if constexpr (TP % 4 == 0) {
#pragma unroll
                    for (int q = 0; q < TP; q += 4) {
                        const float4 t = *reinterpret_cast<const float4 *>(vs + cc * vstep + q);
                        vr[q] = t.x; vr[q + 1] = t.y; vr[q + 2] = t.z; vr[q + 3] = t.w;
                    }
                } else if constexpr (TP % 2 == 0) {
#pragma unroll
                    for (int q = 0; q < TP; q += 2) {
                        const float2 t = *reinterpret_cast<const float2 *>(vs + cc * vstep + q);
                        vr[q] = t.x; vr[q + 1] = t.y;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < TP; ++q) vr[q] = vs[cc * vstep + q];
                }
#pragma unroll
                for (int a = 0; a < TZ; ++a)
#pragma unroll
                    for (int b = 0; b < TP; ++b) acc[j][a][b] = fmaf(ur[a], vr[b], acc[j][a][b]);
            }
        }
    };

    if (P.use_tma) {
        if (tid == 0) {
            for (int s2 = 0; s2 < NS; ++s2) {
                mbar_init(full + s2, 1);
                mbar_init(empty + s2, nwarps);
            }
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0)
            for (int s2 = 0; s2 < NS - 1 && s2 < nchunks; ++s2) tma_issue(s2, s2);
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            const int slot = chunk % NS;
            float *vbuf = v_s + (chunk & 1) * P.v_floats;
            mbar_wait(full + slot, (chunk / NS) & 1);
            transform_inputs(slot, vbuf);
            __syncthreads();   // V[chunk&1] complete; V[(chunk-1)&1] readers done
            gemm(slot, vbuf);
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(empty + slot);
            const int next = chunk + NS - 1;
            if (tid == 0 && next < nchunks) {
                const int nslot = next % NS;
                if (next >= NS) mbar_wait(empty + nslot, ((next / NS) - 1) & 1);
                tma_issue(next, nslot);
            }
        }
    } else {
        const int pre = NS > 1 ? NS - 1 : 1;
        for (int s2 = 0; s2 < pre; ++s2) {
            if (s2 < nchunks) cp_issue(s2, s2);
            cp_async_commit();
        }
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            float *vbuf = v_s + (chunk & 1) * P.v_floats;
            if (NS >= 3) cp_async_wait<1>();
            else cp_async_wait<0>();
            __syncthreads();   // chunk landed for all; slot (chunk-1)%NS and V buffers free
            if (NS >= 2) {
                const int next = chunk + NS - 1;
                if (next < nchunks) cp_issue(next, next % NS);
                cp_async_commit();
            }
            transform_inputs(chunk % NS, vbuf);
            __syncthreads();
            gemm(chunk % NS, vbuf);
            if (NS == 1) {
                __syncthreads();
                if (chunk + 1 < nchunks) cp_issue(chunk + 1, 0);
                cp_async_commit();
            }
        }
    }
    __syncthreads();

    // step 4: exchange through smem O[xi][z][pos], then A^T Pi A per (z, pos)
    float *o_s = smem;
#pragma unroll
    for (int j = 0; j < UPT; ++j) {
        if (!u_ok[j]) continue;
#pragma unroll
        for (int a = 0; a < TZ; ++a) {
            float *dst = o_s + (u_xi[j] * P.bz + u_z[j] + a) * P.o_pitch + u_p[j];
#pragma unroll
            for (int b = 0; b < TP; ++b) dst[b] = acc[j][a][b];
        }
    }
    __syncthreads();
    float *yb = P.y + (int64_t)img * P.ys.n;
    const int tasks = P.bz * P.npos;
    for (int t = tid; t < tasks; t += nthr) {
        const int zz = t / P.npos, pos = t - zz * P.npos;
        const int py = pos / P.px, pxx = pos - py * P.px;
        float m[M][M], out[E][E];
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) m[i][j] = o_s[((i * M + j) * P.bz + zz) * P.o_pitch + pos];
        WinoMats<E>::output(m, out);
        const int kk = k0 + zz;
        const float b = P.bias ? __ldg(P.bias + kk) : 0.0f;
        const int oy = oy0 + py * E, ox = ox0 + pxx * E;
        float *dst = yb + kk * P.ys.c + oy * P.ys.y + ox * P.ys.x;
#pragma unroll
        for (int i = 0; i < E; ++i)
#pragma unroll
            for (int j = 0; j < E; ++j) {
                float v = out[i][j] + b;
                if (P.relu) v = fmaxf(v, 0.0f);
                dst[i * P.ys.y + j * P.ys.x] = v;
            }
    }
}

using WinoKernelFn = void (*)(const WinoParams, const CUtensorMap, const CUtensorMap);
WinoKernelFn find_winograd_kernel(int e, int tz, int tp, int upt);

int winograd_query(const convio_conv_desc *d, const convio_tile *t, convio_launch_info *out);
int64_t winograd_workspace_bytes(const convio_conv_desc *d, const convio_tile *t);

}  // namespace convio
