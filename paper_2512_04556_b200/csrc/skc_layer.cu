// skc_layer.cu -- uniform sparse-layer kernels (sm_100a).
//
// Reference: engine.apply_sparse_layer (engine.py:160-170) -> sample_shifted
// (118-130) -> _accum_shift (106-115); engine.apply_complex (173-178).
//
// Work decomposition: one CTA = one (output tile, channel) pair, channel-
// fastest grid.  The chain's intermediates are fp32 *planar* (B, C, H, W): the
// first layer reads the caller's HWC image (fp16 inputs go through a relayout
// pass first) and the last writes HWC through the tap kernel's staged
// epilogue (or a relayout pass after a stencil), so every inner layer loads its
// halo tile as contiguous rows with 8-byte cp.async (LDGSTS, zero-fill at the
// image edge; interior tiles take a pointer-increment fast path) and stores
// 8-pixel row segments with 16-byte stores.
//
// Tap path (layer_tap_kernel): a uniform tap is 4 integer shifts with constant
// weights; the host folds each tap into (shared-memory offset of corner 00,
// 4 weights) and sorts taps by offset parity.  Each thread owns a KR x 8
// output block (KR odd); per tap it reads a (KR+1) x 9 window -- 4 LDS.64 +
// 1 LDS.32 per row, bank-conflict free for LDS.64 because the row pitch is
// 2 mod 4 and KR is odd -- and issues 32*KR FFMAs with uniform-register
// weights.  Dense path: when the merged corner footprint fits D x D (D <= 9)
// with D^2 < 4S the host merges coincident corners into a stencil; planar
// inner layers with D >= 7 run it with packed-FP32 FFMA2 on output-row pairs
// (layer_stencil2_kernel), the others with constant-bank FFMA operands
// (layer_stencil_kernel).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include <cooperative_groups.h>

#include "skc_tile.cuh"

namespace skc {

constexpr int kLMaxTaps = 256;

struct TapList {
    float4 cw[kLMaxTaps];  // corner weights (00, 10, 01, 11)
    int off[kLMaxTaps];    // smem offset of corner 00 relative to the thread's block origin
    int ix[kLMaxTaps];     // integer parts (direct kernel)
    int iy[kLMaxTaps];
    int n_even;            // taps [0, n_even) have even offsets, [n_even, n) odd
    int n;
};

struct DenseList {
    float k[kMaxDense * kMaxDense];  // K[a][b] multiplies in[y + dy0 + a][x + dx0' + b]
    int D;
    int col_shift;                   // stencil column 0 relative to the smem tile column of x
};

struct LGeom {
    int H, W, C;
    int dx0, dy0;      // smem (0,0) <-> global (tx0 + dx0, ty0 + dy0); dx0 even
    int pitch, rows;   // pitch = 2 mod 4
    int boundary;
    int accumulate;
};

// ---------------------------------------------------------------- loaders ---
__device__ __forceinline__ void cp_async8(float *dst, const float *src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
                 "r"(valid ? 8 : 0));
}

// Interior-row copies with a compile-time chunk count: per lane NCH chunks of
// E floats at lane stride (E = 2: 8-byte pairs of a planar row; E = 1 with a
// global element stride `gs`: one channel of an HWC row).  Constant offsets
// fold into the LDGSTS address fields.
template <int NCH>
__device__ __forceinline__ void row_pairs(unsigned sd, const float *sx, int lane, int pitch) {
#pragma unroll
    for (int u = 0; u < NCH; ++u)
        if (u < NCH - 1 || 2 * lane + 64 * u < pitch) cp_async8s(sd + 256 * u, sx + 64 * u);
}
template <int NCH>
__device__ __forceinline__ void row_elems(unsigned sd, const float *sx, int lane, int pitch, int gs) {
#pragma unroll
    for (int u = 0; u < NCH; ++u)
        if (u < NCH - 1 || lane + 32 * u < pitch) cp_async4s(sd + 128 * u, sx + (32 * u) * gs);
}
__device__ __forceinline__ void row_pairs_any(unsigned sd, const float *sx, int lane, int pitch) {
    switch ((pitch + 63) >> 6) {
        case 1: row_pairs<1>(sd, sx, lane, pitch); break;
        case 2: row_pairs<2>(sd, sx, lane, pitch); break;
        case 3: row_pairs<3>(sd, sx, lane, pitch); break;
        case 4: row_pairs<4>(sd, sx, lane, pitch); break;
        default:
            for (int col = 2 * lane; col < pitch; col += 64, sd += 256, sx += 64) cp_async8s(sd, sx);
    }
}
__device__ __forceinline__ void row_elems_any(unsigned sd, const float *sx, int lane, int pitch, int gs) {
    switch ((pitch + 31) >> 5) {
        case 3: row_elems<3>(sd, sx, lane, pitch, gs); break;
        case 4: row_elems<4>(sd, sx, lane, pitch, gs); break;
        case 5: row_elems<5>(sd, sx, lane, pitch, gs); break;
        case 6: row_elems<6>(sd, sx, lane, pitch, gs); break;
        default:
            for (int col = lane; col < pitch; col += 32, sd += 128, sx += 32 * gs) cp_async4s(sd, sx);
    }
}

// A whole interior tile (no row or column outside the image): every warp walks
// its rows with pointer increments only; the per-row chunk count is a
// compile-time constant.
template <int NCH, int E>
__device__ __forceinline__ void tile_rows(unsigned sd, const float *sx, int lane, int pitch, int r0, int rows,
                                          int nw, unsigned sstep, long long gstep, int gs) {
    for (int r = r0; r < rows; r += nw, sd += sstep, sx += gstep) {
        if constexpr (E == 2) row_pairs<NCH>(sd, sx, lane, pitch);
        else row_elems<NCH>(sd, sx, lane, pitch, gs);
    }
}
template <int E>
__device__ __forceinline__ bool tile_rows_any(unsigned sd, const float *sx, int lane, int pitch, int r0, int rows,
                                              int nw, unsigned sstep, long long gstep, int gs) {
    const int nch = E == 2 ? (pitch + 63) >> 6 : (pitch + 31) >> 5;
    if constexpr (E == 2) {
        switch (nch) {
            case 2: tile_rows<2, 2>(sd, sx, lane, pitch, r0, rows, nw, sstep, gstep, gs); return true;
            case 3: tile_rows<3, 2>(sd, sx, lane, pitch, r0, rows, nw, sstep, gstep, gs); return true;
            case 4: tile_rows<4, 2>(sd, sx, lane, pitch, r0, rows, nw, sstep, gstep, gs); return true;
            default: return false;
        }
    } else {
        switch (nch) {
            case 3: tile_rows<3, 1>(sd, sx, lane, pitch, r0, rows, nw, sstep, gstep, gs); return true;
            case 4: tile_rows<4, 1>(sd, sx, lane, pitch, r0, rows, nw, sstep, gstep, gs); return true;
            case 5: tile_rows<5, 1>(sd, sx, lane, pitch, r0, rows, nw, sstep, gstep, gs); return true;
            case 6: tile_rows<6, 1>(sd, sx, lane, pitch, r0, rows, nw, sstep, gstep, gs); return true;
            default: return false;
        }
    }
}

// Planar fp16 interior rows: each lane moves NCH half2 pairs of four rows per
// iteration (4 * NCH independent 4-byte loads in flight), widened to fp32
// with 8-byte shared stores.  (A cp.async variant staging the raw pairs
// behind the fp32 tile measured slower on config 3: 1.5x shared memory per
// CTA costs a resident CTA per SM; 19.1 vs 21.0 Gpix/s.)
template <int NCH>
__device__ __forceinline__ void half_rows(float *s, const __half *src, int lane, int np, int r0, int rows, int nw,
                                          int spitch, int W) {
    constexpr int RU = 4;  // rows per iteration: RU * NCH independent loads in flight per lane
    const int sstep = nw * spitch;
    const long long gstep = (long long)nw * W;
    for (int r = r0; r < rows; r += RU * nw, s += RU * sstep, src += RU * gstep) {
        __half2 v[RU][NCH];
#pragma unroll
        for (int q = 0; q < RU; ++q)
#pragma unroll
            for (int u = 0; u < NCH; ++u) {
                const bool in = (u < NCH - 1 || lane + 32 * u < np) && r + q * nw < rows;
                if (in) v[q][u] = __ldg(reinterpret_cast<const __half2 *>(src + q * gstep + 64 * u));
            }
#pragma unroll
        for (int q = 0; q < RU; ++q)
#pragma unroll
            for (int u = 0; u < NCH; ++u) {
                const bool in = (u < NCH - 1 || lane + 32 * u < np) && r + q * nw < rows;
                if (in) *reinterpret_cast<float2 *>(s + q * sstep + 64 * u) = __half22float2(v[q][u]);
            }
    }
}

// One channel plane of the halo tile into s[rows][pitch].  `frame` points at
// the (H, W, C) HWC frame or the (C, H, W) planar frame.
template <typename TI, bool PLANAR, bool WAIT = true>
__device__ __forceinline__ void load_plane(float *s, const TI *__restrict__ frame, const LGeom &g,
                                           int c, int gx0, int gy0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const bool clamp = g.boundary == SKC_CLAMP;
    const int H = g.H, W = g.W, C = g.C;
    if constexpr (PLANAR && sizeof(TI) == 2) {
        // planar fp16 intermediates (fp16-storage chains): through registers
        const __half *plane = reinterpret_cast<const __half *>(frame) + (long long)c * H * W;
        const bool pairs_ok = (W & 1) == 0;  // gx0 is even: 4-byte aligned pairs
        const int np = g.pitch >> 1;
        if (pairs_ok && gx0 >= 0 && gx0 + g.pitch <= W && gy0 >= 0 && gy0 + g.rows <= H) {
            float *sd = s + warp * g.pitch + 2 * lane;
            const __half *sx = plane + (long long)(gy0 + warp) * W + gx0 + 2 * lane;
            switch ((np + 31) >> 5) {
                case 1: half_rows<1>(sd, sx, lane, np, warp, g.rows, nw, g.pitch, W); return;
                case 2: half_rows<2>(sd, sx, lane, np, warp, g.rows, nw, g.pitch, W); return;
                case 3: half_rows<3>(sd, sx, lane, np, warp, g.rows, nw, g.pitch, W); return;
                case 4: half_rows<4>(sd, sx, lane, np, warp, g.rows, nw, g.pitch, W); return;
                case 5: half_rows<5>(sd, sx, lane, np, warp, g.rows, nw, g.pitch, W); return;
                default: break;
            }
        }
        for (int r = warp; r < g.rows; r += nw) {
            int gy = gy0 + r;
            const bool rowin = clamp || (gy >= 0 && gy < H);
            gy = min(max(gy, 0), H - 1);
            const __half *src = plane + (long long)gy * W;
            float *dst = s + r * g.pitch;
            for (int p = lane; p < np; p += 32) {
                const int col = 2 * p, gx = gx0 + col;
                if (pairs_ok && rowin && gx >= 0 && gx + 1 < W) {
                    *reinterpret_cast<float2 *>(dst + col) =
                        __half22float2(__ldg(reinterpret_cast<const __half2 *>(src + gx)));
                } else {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int x = gx + u;
                        const bool ok = clamp || (rowin && x >= 0 && x < W);
                        dst[col + u] = ok ? __half2float(__ldg(src + min(max(x, 0), W - 1))) : 0.f;
                    }
                }
            }
        }
    } else if constexpr (PLANAR) {
        static_assert(sizeof(TI) == 4, "planar intermediates are fp32");
        const float *plane = reinterpret_cast<const float *>(frame) + (long long)c * H * W;
        const bool pairs_ok = (W & 1) == 0;  // 8-byte alignment of row starts
        if (pairs_ok && gx0 >= 0 && gx0 + g.pitch <= W && gy0 >= 0 && gy0 + g.rows <= H &&
            tile_rows_any<2>((unsigned)__cvta_generic_to_shared(s + warp * g.pitch + 2 * lane),
                             plane + (long long)(gy0 + warp) * W + gx0 + 2 * lane, lane, g.pitch, warp, g.rows, nw,
                             4u * nw * g.pitch, (long long)nw * W, 1)) {
            if (WAIT) cp_async_wait_all();
            return;
        }
        for (int r = warp; r < g.rows; r += nw) {
            int gy = gy0 + r;
            const bool rowin = clamp || (gy >= 0 && gy < H);
            gy = min(max(gy, 0), H - 1);
            const float *src = plane + (long long)gy * W;
            float *dst = s + r * g.pitch;
            if (pairs_ok && rowin && gx0 >= 0 && gx0 + g.pitch <= W) {  // interior row: no clamping
                row_pairs_any((unsigned)__cvta_generic_to_shared(dst + 2 * lane), src + gx0 + 2 * lane, lane,
                              g.pitch);
                continue;
            }
            for (int p = lane; 2 * p < g.pitch; p += 32) {
                const int col = 2 * p;
                const int gx = gx0 + col;
                if (pairs_ok && gx >= 0 && gx + 1 < W) {
                    cp_async8(dst + col, src + gx, rowin);
                } else {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int x = gx + u;
                        const bool ok = clamp || (rowin && x >= 0 && x < W);
                        cp_async4(dst + col + u, src + min(max(x, 0), W - 1), ok);
                    }
                }
            }
        }
        if (WAIT) cp_async_wait_all();
    } else if constexpr (sizeof(TI) == 4) {
        const float *img = reinterpret_cast<const float *>(frame);
        if (gx0 >= 0 && gx0 + g.pitch <= W && gy0 >= 0 && gy0 + g.rows <= H &&
            tile_rows_any<1>((unsigned)__cvta_generic_to_shared(s + warp * g.pitch + lane),
                             img + ((long long)(gy0 + warp) * W + gx0 + lane) * C + c, lane, g.pitch, warp, g.rows,
                             nw, 4u * nw * g.pitch, (long long)nw * W * C, C)) {
            if (WAIT) if (WAIT) cp_async_wait_all();
            return;
        }
        for (int r = warp; r < g.rows; r += nw) {
            int gy = gy0 + r;
            const bool rowin = clamp || (gy >= 0 && gy < H);
            gy = min(max(gy, 0), H - 1);
            const float *src = img + (long long)gy * W * C + c;
            float *dst = s + r * g.pitch;
            if (rowin && gx0 >= 0 && gx0 + g.pitch <= W) {  // interior row: no clamping
                row_elems_any((unsigned)__cvta_generic_to_shared(dst + lane), src + (long long)(gx0 + lane) * C, lane,
                              g.pitch, C);
                continue;
            }
#pragma unroll 4
            for (int col = lane; col < g.pitch; col += 32) {
                const int gx = gx0 + col;
                const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                cp_async4(dst + col, src + (long long)min(max(gx, 0), W - 1) * C, ok);
            }
        }
        cp_async_wait_all();
    } else {
        constexpr int U = 8;
        if (gx0 >= 0 && gx0 + g.pitch <= W && gy0 >= 0 && gy0 + g.rows <= H) {
            // interior tile: U independent strided loads in flight per lane, no clamping
            const TI *sx = frame + ((long long)(gy0 + warp) * W + gx0 + lane) * C + c;
            float *dx = s + warp * g.pitch + lane;
            const long long gstep = (long long)nw * W * C;
            for (int r = warp; r < g.rows; r += nw, sx += gstep, dx += nw * g.pitch) {
                for (int c0 = lane; c0 < g.pitch; c0 += 32 * U) {
                    float v[U];
                    const int o = c0 - lane;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        v[u] = (c0 + 32 * u < g.pitch) ? IO<TI>::ld(sx + (long long)(o + 32 * u) * C) : 0.f;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (c0 + 32 * u < g.pitch) dx[o + 32 * u] = v[u];
                }
            }
            return;
        }
        for (int r = warp; r < g.rows; r += nw) {
            int gy = gy0 + r;
            const bool rowin = clamp || (gy >= 0 && gy < H);
            gy = min(max(gy, 0), H - 1);
            const TI *src = frame + (long long)gy * W * C + c;
            float *dst = s + r * g.pitch;
            for (int c0 = lane; c0 < g.pitch; c0 += 32 * U) {
                float v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int col = c0 + 32 * u;
                    const int gx = gx0 + col;
                    const bool ok = col < g.pitch && (clamp || (rowin && gx >= 0 && gx < W));
                    v[u] = ok ? IO<TI>::ld(src + (long long)min(max(gx, 0), W - 1) * C) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (c0 + 32 * u < g.pitch) dst[c0 + 32 * u] = v[u];
            }
        }
    }
}

// Shared memory of a layer kernel: the fp32 tile.
template <typename TI, bool IN_PL>
static size_t tile_smem(const LGeom &g) {
    return (size_t)g.rows * g.pitch * sizeof(float);
}

// Store a KR x 8 block of one channel.
template <int KR, typename TO, bool PLANAR>
__device__ __forceinline__ void store_block(TO *__restrict__ frame, const LGeom &g, int c, int gy0,
                                            int gx0, const float (&acc)[KR][8]) {
    const int H = g.H, W = g.W, C = g.C;
#pragma unroll
    for (int r = 0; r < KR; ++r) {
        const int gy = gy0 + r;
        if (gy >= H) continue;
        if constexpr (PLANAR && sizeof(TO) == 2) {
            // planar fp16 intermediates: one 16-byte store of 8 halves per row
            TO *p = frame + ((long long)c * H + gy) * W + gx0;
            if (gx0 + 7 < W && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
                uint4 t;
                unsigned *tw = reinterpret_cast<unsigned *>(&t);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const __half2 h = __floats2half2_rn(acc[r][2 * k], acc[r][2 * k + 1]);
                    tw[k] = *reinterpret_cast<const unsigned *>(&h);
                }
                *reinterpret_cast<uint4 *>(p) = t;
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (gx0 + j < W) IO<TO>::st(p + j, acc[r][j]);
            }
        } else if constexpr (PLANAR) {
            float *row = reinterpret_cast<float *>(frame) + ((long long)c * H + gy) * W;
            float *p = row + gx0;
            if (gx0 + 7 < W && ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && !g.accumulate) {
                reinterpret_cast<float4 *>(p)[0] = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
                reinterpret_cast<float4 *>(p)[1] = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (gx0 + j < W) p[j] = g.accumulate ? p[j] + acc[r][j] : acc[r][j];
            }
        } else {
            TO *row = frame + (long long)gy * W * C + c;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (gx0 + j < W) store_px<TO>(row + (long long)(gx0 + j) * C, acc[r][j], g.accumulate);
        }
    }
}

// --------------------------------------------------------------- tap path ---
// Staged HWC epilogue (see layer_tap_kernel): tile rows of one channel.
constexpr int kStagePitch = 132;  // 128 + 4: STS.128 conflict-free for odd KR (KR * 33 odd)

template <int KR, typename TO>
__device__ __forceinline__ void stage_store_hwc(float *smem, const float (&acc)[KR][8], TO *__restrict__ frame,
                                                const LGeom &g, int c, int ty0, int tx0, int row0, int col0) {
    __syncthreads();  // every warp is done reading the input tile
#pragma unroll
    for (int r = 0; r < KR; ++r) {
        float4 *d = reinterpret_cast<float4 *>(smem + (row0 + r) * kStagePitch + col0);
        d[0] = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
        d[1] = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
    }
    __syncthreads();
    constexpr int TH = 2 * 8 * KR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int C = g.C;
    const int nx = min(128, g.W - tx0), nr = min(TH, g.H - ty0);
    for (int r = warp; r < nr; r += nw) {
        TO *dst = frame + ((long long)(ty0 + r) * g.W + tx0) * C + c;
        const float *src = smem + r * kStagePitch;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int x = lane + 32 * u;
            if (x < nx) IO<TO>::st(dst + (long long)x * C, src[x]);
        }
    }
}


constexpr int kTWX = 4, kTWY = 2;                 // 256 threads, tile 128 x (16 * KR)
constexpr int kTTW = kTWX * 32;

template <int KR>
__device__ __forceinline__ void tap_rows(float (&acc)[KR][8], const float *p, int pitch, float4 w,
                                         bool odd) {
    float a[9], b[9];
    auto load_row = [&](const float *q, float (&v)[9]) {
        if (!odd) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 t = reinterpret_cast<const float2 *>(q)[k];
                v[2 * k] = t.x;
                v[2 * k + 1] = t.y;
            }
            v[8] = q[8];
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 t = reinterpret_cast<const float2 *>(q + 1)[k];
                v[2 * k + 1] = t.x;
                v[2 * k + 2] = t.y;
            }
            v[0] = q[0];
        }
    };
    load_row(p, a);
#pragma unroll
    for (int r = 0; r < KR; ++r) {
        load_row(p + (r + 1) * pitch, b);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float v = acc[r][j];
            v = fmaf(w.x, a[j], v);
            v = fmaf(w.y, a[j + 1], v);
            v = fmaf(w.z, b[j], v);
            v = fmaf(w.w, b[j + 1], v);
            acc[r][j] = v;
        }
#pragma unroll
        for (int j = 0; j < 9; ++j) a[j] = b[j];
    }
}

template <int KR, typename TI, typename TO, bool IN_PL, bool OUT_PL>
__global__ void __launch_bounds__(kTWX *kTWY * 32)
    layer_tap_kernel(const TI *__restrict__ in, TO *__restrict__ out, const LGeom g,
                     const __grid_constant__ TapList tl) {
    extern __shared__ __align__(16) float smem[];
    const int C = g.C;
    const int b = blockIdx.z, c = blockIdx.x % C;
    const long long fs = (long long)g.H * g.W * C;
    constexpr int TH = kTWY * 8 * KR;
    const int tx0 = (blockIdx.x / C) * kTTW, ty0 = blockIdx.y * TH;
    load_plane<TI, IN_PL>(smem, in + b * fs, g, c, tx0 + g.dx0, ty0 + g.dy0);
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane & 3, ly = lane >> 2, wx = warp % kTWX, wy = warp / kTWX;
    const int col0 = wx * 32 + lx * 8;
    const int row0 = wy * 8 * KR + ly * KR;
    const float *base = smem + row0 * g.pitch + col0;

    float acc[KR][8];
#pragma unroll
    for (int r = 0; r < KR; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[r][j] = 0.f;
#pragma unroll 1
    for (int i = 0; i < tl.n_even; ++i) tap_rows<KR>(acc, base + tl.off[i], g.pitch, tl.cw[i], false);
#pragma unroll 1
    for (int i = tl.n_even; i < tl.n; ++i) tap_rows<KR>(acc, base + tl.off[i], g.pitch, tl.cw[i], true);

    if constexpr (IN_PL && !OUT_PL) {
        if (!g.accumulate) {
            // HWC output from a channel CTA: stage the tile in the dead input
            // tile, then every warp writes whole tile rows with lanes along x
            // (stride-C addresses: 32 lanes cover 3-4 contiguous lines, and
            // the C channel CTAs of the tile, which run together, complete
            // the sectors in L2) instead of 8 scattered rows per instruction.
            stage_store_hwc<KR, TO>(smem, acc, out + b * fs, g, c, ty0, tx0, row0, col0);
            return;
        }
    }
    store_block<KR, TO, OUT_PL>(out + b * fs, g, c, ty0 + row0, tx0 + col0, acc);
}

// Cluster-of-C HWC epilogue (opt-in, SKC_TAP_CLUSTER=1): the C channel CTAs
// of a tile form one thread-block cluster.  Each stages its finished channel
// tile in its dead input tile, then -- after a cluster barrier -- writes every
// C-th tile row for *all* channels: each lane reads 4 pixels of every channel
// from the sibling CTAs' shared memory (DSMEM, 16-byte loads) and stores the
// interleaved pixels contiguously (fp16 C = 4: 32 bytes per lane), instead of
// C CTAs each scattering 2- or 4-byte stores at stride C.
template <typename TO, int CC>
__device__ __forceinline__ void store_hwc_pixels(TO *dst, const float (&v)[4][CC], int n) {
    if constexpr (sizeof(TO) == 2 && CC == 4) {
        if (n == 4 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            uint4 t[2];
            unsigned *tw = reinterpret_cast<unsigned *>(t);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const __half2 a = __floats2half2_rn(v[p][0], v[p][1]), b = __floats2half2_rn(v[p][2], v[p][3]);
                tw[2 * p] = *reinterpret_cast<const unsigned *>(&a);
                tw[2 * p + 1] = *reinterpret_cast<const unsigned *>(&b);
            }
            reinterpret_cast<uint4 *>(dst)[0] = t[0];
            reinterpret_cast<uint4 *>(dst)[1] = t[1];
            return;
        }
    }
    if constexpr (sizeof(TO) == 4 && (CC == 4 || CC == 2)) {
        if (n == 4 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            float4 *d4 = reinterpret_cast<float4 *>(dst);
            const float *f = &v[0][0];
#pragma unroll
            for (int q = 0; q < CC; ++q) d4[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
            return;
        }
    }
    for (int p = 0; p < n; ++p)
#pragma unroll
        for (int c = 0; c < CC; ++c) IO<TO>::st(dst + p * CC + c, v[p][c]);
}

template <int KR, typename TI, typename TO, int CC>
__global__ void __launch_bounds__(kTWX *kTWY * 32)
    layer_tap_cluster_kernel(const TI *__restrict__ in, TO *__restrict__ out, const LGeom g,
                             const __grid_constant__ TapList tl) {
    extern __shared__ __align__(16) float smem[];
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int b = blockIdx.z, c = (int)cluster.block_rank();  // cluster (CC,1,1) over the channel-fastest grid
    const long long fs = (long long)g.H * g.W * CC;
    constexpr int TH = kTWY * 8 * KR;
    const int tx0 = (blockIdx.x / CC) * kTTW, ty0 = blockIdx.y * TH;
    load_plane<TI, true>(smem, in + b * fs, g, c, tx0 + g.dx0, ty0 + g.dy0);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane & 3, ly = lane >> 2, wx = warp % kTWX, wy = warp / kTWX;
    const int col0 = wx * 32 + lx * 8;
    const int row0 = wy * 8 * KR + ly * KR;
    const float *base = smem + row0 * g.pitch + col0;
    float acc[KR][8];
#pragma unroll
    for (int r = 0; r < KR; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[r][j] = 0.f;
#pragma unroll 1
    for (int i = 0; i < tl.n_even; ++i) tap_rows<KR>(acc, base + tl.off[i], g.pitch, tl.cw[i], false);
#pragma unroll 1
    for (int i = tl.n_even; i < tl.n; ++i) tap_rows<KR>(acc, base + tl.off[i], g.pitch, tl.cw[i], true);
    __syncthreads();  // every warp is done reading the input tile
#pragma unroll
    for (int r = 0; r < KR; ++r) {
        float4 *d = reinterpret_cast<float4 *>(smem + (row0 + r) * kStagePitch + col0);
        d[0] = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
        d[1] = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
    }
    cluster.sync();  // all C channel tiles staged
    const float *sib[CC];
#pragma unroll
    for (int q = 0; q < CC; ++q) sib[q] = cluster.map_shared_rank(smem, q);
    const int nx = min(128, g.W - tx0), nr = min(TH, g.H - ty0);
    const int nw = blockDim.x >> 5;
    for (int r = c + CC * warp; r < nr; r += CC * nw) {
        const int x = 4 * lane;
        if (x >= nx) continue;
        float v[4][CC];
#pragma unroll
        for (int q = 0; q < CC; ++q) {
            const float4 t = *reinterpret_cast<const float4 *>(sib[q] + r * kStagePitch + x);
            v[0][q] = t.x;
            v[1][q] = t.y;
            v[2][q] = t.z;
            v[3][q] = t.w;
        }
        store_hwc_pixels<TO, CC>(out + ((long long)b * g.H * g.W + (long long)(ty0 + r) * g.W + tx0 + x) * CC, v,
                                 min(4, nx - x));
    }
    cluster.sync();  // keep this CTA's staged tile alive until the siblings are done
}

static bool tap_cluster_enabled() {
    static const bool v = [] {
        const char *e = std::getenv("SKC_TAP_CLUSTER");
        return e && e[0] == '1';
    }();
    return v;
}

template <int KR, typename TI, typename TO, int CC>
static int launch_tap_cluster(const TI *in, TO *out, int B, int H, int W, const LGeom &g, const TapList &tl,
                              size_t smem, cudaStream_t s) {
    auto kern = layer_tap_cluster_kernel<KR, TI, TO, CC>;
    const int attr = set_smem_attr(kern);
    if (attr) return attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ceil_div(W, kTTW) * CC, ceil_div(H, kTWY * 8 * KR), B);
    cfg.blockDim = dim3(kTWX * kTWY * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SKC_CUDA(cudaLaunchKernelEx(&cfg, kern, in, out, g, tl));
    return SKC_OK;
}

// ------------------------------------------------------------- dense path ---
constexpr int kDenKR = 5, kDenWX = 4, kDenWY = 2;  // 256 threads, tile 128 x 80
constexpr int kDenTW = kDenWX * 32, kDenTH = kDenWY * 8 * kDenKR;

// acc = the D x D stencil over a KR x 8 block whose window starts at pc.
template <int D, int KR>
__device__ __forceinline__ void stencil_block(float (&acc)[KR][8], const float *pc, int pitch, const DenseList &dl) {
#pragma unroll
    for (int i = 0; i < KR; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll
    for (int r = 0; r < KR + D - 1; ++r) {
        float w[8 + D - 1];
#pragma unroll
        for (int j = 0; j < 8 + D - 1; ++j) w[j] = pc[r * pitch + j];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int i = r - a;
            if (i < 0 || i >= KR) continue;
#pragma unroll
            for (int bb = 0; bb < D; ++bb) {
                const float k = dl.k[a * D + bb];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(k, w[j + bb], acc[i][j]);
            }
        }
    }
}

// Packed-FP32 dense stencil (FFMA2, sm_100): each thread owns KR2 = 6 rows x
// 8 columns as 3 row pairs; one fma.rn.f32x2 updates (out[2p][j],
// out[2p+1][j]) with the weight pair (K[a][b], K[a-1][b]) -- adjacent in a
// host-prepared table, loaded as one 64-bit operand -- times the broadcast
// input texel w[j+b] (the .F32 scalar operand form).  No register pairing of
// inputs is needed, and every instruction does two FMAs.  Rows a = 0 and a = D
// of the table hold a zero in the missing half (10% padding work at D = 9).
constexpr int kF2KR = 6, kF2TH = kDenWY * 8 * kF2KR;  // tile 128 x 96

struct DenseList2 {
    float2 k2[(kMaxDense + 1) * kMaxDense];  // k2[a][b] = (K[a][b], K[a-1][b]), zero outside 0..D-1
    int D;
    int col_shift;
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long ra = *reinterpret_cast<unsigned long long *>(&a);
    unsigned long long rb = *reinterpret_cast<unsigned long long *>(&b);
    unsigned long long rc = *reinterpret_cast<unsigned long long *>(&c), rd;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
    return *reinterpret_cast<float2 *>(&rd);
}

// Planar fp32 in and out (the chain's inner layers).  SH = col_shift & 1:
// window rows are read with LDS.64 from the 8-byte-aligned column at or before
// the window start.
template <int D, int SH, typename T>
__global__ void __launch_bounds__(kDenWX *kDenWY * 32)
    layer_stencil2_kernel(const T *__restrict__ in, T *__restrict__ out, const LGeom g,
                          const __grid_constant__ DenseList2 dl) {
    extern __shared__ __align__(16) float smem[];
    constexpr int KR = kF2KR, NP = KR / 2;
    const int C = g.C;
    const int b = blockIdx.z, c = blockIdx.x % C;
    const long long fs = (long long)g.H * g.W * C;
    const int tx0 = (blockIdx.x / C) * kDenTW, ty0 = blockIdx.y * kF2TH;
    load_plane<T, true>(smem, in + b * fs, g, c, tx0 + g.dx0, ty0 + g.dy0);
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane & 3, ly = lane >> 2, wx = warp % kDenWX, wy = warp / kDenWX;
    const int col0 = wx * 32 + lx * 8;
    const int row0 = wy * 8 * KR + ly * KR;
    const float *pc = smem + row0 * g.pitch + col0 + dl.col_shift;
    const int pitch = g.pitch;

    float2 acc[NP][8];
#pragma unroll
    for (int i = 0; i < NP; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < KR + D - 1; ++r) {
        float w[8 + D - 1 + 1];
        {
            constexpr int NV = (8 + D - 1 + SH + 1) / 2;
            float raw[2 * NV];
            const float2 *q2 = reinterpret_cast<const float2 *>(pc - SH + r * pitch);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float2 t = q2[v];
                raw[2 * v] = t.x;
                raw[2 * v + 1] = t.y;
            }
#pragma unroll
            for (int j = 0; j < 8 + D - 1; ++j) w[j] = raw[j + SH];
        }
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
            const int a = r - 2 * pp;  // row 2pp takes stencil row a, row 2pp+1 row a-1
            if (a < 0 || a > D) continue;
#pragma unroll
            for (int bb = 0; bb < D; ++bb) {
                const float2 kk = dl.k2[a * D + bb];
                if (a == 0) {         // only row 2pp has a term (K[0][b]); scalar FFMA on that half
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[pp][j].x = fmaf(kk.x, w[j + bb], acc[pp][j].x);
                } else if (a == D) {  // only row 2pp+1 (K[D-1][b])
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[pp][j].y = fmaf(kk.y, w[j + bb], acc[pp][j].y);
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        acc[pp][j] = ffma2(kk, make_float2(w[j + bb], w[j + bb]), acc[pp][j]);
                }
            }
        }
    }
    float res[KR][8];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            res[2 * pp][j] = acc[pp][j].x;
            res[2 * pp + 1][j] = acc[pp][j].y;
        }
    store_block<KR, T, true>(out + b * fs, g, c, ty0 + row0, tx0 + col0, res);
}

// Register caps (4 CTAs per SM, 3 for D = 3 whose body otherwise hoists its
// window loads into 80-104 registers and halves the resident CTAs of these
// HBM-bound layers; at the 64-register cap it would spill).
template <int D, int KR, typename TI, typename TO, bool IN_PL, bool OUT_PL>
__global__ void __launch_bounds__(kDenWX *kDenWY * 32, D == 3 ? 3 : 4)
    layer_stencil_kernel(const TI *__restrict__ in, TO *__restrict__ out, const LGeom g,
                         const __grid_constant__ DenseList dl) {
    extern __shared__ __align__(16) float smem[];
    const int C = g.C;
    const int b = blockIdx.z, c = blockIdx.x % C;
    const long long fs = (long long)g.H * g.W * C;
    const int tx0 = (blockIdx.x / C) * kDenTW, ty0 = blockIdx.y * (kDenWY * 8 * KR);
    load_plane<TI, IN_PL>(smem, in + b * fs, g, c, tx0 + g.dx0, ty0 + g.dy0);
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane & 3, ly = lane >> 2, wx = warp % kDenWX, wy = warp / kDenWX;
    const int col0 = wx * 32 + lx * 8;
    const int row0 = wy * 8 * KR + ly * KR;
    const float *pc = smem + row0 * g.pitch + col0 + dl.col_shift;
    const int pitch = g.pitch;

    float acc[KR][8];
    stencil_block<D, KR>(acc, pc, pitch, dl);
    store_block<KR, TO, OUT_PL>(out + b * fs, g, c, ty0 + row0, tx0 + col0, acc);
}

// ------------------------------------------------ direct (huge halo) path ---
template <typename TI, typename TO, bool IN_PL, bool OUT_PL>
__global__ void __launch_bounds__(256)
    layer_gather_kernel(const TI *__restrict__ in, TO *__restrict__ out, const LGeom g,
                        const __grid_constant__ TapList tl) {
    const int C = g.C;
    const int b = blockIdx.y / C, c = blockIdx.y - (blockIdx.y / C) * C;
    const long long hw = (long long)g.H * g.W, fs = hw * C;
    in += b * fs;
    out += b * fs;
    const long long ps = IN_PL ? 1 : C, cs = IN_PL ? hw : 1;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < hw;
         p += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(p / g.W), x = (int)(p - (long long)y * g.W);
        float acc = 0.f;
        for (int i = 0; i < tl.n; ++i) {
            const float4 w = tl.cw[i];
            const float cw[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int yy = y + tl.iy[i] + (k >> 1), xx = x + tl.ix[i] + (k & 1);
                if (g.boundary == SKC_CLAMP) {
                    yy = min(max(yy, 0), g.H - 1);
                    xx = min(max(xx, 0), g.W - 1);
                } else if (yy < 0 || yy >= g.H || xx < 0 || xx >= g.W) {
                    continue;
                }
                acc = fmaf(cw[k], IO<TI>::ld(in + ((long long)yy * g.W + xx) * ps + c * cs), acc);
            }
        }
        TO *o = OUT_PL ? out + c * hw + p : out + p * C + c;
        store_px<TO>(o, acc, g.accumulate);
    }
}

// ------------------------------------------------------------------ host ---
struct Plan {
    std::vector<int> ix, iy;
    std::vector<double> cw;  // 4 per tap, float64 (sample_shifted order)
    int dx_min = 0, dx_max = 0, dy_min = 0, dy_max = 0;  // corner footprint (inclusive)
};

// sample_shifted (engine.py:118-130): ix = floor(ox), fx = ox - ix, corners 00, 10, 01, 11.
static Plan plan_taps(const double *taps, int S) {
    Plan p;
    p.ix.resize(S);
    p.iy.resize(S);
    p.cw.resize(4 * (size_t)S);
    for (int i = 0; i < S; ++i) {
        const double ox = taps[3 * i], oy = taps[3 * i + 1], w = taps[3 * i + 2];
        const double fx0 = std::floor(ox), fy0 = std::floor(oy);
        const double fx = ox - fx0, fy = oy - fy0;
        p.ix[i] = (int)fx0;
        p.iy[i] = (int)fy0;
        p.cw[4 * i + 0] = w * (1.0 - fx) * (1.0 - fy);
        p.cw[4 * i + 1] = w * fx * (1.0 - fy);
        p.cw[4 * i + 2] = w * (1.0 - fx) * fy;
        p.cw[4 * i + 3] = w * fx * fy;
        if (i == 0 || p.ix[i] < p.dx_min) p.dx_min = p.ix[i];
        if (i == 0 || p.ix[i] + 1 > p.dx_max) p.dx_max = p.ix[i] + 1;
        if (i == 0 || p.iy[i] < p.dy_min) p.dy_min = p.iy[i];
        if (i == 0 || p.iy[i] + 1 > p.dy_max) p.dy_max = p.iy[i] + 1;
    }
    return p;
}

static bool dense_allowed() {
    static const bool on = [] {
        const char *e = std::getenv("SKC_DENSE");
        return !(e && e[0] == '0');
    }();
    return on;
}

static int floor_even(int v) { return v & ~1; }

static LGeom make_geom(int H, int W, int C, int boundary, int accumulate, int tw, int th, int dx_min,
                       int dx_max, int dy_min, int dy_max) {
    LGeom g;
    g.H = H;
    g.W = W;
    g.C = C;
    g.boundary = boundary;
    g.accumulate = accumulate;
    g.dx0 = floor_even(dx_min);
    g.dy0 = dy_min;
    int pitch = tw + (dx_max - g.dx0) + 1;  // +1: the odd-tap window reads one column past
    pitch = (pitch + 3) & ~3;
    pitch += 2;                              // pitch = 2 mod 4
    g.pitch = pitch;
    g.rows = th + (dy_max - dy_min);
    return g;
}

template <typename K>
static int set_smem_attr(K kern) {
    return smem_optin((const void *)kern, kMaxSmem);
}

// Rows per thread of the tap kernel: SKC_TAP_KR (5 or 7) overrides; default 5
// for layers of <= 16 taps (HBM-bound), else 7 when the halo tile of a 7-row
// block still leaves two CTAs per SM, else 5.
static int tap_kr_override() {
    static const int v = [] {
        const char *e = std::getenv("SKC_TAP_KR");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// Rows per thread of the tap tile for a layer of `ntaps` taps with the given
// corner footprint (see tap_kr_override).
static int tap_kr_for(int H, int W, int C, int boundary, int accumulate, int dx_min, int dx_max, int dy_min,
                      int dy_max, int ntaps, bool hwc_out = false) {
    const int KR = tap_kr_override();
    if (KR == 3 || KR == 5 || KR == 7) return KR;
    // latency-bound small layers: smaller tiles, more CTAs in flight (config 3's
    // planar 4-tap layers: KR 3 -> 1.59 ms, 5 -> 1.83, 7 -> ~2.2); the staged HWC
    // epilogue prefers the taller tile (2.44 vs 2.59 ms at KR 3)
    if (ntaps <= 16) return hwc_out ? 5 : 3;
    const LGeom g7 = make_geom(H, W, C, boundary, accumulate, kTTW, kTWY * 8 * 7, dx_min, dx_max, dy_min, dy_max);
    return ((size_t)g7.rows * g7.pitch * sizeof(float) * 2 <= (size_t)kMaxSmem) ? 7 : 5;
}

template <typename TI, typename TO, bool IN_PL, bool OUT_PL>
static int launch_taps(const void *in, void *out, int B, int H, int W, int C, const Plan &pl, int t0,
                       int t1, int boundary, int accumulate, cudaStream_t s) {
    int dx_min = 1 << 30, dx_max = -(1 << 30), dy_min = 1 << 30, dy_max = -(1 << 30);
    for (int i = t0; i < t1; ++i) {
        dx_min = std::min(dx_min, pl.ix[i]);
        dx_max = std::max(dx_max, pl.ix[i] + 1);
        dy_min = std::min(dy_min, pl.iy[i]);
        dy_max = std::max(dy_max, pl.iy[i] + 1);
    }
    const int KR = tap_kr_for(H, W, C, boundary, accumulate, dx_min, dx_max, dy_min, dy_max, t1 - t0, IN_PL && !OUT_PL);
    const int TH = kTWY * 8 * KR;
    LGeom g = make_geom(H, W, C, boundary, accumulate, kTTW, TH, dx_min, dx_max, dy_min, dy_max);
    TapList tl;
    tl.n = t1 - t0;
    int k = 0;
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) tl.n_even = k;
        for (int i = t0; i < t1; ++i) {
            const int off = (pl.iy[i] - g.dy0) * g.pitch + (pl.ix[i] - g.dx0);
            if ((off & 1) != pass) continue;
            tl.off[k] = off;
            tl.ix[k] = pl.ix[i];
            tl.iy[k] = pl.iy[i];
            tl.cw[k] = make_float4((float)pl.cw[4 * i], (float)pl.cw[4 * i + 1], (float)pl.cw[4 * i + 2],
                                   (float)pl.cw[4 * i + 3]);
            ++k;
        }
    }
    const size_t smem = tile_smem<TI, IN_PL>(g);
    const TI *pin = static_cast<const TI *>(in);
    TO *pout = static_cast<TO *>(out);
    if constexpr (IN_PL && !OUT_PL) {
        if (tap_cluster_enabled() && !accumulate && (C == 3 || C == 4) && KR == 5 &&
            std::max(smem, (size_t)kTWY * 8 * 5 * kStagePitch * sizeof(float)) <= (size_t)kMaxSmem) {
            const size_t sm = std::max(smem, (size_t)kTWY * 8 * 5 * kStagePitch * sizeof(float));
            return C == 4 ? launch_tap_cluster<5, TI, TO, 4>(static_cast<const TI *>(in), static_cast<TO *>(out), B, H, W, g, tl, sm, s)
                          : launch_tap_cluster<5, TI, TO, 3>(static_cast<const TI *>(in), static_cast<TO *>(out), B, H, W, g, tl, sm, s);
        }
    }
    if (smem <= (size_t)kMaxSmem) {
        auto kern = KR == 7 ? layer_tap_kernel<7, TI, TO, IN_PL, OUT_PL>
                            : (KR == 5 ? layer_tap_kernel<5, TI, TO, IN_PL, OUT_PL> : layer_tap_kernel<3, TI, TO, IN_PL, OUT_PL>);
        const int attr3 = set_smem_attr(layer_tap_kernel<3, TI, TO, IN_PL, OUT_PL>);
        const int attr5 = set_smem_attr(layer_tap_kernel<5, TI, TO, IN_PL, OUT_PL>);
        const int attr7 = set_smem_attr(layer_tap_kernel<7, TI, TO, IN_PL, OUT_PL>);
        if (attr3 || attr5 || attr7) return attr3 ? attr3 : (attr5 ? attr5 : attr7);
        dim3 grid(ceil_div(W, kTTW) * C, ceil_div(H, TH), B);
        kern<<<grid, kTWX * kTWY * 32, smem, s>>>(pin, pout, g, tl);
        SKC_LAUNCH_CHECK("layer_tap_kernel");
    } else {
        const long long hw = (long long)H * W;
        dim3 grid((unsigned)std::min<long long>((hw + 255) / 256, 148 * 8), B * C);
        layer_gather_kernel<TI, TO, IN_PL, OUT_PL><<<grid, 256, 0, s>>>(pin, pout, g, tl);
        SKC_LAUNCH_CHECK("layer_gather_kernel");
    }
    return SKC_OK;
}

// Packed-FP32 (FFMA2) stencil: default for planar inner layers with D >= 7
// (config 1, D = 9: 2.18 ms against 2.59 ms); SKC_STENCIL_FFMA2=1 forces it
// for every stencil, =0 disables it.
static int stencil_ffma2_mode() {
    static const int v = [] {
        const char *e = std::getenv("SKC_STENCIL_FFMA2");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return v;
}

template <int D, int SH, typename T>
static int launch_stencil2_d(const void *in, void *out, int B, int C, const DenseList2 &dl, const LGeom &g,
                             cudaStream_t s) {
    auto kern = layer_stencil2_kernel<D, SH, T>;
    const int attr = set_smem_attr(kern);
    if (attr) return attr;
    const size_t smem = tile_smem<T, true>(g);
    dim3 grid(ceil_div(g.W, kDenTW) * C, ceil_div(g.H, kF2TH), B);
    kern<<<grid, kDenWX * kDenWY * 32, smem, s>>>(static_cast<const T *>(in), static_cast<T *>(out), g, dl);
    SKC_LAUNCH_CHECK("layer_stencil2_kernel");
    return SKC_OK;
}

template <typename T>
static int launch_stencil2(const void *in, void *out, int B, int C, int D, const DenseList2 &dl, const LGeom &g,
                           cudaStream_t s) {
    const bool odd = dl.col_shift & 1;
    switch (D) {
        case 3: return odd ? launch_stencil2_d<3, 1, T>(in, out, B, C, dl, g, s) : launch_stencil2_d<3, 0, T>(in, out, B, C, dl, g, s);
        case 5: return odd ? launch_stencil2_d<5, 1, T>(in, out, B, C, dl, g, s) : launch_stencil2_d<5, 0, T>(in, out, B, C, dl, g, s);
        case 7: return odd ? launch_stencil2_d<7, 1, T>(in, out, B, C, dl, g, s) : launch_stencil2_d<7, 0, T>(in, out, B, C, dl, g, s);
        default: return odd ? launch_stencil2_d<9, 1, T>(in, out, B, C, dl, g, s) : launch_stencil2_d<9, 0, T>(in, out, B, C, dl, g, s);
    }
}

template <int D, int KR, typename TI, typename TO, bool IN_PL, bool OUT_PL>
static int launch_stencil_d(const void *in, void *out, int B, int H, int W, int C, const DenseList &dl,
                            const LGeom &g, cudaStream_t s) {
    const size_t smem = tile_smem<TI, IN_PL>(g);
    auto kern = layer_stencil_kernel<D, KR, TI, TO, IN_PL, OUT_PL>;
    const int attr = set_smem_attr(kern);
    if (attr) return attr;
    dim3 grid(ceil_div(W, kDenTW) * C, ceil_div(H, kDenWY * 8 * KR), B);
    kern<<<grid, kDenWX * kDenWY * 32, smem, s>>>(static_cast<const TI *>(in), static_cast<TO *>(out), g, dl);
    SKC_LAUNCH_CHECK("layer_stencil_kernel");
    return SKC_OK;
}

static bool odd_head_pitch() {
    static const bool v = [] {
        const char *e = std::getenv("SKC_HEAD_ODD_PITCH");
        return !(e && e[0] == '0');
    }();
    return v;
}

template <typename TI, typename TO, bool IN_PL, bool OUT_PL>
static bool try_stencil(const void *in, void *out, int B, int H, int W, int C, const Plan &pl, int S,
                        int boundary, cudaStream_t s, int *rc) {
    if (!dense_allowed()) return false;
    // planar fp16 inputs of small layers are load-latency bound: the KR = 3 tap
    // tile beats the dense kernel's fewer FMAs (config 3's D3 layer: 1.59 vs
    // 2.05 ms; with fp32 planar input the dense D3 wins, 1.68 vs 1.82 ms)
    if constexpr (IN_PL && sizeof(TI) == 2) {
        if (S <= 16) return false;
    }
    const int sx = pl.dx_max - pl.dx_min + 1, sy = pl.dy_max - pl.dy_min + 1;
    const int D = dense_size_for(std::max(sx, sy));
    if (D == 0 || D * D >= 4 * S) return false;
    DenseList dl;
    double k[kMaxDense * kMaxDense] = {0.0};
    for (int i = 0; i < S; ++i)
        for (int q = 0; q < 4; ++q) {
            const int a = pl.iy[i] + (q >> 1) - pl.dy_min, bb = pl.ix[i] + (q & 1) - pl.dx_min;
            k[a * D + bb] += pl.cw[4 * i + q];
        }
    dl.D = D;
    for (int e = 0; e < kMaxDense * kMaxDense; ++e) dl.k[e] = e < D * D ? (float)k[e] : 0.f;
    // planar inner layers: packed-FP32 stencil (default for D >= 7, forced by
    // SKC_STENCIL_FFMA2=1, disabled by =0)
    if constexpr (IN_PL && OUT_PL && std::is_same<TI, TO>::value) {
        const int f2mode = stencil_ffma2_mode();
        if (f2mode == 1 || (f2mode < 0 && D >= 7)) {
            LGeom g = make_geom(H, W, C, boundary, 0, kDenTW, kF2TH, pl.dx_min, pl.dx_min + D - 1, pl.dy_min,
                                pl.dy_min + D - 1);
            DenseList2 d2;
            std::memset(&d2, 0, sizeof(d2));
            d2.D = D;
            d2.col_shift = pl.dx_min - g.dx0;
            for (int a = 0; a <= D; ++a)
                for (int bb = 0; bb < D; ++bb) {
                    const float hi = a < D ? (float)k[a * D + bb] : 0.f;
                    const float lo = a > 0 ? (float)k[(a - 1) * D + bb] : 0.f;
                    d2.k2[a * D + bb] = make_float2(hi, lo);
                }
            *rc = launch_stencil2<TO>(in, out, B, C, D, d2, g, s);
            return true;
        }
    }
    LGeom g = make_geom(H, W, C, boundary, 0, kDenTW, kDenTH, pl.dx_min, pl.dx_min + D - 1,
                        pl.dy_min, pl.dy_min + D - 1);
    // HWC inputs stage with 4-byte copies, so the pitch may be odd: then the
    // window rows' LDS.32 of the 4 x 8 lane layout (rows KR * pitch apart)
    // hit 32 distinct banks (config 1's D5 head: 51% of its shared-load
    // wavefronts were 2-way conflicts at pitch = 2 mod 4)
    if constexpr (!IN_PL) {
        if (odd_head_pitch() && (g.pitch & 1) == 0) g.pitch += 1;
    }
    dl.col_shift = pl.dx_min - g.dx0;
    switch (D) {
        case 3: *rc = launch_stencil_d<3, kDenKR, TI, TO, IN_PL, OUT_PL>(in, out, B, H, W, C, dl, g, s); break;
        case 5: *rc = launch_stencil_d<5, kDenKR, TI, TO, IN_PL, OUT_PL>(in, out, B, H, W, C, dl, g, s); break;
        case 7: *rc = launch_stencil_d<7, kDenKR, TI, TO, IN_PL, OUT_PL>(in, out, B, H, W, C, dl, g, s); break;
        default: *rc = launch_stencil_d<9, kDenKR, TI, TO, IN_PL, OUT_PL>(in, out, B, H, W, C, dl, g, s); break;
    }
    return true;
}

template <typename TI, typename TO, bool IN_PL, bool OUT_PL>
static int layer_t(const void *in, void *out, int B, int H, int W, int C, const double *taps, int S,
                   int boundary, cudaStream_t s) {
    const Plan pl = plan_taps(taps, S);
    int rc = SKC_OK;
    // generated sparse stencil when it is cheaper (skc_sparse.cu); HWC inputs opt-in (SKC_SPARSE_HWC)
    rc = sparse_layer(in, std::is_same<TI, float>::value, out, std::is_same<TO, float>::value, OUT_PL, B, H, W, C,
                      taps, S, boundary, s, !IN_PL);
    if (rc != -1) return rc;
    rc = SKC_OK;
    if (try_stencil<TI, TO, IN_PL, OUT_PL>(in, out, B, H, W, C, pl, S, boundary, s, &rc)) return rc;
    if (S <= kLMaxTaps)
        return launch_taps<TI, TO, IN_PL, OUT_PL>(in, out, B, H, W, C, pl, 0, S, boundary, 0, s);
    // long layers: accumulate chunks into an fp32 destination
    if constexpr (std::is_same<TO, float>::value) {
        for (int t0 = 0; t0 < S && rc == SKC_OK; t0 += kLMaxTaps)
            rc = launch_taps<TI, TO, IN_PL, OUT_PL>(in, out, B, H, W, C, pl, t0, std::min(S, t0 + kLMaxTaps),
                                                    boundary, t0 > 0, s);
        return rc;
    } else {
        return -1;  // caller routes fp16 outputs of long layers through fp32
    }
}

// Dispatch on (input dtype, output dtype, input planar, output planar).
// Planar intermediates are fp32, or fp16 in chains whose storage is fp16 (see
// chain_mid_dtype): the planar fp16 combinations compiled are HWC fp16 ->
// planar fp16, planar fp16 -> planar fp16 and planar fp16 -> HWC fp16.
int layer_dispatch(const void *in, int idt, bool in_pl, void *out, int odt, bool out_pl, int B, int H,
                   int W, int C, const double *taps, int S, int boundary, cudaStream_t s) {
    const bool h_in = in_pl && idt == SKC_F16, h_out = out_pl && odt == SKC_F16;
    if (h_in || h_out) {
        if (idt != SKC_F16 || odt != SKC_F16)
            return fail(SKC_EBADARG, "planar fp16 tensors pair with fp16 on the other side");
        if (S > kLMaxTaps) return fail(SKC_EBADARG, "planar fp16 layers take at most skc_max_taps() taps");
        if (in_pl && out_pl) return layer_t<__half, __half, true, true>(in, out, B, H, W, C, taps, S, boundary, s);
        if (in_pl) return layer_t<__half, __half, true, false>(in, out, B, H, W, C, taps, S, boundary, s);
        return layer_t<__half, __half, false, true>(in, out, B, H, W, C, taps, S, boundary, s);
    }
    if (in_pl && out_pl) return layer_t<float, float, true, true>(in, out, B, H, W, C, taps, S, boundary, s);
    if (in_pl) {
        if (odt == SKC_F32) return layer_t<float, float, true, false>(in, out, B, H, W, C, taps, S, boundary, s);
        return layer_t<float, __half, true, false>(in, out, B, H, W, C, taps, S, boundary, s);
    }
    if (out_pl) {
        if (idt == SKC_F32) return layer_t<float, float, false, true>(in, out, B, H, W, C, taps, S, boundary, s);
        return layer_t<__half, float, false, true>(in, out, B, H, W, C, taps, S, boundary, s);
    }
    if (idt == SKC_F32 && odt == SKC_F32) return layer_t<float, float, false, false>(in, out, B, H, W, C, taps, S, boundary, s);
    if (idt == SKC_F16 && odt == SKC_F32) return layer_t<__half, float, false, false>(in, out, B, H, W, C, taps, S, boundary, s);
    if (idt == SKC_F32 && odt == SKC_F16) return layer_t<float, __half, false, false>(in, out, B, H, W, C, taps, S, boundary, s);
    return layer_t<__half, __half, false, false>(in, out, B, H, W, C, taps, S, boundary, s);
}

int dense_size_for(int span) {
    if (span <= 3) return 3;
    if (span <= 5) return 5;
    if (span <= 7) return 7;
    if (span <= 9) return 9;
    return 0;
}

bool finite_taps(const double *taps, int n) {
    for (int i = 0; i < 3 * n; ++i)
        if (!std::isfinite(taps[i])) return false;
    return true;
}

int check_image_args(const void *in, int idt, const void *out, int odt, int B, int H, int W, int C,
                     int boundary) {
    if (!in || !out) return fail(SKC_EBADARG, "null image pointer");
    if (B < 1 || H < 1 || W < 1) return fail(SKC_EBADARG, "image dimensions must be positive");
    if (C < 1 || C > 4) return fail(SKC_EBADARG, "channels must be 1..4");
    if ((idt != SKC_F32 && idt != SKC_F16) || (odt != SKC_F32 && odt != SKC_F16))
        return fail(SKC_EBADARG, "dtype must be SKC_F32 or SKC_F16");
    if (boundary != SKC_ZERO && boundary != SKC_CLAMP)
        return fail(SKC_EBADARG, "boundary must be SKC_ZERO or SKC_CLAMP");
    if ((long long)H * W >= (1LL << 31)) return fail(SKC_EBADARG, "image too large (H*W >= 2^31)");
    if (B > 65535) return fail(SKC_EBADARG, "batch must be <= 65535 frames per call");
    return SKC_OK;
}

template <typename TI, typename TO>
__global__ void convert_kernel(const TI *__restrict__ in, TO *__restrict__ out, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        IO<TO>::st(out + i, IO<TI>::ld(in + i));
}

// Layout/dtype conversion between HWC and planar CHW.  Each thread moves 4
// consecutive pixels: on the HWC side that is 4*C contiguous elements
// (vectorised 16-byte accesses when aligned), on the planar side 4 contiguous
// elements of each of the C planes.
template <typename T> struct Vec4;
template <> struct Vec4<float> {
    static __device__ __forceinline__ void ld(const float *p, float *v) {
        const float4 t = *reinterpret_cast<const float4 *>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    static __device__ __forceinline__ void st(float *p, const float *v) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <> struct Vec4<__half> {
    static __device__ __forceinline__ void ld(const __half *p, float *v) {
        const uint2 t = *reinterpret_cast<const uint2 *>(p);
        const __half2 a = *reinterpret_cast<const __half2 *>(&t.x), b = *reinterpret_cast<const __half2 *>(&t.y);
        const float2 fa = __half22float2(a), fb = __half22float2(b);
        v[0] = fa.x; v[1] = fa.y; v[2] = fb.x; v[3] = fb.y;
    }
    static __device__ __forceinline__ void st(__half *p, const float *v) {
        const __half2 a = __floats2half2_rn(v[0], v[1]), b = __floats2half2_rn(v[2], v[3]);
        uint2 t;
        t.x = *reinterpret_cast<const unsigned *>(&a);
        t.y = *reinterpret_cast<const unsigned *>(&b);
        *reinterpret_cast<uint2 *>(p) = t;
    }
};

template <int C, typename TI, typename TO, bool IN_PL, bool OUT_PL>
__global__ void __launch_bounds__(256) relayout_kernel(const TI *__restrict__ in, TO *__restrict__ out, int B,
                                                       long long hw, int vec) {
    const long long nq = (long long)B * ((hw + 3) / 4);
    const long long qpf = (hw + 3) / 4;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
         q += (long long)gridDim.x * blockDim.x) {
        const long long b = q / qpf, p0 = (q - b * qpf) * 4;
        const long long fb = b * hw * C;
        const int np = (int)min(4LL, hw - p0);
        float v[4][4];
        // gather 4 pixels x C channels
        if (IN_PL) {
            _Pragma("unroll") for (int c = 0; c < C; ++c) {
                const TI *src = in + fb + c * hw + p0;
                if (vec && np == 4) {
                    float t[4];
                    Vec4<TI>::ld(src, t);
                    _Pragma("unroll") for (int k = 0; k < 4; ++k) v[k][c] = t[k];
                } else {
                    _Pragma("unroll") for (int k = 0; k < 4; ++k) if (k < np) v[k][c] = IO<TI>::ld(src + k);
                }
            }
        } else {
            const TI *src = in + fb + p0 * C;
            if (vec && np == 4) {
                float t[4 * C];
                _Pragma("unroll") for (int j = 0; j < C; ++j) Vec4<TI>::ld(src + 4 * j, t + 4 * j);
                _Pragma("unroll") for (int k = 0; k < 4; ++k)
                    _Pragma("unroll") for (int c = 0; c < C; ++c) v[k][c] = t[k * C + c];
            } else {
                _Pragma("unroll") for (int k = 0; k < 4; ++k) if (k < np)
                    _Pragma("unroll") for (int c = 0; c < C; ++c) v[k][c] = IO<TI>::ld(src + k * C + c);
            }
        }
        if (OUT_PL) {
            _Pragma("unroll") for (int c = 0; c < C; ++c) {
                TO *dst = out + fb + c * hw + p0;
                if (vec && np == 4) {
                    const float t[4] = {v[0][c], v[1][c], v[2][c], v[3][c]};
                    Vec4<TO>::st(dst, t);
                } else {
                    _Pragma("unroll") for (int k = 0; k < 4; ++k) if (k < np) IO<TO>::st(dst + k, v[k][c]);
                }
            }
        } else {
            TO *dst = out + fb + p0 * C;
            if (vec && np == 4) {
                float t[4 * C];
                _Pragma("unroll") for (int k = 0; k < 4; ++k)
                    _Pragma("unroll") for (int c = 0; c < C; ++c) t[k * C + c] = v[k][c];
                _Pragma("unroll") for (int j = 0; j < C; ++j) Vec4<TO>::st(dst + 4 * j, t + 4 * j);
            } else {
                _Pragma("unroll") for (int k = 0; k < 4; ++k) if (k < np)
                    _Pragma("unroll") for (int c = 0; c < C; ++c) IO<TO>::st(dst + k * C + c, v[k][c]);
            }
        }
    }
}

int relayout(const void *in, int idt, bool in_pl, void *out, int odt, bool out_pl, int B, int H, int W,
             int C, cudaStream_t s) {
    const long long hw = (long long)H * W;
    const unsigned grid = (unsigned)std::min<long long>((B * ((hw + 3) / 4) + 255) / 256, 148 * 16);
    // 16-byte (fp32) / 8-byte (fp16) vector accesses need hw % 4 == 0 and aligned bases
    const size_t ia = idt == SKC_F32 ? 16 : 8, oa = odt == SKC_F32 ? 16 : 8;
    const int vec = (hw % 4 == 0) && ((uintptr_t)in % ia == 0) && ((uintptr_t)out % oa == 0);
#define SKC_RL(TI, TO, IP, OP)                                                                          \
    switch (C) {                                                                                        \
        case 1: relayout_kernel<1, TI, TO, IP, OP><<<grid, 256, 0, s>>>((const TI *)in, (TO *)out, B, hw, vec); break; \
        case 2: relayout_kernel<2, TI, TO, IP, OP><<<grid, 256, 0, s>>>((const TI *)in, (TO *)out, B, hw, vec); break; \
        case 3: relayout_kernel<3, TI, TO, IP, OP><<<grid, 256, 0, s>>>((const TI *)in, (TO *)out, B, hw, vec); break; \
        default: relayout_kernel<4, TI, TO, IP, OP><<<grid, 256, 0, s>>>((const TI *)in, (TO *)out, B, hw, vec); break; \
    }
    if (!in_pl && out_pl && odt == SKC_F16) {
        if (idt != SKC_F16) return fail(SKC_EBADARG, "planar fp16 relayout takes fp16 HWC");
        SKC_RL(__half, __half, false, true);
    } else if (in_pl && !out_pl && idt == SKC_F16) {
        if (odt != SKC_F16) return fail(SKC_EBADARG, "planar fp16 relayout writes fp16 HWC");
        SKC_RL(__half, __half, true, false);
    } else if (!in_pl && out_pl) {
        if (idt == SKC_F32) { SKC_RL(float, float, false, true); } else { SKC_RL(__half, float, false, true); }
    } else if (in_pl && !out_pl) {
        if (odt == SKC_F32) { SKC_RL(float, float, true, false); } else { SKC_RL(float, __half, true, false); }
    } else {
        return fail(SKC_EBADARG, "relayout converts between HWC and planar");
    }
#undef SKC_RL
    SKC_LAUNCH_CHECK("relayout_kernel");
    return SKC_OK;
}

// Chain I/O policy: 0 = the first layer reads HWC and the last writes HWC
// directly; 1 = planar everywhere with relayout passes at both ends; 2 = only
// the output side goes through a relayout pass.  Default (-1): relayout the
// input too when it is fp16 (the per-channel fp16 gather is the slow case).
static int chain_policy_env() {
    static const int v = [] {
        const char *e = std::getenv("SKC_CHAIN_IO");
        return e ? std::atoi(e) : -1;
    }();
    return v;
}
static int chain_policy(int in_dtype) {
    const int v = chain_policy_env();
    if (v >= 0) return v;
    return in_dtype == SKC_F16 ? 1 : 2;
}

// SKC_TAP_HWC_STAGE=0: chains end with planar + relayout even when the last
// layer is a tap layer (whose kernel can write HWC through its staged epilogue).
static bool tap_hwc_stage_enabled() {
    static const bool v = [] {
        const char *e = std::getenv("SKC_TAP_HWC_STAGE");
        return !(e && e[0] == '0');
    }();
    return v;
}

// Would a chain's last layer (planar fp32 in, HWC out) run the tap kernel,
// which writes HWC itself through its staged epilogue?  Mirrors the routing
// of layer_t -> try_stencil -> launch_taps.
static bool last_layer_direct(int H, int W, int C, const double *taps, int S, int boundary) {
    if (!tap_hwc_stage_enabled() || S > kLMaxTaps) return false;
    int np;
    double wpo;
    if (sparse_plan(taps, S, &np, &wpo)) return true;  // the sparse stencil has the same staged epilogue
    const Plan pl = plan_taps(taps, S);
    if (dense_allowed()) {
        const int sx = pl.dx_max - pl.dx_min + 1, sy = pl.dy_max - pl.dy_min + 1;
        const int D = dense_size_for(std::max(sx, sy));
        if (D != 0 && D * D < 4 * S) return false;
    }
    int dx_min = 1 << 30, dx_max = -(1 << 30), dy_min = 1 << 30, dy_max = -(1 << 30);
    for (int i = 0; i < S; ++i) {
        dx_min = std::min(dx_min, pl.ix[i]);
        dx_max = std::max(dx_max, pl.ix[i] + 1);
        dy_min = std::min(dy_min, pl.iy[i]);
        dy_max = std::max(dy_max, pl.iy[i] + 1);
    }
    const LGeom g5 = make_geom(H, W, C, boundary, 0, kTTW, kTWY * 8 * 5, dx_min, dx_max, dy_min, dy_max);
    return (size_t)g5.rows * g5.pitch * sizeof(float) <= (size_t)kMaxSmem;
}

// The chain's I/O passes (see chain_policy); by default the output relayout
// is skipped when the last layer runs the tap kernel's staged HWC epilogue.
static int chain_mid_dtype(int in_dtype, int out_dtype, const int *layout, int L);

static void chain_io(const double *taps, const int *layout, int L, long long total, int H, int W, int C,
                     int in_dtype, int boundary, bool *pre, bool *post, int out_dtype = -1) {
    if (out_dtype < 0) out_dtype = in_dtype;
    const int pol = chain_policy(in_dtype);
    *pre = pol == 1;
    *post = pol == 1 || pol == 2;
    // an fp16 head that runs as the all-channel generated stencil reads the
    // HWC input itself (coalesced), so the input relayout pass goes
    if (*pre && chain_policy_env() < 0 && in_dtype == SKC_F16 &&
        chain_mid_dtype(in_dtype, out_dtype, layout, L) == SKC_F16 && sparse_head_allc(taps, layout[0], C, false))
        *pre = false;
    if (*post && chain_policy_env() < 0) {
        const double *lt = taps + 3 * (total - layout[L - 1]);
        if (last_layer_direct(H, W, C, lt, layout[L - 1], boundary)) *post = false;
    }
}

// Dtype of a chain's planar intermediates: fp16 when the chain's storage is
// fp16 on both ends (config 3: "fp16 storage, fp32 accumulation"; each layer
// still accumulates in fp32 and rounds once on store), else fp32.
// SKC_HALF_MID=0 keeps fp32 intermediates for fp16 chains.
static bool half_mid_enabled() {
    static const bool v = [] {
        const char *e = std::getenv("SKC_HALF_MID");
        return !(e && e[0] == '0');
    }();
    return v;
}
static int chain_mid_dtype(int in_dtype, int out_dtype, const int *layout, int L) {
    if (!half_mid_enabled() || in_dtype != SKC_F16 || out_dtype != SKC_F16) return SKC_F32;
    for (int l = 0; l < L; ++l)
        if (layout[l] > kLMaxTaps) return SKC_F32;
    return SKC_F16;
}

// HWC output layer with the long-layer fp16 fallback (fp32 temporary + convert).
static int last_layer(const void *in, int idt, bool in_pl, void *out, int odt, int B, int H, int W,
                      int C, const double *taps, int S, int boundary, cudaStream_t s) {
    int rc = layer_dispatch(in, idt, in_pl, out, odt, false, B, H, W, C, taps, S, boundary, s);
    if (rc != -1) return rc;
    const long long n = (long long)B * H * W * C;
    void *tmp = nullptr;
    if ((rc = pool_alloc(&tmp, (size_t)n * sizeof(float), s))) return rc;
    rc = layer_dispatch(in, idt, in_pl, tmp, SKC_F32, false, B, H, W, C, taps, S, boundary, s);
    if (rc == SKC_OK) {
        const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148 * 32);
        convert_kernel<float, __half><<<grid, 256, 0, s>>>((const float *)tmp, (__half *)out, n);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = cuda_fail(e, "convert_kernel");
    }
    pool_free(tmp, s);
    return rc;
}

}  // namespace skc

using namespace skc;

extern "C" {

int skc_max_taps(void) { return kLMaxTaps; }

int skc_layer_fwd(const void *in, int in_dtype, void *out, int out_dtype, int B, int H, int W,
                  int C, const double *taps, int S, int boundary, void *stream) {
    int rc = check_image_args(in, in_dtype, out, out_dtype, B, H, W, C, boundary);
    if (rc) return rc;
    if (S < 1 || !taps) return fail(SKC_EBADARG, "sparse layer needs at least one sample");
    if (!finite_taps(taps, S)) return fail(SKC_EBADARG, "sparse layer parameters must be finite");
    return last_layer(in, in_dtype, false, out, out_dtype, B, H, W, C, taps, S, boundary,
                      (cudaStream_t)stream);
}

int skc_layer_fwd_ex(const void *in, int in_dtype, int in_layout, void *out, int out_dtype,
                     int out_layout, int B, int H, int W, int C, const double *taps, int S,
                     int boundary, void *stream) {
    int rc = check_image_args(in, in_dtype, out, out_dtype, B, H, W, C, boundary);
    if (rc) return rc;
    if (S < 1 || !taps) return fail(SKC_EBADARG, "sparse layer needs at least one sample");
    if (!finite_taps(taps, S)) return fail(SKC_EBADARG, "sparse layer parameters must be finite");
    if ((in_layout != SKC_HWC && in_layout != SKC_CHW) || (out_layout != SKC_HWC && out_layout != SKC_CHW))
        return fail(SKC_EBADARG, "layout must be SKC_HWC or SKC_CHW");
    cudaStream_t s = (cudaStream_t)stream;
    if (out_layout == SKC_HWC)
        return last_layer(in, in_dtype, in_layout == SKC_CHW, out, out_dtype, B, H, W, C, taps, S, boundary, s);
    rc = layer_dispatch(in, in_dtype, in_layout == SKC_CHW, out, out_dtype, true, B, H, W, C, taps, S,
                        boundary, s);
    return rc == -1 ? fail(SKC_EBADARG, "planar output of a long layer must be fp32") : rc;
}

int skc_relayout(const void *in, int in_dtype, int in_layout, void *out, int out_dtype, int out_layout,
                 int B, int H, int W, int C, void *stream) {
    int rc = check_image_args(in, in_dtype, out, out_dtype, B, H, W, C, SKC_ZERO);
    if (rc) return rc;
    if (in_layout == out_layout) return fail(SKC_EBADARG, "relayout needs different layouts");
    return relayout(in, in_dtype, in_layout == SKC_CHW, out, out_dtype, out_layout == SKC_CHW, B, H, W, C,
                    (cudaStream_t)stream);
}

int skc_layer_plan(const double *taps, int S, int H, int W, int C, int boundary, int *kind, int *param) {
    if (!taps || S < 1 || H < 1 || W < 1 || C < 1 || !kind || !param) return fail(SKC_EBADARG, "bad layer arguments");
    const Plan pl = plan_taps(taps, S);
    int np;
    double wpo;
    // planar-input layers (the chain's inner and last layers); a single frame of this shape
    if (sparse_plan(taps, S, &np, &wpo, sparse_small_launch(1, H, W, C, false))) {
        *kind = 3;
        *param = np;
        return SKC_OK;
    }
    if (dense_allowed()) {
        const int sx = pl.dx_max - pl.dx_min + 1, sy = pl.dy_max - pl.dy_min + 1;
        const int D = dense_size_for(std::max(sx, sy));
        if (D != 0 && D * D < 4 * S) {
            *kind = 1;
            *param = D;
            return SKC_OK;
        }
    }
    const int n = std::min(S, kLMaxTaps);
    int dx_min = 1 << 30, dx_max = -(1 << 30), dy_min = 1 << 30, dy_max = -(1 << 30);
    for (int i = 0; i < n; ++i) {
        dx_min = std::min(dx_min, pl.ix[i]);
        dx_max = std::max(dx_max, pl.ix[i] + 1);
        dy_min = std::min(dy_min, pl.iy[i]);
        dy_max = std::max(dy_max, pl.iy[i] + 1);
    }
    const int KR = tap_kr_for(H, W, C, boundary, 0, dx_min, dx_max, dy_min, dy_max, n);
    const LGeom g = make_geom(H, W, C, boundary, 0, kTTW, kTWY * 8 * KR, dx_min, dx_max, dy_min, dy_max);
    if ((size_t)g.rows * g.pitch * sizeof(float) > (size_t)kMaxSmem) {
        *kind = 2;
        *param = 0;
    } else {
        *kind = 0;
        *param = KR;
    }
    return SKC_OK;
}

int skc_layer_pair_fwd(const void *in, void *out, int B, int H, int W, int C, const double *taps0, int S0,
                       const double *taps1, int S1, int boundary, void *stream) {
    if (!taps0 || !taps1 || S0 < 1 || S1 < 1) return fail(SKC_EBADARG, "sparse layer needs at least one sample");
    if (!finite_taps(taps0, S0) || !finite_taps(taps1, S1))
        return fail(SKC_EBADARG, "sparse layer parameters must be finite");
    if (!in && !out) {
        if (B < 1 || H < 1 || W < 1 || C < 1) return fail(SKC_EBADARG, "bad image arguments");
        return sparse_pair(nullptr, nullptr, B, H, W, C, taps0, S0, taps1, S1, boundary, nullptr) == SKC_OK ? SKC_OK
                                                                                                     : SKC_ENOTTAKEN;
    }
    int rc = check_image_args(in, SKC_F32, out, SKC_F32, B, H, W, C, boundary);
    if (rc) return rc;
    rc = sparse_pair((const float *)in, (float *)out, B, H, W, C, taps0, S0, taps1, S1, boundary,
                     (cudaStream_t)stream);
    return rc == -1 ? SKC_ENOTTAKEN : rc;
}

int skc_pair_compile_check(const double *taps0, int S0, const double *taps1, int S1) {
    if (!taps0 || !taps1 || S0 < 1 || S1 < 1) return fail(SKC_EBADARG, "bad layer arguments");
    return sparse_pair_compile_check(taps0, S0, taps1, S1);
}

int skc_chain_relayouts(const double *taps, const int *layout, int L, int H, int W, int C, int in_dtype,
                        int boundary) {
    if (!taps || !layout || L < 1 || H < 1 || W < 1 || C < 1) return fail(SKC_EBADARG, "bad chain arguments");
    if (L == 1) return 0;
    long long total = 0;
    for (int l = 0; l < L; ++l) {
        if (layout[l] < 1) return fail(SKC_EBADARG, "sparse layer needs at least one sample");
        total += layout[l];
    }
    bool pre, post;
    chain_io(taps, layout, L, total, H, W, C, in_dtype, boundary, &pre, &post);
    return (pre ? 1 : 0) | (post ? 2 : 0);
}

int skc_chain_mid_dtype(const int *layout, int L, int in_dtype, int out_dtype) {
    if (!layout || L < 1) return fail(SKC_EBADARG, "bad chain arguments");
    return chain_mid_dtype(in_dtype, out_dtype, layout, L);
}

int skc_chain_fwd(const void *in, int in_dtype, void *out, int out_dtype, int B, int H, int W,
                  int C, const double *taps, const int *layout, int L, int boundary, void *stream) {
    int rc = check_image_args(in, in_dtype, out, out_dtype, B, H, W, C, boundary);
    if (rc) return rc;
    if (L < 1 || !layout || !taps) return fail(SKC_EBADARG, "kernel complex needs at least one layer");
    long long total = 0;
    for (int l = 0; l < L; ++l) {
        if (layout[l] < 1) return fail(SKC_EBADARG, "sparse layer needs at least one sample");
        total += layout[l];
    }
    if (!finite_taps(taps, (int)total)) return fail(SKC_EBADARG, "sparse layer parameters must be finite");
    cudaStream_t s = (cudaStream_t)stream;
    // Kawase ladders on fp16 RGBA: one fused separable launch (skc_kawase.cu)
    rc = kawase_chain(in, in_dtype, out, out_dtype, B, H, W, C, taps, layout, L, boundary, s);
    if (rc != -1) return rc;
    if (L == 1) return last_layer(in, in_dtype, false, out, out_dtype, B, H, W, C, taps, layout[0], boundary, s);
    rc = fused_chain(in, in_dtype, out, out_dtype, B, H, W, C, taps, layout, L, boundary, s);
    if (rc != -1) return rc;
    rc = SKC_OK;
    // intermediates: fp32 planar (B, C, H, W), ping-pong; see chain_policy()
    bool pre, post;
    chain_io(taps, layout, L, total, H, W, C, in_dtype, boundary, &pre, &post, out_dtype);
    const int mid = chain_mid_dtype(in_dtype, out_dtype, layout, L);
    const size_t n = (size_t)B * H * W * C;
    void *buf[2] = {nullptr, nullptr};
    const int nbuf = (L > 2 || post || pre) ? 2 : 1;
    for (int i = 0; i < nbuf; ++i) {
        rc = pool_alloc(&buf[i], n * dtype_size(mid), s);
        if (rc) { for (int j = 0; j < i; ++j) pool_free(buf[j], s); return rc; }
    }
    const void *src = in;
    int sdt = in_dtype;
    bool spl = false;
    int k = 0;  // next scratch buffer
    if (pre) {
        rc = relayout(in, in_dtype, false, buf[0], mid, true, B, H, W, C, s);
        src = buf[0];
        sdt = mid;
        spl = true;
        k = 1;
    }
    const double *tp = taps;
    int l0 = 0;
    // layers 0 and 1 as one fused launch (skc_sparse.cu sparse_pair): fp32
    // HWC in, fp32 planar out, the intermediate kept in shared memory
    if (!pre && L >= 3 && in_dtype == SKC_F32 && mid == SKC_F32) {
        const int prc = sparse_pair((const float *)in, (float *)buf[k], B, H, W, C, taps, layout[0],
                                    taps + 3 * layout[0], layout[1], boundary, s);
        if (prc != -1) {
            rc = prc;
            src = buf[k];
            sdt = mid;
            spl = true;
            k ^= 1;
            tp += 3 * (layout[0] + layout[1]);
            l0 = 2;
        }
    }
    for (int l = l0; l < L && rc == SKC_OK; ++l) {
        const bool last = l == L - 1;
        if (last && !post) {
            rc = last_layer(src, sdt, spl, out, out_dtype, B, H, W, C, tp, layout[l], boundary, s);
        } else {
            rc = layer_dispatch(src, sdt, spl, buf[k], mid, true, B, H, W, C, tp, layout[l], boundary, s);
            src = buf[k];
            sdt = mid;
            spl = true;
            k ^= 1;
        }
        tp += 3 * layout[l];
    }
    if (rc == SKC_OK && post) rc = relayout(src, sdt, true, out, out_dtype, false, B, H, W, C, s);
    for (int i = 0; i < nbuf; ++i) pool_free(buf[i], s);
    return rc;
}

}  // extern "C"
