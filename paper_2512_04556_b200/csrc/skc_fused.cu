// skc_fused.cu -- fused L-layer chain for complexes with a small total reach
// (sm_100a).  SURVEY K2/K3: the Kawase-style "Gaussian fast path" (config 3,
// 6 layers x 4 taps, total corner reach 21 px) is memory-bound when every
// layer round-trips HBM (32 B/px/layer planar fp32); fused, the image is read
// once and written once (16 B/px for fp16 RGBA).
//
// Reference: engine.apply_complex (engine.py:173-178) over
// apply_sparse_layer (160-170); boundary re-applied at every layer.
//
// One CTA = one output tile (64 x 48) of one frame, all channels in turn.
// Per channel the tile plus the chain's accumulated corner-reach halo is
// staged in shared memory (fp32), then each layer l computes exactly the
// rectangle layer l+1 needs (needed_L = tile, needed_l = needed_{l+1} +
// footprint_l) into the other plane with the same KR x 8 register blocking as
// the tap kernel (conflict-free LDS.32: odd pitch, odd KR).  Texels of a
// layer output that fall outside the image are reset to zero (ZERO) or to the
// clamped texel (CLAMP) before the next layer reads them, which is exactly the
// per-layer boundary rule of the unfused chain.  The last layer's tile is
// staged per channel and written back as whole HWC pixels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "skc_tile.cuh"

namespace skc {

constexpr int kFuTW = 64, kFuTH = 48;
constexpr int kFuKR = 3;                 // rows per thread block (odd)
constexpr int kFuMaxL = 8, kFuMaxTaps = 16;
constexpr int kFuPadX = 9, kFuPadY = kFuKR + 1;   // plane padding read by partial blocks

struct FuLayer {
    float4 cw[kFuMaxTaps];
    int ix[kFuMaxTaps], iy[kFuMaxTaps];
    int n;
    int x0, y0, w, h;   // output rectangle of this layer in plane coordinates
};

struct FuParams {
    int H, W, C, L, boundary;
    int hlx, hly;       // plane (0,0) <-> global (tx0 - hlx, ty0 - hly)
    int pitch, rows;    // plane geometry (pitch odd)
    int in_w, in_h;     // rectangle of layer 0 input (plane coords, origin 0)
    FuLayer layer[kFuMaxL];
};

template <typename TI>
__device__ __forceinline__ void fu_load(float *plane, const TI *__restrict__ frame, const FuParams &q,
                                        int c, int gx0, int gy0) {
    const bool clamp = q.boundary == SKC_CLAMP;
    const int n = q.in_w * q.in_h;
    for (int e0 = threadIdx.x; e0 < n; e0 += blockDim.x * 4) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * blockDim.x;
            v[u] = 0.f;
            if (e < n) {
                const int r = e / q.in_w, col = e - r * q.in_w;
                int gy = gy0 + r, gx = gx0 + col;
                const bool ok = clamp || (gy >= 0 && gy < q.H && gx >= 0 && gx < q.W);
                gy = min(max(gy, 0), q.H - 1);
                gx = min(max(gx, 0), q.W - 1);
                if (ok) v[u] = IO<TI>::ld(frame + ((long long)gy * q.W + gx) * q.C + c);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < n) {
                const int r = e / q.in_w, col = e - r * q.in_w;
                plane[r * q.pitch + col] = v[u];
            }
        }
    }
}

// One layer: out rectangle of `L` from src plane into dst plane.
__device__ __forceinline__ void fu_layer(const float *src, float *dst, const FuLayer &L, int pitch) {
    constexpr int KR = kFuKR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int lx = lane & 3, ly = lane >> 2;
    const int wtw = (L.w + 31) / 32, wth = (L.h + 8 * KR - 1) / (8 * KR);
    for (int wt = warp; wt < wtw * wth; wt += nw) {
        const int wy = wt / wtw, wx = wt - wy * wtw;
        const int x0 = L.x0 + wx * 32 + lx * 8, y0 = L.y0 + wy * 8 * KR + ly * KR;
        if (x0 >= L.x0 + L.w || y0 >= L.y0 + L.h) continue;
        float acc[KR][8];
#pragma unroll
        for (int r = 0; r < KR; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[r][j] = 0.f;
        for (int i = 0; i < L.n; ++i) {
            const float4 w = L.cw[i];
            const float *p = src + (y0 + L.iy[i]) * pitch + (x0 + L.ix[i]);
            float a[9], b[9];
#pragma unroll
            for (int j = 0; j < 9; ++j) a[j] = p[j];
#pragma unroll
            for (int r = 0; r < KR; ++r) {
#pragma unroll
                for (int j = 0; j < 9; ++j) b[j] = p[(r + 1) * pitch + j];
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
#pragma unroll
        for (int r = 0; r < KR; ++r) {
            if (y0 + r >= L.y0 + L.h) continue;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (x0 + j < L.x0 + L.w) dst[(y0 + r) * pitch + x0 + j] = acc[r][j];
        }
    }
}

// Re-apply the boundary rule to the out-of-image part of a layer output.
__device__ __forceinline__ void fu_fixup(float *plane, const FuLayer &L, const FuParams &q, int gx0, int gy0) {
    const int n = L.w * L.h;
    const bool clamp = q.boundary == SKC_CLAMP;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int r = e / L.w, col = e - r * L.w;
        const int py = L.y0 + r, px = L.x0 + col;
        const int gy = gy0 + py, gx = gx0 + px;
        if (gy >= 0 && gy < q.H && gx >= 0 && gx < q.W) continue;
        float v = 0.f;
        if (clamp) {
            const int cy = min(max(gy, 0), q.H - 1) - gy0, cx = min(max(gx, 0), q.W - 1) - gx0;
            v = plane[cy * q.pitch + cx];
        }
        plane[py * q.pitch + px] = v;
    }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) fused_chain_kernel(const TI *__restrict__ in, TO *__restrict__ out,
                                                          const __grid_constant__ FuParams q) {
    extern __shared__ __align__(16) float smem[];
    const int plane_sz = q.rows * q.pitch;
    float *P[2] = {smem, smem + plane_sz};
    TO *stage = reinterpret_cast<TO *>(smem + 2 * plane_sz);   // (kFuTH, kFuTW, C) output tile
    const int C = q.C;
    const int tx0 = blockIdx.x * kFuTW, ty0 = blockIdx.y * kFuTH;
    const long long fs = (long long)q.H * q.W * C;
    in += blockIdx.z * fs;
    out += blockIdx.z * fs;
    const int gx0 = tx0 - q.hlx, gy0 = ty0 - q.hly;   // global coords of plane (0,0)
    const bool edge = gx0 < 0 || gy0 < 0 || gx0 + q.in_w > q.W || gy0 + q.in_h > q.H;
    for (int c = 0; c < C; ++c) {
        fu_load<TI>(P[0], in, q, c, gx0, gy0);
        __syncthreads();
        int cur = 0;
        for (int l = 0; l < q.L; ++l) {
            const FuLayer &L = q.layer[l];
            fu_layer(P[cur], P[cur ^ 1], L, q.pitch);
            __syncthreads();
            cur ^= 1;
            if (edge && l + 1 < q.L) {
                fu_fixup(P[cur], L, q, gx0, gy0);
                __syncthreads();
            }
        }
        // final rectangle == the tile
        const FuLayer &Lf = q.layer[q.L - 1];
        for (int e = threadIdx.x; e < kFuTW * kFuTH; e += blockDim.x) {
            const int r = e / kFuTW, col = e - r * kFuTW;
            IO<TO>::st(stage + e * C + c, P[cur][(Lf.y0 + r) * q.pitch + Lf.x0 + col]);
        }
        __syncthreads();
    }
    const int th = min(kFuTH, q.H - ty0), tw = min(kFuTW, q.W - tx0);
    for (int e = threadIdx.x; e < th * tw * C; e += blockDim.x) {
        const int r = e / (tw * C), rem = e - r * tw * C;
        out[((long long)(ty0 + r) * q.W + tx0) * C + rem] = stage[(r * kFuTW) * C + rem];
    }
}

// Host: eligibility and launch.  Returns -1 when the chain is not eligible
// (caller falls back to the per-layer path).
int fused_chain(const void *in, int idt, void *out, int odt, int B, int H, int W, int C,
                const double *taps, const int *layout, int L, int boundary, cudaStream_t s, bool dry) {
    static const bool enabled = [] {
        const char *e = std::getenv("SKC_FUSED");
        return !(e && e[0] == '0');
    }();
    if (!enabled || L < 2 || L > kFuMaxL || B > 65535) return -1;
    FuParams q;
    std::memset(&q, 0, sizeof(q));
    q.H = H;
    q.W = W;
    q.C = C;
    q.L = L;
    q.boundary = boundary;
    // per-layer footprints
    std::vector<int> dxmin(L), dxmax(L), dymin(L), dymax(L);
    const double *tp = taps;
    long long fma = 0;
    for (int l = 0; l < L; ++l) {
        if (layout[l] > kFuMaxTaps) return -1;
        FuLayer &F = q.layer[l];
        F.n = layout[l];
        for (int i = 0; i < F.n; ++i) {
            const double ox = tp[3 * i], oy = tp[3 * i + 1], w = tp[3 * i + 2];
            const double fx0 = std::floor(ox), fy0 = std::floor(oy);
            const double fx = ox - fx0, fy = oy - fy0;
            F.ix[i] = (int)fx0;
            F.iy[i] = (int)fy0;
            F.cw[i] = make_float4((float)(w * (1.0 - fx) * (1.0 - fy)), (float)(w * fx * (1.0 - fy)),
                                  (float)(w * (1.0 - fx) * fy), (float)(w * fx * fy));
            dxmin[l] = i ? std::min(dxmin[l], F.ix[i]) : F.ix[i];
            dxmax[l] = i ? std::max(dxmax[l], F.ix[i] + 1) : F.ix[i] + 1;
            dymin[l] = i ? std::min(dymin[l], F.iy[i]) : F.iy[i];
            dymax[l] = i ? std::max(dymax[l], F.iy[i] + 1) : F.iy[i] + 1;
        }
        tp += 3 * layout[l];
        fma += 4LL * layout[l];
    }
    // needed rectangles, backwards from the tile (relative to the tile origin)
    std::vector<int> nx0(L + 1), nx1(L + 1), ny0(L + 1), ny1(L + 1);  // [lo, hi)
    nx0[L] = 0;
    nx1[L] = kFuTW;
    ny0[L] = 0;
    ny1[L] = kFuTH;
    for (int l = L - 1; l >= 0; --l) {
        nx0[l] = nx0[l + 1] + dxmin[l];
        nx1[l] = nx1[l + 1] + dxmax[l];
        ny0[l] = ny0[l + 1] + dymin[l];
        ny1[l] = ny1[l + 1] + dymax[l];
    }
    // every layer's rectangle must contain the tile (footprints straddle the
    // origin) so clamped edge texels are always computed
    for (int l = 0; l <= L; ++l)
        if (nx0[l] > 0 || ny0[l] > 0 || nx1[l] < kFuTW || ny1[l] < kFuTH) return -1;
    q.hlx = -nx0[0];
    q.hly = -ny0[0];
    q.in_w = nx1[0] - nx0[0];
    q.in_h = ny1[0] - ny0[0];
    // fusion pays when the halo is small relative to the tile (redundant work)
    const double redund = (double)q.in_w * q.in_h / (kFuTW * kFuTH);
    if (redund > 4.0) return -1;
    for (int l = 0; l < L; ++l) {
        FuLayer &F = q.layer[l];
        F.x0 = nx0[l + 1] + q.hlx;
        F.y0 = ny0[l + 1] + q.hly;
        F.w = nx1[l + 1] - nx0[l + 1];
        F.h = ny1[l + 1] - ny0[l + 1];
        // taps read plane (y + iy, x + ix): offsets stay as is (plane origin fixed)
    }
    int pitch = q.in_w + kFuPadX;
    if ((pitch & 1) == 0) ++pitch;
    q.pitch = pitch;
    q.rows = q.in_h + kFuPadY;
    const size_t smem = 2 * (size_t)q.rows * q.pitch * sizeof(float) +
                        (size_t)kFuTW * kFuTH * C * (odt == SKC_F16 ? 2 : 4);
    if (smem > (size_t)kMaxSmem) return -1;
    if (dry) return SKC_OK;
    dim3 grid(ceil_div(W, kFuTW), ceil_div(H, kFuTH), B);
#define SKC_FU(TI, TO)                                                                                  \
    do {                                                                                                \
        auto kern = fused_chain_kernel<TI, TO>;                                                         \
        static cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem); \
        if (attr != cudaSuccess) return cuda_fail(attr, "cudaFuncSetAttribute(fused)");               \
        kern<<<grid, 256, smem, s>>>(static_cast<const TI *>(in), static_cast<TO *>(out), q);          \
    } while (0)
    if (idt == SKC_F32 && odt == SKC_F32) SKC_FU(float, float);
    else if (idt == SKC_F16 && odt == SKC_F16) SKC_FU(__half, __half);
    else if (idt == SKC_F16 && odt == SKC_F32) SKC_FU(__half, float);
    else SKC_FU(float, __half);
#undef SKC_FU
    SKC_LAUNCH_CHECK("fused_chain_kernel");
    (void)fma;
    return SKC_OK;
}

}  // namespace skc

extern "C" int skc_chain_is_fused(const double *taps, const int *layout, int L, int H, int W, int C,
                                  int out_dtype) {
    if (!taps || !layout || L < 1) return 0;
    return skc::fused_chain(nullptr, SKC_F32, nullptr, out_dtype, 1, H, W, C, taps, layout, L, SKC_ZERO,
                            nullptr, true) == SKC_OK;
}
