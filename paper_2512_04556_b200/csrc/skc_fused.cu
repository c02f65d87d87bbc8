// skc_fused.cu -- fused L-layer chain for complexes with a small total reach
// (sm_100a).  SURVEY K2/K3: the Kawase-style "Gaussian fast path" (config 3,
// 6 layers x 4 taps, total corner reach 21 px) is memory-bound when every
// layer round-trips HBM (32 B/px/layer planar fp32); fused, each planar pixel
// is read once and written once.
//
// Reference: engine.apply_complex (engine.py:173-178) over
// apply_sparse_layer (160-170); the boundary rule is re-applied at every layer.
//
// One CTA (512 threads) = one (128 x 80 output tile, channel) pair of a
// planar fp32 frame.  The tile plus the chain's accumulated corner-reach halo
// is staged once in shared memory (cp.async); every layer then computes
// exactly the rectangle the next layer needs (needed_L = tile, needed_l =
// needed_{l+1} + footprint_l) into the other plane, with the tap kernel's
// 5 x 8 register blocks and LDS.64 windows (pitch = 2 mod 4; taps sorted by
// window parity per layer).  Texels of a layer output outside the image are
// reset to zero (ZERO) or to the clamped texel (CLAMP) before the next layer
// reads them -- the unfused chain's per-layer boundary rule.  The last layer
// writes the tile straight to the planar output.  HWC callers go through the
// vectorised relayout passes on both sides.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "skc_tile.cuh"

namespace skc {

constexpr int kF2TW = 128, kF2TH = 80, kF2KR = 5;
constexpr int kF2Threads = 512;
constexpr int kF2MaxL = 8, kF2MaxTaps = 16;

struct F2Layer {
    float4 cw[kF2MaxTaps];
    int ix[kF2MaxTaps], iy[kF2MaxTaps];
    int n, n_even;          // taps [0, n_even) have even window columns
    int x0, y0, w, h;       // output rectangle (plane coordinates)
};

struct F2Params {
    int H, W, C, L, boundary;
    int hlx, hly;           // plane (0,0) <-> global (tx0 - hlx, ty0 - hly)
    int in_w, in_h;
    F2Layer layer[kF2MaxL];
};

__device__ __forceinline__ void f2_row(const float *q, float (&v)[9], bool odd) {
    if (!odd) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 t = reinterpret_cast<const float2 *>(q)[k];
            v[2 * k] = t.x;
            v[2 * k + 1] = t.y;
        }
        v[8] = q[8];
    } else {
        v[0] = q[0];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 t = reinterpret_cast<const float2 *>(q + 1)[k];
            v[2 * k + 1] = t.x;
            v[2 * k + 2] = t.y;
        }
    }
}

template <int KR>
__device__ __forceinline__ void f2_taps(float (&acc)[KR][8], const float *base, int pitch, const F2Layer &L,
                                        int i0, int i1, bool odd) {
    for (int i = i0; i < i1; ++i) {
        const float4 w = L.cw[i];
        const float *p = base + L.iy[i] * pitch + L.ix[i];
        float a[9], b[9];
        f2_row(p, a, odd);
#pragma unroll
        for (int r = 0; r < KR; ++r) {
            f2_row(p + (r + 1) * pitch, b, odd);
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
}

__global__ void __launch_bounds__(kF2Threads) fused2_kernel(const float *__restrict__ in, float *__restrict__ out,
                                                            const __grid_constant__ F2Params q, int pitch,
                                                            int rows) {
    extern __shared__ __align__(16) float smem[];
    constexpr int KR = kF2KR;
    const int plane = rows * pitch;
    const int C = q.C;
    const int c = blockIdx.x % C;
    const int tx0 = (blockIdx.x / C) * kF2TW, ty0 = blockIdx.y * kF2TH;
    const long long hw = (long long)q.H * q.W;
    const float *src = in + ((long long)blockIdx.z * C + c) * hw;
    float *dstp = out + ((long long)blockIdx.z * C + c) * hw;
    const int gx0 = tx0 - q.hlx, gy0 = ty0 - q.hly;
    const bool clamp = q.boundary == SKC_CLAMP;

    // stage the region (8-byte cp.async where a pair lies inside a row of the image)
    {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        const bool pairs_ok = (q.W & 1) == 0 && (gx0 & 1) == 0;
        for (int r = warp; r < q.in_h; r += nw) {
            int gy = gy0 + r;
            const bool rowin = clamp || (gy >= 0 && gy < q.H);
            gy = min(max(gy, 0), q.H - 1);
            const float *row = src + (long long)gy * q.W;
            float *d = smem + r * pitch;
            for (int pc = lane; 2 * pc < q.in_w; pc += 32) {
                const int col = 2 * pc, gx = gx0 + col;
                if (pairs_ok && gx >= 0 && gx + 1 < q.W) {
                    const unsigned da = (unsigned)__cvta_generic_to_shared(d + col);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(da), "l"(row + gx),
                                 "r"(rowin ? 8 : 0));
                } else {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int x = gx + u;
                        const bool ok = clamp || (rowin && x >= 0 && x < q.W);
                        cp_async4(d + col + u, row + min(max(x, 0), q.W - 1), ok);
                    }
                }
            }
        }
        cp_async_wait_all();
    }
    __syncthreads();

    const bool edge = gx0 < 0 || gy0 < 0 || gx0 + q.in_w > q.W || gy0 + q.in_h > q.H;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane & 3, ly = lane >> 2;
    int cur = 0;
    for (int l = 0; l < q.L; ++l) {
        const F2Layer &L = q.layer[l];
        const float *P = smem + cur * plane;
        float *Q = smem + (cur ^ 1) * plane;
        const bool last = l == q.L - 1;
        const int wtw = (L.w + 31) / 32, wth = (L.h + 8 * KR - 1) / (8 * KR);
        for (int wt = warp; wt < wtw * wth; wt += kF2Threads / 32) {
            const int wy = wt / wtw, wx = wt - wy * wtw;
            const int x0 = L.x0 + wx * 32 + lx * 8, y0 = L.y0 + wy * 8 * KR + ly * KR;
            if (x0 >= L.x0 + L.w || y0 >= L.y0 + L.h) continue;
            float acc[KR][8];
#pragma unroll
            for (int r = 0; r < KR; ++r)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[r][j] = 0.f;
            const float *base = P + y0 * pitch + x0;
            f2_taps<KR>(acc, base, pitch, L, 0, L.n_even, false);
            f2_taps<KR>(acc, base, pitch, L, L.n_even, L.n, true);
            if (!last) {
#pragma unroll
                for (int r = 0; r < KR; ++r) {
                    if (y0 + r >= L.y0 + L.h) continue;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (x0 + j < L.x0 + L.w) Q[(y0 + r) * pitch + x0 + j] = acc[r][j];
                }
            } else {
                // final rectangle == the tile: write the planar output
#pragma unroll
                for (int r = 0; r < KR; ++r) {
                    const int gy = ty0 + (y0 - L.y0) + r;
                    if (y0 + r >= L.y0 + L.h || gy >= q.H) continue;
                    const int gx = tx0 + (x0 - L.x0);
                    float *o = dstp + (long long)gy * q.W + gx;
                    if (gx + 7 < q.W && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
                        reinterpret_cast<float4 *>(o)[0] = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
                        reinterpret_cast<float4 *>(o)[1] = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            if (gx + j < q.W) o[j] = acc[r][j];
                    }
                }
            }
        }
        if (last) break;
        __syncthreads();
        cur ^= 1;
        if (edge) {
            // re-apply the boundary rule to the out-of-image part of this layer's output
            float *R = smem + cur * plane;
            const int n = L.w * L.h;
            for (int e = threadIdx.x; e < n; e += blockDim.x) {
                const int r = e / L.w, col = e - r * L.w;
                const int py = L.y0 + r, px = L.x0 + col;
                const int gy = gy0 + py, gx = gx0 + px;
                if (gy >= 0 && gy < q.H && gx >= 0 && gx < q.W) continue;
                float v = 0.f;
                if (clamp) {
                    const int cy = min(max(gy, 0), q.H - 1) - gy0, cx = min(max(gx, 0), q.W - 1) - gx0;
                    v = R[cy * pitch + cx];
                }
                R[py * pitch + px] = v;
            }
            __syncthreads();
        }
    }
}

int relayout(const void *in, int idt, bool in_pl, void *out, int odt, bool out_pl, int B, int H, int W,
             int C, cudaStream_t s);

// Plan one fused group of layers (taps/layout point at its first layer):
// fills q, the plane pitch/rows and the shared-memory size.  Returns false
// when the group is not eligible.
static bool plan_fused(const double *taps, const int *layout, int L, int H, int W, int C, int boundary,
                       F2Params &q, int &pitch, int &rows, size_t &smem) {
    if (L < 1 || L > kF2MaxL) return false;
    std::memset(&q, 0, sizeof(q));
    q.H = H;
    q.W = W;
    q.C = C;
    q.L = L;
    q.boundary = boundary;
    std::vector<int> dxmin(L), dxmax(L), dymin(L), dymax(L);
    const double *tp = taps;
    for (int l = 0; l < L; ++l) {
        if (layout[l] > kF2MaxTaps) return false;
        F2Layer &F = q.layer[l];
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
    }
    // needed rectangles, backwards from the tile (relative to the tile origin)
    std::vector<int> nx0(L + 1), nx1(L + 1), ny0(L + 1), ny1(L + 1);
    nx0[L] = 0;
    nx1[L] = kF2TW;
    ny0[L] = 0;
    ny1[L] = kF2TH;
    for (int l = L - 1; l >= 0; --l) {
        nx0[l] = nx0[l + 1] + dxmin[l];
        nx1[l] = nx1[l + 1] + dxmax[l];
        ny0[l] = ny0[l + 1] + dymin[l];
        ny1[l] = ny1[l + 1] + dymax[l];
    }
    // every rectangle must contain the tile (footprints straddle the origin),
    // so clamped edge texels are always computed
    for (int l = 0; l <= L; ++l)
        if (nx0[l] > 0 || ny0[l] > 0 || nx1[l] < kF2TW || ny1[l] < kF2TH) return false;
    // keep the plane origin even so 8-byte loads and LDS.64 windows align
    q.hlx = -nx0[0] + ((-nx0[0]) & 1);
    q.hly = -ny0[0];
    q.in_w = nx1[0] + q.hlx;
    q.in_h = ny1[0] - ny0[0];
    const double redund = (double)(nx1[0] - nx0[0]) * q.in_h / (kF2TW * kF2TH);
    if (redund > 4.0) return false;
    pitch = q.in_w + 10;          // odd-tap windows read 9 columns past the block origin
    pitch = (pitch + 3) & ~3;
    pitch += 2;                   // pitch = 2 mod 4
    rows = q.in_h + kF2KR + 1;
    smem = 2 * (size_t)rows * pitch * sizeof(float);
    if (smem > (size_t)kMaxSmem) return false;
    for (int l = 0; l < L; ++l) {
        F2Layer &F = q.layer[l];
        F.x0 = nx0[l + 1] + q.hlx;
        F.y0 = ny0[l + 1] + q.hly;
        F.w = nx1[l + 1] - nx0[l + 1];
        F.h = ny1[l + 1] - ny0[l + 1];
        // sort taps by window-column parity: block columns are x0 + 8k, x0 = F.x0
        const F2Layer S = F;
        int k = 0;
        for (int pass = 0; pass < 2; ++pass) {
            if (pass == 1) F.n_even = k;
            for (int i = 0; i < S.n; ++i) {
                if (((F.x0 + S.ix[i]) & 1) != pass) continue;
                F.cw[k] = S.cw[i];
                F.ix[k] = S.ix[i];
                F.iy[k] = S.iy[i];
                ++k;
            }
        }
    }
    return true;
}

// Layers per fused launch: SKC_FUSED_GROUP (default: the whole chain).
static int fused_group() {
    static const int v = [] {
        const char *e = std::getenv("SKC_FUSED_GROUP");
        return e ? std::max(1, std::atoi(e)) : 0;
    }();
    return v;
}

// Host: eligibility, plan and launch (relayout -> fused planar groups ->
// relayout).  Returns -1 when the chain is not eligible.
int fused_chain(const void *in, int idt, void *out, int odt, int B, int H, int W, int C,
                const double *taps, const int *layout, int L, int boundary, cudaStream_t s, bool dry) {
    // Opt-in (SKC_FUSED=1): on B200 the fused launch (1 CTA/SM at 186 KB of
    // planes, 2x redundant halo work) measured slower than the unfused
    // planar chain for config 3 (24.9 vs 15.9 ms for 32 frames).
    static const bool enabled = [] {
        const char *e = std::getenv("SKC_FUSED");
        return e && e[0] == '1';
    }();
    if (!enabled || L < 2 || B > 65535) return -1;
    const int G = fused_group() ? fused_group() : L;
    const int ng = (L + G - 1) / G;
    std::vector<F2Params> qs(ng);
    std::vector<int> pitches(ng), rowss(ng);
    std::vector<size_t> smems(ng);
    const double *tp = taps;
    for (int gi = 0; gi < ng; ++gi) {
        const int l0 = gi * G, nl = std::min(G, L - l0);
        if (!plan_fused(tp, layout + l0, nl, H, W, C, boundary, qs[gi], pitches[gi], rowss[gi], smems[gi]))
            return -1;
        for (int l = l0; l < l0 + nl; ++l) tp += 3 * layout[l];
    }
    if (dry) return SKC_OK;

    // planar staging around the fused launches (ping-pong between groups)
    const size_t n = (size_t)B * H * W * C;
    void *buf[2] = {nullptr, nullptr};
    int rc = pool_alloc(&buf[0], n * sizeof(float), s);
    if (rc) return rc;
    if ((rc = pool_alloc(&buf[1], n * sizeof(float), s))) { pool_free(buf[0], s); return rc; }
    rc = relayout(in, idt, false, buf[0], SKC_F32, true, B, H, W, C, s);
    if (rc == SKC_OK) rc = smem_optin((const void *)fused2_kernel, kMaxSmem);
    int k = 0;
    for (int gi = 0; gi < ng && rc == SKC_OK; ++gi, k ^= 1) {
        dim3 grid(ceil_div(W, kF2TW) * C, ceil_div(H, kF2TH), B);
        fused2_kernel<<<grid, kF2Threads, smems[gi], s>>>((const float *)buf[k], (float *)buf[k ^ 1], qs[gi],
                                                          pitches[gi], rowss[gi]);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = cuda_fail(e, "fused2_kernel");
    }
    if (rc == SKC_OK) rc = relayout(buf[k], SKC_F32, true, out, odt, false, B, H, W, C, s);
    pool_free(buf[0], s);
    pool_free(buf[1], s);
    return rc;
}

}  // namespace skc

extern "C" int skc_chain_is_fused(const double *taps, const int *layout, int L, int H, int W, int C,
                                  int out_dtype) {
    if (!taps || !layout || L < 1) return 0;
    if (skc::kawase_chain(nullptr, out_dtype, nullptr, out_dtype, 1, H, W, C, taps, layout, L, SKC_ZERO, nullptr) ==
        SKC_OK)
        return 1;
    return skc::fused_chain(nullptr, SKC_F32, nullptr, out_dtype, 1, H, W, C, taps, layout, L, SKC_ZERO,
                            nullptr, true) == SKC_OK;
}
