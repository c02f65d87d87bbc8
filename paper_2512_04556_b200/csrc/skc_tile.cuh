// skc_tile.cuh -- halo-tile staging shared by the uniform-layer kernels.
#pragma once

#include "skc_common.cuh"

namespace skc {

constexpr int kMaxSmem = 227 * 1024;

struct Geom {
    int H, W;
    int dx0, dy0;      // global offset of smem (0,0) relative to the tile origin
    int pitch, rows;   // smem tile geometry (pitch odd)
    int boundary;
    int accumulate;    // out += result (fp32 outputs only; tap chunking)
    long long in_fs, out_fs;  // frame strides (elements)
};

// ------------------------------------------------------------ tile loader ---
// Stage rows [gy0, gy0+rows) x cols [gx0, gx0+pitch) of an HWC image into C
// planar smem planes; out-of-image texels are 0 (ZERO) or the clamped texel.
// fp32: every element is one 4-byte cp.async (LDGSTS) with zero-fill for
// out-of-image texels, so the whole halo tile is in flight at once instead of
// one dependent LDG->STS round trip per element.  fp16: batches of 8
// independent loads per thread before the stores.
__device__ __forceinline__ void cp_async4(float *dst, const float *src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
                 "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
// Variants on a precomputed shared-window address (no per-call cvta), always valid.
__device__ __forceinline__ void cp_async4s(unsigned saddr, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(src));
}
__device__ __forceinline__ void cp_async8s(unsigned saddr, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(src));
}

template <int C, typename TI>
__device__ __forceinline__ void load_tile(float *s, const TI *__restrict__ in, int H, int W,
                                          int boundary, int gx0, int gy0, int pitch, int rows) {
    const int plane = rows * pitch;
    const int rowlen = pitch * C;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const bool clamp = boundary == SKC_CLAMP;
    if constexpr (sizeof(TI) == 4) {
        for (int r = warp; r < rows; r += nw) {
            int gy = gy0 + r;
            bool rowin = gy >= 0 && gy < H;
            if (clamp) { gy = min(max(gy, 0), H - 1); rowin = true; }
            gy = min(max(gy, 0), H - 1);  // keep the (unused) source address in bounds
            const float *src = reinterpret_cast<const float *>(in) + (long long)gy * W * C;
            float *dst = s + r * pitch;
#pragma unroll 4
            for (int e = lane; e < rowlen; e += 32) {
                const int col = e / C;
                const int c = e - col * C;
                const int gx = gx0 + col;
                const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                const int gxc = min(max(gx, 0), W - 1);
                cp_async4(dst + c * plane + col, src + (long long)gxc * C + c, ok);
            }
        }
        cp_async_wait_all();
    } else {
        constexpr int U = 8;
        for (int r = warp; r < rows; r += nw) {
            int gy = gy0 + r;
            bool rowin = gy >= 0 && gy < H;
            if (clamp) { gy = min(max(gy, 0), H - 1); rowin = true; }
            gy = min(max(gy, 0), H - 1);
            const TI *src = in + (long long)gy * W * C;
            float *dst = s + r * pitch;
            for (int e0 = lane; e0 < rowlen; e0 += 32 * U) {
                float v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = e0 + 32 * u;
                    const int col = e / C;
                    const int c = e - col * C;
                    const int gx = gx0 + col;
                    const bool ok = e < rowlen && (clamp || (rowin && gx >= 0 && gx < W));
                    const int gxc = min(max(gx, 0), W - 1);
                    v[u] = ok ? IO<TI>::ld(src + (long long)gxc * C + c) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int e = e0 + 32 * u;
                    if (e < rowlen) {
                        const int col = e / C;
                        dst[(e - col * C) * plane + col] = v[u];
                    }
                }
            }
        }
    }
}

template <typename TO>
__device__ __forceinline__ void store_px(TO *p, float v, int accumulate) {
    IO<TO>::st(p, v);
}
template <>
__device__ __forceinline__ void store_px<float>(float *p, float v, int accumulate) {
    *p = accumulate ? (*p + v) : v;
}


// Dense-stencil path (skc_layer.cu): a layer whose merged corner footprint
// fits a D x D window (D <= 9) and costs fewer FMAs than 4 per tap.
constexpr int kMaxDense = 9;
int dense_size_for(int span);  // smallest compiled D >= span, or 0

// Fused small-reach chain (skc_fused.cu); -1 = not eligible.
int fused_chain(const void *in, int idt, void *out, int odt, int B, int H, int W, int C,
                const double *taps, const int *layout, int L, int boundary, cudaStream_t s,
                bool dry = false);

// Layer-specialised sparse stencils compiled at run time (skc_sparse.cu):
// planar input, planar or HWC output; -1 = not taken.
int sparse_layer(const void *in, bool in_f32, void *out, bool out_f32, bool out_pl, int B, int H, int W, int C,
                 const double *taps, int S, int boundary, cudaStream_t s, bool in_hwc = false);
bool sparse_plan(const double *taps, int S, int *npos, double *words_per_out, bool small = false);
bool sparse_small_launch(int B, int H, int W, int C, bool allc);
bool sparse_head_allc(const double *taps, int S, int C, bool f32);
// A chain's layers 0 and 1 fused (fp32 HWC -> fp32 planar); -1 = not taken,
// in == nullptr: plan query.
int sparse_pair(const float *in, float *out, int B, int H, int W, int C, const double *t1, int S1, const double *t2,
                int S2, int boundary, cudaStream_t s);
int sparse_pair_compile_check(const double *t1, int S1, const double *t2, int S2);
// Fused separable Kawase chain (skc_kawase.cu): -1 when the chain or image
// does not qualify; with in == nullptr a plan query (SKC_OK = would run).
int kawase_chain(const void *in, int idt, void *out, int odt, int B, int H, int W, int C, const double *taps,
                 const int *layout, int L, int boundary, cudaStream_t s);

// Argument checks shared by the image entry points (skc_layer.cu).
int check_image_args(const void *in, int idt, const void *out, int odt, int B, int H, int W, int C,
                     int boundary);
bool finite_taps(const double *taps, int n);

}  // namespace skc
