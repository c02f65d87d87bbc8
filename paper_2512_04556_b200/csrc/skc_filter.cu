// skc_filter.cu -- uniform sparse-layer filtering and the spatially varying
// filter for sm_100a.
//
// Reference chains replaced (all citations into /root/reference/pkg/src/sparsekern):
//   apply_sparse_layer (engine.py:160-170) -> sample_shifted (118-130) ->
//   _accum_shift (106-115); apply_complex (173-178);
//   sv_filter (svfilter.py:171-203) -> sv_filter_compiled/_sv_pass_loop
//   (_fastpath.py:97-150).
//
// Design:
//   * A uniform layer's tap has the same fractional part at every pixel, so it
//     is 4 integer shifts with constant corner weights.  The host folds each
//     tap into (corner-00 smem offset, 4 weights) in the kernel-parameter
//     constant bank; the kernel never computes floor/frac.
//   * A CTA stages its output tile plus the layer's exact corner-reach halo in
//     shared memory (planar per channel, zero- or clamp-filled at the image
//     edge, so the inner loop is branch-free), then every thread computes a
//     KR x MC register block: per tap and channel it reads a (KR+1) x (MC+1)
//     window and issues 4*KR*MC FFMAs.  KR is odd and the row pitch is odd,
//     which makes the 32 lanes' window origins fall in 32 distinct banks.
//   * Tiles whose halo would not fit shared memory fall back to a direct
//     global-gather kernel (L1/L2 cached) with identical arithmetic.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "skc_tile.cuh"

namespace skc {

constexpr int kMaxTaps = 256;        // taps per launch; longer layers are chunked

struct TapTable {
    float4 cw[kMaxTaps];  // corner weights (00, 10, 01, 11) = w(1-fx)(1-fy), w fx(1-fy), ...
    int off[kMaxTaps];    // shared-memory offset of corner 00 relative to the thread base
    int ix[kMaxTaps];     // integer parts (direct kernel)
    int iy[kMaxTaps];
    int n;
};

// ----------------------------------------------------- uniform layer kernel ---
template <int C, int KR, int MC, int WX, int WY, typename TI, typename TO>
__global__ void __launch_bounds__(WX *WY * 32)
    layer_tile_kernel(const TI *__restrict__ in, TO *__restrict__ out, const Geom g,
                      const __grid_constant__ TapTable tt) {
    extern __shared__ float smem[];
    constexpr int LX = 32 / MC;
    constexpr int LY = MC;
    constexpr int TW = WX * 32;
    constexpr int TH = WY * LY * KR;
    const int tx0 = blockIdx.x * TW, ty0 = blockIdx.y * TH;
    in += (long long)blockIdx.z * g.in_fs;
    out += (long long)blockIdx.z * g.out_fs;

    load_tile<C, TI>(smem, in, g.H, g.W, g.boundary, tx0 + g.dx0, ty0 + g.dy0, g.pitch, g.rows);
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane % LX, ly = lane / LX, wx = warp % WX, wy = warp / WX;
    const int col0 = wx * 32 + lx * MC;
    const int row0 = wy * LY * KR + ly * KR;
    const int plane = g.rows * g.pitch;
    const int pitch = g.pitch;
    const float *sb = smem + row0 * pitch + col0;

    float acc[C][KR][MC];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int r = 0; r < KR; ++r)
#pragma unroll
            for (int j = 0; j < MC; ++j) acc[c][r][j] = 0.f;

#pragma unroll 1
    for (int i = 0; i < tt.n; ++i) {
        const float4 w = tt.cw[i];
        const float *p = sb + tt.off[i];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const float *pc = p + c * plane;
            float a[MC + 1], b[MC + 1];
#pragma unroll
            for (int j = 0; j <= MC; ++j) a[j] = pc[j];
#pragma unroll
            for (int r = 0; r < KR; ++r) {
                const float *q = pc + (r + 1) * pitch;
#pragma unroll
                for (int j = 0; j <= MC; ++j) b[j] = q[j];
#pragma unroll
                for (int j = 0; j < MC; ++j) {
                    float v = acc[c][r][j];
                    v = fmaf(w.x, a[j], v);
                    v = fmaf(w.y, a[j + 1], v);
                    v = fmaf(w.z, b[j], v);
                    v = fmaf(w.w, b[j + 1], v);
                    acc[c][r][j] = v;
                }
#pragma unroll
                for (int j = 0; j <= MC; ++j) a[j] = b[j];
            }
        }
    }

#pragma unroll
    for (int r = 0; r < KR; ++r) {
        const int gy = ty0 + row0 + r;
        if (gy >= g.H) continue;
        TO *orow = out + (long long)gy * g.W * C;
#pragma unroll
        for (int j = 0; j < MC; ++j) {
            const int gx = tx0 + col0 + j;
            if (gx >= g.W) continue;
#pragma unroll
            for (int c = 0; c < C; ++c) store_px<TO>(orow + (long long)gx * C + c, acc[c][r][j], g.accumulate);
        }
    }
}

// Direct global-gather fallback (halo too large for shared memory).
template <int C, typename TI, typename TO>
__global__ void __launch_bounds__(256)
    layer_direct_kernel(const TI *__restrict__ in, TO *__restrict__ out, const Geom g,
                        const __grid_constant__ TapTable tt) {
    const long long npx = (long long)g.H * g.W;
    in += (long long)blockIdx.y * g.in_fs;
    out += (long long)blockIdx.y * g.out_fs;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npx;
         p += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(p / g.W), x = (int)(p - (long long)y * g.W);
        float acc[C];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = 0.f;
        for (int i = 0; i < tt.n; ++i) {
            const float4 w = tt.cw[i];
            const float cw[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int yy = y + tt.iy[i] + (k >> 1), xx = x + tt.ix[i] + (k & 1);
                if (g.boundary == SKC_CLAMP) {
                    yy = min(max(yy, 0), g.H - 1);
                    xx = min(max(xx, 0), g.W - 1);
                } else if (yy < 0 || yy >= g.H || xx < 0 || xx >= g.W) {
                    continue;
                }
                const TI *src = in + ((long long)yy * g.W + xx) * C;
#pragma unroll
                for (int c = 0; c < C; ++c) acc[c] = fmaf(cw[k], IO<TI>::ld(src + c), acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) store_px<TO>(out + p * C + c, acc[c], g.accumulate);
    }
}

template <typename TI, typename TO>
__global__ void convert_kernel(const TI *__restrict__ in, TO *__restrict__ out, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        IO<TO>::st(out + i, IO<TI>::ld(in + i));
}

// ------------------------------------------------------------ host: plans ---
struct LayerPlan {
    std::vector<float4> cw;
    std::vector<int> ix, iy;
    int dx_min = 0, dx_max = 0, dy_min = 0, dy_max = 0;
};

// sample_shifted (engine.py:118-130): ix = floor(ox), fx = ox - ix, corner
// weights in (00, 10, 01, 11) order, computed in float64 then rounded once.
static LayerPlan make_plan(const double *taps, int S) {
    LayerPlan p;
    p.cw.resize(S);
    p.ix.resize(S);
    p.iy.resize(S);
    for (int i = 0; i < S; ++i) {
        const double ox = taps[3 * i], oy = taps[3 * i + 1], w = taps[3 * i + 2];
        const double fx0 = std::floor(ox), fy0 = std::floor(oy);
        const double fx = ox - fx0, fy = oy - fy0;
        p.ix[i] = (int)fx0;
        p.iy[i] = (int)fy0;
        p.cw[i] = make_float4((float)(w * (1.0 - fx) * (1.0 - fy)), (float)(w * fx * (1.0 - fy)),
                              (float)(w * (1.0 - fx) * fy), (float)(w * fx * fy));
        if (i == 0 || p.ix[i] < p.dx_min) p.dx_min = p.ix[i];
        if (i == 0 || p.ix[i] + 1 > p.dx_max) p.dx_max = p.ix[i] + 1;
        if (i == 0 || p.iy[i] < p.dy_min) p.dy_min = p.iy[i];
        if (i == 0 || p.iy[i] + 1 > p.dy_max) p.dy_max = p.iy[i] + 1;
    }
    return p;
}

static bool finite_taps(const double *taps, int S) {
    for (int i = 0; i < 3 * S; ++i)
        if (!std::isfinite(taps[i])) return false;
    return true;
}

// Tile configuration of the uniform-layer kernel.
constexpr int kKR = 5, kMC = 4, kWX = 2, kWY = 4;
constexpr int kTW = kWX * 32, kTH = kWY * kMC * kKR;

template <int C, typename TI, typename TO>
static int launch_layer_t(const void *in, void *out, int B, int H, int W, const LayerPlan &lp,
                          int t0, int t1, int boundary, int accumulate, cudaStream_t s) {
    TapTable tt;
    const int n = t1 - t0;
    tt.n = n;
    int dx_min = 0, dx_max = 0, dy_min = 0, dy_max = 0;
    for (int i = 0; i < n; ++i) {
        const int ix = lp.ix[t0 + i], iy = lp.iy[t0 + i];
        if (i == 0 || ix < dx_min) dx_min = ix;
        if (i == 0 || ix + 1 > dx_max) dx_max = ix + 1;
        if (i == 0 || iy < dy_min) dy_min = iy;
        if (i == 0 || iy + 1 > dy_max) dy_max = iy + 1;
    }
    Geom g;
    g.H = H;
    g.W = W;
    g.boundary = boundary;
    g.accumulate = accumulate;
    g.in_fs = (long long)H * W * C;
    g.out_fs = (long long)H * W * C;
    g.dx0 = dx_min;
    g.dy0 = dy_min;
    int pitch = kTW + (dx_max - dx_min);
    if ((pitch & 1) == 0) ++pitch;
    g.pitch = pitch;
    g.rows = kTH + (dy_max - dy_min);
    const size_t smem = (size_t)C * g.rows * g.pitch * sizeof(float);
    for (int i = 0; i < n; ++i) {
        tt.cw[i] = lp.cw[t0 + i];
        tt.ix[i] = lp.ix[t0 + i];
        tt.iy[i] = lp.iy[t0 + i];
        tt.off[i] = (lp.iy[t0 + i] - dy_min) * pitch + (lp.ix[t0 + i] - dx_min);
    }
    const TI *pin = static_cast<const TI *>(in);
    TO *pout = static_cast<TO *>(out);
    if (smem <= (size_t)kMaxSmem) {
        auto kern = layer_tile_kernel<C, kKR, kMC, kWX, kWY, TI, TO>;
        static bool attr_set = false;
        if (!attr_set) {
            SKC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
            attr_set = true;
        }
        dim3 grid(ceil_div(W, kTW), ceil_div(H, kTH), B);
        kern<<<grid, kWX * kWY * 32, smem, s>>>(pin, pout, g, tt);
        SKC_LAUNCH_CHECK("layer_tile_kernel");
    } else {
        const long long npx = (long long)H * W;
        dim3 grid((unsigned)std::min<long long>((npx + 255) / 256, 148 * 16), B);
        layer_direct_kernel<C, TI, TO><<<grid, 256, 0, s>>>(pin, pout, g, tt);
        SKC_LAUNCH_CHECK("layer_direct_kernel");
    }
    return SKC_OK;
}

template <int C>
static int launch_layer_c(const void *in, int idt, void *out, int odt, int B, int H, int W,
                          const LayerPlan &lp, int t0, int t1, int boundary, int acc,
                          cudaStream_t s) {
    if (idt == SKC_F32 && odt == SKC_F32)
        return launch_layer_t<C, float, float>(in, out, B, H, W, lp, t0, t1, boundary, acc, s);
    if (idt == SKC_F16 && odt == SKC_F32)
        return launch_layer_t<C, __half, float>(in, out, B, H, W, lp, t0, t1, boundary, acc, s);
    if (idt == SKC_F32 && odt == SKC_F16)
        return launch_layer_t<C, float, __half>(in, out, B, H, W, lp, t0, t1, boundary, acc, s);
    return launch_layer_t<C, __half, __half>(in, out, B, H, W, lp, t0, t1, boundary, acc, s);
}

static int launch_layer(const void *in, int idt, void *out, int odt, int B, int H, int W, int C,
                        const LayerPlan &lp, int t0, int t1, int boundary, int acc,
                        cudaStream_t s) {
    switch (C) {
        case 1: return launch_layer_c<1>(in, idt, out, odt, B, H, W, lp, t0, t1, boundary, acc, s);
        case 2: return launch_layer_c<2>(in, idt, out, odt, B, H, W, lp, t0, t1, boundary, acc, s);
        case 3: return launch_layer_c<3>(in, idt, out, odt, B, H, W, lp, t0, t1, boundary, acc, s);
        case 4: return launch_layer_c<4>(in, idt, out, odt, B, H, W, lp, t0, t1, boundary, acc, s);
        default: return fail(SKC_EBADARG, "channels must be 1..4");
    }
}

static int convert(const void *in, int idt, void *out, int odt, long long n, cudaStream_t s) {
    const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148 * 32);
    if (idt == SKC_F32 && odt == SKC_F16)
        convert_kernel<float, __half><<<grid, 256, 0, s>>>((const float *)in, (__half *)out, n);
    else if (idt == SKC_F16 && odt == SKC_F32)
        convert_kernel<__half, float><<<grid, 256, 0, s>>>((const __half *)in, (float *)out, n);
    else if (idt == SKC_F32)
        convert_kernel<float, float><<<grid, 256, 0, s>>>((const float *)in, (float *)out, n);
    else
        convert_kernel<__half, __half><<<grid, 256, 0, s>>>((const __half *)in, (__half *)out, n);
    SKC_LAUNCH_CHECK("convert_kernel");
    return SKC_OK;
}

// One full layer from `in` to `out` with tap chunking.  Chunks after the first
// accumulate into an fp32 destination; an fp16 destination with more than
// kMaxTaps taps goes through an fp32 temporary.
// Dense-stencil eligibility: merged corner footprint D x D (D <= 9) with
// D*D < 4*S FMAs per pixel.  SKC_DENSE=0 in the environment disables it.
static bool dense_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("SKC_DENSE");
        return !(e && e[0] == '0');
    }();
    return on;
}

static bool try_dense(const double *taps, int S, const LayerPlan &lp, DenseTable &dt) {
    if (!dense_enabled()) return false;
    const int sx = lp.dx_max - lp.dx_min + 1, sy = lp.dy_max - lp.dy_min + 1;
    const int D = dense_size_for(std::max(sx, sy));
    if (D == 0 || D * D >= 4 * S) return false;
    double k[kMaxDense * kMaxDense] = {0.0};
    for (int i = 0; i < S; ++i) {
        const double ox = taps[3 * i], oy = taps[3 * i + 1], w = taps[3 * i + 2];
        const double fx0 = std::floor(ox), fy0 = std::floor(oy);
        const double fx = ox - fx0, fy = oy - fy0;
        const double cw[4] = {w * (1.0 - fx) * (1.0 - fy), w * fx * (1.0 - fy), w * (1.0 - fx) * fy,
                              w * fx * fy};
        for (int c = 0; c < 4; ++c) {
            const int a = (int)fy0 + (c >> 1) - lp.dy_min, b = (int)fx0 + (c & 1) - lp.dx_min;
            k[a * D + b] += cw[c];
        }
    }
    dt.D = D;
    for (int e = 0; e < kMaxDense * kMaxDense; ++e) dt.k[e] = e < D * D ? (float)k[e] : 0.f;
    return true;
}

static int run_layer(const void *in, int idt, void *out, int odt, int B, int H, int W, int C,
                     const double *taps, int S, int boundary, cudaStream_t s) {
    LayerPlan lp = make_plan(taps, S);
    DenseTable dt;
    if (try_dense(taps, S, lp, dt))
        return launch_dense(in, idt, out, odt, B, H, W, C, dt, lp.dx_min, lp.dy_min, boundary, s);
    if (S <= kMaxTaps) return launch_layer(in, idt, out, odt, B, H, W, C, lp, 0, S, boundary, 0, s);
    void *dst = out;
    void *tmp = nullptr;
    const long long n = (long long)B * H * W * C;
    if (odt != SKC_F32) {
        int rc = pool_alloc(&tmp, (size_t)n * sizeof(float), s);
        if (rc) return rc;
        dst = tmp;
    }
    for (int t0 = 0; t0 < S; t0 += kMaxTaps) {
        const int t1 = std::min(S, t0 + kMaxTaps);
        int rc = launch_layer(in, idt, dst, SKC_F32, B, H, W, C, lp, t0, t1, boundary, t0 > 0, s);
        if (rc) return rc;
    }
    if (tmp) {
        int rc = convert(tmp, SKC_F32, out, odt, n, s);
        pool_free(tmp, s);
        if (rc) return rc;
    }
    return SKC_OK;
}

static int check_image_args(const void *in, int idt, const void *out, int odt, int B, int H, int W,
                            int C, int boundary) {
    if (!in || !out) return fail(SKC_EBADARG, "null image pointer");
    if (B < 1 || H < 1 || W < 1) return fail(SKC_EBADARG, "image dimensions must be positive");
    if (C < 1 || C > 4) return fail(SKC_EBADARG, "channels must be 1..4");
    if ((idt != SKC_F32 && idt != SKC_F16) || (odt != SKC_F32 && odt != SKC_F16))
        return fail(SKC_EBADARG, "dtype must be SKC_F32 or SKC_F16");
    if (boundary != SKC_ZERO && boundary != SKC_CLAMP)
        return fail(SKC_EBADARG, "boundary must be SKC_ZERO or SKC_CLAMP");
    if ((long long)H * W >= (1LL << 31)) return fail(SKC_EBADARG, "image too large (H*W >= 2^31)");
    return SKC_OK;
}

// ------------------------------------------------------- SV filter kernel ---
constexpr int kSvTW = 64, kSvTH = 32, kSvPx = 8;  // 256 threads x 8 rows
constexpr int kMaxBasis = 64;

struct SvParams {
    int H, W, Mb, n, boundary;
    int dx0, dy0, pitch, rows;
    long long in_fs, out_fs;
    float ps[kMaxBasis];
};

// svfilter._bracket (svfilter.py:129-137) in fp32 on the fp32 map.
__device__ __forceinline__ void bracket(float p, const SvParams &q, int &k0, int &k1, float &t) {
    if (q.Mb == 1) { k0 = 0; k1 = 0; t = 0.f; return; }
    const float pc = fminf(fmaxf(p, q.ps[0]), q.ps[q.Mb - 1]);
    int k = 0;
    for (int j = 1; j < q.Mb - 1; ++j) k += (q.ps[j] <= pc) ? 1 : 0;
    k0 = k;
    k1 = k + 1;
    t = (pc - q.ps[k]) / (q.ps[k + 1] - q.ps[k]);
}

template <int C, typename TI, typename TO>
__global__ void __launch_bounds__(256)
    sv_tile_kernel(const TI *__restrict__ in, TO *__restrict__ out, const float *__restrict__ pmap,
                   const float4 *__restrict__ table, const __grid_constant__ SvParams q) {
    extern __shared__ float4 smem4[];
    float4 *stab = smem4;  // (Mb, n) entries (ox, oy, w, 0)
    float *tile = reinterpret_cast<float *>(smem4 + q.Mb * q.n);
    const int tx0 = blockIdx.x * kSvTW, ty0 = blockIdx.y * kSvTH;
    for (int i = threadIdx.x; i < q.Mb * q.n; i += blockDim.x) stab[i] = table[i];
    load_tile<C, TI>(tile, in, q.H, q.W, q.boundary, tx0 + q.dx0, ty0 + q.dy0, q.pitch, q.rows);
    __syncthreads();

    const int tx = threadIdx.x & (kSvTW - 1), ty = threadIdx.x / kSvTW;
    const int plane = q.rows * q.pitch, pitch = q.pitch;
    const int gx = tx0 + tx;
    int e0[kSvPx], e1[kSvPx];
    float tt[kSvPx];
    float acc[kSvPx][C];
#pragma unroll
    for (int k = 0; k < kSvPx; ++k) {
        const int gy = ty0 + ty + 4 * k;
        float p = 0.f;
        if (gy < q.H && gx < q.W) p = __ldg(pmap + (long long)gy * q.W + gx);
        int k0, k1;
        bracket(p, q, k0, k1, tt[k]);
        e0[k] = k0 * q.n;
        e1[k] = k1 * q.n;
#pragma unroll
        for (int c = 0; c < C; ++c) acc[k][c] = 0.f;
    }
    // smem (0,0) sits at global (tx0 + dx0, ty0 + dy0)
    const int base0 = (ty - q.dy0) * pitch + (tx - q.dx0);
#pragma unroll 1
    for (int i = 0; i < q.n; ++i) {
#pragma unroll
        for (int k = 0; k < kSvPx; ++k) {
            const float4 a = stab[e0[k] + i];
            const float4 b = stab[e1[k] + i];
            const float t = tt[k], u = 1.f - t;
            // _fastpath.py:109-111: lerp of offsets and weight
            const float ox = u * a.x + t * b.x;
            const float oy = u * a.y + t * b.y;
            const float w = u * a.z + t * b.z;
            const float fx0 = floorf(ox), fy0 = floorf(oy);
            const float fx = ox - fx0, fy = oy - fy0;
            const float wa = w * (1.f - fy), wb = w * fy;
            const float c00 = wa * (1.f - fx), c10 = wa * fx, c01 = wb * (1.f - fx), c11 = wb * fx;
            const int off = base0 + (4 * k + (int)fy0) * pitch + (int)fx0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const float *sp = tile + c * plane + off;
                float v = acc[k][c];
                v = fmaf(c00, sp[0], v);
                v = fmaf(c10, sp[1], v);
                v = fmaf(c01, sp[pitch], v);
                v = fmaf(c11, sp[pitch + 1], v);
                acc[k][c] = v;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kSvPx; ++k) {
        const int gy = ty0 + ty + 4 * k;
        if (gy >= q.H || gx >= q.W) continue;
        TO *o = out + ((long long)gy * q.W + gx) * C;
#pragma unroll
        for (int c = 0; c < C; ++c) IO<TO>::st(o + c, acc[k][c]);
    }
}

template <int C, typename TI, typename TO>
__global__ void __launch_bounds__(256)
    sv_direct_kernel(const TI *__restrict__ in, TO *__restrict__ out, const float *__restrict__ pmap,
                     const float4 *__restrict__ table, const __grid_constant__ SvParams q) {
    const long long npx = (long long)q.H * q.W;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npx;
         p += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(p / q.W), x = (int)(p - (long long)y * q.W);
        int k0, k1;
        float t;
        bracket(__ldg(pmap + p), q, k0, k1, t);
        const float u = 1.f - t;
        float acc[C];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = 0.f;
        for (int i = 0; i < q.n; ++i) {
            const float4 a = __ldg(table + k0 * q.n + i);
            const float4 b = __ldg(table + k1 * q.n + i);
            const float ox = u * a.x + t * b.x, oy = u * a.y + t * b.y, w = u * a.z + t * b.z;
            const float fx0 = floorf(ox), fy0 = floorf(oy);
            const float fx = ox - fx0, fy = oy - fy0;
            const float wa = w * (1.f - fy), wb = w * fy;
            const float cw[4] = {wa * (1.f - fx), wa * fx, wb * (1.f - fx), wb * fx};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int yy = y + (int)fy0 + (k >> 1), xx = x + (int)fx0 + (k & 1);
                if (q.boundary == SKC_CLAMP) {
                    yy = min(max(yy, 0), q.H - 1);
                    xx = min(max(xx, 0), q.W - 1);
                } else if (yy < 0 || yy >= q.H || xx < 0 || xx >= q.W) {
                    continue;
                }
                const TI *src = in + ((long long)yy * q.W + xx) * C;
#pragma unroll
                for (int c = 0; c < C; ++c) acc[c] = fmaf(cw[k], IO<TI>::ld(src + c), acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) IO<TO>::st(out + p * C + c, acc[c]);
    }
}

template <int C, typename TI, typename TO>
static int launch_sv_t(const void *in, void *out, const float *pmap, const float4 *table,
                       SvParams q, cudaStream_t s) {
    const size_t smem = (size_t)q.Mb * q.n * sizeof(float4) + (size_t)C * q.rows * q.pitch * 4;
    const TI *pin = static_cast<const TI *>(in);
    TO *pout = static_cast<TO *>(out);
    if (smem <= (size_t)kMaxSmem) {
        auto kern = sv_tile_kernel<C, TI, TO>;
        static bool attr_set = false;
        if (!attr_set) {
            SKC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
            attr_set = true;
        }
        dim3 grid(ceil_div(q.W, kSvTW), ceil_div(q.H, kSvTH));
        kern<<<grid, 256, smem, s>>>(pin, pout, pmap, table, q);
        SKC_LAUNCH_CHECK("sv_tile_kernel");
    } else {
        const long long npx = (long long)q.H * q.W;
        const unsigned grid = (unsigned)std::min<long long>((npx + 255) / 256, 148 * 16);
        sv_direct_kernel<C, TI, TO><<<grid, 256, 0, s>>>(pin, pout, pmap, table, q);
        SKC_LAUNCH_CHECK("sv_direct_kernel");
    }
    return SKC_OK;
}

template <int C>
static int launch_sv_c(const void *in, int idt, void *out, int odt, const float *pmap,
                       const float4 *table, const SvParams &q, cudaStream_t s) {
    if (idt == SKC_F32 && odt == SKC_F32) return launch_sv_t<C, float, float>(in, out, pmap, table, q, s);
    if (idt == SKC_F16 && odt == SKC_F32) return launch_sv_t<C, __half, float>(in, out, pmap, table, q, s);
    if (idt == SKC_F32 && odt == SKC_F16) return launch_sv_t<C, float, __half>(in, out, pmap, table, q, s);
    return launch_sv_t<C, __half, __half>(in, out, pmap, table, q, s);
}

static int launch_sv(const void *in, int idt, void *out, int odt, int C, const float *pmap,
                     const float4 *table, const SvParams &q, cudaStream_t s) {
    switch (C) {
        case 1: return launch_sv_c<1>(in, idt, out, odt, pmap, table, q, s);
        case 2: return launch_sv_c<2>(in, idt, out, odt, pmap, table, q, s);
        case 3: return launch_sv_c<3>(in, idt, out, odt, pmap, table, q, s);
        case 4: return launch_sv_c<4>(in, idt, out, odt, pmap, table, q, s);
        default: return fail(SKC_EBADARG, "channels must be 1..4");
    }
}

}  // namespace skc

using namespace skc;

extern "C" {

int skc_max_taps(void) { return kMaxTaps; }

int skc_layer_fwd(const void *in, int in_dtype, void *out, int out_dtype, int B, int H, int W,
                  int C, const double *taps, int S, int boundary, void *stream) {
    int rc = check_image_args(in, in_dtype, out, out_dtype, B, H, W, C, boundary);
    if (rc) return rc;
    if (S < 1 || !taps) return fail(SKC_EBADARG, "sparse layer needs at least one sample");
    if (!finite_taps(taps, S)) return fail(SKC_EBADARG, "sparse layer parameters must be finite");
    return run_layer(in, in_dtype, out, out_dtype, B, H, W, C, taps, S, boundary,
                     (cudaStream_t)stream);
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
    const size_t n = (size_t)B * H * W * C;
    void *buf[2] = {nullptr, nullptr};
    const int nbuf = L > 2 ? 2 : (L - 1);
    for (int i = 0; i < nbuf; ++i) {
        rc = pool_alloc(&buf[i], n * sizeof(float), s);
        if (rc) { for (int j = 0; j < i; ++j) pool_free(buf[j], s); return rc; }
    }
    const double *tp = taps;
    for (int l = 0; l < L && rc == SKC_OK; ++l) {
        const void *src = l == 0 ? in : buf[(l - 1) & 1];
        const int sdt = l == 0 ? in_dtype : SKC_F32;
        void *dst = l == L - 1 ? out : buf[l & 1];
        const int ddt = l == L - 1 ? out_dtype : SKC_F32;
        rc = run_layer(src, sdt, dst, ddt, B, H, W, C, tp, layout[l], boundary, s);
        tp += 3 * layout[l];
    }
    for (int i = 0; i < nbuf; ++i) pool_free(buf[i], s);
    return rc;
}

int skc_sv_fwd(const void *in, int in_dtype, void *out, int out_dtype, int H, int W, int C,
               const float *pmap, const double *params, int Mb, const double *basis, int nmax,
               const int *layout, int L, int boundary, void *stream) {
    int rc = check_image_args(in, in_dtype, out, out_dtype, 1, H, W, C, boundary);
    if (rc) return rc;
    if (!pmap || !params || !basis || !layout) return fail(SKC_EBADARG, "null argument");
    if (Mb < 1 || Mb > kMaxBasis) return fail(SKC_EBADARG, "basis size must be 1..64");
    if (L < 1 || nmax < 1) return fail(SKC_EBADARG, "basis needs at least one layer");
    for (int k = 1; k < Mb; ++k)
        if (!(params[k] > params[k - 1])) return fail(SKC_EBADARG, "basis parameters must be strictly increasing");
    for (int l = 0; l < L; ++l)
        if (layout[l] < 1 || layout[l] > nmax) return fail(SKC_EBADARG, "bad basis layout");
    if (!finite_taps(basis, Mb * L * nmax)) return fail(SKC_EBADARG, "basis parameters must be finite");
    cudaStream_t s = (cudaStream_t)stream;

    // per-layer tables (Mb, n_l) of (ox, oy, w, 0) in one device upload
    std::vector<float4> host;
    std::vector<size_t> start(L);
    for (int l = 0; l < L; ++l) {
        start[l] = host.size();
        for (int k = 0; k < Mb; ++k)
            for (int i = 0; i < layout[l]; ++i) {
                const double *e = basis + (((size_t)k * L + l) * nmax + i) * 3;
                host.push_back(make_float4((float)e[0], (float)e[1], (float)e[2], 0.f));
            }
    }
    void *dtab = nullptr;
    rc = pool_alloc(&dtab, host.size() * sizeof(float4), s);
    if (rc) return rc;
    cudaError_t ce = cudaMemcpyAsync(dtab, host.data(), host.size() * sizeof(float4),
                                     cudaMemcpyHostToDevice, s);
    if (ce != cudaSuccess) { pool_free(dtab, s); return cuda_fail(ce, "cudaMemcpyAsync(sv table)"); }

    const size_t n = (size_t)H * W * C;
    void *buf[2] = {nullptr, nullptr};
    const int nbuf = L > 2 ? 2 : (L - 1);
    for (int i = 0; i < nbuf && rc == SKC_OK; ++i) rc = pool_alloc(&buf[i], n * sizeof(float), s);

    SvParams q;
    q.H = H;
    q.W = W;
    q.Mb = Mb;
    q.boundary = boundary;
    q.in_fs = q.out_fs = (long long)n;
    for (int k = 0; k < Mb; ++k) q.ps[k] = (float)params[k];
    for (int l = 0; l < L && rc == SKC_OK; ++l) {
        const int nl = layout[l];
        q.n = nl;
        // exact corner reach over every basis entry, +1 texel for fp32 lerp rounding
        double lo_x = 0, hi_x = 0, lo_y = 0, hi_y = 0;
        bool first = true;
        for (int k = 0; k < Mb; ++k)
            for (int i = 0; i < nl; ++i) {
                const double *e = basis + (((size_t)k * L + l) * nmax + i) * 3;
                if (first || e[0] < lo_x) lo_x = e[0];
                if (first || e[0] > hi_x) hi_x = e[0];
                if (first || e[1] < lo_y) lo_y = e[1];
                if (first || e[1] > hi_y) hi_y = e[1];
                first = false;
            }
        const int dx_min = (int)std::floor(lo_x) - 1, dx_max = (int)std::floor(hi_x) + 2;
        const int dy_min = (int)std::floor(lo_y) - 1, dy_max = (int)std::floor(hi_y) + 2;
        q.dx0 = dx_min;
        q.dy0 = dy_min;
        int pitch = kSvTW + (dx_max - dx_min);
        if ((pitch & 1) == 0) ++pitch;
        q.pitch = pitch;
        q.rows = kSvTH + (dy_max - dy_min);
        const void *src = l == 0 ? in : buf[(l - 1) & 1];
        const int sdt = l == 0 ? in_dtype : SKC_F32;
        void *dst = l == L - 1 ? out : buf[l & 1];
        const int ddt = l == L - 1 ? out_dtype : SKC_F32;
        rc = launch_sv(src, sdt, dst, ddt, C, pmap, (const float4 *)dtab + start[l], q, s);
    }
    for (int i = 0; i < nbuf; ++i)
        if (buf[i]) pool_free(buf[i], s);
    pool_free(dtab, s);
    return rc;
}

}  // extern "C"
