// skc_filter.cu -- the spatially varying filter for sm_100a.
//
// Reference chains replaced (all citations into /root/reference/pkg/src/sparsekern):
//   apply_sparse_layer (engine.py:160-170) -> sample_shifted (118-130) ->
//   _accum_shift (106-115); apply_complex (173-178);
//   sv_filter (svfilter.py:171-203) -> sv_filter_compiled/_sv_pass_loop
//   (_fastpath.py:97-150).
//
// This file holds the spatially varying filter; the uniform-layer kernels
// live in skc_layer.cu.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "skc_tile.cuh"

namespace skc {

// ------------------------------------------------------- SV filter kernel ---
constexpr int kSvTW = 64, kSvPx = 8;  // 64 x (8 * thread rows) tile; 8 pixels per thread
constexpr int kMaxBasis = 64;

struct SvParams {
    int H, W, Mb, n, boundary;
    int pairs;  // packed-FP32 pixel pairs on the bracket-uniform path (SKC_SV_PAIRS, default on)
    int dx0, dy0, pitch, rows;
    long long in_fs, out_fs;
    float ps[kMaxBasis];
};

// svfilter._bracket (svfilter.py:129-137) in fp32 on the fp32 map.
__device__ __forceinline__ void bracket_ps(float p, const float *ps, int Mb, int &k0, int &k1, float &t) {
    if (Mb == 1) { k0 = 0; k1 = 0; t = 0.f; return; }
    const float pc = fminf(fmaxf(p, ps[0]), ps[Mb - 1]);
    int k = 0;
    for (int j = 1; j < Mb - 1; ++j) k += (ps[j] <= pc) ? 1 : 0;
    k0 = k;
    k1 = k + 1;
    t = (pc - ps[k]) / (ps[k + 1] - ps[k]);
}
__device__ __forceinline__ void bracket(float p, const SvParams &q, int &k0, int &k1, float &t) {
    bracket_ps(p, q.ps, q.Mb, k0, k1, t);
}

// Table rows are per bracket k0: entry (k0, i) = {o[k0] (ox, oy, w), o[k0+1] - o[k0]},
// so the per-pixel lerp is one FFMA per component.
template <int C, int TR, typename TI, typename TO>
__global__ void __launch_bounds__(TR * 64)
    sv_tile_kernel(const TI *__restrict__ in, TO *__restrict__ out, const float *__restrict__ pmap,
                   const float4 *__restrict__ table, const __grid_constant__ SvParams q) {
    extern __shared__ float4 smem4[];
    constexpr int TH = TR * kSvPx;
    const int nrow = q.Mb > 1 ? q.Mb - 1 : 1;
    float4 *stab = smem4;  // (nrow, n, 2)
    float *tile = reinterpret_cast<float *>(smem4 + 2 * nrow * q.n);
    const int tx0 = blockIdx.x * kSvTW, ty0 = blockIdx.y * TH;
    for (int i = threadIdx.x; i < 2 * nrow * q.n; i += blockDim.x) stab[i] = table[i];
    load_tile<C, TI>(tile, in, q.H, q.W, q.boundary, tx0 + q.dx0, ty0 + q.dy0, q.pitch, q.rows);
    __syncthreads();

    const int tx = threadIdx.x & (kSvTW - 1), ty = threadIdx.x / kSvTW;
    const int plane = q.rows * q.pitch, pitch = q.pitch;
    const int gx = tx0 + tx;
    int e0[kSvPx];
    float tt[kSvPx];
    float acc[kSvPx][C];
#pragma unroll
    for (int k = 0; k < kSvPx; ++k) {
        const int gy = ty0 + ty + TR * k;
        float p = 0.f;
        if (gy < q.H && gx < q.W) p = __ldg(pmap + (long long)gy * q.W + gx);
        int k0, k1;
        bracket(p, q, k0, k1, tt[k]);
        e0[k] = 2 * k0 * q.n;
#pragma unroll
        for (int c = 0; c < C; ++c) acc[k][c] = 0.f;
    }
    // smem (0,0) sits at global (tx0 + dx0, ty0 + dy0)
    const int base0 = (ty - q.dy0) * pitch + (tx - q.dx0);
#pragma unroll 1
    for (int i = 0; i < q.n; ++i) {
#pragma unroll
        for (int k = 0; k < kSvPx; ++k) {
            const float4 a = stab[e0[k] + 2 * i];
            const float4 d = stab[e0[k] + 2 * i + 1];
            const float t = tt[k];
            // _fastpath.py:109-111: lerp of offsets and weight between the bracket
            const float ox = fmaf(t, d.x, a.x);
            const float oy = fmaf(t, d.y, a.y);
            const float w = fmaf(t, d.z, a.z);
            const float fx0 = floorf(ox), fy0 = floorf(oy);
            const float fx = ox - fx0, fy = oy - fy0;
            const float wb = w * fy, wa = w - wb;
            const float c10 = wa * fx, c00 = wa - c10, c11 = wb * fx, c01 = wb - c11;
            const int off = base0 + (TR * k + (int)fy0) * pitch + (int)fx0;
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
        const int gy = ty0 + ty + TR * k;
        if (gy >= q.H || gx >= q.W) continue;
        TO *o = out + ((long long)gy * q.W + gx) * C;
#pragma unroll
        for (int c = 0; c < C; ++c) IO<TO>::st(o + c, acc[k][c]);
    }
}

// Interleaved-tile variant: the halo tile keeps the image's pixel-interleaved
// layout in shared memory (pixel stride PS = C, or C + 1 for even C so that
// neighbouring lanes stay bank-disjoint), so the 2 x 2 corners of all C
// channels of one tap sit at compile-time offsets {0, PS} x {0, RS} + c from
// a single per-(tap, pixel) address: 2 integer ops of addressing per
// tap-pixel instead of ~14 with C separate planes (SASS count).  The floor
// of the lerped offset uses the round-down add of 1.5 * 2^23 (exact for
// |o| < 2^22), which yields the integer and the fraction on the FMA pipe.
template <int C>
struct SvPix {
    static constexpr int PS = (C % 2 == 1) ? C : C + 1;
};

template <int C, typename TI>
__device__ __forceinline__ void load_tile_il(float *s, const TI *__restrict__ in, int H, int W, int boundary,
                                             int gx0, int gy0, int pitch, int rows) {
    constexpr int PS = SvPix<C>::PS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const bool clamp = boundary == SKC_CLAMP;
    const int rowlen = pitch * C, rs = pitch * PS;
    for (int r = warp; r < rows; r += nw) {
        int gy = gy0 + r;
        const bool rowin = clamp || (gy >= 0 && gy < H);
        gy = min(max(gy, 0), H - 1);
        const TI *src = in + (long long)gy * W * C;
        float *dst = s + r * rs;
        const bool interior = rowin && gx0 >= 0 && gx0 + pitch <= W;
        if constexpr (sizeof(TI) == 4) {
            const float *sf = reinterpret_cast<const float *>(src);
            if (interior && PS == C) {
                const float *sx = sf + (long long)gx0 * C + lane;
                unsigned sd = (unsigned)__cvta_generic_to_shared(dst + lane);
#pragma unroll 4
                for (int e = lane; e < rowlen; e += 32, sd += 128, sx += 32) cp_async4s(sd, sx);
                continue;
            }
#pragma unroll 4
            for (int e = lane; e < rowlen; e += 32) {
                const int col = e / C, c = e - col * C;
                const int gx = gx0 + col;
                const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                cp_async4(dst + col * PS + c, sf + (long long)min(max(gx, 0), W - 1) * C + c, ok);
            }
        } else {
            for (int e = lane; e < rowlen; e += 32) {
                const int col = e / C, c = e - col * C;
                const int gx = gx0 + col;
                const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                dst[col * PS + c] = ok ? IO<TI>::ld(src + (long long)min(max(gx, 0), W - 1) * C + c) : 0.f;
            }
        }
    }
    cp_async_wait_all();
}

// Packed-FP32 helpers (sm_100 f32x2): one instruction per pixel pair.
__device__ __forceinline__ unsigned long long f2_bits(float2 v) { return *reinterpret_cast<unsigned long long *>(&v); }
__device__ __forceinline__ float2 f2_val(unsigned long long r) { return *reinterpret_cast<float2 *>(&r); }
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
    return f2_val(d);
}
__device__ __forceinline__ float2 f2_add_rm(float2 a, float2 b) {  // round toward -inf (__fadd_rd)
    unsigned long long d;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_val(d);
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_val(d);
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_val(d);
}

template <int C, int TR, typename TI, typename TO>
__global__ void __launch_bounds__(TR * 64)
    sv_tile_il_kernel(const TI *__restrict__ in, TO *__restrict__ out, const float *__restrict__ pmap,
                      const float4 *__restrict__ table, const __grid_constant__ SvParams q) {
    extern __shared__ float4 smem4[];
    constexpr int TH = TR * kSvPx, PS = SvPix<C>::PS;
    const int nrow = q.Mb > 1 ? q.Mb - 1 : 1;
    float4 *stab = smem4;  // (nrow, n, 2)
    float *tile = reinterpret_cast<float *>(smem4 + 2 * nrow * q.n);
    const int tx0 = blockIdx.x * kSvTW, ty0 = blockIdx.y * TH;
    for (int i = threadIdx.x; i < 2 * nrow * q.n; i += blockDim.x) stab[i] = table[i];
    load_tile_il<C, TI>(tile, in, q.H, q.W, q.boundary, tx0 + q.dx0, ty0 + q.dy0, q.pitch, q.rows);
    __syncthreads();

    const int tx = threadIdx.x & (kSvTW - 1), ty = threadIdx.x / kSvTW;
    const int rs = q.pitch * PS;
    const int gx = tx0 + tx;
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
    constexpr int kMagicBits = 0x4B400000;
    int e0[kSvPx], pb[kSvPx];
    float tt[kSvPx];
    float acc[kSvPx][C];
#pragma unroll
    for (int k = 0; k < kSvPx; ++k) {
        const int gy = ty0 + ty + TR * k;
        float p = 0.f;
        if (gy < q.H && gx < q.W) p = __ldg(pmap + (long long)gy * q.W + gx);
        int k0, k1;
        bracket(p, q, k0, k1, tt[k]);
        e0[k] = 2 * k0 * q.n;
        pb[k] = (ty + TR * k - q.dy0) * rs + (tx - q.dx0) * PS;  // word offset of the pixel's (0, 0) texel
#pragma unroll
        for (int c = 0; c < C; ++c) acc[k][c] = 0.f;
    }
    // One (tap, pixel): lerp the tap between the bracket's basis entries
    // (_fastpath.py:109-111), split the offset into floor and fraction and
    // gather the 2 x 2 corners of all C channels.
    auto tap_px = [&](const float4 a, const float4 d, int k) {
        const float t = tt[k];
        const float ox = fmaf(t, d.x, a.x);
        const float oy = fmaf(t, d.y, a.y);
        const float w = fmaf(t, d.z, a.z);
        const float bx = __fadd_rd(ox, kMagic), by = __fadd_rd(oy, kMagic);  // kMagic + floor(o)
        const float fx = ox - (bx - kMagic), fy = oy - (by - kMagic);
        const float wb = w * fy, wa = w - wb;
        const float c10 = wa * fx, c00 = wa - c10, c11 = wb * fx, c01 = wb - c11;
        int iy = __float_as_int(by) - kMagicBits, ix = __float_as_int(bx) - kMagicBits;
        // opaque to the optimiser: otherwise the magic bias is re-associated into
        // a separate add in front of every shared load (no room in the LDS offset)
        asm("" : "+r"(iy), "+r"(ix));
        const float *sp = tile + (pb[k] + iy * rs + ix * PS);
        const float *sq = sp + rs;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            float v = acc[k][c];
            v = fmaf(c00, sp[c], v);
            v = fmaf(c10, sp[PS + c], v);
            v = fmaf(c01, sq[c], v);
            v = fmaf(c11, sq[PS + c], v);
            acc[k][c] = v;
        }
    };
    // Smooth size maps put a thread's 8 pixels (one column, TR rows apart) in
    // the same bracket almost everywhere: then one table read per tap serves
    // all 8 (the per-pixel reads were ~2 of ~17 shared wavefronts per
    // warp-tap-pixel).  Warp-uniform choice, so no divergence between paths.
    bool same = true;
#pragma unroll
    for (int k = 1; k < kSvPx; ++k) same &= e0[k] == e0[0];
    if (__all_sync(0xffffffffu, same)) {
        const float4 *row = stab + e0[0];
        if (q.pairs) {
            // Pixel pairs in packed FP32 (f32x2): lerp, floor/fraction and corner
            // weights of pixels k and k+1 in one instruction each, and the corner
            // FMAs on (acc[k][c], acc[k+1][c]) pairs -- the same per-lane
            // operations as tap_px, ~2/3 of its instructions.
            float2 tp[kSvPx / 2];
            float2 accp[kSvPx / 2][C];
#pragma unroll
            for (int m = 0; m < kSvPx / 2; ++m) {
                tp[m] = make_float2(tt[2 * m], tt[2 * m + 1]);
#pragma unroll
                for (int c = 0; c < C; ++c) accp[m][c] = make_float2(0.f, 0.f);
            }
            const float2 mg = make_float2(kMagic, kMagic);
#pragma unroll 1
            for (int i = 0; i < q.n; ++i) {
                const float4 a = row[2 * i], d = row[2 * i + 1];
#pragma unroll
                for (int m = 0; m < kSvPx / 2; ++m) {
                    const float2 ox = f2_fma(tp[m], make_float2(d.x, d.x), make_float2(a.x, a.x));
                    const float2 oy = f2_fma(tp[m], make_float2(d.y, d.y), make_float2(a.y, a.y));
                    const float2 w = f2_fma(tp[m], make_float2(d.z, d.z), make_float2(a.z, a.z));
                    const float2 bx = f2_add_rm(ox, mg), by = f2_add_rm(oy, mg);
                    const float2 fx = f2_sub(ox, f2_sub(bx, mg)), fy = f2_sub(oy, f2_sub(by, mg));
                    const float2 wb = f2_mul(w, fy), wa = f2_sub(w, wb);
                    const float2 c10 = f2_mul(wa, fx), c00 = f2_sub(wa, c10), c11 = f2_mul(wb, fx), c01 = f2_sub(wb, c11);
                    int iy0 = __float_as_int(by.x) - kMagicBits, ix0 = __float_as_int(bx.x) - kMagicBits;
                    int iy1 = __float_as_int(by.y) - kMagicBits, ix1 = __float_as_int(bx.y) - kMagicBits;
                    asm("" : "+r"(iy0), "+r"(ix0), "+r"(iy1), "+r"(ix1));
                    const float *sp0 = tile + (pb[2 * m] + iy0 * rs + ix0 * PS), *sq0 = sp0 + rs;
                    const float *sp1 = tile + (pb[2 * m + 1] + iy1 * rs + ix1 * PS), *sq1 = sp1 + rs;
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        float2 v = accp[m][c];
                        v = f2_fma(c00, make_float2(sp0[c], sp1[c]), v);
                        v = f2_fma(c10, make_float2(sp0[PS + c], sp1[PS + c]), v);
                        v = f2_fma(c01, make_float2(sq0[c], sq1[c]), v);
                        v = f2_fma(c11, make_float2(sq0[PS + c], sq1[PS + c]), v);
                        accp[m][c] = v;
                    }
                }
            }
#pragma unroll
            for (int m = 0; m < kSvPx / 2; ++m)
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    acc[2 * m][c] = accp[m][c].x;
                    acc[2 * m + 1][c] = accp[m][c].y;
                }
        } else {
#pragma unroll 1
            for (int i = 0; i < q.n; ++i) {
                const float4 a = row[2 * i], d = row[2 * i + 1];
#pragma unroll
                for (int k = 0; k < kSvPx; ++k) tap_px(a, d, k);
            }
        }
    } else {
#pragma unroll 1
        for (int i = 0; i < q.n; ++i) {
#pragma unroll
            for (int k = 0; k < kSvPx; ++k) tap_px(stab[e0[k] + 2 * i], stab[e0[k] + 2 * i + 1], k);
        }
    }
#pragma unroll
    for (int k = 0; k < kSvPx; ++k) {
        const int gy = ty0 + ty + TR * k;
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
        float acc[C];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = 0.f;
        for (int i = 0; i < q.n; ++i) {
            const float4 a = __ldg(table + 2 * (k0 * q.n + i));
            const float4 d = __ldg(table + 2 * (k0 * q.n + i) + 1);
            const float ox = fmaf(t, d.x, a.x), oy = fmaf(t, d.y, a.y), w = fmaf(t, d.z, a.z);
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

// SKC_SV_PLANAR=1 keeps the channel-planar SV tile (the interleaved one is the default).
static bool sv_interleaved() {
    static const bool v = [] {
        const char *e = std::getenv("SKC_SV_PLANAR");
        return !(e && e[0] == '1');
    }();
    return v;
}

template <int C, int TR, typename TI, typename TO>
static int launch_sv_tile(const void *in, void *out, const float *pmap, const float4 *table, SvParams q,
                          int span_y, cudaStream_t s) {
    q.rows = TR * kSvPx + span_y;
    const int nrow = q.Mb > 1 ? q.Mb - 1 : 1;
    if (sv_interleaved()) {
        const size_t smem =
            (size_t)2 * nrow * q.n * sizeof(float4) + (size_t)SvPix<C>::PS * q.rows * q.pitch * 4;
        if (smem > (size_t)kMaxSmem) return -1;
        auto kern = sv_tile_il_kernel<C, TR, TI, TO>;
        if (int rc_ = smem_optin((const void *)kern, kMaxSmem)) return rc_;
        dim3 grid(ceil_div(q.W, kSvTW), ceil_div(q.H, TR * kSvPx));
        kern<<<grid, TR * 64, smem, s>>>(static_cast<const TI *>(in), static_cast<TO *>(out), pmap, table, q);
        SKC_LAUNCH_CHECK("sv_tile_il_kernel");
        return SKC_OK;
    }
    const size_t smem = (size_t)2 * nrow * q.n * sizeof(float4) + (size_t)C * q.rows * q.pitch * 4;
    if (smem > (size_t)kMaxSmem) return -1;
    auto kern = sv_tile_kernel<C, TR, TI, TO>;
    if (int rc_ = smem_optin((const void *)kern, kMaxSmem)) return rc_;
    dim3 grid(ceil_div(q.W, kSvTW), ceil_div(q.H, TR * kSvPx));
    kern<<<grid, TR * 64, smem, s>>>(static_cast<const TI *>(in), static_cast<TO *>(out), pmap, table, q);
    SKC_LAUNCH_CHECK("sv_tile_kernel");
    return SKC_OK;
}

// Big halos get the taller 64 x 64 tile (16 warps, half the halo overfetch);
// small halos the 64 x 32 tile (more CTAs per SM).
template <int C, typename TI, typename TO>
static int launch_sv_t(const void *in, void *out, const float *pmap, const float4 *table,
                       SvParams q, cudaStream_t s) {
    const int span_y = q.rows;  // caller passes the vertical halo span in rows
    int rc = -1;
    if (span_y > 24) rc = launch_sv_tile<C, 8, TI, TO>(in, out, pmap, table, q, span_y, s);
    if (rc == -1) rc = launch_sv_tile<C, 4, TI, TO>(in, out, pmap, table, q, span_y, s);
    if (rc != -1) return rc;
    const long long npx = (long long)q.H * q.W;
    const unsigned grid = (unsigned)std::min<long long>((npx + 255) / 256, 148 * 16);
    sv_direct_kernel<C, TI, TO><<<grid, 256, 0, s>>>(static_cast<const TI *>(in), static_cast<TO *>(out), pmap,
                                                     table, q);
    SKC_LAUNCH_CHECK("sv_direct_kernel");
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

// ------------------------------------------------ 2-D grid SV (next row) ---
// svfilter.sv_filter_grid (svfilter.py:292-319): per pixel two brackets
// (u, v) and a bilinear blend of the four surrounding basis entries' taps
// (weights (1-tu)(1-tv), tu(1-tv), (1-tu)tv, tu tv), then the same bilinear
// gather from the staged halo tile as the 1-D SV kernel.
struct SvGridParams {
    int H, W, Mu, Mv, n, boundary;
    int dx0, dy0, pitch, rows;
    float pu[kMaxBasis], pv[kMaxBasis];
};

template <int C, typename TI, typename TO>
__global__ void __launch_bounds__(256)
    sv_grid_kernel(const TI *__restrict__ in, TO *__restrict__ out, const float2 *__restrict__ pmap2,
                   const float4 *__restrict__ table, const __grid_constant__ SvGridParams q) {
    extern __shared__ float4 smem4[];
    constexpr int TR = 4, TH = TR * kSvPx;
    const int nent = q.Mu * q.Mv * q.n;
    float4 *stab = smem4;  // (Mu, Mv, n) entries (ox, oy, w, 0)
    float *tile = reinterpret_cast<float *>(smem4 + nent);
    const int tx0 = blockIdx.x * kSvTW, ty0 = blockIdx.y * TH;
    for (int i = threadIdx.x; i < nent; i += blockDim.x) stab[i] = table[i];
    load_tile<C, TI>(tile, in, q.H, q.W, q.boundary, tx0 + q.dx0, ty0 + q.dy0, q.pitch, q.rows);
    __syncthreads();
    const int tx = threadIdx.x & (kSvTW - 1), ty = threadIdx.x / kSvTW;
    const int plane = q.rows * q.pitch, pitch = q.pitch;
    const int gx = tx0 + tx;
    const int base0 = (ty - q.dy0) * pitch + (tx - q.dx0);
#pragma unroll 1
    for (int k = 0; k < kSvPx; ++k) {
        const int gy = ty0 + ty + TR * k;
        float2 pm = make_float2(0.f, 0.f);
        if (gy < q.H && gx < q.W) pm = pmap2[(long long)gy * q.W + gx];
        int u0, u1, v0, v1;
        float tu, tv;
        bracket_ps(pm.x, q.pu, q.Mu, u0, u1, tu);
        bracket_ps(pm.y, q.pv, q.Mv, v0, v1, tv);
        const float b00 = (1.f - tu) * (1.f - tv), b10 = tu * (1.f - tv), b01 = (1.f - tu) * tv, b11 = tu * tv;
        const int e00 = (u0 * q.Mv + v0) * q.n, e10 = (u1 * q.Mv + v0) * q.n;
        const int e01 = (u0 * q.Mv + v1) * q.n, e11 = (u1 * q.Mv + v1) * q.n;
        float acc[C];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = 0.f;
        for (int i = 0; i < q.n; ++i) {
            const float4 a = stab[e00 + i], b = stab[e10 + i], cc = stab[e01 + i], d = stab[e11 + i];
            const float ox = b00 * a.x + b10 * b.x + b01 * cc.x + b11 * d.x;
            const float oy = b00 * a.y + b10 * b.y + b01 * cc.y + b11 * d.y;
            const float w = b00 * a.z + b10 * b.z + b01 * cc.z + b11 * d.z;
            const float fx0 = floorf(ox), fy0 = floorf(oy);
            const float fx = ox - fx0, fy = oy - fy0;
            const float wb = w * fy, wa = w - wb;
            const float c10 = wa * fx, c00 = wa - c10, c11 = wb * fx, c01 = wb - c11;
            const int off = base0 + (TR * k + (int)fy0) * pitch + (int)fx0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const float *sp = tile + c * plane + off;
                float v = acc[c];
                v = fmaf(c00, sp[0], v);
                v = fmaf(c10, sp[1], v);
                v = fmaf(c01, sp[pitch], v);
                v = fmaf(c11, sp[pitch + 1], v);
                acc[c] = v;
            }
        }
        if (gy < q.H && gx < q.W) {
            TO *o = out + ((long long)gy * q.W + gx) * C;
#pragma unroll
            for (int c = 0; c < C; ++c) IO<TO>::st(o + c, acc[c]);
        }
    }
}

template <int C>
static int launch_sv_grid_c(const void *in, void *out, const float2 *pmap2, const float4 *table,
                            const SvGridParams &q, cudaStream_t s) {
    const size_t smem = (size_t)q.Mu * q.Mv * q.n * sizeof(float4) + (size_t)C * q.rows * q.pitch * 4;
    if (smem > (size_t)kMaxSmem) return fail(SKC_EBADARG, "grid SV basis/halo too large for shared memory");
    auto kern = sv_grid_kernel<C, float, float>;
    if (int rc_ = smem_optin((const void *)kern, kMaxSmem)) return rc_;
    dim3 grid(ceil_div(q.W, kSvTW), ceil_div(q.H, 4 * kSvPx));
    kern<<<grid, 256, smem, s>>>(static_cast<const float *>(in), static_cast<float *>(out), pmap2, table, q);
    SKC_LAUNCH_CHECK("sv_grid_kernel");
    return SKC_OK;
}

}  // namespace skc

using namespace skc;

extern "C" {

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
    // rows per bracket k0: {o[k0], o[k0+1] - o[k0]} (the difference in float64)
    std::vector<float4> host;
    std::vector<size_t> start(L);
    const int nrow = Mb > 1 ? Mb - 1 : 1;
    for (int l = 0; l < L; ++l) {
        start[l] = host.size();
        for (int k = 0; k < nrow; ++k)
            for (int i = 0; i < layout[l]; ++i) {
                const double *e0 = basis + (((size_t)k * L + l) * nmax + i) * 3;
                const double *e1 = Mb > 1 ? basis + (((size_t)(k + 1) * L + l) * nmax + i) * 3 : e0;
                host.push_back(make_float4((float)e0[0], (float)e0[1], (float)e0[2], 0.f));
                host.push_back(make_float4((float)(e1[0] - e0[0]), (float)(e1[1] - e0[1]),
                                           (float)(e1[2] - e0[2]), 0.f));
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
    {
        const char *e = std::getenv("SKC_SV_PAIRS");
        q.pairs = !(e && e[0] == '0');
    }
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
        q.rows = dy_max - dy_min;   // vertical halo span; the launcher adds the tile height
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

int skc_sv_grid_fwd(const void *in, void *out, int H, int W, int C, const float *pmap2,
                    const double *params_u, int Mu, const double *params_v, int Mv, const double *basis,
                    int nmax, const int *layout, int L, int boundary, void *stream) {
    int rc = check_image_args(in, SKC_F32, out, SKC_F32, 1, H, W, C, boundary);
    if (rc) return rc;
    if (!pmap2 || !params_u || !params_v || !basis || !layout) return fail(SKC_EBADARG, "null argument");
    if (Mu < 1 || Mu > kMaxBasis || Mv < 1 || Mv > kMaxBasis) return fail(SKC_EBADARG, "grid axes must be 1..64");
    if (L < 1 || nmax < 1) return fail(SKC_EBADARG, "basis needs at least one layer");
    for (int k = 1; k < Mu; ++k)
        if (!(params_u[k] > params_u[k - 1])) return fail(SKC_EBADARG, "grid parameters must be strictly increasing");
    for (int k = 1; k < Mv; ++k)
        if (!(params_v[k] > params_v[k - 1])) return fail(SKC_EBADARG, "grid parameters must be strictly increasing");
    for (int l = 0; l < L; ++l)
        if (layout[l] < 1 || layout[l] > nmax) return fail(SKC_EBADARG, "bad basis layout");
    if (!finite_taps(basis, Mu * Mv * L * nmax)) return fail(SKC_EBADARG, "basis parameters must be finite");
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<float4> host;
    std::vector<size_t> start(L);
    for (int l = 0; l < L; ++l) {
        start[l] = host.size();
        for (int k = 0; k < Mu * Mv; ++k)
            for (int i = 0; i < layout[l]; ++i) {
                const double *e = basis + (((size_t)k * L + l) * nmax + i) * 3;
                host.push_back(make_float4((float)e[0], (float)e[1], (float)e[2], 0.f));
            }
    }
    void *dtab = nullptr;
    if ((rc = pool_alloc(&dtab, host.size() * sizeof(float4), s))) return rc;
    cudaError_t ce = cudaMemcpyAsync(dtab, host.data(), host.size() * sizeof(float4), cudaMemcpyHostToDevice, s);
    if (ce != cudaSuccess) { pool_free(dtab, s); return cuda_fail(ce, "cudaMemcpyAsync(grid table)"); }
    const size_t n = (size_t)H * W * C;
    void *buf[2] = {nullptr, nullptr};
    const int nbuf = L > 2 ? 2 : (L - 1);
    for (int i = 0; i < nbuf && rc == SKC_OK; ++i) rc = pool_alloc(&buf[i], n * sizeof(float), s);
    SvGridParams q;
    q.H = H;
    q.W = W;
    q.Mu = Mu;
    q.Mv = Mv;
    q.boundary = boundary;
    for (int k = 0; k < Mu; ++k) q.pu[k] = (float)params_u[k];
    for (int k = 0; k < Mv; ++k) q.pv[k] = (float)params_v[k];
    for (int l = 0; l < L && rc == SKC_OK; ++l) {
        const int nl = layout[l];
        q.n = nl;
        double lo_x = 0, hi_x = 0, lo_y = 0, hi_y = 0;
        bool first = true;
        for (int k = 0; k < Mu * Mv; ++k)
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
        q.rows = 4 * kSvPx + (dy_max - dy_min);
        const void *src = l == 0 ? in : buf[(l - 1) & 1];
        void *dst = l == L - 1 ? out : buf[l & 1];
        const float4 *tab = (const float4 *)dtab + start[l];
        const float2 *pm = (const float2 *)pmap2;
        switch (C) {
            case 1: rc = launch_sv_grid_c<1>(src, dst, pm, tab, q, s); break;
            case 2: rc = launch_sv_grid_c<2>(src, dst, pm, tab, q, s); break;
            case 3: rc = launch_sv_grid_c<3>(src, dst, pm, tab, q, s); break;
            default: rc = launch_sv_grid_c<4>(src, dst, pm, tab, q, s); break;
        }
    }
    for (int i = 0; i < nbuf; ++i)
        if (buf[i]) pool_free(buf[i], s);
    pool_free(dtab, s);
    return rc;
}

}  // extern "C"

