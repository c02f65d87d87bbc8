// skc_fit.cu -- impulse-response synthesis, analytic backward and the
// persistent batched fitting loop for sm_100a.
//
// Reference (citations into /root/reference/pkg/src/sparsekern):
//   synthesize_ir (engine.py:191-209), synthesize_ir_batch (251-303),
//   _ir_batch_loop (_fastpath.py:33-85); optim.py: _loss_value/_loss_grad
//   (133-146), _forward_ir (204-222), _first_nonfinite_sample (225-228),
//   _backward_pass (231-263), _chain_weight_norm (266-275), backward
//   (278-292), _project_kws (312-325), _project_sum (328-335), adam_step
//   (338-369), fit (390-469).
//
// One CTA owns one complex (one target kernel) for the whole call.  Every
// step runs on device: effective weights, the canvas growth rule, per-layer
// live boxes (the support of each intermediate, clipped to the canvas -- the
// reference's "live region", _fastpath.py:42-56), the forward chain, the
// loss, the reverse sweep (per-tap <g, sample>, <g, d sample/dx>,
// <g, d sample/dy> reductions in float64, then the adjoint gather at negated
// offsets), the weight-norm chain rule, Adam and the projections.  Reductions
// are fixed-order (warp shuffle tree, then warps in index order), so results
// are bit-reproducible run to run.  The per-step loss goes to a device trace;
// the host reads it once at the end.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "skc_common.cuh"

namespace skc {

constexpr int kFitThreads = 256;       // two CTAs (two targets) per SM
constexpr int kFitWarps = kFitThreads / 32;
constexpr int kFitMaxL = 8;
constexpr int kFitMaxP = 256;     // total taps per complex
constexpr int kNeedGrow = 100;    // internal status: scratch canvas too small
constexpr int kFitSmem = 110 * 1024;   // dynamic shared memory per CTA (state + arena)
constexpr int kFKR = 5, kFMC = 4;      // register block of the pixel passes (KR odd)
constexpr int kMaxTapsPerWarp = 4;     // correlation taps a warp carries at once

enum FitMode { MODE_FIT = 0, MODE_BACKWARD = 1, MODE_IR = 2, MODE_ENERGY = 3 };

// Live box of an intermediate in canvas coordinates; empty when w or h <= 0.
__host__ __device__ __forceinline__ int odd_stride(int w) { return w | 1; }
struct Box {
    int x0, y0, w, h;
};

// A box plus its compact row-major data (row stride = w).  `p` is a generic
// pointer into the shared-memory arena or, when the arena is full, into the
// CTA's global scratch slot -- the passes do not care which.
struct Buf {
    float *p;
    int x0, y0, w, h;
    int s;   // row stride, odd: with KR odd the 32 lanes' 5x4 block origins hit 32 banks
    int so;  // p's offset (floats) from the CTA's dynamic shared memory, -1 for a global overflow slot
};

// The CTA's dynamic shared memory as floats: window loads indexed from this
// symbol compile to LDS with 32-bit addressing (through Buf::p they are
// generic LD with 64-bit address arithmetic -- 8% of the fit kernel's stall
// samples sat on those loads and 13% on their IMADs, profiles/r02_c4_fit_final.md).
__device__ __forceinline__ const float *smem_f32() {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    return reinterpret_cast<const float *>(smem_raw);
}

struct FitParams {
    int B, L, nmax, P, M, mode;
    int layout[kFitMaxL];
    int start[kFitMaxL + 1];
    skc_fit_cfg cfg;
    int cap;            // scratch canvas capacity (global slots are cap*cap floats)
    int canvas_fixed;   // MODE_BACKWARD / MODE_IR canvas
    float *state;       // MODE_FIT
    const float *tgts;  // (B, M, M)
    float *trace;       // (B, steps+1)
    int *status;        // (B, 4)
    float *scratch;     // (B, L+1, cap, cap) global overflow slots
    const float *taps_in;  // MODE_BACKWARD / MODE_IR: (B, L, nmax, 3)
    float *loss_out;       // MODE_BACKWARD
    float *grads_out;      // MODE_BACKWARD: (B, L, nmax, 3)
    float *ir_out;         // MODE_IR: (B, canvas, canvas)
    double *energy_out;    // MODE_ENERGY: (B,)
    int tgt_shared;        // MODE_ENERGY: every complex uses target 0
    const int *idx;        // MODE_FIT relaunch: CTA i runs target idx[i] (null = i)
};

struct FitSmem {
    float2 off[kFitMaxP];   // current offsets
    float wp[kFitMaxP];     // weight parameters (weights or logits)
    float w[kFitMaxP];      // effective weights
    float4 cw[kFitMaxP];    // corner weights
    float2 frac[kFitMaxP];  // fx, fy
    int2 ixy[kFitMaxP];     // floor(ox), floor(oy)
    float3 grad[kFitMaxP];  // d_ox, d_oy, d_w
    double red[kFitWarps];
    Box box[kFitMaxL + 1];
    int4 dr[kFitMaxL];      // per layer corner range: dxmin, dxmax, dymin, dymax
    float *bufp[kFitMaxL + 1];
    float one;
    int canvas;
    int flag;
    int bad_layer, bad_sample;
};

constexpr int kArenaFloats = (kFitSmem - (int)((sizeof(FitSmem) + 15) / 16 * 16)) / 4;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum of one double (result returned to all threads).
__device__ double block_sum(FitSmem &S, double v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) S.red[warp] = v;
    __syncthreads();
    double tot = 0.0;
    for (int k = 0; k < kFitWarps; ++k) tot += S.red[k];
    return tot;
}

// optim.py:133-146
__device__ __forceinline__ float loss_term(float d, int kind, float eps) {
    if (kind == SKC_LOSS_CHARBONNIER) return sqrtf(d * d + eps * eps);
    if (kind == SKC_LOSS_L1) return fabsf(d);
    return d * d;
}
__device__ __forceinline__ float loss_grad(float d, int kind, float eps) {
    if (kind == SKC_LOSS_CHARBONNIER) return d / sqrtf(d * d + eps * eps);
    if (kind == SKC_LOSS_L1) return d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    return 2.f * d;
}

__device__ __forceinline__ float ld_chk(const Buf &b, int y, int x) {
    const unsigned dy = (unsigned)(y - b.y0), dx = (unsigned)(x - b.x0);
    return (dy < (unsigned)b.h && dx < (unsigned)b.w) ? b.p[dy * b.s + dx] : 0.f;
}

__device__ __forceinline__ Buf buf_of(const FitSmem &S, int l) {
    const Box &bx = S.box[l];
    float *const bp = S.bufp[l];
    return Buf{bp, bx.x0, bx.y0, bx.w, bx.h, l == 0 ? 1 : odd_stride(bx.w),
               __isShared(bp) ? (int)(bp - smem_f32()) : -1};
}

// Effective weights (optim.py:164-165; softmax 159-161) -- one thread per layer.
__device__ void effective_weights(const FitParams &p, FitSmem &S) {
    const int l = threadIdx.x;
    if (l < p.L) {
        const int s0 = p.start[l], n = p.layout[l];
        if (p.cfg.weight_norm == SKC_WN_SOFM) {
            float m = S.wp[s0];
            for (int i = 1; i < n; ++i) m = fmaxf(m, S.wp[s0 + i]);
            float sum = 0.f;
            for (int i = 0; i < n; ++i) {
                const float e = expf(S.wp[s0 + i] - m);
                S.w[s0 + i] = e;
                sum += e;
            }
            for (int i = 0; i < n; ++i) S.w[s0 + i] /= sum;
        } else {
            for (int i = 0; i < n; ++i) S.w[s0 + i] = S.wp[s0 + i];
        }
    }
    __syncthreads();
}

// Tap tables (sample_shifted, engine.py:118-130), live boxes and the buffer
// arena: the IR's box first, then intermediates from the last layer down, go
// to shared memory while they fit, the rest to the CTA's global slots.
__device__ void build_taps_and_boxes(const FitParams &p, FitSmem &S, float *arena, float *gslots) {
    for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
        const float ox = S.off[q].x, oy = S.off[q].y, w = S.w[q];
        const float fx0 = floorf(ox), fy0 = floorf(oy);
        const float fx = ox - fx0, fy = oy - fy0;
        S.ixy[q] = make_int2((int)fx0, (int)fy0);
        S.frac[q] = make_float2(fx, fy);
        S.cw[q] = make_float4(w * (1.f - fx) * (1.f - fy), w * fx * (1.f - fy),
                              w * (1.f - fx) * fy, w * fx * fy);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int c = S.canvas / 2, last = S.canvas - 1;
        S.box[0] = Box{c, c, 1, 1};
        S.one = 1.f;
        S.bufp[0] = &S.one;
        for (int l = 0; l < p.L; ++l) {
            int dxmin = 1 << 30, dxmax = -(1 << 30), dymin = 1 << 30, dymax = -(1 << 30);
            for (int i = 0; i < p.layout[l]; ++i) {
                const int2 d = S.ixy[p.start[l] + i];
                dxmin = min(dxmin, d.x);
                dxmax = max(dxmax, d.x + 1);
                dymin = min(dymin, d.y);
                dymax = max(dymax, d.y + 1);
            }
            S.dr[l] = make_int4(dxmin, dxmax, dymin, dymax);
            const Box a = S.box[l];
            Box nb{0, 0, 0, 0};
            if (a.w > 0 && a.h > 0) {
                // I_{l+1}[y] = sum cw I_l[y + d]  =>  support(I_{l+1}) = support(I_l) - d
                const int x0 = max(0, a.x0 - dxmax), x1 = min(last, a.x0 + a.w - 1 - dxmin);
                const int y0 = max(0, a.y0 - dymax), y1 = min(last, a.y0 + a.h - 1 - dymin);
                nb = Box{x0, y0, x1 - x0 + 1, y1 - y0 + 1};
            }
            S.box[l + 1] = nb;
        }
        int used = 0;
        for (int l = p.L; l >= 1; --l) {
            const Box &bx = S.box[l];
            const int n = (max(bx.w, 0) > 0 ? odd_stride(bx.w) * max(bx.h, 0) : 0) + 3 & ~3;
            if (used + n <= kArenaFloats) {
                S.bufp[l] = arena + used;
                used += n;
            } else {
                S.bufp[l] = gslots + (size_t)(l - 1) * p.cap * p.cap;
            }
        }
    }
    __syncthreads();
}

// Block b of a box with nbx x nby blocks: full groups of 8 block-columns are
// enumerated 8-wide row by row (a warp's 32 consecutive blocks form an 8 x 4
// tile: conflict-free with odd strides), the remainder group rem-wide.  Every
// index in [0, nbx*nby) is a real block, so a linear distribution over threads
// is perfectly balanced.
__device__ __forceinline__ void block_of(int b, int nbx, int nby, int &bx, int &by) {
    const int full = (nbx >> 3) * 8 * nby;
    if (b < full) {
        const int g = b / (8 * nby), r = b - g * 8 * nby;
        by = r >> 3;
        bx = g * 8 + (r & 7);
    } else {
        const int rem = nbx & 7, r = b - full;
        by = r / rem;
        bx = (nbx & ~7) + (r - by * rem);
    }
}

// out(y, x) += sum over taps of the 4 corner products, for one KR x MC block.
// `rd(y, x)` returns the source value at canvas (y, x) (checked or not); the
// window of tap i starts at source (y0 + sy(i), x0 + sx(i)).
template <bool ADJ, bool CHECK>
__device__ __forceinline__ void block_taps(float (&acc)[kFKR][kFMC], const FitSmem &S, const Buf &src,
                                           int s0, int n, int y0, int x0, int i0 = 0, int di = 1) {
    for (int i = i0; i < n; i += di) {
        const int2 d = S.ixy[s0 + i];
        const float4 w = S.cw[s0 + i];
        // forward: out(y,x) reads src(y + d + corner); adjoint: src(y - d - corner)
        const int wy = ADJ ? y0 - d.y - 1 : y0 + d.y;
        const int wx = ADJ ? x0 - d.x - 1 : x0 + d.x;
        // a window that misses src's box entirely adds exact zeros: skip it
        if (CHECK && (wy > src.y0 + src.h - 1 || wy + kFKR < src.y0 || wx > src.x0 + src.w - 1 ||
                      wx + kFMC < src.x0))
            continue;
        float win[kFKR + 1][kFMC + 1];
        // an edge block (CHECK) still reads most taps' windows entirely inside
        // src: when every active lane's window is, take the unchecked loads
        const bool tin = !CHECK || (wy >= src.y0 && wy + kFKR < src.y0 + src.h && wx >= src.x0 &&
                                    wx + kFMC < src.x0 + src.w);
        if (CHECK && !__all_sync(__activemask(), tin)) {
#pragma unroll
            for (int r = 0; r <= kFKR; ++r)
#pragma unroll
                for (int c = 0; c <= kFMC; ++c) win[r][c] = ld_chk(src, wy + r, wx + c);
        } else if (src.so >= 0) {
            const float *sb = smem_f32();
            const int o = src.so + (wy - src.y0) * src.s + (wx - src.x0);
#pragma unroll
            for (int r = 0; r <= kFKR; ++r)
#pragma unroll
                for (int c = 0; c <= kFMC; ++c) win[r][c] = sb[o + r * src.s + c];
        } else {
            const float *q = src.p + (wy - src.y0) * src.s + (wx - src.x0);
#pragma unroll
            for (int r = 0; r <= kFKR; ++r)
#pragma unroll
                for (int c = 0; c <= kFMC; ++c) win[r][c] = q[r * src.s + c];
        }
#pragma unroll
        for (int r = 0; r < kFKR; ++r)
#pragma unroll
            for (int c = 0; c < kFMC; ++c) {
                float v = acc[r][c];
                if (!ADJ) {
                    v = fmaf(w.x, win[r][c], v);
                    v = fmaf(w.y, win[r][c + 1], v);
                    v = fmaf(w.z, win[r + 1][c], v);
                    v = fmaf(w.w, win[r + 1][c + 1], v);
                } else {
                    v = fmaf(w.x, win[r + 1][c + 1], v);
                    v = fmaf(w.y, win[r + 1][c], v);
                    v = fmaf(w.z, win[r][c + 1], v);
                    v = fmaf(w.w, win[r][c], v);
                }
                acc[r][c] = v;
            }
    }
}

// One gather pass over dst's box: forward layer l (ADJ=false, dst = I_{l+1})
// or the adjoint of layer l (ADJ=true, src = g_{l+1}, dst = g_l).  Returns the
// block-wide "non-finite seen" flag.
template <bool ADJ>
__device__ int gather_pass(const FitParams &p, FitSmem &S, int l, const Buf src, const Buf dst) {
    const int s0 = p.start[l], n = p.layout[l];
    const int4 dr = S.dr[l];
    // rows/cols of src a block's window can touch, relative to its origin
    const int ry0 = ADJ ? -dr.w : dr.z, ry1 = ADJ ? kFKR - 1 - dr.z : kFKR - 1 + dr.w;
    const int rx0 = ADJ ? -dr.y : dr.x, rx1 = ADJ ? kFMC - 1 - dr.x : kFMC - 1 + dr.y;
    const int nbx = (dst.w + kFMC - 1) / kFMC, nby = (dst.h + kFKR - 1) / kFKR;
    int bad = 0;
    // Small boxes (the first layers of an impulse response): fewer blocks than
    // threads, so G = 2^k consecutive lanes share a block and split its taps
    // (lane g takes taps g, g + G, ...); the G partial sums are combined by a
    // fixed xor-shuffle tree -- deterministic, and every thread stays busy.
    int G = 1;
    while (G < 32 && 2 * G * nbx * nby <= (int)blockDim.x && 2 * G <= n) G *= 2;
    if (G > 1) {
        const int b = threadIdx.x / G, g = threadIdx.x & (G - 1);
        const bool live = b < nbx * nby;
        float acc[kFKR][kFMC];
#pragma unroll
        for (int r = 0; r < kFKR; ++r)
#pragma unroll
            for (int c = 0; c < kFMC; ++c) acc[r][c] = 0.f;
        int y0 = 0, x0 = 0;
        if (live) {
            int bx, by;
            block_of(b, nbx, nby, bx, by);
            y0 = dst.y0 + by * kFKR;
            x0 = dst.x0 + bx * kFMC;
            const bool inside = y0 + ry0 >= src.y0 && y0 + ry1 < src.y0 + src.h && x0 + rx0 >= src.x0 &&
                                x0 + rx1 < src.x0 + src.w;
            if (inside)
                block_taps<ADJ, false>(acc, S, src, s0, n, y0, x0, g, G);
            else
                block_taps<ADJ, true>(acc, S, src, s0, n, y0, x0, g, G);
        }
        for (int o = G >> 1; o > 0; o >>= 1)
#pragma unroll
            for (int r = 0; r < kFKR; ++r)
#pragma unroll
                for (int c = 0; c < kFMC; ++c) acc[r][c] += __shfl_xor_sync(0xffffffffu, acc[r][c], o);
        if (live && g == 0) {
#pragma unroll
            for (int r = 0; r < kFKR; ++r)
#pragma unroll
                for (int c = 0; c < kFMC; ++c) {
                    const int y = y0 + r, x = x0 + c;
                    if (y < dst.y0 + dst.h && x < dst.x0 + dst.w) {
                        dst.p[(y - dst.y0) * dst.s + (x - dst.x0)] = acc[r][c];
                        bad |= !isfinite(acc[r][c]);
                    }
                }
        }
        return __syncthreads_or(bad);
    }
    for (int b = threadIdx.x; b < nbx * nby; b += blockDim.x) {
        int bx, by;
        block_of(b, nbx, nby, bx, by);
        const int y0 = dst.y0 + by * kFKR, x0 = dst.x0 + bx * kFMC;
        float acc[kFKR][kFMC];
#pragma unroll
        for (int r = 0; r < kFKR; ++r)
#pragma unroll
            for (int c = 0; c < kFMC; ++c) acc[r][c] = 0.f;
        const bool inside = y0 + ry0 >= src.y0 && y0 + ry1 < src.y0 + src.h && x0 + rx0 >= src.x0 &&
                            x0 + rx1 < src.x0 + src.w;
        if (inside)
            block_taps<ADJ, false>(acc, S, src, s0, n, y0, x0);
        else
            block_taps<ADJ, true>(acc, S, src, s0, n, y0, x0);
#pragma unroll
        for (int r = 0; r < kFKR; ++r)
#pragma unroll
            for (int c = 0; c < kFMC; ++c) {
                const int y = y0 + r, x = x0 + c;
                if (y < dst.y0 + dst.h && x < dst.x0 + dst.w) {
                    dst.p[(y - dst.y0) * dst.s + (x - dst.x0)] = acc[r][c];
                    bad |= !isfinite(acc[r][c]);
                }
            }
    }
    return __syncthreads_or(bad);
}

// Forward chain on the live boxes (_forward_ir, optim.py:204-222).  Returns
// false (and fills bad_layer/bad_sample) on a non-finite intermediate.
__device__ bool forward(const FitParams &p, FitSmem &S) {
    for (int l = 0; l < p.L; ++l) {
        const Box o = S.box[l + 1];
        int bad = 0;
        if (o.w > 0 && o.h > 0) bad = gather_pass<false>(p, S, l, buf_of(S, l), buf_of(S, l + 1));
        if (bad) {
            if (threadIdx.x == 0) {
                S.bad_layer = l;
                S.bad_sample = -1;
                for (int i = 0; i < p.layout[l]; ++i) {
                    const int q = p.start[l] + i;
                    if (!(isfinite(S.off[q].x) && isfinite(S.off[q].y) && isfinite(S.w[q]))) {
                        S.bad_sample = i;
                        break;
                    }
                }
            }
            __syncthreads();
            return false;
        }
    }
    return true;
}

__device__ __forceinline__ float tgt_at(const FitParams &p, int b, int canvas, int y, int x) {
    const int pad = (canvas - p.M) / 2;   // DenseKernel.embedded (kernels.py:75-82)
    const int ty = y - pad, tx = x - pad;
    if (ty < 0 || ty >= p.M || tx < 0 || tx >= p.M) return 0.f;
    return __ldg(p.tgts + ((size_t)b * p.M + ty) * p.M + tx);
}

// Loss over the whole canvas (the IR is zero outside its live box); the loss
// gradient overwrites the IR on its box -- the reverse sweep reads it nowhere else.
__device__ double loss_and_grad(const FitParams &p, FitSmem &S, int b) {
    const int canvas = S.canvas;
    const Buf g = buf_of(S, p.L);
    double part = 0.0;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int y = ty; y < canvas; y += kFitWarps) {
        for (int x = tx; x < canvas; x += 32) {
            const unsigned dy = (unsigned)(y - g.y0), dx = (unsigned)(x - g.x0);
            const bool in = dy < (unsigned)g.h && dx < (unsigned)g.w;
            const float v = in ? g.p[dy * g.s + dx] : 0.f;
            const float d = v - tgt_at(p, b, canvas, y, x);
            part += (double)loss_term(d, p.cfg.loss_kind, p.cfg.loss_eps);
            if (in) g.p[dy * g.s + dx] = loss_grad(d, p.cfg.loss_kind, p.cfg.loss_eps);
        }
    }
    return block_sum(S, part);
}

// Per-tap gradients of layer l (_backward_pass, optim.py:231-263) from the
// four corner correlations C_c = <g_{l+1}, I_l shifted by corner c>:
//   d_w = sum_c a_c C_c, d_ox = w[(1-fy)(C10-C00) + fy(C11-C01)],
//   d_oy = w[(1-fx)(C01-C00) + fx(C11-C10)].
// Each warp owns up to kMaxTapsPerWarp taps and sweeps the whole box of
// g_{l+1}; per-block sums are fp32, accumulated across blocks in float64 and
// reduced by a fixed shuffle tree (deterministic, no atomics).
__device__ void correlate(const FitParams &p, FitSmem &S, int l, const Buf I, const Buf g) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s0 = p.start[l], n = p.layout[l];
    const int nbx = (g.w + kFMC - 1) / kFMC, nby = (g.h + kFKR - 1) / kFKR;
    const int4 dr = S.dr[l];
    // taps spread evenly over the warps, at most kMaxTapsPerWarp per sweep
    const int tpw = min(kMaxTapsPerWarp, (n + kFitWarps - 1) / kFitWarps);
    for (int t0 = warp * tpw; t0 < n; t0 += kFitWarps * tpw) {
        const int nt = min(tpw, n - t0);
        double C[kMaxTapsPerWarp][4];
#pragma unroll
        for (int k = 0; k < kMaxTapsPerWarp; ++k)
#pragma unroll
            for (int c = 0; c < 4; ++c) C[k][c] = 0.0;
        for (int b = lane; b < nbx * nby; b += 32) {
            int bx, by;
            block_of(b, nbx, nby, bx, by);
            const int y0 = g.y0 + by * kFKR, x0 = g.x0 + bx * kFMC;
            float gv[kFKR][kFMC];
#pragma unroll
            for (int r = 0; r < kFKR; ++r)
#pragma unroll
                for (int c = 0; c < kFMC; ++c) {
                    const int y = y0 + r, x = x0 + c;
                    gv[r][c] = (y < g.y0 + g.h && x < g.x0 + g.w) ? g.p[(y - g.y0) * g.s + (x - g.x0)] : 0.f;
                }
            const bool inside = y0 + dr.z >= I.y0 && y0 + kFKR - 1 + dr.w < I.y0 + I.h &&
                                x0 + dr.x >= I.x0 && x0 + kFMC - 1 + dr.y < I.x0 + I.w;
#pragma unroll
            for (int k = 0; k < kMaxTapsPerWarp; ++k) {
                if (k >= nt) break;
                const int2 d = S.ixy[s0 + t0 + k];
                float win[kFKR + 1][kFMC + 1];
                const int wy = y0 + d.y, wx = x0 + d.x;
                // a window that misses I's box reads only zeros: its products add
                // exact zeros, so the lane skips it (I is the small support of an
                // early intermediate, g the much larger box of a later gradient)
                if (wy > I.y0 + I.h - 1 || wy + kFKR < I.y0 || wx > I.x0 + I.w - 1 || wx + kFMC < I.x0) continue;
                const bool tin = inside || (wy >= I.y0 && wy + kFKR < I.y0 + I.h && wx >= I.x0 &&
                                            wx + kFMC < I.x0 + I.w);
                if (inside || __all_sync(__activemask(), tin)) {
                    if (I.so >= 0) {
                        const float *sb = smem_f32();
                        const int o = I.so + (y0 + d.y - I.y0) * I.s + (x0 + d.x - I.x0);
#pragma unroll
                        for (int r = 0; r <= kFKR; ++r)
#pragma unroll
                            for (int c = 0; c <= kFMC; ++c) win[r][c] = sb[o + r * I.s + c];
                    } else {
                        const float *q = I.p + (y0 + d.y - I.y0) * I.s + (x0 + d.x - I.x0);
#pragma unroll
                        for (int r = 0; r <= kFKR; ++r)
#pragma unroll
                            for (int c = 0; c <= kFMC; ++c) win[r][c] = q[r * I.s + c];
                    }
                } else {
#pragma unroll
                    for (int r = 0; r <= kFKR; ++r)
#pragma unroll
                        for (int c = 0; c <= kFMC; ++c) win[r][c] = ld_chk(I, y0 + d.y + r, x0 + d.x + c);
                }
                float c00 = 0.f, c10 = 0.f, c01 = 0.f, c11 = 0.f;
#pragma unroll
                for (int r = 0; r < kFKR; ++r)
#pragma unroll
                    for (int c = 0; c < kFMC; ++c) {
                        const float v = gv[r][c];
                        c00 = fmaf(v, win[r][c], c00);
                        c10 = fmaf(v, win[r][c + 1], c10);
                        c01 = fmaf(v, win[r + 1][c], c01);
                        c11 = fmaf(v, win[r + 1][c + 1], c11);
                    }
                C[k][0] += c00;
                C[k][1] += c10;
                C[k][2] += c01;
                C[k][3] += c11;
            }
        }
#pragma unroll
        for (int k = 0; k < kMaxTapsPerWarp; ++k) {
            if (k >= nt) break;
            double c4[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) c4[c] = warp_sum(C[k][c]);
            if (lane == 0) {
                const int q = s0 + t0 + k;
                const double fx = S.frac[q].x, fy = S.frac[q].y, w = S.w[q];
                const double dw = (1 - fx) * (1 - fy) * c4[0] + fx * (1 - fy) * c4[1] + (1 - fx) * fy * c4[2] +
                                  fx * fy * c4[3];
                const double dx = w * ((1 - fy) * (c4[1] - c4[0]) + fy * (c4[3] - c4[2]));
                const double dy = w * ((1 - fx) * (c4[2] - c4[0]) + fx * (c4[3] - c4[1]));
                S.grad[q] = make_float3((float)dx, (float)dy, (float)dw);
            }
        }
    }
}

// Reverse sweep: gradients of layer l, then (l > 0) the adjoint into I_l's
// buffer, which corr(l) no longer needs.
__device__ void backward_sweep(const FitParams &p, FitSmem &S) {
    for (int l = p.L - 1; l >= 0; --l) {
        const Buf I = buf_of(S, l), g = buf_of(S, l + 1);
        if (g.w > 0 && g.h > 0) {
            correlate(p, S, l, I, g);
        } else {
            for (int q = p.start[l] + threadIdx.x; q < p.start[l + 1]; q += blockDim.x)
                S.grad[q] = make_float3(0.f, 0.f, 0.f);
        }
        __syncthreads();
        if (l > 0 && I.w > 0 && I.h > 0) {
            if (g.w > 0 && g.h > 0) {
                gather_pass<true>(p, S, l, g, I);
            } else {
                for (int e = threadIdx.x; e < I.s * I.h; e += blockDim.x) I.p[e] = 0.f;
                __syncthreads();
            }
        }
    }
}

__device__ __forceinline__ int param_index(const FitParams &p, int q) {
    // flat tap q -> (l, i) -> row in the (L, nmax) parameter block
    int l = 0;
    while (l + 1 < p.L && q >= p.start[l + 1]) ++l;
    return l * p.nmax + (q - p.start[l]);
}

// KWS tie (optim.py:312-325) then SUM projection (328-335).  Returns the
// degenerate layer or -1.
__device__ int project(const FitParams &p, FitSmem &S) {
    if (p.cfg.kws) {
        const int ngroups = p.P / 4;
        for (int gq = threadIdx.x; gq < ngroups; gq += blockDim.x) {
            const int q = 4 * gq;  // layers are multiples of 4, so groups never straddle layers
            const float sx[4] = {1.f, -1.f, -1.f, 1.f}, sy[4] = {1.f, 1.f, -1.f, -1.f};
            float dx = 0.f, dy = 0.f, mw = 0.f;
            for (int k = 0; k < 4; ++k) {
                dx += sx[k] * S.off[q + k].x;
                dy += sy[k] * S.off[q + k].y;
                mw += S.wp[q + k];
            }
            dx /= 4.f;
            dy /= 4.f;
            mw /= 4.f;
            for (int k = 0; k < 4; ++k) {
                S.off[q + k] = make_float2(sx[k] * dx, sy[k] * dy);
                S.wp[q + k] = mw;
            }
        }
        __syncthreads();
    }
    int bad = -1;
    if (p.cfg.weight_norm == SKC_WN_SUM) {
        if (threadIdx.x == 0) {
            S.flag = -1;
            for (int l = 0; l < p.L; ++l) {
                float s = 0.f;
                for (int i = 0; i < p.layout[l]; ++i) s += S.wp[p.start[l] + i];
                if (fabsf(s) < 1e-8f) { S.flag = l; break; }
                for (int i = 0; i < p.layout[l]; ++i) S.wp[p.start[l] + i] /= s;
            }
        }
        __syncthreads();
        bad = S.flag;
        __syncthreads();
    }
    return bad;
}

__device__ __forceinline__ int &hdr_i(float *st, int k) { return reinterpret_cast<int *>(st)[k]; }

__global__ void __launch_bounds__(kFitThreads, 2) fit_kernel(const __grid_constant__ FitParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FitSmem &S = *reinterpret_cast<FitSmem *>(smem_raw);
    float *arena = reinterpret_cast<float *>(smem_raw + (sizeof(FitSmem) + 15) / 16 * 16);
    const int b = p.idx ? p.idx[blockIdx.x] : blockIdx.x;
    const int blk = p.L * p.nmax * 3;
    int *status = p.status + 4 * b;
    // overflow slots are per launched CTA: a relaunch of parked targets only
    // sizes scratch for those
    float *gslots = p.scratch + (size_t)blockIdx.x * p.L * p.cap * p.cap;

    if (p.mode != MODE_FIT) {
        // backward()/synthesize_ir(): parameters come in as effective weights
        const float *t = p.taps_in + (size_t)b * blk;
        for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
            const int r = param_index(p, q);
            S.off[q] = make_float2(t[3 * r], t[3 * r + 1]);
            S.w[q] = t[3 * r + 2];
            S.wp[q] = S.w[q];
        }
        if (threadIdx.x == 0) S.canvas = p.canvas_fixed;
        __syncthreads();
        build_taps_and_boxes(p, S, arena, gslots);
        const bool ok = forward(p, S);
        if (!ok && p.mode == MODE_ENERGY) {
            if (threadIdx.x == 0) p.energy_out[b] = INFINITY;   // rejected like a non-finite proposal
            return;
        }
        if (!ok) {
            if (threadIdx.x == 0) {
                status[0] = SKC_ENONFINITE;
                status[1] = S.bad_layer;
                status[2] = S.bad_sample;
                status[3] = 0;
            }
            return;
        }
        if (p.mode == MODE_ENERGY) {
            // baselines.pst_fit energies_of (baselines.py:175-191): pixel-summed
            // loss against the shared target, plus the "leak wall": a response
            // whose mass differs from prod_l sum_i w_li (truncated off the
            // canvas) is invalid (energy +inf)
            const int cv = S.canvas;
            const Buf ir = buf_of(S, p.L);
            const int bt = p.tgt_shared ? 0 : b;
            double part = 0.0, mass = 0.0;
            const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
            for (int y = ty; y < cv; y += kFitWarps)
                for (int x = tx; x < cv; x += 32) {
                    const float v = ld_chk(ir, y, x);
                    mass += (double)v;
                    part += (double)loss_term(v - tgt_at(p, bt, cv, y, x), p.cfg.loss_kind, p.cfg.loss_eps);
                }
            const double e = block_sum(S, part);
            const double m = block_sum(S, mass);
            if (threadIdx.x == 0) {
                double expected = 1.0;
                for (int l = 0; l < p.L; ++l) {
                    double sw = 0.0;
                    for (int i = 0; i < p.layout[l]; ++i) sw += (double)S.w[p.start[l] + i];
                    expected *= sw;
                }
                const double tol = 1e-6 * fmax(fabs(expected), 1.0);
                p.energy_out[b] = fabs(m - expected) > tol ? INFINITY : e;
            }
            return;
        }
        if (p.mode == MODE_IR) {
            const int cv = S.canvas;
            const Buf ir = buf_of(S, p.L);
            float *out = p.ir_out + (size_t)b * cv * cv;
            for (int e = threadIdx.x; e < cv * cv; e += blockDim.x) {
                const int y = e / cv, x = e - y * cv;
                out[e] = ld_chk(ir, y, x);
            }
            if (threadIdx.x == 0) status[0] = SKC_OK;
            return;
        }
        const double loss = loss_and_grad(p, S, b);
        __syncthreads();
        backward_sweep(p, S);
        float *go = p.grads_out + (size_t)b * blk;
        for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
            const int r = param_index(p, q);
            go[3 * r] = S.grad[q].x;
            go[3 * r + 1] = S.grad[q].y;
            go[3 * r + 2] = S.grad[q].z;
        }
        if (threadIdx.x == 0) {
            p.loss_out[b] = (float)loss;
            status[0] = SKC_OK;
        }
        return;
    }

    // ---------------------------------------------------------- MODE_FIT ---
    float *st = p.state + (size_t)b * SKC_FIT_STATE_FLOATS(p.L, p.nmax);
    float *prm = st + SKC_FIT_HDR;
    float *am = prm + blk;
    float *av = am + blk;
    float *best = av + blk;
    float *trace = p.trace + (size_t)b * (p.cfg.steps + 1);
    if (status[0] != SKC_OK && status[0] != kNeedGrow) return;  // failed earlier
    int step = hdr_i(st, 0);
    if (step > p.cfg.steps) return;                              // finished
    for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
        const int r = param_index(p, q);
        S.off[q] = make_float2(prm[3 * r], prm[3 * r + 1]);
        S.wp[q] = prm[3 * r + 2];
    }
    if (threadIdx.x == 0) S.canvas = hdr_i(st, 1);
    __syncthreads();
    float best_loss = st[2];
    int best_step = hdr_i(st, 3);
    const float scale = (float)p.M;  // offset_lr_scale = k_tgt.size (optim.py:411)
    int code = SKC_OK, err_layer = 0, err_sample = -1;

    for (;; ++step) {
        effective_weights(p, S);
        // embed_if_grown (optim.py:429-434): reach = sum_l max |o| (engine.py:68-71, 101-103)
        if (threadIdx.x == 0) {
            float reach = 0.f;
            for (int l = 0; l < p.L; ++l) {
                float m = 0.f;
                for (int i = 0; i < p.layout[l]; ++i) {
                    const float2 o = S.off[p.start[l] + i];
                    m = fmaxf(m, fmaxf(fabsf(o.x), fabsf(o.y)));
                }
                reach += m;
            }
            const int need = 2 * (int)ceilf(reach) + 1;
            if (need > S.canvas) S.canvas = need + 4;
            S.flag = S.canvas > p.cap;
        }
        __syncthreads();
        if (S.flag) { code = kNeedGrow; break; }
        build_taps_and_boxes(p, S, arena, gslots);
        if (!forward(p, S)) {
            code = SKC_ENONFINITE;
            err_layer = S.bad_layer;
            err_sample = S.bad_sample;
            break;
        }
        const double loss = loss_and_grad(p, S, b);
        const float lossf = (float)loss;
        if (threadIdx.x == 0) trace[step] = lossf;
        if (lossf < best_loss) {   // strict improvement, optim.py:442-445
            best_loss = lossf;
            best_step = step;
            for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
                const int r = param_index(p, q);
                best[3 * r] = S.off[q].x;
                best[3 * r + 1] = S.off[q].y;
                best[3 * r + 2] = S.w[q];
            }
        }
        if (step == p.cfg.steps) { step = p.cfg.steps + 1; break; }
        __syncthreads();
        backward_sweep(p, S);
        // _chain_weight_norm (optim.py:266-275)
        if (p.cfg.weight_norm == SKC_WN_SOFM) {
            if (threadIdx.x < p.L) {
                const int s0 = p.start[threadIdx.x], n = p.layout[threadIdx.x];
                float dot = 0.f;
                for (int i = 0; i < n; ++i) dot += S.grad[s0 + i].z * S.w[s0 + i];
                for (int i = 0; i < n; ++i) S.grad[s0 + i].z = S.w[s0 + i] * (S.grad[s0 + i].z - dot);
            }
            __syncthreads();
        }
        // adam_step (optim.py:338-369), bias correction at t = step + 1
        {
            const int T = p.cfg.steps;
            const int tc = min(max(step, 0), T - 1);
            const double lr = (T == 1) ? (double)p.cfg.lr_start
                                       : (double)p.cfg.lr_start + ((double)p.cfg.lr_end - (double)p.cfg.lr_start) * tc / (double)(T - 1);
            const double tt = (double)(step + 1);
            const float c1 = (float)(1.0 - pow((double)p.cfg.beta1, tt));
            const float c2 = (float)(1.0 - pow((double)p.cfg.beta2, tt));
            const float b1 = p.cfg.beta1, b2 = p.cfg.beta2, eps = p.cfg.eps;
            const float lrf = (float)lr;
            for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
                const int r = param_index(p, q);
                const float g3[3] = {S.grad[q].x, S.grad[q].y, S.grad[q].z};
                float pv[3] = {S.off[q].x, S.off[q].y, S.wp[q]};
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const float g = g3[k];
                    const float m = am[3 * r + k] * b1 + (1.f - b1) * g;
                    const float v = av[3 * r + k] * b2 + (1.f - b2) * g * g;
                    am[3 * r + k] = m;
                    av[3 * r + k] = v;
                    const float s = k < 2 ? scale : 1.f;
                    pv[k] = pv[k] - s * lrf * (m / c1) / (sqrtf(v / c2) + eps);
                }
                S.off[q] = make_float2(pv[0], pv[1]);
                S.wp[q] = pv[2];
            }
            __syncthreads();
        }
        const int badl = project(p, S);
        if (badl >= 0) {
            code = SKC_EDEGENERATE;
            err_layer = badl;
            break;
        }
    }

    // persist state (resumable after kNeedGrow)
    __syncthreads();
    for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
        const int r = param_index(p, q);
        prm[3 * r] = S.off[q].x;
        prm[3 * r + 1] = S.off[q].y;
        prm[3 * r + 2] = S.wp[q];
    }
    if (threadIdx.x == 0) {
        hdr_i(st, 0) = step;
        hdr_i(st, 1) = S.canvas;
        st[2] = best_loss;
        hdr_i(st, 3) = best_step;
        status[0] = code;
        status[1] = err_layer;
        status[2] = err_sample;
        status[3] = step;
    }
}

// Initialise fit state from an explicit init complex: parameters
// (_params_from_complex, optim.py:168-176), KWS/SUM projections (414-417),
// the initial canvas max(auto_canvas, M) (419-420).
__global__ void fit_init_kernel(const __grid_constant__ FitParams p, const float *init) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FitSmem &S = *reinterpret_cast<FitSmem *>(smem_raw);
    const int b = blockIdx.x;
    const int blk = p.L * p.nmax * 3;
    float *st = p.state + (size_t)b * SKC_FIT_STATE_FLOATS(p.L, p.nmax);
    float *prm = st + SKC_FIT_HDR;
    const float *t = init + (size_t)b * blk;
    for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
        const int r = param_index(p, q);
        S.off[q] = make_float2(t[3 * r], t[3 * r + 1]);
        const float w = t[3 * r + 2];
        S.wp[q] = (p.cfg.weight_norm == SKC_WN_SOFM) ? logf(fmaxf(w, 1e-12f)) : w;
    }
    for (int e = threadIdx.x; e < SKC_FIT_STATE_FLOATS(p.L, p.nmax) - SKC_FIT_HDR; e += blockDim.x)
        prm[e] = 0.f;
    __syncthreads();
    const int bad = project(p, S);
    for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
        const int r = param_index(p, q);
        prm[3 * r] = S.off[q].x;
        prm[3 * r + 1] = S.off[q].y;
        prm[3 * r + 2] = S.wp[q];
    }
    if (threadIdx.x == 0) {
        float reach = 0.f;
        for (int l = 0; l < p.L; ++l) {
            float m = 0.f;
            for (int i = 0; i < p.layout[l]; ++i) {
                const float2 o = S.off[p.start[l] + i];
                m = fmaxf(m, fmaxf(fabsf(o.x), fabsf(o.y)));
            }
            reach += m;
        }
        const int canvas = max(2 * (int)ceilf(reach) + 1 + 4, p.M);
        hdr_i(st, 0) = 0;
        hdr_i(st, 1) = canvas;
        st[2] = INFINITY;
        hdr_i(st, 3) = 0;
        int *status = p.status + 4 * b;
        status[0] = bad >= 0 ? SKC_EDEGENERATE : SKC_OK;
        status[1] = bad >= 0 ? bad : 0;
        status[2] = -1;
        status[3] = 0;
    }
}

// Standalone Adam step on one complex (optim.adam_step): a single CTA.
__global__ void adam_kernel(float *params, const float *grads, float *m, float *v,
                            const __grid_constant__ FitParams p, int step, float scale, int *status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FitSmem &S = *reinterpret_cast<FitSmem *>(smem_raw);
    const int T = p.cfg.steps;
    const int tc = min(max(step, 0), T - 1);
    const double lr = (T == 1) ? (double)p.cfg.lr_start
                               : (double)p.cfg.lr_start + ((double)p.cfg.lr_end - (double)p.cfg.lr_start) * tc / (double)(T - 1);
    const double tt = (double)(step + 1);
    const float c1 = (float)(1.0 - pow((double)p.cfg.beta1, tt));
    const float c2 = (float)(1.0 - pow((double)p.cfg.beta2, tt));
    for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
        float pv[3];
        for (int k = 0; k < 3; ++k) {
            const float g = grads[3 * q + k];
            const float mm = m[3 * q + k] * p.cfg.beta1 + (1.f - p.cfg.beta1) * g;
            const float vv = v[3 * q + k] * p.cfg.beta2 + (1.f - p.cfg.beta2) * g * g;
            m[3 * q + k] = mm;
            v[3 * q + k] = vv;
            const float s = k < 2 ? scale : 1.f;
            pv[k] = params[3 * q + k] - s * (float)lr * (mm / c1) / (sqrtf(vv / c2) + p.cfg.eps);
        }
        S.off[q] = make_float2(pv[0], pv[1]);
        S.wp[q] = pv[2];
    }
    __syncthreads();
    const int bad = project(p, S);
    for (int q = threadIdx.x; q < p.P; q += blockDim.x) {
        params[3 * q] = S.off[q].x;
        params[3 * q + 1] = S.off[q].y;
        params[3 * q + 2] = S.wp[q];
    }
    if (threadIdx.x == 0) {
        status[0] = bad >= 0 ? SKC_EDEGENERATE : SKC_OK;
        status[1] = bad >= 0 ? bad : 0;
        status[2] = -1;
        status[3] = step;
    }
}

static int fill_params(FitParams &p, int B, const int *layout, int L, int nmax, int M) {
    if (B < 1) return fail(SKC_EBADARG, "batch must be positive");
    if (L < 1 || L > kFitMaxL) return fail(SKC_EBADARG, "fit supports 1..8 layers");
    if (!layout) return fail(SKC_EBADARG, "null layout");
    std::memset(&p, 0, sizeof(p));
    p.B = B;
    p.L = L;
    p.nmax = nmax;
    p.M = M;
    p.start[0] = 0;
    for (int l = 0; l < L; ++l) {
        if (layout[l] < 1 || layout[l] > nmax) return fail(SKC_EBADARG, "layout entries must be 1..nmax");
        p.layout[l] = layout[l];
        p.start[l + 1] = p.start[l] + layout[l];
    }
    p.P = p.start[L];
    if (p.P > kFitMaxP) return fail(SKC_EBADARG, "fit supports at most 256 taps per complex");
    return SKC_OK;
}

static int set_fit_attrs() {
    int rc;
    if ((rc = smem_optin((const void *)fit_kernel, kFitSmem))) return rc;
    if ((rc = smem_optin((const void *)fit_init_kernel, kFitSmem))) return rc;
    return smem_optin((const void *)adam_kernel, kFitSmem);
}

static int fit_launch(const FitParams &p, cudaStream_t s, int grid = -1) {
    int rc = set_fit_attrs();
    if (rc) return rc;
    fit_kernel<<<grid < 0 ? p.B : grid, kFitThreads, kFitSmem, s>>>(p);
    SKC_LAUNCH_CHECK("fit_kernel");
    return SKC_OK;
}

static int alloc_scratch(FitParams &p, int cap, cudaStream_t s, int ctas = -1) {
    p.cap = cap;
    const size_t bytes = (size_t)(ctas < 0 ? p.B : ctas) * p.L * cap * cap * sizeof(float);
    void *ptr = nullptr;
    int rc = pool_alloc(&ptr, bytes, s);
    if (rc) return rc;
    p.scratch = (float *)ptr;
    return SKC_OK;
}

static bool cfg_ok(const skc_fit_cfg *c) {
    return c && c->steps >= 1 && c->lr_start >= c->lr_end && c->lr_end > 0 &&
           (c->weight_norm == SKC_WN_NONE || c->weight_norm == SKC_WN_SUM || c->weight_norm == SKC_WN_SOFM) &&
           (c->loss_kind >= 0 && c->loss_kind <= 2) && c->loss_eps > 0;
}


// ------------------------------------------------- PST energy evaluation ---
// skc_pst.cu replays the MODE_ENERGY launch once per tempering iteration on
// fixed device buffers (proposal taps in, chain energies out), so its
// parameter block is built once and the launch is CUDA-graph capturable.
struct EnergyPlan {
    FitParams p;
};

int energy_plan_create(EnergyPlan **out, int B, const int *layout, int L, int nmax, int canvas,
                       const float *tgt, int M, int loss_kind, float loss_eps, const float *taps,
                       double *energies, cudaStream_t s) {
    *out = nullptr;
    EnergyPlan *e = new EnergyPlan();
    FitParams &p = e->p;
    int rc = fill_params(p, B, layout, L, nmax, M);
    if (!rc && (canvas < M || (canvas & 1) == 0 || (M & 1) == 0))
        rc = fail(SKC_EBADARG, "canvas/target must be odd, canvas >= M");
    if (!rc && (loss_kind < 0 || loss_kind > 2 || !(loss_eps > 0))) rc = fail(SKC_EBADARG, "bad loss kind");
    if (rc) { delete e; return rc; }
    p.mode = MODE_ENERGY;
    p.canvas_fixed = canvas;
    p.taps_in = taps;
    p.tgts = tgt;
    p.tgt_shared = 1;
    p.energy_out = energies;
    p.cfg.steps = 1;
    p.cfg.loss_kind = loss_kind;
    p.cfg.loss_eps = loss_eps;
    void *st = nullptr;
    if ((rc = pool_alloc(&st, (size_t)B * 4 * sizeof(int), s))) { delete e; return rc; }
    p.status = (int *)st;
    if ((rc = alloc_scratch(p, canvas, s))) { pool_free(st, s); delete e; return rc; }
    if ((rc = set_fit_attrs())) { pool_free(p.scratch, s); pool_free(st, s); delete e; return rc; }
    *out = e;
    return SKC_OK;
}

int energy_plan_launch(const EnergyPlan *e, cudaStream_t s) {
    fit_kernel<<<e->p.B, kFitThreads, kFitSmem, s>>>(e->p);
    SKC_LAUNCH_CHECK("fit_kernel (energies)");
    return SKC_OK;
}

void energy_plan_destroy(EnergyPlan *e, cudaStream_t s) {
    if (!e) return;
    pool_free(e->p.scratch, s);
    pool_free(e->p.status, s);
    delete e;
}

}  // namespace skc

using namespace skc;

extern "C" {

int skc_ir_batch(const float *taps, int B, const int *layout, int L, int nmax, int canvas,
                 float *out, void *stream) {
    FitParams p;
    int rc = fill_params(p, B, layout, L, nmax, 1);
    if (rc) return rc;
    if (!taps || !out) return fail(SKC_EBADARG, "null pointer");
    if (canvas < 1 || (canvas & 1) == 0) return fail(SKC_EBADARG, "canvas must be odd");
    cudaStream_t s = (cudaStream_t)stream;
    p.mode = MODE_IR;
    p.canvas_fixed = canvas;
    p.taps_in = taps;
    p.ir_out = out;
    p.cfg.steps = 1;
    void *st = nullptr;
    if ((rc = pool_alloc(&st, (size_t)B * 4 * sizeof(int), s))) return rc;
    p.status = (int *)st;
    if ((rc = alloc_scratch(p, canvas, s))) { pool_free(st, s); return rc; }
    rc = fit_launch(p, s);
    std::vector<int> hs((size_t)B * 4);
    if (rc == SKC_OK) {
        cudaError_t e = cudaMemcpyAsync(hs.data(), st, hs.size() * sizeof(int), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) rc = cuda_fail(e, "skc_ir_batch status");
    }
    pool_free(p.scratch, s);
    pool_free(st, s);
    if (rc) return rc;
    for (int b = 0; b < B; ++b)
        if (hs[4 * b] == SKC_ENONFINITE)
            return fail(SKC_ENONFINITE, "non-finite intermediate at layer " + std::to_string(hs[4 * b + 1]));
    return SKC_OK;
}

int skc_ir_energies(const float *taps, int B, const int *layout, int L, int nmax, int canvas,
                    const float *tgt, int M, int loss_kind, float loss_eps, double *energies,
                    void *stream) {
    FitParams p;
    int rc = fill_params(p, B, layout, L, nmax, M);
    if (rc) return rc;
    if (!taps || !tgt || !energies) return fail(SKC_EBADARG, "null pointer");
    if (canvas < M || (canvas & 1) == 0 || (M & 1) == 0) return fail(SKC_EBADARG, "canvas/target must be odd, canvas >= M");
    if (loss_kind < 0 || loss_kind > 2 || !(loss_eps > 0)) return fail(SKC_EBADARG, "bad loss kind");
    cudaStream_t s = (cudaStream_t)stream;
    p.mode = MODE_ENERGY;
    p.canvas_fixed = canvas;
    p.taps_in = taps;
    p.tgts = tgt;
    p.tgt_shared = 1;
    p.energy_out = energies;
    p.cfg.steps = 1;
    p.cfg.loss_kind = loss_kind;
    p.cfg.loss_eps = loss_eps;
    void *st = nullptr;
    if ((rc = pool_alloc(&st, (size_t)B * 4 * sizeof(int), s))) return rc;
    p.status = (int *)st;
    if ((rc = alloc_scratch(p, canvas, s))) { pool_free(st, s); return rc; }
    rc = fit_launch(p, s);
    pool_free(p.scratch, s);
    pool_free(st, s);
    return rc;
}

int skc_backward_batch(const float *taps, int B, const int *layout, int L, int nmax,
                       const float *tgts, int M, int canvas, int loss_kind, float loss_eps,
                       float *loss, float *grads, int *status, void *stream) {
    FitParams p;
    int rc = fill_params(p, B, layout, L, nmax, M);
    if (rc) return rc;
    if (!taps || !tgts || !loss || !grads || !status) return fail(SKC_EBADARG, "null pointer");
    if (canvas < M || (canvas & 1) == 0 || (M & 1) == 0) return fail(SKC_EBADARG, "canvas/target must be odd, canvas >= M");
    if (loss_kind < 0 || loss_kind > 2 || !(loss_eps > 0)) return fail(SKC_EBADARG, "bad loss kind");
    cudaStream_t s = (cudaStream_t)stream;
    p.mode = MODE_BACKWARD;
    p.canvas_fixed = canvas;
    p.taps_in = taps;
    p.tgts = tgts;
    p.loss_out = loss;
    p.grads_out = grads;
    p.status = status;
    p.cfg.steps = 1;
    p.cfg.loss_kind = loss_kind;
    p.cfg.loss_eps = loss_eps;
    if ((rc = alloc_scratch(p, canvas, s))) return rc;
    SKC_CUDA(cudaMemsetAsync(grads, 0, (size_t)B * L * nmax * 3 * sizeof(float), s));
    rc = fit_launch(p, s);
    pool_free(p.scratch, s);
    return rc;
}

int skc_fit_init(float *state, const float *init_taps, int B, const int *layout, int L, int nmax,
                 int M, const skc_fit_cfg *cfg, int *status, void *stream) {
    FitParams p;
    int rc = fill_params(p, B, layout, L, nmax, M);
    if (rc) return rc;
    if (!state || !init_taps || !status) return fail(SKC_EBADARG, "null pointer");
    if (!cfg_ok(cfg)) return fail(SKC_EBADARG, "invalid fit configuration");
    if (cfg->kws)
        for (int l = 0; l < L; ++l)
            if (layout[l] % 4) return fail(SKC_EBADARG, "KWS symmetry needs sample counts divisible by 4");
    cudaStream_t s = (cudaStream_t)stream;
    p.mode = MODE_FIT;
    p.cfg = *cfg;
    p.state = state;
    p.status = status;
    if ((rc = set_fit_attrs())) return rc;
    fit_init_kernel<<<B, kFitThreads, sizeof(FitSmem), s>>>(p, init_taps);
    SKC_LAUNCH_CHECK("fit_init_kernel");
    return SKC_OK;
}

int skc_fit_run(float *state, int B, const int *layout, int L, int nmax, const float *tgts, int M,
                const skc_fit_cfg *cfg, float *trace, int *status, void *stream) {
    FitParams p;
    int rc = fill_params(p, B, layout, L, nmax, M);
    if (rc) return rc;
    if (!state || !tgts || !trace || !status) return fail(SKC_EBADARG, "null pointer");
    if (!cfg_ok(cfg)) return fail(SKC_EBADARG, "invalid fit configuration");
    cudaStream_t s = (cudaStream_t)stream;
    p.mode = MODE_FIT;
    p.cfg = *cfg;
    p.state = state;
    p.tgts = tgts;
    p.trace = trace;
    p.status = status;
    const size_t stride = SKC_FIT_STATE_FLOATS(L, nmax);
    std::vector<int> hdr((size_t)B * 4), hs((size_t)B * 4);
    // Every target starts in one launch with a generous scratch canvas.  A
    // target whose canvas outgrows it parks (kNeedGrow); only the parked
    // targets are relaunched, compacted through an index list with scratch
    // sized for them (optim.py:429-434 grows only that fit's canvas).  A
    // canvas beyond kMaxFitCanvas stops that target with SKC_ETRUNC in its
    // status row; the rest of the batch is unaffected.
    constexpr int kMaxFitCanvas = 4097;
    SKC_CUDA(cudaMemcpy2DAsync(hdr.data(), 4 * sizeof(int), state, stride * sizeof(float),
                               4 * sizeof(int), B, cudaMemcpyDeviceToHost, s));
    SKC_CUDA(cudaStreamSynchronize(s));
    int cap = 1;
    for (int b = 0; b < B; ++b) cap = std::max(cap, hdr[4 * b + 1]);
    cap = std::min(2 * cap + 32, kMaxFitCanvas);
    std::vector<int> parked;
    int *d_idx = nullptr;
    for (int attempt = 0;; ++attempt) {
        const int ctas = attempt == 0 ? B : (int)parked.size();
        p.idx = attempt == 0 ? nullptr : d_idx;
        if ((rc = alloc_scratch(p, cap, s, ctas))) break;
        rc = fit_launch(p, s, ctas);
        if (rc == SKC_OK) {
            cudaError_t e = cudaMemcpyAsync(hs.data(), status, hs.size() * sizeof(int),
                                            cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaMemcpy2DAsync(hdr.data(), 4 * sizeof(int), state, stride * sizeof(float),
                                                        4 * sizeof(int), B, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) rc = cuda_fail(e, "skc_fit_run status");
        }
        pool_free(p.scratch, s);
        if (rc) break;
        parked.clear();
        int need = 0;
        for (int b = 0; b < B; ++b) {
            if (hs[4 * b] != kNeedGrow) continue;
            if (hdr[4 * b + 1] > kMaxFitCanvas) {
                const int row[4] = {SKC_ETRUNC, 0, -1, hs[4 * b + 3]};
                cudaError_t e = cudaMemcpyAsync(status + 4 * b, row, sizeof(row), cudaMemcpyHostToDevice, s);
                if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                if (e != cudaSuccess) { rc = cuda_fail(e, "skc_fit_run status"); break; }
                continue;
            }
            parked.push_back(b);
            need = std::max(need, hdr[4 * b + 1]);
        }
        if (rc || parked.empty()) break;
        cap = std::min(need + need / 2 + 64, kMaxFitCanvas);
        // bound one relaunch's scratch; targets left out stay parked and run
        // in a later round of this loop
        const size_t per = (size_t)L * cap * cap * sizeof(float);
        const size_t fit = std::max<size_t>(1, (size_t(8) << 30) / per);
        if (parked.size() > fit) parked.resize(fit);
        if (d_idx) pool_free(d_idx, s);
        d_idx = nullptr;
        if ((rc = pool_alloc((void **)&d_idx, parked.size() * sizeof(int), s))) break;
        cudaError_t e = cudaMemcpyAsync(d_idx, parked.data(), parked.size() * sizeof(int), cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);   // `parked` is reused next round
        if (e != cudaSuccess) { rc = cuda_fail(e, "skc_fit_run index"); break; }
    }
    if (d_idx) pool_free(d_idx, s);
    return rc;
}

int skc_adam_step(float *params, const float *grads, float *m, float *v, const int *layout, int L,
                  int step_index, const skc_fit_cfg *cfg, float offset_lr_scale, int *status,
                  void *stream) {
    FitParams p;
    int nmax = 1;
    for (int l = 0; layout && l < L; ++l) nmax = std::max(nmax, layout[l]);
    int rc = fill_params(p, 1, layout, L, nmax, 1);
    if (rc) return rc;
    if (!params || !grads || !m || !v || !status) return fail(SKC_EBADARG, "null pointer");
    if (!cfg_ok(cfg)) return fail(SKC_EBADARG, "invalid fit configuration");
    if (cfg->kws)
        for (int l = 0; l < L; ++l)
            if (layout[l] % 4) return fail(SKC_EBADARG, "KWS symmetry needs sample counts divisible by 4");
    p.cfg = *cfg;
    if ((rc = set_fit_attrs())) return rc;
    adam_kernel<<<1, kFitThreads, sizeof(FitSmem), (cudaStream_t)stream>>>(
        params, grads, m, v, p, step_index, offset_lr_scale, status);
    SKC_LAUNCH_CHECK("adam_kernel");
    return SKC_OK;
}

}  // extern "C"
