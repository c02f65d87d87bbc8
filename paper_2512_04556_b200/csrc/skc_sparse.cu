// skc_sparse.cu -- layer-specialised sparse stencils, generated and compiled at
// run time with NVRTC (sm_100a).
//
// Reference: engine.apply_sparse_layer (engine.py:160-170) -> sample_shifted
// (118-130) -> _accum_shift (106-115).  A uniform layer of S bilinear taps is
// an integer stencil with at most 4S nonzero positions: the tap's 4 corners,
// coincident corners merged in float64 and rounded once (the dense path's
// rule, skc_layer.cu try_stencil).  For footprints wider than the 9 x 9 dense
// kernels the tap kernel is shared-memory bound (~1.3 window words per
// output per tap, SMEM 32 words/clk/SM against 128 FMA/clk/SM).  Knowing the
// positions at compile time removes that bound: each thread slides down the
// input rows of its KR x 8 output block once, loads only the columns the
// stencil rows touching that input row need (LDS.128, conflict-free), and
// issues one FFMA with an immediate weight per (position, output) -- no
// per-tap window reloads, no zero work.  Config 1's radius-8 layer (32 taps ->
// 102 positions in 15 x 17) reads ~10 words per output instead of ~41.
//
// The kernel source is emitted per position pattern (the merged weights are a
// kernel parameter), compiled with NVRTC (dlopen'ed libnvrtc.so.12, no
// link-time dependency) on a background thread while the tap / dense kernels
// serve the layer (SKC_JIT=sync waits instead), loaded with
// cudaLibraryLoadData and kept in a bounded LRU cache keyed by the source.
// SKC_SPARSE=0 disables the path; SKC_SPARSE=1 forces it for every eligible
// layer regardless of the cost model; SKC_SPARSE_DUMP=<dir> writes the
// generated sources.
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <memory>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "skc_tile.cuh"

namespace skc {
namespace {

constexpr int kSpTW = 128;

int env_int(const char *name, int dflt) {
    const char *e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
// Rows per thread KR (odd: LDS.128 conflict-free with pitch = 4 mod 8; tile
// 128 x 16 KR), barrier period in input rows (0 = none) and minimum resident
// CTAs per SM of the generated kernel (SKC_SPARSE_KR / _SYNC / _MINB).
int sp_kr() {
    static const int v = [] { const int k = env_int("SKC_SPARSE_KR", 3); return (k == 1 || k == 3 || k == 5 || k == 7 || k == 9) ? k : 3; }();
    return v;
}
int sp_kr_wide() {
    static const int v = [] { const int k = env_int("SKC_SPARSE_KR_WIDE", 5); return (k == 3 || k == 5 || k == 7) ? k : 5; }();
    return v;
}
int sp_sync() {
    static const int v = env_int("SKC_SPARSE_SYNC", 0);
    return v;
}
// Packed-FP32 body (default; SKC_SPARSE_F2=0 emits scalar FFMAs with
// immediate weights): fma.rn.f32x2 on horizontal output pairs, the weight
// broadcast as a (K, K) pair from a __constant__ table (uniform registers).
int sp_f2() {
    static const int v = env_int("SKC_SPARSE_F2", 1);
    return v;
}
// HWC-input layers (a chain's head): SKC_SPARSE_HWC=2 (default) runs an
// fp32 head that writes planar as an all-channel sparse stencil (the
// interleaved tile lands with coalesced cp.async; config 1's D5 head 1.60 ->
// 1.25 ms) when the layer would run a dense or sparse stencil and two CTAs
// fit per SM; 1 = per-channel CTAs with strided loads (measured slower);
// 0 = the dense / tap kernels.
int sp_hwc() {
    static const int v = env_int("SKC_SPARSE_HWC", 2);
    return v;
}
// Warps along y per CTA (SKC_SPARSE_WY, 2 or 4; 4 along x): taller tiles
// amortise the vertical halo of wide layers.
int sp_wy() {
    static const int v = [] { const int w = env_int("SKC_SPARSE_WY", 2); return w == 4 ? 4 : 2; }();
    return v;
}
// Interior fp32 planar tiles fill with one bulk (TMA) copy per row
// (SKC_SPARSE_TMA=1; measured no faster: config 1 25.6 vs 25.8 Gpix/s) or
// per-lane 16-byte cp.async (=0, default).
int sp_tma() {
    static const int v = env_int("SKC_SPARSE_TMA", 0);
    return v;
}
int sp_minb() {
    static const int v = std::max(1, env_int("SKC_SPARSE_MINB", 3));
    return v;
}
constexpr int kSpStagePitch = 132;        // staged HWC epilogue (as skc_layer.cu)
constexpr int kSpMaxFfma = 4096;          // code-size guard: FFMAs per thread (instruction cache)

struct SpPos {
    int b;
    float k;
};

struct SpPlan {
    int KR = 7, TH = 112, WY = 2;  // rows per thread, tile height, warps along y (4 along x)
    int dx_min = 0, dy_min = 0, Dx = 0, Dy = 0, npos = 0;
    std::vector<std::vector<SpPos>> rows;  // rows[a]: nonzero (b, K) of stencil row a
    int DX0 = 0, SH = 0, pitch = 0, nrows = 0, nw = 0;
    double words_per_out = 0.0;            // LDS words per output (all loads / (8 * KR))
    size_t smem = 0;
};

SpPlan make_plan(const double *taps, int S, int wy = 0, int kr = 0) {
    SpPlan p;
    p.KR = kr > 0 ? kr : sp_kr();
    p.WY = wy > 0 ? wy : sp_wy();
    p.TH = 8 * p.KR * p.WY;
    std::map<std::pair<int, int>, double> acc;  // (dy, dx) -> merged weight
    for (int i = 0; i < S; ++i) {
        const double ox = taps[3 * i], oy = taps[3 * i + 1], w = taps[3 * i + 2];
        const double fx0 = std::floor(ox), fy0 = std::floor(oy);
        const double fx = ox - fx0, fy = oy - fy0;
        const int ix = (int)fx0, iy = (int)fy0;
        acc[{iy, ix}] += w * (1.0 - fx) * (1.0 - fy);
        acc[{iy, ix + 1}] += w * fx * (1.0 - fy);
        acc[{iy + 1, ix}] += w * (1.0 - fx) * fy;
        acc[{iy + 1, ix + 1}] += w * fx * fy;
    }
    int xmin = 1 << 30, xmax = -(1 << 30), ymin = 1 << 30, ymax = -(1 << 30);
    for (const auto &kv : acc) {
        if ((float)kv.second == 0.f) continue;
        ymin = std::min(ymin, kv.first.first);
        ymax = std::max(ymax, kv.first.first);
        xmin = std::min(xmin, kv.first.second);
        xmax = std::max(xmax, kv.first.second);
    }
    if (xmin > xmax) return p;  // all-zero layer: npos = 0
    p.dx_min = xmin;
    p.dy_min = ymin;
    p.Dx = xmax - xmin + 1;
    p.Dy = ymax - ymin + 1;
    // tall footprints re-read fewer window rows per output at a larger KR
    // ((KR + Dy - 1) / KR rows per output row): SKC_SPARSE_KR_WIDE (default 5)
    // for Dy >= 24
    if (p.Dy >= 24 && kr == 0) {
        p.KR = sp_kr_wide();
        p.TH = 8 * p.KR * p.WY;
    }
    p.rows.assign(p.Dy, {});
    for (const auto &kv : acc) {
        const float k = (float)kv.second;
        if (k == 0.f) continue;
        p.rows[kv.first.first - ymin].push_back({kv.first.second - xmin, k});
        ++p.npos;
    }
    // smem geometry: column 0 <-> global tx0 + DX0 (DX0 = dx_min floored to 4)
    p.DX0 = xmin & ~3;
    p.SH = xmin - p.DX0;
    const int wmax = p.SH + p.Dx - 1 + (sp_f2() == 2 ? 8 : 7);  // last window word of a thread
    p.nw = (wmax / 4 + 1) * 4;
    int pitch = 120 + p.nw;                        // last thread's col0 = 120
    while (pitch % 8 != 4) ++pitch;
    p.pitch = pitch;
    p.nrows = p.TH + p.Dy - 1;
    p.smem = (size_t)std::max(p.nrows * p.pitch, p.TH * kSpStagePitch) * sizeof(float);
    // LDS words per output: per input row, the chunks the touching stencil rows need
    long long words = 0;
    for (int q = 0; q < p.KR + p.Dy - 1; ++q) {
        int kmin = 1 << 30, kmax = -1;
        for (int a = std::max(0, q - p.KR + 1); a <= std::min(p.Dy - 1, q); ++a)
            for (const SpPos &e : p.rows[a]) {
                kmin = std::min(kmin, p.SH + e.b);
                kmax = std::max(kmax, p.SH + e.b + 7);
            }
        if (kmax >= 0) words += 4 * (kmax / 4 - kmin / 4 + 1);
    }
    p.words_per_out = (double)words / (8.0 * p.KR);
    return p;
}

int sparse_mode() {
    static const int v = [] {
        const char *e = std::getenv("SKC_SPARSE");
        return e ? (e[0] == '0' ? 0 : (e[0] == '1' ? 1 : -1)) : -1;
    }();
    return v;
}

// Eligibility + cost model (per output and channel, in SM clocks): the tap
// kernel at KR = 7 reads S * 72 / 56 words (32 words/clk) and issues 4S FFMAs
// (128/clk), shared-memory bound; the sparse stencil issues npos FFMAs and
// reads words_per_out words.  Taken when clearly cheaper (< 0.8x).
// Footprints the dense kernels cover (D <= 9 with D^2 < 4S, skc_layer.cu
// try_stencil) run sparse only when it skips enough zeros: npos < 0.8 D^2.
// `small`: the launch fills less than two waves (config 0's 512^2 frame): a
// layer there is bound by one CTA's latency, not by throughput, and the
// generated stencil's CTA is shorter than the tap kernel's (config 0's
// 12-tap radius-16 layer: 10.0 vs 13.4 us), so wide layers skip the
// throughput comparison (SKC_SPARSE_SMALL_PREFER=0 restores it)
bool eligible(const SpPlan &p, int S, bool small = false) {
    const int mode = sparse_mode();
    if (mode == 0 || p.npos == 0) return false;
    if ((long long)p.npos * p.KR * (sp_f2() ? 5 : 8) > kSpMaxFfma) return false;
    if (p.smem > (size_t)kMaxSmem) return false;
    if (mode == 1) return true;
    const int D = dense_size_for(std::max(p.Dx, p.Dy));
    if (D != 0 && D * D < 4 * S) return p.npos < 0.8 * D * D;
    if (small && p.npos <= 160 && env_int("SKC_SPARSE_SMALL_PREFER", 1)) return true;
    const double tap = S * (7 + 1) * 9.0 / (7 * 8.0) / 32.0;  // the tap kernel at KR = 7
    const double sp = std::max(p.npos / 128.0, p.words_per_out / 32.0);
    return sp < 0.8 * tap;
}

// ------------------------------------------------------------ generator ---
const char *kSpPrelude = R"CUDA(
typedef unsigned short half_t;
__device__ __forceinline__ float h2f(unsigned h) { float f; asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"((unsigned short)h)); return f; }
__device__ __forceinline__ half_t f2h(float f) { half_t h; asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f)); return h; }
__device__ __forceinline__ float ldx(const float *p) { return __ldg(p); }
__device__ __forceinline__ float ldx(const half_t *p) { return h2f(__ldg(p)); }
__device__ __forceinline__ void stx(float *p, float v) { *p = v; }
__device__ __forceinline__ void stx(half_t *p, float v) { *p = f2h(v); }
__device__ __forceinline__ void cp4(float *dst, const float *src, int n) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp16(float *dst, const float *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
}

extern "C" __global__ void __launch_bounds__(NWARP * 32, MINB)
skc_sparse_stencil(const TI *__restrict__ in, TO *__restrict__ out, int H, int W, int C, int clamp,
                   const __grid_constant__ KWT kw) {
    extern __shared__ __align__(16) float smem[];
    const long long hw = (long long)H * W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if PDL
    // programmatic dependent launch (small launches): let the next layer's grid
    // start launching now, then wait for the previous layer's grid and its writes
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
#if ALLC
    // all channels per CTA (HWC chain head): the interleaved halo tile lands
    // with coalesced 4-byte cp.async (RS = PITCH * CC + 1 words per row: odd, so
    // the body's stride-CC window loads of the 4 x 8 lane layout are
    // conflict-free); the body then runs once per channel on that tile
    const int b = blockIdx.z;
    const int tx0 = blockIdx.x * 128, ty0 = blockIdx.y * TH;
#if !IN_F32
    {   // fp16 head: the raw interleaved halves land with 4-byte cp.async (RSH
        // halves per row, even); the body widens each window word it reads
        const half_t *frame = (const half_t *)in + (long long)b * hw * CC;
        const int gx0 = tx0 + DX0, gy0 = ty0 + DY0;
        half_t *sh = (half_t *)smem;
        for (int r = warp; r < ROWS; r += NWARP) {
            int gy = gy0 + r;
            const bool rowin = clamp || (gy >= 0 && gy < H);
            gy = min(max(gy, 0), H - 1);
            const half_t *src = frame + (long long)gy * W * CC;
            half_t *dst = sh + r * RSH;
            if (rowin && ((W * CC) & 1) == 0 && gx0 >= 0 && gx0 + PITCH <= W) {
                const float *s1 = (const float *)(src + (long long)gx0 * CC);
#pragma unroll 4
                for (int e = lane; e < PITCH * CC / 2; e += 32) cp4((float *)dst + e, s1 + e, 4);
            } else {
                for (int e = lane; e < PITCH * CC; e += 32) {
                    const int px = e / CC, ch = e - px * CC, gx = gx0 + px;
                    const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                    dst[e] = ok ? __ldg(src + (long long)min(max(gx, 0), W - 1) * CC + ch) : (half_t)0;
                }
            }
        }
        asm volatile("cp.async.wait_all;");
    }
#else
    {
        const float *frame = (const float *)in + (long long)b * hw * CC;
        const int gx0 = tx0 + DX0, gy0 = ty0 + DY0;
        for (int r = warp; r < ROWS; r += NWARP) {
            int gy = gy0 + r;
            const bool rowin = clamp || (gy >= 0 && gy < H);
            gy = min(max(gy, 0), H - 1);
            const float *src = frame + (long long)gy * W * CC;
            float *dst = smem + r * RS;
            if (rowin && gx0 >= 0 && gx0 + PITCH <= W) {
                const float *s1 = src + (long long)gx0 * CC;
#pragma unroll 4
                for (int e = lane; e < PITCH * CC; e += 32) cp4(dst + e, s1 + e, 4);
            } else {
                for (int e = lane; e < PITCH * CC; e += 32) {
                    const int px = e / CC, ch = e - px * CC, gx = gx0 + px;
                    const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                    cp4(dst + e, src + (long long)min(max(gx, 0), W - 1) * CC + ch, ok ? 4 : 0);
                }
            }
        }
        asm volatile("cp.async.wait_all;");
    }
#endif
#else
    const int b = blockIdx.z, c = blockIdx.x % C;
    const int tx0 = (blockIdx.x / C) * 128, ty0 = blockIdx.y * TH;
#endif
#if ALLC
#elif IN_HWC
    {   // channel c of the HWC halo tile: 4-byte copies at element stride C
        const TI *frame = in + (long long)b * hw * C;
        const int gx0 = tx0 + DX0, gy0 = ty0 + DY0;
        for (int r = warp; r < ROWS; r += NWARP) {
            int gy = gy0 + r;
            const bool rowin = clamp || (gy >= 0 && gy < H);
            gy = min(max(gy, 0), H - 1);
            const TI *src = frame + (long long)gy * W * C + c;
            float *dst = smem + r * PITCH;
            const bool inner = rowin && gx0 >= 0 && gx0 + PITCH <= W;
            for (int col = lane; col < PITCH; col += 32) {
                const int gx = gx0 + col;
                const bool ok = inner || clamp || (rowin && gx >= 0 && gx < W);
                const long long e = (long long)(inner ? gx : min(max(gx, 0), W - 1)) * C;
                if (IN_F32) cp4(dst + col, (const float *)src + e, ok ? 4 : 0);
                else dst[col] = ok ? ldx(src + e) : 0.f;
            }
        }
        asm volatile("cp.async.wait_all;");
    }
#else
    {   // halo tile of channel plane c: rows [ty0 + DY0, +ROWS), cols [tx0 + DX0, +PITCH)
        const TI *plane = in + ((long long)b * C + c) * hw;
        const int gx0 = tx0 + DX0, gy0 = ty0 + DY0;
        const bool interior = (W & 3) == 0 && gx0 >= 0 && gx0 + PITCH <= W && gy0 >= 0 && gy0 + ROWS <= H;
#if USE_TMA
        if (IN_F32 && interior) {
            // interior tile: one bulk (TMA) copy per row, completion counted in
            // bytes on an mbarrier -- the fill bypasses the LSU (no per-lane
            // LDGSTS, none of its shared-store wavefronts)
            __shared__ __align__(8) unsigned long long mbar;
            const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
            if (threadIdx.x == 0) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
                asm volatile("fence.mbarrier_init.release.cluster;");
            }
            __syncthreads();
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(ROWS * PITCH * 4));
            if (lane == 0) {
                const float *src = (const float *)plane + (long long)(gy0 + warp) * W + gx0;
                unsigned dst = (unsigned)__cvta_generic_to_shared(smem + warp * PITCH);
                for (int r = warp; r < ROWS; r += NWARP, src += (long long)NWARP * W, dst += NWARP * PITCH * 4)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(dst), "l"(src), "r"(PITCH * 4), "r"(mb) : "memory");
            }
            unsigned done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(mb) : "memory");
        } else
#endif
        if (IN_F32 && interior) {
            const float *src = (const float *)plane + (long long)(gy0 + warp) * W + gx0;
            float *dst = smem + warp * PITCH;
            for (int r = warp; r < ROWS; r += NWARP, src += (long long)NWARP * W, dst += NWARP * PITCH)
#pragma unroll
                for (int u = 0; u < (PITCH / 4 + 31) / 32; ++u)
                    if (lane + 32 * u < PITCH / 4) cp16(dst + 4 * (lane + 32 * u), src + 4 * (lane + 32 * u));
        } else {
            for (int r = warp; r < ROWS; r += NWARP) {
                int gy = gy0 + r;
                const bool rowin = clamp || (gy >= 0 && gy < H);
                gy = min(max(gy, 0), H - 1);
                const TI *src = plane + (long long)gy * W;
                float *dst = smem + r * PITCH;
                if (IN_F32) {
                    for (int col = lane; col < PITCH; col += 32) {
                        const int gx = gx0 + col;
                        const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                        cp4(dst + col, (const float *)src + min(max(gx, 0), W - 1), ok ? 4 : 0);
                    }
                } else if (rowin && (W & 1) == 0 && gx0 >= 0 && gx0 + PITCH <= W) {
                    const unsigned *s2 = (const unsigned *)(src + gx0);
#pragma unroll 4
                    for (int p = lane; p < PITCH / 2; p += 32) {
                        const unsigned v = __ldg(s2 + p);
                        *(float2 *)(dst + 2 * p) = make_float2(h2f(v & 0xffffu), h2f(v >> 16));
                    }
                } else {
                    for (int col = lane; col < PITCH; col += 32) {
                        const int gx = gx0 + col;
                        const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                        dst[col] = ok ? ldx(src + min(max(gx, 0), W - 1)) : 0.f;
                    }
                }
            }
        }
        asm volatile("cp.async.wait_all;");
    }
#endif
    __syncthreads();
    const int lx = lane & 3, ly = lane >> 2, wx = warp & 3, wy = warp >> 2;
    const int col0 = wx * 32 + lx * 8, row0 = wy * 8 * KR + ly * KR;
#if ALLC
#pragma unroll 1
    for (int c = 0; c < CC; ++c) {
#if IN_F32
    const float *base = smem + row0 * RS + col0 * CC + c;
#else
    const half_t *base = (const half_t *)smem + row0 * RSH + col0 * CC + c;
#endif
#else
    const float *base = smem + row0 * PITCH + col0;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(base);
#endif
)CUDA";

const char *kSpPlanarEpilogue = R"CUDA(
    TO *o = out + ((long long)b * C + c) * hw;
    const int gx = tx0 + col0;
#pragma unroll
    for (int i = 0; i < KR; ++i) {
        const int gy = ty0 + row0 + i;
        if (gy >= H) continue;
        TO *p = o + (long long)gy * W + gx;
        if (OUT_F32) {
            if (gx + 7 < W && (W & 3) == 0) {
                ((float4 *)p)[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                ((float4 *)p)[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
                continue;
            }
        } else if (gx + 7 < W && (W & 7) == 0) {
            uint4 t;
            t.x = (unsigned)f2h(acc[i][0]) | ((unsigned)f2h(acc[i][1]) << 16);
            t.y = (unsigned)f2h(acc[i][2]) | ((unsigned)f2h(acc[i][3]) << 16);
            t.z = (unsigned)f2h(acc[i][4]) | ((unsigned)f2h(acc[i][5]) << 16);
            t.w = (unsigned)f2h(acc[i][6]) | ((unsigned)f2h(acc[i][7]) << 16);
            *(uint4 *)p = t;
            continue;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (gx + j < W) stx(p + j, acc[i][j]);
    }
)CUDA";

const char *kSpHwcEpilogue = R"CUDA(
    __syncthreads();  // every warp is done reading the input tile
#pragma unroll
    for (int i = 0; i < KR; ++i) {
        float4 *d = (float4 *)(smem + (row0 + i) * 132 + col0);
        d[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        d[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
    __syncthreads();
    const int nx = min(128, W - tx0), nr = min(TH, H - ty0);
    // lane x of row r writes pixel (ty0 + r, tx0 + x + 32 u): pointers stepped
    // per row (no per-element index arithmetic), full-width tiles unguarded
    const int s32 = 32 * C;
    const long long rstep = (long long)W * C * NWARP;
    TO *dst = out + (((long long)b * H + ty0 + warp) * W + tx0 + lane) * C + c;
    const float *srow = smem + warp * 132 + lane;
    if (nx == 128) {
#pragma unroll 2
        for (int r = warp; r < nr; r += NWARP, dst += rstep, srow += NWARP * 132) {
            const float v0 = srow[0], v1 = srow[32], v2 = srow[64], v3 = srow[96];
            stx(dst, v0);
            stx(dst + s32, v1);
            stx(dst + 2 * s32, v2);
            stx(dst + 3 * s32, v3);
        }
    } else {
        for (int r = warp; r < nr; r += NWARP, dst += rstep, srow += NWARP * 132) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (lane + 32 * u < nx) stx(dst + u * s32, srow[32 * u]);
        }
    }
)CUDA";


// The default HWC epilogue: per-element index arithmetic and guards.  The
// pointer-stepped form above (SKC_SPARSE_EPI=1) has fewer instructions per
// row but measured slower on config 1's 116-position KR 5 layer (3.36 vs
// 3.17 ms; its unrolled loads lengthen the tail every CTA serialises on).
const char *kSpHwcEpilogueIdx = R"CUDA(
    __syncthreads();  // every warp is done reading the input tile
#pragma unroll
    for (int i = 0; i < KR; ++i) {
        float4 *d = (float4 *)(smem + (row0 + i) * 132 + col0);
        d[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        d[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
    __syncthreads();
    const int nx = min(128, W - tx0), nr = min(TH, H - ty0);
    for (int r = warp; r < nr; r += NWARP) {
        TO *dst = out + (((long long)b * H + ty0 + r) * W + tx0) * C + c;
        const float *srow = smem + r * 132;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int x = lane + 32 * u;
            if (x < nx) stx(dst + (long long)x * C, srow[x]);
        }
    }
)CUDA";

int sp_epi() {
    static const int v = env_int("SKC_SPARSE_EPI", 0);
    return v;
}

// The kernel parameter the generated body reads: (K, K) per position, in
// the body's order (stencil row a, then position within the row).
std::vector<float> kw_table(const SpPlan &p) {
    std::vector<float> t;
    t.reserve(2 * std::max(1, p.npos));
    for (int a = 0; a < p.Dy; ++a)
        for (const SpPos &e : p.rows[a]) {
            t.push_back(e.k);
            t.push_back(e.k);
        }
    if (t.empty()) t.assign(2, 0.f);
    return t;
}

std::string generate(const SpPlan &p, bool in_f32, bool out_f32, bool out_pl, bool in_hwc = false, int allc = 0,
                     bool pdl = false) {
    std::ostringstream s;
    s << "#define PDL " << (pdl ? 1 : 0) << "\n";
    s << "#define ALLC " << (allc ? 1 : 0) << "\n#define CC " << std::max(1, allc) << "\n#define RS "
      << p.pitch * std::max(1, allc) + 1 << "\n#define RSH " << p.pitch * std::max(1, allc) + 2 << "\n";
    s << "// generated by libskc (skc_sparse.cu): " << p.npos << " positions, footprint " << p.Dx << " x " << p.Dy
      << "\n";
    s << "#define TI " << (in_f32 ? "float" : "half_t") << "\n#define TO " << (out_f32 ? "float" : "half_t") << "\n";
    s << "#define IN_F32 " << (in_f32 ? 1 : 0) << "\n#define OUT_F32 " << (out_f32 ? 1 : 0) << "\n#define IN_HWC "
      << (in_hwc ? 1 : 0) << "\n";
    // resident CTAs per SM: 3 at KR = 3 (<= 85 registers), 2 for all-channel heads
    // and KR >= 5 bodies (config 1's tall layer: 3.15 vs 3.23 ms at KR 5 / 2 CTAs),
    // and 4 for small, narrow KR = 3 bodies (64 registers: config 1's 58-position
    // 9 x 9 layer 1.58 -> 1.47 ms; 5 CTAs spill)
    int minb = (allc || p.KR >= 5) ? std::min(2, sp_minb()) : sp_minb();
    if (!allc && (sp_f2() == 1 || sp_f2() == 3) && p.KR < 5 && p.npos <= 64 && p.nw <= 20) minb = env_int("SKC_SPARSE_MINB_SMALL", 4);
    // one warp row (128 threads, half-height tiles: small images): twice the
    // CTAs at the same registers per thread
    if (p.WY == 1 && sp_wy() == 2) minb *= 2;
    s << "#define MINB " << minb << "\n#define F2MODE " << sp_f2() << "\n";
    s << "#define USE_TMA " << sp_tma() << "\n";
    s << "#define NWARP " << 4 * p.WY << "\n";
    s << "#define KR " << p.KR << "\n#define TH " << p.TH << "\n#define PITCH " << p.pitch << "\n#define ROWS "
      << p.nrows << "\n#define DX0 " << p.DX0 << "\n#define DY0 " << p.dy_min << "\n#define NW " << p.nw << "\n";
    const bool f2 = sp_f2() != 0;
    // the merged weights arrive as a kernel parameter (constant bank 0), one
    // (K, K) pair per position in the body's order: the source -- and so the
    // compiled kernel -- depends only on the position pattern, and a layer
    // with new weights at the same positions reuses it
    s << "#define NPOS " << std::max(1, p.npos) << "\nstruct KWT { float2 k[NPOS]; };\n";
    if (f2) {
        // register-only packing (no address-taken temporaries: thousands of
        // inlined calls otherwise cost the front end tens of seconds)
        s << "__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {\n"
             "    float2 d;\n"
             "    asm(\"{ .reg .b64 ra, rb, rc, rd; mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5}; mov.b64 rc, {%6, %7};\"\n"
             "        \" fma.rn.f32x2 rd, ra, rb, rc; mov.b64 {%0, %1}, rd; }\"\n"
             "        : \"=f\"(d.x), \"=f\"(d.y) : \"f\"(a.x), \"f\"(a.y), \"f\"(b.x), \"f\"(b.y), \"f\"(c.x), \"f\"(c.y));\n"
             "    return d;\n}\n";
    }
    s << kSpPrelude;
    // one named value per position, read once from the parameter struct: the
    // body indexing the struct directly (1000+ reads) made NVRTC's optimizer
    // take minutes on the widest layers; ptxas still folds these into
    // constant-bank operands
    for (int q = 0; q < std::max(1, p.npos); ++q) s << "    const float2 kw" << q << " = kw.k[" << q << "];\n";
    std::vector<int> first(p.Dy + 1, 0);  // index of stencil row a's first position in KW
    for (int a = 0; a < p.Dy; ++a) first[a + 1] = first[a] + (int)p.rows[a].size();
    if (f2) {
        // Window words as aligned pairs wp<m> = (w[2m], w[2m+1]).  A position at
        // window column c0 feeds output j from w[c0 + j]: for even c0 the output
        // pairs (2m, 2m+1) meet aligned window pairs; for odd c0 the pairs
        // (2m+1, 2m+2) do, with outputs 0 and 7 as scalar FFMAs -- two
        // accumulator sets (e: even-paired, o: odd-paired + 2 scalars), summed
        // in the epilogue.  No register moves to re-pair the window.
        s << "    float2";
        for (int i = 0; i < p.KR; ++i)
            for (int j = 0; j < 4; ++j) s << (i || j ? ", " : " ") << "e" << i << "_" << j << " = make_float2(0.f, 0.f)";
        const bool xchg = sp_f2() == 2;  // odd positions: 4 pairs (1,2)..(7,8), output 8 to the right neighbour
        const bool pair_ends = sp_f2() == 3;  // odd positions: outputs 0 and 7 as one FFMA2
        for (int i = 0; i < p.KR; ++i)
            for (int j = 0; j < (xchg ? 4 : 3); ++j) s << ", o" << i << "_" << j << " = make_float2(0.f, 0.f)";
        s << ";\n    float";
        for (int i = 0; i < p.KR; ++i) s << (i ? ", " : " ") << "s" << i << "_0 = 0.f, s" << i << "_7 = 0.f";
        if (pair_ends) {
            s << ";\n    float2";
            for (int i = 0; i < p.KR; ++i) s << (i ? ", " : " ") << "z" << i << " = make_float2(0.f, 0.f)";
        }
        s << ";\n    float2";
        for (int m = 0; m < p.nw / 2; ++m) s << (m ? ", " : " ") << "wp" << m;
        s << ";\n";
        for (int q = 0; q < p.KR + p.Dy - 1; ++q) {
            const int a_lo = std::max(0, q - p.KR + 1), a_hi = std::min(p.Dy - 1, q);
            int kmin = 1 << 30, kmax = -1;
            for (int a = a_lo; a <= a_hi; ++a)
                for (const SpPos &e : p.rows[a]) {
                    kmin = std::min(kmin, p.SH + e.b);
                    kmax = std::max(kmax, p.SH + e.b + (xchg && (p.SH + e.b) % 2 ? 8 : 7));
                }
            if (kmax < 0) continue;
            if (allc && in_f32) {
                s << "    {\n        const float *rp = base + " << q << " * RS;\n";
                for (int m = kmin / 2; m <= kmax / 2; ++m)
                    s << "        wp" << m << " = make_float2(rp[" << 2 * m << " * CC], rp[" << 2 * m + 1 << " * CC]);\n";
            } else if (allc) {
                s << "    {\n        const half_t *rp = base + " << q << " * RSH;\n";
                for (int m = kmin / 2; m <= kmax / 2; ++m)
                    s << "        wp" << m << " = make_float2(h2f(rp[" << 2 * m << " * CC]), h2f(rp[" << 2 * m + 1
                      << " * CC]));\n";
            } else {
                // full-width LDS.128 through inline PTX: a chunk whose words are only
                // partly used would otherwise be narrowed to LDS.32/64, which the 4 x 8
                // lane layout turns into 4-way bank conflicts (ncu source page, config 1)
                s << "    {\n";
                for (int ch = kmin / 4; ch <= kmax / 4; ++ch)
                    s << "        asm(\"ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4+" << 4 * (q * p.pitch + 4 * ch)
                      << "];\" : \"=f\"(wp" << 2 * ch << ".x), \"=f\"(wp" << 2 * ch << ".y), \"=f\"(wp" << 2 * ch + 1
                      << ".x), \"=f\"(wp" << 2 * ch + 1 << ".y) : \"r\"(sbase));\n";
            }
            std::ostringstream first_col;  // exchange mode: output 0 of the tile's first column block
            for (int a = a_lo; a <= a_hi; ++a) {
                const int i = q - a;
                for (size_t e = 0; e < p.rows[a].size(); ++e) {
                    const int c0 = p.SH + p.rows[a][e].b;
                    const std::string kw = "kw" + std::to_string(first[a] + (int)e);
                    if (c0 % 2 == 0) {
                        for (int j = 0; j < 4; ++j)
                            s << "        e" << i << "_" << j << " = ffma2(" << kw << ", wp" << c0 / 2 + j << ", e" << i << "_"
                              << j << ");\n";
                    } else if (xchg) {
                        first_col << "            s" << i << "_0 = fmaf(" << kw << ".x, wp" << (c0 - 1) / 2 << ".y, s" << i
                                  << "_0);\n";
                        for (int j = 0; j < 4; ++j)
                            s << "        o" << i << "_" << j << " = ffma2(" << kw << ", wp" << (c0 + 1) / 2 + j << ", o" << i
                              << "_" << j << ");\n";
                    } else if (pair_ends) {
                        // outputs 0 and 7 as one FFMA2 on the accumulator pair
                        // z<i> = (out 0, out 7) with the operand pair (w[c0], w[c0+7])
                        s << "        z" << i << " = ffma2(" << kw << ", make_float2(wp" << (c0 - 1) / 2 << ".y, wp"
                          << (c0 + 7) / 2 << ".x), z" << i << ");\n";
                        for (int j = 0; j < 3; ++j)
                            s << "        o" << i << "_" << j << " = ffma2(" << kw << ", wp" << (c0 + 1) / 2 + j << ", o" << i
                              << "_" << j << ");\n";
                    } else {
                        s << "        s" << i << "_0 = fmaf(" << kw << ".x, wp" << (c0 - 1) / 2 << ".y, s" << i << "_0);\n";
                        for (int j = 0; j < 3; ++j)
                            s << "        o" << i << "_" << j << " = ffma2(" << kw << ", wp" << (c0 + 1) / 2 + j << ", o" << i
                              << "_" << j << ");\n";
                        s << "        s" << i << "_7 = fmaf(" << kw << ".x, wp" << (c0 + 7) / 2 << ".x, s" << i << "_7);\n";
                    }
                }
            }
            if (!first_col.str().empty()) s << "        if (wx == 0) {\n" << first_col.str() << "        }\n";
            s << "    }\n";
        }
        s << "    float acc[KR][8];\n";
        if (xchg) {
            // output 8 of each column block is output 0 of the block to its right:
            // exchange through the dead tile (16 column blocks per tile row); the
            // tile's first block keeps its own scalar sums s<i>_0
            s << "    __syncthreads();\n";
            for (int i = 0; i < p.KR; ++i)
                s << "    smem[(row0 + " << i << ") * 16 + (col0 >> 3)] = o" << i << "_3.y;\n";
            s << "    __syncthreads();\n";
            for (int i = 0; i < p.KR; ++i)
                s << "    const float x" << i << " = col0 > 0 ? smem[(row0 + " << i << ") * 16 + (col0 >> 3) - 1] : s" << i
                  << "_0;\n";
        }
        for (int i = 0; i < p.KR; ++i) {
            for (int j = 0; j < 4; ++j)
                s << "    acc[" << i << "][" << 2 * j << "] = e" << i << "_" << j << ".x; acc[" << i << "][" << 2 * j + 1
                  << "] = e" << i << "_" << j << ".y;\n";
            if (xchg) {
                s << "    acc[" << i << "][0] += x" << i << "; acc[" << i << "][7] += o" << i << "_3.x;\n";
            } else if (pair_ends) {
                s << "    acc[" << i << "][0] += z" << i << ".x; acc[" << i << "][7] += z" << i << ".y;\n";
            } else {
                s << "    acc[" << i << "][0] += s" << i << "_0; acc[" << i << "][7] += s" << i << "_7;\n";
            }
            for (int j = 0; j < 3; ++j)
                s << "    acc[" << i << "][" << 2 * j + 1 << "] += o" << i << "_" << j << ".x; acc[" << i << "][" << 2 * j + 2
                  << "] += o" << i << "_" << j << ".y;\n";
        }
        s << (out_pl ? kSpPlanarEpilogue : sp_epi() ? kSpHwcEpilogue : kSpHwcEpilogueIdx);
        s << (allc ? "    }\n}\n" : "}\n");
        return s.str();
    }
    // scalar accumulators a<i>_<j> and window words w<k> (not arrays: the front
    // end's array scalarisation is ~10x slower on bodies of this size)
    s << "    float";
    for (int i = 0; i < p.KR; ++i)
        for (int j = 0; j < 8; ++j) s << (i || j ? ", " : " ") << "a" << i << "_" << j << " = 0.f";
    s << ";\n    float";
    for (int k = 0; k < p.nw; ++k) s << (k ? ", " : " ") << "w" << k;
    s << ";\n";
    const int sync = sp_sync();
    for (int q = 0; q < p.KR + p.Dy - 1; ++q) {
        if (sync > 0 && q > 0 && q % sync == 0) s << "    __syncthreads();\n";
        const int a_lo = std::max(0, q - p.KR + 1), a_hi = std::min(p.Dy - 1, q);
        int kmin = 1 << 30, kmax = -1;
        for (int a = a_lo; a <= a_hi; ++a)
            for (const SpPos &e : p.rows[a]) {
                kmin = std::min(kmin, p.SH + e.b);
                kmax = std::max(kmax, p.SH + e.b + 7);
            }
        if (kmax < 0) continue;
        s << "    {\n        const float4 *rp = (const float4 *)(base + " << q << " * PITCH);\n";
        for (int ch = kmin / 4; ch <= kmax / 4; ++ch)
            s << "        { const float4 t = rp[" << ch << "]; w" << 4 * ch << " = t.x; w" << 4 * ch + 1
              << " = t.y; w" << 4 * ch + 2 << " = t.z; w" << 4 * ch + 3 << " = t.w; }\n";
        for (int a = a_lo; a <= a_hi; ++a) {
            const int i = q - a;
            for (size_t ei = 0; ei < p.rows[a].size(); ++ei) {
                const SpPos &e = p.rows[a][ei];
                const std::string k = "kw" + std::to_string(first[a] + (int)ei) + ".x";
                for (int j = 0; j < 8; ++j)
                    s << "        a" << i << "_" << j << " = fmaf(" << k << ", w" << p.SH + e.b + j << ", a" << i << "_" << j
                      << ");\n";
            }
        }
        s << "    }\n";
    }
    s << "    float acc[KR][8];\n";
 for (int i = 0; i < p.KR; ++i)
        for (int j = 0; j < 8; ++j) s << "    acc[" << i << "][" << j << "] = a" << i << "_" << j << ";\n";
    s << (out_pl ? kSpPlanarEpilogue : sp_epi() ? kSpHwcEpilogue : kSpHwcEpilogueIdx);
    s << (allc ? "    }\n}\n" : "}\n");
    return s.str();
}

// ------------------------------------------------- fused head pair ---
// Layers 0 and 1 of a chain in one launch (north_star: consecutive layers
// fused inside one CTA where the accumulated halo fits in shared memory).
// A CTA owns one channel of a 128-column strip over a chunk of rows and
// streams down it in blocks of TH output rows:
//   IN  (TH + Dy0 - 1) x P1 : the channel's input rows (4-byte cp.async at
//       element stride C from the HWC frame, the boundary rule applied);
//   MID (TH + Dy1 - 1) x MP : layer 0's output, the rows layer 1 reads.
// Per block: layer 0 computes the TH new MID rows (8-row x 32-column warp
// jobs, one row and 8 columns per lane) and re-applies the boundary rule
// outside the image (zero: 0; clamp: the clamped in-image value -- what the
// reference's materialised intermediate holds); the last Dy0 - 1 IN rows and
// Dy1 - 1 MID rows move to the top of their buffers (register round trip),
// the next block's TH input rows are prefetched behind layer 1, and layer 1
// runs from MID into registers and the planar output.  Only the horizontal
// halo of layer 0 is recomputed (the vertical one streams), and the
// intermediate never reaches HBM: config 1 drops one 5.2 GB round trip.
struct PairPlan {
    SpPlan p1, p2;     // layer 0 (KR 1: one row per lane job), layer 1 (KR, TH, WY)
    int MP = 0, P1 = 0, NCJ = 0, RIN = 0, RMID = 0, RJ0 = 0, minb = 2;
    size_t smem = 0;
    bool ok = false;
};

int pair_kr() {
    static const int v = [] { const int k = env_int("SKC_PAIR_KR", 3); return (k == 3 || k == 5) ? k : 3; }();
    return v;
}
// Opt-in (SKC_PAIR=1, read per call): on config 1 the pair measured 3.35 ms
// against 2.74 ms for the two unfused launches -- the per-channel fill at
// element stride C (4-byte LDGSTS) took a quarter of the L1 wavefronts
// (profiles/r02_c1_pair.md), and an all-channel fill does not leave room
// for more than one CTA per SM.
int pair_mode() { return env_int("SKC_PAIR", 0); }

PairPlan make_pair_plan(const double *t1, int S1, const double *t2, int S2, int wy = 2) {
    PairPlan q;
    q.p1 = make_plan(t1, S1, wy, 1);
    q.p2 = make_plan(t2, S2, wy, pair_kr());
    const SpPlan &a = q.p1, &b = q.p2;
    if (a.npos == 0 || b.npos == 0) return q;
    const int TH = b.TH;
    q.MP = b.pitch;
    q.NCJ = (b.pitch + 31) / 32;
    // input plane: the last lane job's window (col0 = NCJ * 32 - 8) ends at
    // word NCJ * 32 - 8 + a.nw; pitch = 4 mod 8 keeps LDS.128 conflict-free
    int p1 = q.NCJ * 32 - 8 + a.nw;
    while (p1 % 8 != 4) ++p1;
    q.P1 = p1;
    q.RIN = TH + a.Dy - 1;
    q.RMID = TH + b.Dy - 1;
    q.RJ0 = (TH - (b.Dy - 1)) / 8;   // the prologue block computes only the rows it carries
    q.smem = (size_t)(q.RIN * q.P1 + q.RMID * q.MP) * sizeof(float);
    // layer 1 must reach both ways in x and y (the clamp rule's source rows
    // and columns are then inside the buffers); two CTAs per SM at least
    q.ok = b.dy_min < 0 && b.dy_min + b.Dy - 1 > 0 && b.DX0 + b.SH < 0 && b.DX0 + b.SH + b.Dx - 1 > 0 &&
           b.Dy - 1 <= TH && 2 * (q.smem + 1024) <= (size_t)kMaxSmem + 1024 &&
           (long long)a.npos * 5 <= kSpMaxFfma && (long long)b.npos * b.KR * 5 <= kSpMaxFfma;
    // resident CTAs per SM: as many as shared memory allows, at most 3 (KR 3:
    // 80 registers); KR 5 bodies keep 2
    q.minb = std::max(1, std::min(b.KR >= 5 ? 2 : 3, (int)((size_t)(kMaxSmem + 1024) / (q.smem + 1024))));
    if (const int m = env_int("SKC_PAIR_MINB", 0)) q.minb = m;
    return q;
}

// Packed-FP32 body of one plan reading a planar shared tile through LDS.128
// at byte address `sb` (row pitch `pitch` words), accumulating kr x 8 outputs
// into the float array `acc` (declared by the caller); weights kw<kwbase + n>.
void emit_f2_body(std::ostringstream &s, const SpPlan &p, int kr, int kwbase, const std::string &sb, int pitch,
                  const std::string &acc) {
    std::vector<int> first(p.Dy + 1, 0);
    for (int a = 0; a < p.Dy; ++a) first[a + 1] = first[a] + (int)p.rows[a].size();
    s << "    {\n    float2";
    for (int i = 0; i < kr; ++i)
        for (int j = 0; j < 4; ++j) s << (i || j ? ", " : " ") << "e" << i << "_" << j << " = make_float2(0.f, 0.f)";
    for (int i = 0; i < kr; ++i)
        for (int j = 0; j < 3; ++j) s << ", o" << i << "_" << j << " = make_float2(0.f, 0.f)";
    s << ";\n    float";
    for (int i = 0; i < kr; ++i) s << (i ? ", " : " ") << "s" << i << "_0 = 0.f, s" << i << "_7 = 0.f";
    s << ";\n    float2";
    for (int m = 0; m < p.nw / 2; ++m) s << (m ? ", " : " ") << "wp" << m;
    s << ";\n";
    for (int q = 0; q < kr + p.Dy - 1; ++q) {
        const int a_lo = std::max(0, q - kr + 1), a_hi = std::min(p.Dy - 1, q);
        int kmin = 1 << 30, kmax = -1;
        for (int a = a_lo; a <= a_hi; ++a)
            for (const SpPos &e : p.rows[a]) {
                kmin = std::min(kmin, p.SH + e.b);
                kmax = std::max(kmax, p.SH + e.b + 7);
            }
        if (kmax < 0) continue;
        s << "    {\n";
        // asm volatile: the loads depend on shared memory the CTA rewrites
        // between passes (a plain asm is a pure function of its address
        // operand to the compiler, which then hoists it out of the channel loop)
        for (int ch = kmin / 4; ch <= kmax / 4; ++ch)
            s << "        asm volatile(\"ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4+" << 4 * (q * pitch + 4 * ch)
              << "];\" : \"=f\"(wp" << 2 * ch << ".x), \"=f\"(wp" << 2 * ch << ".y), \"=f\"(wp" << 2 * ch + 1
              << ".x), \"=f\"(wp" << 2 * ch + 1 << ".y) : \"r\"(" << sb << "));\n";
        for (int a = a_lo; a <= a_hi; ++a) {
            const int i = q - a;
            for (size_t e = 0; e < p.rows[a].size(); ++e) {
                const int c0 = p.SH + p.rows[a][e].b;
                const std::string kw = "kw" + std::to_string(kwbase + first[a] + (int)e);
                if (c0 % 2 == 0) {
                    for (int j = 0; j < 4; ++j)
                        s << "        e" << i << "_" << j << " = ffma2(" << kw << ", wp" << c0 / 2 + j << ", e" << i << "_"
                          << j << ");\n";
                } else {
                    s << "        s" << i << "_0 = fmaf(" << kw << ".x, wp" << (c0 - 1) / 2 << ".y, s" << i << "_0);\n";
                    for (int j = 0; j < 3; ++j)
                        s << "        o" << i << "_" << j << " = ffma2(" << kw << ", wp" << (c0 + 1) / 2 + j << ", o" << i
                          << "_" << j << ");\n";
                    s << "        s" << i << "_7 = fmaf(" << kw << ".x, wp" << (c0 + 7) / 2 << ".x, s" << i << "_7);\n";
                }
            }
        }
        s << "    }\n";
    }
    for (int i = 0; i < kr; ++i) {
        for (int j = 0; j < 4; ++j)
            s << "    " << acc << "[" << i << "][" << 2 * j << "] = e" << i << "_" << j << ".x; " << acc << "[" << i << "]["
              << 2 * j + 1 << "] = e" << i << "_" << j << ".y;\n";
        s << "    " << acc << "[" << i << "][0] += s" << i << "_0; " << acc << "[" << i << "][7] += s" << i << "_7;\n";
        for (int j = 0; j < 3; ++j)
            s << "    " << acc << "[" << i << "][" << 2 * j + 1 << "] += o" << i << "_" << j << ".x; " << acc << "[" << i
              << "][" << 2 * j + 2 << "] += o" << i << "_" << j << ".y;\n";
    }
    s << "    }\n";
}

const char *kPairHead = R"CUDA(struct KWT { float2 k[NPOS]; };
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{ .reg .b64 ra, rb, rc, rd; mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5}; mov.b64 rc, {%6, %7};"
        " fma.rn.f32x2 rd, ra, rb, rc; mov.b64 {%0, %1}, rd; }"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ void cp4(float *dst, const float *src, int n) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
// IN rows [r_lo, r_hi) <- channel c of the HWC frame, global rows gyb + r,
// columns gx0 + [0, P1), the boundary rule applied
__device__ __forceinline__ void fill_rows(float *inb, const float *frame, int c, int C, int H, int W, int clamp,
                                          int gx0, int gyb, int r_lo, int r_hi, int warp, int lane) {
    const bool colin = gx0 >= 0 && gx0 + P1 <= W;
    for (int r = r_lo + warp; r < r_hi; r += NWARP) {
        int gy = gyb + r;
        const bool rowin = clamp || (gy >= 0 && gy < H);
        gy = min(max(gy, 0), H - 1);
        const float *src = frame + (long long)gy * W * C + c;
        float *dst = inb + r * P1;
        if (rowin && colin) {
            const float *sp = src + (long long)(gx0 + lane) * C;
#pragma unroll 2
            for (int col = lane; col < P1; col += 32, sp += 32 * C) cp4(dst + col, sp, 4);
        } else {
            for (int col = lane; col < P1; col += 32) {
                const int gx = gx0 + col;
                const bool ok = clamp || (rowin && gx >= 0 && gx < W);
                cp4(dst + col, src + (long long)min(max(gx, 0), W - 1) * C, ok ? 4 : 0);
            }
        }
    }
}

extern "C" __global__ void __launch_bounds__(NWARP * 32, MINB)
skc_sparse_pair(const float *__restrict__ in, float *__restrict__ out, int H, int W, int C, int clamp, int CH,
                const __grid_constant__ KWT kw) {
    extern __shared__ __align__(16) float smem[];
    float *inb = smem;                  // RIN x P1: layer 0's input rows (channel c)
    float *mid = smem + RIN * P1;       // RMID x MP: layer 0's output = layer 1's input rows
    const long long hw = (long long)H * W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x % C, tx0 = (blockIdx.x / C) * 128, b = blockIdx.z;
    const int y0 = blockIdx.y * CH, y1 = min(H, y0 + CH), nblk = (y1 - y0 + TH - 1) / TH;
    const float *frame = in + (long long)b * hw * C;
    float *o = out + ((long long)b * C + c) * hw;
    const int lx = lane & 3, ly = lane >> 2, wx = warp & 3, wy = warp >> 2;
    const int col0 = wx * 32 + lx * 8, row0 = wy * 8 * KR + ly * KR;
    const int mx0 = tx0 + DX0_2;                        // global column of MID column 0
    const int gx0 = mx0 + DX0_1;                        // global column of IN column 0
    const bool xedge = mx0 < 0 || mx0 + MP > W;
    const unsigned sbin = (unsigned)__cvta_generic_to_shared(inb), sbmid = (unsigned)__cvta_generic_to_shared(mid);
)CUDA";

// block k covers output rows [Y, Y + TH), Y = y0 + k * TH; MID row j <-> global
// Y + DY0_2 + j; IN row i <-> global Y + DY0_2 + DY1M + DY0_1 + i (DY1M = Dy1 - 1)
const char *kPairLoop = R"CUDA(    fill_rows(inb, frame, c, C, H, W, clamp, gx0, y0 - TH + DY0_2 + DY1M + DY0_1, 0, RIN, warp, lane);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#pragma unroll 1
    for (int k = -1; k < nblk; ++k) {
        const int Y = y0 + k * TH;
        // layer 0: the TH new MID rows [DY1M, DY1M + TH) (the prologue block only those it carries)
#pragma unroll 1
        for (int job = warp + (k < 0 ? RJ0 * NCJ : 0); job < (TH / 8) * NCJ; job += NWARP) {
            const int rj = job / NCJ, cj = job - rj * NCJ;
            const int r0 = rj * 8 + ly, c0 = cj * 32 + lx * 8;
            const unsigned sb1 = sbin + 4u * (unsigned)(r0 * P1 + c0);
            float acc1[1][8];
)CUDA";

const char *kPairMid = R"CUDA(            float *d = mid + (DY1M + r0) * MP + c0;
            if (c0 < MP) *(float4 *)d = make_float4(acc1[0][0], acc1[0][1], acc1[0][2], acc1[0][3]);
            if (c0 + 4 < MP) *(float4 *)(d + 4) = make_float4(acc1[0][4], acc1[0][5], acc1[0][6], acc1[0][7]);
        }
        __syncthreads();
        const int gm0 = Y + DY0_2 + DY1M;   // global row of new MID row 0
        if (xedge || gm0 < 0 || gm0 + TH > H) {
            // outside the image the intermediate is the boundary rule's value
            const int r_lo = k < 0 ? RJ0 * 8 : 0;
            for (int e = r_lo * MP + threadIdx.x; e < TH * MP; e += NWARP * 32) {
                const int r = e / MP, m = e - r * MP;
                const int gy = gm0 + r, gx = mx0 + m;
                if (gy >= 0 && gy < H && gx >= 0 && gx < W) continue;
                float v = 0.f;
                if (clamp) v = mid[(min(max(gy, 0), H - 1) - Y - DY0_2) * MP + min(max(gx, 0), W - 1) - mx0];
                mid[(DY1M + r) * MP + m] = v;
            }
            __syncthreads();
        }
        // carries: IN rows [TH, TH + DY0M) and MID rows [TH, TH + DY1M) move to the top
        float cin[CIN], cmid[CMID];
#pragma unroll
        for (int i = 0; i < CIN; ++i) {
            const int e = threadIdx.x + i * NWARP * 32;
            if (e < DY0M * P1) cin[i] = inb[TH * P1 + e];
        }
#pragma unroll
        for (int i = 0; i < CMID; ++i) {
            const int e = threadIdx.x + i * NWARP * 32;
            if (e < DY1M * MP) cmid[i] = mid[TH * MP + e];
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < CIN; ++i) {
            const int e = threadIdx.x + i * NWARP * 32;
            if (e < DY0M * P1) inb[e] = cin[i];
        }
        if (k + 1 < nblk)
            fill_rows(inb, frame, c, C, H, W, clamp, gx0, Y + TH + DY0_2 + DY1M + DY0_1, DY0M, RIN, warp, lane);
        if (k >= 0) {
            const unsigned sbase = sbmid + 4u * (unsigned)(row0 * MP + col0);
            float acc[KR][8];
)CUDA";

const char *kPairTail = R"CUDA(            const int gx = tx0 + col0;
#pragma unroll
            for (int i = 0; i < KR; ++i) {
                const int gy = Y + row0 + i;
                if (gy >= y1) continue;
                float *p = o + (long long)gy * W + gx;
                if (gx + 7 < W && (W & 3) == 0) {
                    ((float4 *)p)[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                    ((float4 *)p)[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
                    continue;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (gx + j < W) p[j] = acc[i][j];
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < CMID; ++i) {
            const int e = threadIdx.x + i * NWARP * 32;
            if (e < DY1M * MP) mid[e] = cmid[i];
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
}
)CUDA";

std::string generate_pair(const PairPlan &q) {
    const SpPlan &a = q.p1, &b = q.p2;
    const int nt = 128 * b.WY;
    std::ostringstream s;
    s << "// generated by libskc (skc_sparse.cu): fused head pair, " << a.npos << " + " << b.npos << " positions\n";
    s << "#define NWARP " << 4 * b.WY << "\n#define KR " << b.KR << "\n#define TH " << b.TH << "\n#define MP " << q.MP
      << "\n#define P1 " << q.P1 << "\n#define RIN " << q.RIN << "\n#define RMID " << q.RMID << "\n#define DX0_2 "
      << b.DX0 << "\n#define DY0_2 " << b.dy_min << "\n#define DX0_1 " << a.DX0 << "\n#define DY0_1 " << a.dy_min
      << "\n#define DY0M " << a.Dy - 1 << "\n#define DY1M " << b.Dy - 1 << "\n#define NCJ " << q.NCJ
      << "\n#define RJ0 " << q.RJ0 << "\n#define CIN " << std::max(1, ((a.Dy - 1) * q.P1 + nt - 1) / nt)
      << "\n#define CMID " << std::max(1, ((b.Dy - 1) * q.MP + nt - 1) / nt) << "\n#define NPOS " << a.npos + b.npos
      << "\n#define MINB " << q.minb << "\n";
    s << kPairHead;
    for (int n = 0; n < a.npos + b.npos; ++n) s << "    const float2 kw" << n << " = kw.k[" << n << "];\n";
    s << kPairLoop;
    emit_f2_body(s, a, 1, 0, "sb1", q.P1, "acc1");
    s << kPairMid;
    emit_f2_body(s, b, b.KR, a.npos, "sbase", q.MP, "acc");
    s << kPairTail;
    return s.str();
}

std::vector<float> pair_kw_table(const PairPlan &q) {
    std::vector<float> t = kw_table(q.p1), t2 = kw_table(q.p2);
    t.insert(t.end(), t2.begin(), t2.end());
    return t;
}

// ---------------------------------------------------------------- NVRTC ---
struct Nvrtc {
    bool ok = false;
    std::string why;
    nvrtcResult (*create)(nvrtcProgram *, const char *, const char *, int, const char *const *,
                          const char *const *) = nullptr;
    nvrtcResult (*compile)(nvrtcProgram, int, const char *const *) = nullptr;
    nvrtcResult (*log_size)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*get_log)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*cubin_size)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*get_cubin)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*destroy)(nvrtcProgram *) = nullptr;
    nvrtcResult (*version)(int *, int *) = nullptr;
};

Nvrtc &nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        void *h = nullptr;
        for (const char *name : {"libnvrtc.so.12", "libnvrtc.so"})
            if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) {
            r.why = std::string("dlopen libnvrtc: ") + dlerror();
            return r;
        }
        r.create = (decltype(r.create))dlsym(h, "nvrtcCreateProgram");
        r.compile = (decltype(r.compile))dlsym(h, "nvrtcCompileProgram");
        r.log_size = (decltype(r.log_size))dlsym(h, "nvrtcGetProgramLogSize");
        r.get_log = (decltype(r.get_log))dlsym(h, "nvrtcGetProgramLog");
        r.cubin_size = (decltype(r.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
        r.get_cubin = (decltype(r.get_cubin))dlsym(h, "nvrtcGetCUBIN");
        r.destroy = (decltype(r.destroy))dlsym(h, "nvrtcDestroyProgram");
        r.version = (decltype(r.version))dlsym(h, "nvrtcVersion");
        r.ok = r.create && r.compile && r.log_size && r.get_log && r.cubin_size && r.get_cubin && r.destroy;
        if (!r.ok) r.why = "libnvrtc lacks an expected symbol";
        return r;
    }();
    return n;
}

// Compile `src` to an sm_100a cubin; empty on failure (reason in *why).
std::vector<char> compile_cubin(const std::string &src, std::string *why) {
    if (const char *dir = std::getenv("SKC_SPARSE_DUMP")) {
        static int seq = 0;
        const std::string path = std::string(dir) + "/skc_sparse_" + std::to_string(seq++) + ".cu";
        if (FILE *f = std::fopen(path.c_str(), "w")) {
            std::fwrite(src.data(), 1, src.size(), f);
            std::fclose(f);
        }
    }
    Nvrtc &n = nvrtc();
    if (!n.ok) {
        *why = n.why;
        return {};
    }
    nvrtcProgram prog;
    if (n.create(&prog, src.c_str(), "skc_sparse.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        *why = "nvrtcCreateProgram failed";
        return {};
    }
    const char *opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true"};
    const nvrtcResult rc = n.compile(prog, 4, opts);
    std::vector<char> cubin;
    if (rc != NVRTC_SUCCESS) {
        size_t ls = 0;
        n.log_size(prog, &ls);
        std::string log(ls, '\0');
        if (ls) n.get_log(prog, &log[0]);
        *why = "nvrtc compile failed: " + log;
    } else {
        size_t cs = 0;
        n.cubin_size(prog, &cs);
        cubin.resize(cs);
        n.get_cubin(prog, cubin.data());
    }
    n.destroy(&prog);
    return cubin;
}

unsigned long long fnv1a(const std::string &src) {
    unsigned long long h = 1469598103934665603ULL;
    for (unsigned char ch : src) h = (h ^ ch) * 1099511628211ULL;
    return h;
}

// Optional on-disk cubin cache (a cold cache only costs compile time).  Off
// unless SKC_CACHE_DIR names a directory; the directory must belong to this
// user and must not be group/world-writable (a shared writable cache could
// inject code).  The key covers the generated source (FNV-1a + length), the
// NVRTC version and the driver version.
std::string cache_path(const std::string &src) {
    const char *d = std::getenv("SKC_CACHE_DIR");
    if (!d || !*d || std::string(d) == "0") return "";
    const std::string dir = d;
    for (size_t i = 1; i <= dir.size(); ++i)  // mkdir -p without a shell
        if (i == dir.size() || dir[i] == '/') ::mkdir(dir.substr(0, i).c_str(), 0700);
    struct stat st;
    if (::stat(dir.c_str(), &st) != 0 || !S_ISDIR(st.st_mode) || st.st_uid != ::geteuid() || (st.st_mode & 022))
        return "";
    int nv_major = 0, nv_minor = 0, drv = 0;
    Nvrtc &n = nvrtc();
    if (n.ok && n.version) n.version(&nv_major, &nv_minor);
    cudaDriverGetVersion(&drv);
    char name[160];
    std::snprintf(name, sizeof name, "/sparse_sm100a_nvrtc%d.%d_drv%d_%016llx_%zu.cubin", nv_major, nv_minor, drv,
                  fnv1a(src), src.size());
    return dir + name;
}

std::vector<char> cached_cubin(const std::string &src, std::string *why) {
    const std::string path = cache_path(src);
    if (!path.empty()) {
        if (FILE *f = std::fopen(path.c_str(), "rb")) {
            std::vector<char> buf;
            char tmp[65536];
            size_t n;
            while ((n = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + n);
            std::fclose(f);
            if (!buf.empty()) return buf;
        }
    }
    std::vector<char> cubin = compile_cubin(src, why);
    if (!cubin.empty() && !path.empty()) {
        const std::string tmpp = path + ".tmp" + std::to_string((long long)getpid());
        if (FILE *f = std::fopen(tmpp.c_str(), "wb")) {
            const bool ok = std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
            std::fclose(f);
            if (ok) std::rename(tmpp.c_str(), path.c_str());
            else std::remove(tmpp.c_str());
        }
    }
    return cubin;
}

// ------------------------------------------------------- kernel cache ---
// Compiled kernels keyed by their source (hash + length; the source names
// only the position pattern and the variant).  A miss starts an NVRTC
// compile on a background thread and returns nullptr, so the caller serves
// the layer with the tap / dense kernels until the kernel is ready (first
// calls on a new complex are not stalled by the 1-3 s compile); in sync mode
// (SKC_JIT=sync or skc_set_jit_mode(1)) the caller waits instead, so every
// call of a layer runs the same kernel.  At most kMaxKernels stay loaded
// (least recently used are unloaded).
enum { kCompiling = 0, kReady = 1, kFailed = 2 };
struct SpKernel {
    int state = kCompiling;
    bool built = false;          // background compile finished (cubin or why set)
    std::vector<char> cubin;
    std::string why;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    unsigned long long devmask = 0;  // devices whose shared-memory opt-in is set
    size_t smem = 0;
    unsigned long long last_use = 0;
    const char *name = "skc_sparse_stencil";  // entry point of the generated source
};
struct Key {
    unsigned long long h;
    size_t n;
    bool operator==(const Key &o) const { return h == o.h && n == o.n; }
};
struct KeyHash {
    size_t operator()(const Key &k) const { return (size_t)(k.h ^ (k.n * 0x9e3779b97f4a7c15ULL)); }
};
constexpr size_t kMaxKernels = 128;
std::mutex g_mu;
std::condition_variable g_cv;
std::unordered_map<Key, std::shared_ptr<SpKernel>, KeyHash> g_cache;
unsigned long long g_clock = 0;
std::atomic<int> g_jit_mode{-1};

int jit_sync() {
    int m = g_jit_mode.load();
    if (m < 0) {
        const char *e = std::getenv("SKC_JIT");
        m = (e && std::string(e) == "sync") ? 1 : 0;
        g_jit_mode.store(m);
    }
    return m;
}

void evict_lru_locked() {
    while (g_cache.size() > kMaxKernels) {
        auto victim = g_cache.end();
        for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
            if (it->second->state != kCompiling && (victim == g_cache.end() || it->second->last_use < victim->second->last_use))
                victim = it;
        if (victim == g_cache.end()) return;
        SpKernel &k = *victim->second;
        if (k.lib) {
            // launches of this kernel may still be queued: drain the devices it ran on
            int cur = 0;
            cudaGetDevice(&cur);
            for (int d = 0; d < 64; ++d)
                if (k.devmask >> d & 1ULL) {
                    cudaSetDevice(d);
                    cudaDeviceSynchronize();
                }
            cudaSetDevice(cur);
            cudaLibraryUnload(k.lib);
            cudaGetLastError();
        }
        g_cache.erase(victim);
    }
}

// Load a finished cubin (caller holds g_mu).
void finish_locked(SpKernel &k) {
    if (k.cubin.empty() ||
        cudaLibraryLoadData(&k.lib, k.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&k.kern, k.lib, k.name) != cudaSuccess) {
        cudaGetLastError();
        k.state = kFailed;
        if (std::getenv("SKC_SPARSE_VERBOSE")) std::fprintf(stderr, "skc sparse stencil unavailable: %s\n", k.why.c_str());
    } else {
        k.state = kReady;
    }
    std::vector<char>().swap(k.cubin);
}

// The compiled kernel for `src` (see above); nullptr while it compiles in
// the background or when the run-time compiler is unavailable / failed.
std::shared_ptr<SpKernel> get_kernel(const Key &key, const std::string &src, size_t smem,
                                     const char *name = "skc_sparse_stencil") {
    std::unique_lock<std::mutex> lock(g_mu);
    auto it = g_cache.find(key);
    std::shared_ptr<SpKernel> k;
    if (it == g_cache.end()) {
        k = std::make_shared<SpKernel>();
        k->smem = smem;
        k->name = name;
        g_cache.emplace(key, k);
        evict_lru_locked();
        if (jit_sync()) {
            lock.unlock();
            std::string why;
            std::vector<char> cubin = cached_cubin(src, &why);
            lock.lock();
            k->cubin.swap(cubin);
            k->why = why;
            k->built = true;
        } else {
            std::thread([k, src] {
                std::string why;
                std::vector<char> cubin = cached_cubin(src, &why);
                std::lock_guard<std::mutex> lk(g_mu);
                k->cubin.swap(cubin);
                k->why = why;
                k->built = true;
                g_cv.notify_all();
            }).detach();
        }
    } else {
        k = it->second;
    }
    if (k->state == kCompiling && !k->built && jit_sync()) g_cv.wait(lock, [&] { return k->built; });
    if (k->state == kCompiling && k->built) finish_locked(*k);
    k->last_use = ++g_clock;
    return k->state == kReady ? k : nullptr;
}

// Wait for every background compile to finish (skc_jit_wait).
void wait_all_compiles() {
    std::unique_lock<std::mutex> lock(g_mu);
    g_cv.wait(lock, [] {
        for (auto &kv : g_cache)
            if (kv.second->state == kCompiling && !kv.second->built) return false;
        return true;
    });
    for (auto &kv : g_cache)
        if (kv.second->state == kCompiling && kv.second->built) finish_locked(*kv.second);
}

// All-channel head eligibility (and its shared memory in p.smem): C
// interleaved channels staged per CTA, stencil-type layers, two CTAs per SM.
bool allc_ok(SpPlan &p, int S, int C, bool in_f32) {
    p.smem = in_f32 ? (size_t)p.nrows * (C * p.pitch + 1) * sizeof(float) : (size_t)p.nrows * (C * p.pitch + 2) * 2;
    const int D = dense_size_for(std::max(p.Dx, p.Dy));
    const bool stencil_like = eligible(p, S) || (D != 0 && D * D < 4 * S);
    return sparse_mode() != 0 && sp_hwc() == 2 && (sp_f2() == 1 || sp_f2() == 3) && stencil_like && p.npos > 0 &&
           (long long)p.npos * p.KR * 8 <= kSpMaxFfma && 2 * p.smem <= (size_t)kMaxSmem;
}

// Per-layer memo (host cost per launch is a hash lookup, not a plan and a
// 300 KB source string): keyed by the tap bytes, the variant and the knobs;
// holds the launch geometry, the kernel's cache key and the layer's weight
// table.  Bounded: cleared when it exceeds kMaxMemo entries.
struct SpLaunch {
    bool eligible = false;
    int npos = 0, TH = 0;
    double words_per_out = 0.0;
    size_t smem = 0;
    Key key{0, 0};
    std::string src;           // kept until the kernel is ready
    std::vector<float> kw;     // (K, K) per position: the kernel parameter
    int WY = 2;                // warps along y (CTA = 128 * WY threads)
    int minb = 2;              // resident CTAs per SM the kernel is built for
};
constexpr size_t kMaxMemo = 4096;
std::mutex g_memo_mu;
std::unordered_map<std::string, std::shared_ptr<SpLaunch>> g_memo;

std::string memo_key(const double *taps, int S, int variant) {
    std::string k((const char *)taps, sizeof(double) * 3 * (size_t)S);
    const int knobs[11] = {variant, sparse_mode(), sp_kr(), sp_sync(), sp_minb(), sp_f2(), sp_hwc(), sp_wy(), sp_tma(),
                           sp_kr_wide(), env_int("SKC_SPARSE_MINB_SMALL", 0)};
    k.append((const char *)knobs, sizeof knobs);
    return k;
}

void memo_put(const std::string &key, std::shared_ptr<SpLaunch> l) {
    std::lock_guard<std::mutex> lock(g_memo_mu);
    if (g_memo.size() >= kMaxMemo) g_memo.clear();
    g_memo[key] = std::move(l);
}

std::shared_ptr<SpLaunch> memo_get(const std::string &key) {
    std::lock_guard<std::mutex> lock(g_memo_mu);
    auto it = g_memo.find(key);
    return it == g_memo.end() ? nullptr : it->second;
}

}  // namespace

// Plan query for skc_layer_plan: 1 and the position count / LDS words per
// output when the layer would take the sparse path (cost model only; the
// run-time compiler is not consulted).
bool sparse_plan(const double *taps, int S, int *npos, double *words_per_out, bool small) {
    const std::string key = memo_key(taps, S, small ? -2 : -1);
    std::shared_ptr<SpLaunch> l = memo_get(key);
    if (!l) {
        const SpPlan p = make_plan(taps, S, small ? 1 : 0);
        l = std::make_shared<SpLaunch>();
        l->eligible = eligible(p, S, small);
        l->npos = p.npos;
        l->words_per_out = p.words_per_out;
        memo_put(key, l);
    }
    *npos = l->npos;
    *words_per_out = l->words_per_out;
    return l->eligible;
}

// Would an HWC head (fp32 or fp16 storage, planar output of the same dtype)
// run as the all-channel generated stencil?  skc_chain_fwd then skips its
// input relayout pass.
bool sparse_head_allc(const double *taps, int S, int C, bool f32) {
    SpPlan p = make_plan(taps, S);
    return allc_ok(p, S, C, f32);
}

// One layer through a generated sparse stencil: planar input (fp32 or fp16),
// planar or HWC output.  Returns -1 when the layer does not take this path
// (ineligible, or no run-time compiler), else a status code.
// Does a launch of this shape fill less than two waves of the default tiles
// (sparse_layer's `small` rule)?
bool sparse_small_launch(int B, int H, int W, int C, bool allc) {
    int cur_dev = 0, nsm = 148;
    if (cudaGetDevice(&cur_dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cur_dev);
    cudaGetLastError();
    const int th_default = 8 * sp_wy() * sp_kr();
    const long long ctas = (long long)ceil_div(W, kSpTW) * (allc ? 1 : C) * ceil_div(H, th_default) * B;
    return sp_wy() == 2 && ctas < 2LL * nsm && env_int("SKC_SPARSE_SMALL", 1);
}

int sparse_layer(const void *in, bool in_f32, void *out, bool out_f32, bool out_pl, int B, int H, int W, int C,
                 const double *taps, int S, int boundary, cudaStream_t s, bool in_hwc) {
    // HWC input: the all-channel head (fp32 in, planar out), or with
    // SKC_SPARSE_HWC=1 the per-channel variant; otherwise the dense / tap kernels
    const int allc = (in_hwc && sp_hwc() == 2 && in_f32 == out_f32 && out_pl && (sp_f2() == 1 || sp_f2() == 3)) ? C : 0;
    if (in_hwc && !allc && sp_hwc() != 1) return -1;
    // a grid below two waves at the default tile height (small images, e.g.
    // config 0's 512^2 frame) runs half-height tiles of one warp row instead
    int cur_dev = 0, nsm = 148;
    if (cudaGetDevice(&cur_dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cur_dev);
    const int th_default = 8 * sp_wy() * sp_kr();
    const long long ctas = (long long)ceil_div(W, kSpTW) * (allc ? 1 : C) * ceil_div(H, th_default) * B;
    const bool small = sp_wy() == 2 && ctas < 2LL * nsm && env_int("SKC_SPARSE_SMALL", 1);
    int wy = small ? 1 : 0;
    // all-channel heads run one-warp-row tiles (twice the resident CTAs, so
    // more tiles' loads in flight per SM: config 1's head 1.25 -> 1.12 ms;
    // SKC_SPARSE_HEAD_WY=2 keeps two warp rows)
    if (allc && sp_wy() == 2 && env_int("SKC_SPARSE_HEAD_WY", 1) == 1) wy = 1;
    // SKC_SPARSE_WY1=1: one-warp-row tiles for every generated layer (measurement switch)
    if (!allc && sp_wy() == 2 && env_int("SKC_SPARSE_WY1", 0) == 1) wy = 1;
    // small launches: all-channel heads at one row per thread (three times the CTAs, each a
    // third as long: config 0's head 7.5 -> 5.5 us; SKC_SPARSE_SMALL_KR=0 keeps the default)
    int kr_small = (small && allc) ? env_int("SKC_SPARSE_SMALL_KR", 1) : 0;
    // SKC_SPARSE_HEAD_KR: rows per thread of the all-channel head on large launches (measurement switch)
    if (allc && !small) kr_small = env_int("SKC_SPARSE_HEAD_KR", 0);
    // small launches chain through programmatic dependent launch: the next layer's CTAs are
    // resident and past their prologue when the previous layer's grid drains (SKC_PDL=0: plain launches)
    const bool pdl = small && env_int("SKC_PDL", 1) != 0;
    const std::string key = memo_key(taps, S, (in_f32 ? 1 : 0) | (out_f32 ? 2 : 0) | (out_pl ? 4 : 0) |
                                                  (in_hwc ? 8 : 0) | (allc << 4) | (wy << 12) | ((small ? 1 : 0) << 14) |
                                                  (kr_small << 15) | ((pdl ? 1 : 0) << 19));
    std::shared_ptr<SpLaunch> l = memo_get(key);
    if (!l) {
        SpPlan p = make_plan(taps, S, wy, kr_small);
        l = std::make_shared<SpLaunch>();
        l->eligible = eligible(p, S, small);
        if (allc) l->eligible = allc_ok(p, S, allc, in_f32);
        l->npos = p.npos;
        l->TH = p.TH;
        l->WY = p.WY;
        l->words_per_out = p.words_per_out;
        l->smem = p.smem;
        if (l->eligible) {
            l->src = generate(p, in_f32, out_f32, out_pl, in_hwc, allc, pdl);
            l->key = Key{fnv1a(l->src), l->src.size()};
            l->kw = kw_table(p);
        }
        memo_put(key, l);
    }
    if (!l->eligible) return -1;
    std::shared_ptr<SpKernel> k = get_kernel(l->key, l->src, l->smem);
    if (!k) return -1;   // compiling in the background (or unavailable): tap / dense kernels
    {   // the shared-memory opt-in is per device: set it once for each device used
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && dev < 64) {
            std::lock_guard<std::mutex> lock(g_mu);
            if (!(k->devmask >> dev & 1ULL)) {
                const cudaError_t ae = cudaFuncSetAttribute((const void *)k->kern,
                                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l->smem);
                if (ae != cudaSuccess) return cuda_fail(ae, "cudaFuncSetAttribute(skc_sparse_stencil)");
                k->devmask |= 1ULL << dev;
            }
        }
    }
    dim3 grid(ceil_div(W, kSpTW) * (allc ? 1 : C), ceil_div(H, l->TH), B);
    int clamp = boundary == SKC_CLAMP ? 1 : 0;
    void *kwp = (void *)l->kw.data();
    void *args[] = {(void *)&in, (void *)&out, (void *)&H, (void *)&W, (void *)&C, (void *)&clamp, kwp};
    cudaError_t e;
    if (pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(128 * l->WY);
        cfg.dynamicSmemBytes = l->smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelExC(&cfg, (const void *)k->kern, args);
    } else {
        e = cudaLaunchKernel((const void *)k->kern, grid, dim3(128 * l->WY), args, l->smem, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "skc_sparse_stencil");
    return SKC_OK;
}

// Layers 0 and 1 of a chain as one fused launch (generated skc_sparse_pair):
// fp32 HWC input -> fp32 planar output.  With in == nullptr a plan query
// (SKC_OK = the pair would run, -1 = it would not: ineligible, disabled with
// SKC_PAIR=0, or, outside sync JIT mode, still compiling).
int sparse_pair(const float *in, float *out, int B, int H, int W, int C, const double *t1, int S1, const double *t2,
                int S2, int boundary, cudaStream_t s) {
    if (pair_mode() == 0 || sparse_mode() == 0) return -1;
    int cur_dev = 0, nsm = 148;
    if (cudaGetDevice(&cur_dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cur_dev);
    std::string key((const char *)t1, sizeof(double) * 3 * (size_t)S1);
    key.append((const char *)t2, sizeof(double) * 3 * (size_t)S2);
    const int knobs[4] = {0x9a13, pair_kr(), S1, env_int("SKC_PAIR_MINB", 0)};
    key.append((const char *)knobs, sizeof knobs);
    std::shared_ptr<SpLaunch> l = memo_get(key);
    int minb = 2;
    if (!l) {
        const PairPlan q = make_pair_plan(t1, S1, t2, S2);
        l = std::make_shared<SpLaunch>();
        // both layers stencil-like (the sparse or dense paths would take them alone)
        const int D1 = dense_size_for(std::max(q.p1.Dx, q.p1.Dy));
        l->eligible = q.ok && (eligible(q.p1, S1) || (D1 != 0 && D1 * D1 < 4 * S1)) && eligible(q.p2, S2);
        l->npos = q.p1.npos + q.p2.npos;
        l->minb = q.minb;
        l->TH = q.p2.TH;
        l->WY = q.p2.WY;
        l->smem = q.smem;
        if (l->eligible) {
            l->src = generate_pair(q);
            l->key = Key{fnv1a(l->src), l->src.size()};
            l->kw = pair_kw_table(q);
        }
        memo_put(key, l);
    }
    if (!l->eligible) return -1;
    minb = l->minb;
    // rows per CTA (chunk, a multiple of TH): enough CTAs for ~16 waves; a
    // frame too small to fill two waves of single-block chunks runs unfused
    // (each chunk re-runs layer 0 on the rows it carries in)
    const long long cols = (long long)ceil_div(W, kSpTW) * C * B, nb = ceil_div(H, l->TH);
    const long long slots = (long long)nsm * minb;
    // (SKC_PAIR_SMALL=1, read per call, fuses them anyway: tests of the edge logic)
    if (cols * nb < 2 * slots && env_int("SKC_PAIR_SMALL", 0) == 0) return -1;
    const long long chunks = std::min<long long>(nb, std::max<long long>(1, (16 * slots + cols - 1) / cols));
    int CH = (int)(ceil_div((int)nb, (int)chunks) * l->TH);
    if (const int ch = env_int("SKC_PAIR_CH", 0)) CH = std::max(1, ch / l->TH) * l->TH;
    std::shared_ptr<SpKernel> k = get_kernel(l->key, l->src, l->smem, "skc_sparse_pair");
    if (!k) return -1;
    if (!in) return SKC_OK;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && dev < 64) {
            std::lock_guard<std::mutex> lock(g_mu);
            if (!(k->devmask >> dev & 1ULL)) {
                const cudaError_t ae = cudaFuncSetAttribute((const void *)k->kern,
                                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l->smem);
                if (ae != cudaSuccess) return cuda_fail(ae, "cudaFuncSetAttribute(skc_sparse_pair)");
                k->devmask |= 1ULL << dev;
            }
        }
    }
    dim3 grid(ceil_div(W, kSpTW) * C, ceil_div(H, CH), B);
    int clamp = boundary == SKC_CLAMP ? 1 : 0;
    void *kwp = (void *)l->kw.data();
    void *args[] = {(void *)&in, (void *)&out, (void *)&H, (void *)&W, (void *)&C, (void *)&clamp, (void *)&CH, kwp};
    const cudaError_t e = cudaLaunchKernel((const void *)k->kern, grid, dim3(128 * l->WY), args, l->smem, s);
    if (e != cudaSuccess) return cuda_fail(e, "skc_sparse_pair");
    return SKC_OK;
}

// Build check for the fused pair (no device needed): 0 = compiled, 1 = the
// pair is not eligible, SKC_ECUDA = NVRTC rejected it.
int sparse_pair_compile_check(const double *t1, int S1, const double *t2, int S2) {
    const PairPlan q = make_pair_plan(t1, S1, t2, S2);
    if (!q.ok) return SKC_ENOTTAKEN;
    std::string why;
    const std::vector<char> cubin = compile_cubin(generate_pair(q), &why);
    return cubin.empty() ? fail(SKC_ECUDA, why) : SKC_OK;
}

}  // namespace skc

extern "C" {

// Generate and compile (NVRTC, no device needed) the sparse stencil this layer
// would run: 0 = compiled, 1 = the layer does not take the sparse path,
// SKC_ECUDA = the run-time compiler is missing or rejected the source
// (message in skc_last_error).
int skc_sparse_compile_check(const double *taps, int S, int in_dtype, int in_layout, int out_dtype, int out_layout) {
    using namespace skc;
    if (!taps || S < 1) return fail(SKC_EBADARG, "bad layer arguments");
    const SpPlan p = make_plan(taps, S);
    // the all-channel head variant (SKC_SPARSE_HWC=2) is checked for C = 3
    const int allc = (in_layout == SKC_HWC && sp_hwc() == 2 && in_dtype == out_dtype && out_layout == SKC_CHW && (sp_f2() == 1 || sp_f2() == 3))
                         ? (in_dtype == SKC_F32 ? 3 : 4) : 0;
    if (!allc && !eligible(p, S)) return 1;
    std::string why;
    const std::vector<char> cubin = compile_cubin(
        generate(p, in_dtype == SKC_F32, out_dtype == SKC_F32, out_layout == SKC_CHW, in_layout == SKC_HWC, allc), &why);
    return cubin.empty() ? fail(SKC_ECUDA, why) : SKC_OK;
}

int skc_set_jit_mode(int mode) {
    if (mode != 0 && mode != 1) return skc::fail(SKC_EBADARG, "jit mode must be 0 (async) or 1 (sync)");
    skc::g_jit_mode.store(mode);
    return SKC_OK;
}

int skc_jit_wait(void) {
    skc::wait_all_compiles();
    return SKC_OK;
}

}  // extern "C"
