// skc_kawase.cu -- fused, separable Kawase chains (BASELINE config 3, SURVEY
// §2.2 K3) in one persistent launch per call, TMA-fed.
//
// Reference: engine.apply_complex (engine.py:173-178) materialises every
// layer; a layer is apply_sparse_layer (engine.py:160-170) -> sample_shifted
// (118-130) -> _accum_shift (106-115) with zero padding.
//
// A Kawase layer has 4 taps (+-r, +-r) with r = b + 1/2 (b >= 0 integer) and
// one weight w.  Each bilinear tap sits at fraction 1/2 on both axes, so the
// layer is w/4 * (H4 (x) V4) with the unweighted 1-D sum
//     H4 x(p) = x(p-b-1) + x(p-b) + x(p+b) + x(p+b+1),
// and zero padding is a separable mask applied after every layer.  The whole
// chain is therefore  prod_l(w_l/4) * [prod_l My V4_l] [prod_l Mx H4_l] in
// (verified equal to the 2-D chain for zero padding).  Each 1-D
// pass is a pair sum s(p) = x(p) + x(p-1) followed by y(p) = s(p) + s(p-2b-1):
// two adds per output per layer per axis, the scale applied once at the end
// (a power of two for w = 1/4, so exact).
//
// Kernel: persistent CTAs walk work items (frame, 128-column band, row
// segment).  Per 32-row iteration:
//   * one elected producer thread loads the band's rows with one 3-D TMA box
//     (cp.async.bulk.tensor, 64-bit elements = one fp16 RGBA pixel) into a
//     2-stage ring; out-of-image columns/rows arrive as zeros;
//   * 2 H warps (lane = row x channel pair) stream their row along x through
//     the L horizontal passes in registers (fully unrolled; intermediate
//     columns outside the image are zeroed per layer in edge bands) and store
//     128 fp32 channel-pair columns into a 2-stage H-result ring;
//   * 8 V warps (lane = column x channel pair) stream down the rows with the
//     vertical passes' delay lines carried in registers across iterations
//     and across the whole segment (no vertical halo recompute), zero rows
//     outside the image per layer at the top/bottom, scale, round to fp16
//     once and store coalesced.
// HBM traffic per pixel: 8 B in + 8 B out (the horizontal halo of 2 x reach
// columns per 128 is re-read from L2); fp32 arithmetic throughout; one fp16
// rounding of the output.
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "skc_tile.cuh"

namespace skc {
namespace {

constexpr int kKwTW = 128;        // output columns per band
constexpr int kKwR = 32;          // rows per iteration
constexpr int kKwNV = kKwTW / 16; // V warps (16 columns x 2 channel pairs each)
// H warps: 2 per row segment (16 rows x 2 channel pairs each); HS = 1 runs
// the band's whole row per lane, HS = 2 splits it into two 64-column halves
// (each with its own 2 x reach halo) over twice the lanes
// SC (HS = 2 only, opt-in SKC_KAWASE_SC=1): one channel per H lane (scalar
// fp32 state) -- 8 H warps of 8 rows x 4 channels, each with half the register
// state and FADD (one pipe cycle) where the channel-pair lanes issue FADD2
// (two).  A single warp issues an FADD2 every other cycle at best, and the 4
// pair-lane H warps are the critical path (V warps wait half their time on the
// H results, profiles/r02_kawase_peel.md).  The 16 warps launch at 128
// registers and rebalance with setmaxnreg: H warpgroups drop to 96, V
// warpgroups (128 registers of delay lines) take 160.  Measured slower (config
// 3: 1.72 vs 1.50 ms): the V warps' wait disappears (10% of samples) but twice
// the H instructions fill the issue slots (issue 72%, math-pipe throttle the
// top stall at 63% FMA-pipe cycles), profiles/r02_kawase_sc.md.
template <int HS, bool SC = false> __host__ __device__ constexpr int kw_nh() { return SC ? 8 : 2 * HS; }
// the TMA producer is lane 0 of H warp 0 (a separate warp would make 13
// warps for HS = 2: four on one SM sub-partition caps registers at 128)
template <int HS, bool SC = false> __host__ __device__ constexpr int kw_threads() { return 32 * (kw_nh<HS, SC>() + kKwNV); }
// H-result row pitch (words): 2 mod 32 for the float2 stores of the pair
// lanes, 4 mod 32 for the scalar lanes (8 rows x 4 channels per warp: banks 4 r + c)
// (LVW > 0: the LV tile of LVW columns, see KwGen::kLvW)
template <bool SC = false, int LVW = 0> __host__ __device__ constexpr int kw_hp() {
    return LVW > 0 ? LVW * 4 + 2 : kKwTW * 4 + (SC ? 4 : 2);
}

struct KwParams {
    __half *out;
    int B, H, W;
    int bands, segs, seglen, items;
    float scale;
    int dbg;   // SKC_KAWASE_DBG bits (bring-up): 1 = no TMA, 2 = no H math, 4 = no V math
    int hint;  // mbarrier.try_wait suspend-time hint, ns (SKC_KAWASE_HINT, default 1000)
    int peel;  // interior rows run the H passes with the warm-up peeled (SKC_KAWASE_PEEL, default 1)
};

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// `hint` = suspend-time hint in ns: the warp sleeps (instead of spinning on the
// issue slots the other warps need) until the phase completes or the hint
// expires.  The wake-up on completion is not reliable enough to sleep long: at
// 131 us per try some CTAs of config 3 lost 1 ms to expired sleeps (SM active
// cycles 3.0 M .. 5.4 M across the grid, profiles/r02_kawase_hint.md), so the
// default is 1 us (KwParams::hint, SKC_KAWASE_HINT).
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity, unsigned hint) {
    const unsigned a = smem_u32(bar);
    unsigned done = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity), "r"(hint)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, unsigned long long *bar, int x, int y,
                                            int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long ra, rb, rd;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
    return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long ra, rb, rd;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
    float2 d;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
    return d;
}

// one fp16 pair, rounded once, to global memory (st.global: the V lanes' row
// pointer is kept opaque to the optimiser, which would otherwise lose the
// address space with it)
__device__ __forceinline__ void st_h2(char *p, float2 v) {
    const __half2 h = __float22half2_rn(v);
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(*reinterpret_cast<const unsigned *>(&h)) : "memory");
}

__device__ __forceinline__ float2 h2f2(unsigned hv) {
    return __half22float2(*reinterpret_cast<const __half2 *>(&hv));
}

// The pass bodies for the ladders b_l = l (generated: build/skc_kawase_gen.inc)
#include "skc_kawase_gen.inc"

struct Item {
    int f, x0, y0, y1, iters;
};

// TMA box geometry.  The box's first column must sit on a 16-byte boundary
// (an odd 8-byte pixel start faults), so the box starts one pixel early when
// the reach is odd; its width is padded to 2 mod 4 pixels so the staged row
// pitch spreads the H lanes' half2 reads over 16 banks (2-way at worst).
// (LV: the wider H-result tile leaves no room for the pad: the box is the next
// even width, 4-way conflicts on the H lanes' one load per step)
template <int L, bool LV = false>
struct KwBox {
    static constexpr int RX = KwGen<L>::kReach;
    static constexpr int OFF = RX & 1;                       // leading pad pixels
    static constexpr int IW = kKwTW + 2 * RX;                // pixels the passes read
    static constexpr int IWB2 = ((IW + OFF + 1) / 4) * 4 + 2 >= IW + OFF ? ((IW + OFF + 1) / 4) * 4 + 2
                                                                         : ((IW + OFF + 1) / 4) * 4 + 6;
    static constexpr int IWB = LV ? ((IW + OFF + 1) & ~1) : IWB2;
    static constexpr unsigned kStageBytes = (unsigned)kKwR * IWB * 8;
};

template <int L>
__device__ __forceinline__ Item item_of(const KwParams &p, int it) {
    Item r;
    const int seg = it % p.segs;
    const int rest = it / p.segs;
    const int band = rest % p.bands;
    r.f = rest / p.bands;
    r.x0 = band * kKwTW;
    r.y0 = seg * p.seglen;
    r.y1 = min(p.H, r.y0 + p.seglen);
    // the vertical wavefront is skewed by one step per layer: L - 1 extra steps
    r.iters = (r.y1 - r.y0 + 2 * KwGen<L>::kReach + (L - 1) + kKwR - 1) / kKwR;
    return r;
}

// one CTA per SM: the register budget is the whole file / the CTA's threads
// LV (HS = 2, pair lanes, L >= 2): the H warps run the first L - 1 horizontal
// layers over the band plus b + 1 halo columns each side and the V lanes apply
// the last horizontal layer as they load (4 loads + 3 adds instead of 1 load):
// the 4 H warps are the critical path (an H warp issues at most one FADD2 every
// other cycle) and the 8 V warps wait on them half their time.  Opt-in
// (SKC_KAWASE_LV=1): measured 2.43 vs 1.50 ms on config 3 -- the H warps alone
// do not get faster (1.00 vs 0.99 ms: with the 140-column tile the input box
// loses its bank-spreading pad and its loads conflict 4-way), the V lanes
// alone slow from 0.73 to 0.95 ms, and together they overlap worse
// (profiles/r02_kawase_lv.md: issue 40%, FMA pipe 48%).
template <int L, int HS, bool SC, bool LV>
__global__ void __maxnreg__((HS == 4 || SC) ? 128 : 168)
    kawase_sep_kernel(const __grid_constant__ CUtensorMap tmap, const KwParams p) {
    constexpr int kKwNH = kw_nh<HS, SC>();
    using G = KwGen<L>;
    constexpr int kKwHP = kw_hp<SC, LV ? G::kLvW : 0>();
    constexpr int RX = G::kReach;
    using BX = KwBox<L, LV>;
    constexpr unsigned kStageBytes = BX::kStageBytes;
    extern __shared__ __align__(128) unsigned char smem[];
    // stage s of the input ring at smem + s * kStageBytes, of the H-result
    // ring at hres0 + s * kKwR * kKwHP (arithmetic, not a pointer array: an
    // array indexed by s would live in local memory)
    float *const hres0 = reinterpret_cast<float *>(smem + 2 * kStageBytes);
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(smem + 2 * kStageBytes + 2 * kKwR * kKwHP * 4);
    unsigned long long *full_in = bars, *empty_in = bars + 2, *full_h = bars + 4, *empty_h = bars + 6;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned hint = (unsigned)p.hint;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full_in[i], 1);
            mbar_init(&empty_in[i], 32 * kKwNH);
            mbar_init(&full_h[i], 32 * kKwNH);
            mbar_init(&empty_h[i], 32 * kKwNV);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp < kKwNH) {
        // ------------------------------------------ horizontal passes ---
        if (SC) asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
        constexpr int SW = kKwTW / HS;            // output columns per lane
        // pair lanes: 16 rows x 2 channel pairs per warp; scalar lanes: 8 rows x 4 channels
        const int seg = SC ? warp >> 2 : warp >> 1;
        const int r = SC ? (warp & 3) * 8 + (lane >> 2) : (warp & 1) * 16 + (lane & 15);
        const int pr = SC ? (lane & 3) : lane >> 4;
        // TMA producer (lane 0 of warp 0): loads run one chunk ahead of the
        // passes; chunk c lands in stage c & 1 (the (c >> 1)-th use of it)
        const bool prod = warp == 0 && lane == 0;
        int l_it = blockIdx.x, l_i = 0;
        Item lm;
        if (l_it < p.items) lm = item_of<L>(p, l_it);
        auto issue = [&](int stage) {
            if (p.dbg & 1) {
                mbar_arrive(&full_in[stage]);
            } else {
                mbar_expect_tx(&full_in[stage], kStageBytes);
                tma_load_3d(smem + stage * kStageBytes, &tmap, &full_in[stage], lm.x0 - RX - BX::OFF,
                            lm.y0 - RX + l_i * kKwR, lm.f);
            }
            if (++l_i >= lm.iters) {
                l_i = 0;
                l_it += gridDim.x;
                if (l_it < p.items) lm = item_of<L>(p, l_it);
            }
        };
        if (prod && l_it < p.items) issue(0);
        unsigned g = 0;
        for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
            const Item m = item_of<L>(p, it);
            const int xs = m.x0 + seg * SW;
            const bool edge = xs - RX < 0 || xs + SW + RX > p.W;
            for (int i = 0; i < m.iters; ++i, ++g) {
                const int s = g & 1;
                if (prod && l_it < p.items) {
                    // chunk g + 1 reuses the stage of chunk g - 1: wait until every H lane released it
                    if (g >= 1) mbar_wait(&empty_in[s ^ 1], ((g - 1) >> 1) & 1, hint);
                    issue(s ^ 1);
                }
                mbar_wait(&full_in[s], (g >> 1) & 1, hint);
                if (g >= 2) mbar_wait(&empty_h[s], ((g >> 1) - 1) & 1, hint);
                const unsigned *row = reinterpret_cast<const unsigned *>(smem + s * kStageBytes) +
                                      (r * BX::IWB + BX::OFF + seg * SW) * 2 + pr;
                float2 *orow = reinterpret_cast<float2 *>(hres0 + s * kKwR * kKwHP + r * kKwHP) + seg * SW * 2 + pr;
                if (p.dbg & 2) {
                } else if constexpr (LV) {
                    constexpr int LW = G::kLvW / 2;               // H-result columns per lane
                    constexpr int RXH = G::kLvReach;              // reach of the layers the H warps run
                    const int xo = m.x0 - (RX - RXH) + seg * LW;  // first column this lane stores (global)
                    const unsigned *rowl = reinterpret_cast<const unsigned *>(smem + s * kStageBytes) +
                                           (r * BX::IWB + BX::OFF + seg * LW) * 2 + pr;
                    float2 *orowl = reinterpret_cast<float2 *>(hres0 + s * kKwR * kKwHP + r * kKwHP) + seg * LW * 2 + pr;
                    if (xo - RXH < 0 || xo + LW + RXH > p.W) G::template h_half_lv<true>(rowl, orowl, xo - RXH, p.W);
                    else if (p.peel) G::h_half_lv_peel(rowl, orowl);
                    else G::template h_half_lv<false>(rowl, orowl, xo - RXH, p.W);
                } else if (SC) {
                    const __half *rowh = reinterpret_cast<const __half *>(smem + s * kStageBytes) +
                                         (r * BX::IWB + BX::OFF + seg * SW) * 4 + pr;
                    float *oroww = hres0 + s * kKwR * kKwHP + r * kKwHP + seg * SW * 4 + pr;
                    if (edge) G::template h_half_sc<true>(rowh, oroww, xs - RX, p.W);
                    else if (p.peel) G::h_half_peel_sc(rowh, oroww);
                    else G::template h_half_sc<false>(rowh, oroww, xs - RX, p.W);
                } else if (HS == 1) {
                    if (edge) G::template h<true>(row, orow, xs - RX, p.W);
                    else if (p.peel) G::h_peel(row, orow);
                    else G::template h<false>(row, orow, xs - RX, p.W);
                } else if (HS == 2) {
                    if (edge) G::template h_half<true>(row, orow, xs - RX, p.W);
                    else if (p.peel) G::h_half_peel(row, orow);
                    else G::template h_half<false>(row, orow, xs - RX, p.W);
                } else {
                    if (edge) G::template h_quarter<true>(row, orow, xs - RX, p.W);
                    else if (p.peel) G::h_quarter_peel(row, orow);
                    else G::template h_quarter<false>(row, orow, xs - RX, p.W);
                }
                mbar_arrive(&empty_in[s]);
                mbar_arrive(&full_h[s]);
            }
        }
        return;
    }
    // ------------------------------------------------ vertical passes ---
    if (SC) asm volatile("setmaxnreg.inc.sync.aligned.u32 160;");
    const int vw = warp - kKwNH;
    const int xl = vw * 16 + (lane >> 1), pr = lane & 1;
    unsigned g = 0;
    for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
        const Item m = item_of<L>(p, it);
        typename G::State S;
        G::zero(S);
        const int x = m.x0 + xl;
        __half *outp = p.out + (((long long)m.f * p.H) * p.W + x) * 4 + 2 * pr;
        const float2 sc = make_float2(p.scale, p.scale);
        for (int i = 0; i < m.iters; ++i, ++g) {
            const int s = g & 1;
            mbar_wait(&full_h[s], (g >> 1) & 1, hint);
            const float2 *col = reinterpret_cast<const float2 *>(hres0 + s * kKwR * kKwHP) + 2 * xl + pr;
            const int yin0 = m.y0 - RX + i * kKwR;
            // intermediate rows outside the image occur only near the top and
            // bottom: those iterations zero them per layer
            const bool mask = yin0 - RX - (L - 1) < 0 || yin0 + kKwR - 1 >= p.H;
            // a column past the image edge runs the stream (its lanes share the
            // warp's barriers) but stores nothing
            const int y1 = x < p.W ? m.y1 : m.y0;
            if (p.dbg & 4) {
            } else if constexpr (LV) {
                // col = the H-result tile at column x - (b + 1): the last horizontal layer runs on load
                if (mask) G::template v_lv<true, kKwHP / 2>(col, S, yin0, p.H, yin0 - RX, m.y0, y1, outp, (long long)p.W * 4, sc);
                else G::template v_lv<false, kKwHP / 2>(col, S, yin0, p.H, yin0 - RX, m.y0, y1, outp, (long long)p.W * 4, sc);
            } else if (mask) G::template v<true, kKwHP / 2>(col, S, yin0, p.H, yin0 - RX, m.y0, y1, outp, (long long)p.W * 4, sc);
            else G::template v<false, kKwHP / 2>(col, S, yin0, p.H, yin0 - RX, m.y0, y1, outp, (long long)p.W * 4, sc);
            mbar_arrive(&empty_h[s]);
        }
    }
}

// ------------------------------------------------------------------ host ---
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        cudaGetLastError();
        return (EncodeTiledFn)f;
    }();
    return fn;
}

int kawase_env() {
    static const int v = [] {
        const char *e = std::getenv("SKC_KAWASE");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// The chain as (L, b_l) when every layer is a Kawase quadruple (+-r, +-r),
// r = b + 1/2, with equal weights; scale = prod_l w_l / 4.
bool kawase_pattern(const double *taps, const int *layout, int L, int *b, double *scale) {
    if (L < 1 || L > 8) return false;
    double sc = 1.0;
    const double *t = taps;
    for (int l = 0; l < L; ++l, t += 3 * layout[l - 1]) {
        if (layout[l] != 4) return false;
        const double r = std::fabs(t[0]);
        const double w = t[2];
        const double bb = r - 0.5;
        if (!(bb >= 0) || bb != std::floor(bb) || bb > 15) return false;
        bool seen[4] = {false, false, false, false};
        for (int i = 0; i < 4; ++i) {
            const double ox = t[3 * i], oy = t[3 * i + 1];
            if (t[3 * i + 2] != w || std::fabs(ox) != r || std::fabs(oy) != r) return false;
            seen[(ox > 0 ? 1 : 0) | (oy > 0 ? 2 : 0)] = true;
        }
        if (!(seen[0] && seen[1] && seen[2] && seen[3])) return false;
        b[l] = (int)bb;
        sc *= w / 4.0;
    }
    *scale = sc;
    return true;
}

int kawase_hs() {
    static const int v = [] {
        const char *e = std::getenv("SKC_KAWASE_HS");
        const int v = e ? std::atoi(e) : 2;
        return (v == 1 || v == 4) ? v : 2;
    }();
    return v;
}

// the last horizontal layer applied by the V lanes (kawase_sep_kernel<L, 2, false, true>):
// SKC_KAWASE_LV, default 0 -- measured slower (config 3: 2.43 vs 1.50 ms)
int kawase_lv() {
    static const int v = [] {
        const char *e = std::getenv("SKC_KAWASE_LV");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// scalar H lanes (kawase_sep_kernel<L, 2, true>): SKC_KAWASE_SC, default 0
int kawase_sc() {
    static const int v = [] {
        const char *e = std::getenv("SKC_KAWASE_SC");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

template <int L, int HS, bool SC = false, bool LV = false>
int launch_kawase(const void *in, void *out, int B, int H, int W, float scale, cudaStream_t s) {
    constexpr int kKwHP = kw_hp<SC, LV ? KwGen<L>::kLvW : 0>();
    constexpr int RX = KwGen<L>::kReach;
    using BX = KwBox<L, LV>;
    static_assert(BX::IWB <= 256 && BX::IWB % 2 == 0 && BX::IWB >= BX::IW + BX::OFF, "TMA box width");
    const size_t smem = 2 * (size_t)BX::kStageBytes + 2 * (size_t)kKwR * kKwHP * 4 + 8 * sizeof(unsigned long long);
    if (smem > (size_t)kMaxSmem) return -1;
    EncodeTiledFn enc = encode_fn();
    if (!enc) return -1;
    CUtensorMap map;
    const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    const cuuint64_t strides[2] = {(cuuint64_t)W * 8, (cuuint64_t)W * H * 8};
    const cuuint32_t box[3] = {(cuuint32_t)BX::IWB, (cuuint32_t)kKwR, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void *>(in), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -1;
    KwParams p;
    p.out = static_cast<__half *>(out);
    p.B = B;
    p.H = H;
    p.W = W;
    p.bands = ceil_div(W, kKwTW);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // row segments: enough items to balance the persistent grid, each segment
    // long against its 2 x reach warm-up rows
    const long long cols = (long long)B * p.bands;
    int segs = 1;
    double best = 1e30;
    for (int k = 1; k <= 64; ++k) {
        const int len = ceil_div(H, k);
        if (k > 1 && len < 8 * RX) break;
        const long long items = cols * k;
        const long long rounds = (items + nsm - 1) / nsm;
        const double cost = (double)rounds * (len + 2 * RX + kKwR);
        if (cost < best * 0.98) {
            best = cost;
            segs = k;
        }
    }
    p.segs = segs;
    p.seglen = ceil_div(H, segs);
    p.items = (int)(cols * segs);
    p.scale = scale;
    {
        const char *e = std::getenv("SKC_KAWASE_DBG");
        p.dbg = e ? std::atoi(e) : 0;
        e = std::getenv("SKC_KAWASE_HINT");
        p.hint = e ? std::max(0, std::atoi(e)) : 1000;
        e = std::getenv("SKC_KAWASE_PEEL");
        p.peel = e ? std::atoi(e) : 1;
    }
    auto kern = kawase_sep_kernel<L, HS, SC, LV>;
    if (int rc = smem_optin((const void *)kern, (int)smem)) return rc;
    const int grid = std::min(p.items, nsm);
    kern<<<grid, kw_threads<HS, SC>(), smem, s>>>(map, p);
    SKC_LAUNCH_CHECK("kawase_sep_kernel");
    return SKC_OK;
}

}  // namespace

// Fused separable Kawase chain (see top of file) for fp16 RGBA, zero
// boundary; -1 when the chain or the image does not qualify (the per-layer
// path runs instead).
int kawase_chain(const void *in, int idt, void *out, int odt, int B, int H, int W, int C, const double *taps,
                 const int *layout, int L, int boundary, cudaStream_t s) {
    if (kawase_env() == 0) return -1;
    if (C != 4 || idt != SKC_F16 || odt != SKC_F16 || boundary != SKC_ZERO || (W & 1)) return -1;
    if (in && ((reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 7))) return -1;
    int b[8];
    double scale;
    if (!kawase_pattern(taps, layout, L, b, &scale)) return -1;
    for (int l = 0; l < L; ++l)
        if (b[l] != l) return -1;  // instantiated: the standard Kawase ladder r_l = l + 1/2
    if (!in) return encode_fn() ? SKC_OK : -1;  // plan query
    const int hs = kawase_hs();
#define SKC_KW_CASE(LL)                                                                              \
    case LL:                                                                                         \
        if (hs == 2 && kawase_sc()) return launch_kawase<LL, 2, true>(in, out, B, H, W, (float)scale, s); \
        if (hs == 2 && LL >= 2 && kawase_lv()) {                                                     \
            const int rc = launch_kawase<LL, 2, false, (LL >= 2)>(in, out, B, H, W, (float)scale, s); \
            if (rc != -1) return rc;                                                                 \
        }                                                                                            \
        return hs == 1 ? launch_kawase<LL, 1>(in, out, B, H, W, (float)scale, s)                     \
                       : hs == 4 ? launch_kawase<LL, 4>(in, out, B, H, W, (float)scale, s)          \
                                 : launch_kawase<LL, 2>(in, out, B, H, W, (float)scale, s);
    switch (L) {
        SKC_KW_CASE(1)
        SKC_KW_CASE(2)
        SKC_KW_CASE(3)
        SKC_KW_CASE(4)
        SKC_KW_CASE(5)
        SKC_KW_CASE(6)
        default: return -1;
    }
#undef SKC_KW_CASE
}

}  // namespace skc
