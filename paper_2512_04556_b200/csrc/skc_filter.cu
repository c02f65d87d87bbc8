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
