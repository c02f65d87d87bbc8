// skc_dense.cu -- dense-stencil form of a uniform sparse layer (sm_100a).
//
// A uniform layer (engine.apply_sparse_layer, engine.py:160-170) is a sum of
// 4*S integer shifts with constant weights (sample_shifted, engine.py:118-130).
// When its corner footprint fits a D x D window with D*D < 4*S -- e.g. the
// radius-2 and radius-4 layers of the config-1 complex (5x5 and 9x9 windows
// for 128 corner terms) -- the host merges coincident corners into a D x D
// stencil and this kernel evaluates it with every weight a compile-time
// offset into the kernel-parameter constant bank (FFMA with a c[][] operand).
// Each thread owns a KR x MC output block; every staged input row is read
// once into registers and feeds up to D output rows, so shared-memory
// traffic is (KR+D-1)(MC+D-1) words per D*D*KR*MC FMAs.
#include "skc_tile.cuh"

namespace skc {

constexpr int kDKR = 5, kDMC = 4, kDWX = 2, kDWY = 4;
constexpr int kDTW = kDWX * 32, kDTH = kDWY * kDMC * kDKR;

template <int C, int D, typename TI, typename TO>
__global__ void __launch_bounds__(kDWX *kDWY * 32)
    layer_dense_kernel(const TI *__restrict__ in, TO *__restrict__ out, const Geom g,
                       const __grid_constant__ DenseTable dt) {
    extern __shared__ float smem[];
    constexpr int KR = kDKR, MC = kDMC, LX = 32 / MC, LY = MC;
    const int tx0 = blockIdx.x * kDTW, ty0 = blockIdx.y * kDTH;
    in += (long long)blockIdx.z * g.in_fs;
    out += (long long)blockIdx.z * g.out_fs;
    load_tile<C, TI>(smem, in, g.H, g.W, g.boundary, tx0 + g.dx0, ty0 + g.dy0, g.pitch, g.rows);
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = lane % LX, ly = lane / LX, wx = warp % kDWX, wy = warp / kDWX;
    const int col0 = wx * 32 + lx * MC;
    const int row0 = wy * LY * KR + ly * KR;
    const int plane = g.rows * g.pitch;
    const int pitch = g.pitch;

#pragma unroll 1
    for (int c = 0; c < C; ++c) {
        const float *pc = smem + c * plane + row0 * pitch + col0;
        float acc[KR][MC];
#pragma unroll
        for (int i = 0; i < KR; ++i)
#pragma unroll
            for (int j = 0; j < MC; ++j) acc[i][j] = 0.f;
#pragma unroll
        for (int r = 0; r < KR + D - 1; ++r) {
            float w[MC + D - 1];
#pragma unroll
            for (int j = 0; j < MC + D - 1; ++j) w[j] = pc[r * pitch + j];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int i = r - a;
                if (i < 0 || i >= KR) continue;
#pragma unroll
                for (int b = 0; b < D; ++b) {
                    const float k = dt.k[a * D + b];
#pragma unroll
                    for (int j = 0; j < MC; ++j) acc[i][j] = fmaf(k, w[j + b], acc[i][j]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < KR; ++i) {
            const int gy = ty0 + row0 + i;
            if (gy >= g.H) continue;
            TO *orow = out + (long long)gy * g.W * C + c;
#pragma unroll
            for (int j = 0; j < MC; ++j) {
                const int gx = tx0 + col0 + j;
                if (gx < g.W) store_px<TO>(orow + (long long)gx * C, acc[i][j], g.accumulate);
            }
        }
    }
}

int dense_size_for(int span) {
    if (span <= 3) return 3;
    if (span <= 5) return 5;
    if (span <= 7) return 7;
    if (span <= 9) return 9;
    return 0;
}

template <int C, int D, typename TI, typename TO>
static int launch_dense_t(const void *in, void *out, int B, int H, int W, const DenseTable &dt,
                          int dx0, int dy0, int boundary, cudaStream_t s) {
    Geom g;
    g.H = H;
    g.W = W;
    g.boundary = boundary;
    g.accumulate = 0;
    g.in_fs = g.out_fs = (long long)H * W * C;
    g.dx0 = dx0;
    g.dy0 = dy0;
    int pitch = kDTW + D - 1;
    if ((pitch & 1) == 0) ++pitch;
    g.pitch = pitch;
    g.rows = kDTH + D - 1;
    const size_t smem = (size_t)C * g.rows * g.pitch * sizeof(float);
    auto kern = layer_dense_kernel<C, D, TI, TO>;
    static bool attr = false;
    if (!attr) {
        SKC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
        attr = true;
    }
    dim3 grid(ceil_div(W, kDTW), ceil_div(H, kDTH), B);
    kern<<<grid, kDWX * kDWY * 32, smem, s>>>(static_cast<const TI *>(in), static_cast<TO *>(out), g, dt);
    SKC_LAUNCH_CHECK("layer_dense_kernel");
    return SKC_OK;
}

template <int C, int D>
static int launch_dense_cd(const void *in, int idt, void *out, int odt, int B, int H, int W,
                           const DenseTable &dt, int dx0, int dy0, int boundary, cudaStream_t s) {
    if (idt == SKC_F32 && odt == SKC_F32) return launch_dense_t<C, D, float, float>(in, out, B, H, W, dt, dx0, dy0, boundary, s);
    if (idt == SKC_F16 && odt == SKC_F32) return launch_dense_t<C, D, __half, float>(in, out, B, H, W, dt, dx0, dy0, boundary, s);
    if (idt == SKC_F32 && odt == SKC_F16) return launch_dense_t<C, D, float, __half>(in, out, B, H, W, dt, dx0, dy0, boundary, s);
    return launch_dense_t<C, D, __half, __half>(in, out, B, H, W, dt, dx0, dy0, boundary, s);
}

template <int C>
static int launch_dense_c(const void *in, int idt, void *out, int odt, int B, int H, int W,
                          const DenseTable &dt, int dx0, int dy0, int boundary, cudaStream_t s) {
    switch (dt.D) {
        case 3: return launch_dense_cd<C, 3>(in, idt, out, odt, B, H, W, dt, dx0, dy0, boundary, s);
        case 5: return launch_dense_cd<C, 5>(in, idt, out, odt, B, H, W, dt, dx0, dy0, boundary, s);
        case 7: return launch_dense_cd<C, 7>(in, idt, out, odt, B, H, W, dt, dx0, dy0, boundary, s);
        case 9: return launch_dense_cd<C, 9>(in, idt, out, odt, B, H, W, dt, dx0, dy0, boundary, s);
        default: return fail(SKC_EBADARG, "dense stencil size must be 3, 5, 7 or 9");
    }
}

int launch_dense(const void *in, int idt, void *out, int odt, int B, int H, int W, int C,
                 const DenseTable &dt, int dx0, int dy0, int boundary, cudaStream_t s) {
    switch (C) {
        case 1: return launch_dense_c<1>(in, idt, out, odt, B, H, W, dt, dx0, dy0, boundary, s);
        case 2: return launch_dense_c<2>(in, idt, out, odt, B, H, W, dt, dx0, dy0, boundary, s);
        case 3: return launch_dense_c<3>(in, idt, out, odt, B, H, W, dt, dx0, dy0, boundary, s);
        case 4: return launch_dense_c<4>(in, idt, out, odt, B, H, W, dt, dx0, dy0, boundary, s);
        default: return fail(SKC_EBADARG, "channels must be 1..4");
    }
}

}  // namespace skc
