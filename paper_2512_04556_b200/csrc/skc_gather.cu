// skc_gather.cu -- per-element bilinear lookup and the spatially varying
// dense ground truth, for sm_100a.
//
// Reference (citations into /root/reference/pkg/src/sparsekern):
//   bilinear_sample (engine.py:212-248): per-element fractional coordinates,
//     batched leading dims, zero padding; corners accumulated in the order
//     (dy, dx) = (0,0), (0,1), (1,0), (1,1) with weights
//     (1-fx)(1-fy), fx(1-fy), (1-fx)fy, fx fy.
//   sv_ground_truth (svfilter.py:206-235): at every pixel the dense kernel of
//     target_family(pmap[y, x]) applied as a zero-padded convolution,
//     out[y, x] = sum_{u, v} img[u, v] * k[r + y - u, r + x - v].
//
// bilinear_sample is a pure gather (HBM / L2 bound): one thread per output
// element, float64 coordinates and weights, image in float32 or float64.
// sv_ground_truth is the brute-force quality oracle: the host evaluates the
// family once per distinct map value and uploads the kernels (K, Mk, Mk) plus
// a per-pixel kernel index; one CTA computes a 32 x 8 output tile of one
// channel from a shared-memory copy of the tile plus its radius-r halo,
// accumulating each kernel row in fp32 and the rows in fp64.
#include <cmath>

#include "skc_common.cuh"

namespace skc {
namespace {

template <typename T>
__global__ void bilinear_sample_kernel(const T *__restrict__ img, int H, int W, const double *__restrict__ xs,
                                       const double *__restrict__ ys, const long long *__restrict__ bidx,
                                       long long n, long long inner, double *__restrict__ out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = bidx ? bidx[e] : (inner > 0 ? e / inner : 0);
        const T *im = img + (size_t)b * H * W;
        const double x = xs[e], y = ys[e];
        const double x0 = floor(x), y0 = floor(y);
        const double fx = x - x0, fy = y - y0;
        double acc = 0.0;
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                const double wgt = __dmul_rn(dx ? fx : 1.0 - fx, dy ? fy : 1.0 - fy);
                // NaN / huge coordinates fall outside like the reference's
                // validity mask (the corner is treated as zero padding)
                const double xi = x0 + dx, yi = y0 + dy;
                double v = 0.0;
                if (xi >= 0.0 && xi < (double)W && yi >= 0.0 && yi < (double)H)
                    v = (double)im[(size_t)yi * W + (size_t)xi];
                acc = __dadd_rn(acc, __dmul_rn(wgt, v));
            }
        out[e] = acc;
    }
}

constexpr int kGtTx = 32, kGtTy = 8;

// One CTA = a 32 x 8 tile of one channel.  img planar fp32 (C, H, W),
// kidx (H, W) int32, kern (K, M, M) fp32, out planar (C, H, W) fp32.
__global__ void __launch_bounds__(kGtTx * kGtTy) sv_gt_kernel(const float *__restrict__ img, int H, int W,
                                                              const int *__restrict__ kidx,
                                                              const float *__restrict__ kern, int M,
                                                              float *__restrict__ out, int use_smem) {
    extern __shared__ float tile[];
    const int r = M / 2;
    const int c = blockIdx.z;
    const int tx0 = blockIdx.x * kGtTx, ty0 = blockIdx.y * kGtTy;
    const float *plane = img + (size_t)c * H * W;
    const int tw = kGtTx + 2 * r, th = kGtTy + 2 * r;
    if (use_smem) {
        for (int e = threadIdx.x; e < tw * th; e += blockDim.x) {
            const int yy = e / tw, xx = e - yy * tw;
            const int gy = ty0 - r + yy, gx = tx0 - r + xx;
            tile[e] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? __ldg(plane + (size_t)gy * W + gx) : 0.f;
        }
        __syncthreads();
    }
    const int lx = threadIdx.x % kGtTx, ly = threadIdx.x / kGtTx;
    const int x = tx0 + lx, y = ty0 + ly;
    if (x >= W || y >= H) return;
    const float *k = kern + (size_t)__ldg(kidx + (size_t)y * W + x) * M * M;
    double acc = 0.0;
    // out[y, x] = sum_{dy, dx} k[r + dy][r + dx] * img[y - dy][x - dx]
    for (int a = 0; a < M; ++a) {          // a = r + dy
        const int dy = a - r;
        float row = 0.f;
        if (use_smem) {
            const float *src = tile + (size_t)(ly + r - dy) * tw + (lx + r);
            const float *kr = k + (size_t)a * M;
            for (int b = 0; b < M; ++b) row = fmaf(__ldg(kr + b), src[r - b], row);
        } else {
            const int yy = y - dy;
            if (yy < 0 || yy >= H) continue;
            const float *src = plane + (size_t)yy * W;
            const float *kr = k + (size_t)a * M;
            for (int b = 0; b < M; ++b) {
                const int xx = x - (b - r);
                if (xx >= 0 && xx < W) row = fmaf(__ldg(kr + b), __ldg(src + xx), row);
            }
        }
        acc += (double)row;
    }
    out[(size_t)c * H * W + (size_t)y * W + x] = (float)acc;
}

}  // namespace
}  // namespace skc

using namespace skc;

extern "C" {

int skc_bilinear_sample(const void *img, int img_dtype, int NB, int H, int W, const double *x, const double *y,
                        const long long *bidx, long long n, long long inner, double *out, void *stream) {
    if (n < 0 || NB < 1 || H < 1 || W < 1) return fail(SKC_EBADARG, "bad sizes");
    if (n == 0) return SKC_OK;
    if (!img || !x || !y || !out) return fail(SKC_EBADARG, "null pointer");
    if (img_dtype != SKC_F32 && img_dtype != SKC_F64) return fail(SKC_EBADARG, "image must be fp32 or fp64");
    cudaStream_t s = (cudaStream_t)stream;
    const int threads = 256;
    const long long blocks = std::min<long long>((n + threads - 1) / threads, 148LL * 16);
    if (img_dtype == SKC_F32)
        bilinear_sample_kernel<float><<<(int)blocks, threads, 0, s>>>((const float *)img, H, W, x, y, bidx, n,
                                                                    inner, out);
    else
        bilinear_sample_kernel<double><<<(int)blocks, threads, 0, s>>>((const double *)img, H, W, x, y, bidx, n,
                                                                     inner, out);
    SKC_LAUNCH_CHECK("bilinear_sample_kernel");
    return SKC_OK;
}

int skc_sv_ground_truth(const float *img, int H, int W, int C, const int *kidx, const float *kernels, int K,
                        int M, float *out, void *stream) {
    if (H < 1 || W < 1 || C < 1 || K < 1 || M < 1 || (M & 1) == 0)
        return fail(SKC_EBADARG, "bad sizes (kernel size must be odd)");
    if (!img || !kidx || !kernels || !out) return fail(SKC_EBADARG, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const int r = M / 2;
    const size_t smem = (size_t)(kGtTx + 2 * r) * (kGtTy + 2 * r) * sizeof(float);
    int use_smem = smem <= 200 * 1024;
    if (use_smem) {
        int rc = smem_optin((const void *)sv_gt_kernel, (int)smem);
        if (rc) return rc;
    }
    dim3 grid(ceil_div(W, kGtTx), ceil_div(H, kGtTy), C);
    sv_gt_kernel<<<grid, kGtTx * kGtTy, use_smem ? smem : 0, s>>>(img, H, W, kidx, kernels, M, out, use_smem);
    SKC_LAUNCH_CHECK("sv_gt_kernel");
    return SKC_OK;
}

}  // extern "C"
