// smem_peak.cu -- measure the shared-memory load bandwidth of one B200
// (conflict-free LDS.128 and LDS.64 streams, all SMs), the roofline
// denominator SURVEY 8(d) asks to measure instead of assuming the nominal
// 148 SM x 128 B/clk.  Build and run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_peak tools/smem_peak.cu && /tmp/smem_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int VEC>
__global__ void __launch_bounds__(1024) smem_read(float *out, int iters) {
    __shared__ __align__(16) float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = (float)i;
    __syncthreads();
    float acc = 0.f;
    // each warp streams a private 2 KB window; lanes read consecutive vectors
    const int base = (threadIdx.x >> 5) * 512 + (threadIdx.x & 31) * VEC;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int idx = (base + k * 32 * VEC + it * VEC) & 8191 & ~(VEC - 1);
            if (VEC == 4) {
                const float4 v = *reinterpret_cast<const float4 *>(buf + idx);
                acc += v.x + v.y + v.z + v.w;
            } else if (VEC == 2) {
                const float2 v = *reinterpret_cast<const float2 *>(buf + idx);
                acc += v.x + v.y;
            } else {
                acc += buf[idx];
            }
        }
    }
    if (acc == 12345.f) out[threadIdx.x] = acc;
}

template <int VEC>
static double run(int sms) {
    float *out;
    cudaMalloc(&out, 4096);
    const int iters = 4096, blocks = sms * 2, threads = 1024;
    smem_read<VEC><<<blocks, threads>>>(out, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    smem_read<VEC><<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)blocks * threads * iters * 8 * VEC * 4;
    cudaFree(out);
    return bytes / (ms * 1e-3) / 1e9;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double v4 = run<4>(sms), v2 = run<2>(sms), v1 = run<1>(sms);
    printf("{\"sms\": %d, \"clock_khz\": %d, \"lds128_GBps\": %.1f, \"lds64_GBps\": %.1f, \"lds32_GBps\": %.1f, "
           "\"nominal_GBps\": %.1f}\n",
           sms, clk, v4, v2, v1, sms * 128.0 * clk * 1e3 / 1e9);
    return 0;
}
