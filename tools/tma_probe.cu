// TMA bring-up probe: which tensor-map forms load without faulting on this
// driver/GPU (round-2 Kawase kernel bring-up).  One case per process run.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int RANK>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, int x, int y, int z, int w, unsigned bytes,
                      unsigned long long *out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
        if (RANK == 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(smem_u32(smem)), "l"(&tmap), "r"(x), "r"(y), "r"(smem_u32(&bar)) : "memory");
        else if (RANK == 3)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(smem_u32(smem)), "l"(&tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(smem_u32(smem)), "l"(&tmap), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(&bar)) : "memory");
        unsigned done = 0;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        } while (!done);
        unsigned long long s = 0;
        for (unsigned i = 0; i < bytes / 8; ++i) s += reinterpret_cast<unsigned long long *>(smem)[i];
        *out = s;
    }
}

int main(int argc, char **argv) {
    const int which = atoi(argv[1]);
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    EncodeTiledFn enc = (EncodeTiledFn)f;
    const int W = 256, H = 64, B = 2;
    void *buf;
    cudaMalloc(&buf, (size_t)W * H * B * 8);
    cudaMemset(buf, 1, (size_t)W * H * B * 8);
    unsigned long long *out;
    cudaMalloc(&out, 8);
    CUtensorMap map;
    memset(&map, 0, sizeof map);
    CUresult r = CUDA_SUCCESS;
    unsigned bytes = 0;
    int rank = 3, x = 0, y = 0, z = 0, w = 0;
    const CUtensorMapL2promotion l2 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (which == 0 || which == 1 || which == 2) {  // 3-D uint64 pixels, box 170 x 32 x 1
        cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
        cuuint64_t str[2] = {(cuuint64_t)W * 8, (cuuint64_t)W * H * 8};
        cuuint32_t box[3] = {which == 2 ? 128u : 170u, 32, 1}, es[3] = {1, 1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        bytes = box[0] * 32 * 8;
        x = which == 1 ? -21 : 0;
    } else if (which == 3 || which == 4) {  // 4-D fp16: (8 halves, W/2, H, B), box 8 x 85 x 32 x 1
        cuuint64_t dims[4] = {8, (cuuint64_t)W / 2, (cuuint64_t)H, (cuuint64_t)B};
        cuuint64_t str[3] = {16, (cuuint64_t)W * 8, (cuuint64_t)W * H * 8};
        cuuint32_t box[4] = {8, 85, 32, 1}, es[4] = {1, 1, 1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        bytes = 8 * 85 * 32 * 2;
        rank = 4;
        y = which == 4 ? -11 : 0;
    } else if (which == 5 || which == 6) {  // 3-D uint32 halves pairs: (2W, H, B) box 256 x 32 x 1 (uint32 = half2)
        cuuint64_t dims[3] = {(cuuint64_t)W * 2, (cuuint64_t)H, (cuuint64_t)B};
        cuuint64_t str[2] = {(cuuint64_t)W * 8, (cuuint64_t)W * H * 8};
        cuuint32_t box[3] = {256, 32, 1}, es[3] = {1, 1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        bytes = 256 * 32 * 4;
        x = which == 6 ? -42 : 0;
    } else if (which == 7) {  // 2-D float32 (W*2, H*B), box 64 x 32
        cuuint64_t dims[2] = {(cuuint64_t)W * 2, (cuuint64_t)H * B};
        cuuint64_t str[1] = {(cuuint64_t)W * 8};
        cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
        r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        bytes = 64 * 32 * 4;
        rank = 2;
    }
    printf("case %d: encode=%d ", which, (int)r);
    const int smem = 64 * 1024;
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (rank == 2) probe<2><<<1, 32, smem>>>(map, x, y, z, w, bytes, out);
    else if (rank == 3) probe<3><<<1, 32, smem>>>(map, x, y, z, w, bytes, out);
    else probe<4><<<1, 32, smem>>>(map, x, y, z, w, bytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("kernel=%s sum=%llx\n", cudaGetErrorName(e), h);
    return 0;
}
