// skc_common.cuh -- shared helpers for the sm_100a Sparse Kernel Complex library.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/skc.h"

namespace skc {

// ---------------------------------------------------------------- errors ---
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define SKC_CUDA(call)                                   \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

#define SKC_LAUNCH_CHECK(what)                             \
    do {                                                   \
        cudaError_t _e = cudaGetLastError();               \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

// ------------------------------------------------- stream-ordered scratch ---
// Scratch comes from a private per-device pool (skc_api.cu); the pool keeps
// freed blocks cached so steady-state calls do not hit the driver allocator.
int pool_alloc(void **p, size_t bytes, cudaStream_t s);
void pool_free(void *p, cudaStream_t s);
int release_scratch();

// Opt a kernel into `bytes` of dynamic shared memory on the current device
// (remembered per function and device; a failure is reported, not cached).
int smem_optin(const void *fn, int bytes);

// ----------------------------------------------------- dtype conversions ---
template <typename T> struct IO;
template <> struct IO<float> {
    static __device__ __forceinline__ float ld(const float *p) { return __ldg(p); }
    static __device__ __forceinline__ void st(float *p, float v) { *p = v; }
};
template <> struct IO<__half> {
    static __device__ __forceinline__ float ld(const __half *p) { return __half2float(__ldg(p)); }
    static __device__ __forceinline__ void st(__half *p, float v) { *p = __float2half_rn(v); }
};

__host__ __device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

inline size_t dtype_size(int dt) { return dt == SKC_F16 ? 2 : 4; }

}  // namespace skc
