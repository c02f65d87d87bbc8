// skc_api.cu -- error reporting, scratch pool and version for libskc.so.
#include <cstdint>
#include <string>

#include "skc_common.cuh"

namespace skc {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return SKC_ECUDA;
}

int pool_alloc(void **p, size_t bytes, cudaStream_t s) {
    static thread_local int configured_dev = -1;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (configured_dev != dev) {
        // keep freed blocks in the pool instead of returning them at every sync
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        configured_dev = dev;
    }
    e = cudaMallocAsync(p, bytes ? bytes : 16, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    return SKC_OK;
}

void pool_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

}  // namespace skc

extern "C" {

int skc_version(void) { return 100; }  // 0.1.0

const char *skc_last_error(void) { return skc::g_last_error.c_str(); }

}  // extern "C"
