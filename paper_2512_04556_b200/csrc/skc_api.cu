// skc_api.cu -- error reporting, scratch pool and version for libskc.so.
#include <cstdint>
#include <mutex>
#include <set>
#include <tuple>
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

// Scratch comes from a PRIVATE stream-ordered pool per device
// (cudaMemPoolCreate): the process-wide default pool and its release
// threshold stay untouched, and skc_release_scratch() hands the cached
// blocks back to the driver.
static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[64];

static cudaError_t device_pool(int dev, cudaMemPool_t *out) {
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool;
        cudaError_t e = cudaMemPoolCreate(&pool, &props);
        if (e != cudaSuccess) return e;
        // keep freed blocks cached between calls (steady-state calls do not hit
        // the driver allocator); skc_release_scratch() trims them
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        g_pools[dev] = pool;
    }
    *out = g_pools[dev];
    return cudaSuccess;
}

int pool_alloc(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    cudaMemPool_t pool;
    e = device_pool(dev, &pool);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemPoolCreate");
    e = cudaMallocFromPoolAsync(p, bytes ? bytes : 16, pool, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocFromPoolAsync");
    return SKC_OK;
}

void pool_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

int smem_optin(const void *fn, int bytes) {
    // cudaFuncSetAttribute is per device: remember (function, device, bytes)
    // so each device gets its own opt-in; failures are not remembered
    static std::mutex mu;
    static std::set<std::tuple<const void *, int, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const auto key = std::make_tuple(fn, dev, bytes);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (done.count(key)) return SKC_OK;
    }
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    std::lock_guard<std::mutex> lk(mu);
    done.insert(key);
    return SKC_OK;
}

int release_scratch() {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (int d = 0; d < 64; ++d) {
        if (!g_pools[d]) continue;
        cudaError_t e = cudaMemPoolTrimTo(g_pools[d], 0);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemPoolTrimTo");
    }
    return SKC_OK;
}

}  // namespace skc

extern "C" {

int skc_version(void) { return 200; }  // 0.2.0

int skc_release_scratch(void) { return skc::release_scratch(); }

const char *skc_last_error(void) { return skc::g_last_error.c_str(); }

}  // extern "C"
