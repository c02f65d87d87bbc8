// skc_pst.cu -- device-resident parallel simulated tempering (PST) for sm_100a.
//
// Reference: baselines.pst_fit (/root/reference/pkg/src/sparsekern/
// baselines.py:143-254) with its energy function energies_of (175-191) and
// swap sweep _attempt_swaps (132-140).  The reference runs the chain loop on
// the host: per iteration it draws Gaussian proposals for every chain,
// renormalises each layer's weights, synthesises all chains' impulse
// responses, applies Metropolis acceptance at the chain's ladder temperature,
// tracks the best state and every `swap_interval` iterations sweeps
// adjacent-pair exchanges.
//
// Here the whole run is resident on the device.  Per iteration three
// stream-ordered launches, with no host round trip:
//   pst_propose_kernel  one CTA per chain: noise (Philox, or a caller-supplied
//                       buffer in the reference's draw order), inactive-slot
//                       masking, per-layer sum normalisation (numpy's pairwise
//                       summation order, so proposals are bit-identical to the
//                       reference's when the noise is), fp32 tap table out;
//   fit_kernel          MODE_ENERGY (skc_fit.cu): every chain's impulse
//                       response, pixel-summed loss and the leak wall;
//   pst_accept_kernel   one CTA: Metropolis accept, state update, best
//                       tracking, the sequential swap sweep, the trace row and
//                       the iteration counter.
// The three launches of a block of iterations are captured once into a CUDA
// graph and the graph is replayed; kernels past the last iteration return
// early (the counter lives on the device).  The chain state is float64 like
// the reference's; only the energy evaluation is fp32 (skc_ir_energies).
#include <curand_kernel.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "skc_common.cuh"

namespace skc {

struct EnergyPlan;
int energy_plan_create(EnergyPlan **out, int B, const int *layout, int L, int nmax, int canvas,
                       const float *tgt, int M, int loss_kind, float loss_eps, const float *taps,
                       double *energies, cudaStream_t s);
int energy_plan_launch(const EnergyPlan *e, cudaStream_t s);
void energy_plan_destroy(EnergyPlan *e, cudaStream_t s);

namespace {

constexpr int kPstMaxL = 8;
constexpr int kProposeThreads = 128;
constexpr int kAcceptThreads = 256;
constexpr int kGraphIters = 32;   // iterations per captured graph

struct PstDev {
    int chains, L, nmax, iterations, swap_interval, sum_normalize, host_noise;
    int layout[kPstMaxL];
    double sigma_o, sigma_w;
    unsigned long long seed;
    int rec;                 // noise doubles per iteration (host-noise mode)
    const double *noise;     // (iterations, rec) or null
    double *off, *w;         // state (chains, L, nmax, 2) / (chains, L, nmax)
    double *poff, *pw;       // proposals, same shapes
    float *taps;             // proposal tap table (chains, L, nmax, 3) for fit_kernel
    int *bad;                // (chains) proposal failed sum normalisation
    double *energy, *eprop;  // (chains)
    const double *ladder;    // (chains)
    double *best_off, *best_w, *best_e;   // (L, nmax, 2), (L, nmax), (1)
    double *trace;           // (iterations, 2 + chains)
    long long *accepts;      // (chains) accepted proposals per ladder slot
    long long *swaps;        // (chains - 1) accepted exchanges per pair
    int *counter;            // iterations done
};

// numpy's pairwise summation (add.reduce over a contiguous axis): blocks of
// 8 partial sums up to 128 elements, recursive halving above.
__device__ double np_pairwise_sum(const double *a, int n) {
    // iterative form of the recursion: n <= 256 here (fit taps per layer)
    if (n > 128) {
        int n2 = n / 2;
        n2 -= n2 % 8;
        double lhs = 0.0, rhs = 0.0;
        {
            const double *b = a;
            int m = n2;
            // m <= 128 since n <= 256
            double r[8];
            for (int j = 0; j < 8; ++j) r[j] = b[j];
            int i = 8;
            for (; i < m - (m % 8); i += 8)
                for (int j = 0; j < 8; ++j) r[j] += b[i + j];
            lhs = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
            for (; i < m; ++i) lhs += b[i];
        }
        rhs = np_pairwise_sum(a + n2, n - n2);
        return lhs + rhs;
    }
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res += a[i];
        return res;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
}

// Philox stream id of one draw: iteration-major, then a slot within the
// iteration (proposal params, acceptance, swaps); each id is its own
// subsequence, so results do not depend on the launch geometry.
__device__ __forceinline__ curandStatePhilox4_32_10_t philox(const PstDev &d, int it, long long slot) {
    curandStatePhilox4_32_10_t st;
    const long long per_it = (long long)d.chains * d.L * d.nmax + 2LL * d.chains;
    curand_init(d.seed, (unsigned long long)((long long)it * per_it + slot), 0ULL, &st);
    return st;
}

__global__ void __launch_bounds__(kProposeThreads) pst_propose_kernel(const __grid_constant__ PstDev d) {
    const int it = *d.counter;
    if (it >= d.iterations) return;
    const int c = blockIdx.x;
    const int per = d.L * d.nmax;
    const double *off = d.off + (size_t)c * per * 2;
    const double *w = d.w + (size_t)c * per;
    double *poff = d.poff + (size_t)c * per * 2;
    double *pw = d.pw + (size_t)c * per;
    const double *nz = d.host_noise ? d.noise + (size_t)it * d.rec : nullptr;
    for (int q = threadIdx.x; q < per; q += blockDim.x) {
        const int l = q / d.nmax, i = q - l * d.nmax;
        double zx, zy, zw;
        if (nz) {
            // rng.normal(size=off.shape) then rng.normal(size=wts.shape)
            // (baselines.py:212-213): C-order (chains, L, nmax, 2) / (chains, L, nmax)
            zx = nz[((size_t)c * per + q) * 2];
            zy = nz[((size_t)c * per + q) * 2 + 1];
            zw = nz[(size_t)d.chains * per * 2 + (size_t)c * per + q];
        } else {
            curandStatePhilox4_32_10_t st = philox(d, it, (long long)c * per + q);
            const double2 z2 = curand_normal2_double(&st);
            zx = z2.x;
            zy = z2.y;
            zw = curand_normal_double(&st);
        }
        const bool act = i < d.layout[l];
        // normal(0, s) = 0 + s * standard_normal (numpy's Generator.normal),
        // each operation rounded separately (no FMA contraction), as numpy
        poff[2 * q] = act ? __dadd_rn(off[2 * q], __dadd_rn(0.0, __dmul_rn(d.sigma_o, zx))) : 0.0;
        poff[2 * q + 1] = act ? __dadd_rn(off[2 * q + 1], __dadd_rn(0.0, __dmul_rn(d.sigma_o, zy))) : 0.0;
        pw[q] = act ? __dadd_rn(w[q], __dadd_rn(0.0, __dmul_rn(d.sigma_w, zw))) : 0.0;
    }
    __syncthreads();
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    if (d.sum_normalize) {
        // baselines.py:216-220: per layer sum over all nmax slots (numpy
        // pairwise order); |sum| < 1e-8 leaves the layer as is and marks the
        // chain's proposal invalid
        __shared__ double s_sum[kPstMaxL];
        if (threadIdx.x < d.L) {
            const double sm = np_pairwise_sum(pw + threadIdx.x * d.nmax, d.nmax);
            s_sum[threadIdx.x] = sm;
            if (!(fabs(sm) >= 1e-8)) atomicOr(&s_bad, 1);
        }
        __syncthreads();
        for (int q = threadIdx.x; q < per; q += blockDim.x) {
            const double sm = s_sum[q / d.nmax];
            if (fabs(sm) >= 1e-8) pw[q] = __ddiv_rn(pw[q], sm);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) d.bad[c] = s_bad;
    float *t = d.taps + (size_t)c * per * 3;
    for (int q = threadIdx.x; q < per; q += blockDim.x) {
        t[3 * q] = (float)poff[2 * q];
        t[3 * q + 1] = (float)poff[2 * q + 1];
        t[3 * q + 2] = (float)pw[q];
    }
}

__device__ __forceinline__ double draw_uniform(const PstDev &d, int it, long long slot, size_t host_idx) {
    if (d.host_noise) return d.noise[(size_t)it * d.rec + host_idx];
    curandStatePhilox4_32_10_t st = philox(d, it, slot);
    // curand_uniform_double is in (0, 1]; 1 - u is in [0, 1) like numpy's
    return 1.0 - curand_uniform_double(&st);
}

__device__ void copy_rows(double *dst_o, double *dst_w, const double *src_o, const double *src_w, int per) {
    for (int q = threadIdx.x; q < per; q += blockDim.x) {
        dst_o[2 * q] = src_o[2 * q];
        dst_o[2 * q + 1] = src_o[2 * q + 1];
        dst_w[q] = src_w[q];
    }
}

__device__ void swap_rows(double *ao, double *aw, double *bo, double *bw, int per) {
    for (int q = threadIdx.x; q < per; q += blockDim.x) {
        double t = ao[2 * q]; ao[2 * q] = bo[2 * q]; bo[2 * q] = t;
        t = ao[2 * q + 1]; ao[2 * q + 1] = bo[2 * q + 1]; bo[2 * q + 1] = t;
        t = aw[q]; aw[q] = bw[q]; bw[q] = t;
    }
}

// Best-so-far: strictly lower minimum, first chain index on ties (argmin).
__device__ void update_best(const PstDev &d, int per) {
    __shared__ int s_k;
    if (threadIdx.x == 0) {
        int k = 0;
        double e = d.energy[0];
        for (int c = 1; c < d.chains; ++c)
            if (d.energy[c] < e || (isnan(e) && !isnan(d.energy[c]))) { e = d.energy[c]; k = c; }
        s_k = e < *d.best_e ? k : -1;
        if (s_k >= 0) *d.best_e = e;
    }
    __syncthreads();
    if (s_k >= 0) copy_rows(d.best_off, d.best_w, d.off + (size_t)s_k * per * 2, d.w + (size_t)s_k * per, per);
    __syncthreads();
}

__global__ void __launch_bounds__(kAcceptThreads) pst_accept_kernel(const __grid_constant__ PstDev d) {
    const int it = *d.counter;
    if (it >= d.iterations) return;
    const int per = d.L * d.nmax;
    const size_t prop_n = (size_t)d.chains * per * 3;
    __shared__ unsigned char s_acc[1024];
    for (int c = threadIdx.x; c < d.chains; c += blockDim.x) {
        // baselines.py:222-229
        const double enew = d.bad[c] ? INFINITY : d.eprop[c];
        const double de = enew - d.energy[c];
        const double u = draw_uniform(d, it, (long long)d.chains * per + c, prop_n + c);
        bool acc = (de <= 0.0) || (u < exp(-(de > 0.0 ? de : 0.0) / d.ladder[c]));
        acc = acc && isfinite(enew);
        s_acc[c] = acc;
        if (acc) {
            d.energy[c] = enew;
            d.accepts[c] += 1;
        }
    }
    __syncthreads();
    for (int c = 0; c < d.chains; ++c)
        if (s_acc[c])
            copy_rows(d.off + (size_t)c * per * 2, d.w + (size_t)c * per, d.poff + (size_t)c * per * 2,
                      d.pw + (size_t)c * per, per);
    __syncthreads();
    update_best(d, per);                         // baselines.py:231-236
    if ((it + 1) % d.swap_interval == 0) {       // baselines.py:237-238 -> 132-140
        __shared__ int s_sw;
        for (int c = 0; c + 1 < d.chains; ++c) {
            if (threadIdx.x == 0) {
                const double x = (1.0 / d.ladder[c] - 1.0 / d.ladder[c + 1]) * (d.energy[c] - d.energy[c + 1]);
                const double prob = x >= 0.0 ? 1.0 : exp(fmax(x, -745.0));
                const double u = draw_uniform(d, it, (long long)d.chains * per + d.chains + c,
                                              prop_n + d.chains + c);
                s_sw = u < prob;
                if (s_sw) {
                    const double t = d.energy[c];
                    d.energy[c] = d.energy[c + 1];
                    d.energy[c + 1] = t;
                    d.swaps[c] += 1;
                }
            }
            __syncthreads();
            if (s_sw)
                swap_rows(d.off + (size_t)c * per * 2, d.w + (size_t)c * per,
                          d.off + (size_t)(c + 1) * per * 2, d.w + (size_t)(c + 1) * per, per);
            __syncthreads();
        }
    }
    double *row = d.trace + (size_t)it * (2 + d.chains);
    for (int c = threadIdx.x; c < d.chains; c += blockDim.x) row[2 + c] = d.energy[c];
    if (threadIdx.x == 0) {
        row[0] = (double)it;
        row[1] = *d.best_e;
        *d.counter = it + 1;
    }
}

__global__ void pst_start_kernel(const __grid_constant__ PstDev d, const double *start) {
    // every chain starts from the init complex (baselines.py:157-166); the
    // initial energies are in d.energy already
    const int per = d.L * d.nmax;
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < d.chains * per; e += blockDim.x * gridDim.x) {
        const int q = e % per;
        d.off[2 * e] = start[3 * q];
        d.off[2 * e + 1] = start[3 * q + 1];
        d.w[e] = start[3 * q + 2];
        d.taps[3 * e] = (float)start[3 * q];
        d.taps[3 * e + 1] = (float)start[3 * q + 1];
        d.taps[3 * e + 2] = (float)start[3 * q + 2];
    }
}

__global__ void pst_init_best_kernel(const __grid_constant__ PstDev d) {
    const int per = d.L * d.nmax;
    if (threadIdx.x == 0) {
        *d.best_e = INFINITY;
        *d.counter = 0;
    }
    for (int c = threadIdx.x; c < d.chains; c += blockDim.x) {
        d.accepts[c] = 0;
        if (c + 1 < d.chains) d.swaps[c] = 0;
    }
    __syncthreads();
    // baselines.py:202-205: best = argmin of the initial energies (the
    // comparison against +inf keeps a finite minimum; an all-inf start keeps
    // chain 0's state, like the reference's argmin)
    __shared__ int s_k;
    if (threadIdx.x == 0) {
        int k = 0;
        double e = d.energy[0];
        for (int c = 1; c < d.chains; ++c)
            if (d.energy[c] < e) { e = d.energy[c]; k = c; }
        *d.best_e = e;
        s_k = k;
    }
    __syncthreads();
    copy_rows(d.best_off, d.best_w, d.off + (size_t)s_k * per * 2, d.w + (size_t)s_k * per, per);
}

}  // namespace
}  // namespace skc

using namespace skc;

extern "C" {

int skc_pst_run(const double *start_taps, const int *layout, int L, int nmax, int canvas, const float *tgt,
                int M, const skc_pst_cfg *cfg, const double *noise, double *ladder_out, double *trace,
                double *best_taps, double *best_energy, long long *accepts, long long *swaps, void *stream) {
    if (!cfg || !start_taps || !layout || !tgt || !ladder_out || !trace || !best_taps || !best_energy ||
        !accepts || !swaps)
        return fail(SKC_EBADARG, "null pointer");
    if (L < 1 || L > kPstMaxL) return fail(SKC_EBADARG, "PST supports 1..8 layers");
    if (cfg->chains < 2 || cfg->chains > 1024) return fail(SKC_EBADARG, "PST needs 2..1024 chains");
    if (cfg->iterations < 1) return fail(SKC_EBADARG, "PST needs >= 1 iteration");
    if (cfg->swap_interval < 1) return fail(SKC_EBADARG, "swap interval must be >= 1");
    if (!(cfg->sigma_offset >= 0) || !(cfg->sigma_weight >= 0)) return fail(SKC_EBADARG, "sigmas must be >= 0");
    for (int l = 0; l < L; ++l)
        if (layout[l] < 1 || layout[l] > nmax) return fail(SKC_EBADARG, "layout entries must be 1..nmax");
    cudaStream_t s = (cudaStream_t)stream;
    const int C = cfg->chains, per = L * nmax;
    PstDev d;
    std::memset(&d, 0, sizeof(d));
    d.chains = C;
    d.L = L;
    d.nmax = nmax;
    d.iterations = cfg->iterations;
    d.swap_interval = cfg->swap_interval;
    d.sum_normalize = cfg->sum_normalize;
    d.host_noise = noise != nullptr;
    for (int l = 0; l < L; ++l) d.layout[l] = layout[l];
    d.sigma_o = cfg->sigma_offset;
    d.sigma_w = cfg->sigma_weight;
    d.seed = cfg->seed;
    d.rec = C * per * 3 + C + (C - 1);
    d.noise = noise;

    // one pool block for the whole state
    const size_t nd = (size_t)C * per * 6 + 4 * (size_t)C + (size_t)per * 3 + 1;
    const size_t bytes = nd * sizeof(double) + (size_t)C * per * 3 * sizeof(float) + (size_t)C * sizeof(int) +
                         2 * (size_t)C * sizeof(long long) + 64;
    void *blk = nullptr;
    int rc = pool_alloc(&blk, bytes, s);
    if (rc) return rc;
    double *dp = (double *)blk;
    d.off = dp; dp += (size_t)C * per * 2;
    d.w = dp; dp += (size_t)C * per;
    d.poff = dp; dp += (size_t)C * per * 2;
    d.pw = dp; dp += (size_t)C * per;
    d.energy = dp; dp += C;
    d.eprop = dp; dp += C;
    double *lad = dp; dp += C;
    dp += C;   // pad
    d.best_off = dp; dp += (size_t)per * 2;
    d.best_w = dp; dp += per;
    d.best_e = dp; dp += 1;
    long long *lp = (long long *)dp;
    d.accepts = lp; lp += C;
    d.swaps = lp; lp += C;
    float *fp = (float *)lp;
    d.taps = fp; fp += (size_t)C * per * 3;
    d.bad = (int *)fp;
    d.ladder = lad;
    d.trace = trace;
    int *counter = nullptr;
    if ((rc = pool_alloc((void **)&counter, sizeof(int) * 4, s))) { pool_free(blk, s); return rc; }
    d.counter = counter;

    EnergyPlan *plan = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    auto cleanup = [&]() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        energy_plan_destroy(plan, s);
        pool_free(counter, s);
        pool_free(blk, s);
    };
    if ((rc = energy_plan_create(&plan, C, layout, L, nmax, canvas, tgt, M, cfg->loss_kind, cfg->loss_eps,
                                 d.taps, d.energy, s))) {
        plan = nullptr;
        cleanup();
        return rc;
    }
    // initial energies of the start state (baselines.py:194)
    pst_start_kernel<<<ceil_div(C * per, 256), 256, 0, s>>>(d, start_taps);
    if ((rc = energy_plan_launch(plan, s))) { cleanup(); return rc; }
    energy_plan_destroy(plan, s);
    plan = nullptr;
    // the temperature ladder needs the initial energy on the host (one sync
    // per run, like the reference's float(energies[0]), baselines.py:195-200)
    double e0 = 0.0;
    cudaError_t e = cudaMemcpyAsync(&e0, d.energy, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "skc_pst_run initial energy"); }
    const double scale = e0 > 0 ? e0 : 1.0;
    const double t_max = std::isnan(cfg->t_max) ? 1e-2 * scale : cfg->t_max;
    const double t_min = std::isnan(cfg->t_min) ? 1e-6 * scale : cfg->t_min;
    if (!(t_max >= t_min && t_min > 0)) {
        cleanup();
        return fail(SKC_EBADARG, "bad temperature ladder: t_max=" + std::to_string(t_max) +
                                     ", t_min=" + std::to_string(t_min));
    }
    std::vector<double> lh((size_t)C);
    if (t_max > t_min) {
        // _ladder (baselines.py:124-129): t_max * ratio ** (arange(C) / (C - 1))
        const double ratio = t_min / t_max;
        for (int c = 0; c < C; ++c) lh[c] = t_max * std::pow(ratio, (double)c / (double)(C - 1));
    } else {
        std::fill(lh.begin(), lh.end(), t_max);
    }
    std::memcpy(ladder_out, lh.data(), sizeof(double) * C);
    e = cudaMemcpyAsync(lad, lh.data(), sizeof(double) * C, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "skc_pst_run ladder"); }
    pst_init_best_kernel<<<1, kAcceptThreads, 0, s>>>(d);
    if ((rc = energy_plan_create(&plan, C, layout, L, nmax, canvas, tgt, M, cfg->loss_kind, cfg->loss_eps,
                                 d.taps, d.eprop, s))) {
        plan = nullptr;
        cleanup();
        return rc;
    }
    // capture kGraphIters iterations (or fewer for short runs) once, replay
    const int per_graph = std::min(kGraphIters, cfg->iterations);
    cudaStream_t cs = nullptr;
    e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "cudaStreamCreate"); }
    e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        for (int k = 0; k < per_graph && rc == SKC_OK; ++k) {
            pst_propose_kernel<<<C, kProposeThreads, 0, cs>>>(d);
            rc = energy_plan_launch(plan, cs);
            if (rc == SKC_OK) pst_accept_kernel<<<1, kAcceptThreads, 0, cs>>>(d);
        }
        cudaError_t e2 = cudaStreamEndCapture(cs, &graph);
        if (e == cudaSuccess) e = e2;
    }
    if (e == cudaSuccess && rc == SKC_OK) e = cudaGraphInstantiate(&exec, graph, 0);
    cudaStreamDestroy(cs);
    if (rc == SKC_OK && e != cudaSuccess) rc = cuda_fail(e, "PST graph capture");
    if (rc) { cleanup(); return rc; }
    const int launches = ceil_div(cfg->iterations, per_graph);
    for (int k = 0; k < launches; ++k) {
        e = cudaGraphLaunch(exec, s);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(e, "cudaGraphLaunch (PST)"); }
    }
    // results: best taps (L, nmax, 3) float64, best energy, counters
    std::vector<double> bo((size_t)per * 2), bw((size_t)per);
    e = cudaMemcpyAsync(bo.data(), d.best_off, sizeof(double) * per * 2, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bw.data(), d.best_w, sizeof(double) * per, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(best_energy, d.best_e, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(accepts, d.accepts, sizeof(long long) * C, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(swaps, d.swaps, sizeof(long long) * (C - 1), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cleanup();
    if (e != cudaSuccess) return cuda_fail(e, "skc_pst_run results");
    for (int q = 0; q < per; ++q) {
        best_taps[3 * q] = bo[2 * q];
        best_taps[3 * q + 1] = bo[2 * q + 1];
        best_taps[3 * q + 2] = bw[q];
    }
    return SKC_OK;
}

}  // extern "C"
