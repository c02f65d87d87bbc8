/*
 * skc.h -- C ABI of libskc.so, the B200 (sm_100a) Sparse Kernel Complex hot path.
 *
 * Drop-in boundary for the reference `sparsekern` package
 * (/root/reference/pkg/src/sparsekern).  The reference switches its compiled
 * fast path in at call time through `_fastpath.HAVE_NUMBA`
 * (svfilter.py:18, svfilter.py:189-190, baselines.py:17, baselines.py:173);
 * paper_2512_04556_b200 does the same through `HAVE_CUDA`, and every entry
 * point below replaces the bottom of one reference call chain (cited per
 * function).  Binding recipe (ctypes) is in INTEGRATION.md.
 *
 * Conventions
 *   - plain C types only; images/maps/parameters live in device memory unless
 *     the argument is documented as a host array (small tap tables);
 *   - images are HWC interleaved (the reference's (H, W, C) layout,
 *     engine.py:133-136), batched as (B, H, W, C), contiguous;
 *   - every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream), re-entrant; scratch comes from a private per-device
 *     stream-ordered memory pool (skc_release_scratch), the only process
 *     state the library keeps besides its generated-kernel cache;
 *   - the return value is a status code; no C++ exception crosses the ABI;
 *     skc_last_error() returns a thread-local message for the last failure.
 */
#ifndef SKC_H
#define SKC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define SKC_OK 0
#define SKC_EBADARG 1      /* maps to EngineError / OptimError (argument)   */
#define SKC_ENONFINITE 2   /* maps to OptimError "non-finite intermediate"  */
#define SKC_ETRUNC 3       /* maps to TruncationError                        */
#define SKC_ECUDA 4        /* CUDA runtime failure; see skc_last_error()     */
#define SKC_EDEGENERATE 5  /* maps to OptimError "SUM normalization degenerate" */
#define SKC_ENOTTAKEN 6    /* a fused path does not apply: run the layers one by one */

/* storage dtypes (arithmetic is always fp32) */
#define SKC_F32 0
#define SKC_F16 1
#define SKC_F64 2          /* skc_bilinear_sample images only              */

/* boundary modes: ZERO = reference zero padding (engine.py:106-115);
 * CLAMP = clamp-to-edge (BASELINE config 0) */
#define SKC_ZERO 0
#define SKC_CLAMP 1

/* loss kinds (optim.py:59-68) and weight normalisations (optim.py:71-80) */
#define SKC_LOSS_CHARBONNIER 0
#define SKC_LOSS_L1 1
#define SKC_LOSS_L2 2
#define SKC_WN_NONE 0
#define SKC_WN_SUM 1
#define SKC_WN_SOFM 2

int skc_version(void);
const char *skc_last_error(void);

/* Scratch (chain ping-pong planes, fit arenas) comes from a private
 * stream-ordered memory pool per device that keeps freed blocks cached
 * between calls; this returns every cached block to the driver (call after
 * synchronising the streams that used the library).  No reference
 * counterpart: numpy frees its temporaries itself. */
int skc_release_scratch(void);

/* Upper bound on taps per layer accepted by the filter entry points. */
int skc_max_taps(void);

/*
 * One sparse layer, out[b,y,x,c] = sum_i w_i * bilinear(in[b], x+ox_i, y+oy_i)[c].
 * Replaces engine.apply_sparse_layer (engine.py:160-170) and its inner
 * sample_shifted/_accum_shift (engine.py:106-130).
 *   in/out : device, (B, H, W, C) of in_dtype / out_dtype
 *   taps   : HOST float64 array (S, 3) = (ox, oy, w) per tap
 */
int skc_layer_fwd(const void *in, int in_dtype, void *out, int out_dtype,
                  int B, int H, int W, int C,
                  const double *taps, int S, int boundary, void *stream);

/* memory layouts for skc_layer_fwd_ex: HWC interleaved (the reference's) or
 * planar CHW (the chain's internal intermediate layout: fp32, or fp16 in
 * fp16-storage chains, see skc_chain_mid_dtype) */
#define SKC_HWC 0
#define SKC_CHW 1

/*
 * skc_layer_fwd with explicit layouts: in/out each (B, H, W, C) HWC or
 * (B, C, H, W) planar.  Planar tensors are fp32, or fp16 with fp16 on the
 * other side too (at most skc_max_taps() taps).  This is the per-layer
 * step skc_chain_fwd runs (first layer HWC -> CHW, inner CHW -> CHW, last
 * CHW -> HWC), exposed so callers can drive/time layers individually.
 */
int skc_layer_fwd_ex(const void *in, int in_dtype, int in_layout, void *out, int out_dtype,
                     int out_layout, int B, int H, int W, int C,
                     const double *taps, int S, int boundary, void *stream);

/* 1 when skc_chain_fwd runs this complex as one fused launch (in = out
 * dtype, zero boundary), else 0: Kawase ladders (4 taps (+-r_l, +-r_l),
 * r_l = l + 1/2, equal weights per layer, L <= 6) on fp16 RGBA with even W
 * run the separable TMA-fed kernel of skc_kawase.cu (config 3); other small-
 * reach chains the opt-in fused tile kernel (SKC_FUSED=1). */
int skc_chain_is_fused(const double *taps, const int *layout, int L, int H, int W, int C,
                       int out_dtype);

/* The I/O passes skc_chain_fwd brackets a (non-fused) chain with: bit 0 set =
 * an HWC -> planar relayout before the first layer, bit 1 set = a planar ->
 * HWC relayout after the last layer (clear when the last layer writes HWC
 * itself through the cluster epilogue).  Negative on bad arguments. */
int skc_chain_relayouts(const double *taps, const int *layout, int L, int H, int W, int C,
                        int in_dtype, int boundary);

/* Which kernel family skc_layer_fwd(_ex) runs for this layer with the default
 * switches: *kind = 0 tap tile (*param = rows per thread KR), 1 dense stencil
 * (*param = D), 2 direct gather, 3 generated sparse stencil (*param = nonzero
 * positions; planar-input layers, see skc_sparse_compile_check).  Lets callers compute a launch's algorithmic
 * shared-memory traffic (bench roofline). */
int skc_layer_plan(const double *taps, int S, int H, int W, int C, int boundary, int *kind, int *param);

/* Layers with planar input (and, with SKC_SPARSE_HWC=1, HWC input) run a
 * sparse stencil generated for the layer (its merged positions unrolled, the
 * weights a kernel parameter) and compiled at run time with NVRTC
 * (skc_sparse.cu) when the cost model prefers it.  This compiles the kernel
 * such a layer would run, without a device: 0 = compiled, 1 = the layer does
 * not take that path, SKC_ECUDA = the run-time compiler is missing or rejected
 * it (skc_last_error).  Layouts are SKC_HWC / SKC_CHW. */
int skc_sparse_compile_check(const double *taps, int S, int in_dtype, int in_layout, int out_dtype, int out_layout);

/*
 * A chain's first two layers as ONE fused launch (engine.apply_complex,
 * engine.py:173-178, layers 0 and 1 without the materialised intermediate):
 * fp32 HWC (B, H, W, C) in -> fp32 planar (B, C, H, W) out, the output of
 * layer 1.  Layer 0's output lives only in shared memory; outside the image
 * it takes the boundary rule's value, as the reference's materialised image
 * would give.  With SKC_PAIR=1 (opt-in: measured slower than the two
 * unfused launches on config 1) skc_chain_fwd runs it for fp32
 * chains of >= 3 layers when both layers are stencil-type and the generated
 * kernel fits.  Returns SKC_OK, or SKC_ENOTTAKEN when the pair does not take this
 * path (the caller runs the layers one by one).  With in == NULL and out ==
 * NULL a plan query: SKC_OK = would run, SKC_ENOTTAKEN = would not.
 */
int skc_layer_pair_fwd(const void *in, void *out, int B, int H, int W, int C, const double *taps0, int S0,
                       const double *taps1, int S1, int boundary, void *stream);

/* Build check of the fused pair's generated kernel (no device needed):
 * SKC_OK = compiled, SKC_ENOTTAKEN = not eligible, SKC_ECUDA = NVRTC rejected it. */
int skc_pair_compile_check(const double *taps0, int S0, const double *taps1, int S1);

/* Generated stencils compile in the background by default: a layer whose
 * kernel is not ready yet runs on the tap / dense kernels (same result to
 * fp32 rounding, so the first calls on a new position pattern can differ from
 * later ones in the last bits).  mode 1 = compile synchronously on first use
 * (every call of a layer runs the same kernel; also SKC_JIT=sync), 0 = async
 * (default).  skc_jit_wait blocks until every pending compile finished. */
int skc_set_jit_mode(int mode);
int skc_jit_wait(void);

/* Dtype of skc_chain_fwd's planar intermediates for this chain: SKC_F16 when
 * in and out are both fp16 ("fp16 storage, fp32 accumulation": every layer
 * accumulates in fp32 and rounds once on store) and no layer exceeds
 * skc_max_taps(), else SKC_F32 (SKC_HALF_MID=0 forces fp32).  Lets callers
 * drive the chain's launches themselves.  Negative on bad arguments. */
int skc_chain_mid_dtype(const int *layout, int L, int in_dtype, int out_dtype);

/* Layout/dtype conversion HWC <-> planar (fp32, or fp16 <-> fp16): the chain's
 * bracketing passes. */
int skc_relayout(const void *in, int in_dtype, int in_layout, void *out, int out_dtype,
                 int out_layout, int B, int H, int W, int C, void *stream);

/*
 * A chain of L layers (engine.apply_complex, engine.py:173-178).  Intermediate
 * images stay in pool scratch, planar, in skc_chain_mid_dtype's dtype.
 *   taps   : HOST float64 (sum(layout), 3), layers concatenated in order
 *   layout : HOST int32 (L,) taps per layer
 */
int skc_chain_fwd(const void *in, int in_dtype, void *out, int out_dtype,
                  int B, int H, int W, int C,
                  const double *taps, const int *layout, int L, int boundary, void *stream);

/*
 * Spatially varying filtering (svfilter.sv_filter, svfilter.py:171-203 ->
 * _fastpath.sv_filter_compiled / _sv_pass_loop, _fastpath.py:97-150).
 *   pmap   : device float32 (H, W) per-pixel parameter
 *   params : HOST float64 (Mb,) strictly increasing basis parameters
 *   basis  : HOST float64 (Mb, L, nmax, 3) = (ox, oy, w), zero padded
 *            (svfilter._stacked_params, svfilter.py:155-168)
 *   layout : HOST int32 (L,)
 */
int skc_sv_fwd(const void *in, int in_dtype, void *out, int out_dtype,
               int H, int W, int C, const float *pmap,
               const double *params, int Mb, const double *basis, int nmax,
               const int *layout, int L, int boundary, void *stream);

/*
 * 2-D parameter SV filtering (svfilter.sv_filter_grid, svfilter.py:292-319):
 * a (Mu, Mv) grid of basis complexes, per-pixel bilinear blend of the four
 * bracketing entries' taps.  fp32 images only.
 *   pmap2  : device float32 (H, W, 2) = (u, v) per pixel
 *   basis  : HOST float64 (Mu, Mv, L, nmax, 3)
 */
int skc_sv_grid_fwd(const void *in, void *out, int H, int W, int C, const float *pmap2,
                    const double *params_u, int Mu, const double *params_v, int Mv,
                    const double *basis, int nmax, const int *layout, int L, int boundary,
                    void *stream);

/*
 * Batched impulse responses (engine.synthesize_ir / synthesize_ir_batch,
 * engine.py:191-209, 251-303; _fastpath.ir_batch_compiled, _fastpath.py:33-94).
 *   taps : device float32 (B, L, nmax, 3) = (ox, oy, w); zero weights inert
 *   out  : device float32 (B, canvas, canvas)
 *   layout : HOST int32 (L,)
 */
int skc_ir_batch(const float *taps, int B, const int *layout, int L, int nmax,
                 int canvas, float *out, void *stream);

/*
 * Energies of B complexes against ONE shared target for parallel tempering
 * (baselines.pst_fit -> energies_of, baselines.py:175-191, whose IRs come from
 * ir_batch_compiled, _fastpath.py:88-94): pixel-summed loss of each impulse
 * response (canvas^2) against the zero-embedded target, +inf where the
 * response's mass differs from prod_l sum_i w_li by > 1e-6*max(|.|,1) (the
 * "leak wall") or where an intermediate is non-finite.
 *   taps : device float32 (B, L, nmax, 3); tgt : device float32 (M, M)
 *   energies : device float64 (B,)
 */
int skc_ir_energies(const float *taps, int B, const int *layout, int L, int nmax, int canvas,
                    const float *tgt, int M, int loss_kind, float loss_eps, double *energies,
                    void *stream);

/* Parallel simulated tempering configuration (baselines.PSTConfig,
 * baselines.py:93-114).  t_max / t_min NaN = the reference defaults 1e-2 and
 * 1e-6 times the start state's energy (baselines.py:195-198). */
typedef struct skc_pst_cfg {
    int chains;               /* PSTConfig.chains (2..1024)                   */
    int iterations;           /* PSTConfig.iterations                         */
    int swap_interval;        /* PSTConfig.swap_interval                      */
    int sum_normalize;        /* PSTConfig.sum_normalize                      */
    double t_max, t_min;      /* ladder ends, NaN = default                   */
    double sigma_offset;      /* resolved PSTConfig.sigma_offset (px)         */
    double sigma_weight;      /* PSTConfig.sigma_weight                       */
    unsigned long long seed;  /* Philox key (PSTConfig.seed)                  */
    int loss_kind;            /* SKC_LOSS_*                                   */
    float loss_eps;           /* LossKind.epsilon                             */
} skc_pst_cfg;
/*
 * A whole PST run on the device (baselines.pst_fit, baselines.py:143-254):
 * per iteration Gaussian proposals for every chain, per-layer weight sum
 * normalisation, every chain's energy (as skc_ir_energies), Metropolis
 * acceptance at the chain's ladder temperature, best-state tracking and
 * every swap_interval iterations the adjacent-pair swap sweep
 * (baselines.py:132-140).  No host round trip per iteration: the loop is a
 * replayed CUDA graph; the host syncs once for the start energy (the ladder)
 * and once at the end.
 *   start_taps : device float64 (L, nmax, 3) init complex, zero padded
 *                (the chain state is float64 like the reference's)
 *   tgt        : device float32 (M, M) target; canvas odd >= M
 *   noise      : NULL = Philox(seed) draws; else device float64
 *                (iterations, chains*L*nmax*3 + 2*chains - 1) standard
 *                normals / uniforms in the reference's numpy draw order
 *                (offset normals (chains,L,nmax,2), weight normals
 *                (chains,L,nmax), acceptance uniforms (chains), swap
 *                uniforms (chains-1)), so a seeded reference run replays
 *   ladder_out : HOST float64 (chains) temperature ladder
 *   trace      : device float64 (iterations, 2 + chains) rows
 *                (iteration, best energy, chain energies)
 *   best_taps  : HOST float64 (L, nmax, 3); best_energy HOST float64 (1)
 *   accepts    : HOST int64 (chains) accepted proposals per ladder slot;
 *   swaps      : HOST int64 (chains - 1) accepted exchanges per pair
 */
int skc_pst_run(const double *start_taps, const int *layout, int L, int nmax, int canvas, const float *tgt,
                int M, const skc_pst_cfg *cfg, const double *noise, double *ladder_out, double *trace,
                double *best_taps, double *best_energy, long long *accepts, long long *swaps, void *stream);
/*
 * Per-element bilinear lookup with zero padding (engine.bilinear_sample,
 * engine.py:212-248).  img device (NB, H, W) SKC_F32 or SKC_F64; x, y device
 * float64 (n,) coordinates; element e samples image bidx[e] (device int64,
 * or NULL: e / inner, or image 0 when inner == 0); out device float64 (n,).
 * Float64 weights and corner order (0,0), (0,1), (1,0), (1,1) as the
 * reference, so float64 images reproduce its values.
 */
int skc_bilinear_sample(const void *img, int img_dtype, int NB, int H, int W, const double *x, const double *y,
                        const long long *bidx, long long n, long long inner, double *out, void *stream);
/*
 * Spatially varying dense ground truth (svfilter.sv_ground_truth,
 * svfilter.py:206-235): out[c, y, x] = sum_{u,v} img[c, u, v] *
 * K_k[r + y - u, r + x - v], k = kidx[y, x], zero padding.
 *   img / out : device float32 planar (C, H, W)
 *   kidx      : device int32 (H, W) kernel index per pixel
 *   kernels   : device float32 (K, M, M), M odd, each centred (zero padded)
 */
int skc_sv_ground_truth(const float *img, int H, int W, int C, const int *kidx, const float *kernels, int K,
                        int M, float *out, void *stream);
/* Fit configuration (optim.TrainConfig, ConstraintConfig, LossKind). */
typedef struct skc_fit_cfg {
    int steps;            /* TrainConfig.steps                          */
    float lr_start;       /* TrainConfig.lr_start                       */
    float lr_end;         /* TrainConfig.lr_end                         */
    float beta1, beta2, eps;
    int weight_norm;      /* SKC_WN_*                                   */
    int kws;              /* ConstraintConfig.symmetry == "kws"         */
    int loss_kind;        /* SKC_LOSS_*                                 */
    float loss_eps;       /* LossKind.epsilon                           */
} skc_fit_cfg;

/*
 * Loss and gradients of B independent complexes (optim.backward,
 * optim.py:278-292 -> _forward_ir 204-222, _loss_value/_loss_grad 133-146,
 * _backward_pass 231-263), each against its own target embedded in `canvas`.
 *   taps    : device float32 (B, L, nmax, 3), effective weights
 *   tgts    : device float32 (B, M, M), M odd, M <= canvas
 *   loss    : device float32 (B,)
 *   grads   : device float32 (B, L, nmax, 3) = (d_ox, d_oy, d_w)
 *   status  : device int32 (B, 4) = (code, layer, sample, 0)
 */
int skc_backward_batch(const float *taps, int B, const int *layout, int L, int nmax,
                       const float *tgts, int M, int canvas, int loss_kind, float loss_eps,
                       float *loss, float *grads, int *status, void *stream);

/*
 * Persistent batched fitting (optim.fit, optim.py:390-469 with an explicit
 * KernelComplex init, optim.py:404-405): one CTA owns one target kernel and
 * runs every step on device -- forward on the impulse, loss, backward, Adam
 * (optim.py:338-369) with the offset learning-rate scale M (optim.py:411),
 * KWS/SUM projections (312-335), best-so-far tracking (442-445) and the
 * canvas growth rule (429-434).
 *   state  : device float32 (B, SKC_FIT_STATE_FLOATS(L, nmax)); initialise
 *            with skc_fit_init, read back with the SKC_FIT_OFF_* accessors
 *   tgts   : device float32 (B, M, M)
 *   trace  : device float32 (B, steps + 1) per-step loss
 *   status : device int32 (B, 4) = (code, layer, sample, step)
 * Returns SKC_OK when every kernel finished; per-kernel failures are in
 * status (code SKC_ENONFINITE / SKC_EDEGENERATE).
 */
#define SKC_FIT_HDR 8
#define SKC_FIT_STATE_FLOATS(L, nmax) (SKC_FIT_HDR + 6 * (L) * (nmax) * 3)
/* state layout (floats): hdr[0]=step done, hdr[1]=canvas, hdr[2]=best loss,
 * hdr[3]=best step; then params, adam m, adam v, best params, scratch, scratch
 * each (L, nmax, 3) = (ox, oy, wparam). */
int skc_fit_init(float *state, const float *init_taps, int B, const int *layout, int L,
                 int nmax, int M, const skc_fit_cfg *cfg, int *status, void *stream);
int skc_fit_run(float *state, int B, const int *layout, int L, int nmax,
                const float *tgts, int M, const skc_fit_cfg *cfg,
                float *trace, int *status, void *stream);

/*
 * One Adam update with projections (optim.adam_step, optim.py:338-369) on
 * device arrays of one complex: params/grads/m/v float32 (P, 3) rows
 * (ox, oy, wparam), P = sum(layout).  status int32 (4,).
 */
int skc_adam_step(float *params, const float *grads, float *m, float *v, const int *layout,
                  int L, int step_index, const skc_fit_cfg *cfg, float offset_lr_scale,
                  int *status, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SKC_H */
