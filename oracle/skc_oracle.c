/*
 * skc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU float64 restatement of the reference `sparsekern` hot path
 * (/root/reference/pkg/src/sparsekern).  This file is the parity checker for
 * the CUDA product path and the CPU baseline timed by bench.py; it is never
 * linked into, called by, or shipped with the product library (libskc.so).
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load it.
 *
 * Each function cites the reference file:line it restates.  Summation order
 * follows the reference wherever the reference order is numpy-elementwise
 * (filter, IR synthesis, adjoint), so with -ffp-contract=off the forward
 * filter results are bit-identical to the reference (pinned by
 * tests/test_oracle.py against the npz fixtures under tests/golden made by the reference).
 * Dot products (np.vdot -> BLAS ddot) and numpy pairwise sums are restated as
 * plain sequential sums; they agree with the reference to ~1e-15 relative.
 *
 * Build: see oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_ZERO 0
#define OR_CLAMP 1

static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Per-tap bilinear corner table, engine.py:118-130 (sample_shifted):
 * ix = floor(ox), fx = ox - ix; corner order 00, 10, 01, 11 with weights
 * w(1-fx)(1-fy), w fx (1-fy), w (1-fx) fy, w fx fy (left-to-right products). */
typedef struct {
    int64_t ix, iy;
    double cw[4];
} or_tap;

static void make_taps(const double *off, const double *w, int64_t S, or_tap *t) {
    for (int64_t i = 0; i < S; ++i) {
        double ox = off[2 * i], oy = off[2 * i + 1];
        double fx0 = floor(ox), fy0 = floor(oy);
        double fx = ox - fx0, fy = oy - fy0;
        t[i].ix = (int64_t)fx0;
        t[i].iy = (int64_t)fy0;
        t[i].cw[0] = w[i] * (1.0 - fx) * (1.0 - fy);
        t[i].cw[1] = w[i] * fx * (1.0 - fy);
        t[i].cw[2] = w[i] * (1.0 - fx) * fy;
        t[i].cw[3] = w[i] * fx * fy;
    }
}

/* engine.py:160-170 apply_sparse_layer (+ _accum_shift 106-115, _per_channel
 * 133-136).  The reference accumulates tap-by-tap, corner-by-corner into a
 * zeroed plane, skipping zero corner weights (engine.py:108) and reads outside
 * the image (zero padding).  Per output pixel that is exactly the sequence
 * below, so the pixel-outer loop is bit-identical.  boundary=OR_CLAMP is the
 * BASELINE config-0 edge mode: the per-layer edge-pad wrapper
 * around the reference is equivalent to clamping every corner read. */
void or_apply_layer(const double *in, double *out, int64_t H, int64_t W, int64_t C,
                    const double *off, const double *w, int64_t S, int boundary) {
    or_tap *t = (or_tap *)malloc(sizeof(or_tap) * (size_t)(S > 0 ? S : 1));
    make_taps(off, w, S, t);
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < H; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            for (int64_t c = 0; c < C; ++c) {
                double acc = 0.0;
                for (int64_t i = 0; i < S; ++i) {
                    for (int k = 0; k < 4; ++k) {
                        double cw = t[i].cw[k];
                        if (cw == 0.0) continue;
                        int64_t yy = y + t[i].iy + (k >> 1);
                        int64_t xx = x + t[i].ix + (k & 1);
                        if (boundary == OR_CLAMP) {
                            yy = clampi(yy, 0, H - 1);
                            xx = clampi(xx, 0, W - 1);
                        } else if (yy < 0 || yy >= H || xx < 0 || xx >= W) {
                            continue;
                        }
                        acc += cw * in[(yy * W + xx) * C + c];
                    }
                }
                out[(y * W + x) * C + c] = acc;
            }
        }
    }
    free(t);
}

/* engine.py:173-178 apply_complex: layers in order.  taps for layer l start at
 * off + 2*sum(layout[:l]), w + sum(layout[:l]). */
void or_apply_complex(const double *in, double *out, int64_t H, int64_t W, int64_t C,
                      const double *off, const double *w, const int64_t *layout, int64_t L,
                      int boundary) {
    size_t n = (size_t)(H * W * C);
    double *a = (double *)malloc(sizeof(double) * (n ? n : 1));
    double *b = (double *)malloc(sizeof(double) * (n ? n : 1));
    memcpy(a, in, sizeof(double) * n);
    int64_t base = 0;
    for (int64_t l = 0; l < L; ++l) {
        or_apply_layer(a, b, H, W, C, off + 2 * base, w + base, layout[l], boundary);
        double *tmp = a; a = b; b = tmp;
        base += layout[l];
    }
    memcpy(out, a, sizeof(double) * n);
    free(a);
    free(b);
}

/* engine.py:191-209 synthesize_ir (canvas validation is host logic): apply the
 * complex to a centred delta on an odd canvas, zero padding.  Batched over B
 * complexes sharing one layout (engine.py:251-303 / _fastpath.py:33-94 give
 * identical values to 1e-15). */
void or_ir_batch(const double *off, const double *w, const int64_t *layout, int64_t L,
                 int64_t B, int64_t nmax, int64_t canvas, double *out) {
    int64_t n = canvas * canvas;
    for (int64_t b = 0; b < B; ++b) {
        double *a = (double *)calloc((size_t)n, sizeof(double));
        double *t = (double *)malloc(sizeof(double) * (size_t)n);
        a[(canvas / 2) * canvas + canvas / 2] = 1.0;
        for (int64_t l = 0; l < L; ++l) {
            const double *lo = off + ((b * L + l) * nmax) * 2;
            const double *lw = w + (b * L + l) * nmax;
            or_apply_layer(a, t, canvas, canvas, 1, lo, lw, layout[l], OR_ZERO);
            double *s = a; a = t; t = s;
        }
        memcpy(out + b * n, a, sizeof(double) * (size_t)n);
        free(a);
        free(t);
    }
}

/* svfilter.py:129-137 _bracket: clamp p into [p0, pM], k0 = searchsorted
 * (side=right) - 1 clipped to [0, Mb-2], t = (pc - p[k0]) / (p[k0+1] - p[k0]);
 * Mb == 1 gives k0 = k1 = 0, t = 0. */
static void bracket(double p, const double *ps, int64_t Mb, int64_t *k0, double *t) {
    if (Mb == 1) { *k0 = 0; *t = 0.0; return; }
    double pc = p < ps[0] ? ps[0] : (p > ps[Mb - 1] ? ps[Mb - 1] : p);
    int64_t r = 0;
    while (r < Mb && ps[r] <= pc) ++r;      /* searchsorted(side="right") */
    int64_t k = r - 1;
    if (k < 0) k = 0;
    if (k > Mb - 2) k = Mb - 2;
    *k0 = k;
    *t = (pc - ps[k]) / (ps[k + 1] - ps[k]);
}

/* svfilter.py:171-203 sv_filter -> _fastpath.py:97-150 (_sv_pass_loop).
 * basis: (Mb, L, nmax, 3) = (ox, oy, w), zero-padded per _stacked_params
 * (svfilter.py:155-168).  Per pixel and tap: lerp offsets and weight between
 * the bracketing entries, bilinear read of the previous pass at absolute
 * coordinates with per-corner bounds checks (zero) or clamped reads (clamp).
 * Channels are independent (svfilter.py:180-183). */
void or_sv_filter(const double *img, double *out, int64_t H, int64_t W, int64_t C,
                  const double *pmap, const double *ps, int64_t Mb, const double *basis,
                  const int64_t *layout, int64_t L, int64_t nmax, int boundary) {
    int64_t np_ = H * W;
    int64_t *k0 = (int64_t *)malloc(sizeof(int64_t) * (size_t)np_);
    double *tt = (double *)malloc(sizeof(double) * (size_t)np_);
    for (int64_t i = 0; i < np_; ++i) bracket(pmap[i], ps, Mb, &k0[i], &tt[i]);
    double *cur = (double *)malloc(sizeof(double) * (size_t)np_);
    double *nxt = (double *)malloc(sizeof(double) * (size_t)np_);
    for (int64_t c = 0; c < C; ++c) {
        for (int64_t i = 0; i < np_; ++i) cur[i] = img[i * C + c];
        for (int64_t l = 0; l < L; ++l) {
            int64_t n = layout[l];
#pragma omp parallel for schedule(static)
            for (int64_t y = 0; y < H; ++y) {
                for (int64_t x = 0; x < W; ++x) {
                    int64_t kk0 = k0[y * W + x];
                    int64_t kk1 = (Mb == 1) ? 0 : kk0 + 1;
                    double t = tt[y * W + x];
                    double acc = 0.0;
                    for (int64_t i = 0; i < n; ++i) {
                        const double *b0 = basis + ((kk0 * L + l) * nmax + i) * 3;
                        const double *b1 = basis + ((kk1 * L + l) * nmax + i) * 3;
                        double ox = (1.0 - t) * b0[0] + t * b1[0];
                        double oy = (1.0 - t) * b0[1] + t * b1[1];
                        double wt = (1.0 - t) * b0[2] + t * b1[2];
                        double sx = (double)x + ox, sy = (double)y + oy;
                        double fx0 = floor(sx), fy0 = floor(sy);
                        int64_t x0 = (int64_t)fx0, y0 = (int64_t)fy0;
                        double fx = sx - fx0, fy = sy - fy0;
                        double val = 0.0;
                        if (boundary == OR_CLAMP) {
                            int64_t ya = clampi(y0, 0, H - 1), yb = clampi(y0 + 1, 0, H - 1);
                            int64_t xa = clampi(x0, 0, W - 1), xb = clampi(x0 + 1, 0, W - 1);
                            val += (1.0 - fx) * (1.0 - fy) * cur[ya * W + xa];
                            val += fx * (1.0 - fy) * cur[ya * W + xb];
                            val += (1.0 - fx) * fy * cur[yb * W + xa];
                            val += fx * fy * cur[yb * W + xb];
                        } else {
                            if (0 <= y0 && y0 < H) {
                                if (0 <= x0 && x0 < W) val += (1.0 - fx) * (1.0 - fy) * cur[y0 * W + x0];
                                if (0 <= x0 + 1 && x0 + 1 < W) val += fx * (1.0 - fy) * cur[y0 * W + x0 + 1];
                            }
                            if (0 <= y0 + 1 && y0 + 1 < H) {
                                if (0 <= x0 && x0 < W) val += (1.0 - fx) * fy * cur[(y0 + 1) * W + x0];
                                if (0 <= x0 + 1 && x0 + 1 < W) val += fx * fy * cur[(y0 + 1) * W + x0 + 1];
                            }
                        }
                        acc += wt * val;
                    }
                    nxt[y * W + x] = acc;
                }
            }
            double *s = cur; cur = nxt; nxt = s;
        }
        for (int64_t i = 0; i < np_; ++i) out[i * C + c] = cur[i];
    }
    free(k0); free(tt); free(cur); free(nxt);
}

/* ------------------------------------------------------------------------ */
/* Fitting: optim.py                                                         */

#define LOSS_CHARB 0
#define LOSS_L1 1
#define LOSS_L2 2
#define WN_NONE 0
#define WN_SUM 1
#define WN_SOFM 2

/* optim.py:133-146 */
static double loss_term(double d, int kind, double eps) {
    if (kind == LOSS_CHARB) return sqrt(d * d + eps * eps);
    if (kind == LOSS_L1) return fabs(d);
    return d * d;
}
static double loss_grad(double d, int kind, double eps) {
    if (kind == LOSS_CHARB) return d / sqrt(d * d + eps * eps);
    if (kind == LOSS_L1) return (d > 0) ? 1.0 : ((d < 0) ? -1.0 : 0.0);
    return 2.0 * d;
}

/* sample_shifted(img, ox, oy, w, out) on a single plane (engine.py:118-130). */
static void sample_shifted_plane(const double *img, double *out, int64_t n,
                                 double ox, double oy, double w) {
    double fx0 = floor(ox), fy0 = floor(oy);
    double fx = ox - fx0, fy = oy - fy0;
    int64_t ix = (int64_t)fx0, iy = (int64_t)fy0;
    double cw[4] = {w * (1.0 - fx) * (1.0 - fy), w * fx * (1.0 - fy),
                    w * (1.0 - fx) * fy, w * fx * fy};
    for (int k = 0; k < 4; ++k) {
        if (cw[k] == 0.0) continue;
        int64_t a = ix + (k & 1), b = iy + (k >> 1);
        int64_t y0 = b < 0 ? -b : 0, y1 = n - b < n ? n - b : n;
        int64_t x0 = a < 0 ? -a : 0, x1 = n - a < n ? n - a : n;
        if (y1 <= y0 || x1 <= x0) continue;
        for (int64_t y = y0; y < y1; ++y)
            for (int64_t x = x0; x < x1; ++x)
                out[y * n + x] += cw[k] * img[(y + b) * n + (x + a)];
    }
}

/* optim.py:159-165 */
static void softmax(const double *z, double *e, int64_t n) {
    double m = z[0];
    for (int64_t i = 1; i < n; ++i) if (z[i] > m) m = z[i];
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) { e[i] = exp(z[i] - m); s += e[i]; }
    for (int64_t i = 0; i < n; ++i) e[i] = e[i] / s;
}

/* Parameters: off (P,2) and wp (P,) flattened over layers by layout. */
static void effective_weights(const double *wp, double *w, const int64_t *layout, int64_t L,
                              int wn) {
    int64_t base = 0;
    for (int64_t l = 0; l < L; ++l) {
        if (wn == WN_SOFM) softmax(wp + base, w + base, layout[l]);
        else memcpy(w + base, wp + base, sizeof(double) * (size_t)layout[l]);
        base += layout[l];
    }
}

/* optim.py:204-222 _forward_ir.  inter: (L+1) planes of canvas^2.  Returns -1
 * on success, else the failing layer index; *bad_sample gets the first tap
 * with a non-finite parameter (optim.py:225-228) or -1. */
static int64_t forward_ir(const double *off, const double *w, const int64_t *layout, int64_t L,
                          int64_t canvas, double *inter, int64_t *bad_sample) {
    int64_t n = canvas * canvas;
    memset(inter, 0, sizeof(double) * (size_t)n);
    inter[(canvas / 2) * canvas + canvas / 2] = 1.0;
    int64_t base = 0;
    for (int64_t l = 0; l < L; ++l) {
        double *prev = inter + l * n, *nxt = inter + (l + 1) * n;
        memset(nxt, 0, sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < layout[l]; ++i)
            sample_shifted_plane(prev, nxt, canvas, off[2 * (base + i)], off[2 * (base + i) + 1],
                                 w[base + i]);
        for (int64_t p = 0; p < n; ++p) {
            if (!isfinite(nxt[p])) {
                *bad_sample = -1;
                for (int64_t i = 0; i < layout[l]; ++i) {
                    if (!(isfinite(off[2 * (base + i)]) && isfinite(off[2 * (base + i) + 1]) &&
                          isfinite(w[base + i]))) { *bad_sample = i; break; }
                }
                return l;
            }
        }
        base += layout[l];
    }
    return -1;
}

/* optim.py:231-263 _backward_pass. g (canvas^2) is consumed. d_off (P,2), d_w (P,). */
static void backward_pass(const double *off, const double *w, const int64_t *layout, int64_t L,
                          int64_t canvas, const double *inter, double *g, double *d_off,
                          double *d_w) {
    int64_t n = canvas * canvas;
    int64_t *starts = (int64_t *)malloc(sizeof(int64_t) * (size_t)(L + 1));
    starts[0] = 0;
    for (int64_t l = 0; l < L; ++l) starts[l + 1] = starts[l] + layout[l];
    double *s = (double *)malloc(sizeof(double) * (size_t)n * 4);
    double *gp = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t l = L - 1; l >= 0; --l) {
        const double *prev = inter + l * n;
        for (int64_t i = 0; i < layout[l]; ++i) {
            int64_t q = starts[l] + i;
            double ox = off[2 * q], oy = off[2 * q + 1];
            /* _corner_shifts optim.py:185-201 */
            double fx0 = floor(ox), fy0 = floor(oy);
            double fx = ox - fx0, fy = oy - fy0;
            int64_t ix = (int64_t)fx0, iy = (int64_t)fy0;
            memset(s, 0, sizeof(double) * (size_t)n * 4);
            for (int k = 0; k < 4; ++k) {
                int64_t a = ix + (k & 1), b = iy + (k >> 1);
                int64_t y0 = b < 0 ? -b : 0, y1 = canvas - b < canvas ? canvas - b : canvas;
                int64_t x0 = a < 0 ? -a : 0, x1 = canvas - a < canvas ? canvas - a : canvas;
                for (int64_t y = y0; y < y1; ++y)
                    for (int64_t x = x0; x < x1; ++x)
                        s[k * n + y * canvas + x] = prev[(y + b) * canvas + (x + a)];
            }
            const double *s00 = s, *s10 = s + n, *s01 = s + 2 * n, *s11 = s + 3 * n;
            double a00 = (1 - fx) * (1 - fy), a10 = fx * (1 - fy), a01 = (1 - fx) * fy, a11 = fx * fy;
            double dw = 0.0, dx = 0.0, dy = 0.0;
            for (int64_t p = 0; p < n; ++p) {
                double sample = a00 * s00[p] + a10 * s10[p] + a01 * s01[p] + a11 * s11[p];
                double ddx = (1 - fy) * (s10[p] - s00[p]) + fy * (s11[p] - s01[p]);
                double ddy = (1 - fx) * (s01[p] - s00[p]) + fx * (s11[p] - s10[p]);
                dw += g[p] * sample;
                dx += g[p] * ddx;
                dy += g[p] * ddy;
            }
            d_w[q] = dw;
            d_off[2 * q] = w[q] * dx;
            d_off[2 * q + 1] = w[q] * dy;
        }
        if (l > 0) {
            memset(gp, 0, sizeof(double) * (size_t)n);
            for (int64_t i = 0; i < layout[l]; ++i) {
                int64_t q = starts[l] + i;
                sample_shifted_plane(g, gp, canvas, -off[2 * q], -off[2 * q + 1], w[q]);
            }
            memcpy(g, gp, sizeof(double) * (size_t)n);
        }
    }
    free(s); free(gp); free(starts);
}

/* optim.py:278-292 backward(): loss value and gradients at a given canvas,
 * target already embedded (canvas^2).  Returns -1 or the failing layer. */
int64_t or_backward(const double *off, const double *w, const int64_t *layout, int64_t L,
                    int64_t canvas, const double *tgt, int loss_kind, double eps,
                    double *value, double *d_off, double *d_w, int64_t *bad_sample) {
    int64_t n = canvas * canvas;
    double *inter = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(L + 1));
    int64_t bad = forward_ir(off, w, layout, L, canvas, inter, bad_sample);
    if (bad >= 0) { free(inter); return bad; }
    double *g = (double *)malloc(sizeof(double) * (size_t)n);
    const double *ir = inter + L * n;
    double v = 0.0;
    for (int64_t p = 0; p < n; ++p) {
        double d = ir[p] - tgt[p];
        v += loss_term(d, loss_kind, eps);
        g[p] = loss_grad(d, loss_kind, eps);
    }
    *value = v;
    backward_pass(off, w, layout, L, canvas, inter, g, d_off, d_w);
    free(g);
    free(inter);
    return -1;
}

/* _backward_pass (optim.py:231-263) with a caller-given upstream gradient g
 * (canvas^2) instead of the loss gradient: lets a test feed the sign pattern
 * an fp32 implementation evaluated, so an L1 gradient comparison is not
 * dominated by pixels where |IR - target| is below fp32 resolution.
 * Returns -1 or the failing layer. */
int64_t or_backward_g(const double *off, const double *w, const int64_t *layout, int64_t L,
                      int64_t canvas, const double *g_in, double *d_off, double *d_w,
                      int64_t *bad_sample) {
    int64_t n = canvas * canvas;
    double *inter = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(L + 1));
    int64_t bad = forward_ir(off, w, layout, L, canvas, inter, bad_sample);
    if (bad >= 0) { free(inter); return bad; }
    double *g = (double *)malloc(sizeof(double) * (size_t)n);
    memcpy(g, g_in, sizeof(double) * (size_t)n);
    backward_pass(off, w, layout, L, canvas, inter, g, d_off, d_w);
    free(g);
    free(inter);
    return -1;
}

/* optim.py:312-325 _project_kws */
static int project_kws(double *off, double *wp, const int64_t *layout, int64_t L) {
    static const double SX[4] = {1.0, -1.0, -1.0, 1.0};
    static const double SY[4] = {1.0, 1.0, -1.0, -1.0};
    int64_t base = 0;
    for (int64_t l = 0; l < L; ++l) {
        if (layout[l] % 4) return 1;
        for (int64_t g = 0; g < layout[l] / 4; ++g) {
            int64_t q = base + 4 * g;
            double dx = 0.0, dy = 0.0, mw = 0.0;
            for (int k = 0; k < 4; ++k) {
                dx += SX[k] * off[2 * (q + k)];
                dy += SY[k] * off[2 * (q + k) + 1];
                mw += wp[q + k];
            }
            dx /= 4.0; dy /= 4.0; mw /= 4.0;
            for (int k = 0; k < 4; ++k) {
                off[2 * (q + k)] = SX[k] * dx;
                off[2 * (q + k) + 1] = SY[k] * dy;
                wp[q + k] = mw;
            }
        }
        base += layout[l];
    }
    return 0;
}

/* optim.py:328-335 _project_sum; returns failing layer or -1. */
static int64_t project_sum(double *wp, const int64_t *layout, int64_t L) {
    int64_t base = 0;
    for (int64_t l = 0; l < L; ++l) {
        double s = 0.0;
        for (int64_t i = 0; i < layout[l]; ++i) s += wp[base + i];
        if (fabs(s) < 1e-8) return l;
        for (int64_t i = 0; i < layout[l]; ++i) wp[base + i] /= s;
        base += layout[l];
    }
    return -1;
}

static double reach_of(const double *off, const int64_t *layout, int64_t L) {
    /* engine.py:68-71, 101-103 */
    double r = 0.0;
    int64_t base = 0;
    for (int64_t l = 0; l < L; ++l) {
        double m = 0.0;
        for (int64_t i = 0; i < 2 * layout[l]; ++i) {
            double a = fabs(off[2 * base + i]);
            if (a > m) m = a;
        }
        r += m;
        base += layout[l];
    }
    return r;
}

static int64_t required_canvas(double reach) { return 2 * (int64_t)ceil(reach) + 1; }

static void embed(const double *tgt, int64_t m, int64_t canvas, double *out) {
    /* kernels.py:75-82 DenseKernel.embedded */
    int64_t pad = (canvas - m) / 2;
    memset(out, 0, sizeof(double) * (size_t)(canvas * canvas));
    for (int64_t y = 0; y < m; ++y)
        for (int64_t x = 0; x < m; ++x) out[(y + pad) * canvas + x + pad] = tgt[y * m + x];
}

typedef struct {
    int64_t steps;
    double lr_start, lr_end, beta1, beta2, eps;
    int weight_norm;  /* WN_* */
    int kws;
    int loss_kind;
    double loss_eps;
} or_fit_cfg;

static double lr_at(const or_fit_cfg *c, int64_t step) {
    /* optim.py:101-105 */
    if (c->steps == 1) return c->lr_start;
    int64_t t = step < 0 ? 0 : (step > c->steps - 1 ? c->steps - 1 : step);
    return c->lr_start + (c->lr_end - c->lr_start) * (double)t / (double)(c->steps - 1);
}

/* optim.py:390-469 fit() with an explicit KernelComplex init (optim.py:404-405).
 * off0 (P,2), w0 (P,) are the init's effective weights.  Outputs:
 *   trace (steps+1) losses, best_off (P,2), best_w (P,) effective weights,
 *   info[0]=best_step, info[1]=final canvas.  Returns 0 ok, 1 nonfinite
 *   (err_layer), 2 sum degenerate (err_layer), 3 kws layout. */
int or_fit(const double *tgt, int64_t m, const double *off0, const double *w0,
           const int64_t *layout, int64_t L, const or_fit_cfg *cfg, double *trace,
           double *best_off, double *best_w, double *best_loss_out, int64_t *info,
           int64_t *err_layer) {
    int64_t P = 0;
    for (int64_t l = 0; l < L; ++l) P += layout[l];
    double *off = (double *)malloc(sizeof(double) * (size_t)(2 * P));
    double *wp = (double *)malloc(sizeof(double) * (size_t)P);
    double *w = (double *)malloc(sizeof(double) * (size_t)P);
    double *m_off = (double *)calloc((size_t)(2 * P), sizeof(double));
    double *v_off = (double *)calloc((size_t)(2 * P), sizeof(double));
    double *m_w = (double *)calloc((size_t)P, sizeof(double));
    double *v_w = (double *)calloc((size_t)P, sizeof(double));
    double *g_off = (double *)malloc(sizeof(double) * (size_t)(2 * P));
    double *g_w = (double *)malloc(sizeof(double) * (size_t)P);
    double *bo = (double *)malloc(sizeof(double) * (size_t)(2 * P));
    double *bw = (double *)malloc(sizeof(double) * (size_t)P);
    int rc = 0;
    memcpy(off, off0, sizeof(double) * (size_t)(2 * P));
    /* optim.py:168-176 _params_from_complex */
    for (int64_t q = 0; q < P; ++q)
        wp[q] = (cfg->weight_norm == WN_SOFM) ? log(w0[q] < 1e-12 ? 1e-12 : w0[q]) : w0[q];
    if (cfg->kws && project_kws(off, wp, layout, L)) { rc = 3; goto done; }
    if (cfg->weight_norm == WN_SUM) {
        int64_t bad = project_sum(wp, layout, L);
        if (bad >= 0) { *err_layer = bad; rc = 2; goto done; }
    }
    double offset_lr_scale = (double)m;   /* optim.py:411 */
    int64_t canvas = required_canvas(reach_of(off, layout, L)) + 4;
    if (canvas < m) canvas = m;
    double *tgt_c = NULL, *inter = NULL, *g = NULL;
    int64_t cap = 0;
    double best_loss = INFINITY;
    int64_t best_step = 0;
    for (int64_t step = 0; step <= cfg->steps; ++step) {
        /* embed_if_grown optim.py:429-434 */
        int64_t need = required_canvas(reach_of(off, layout, L));
        if (need > canvas) canvas = need + 4;
        int64_t n = canvas * canvas;
        if (n > cap) {
            free(tgt_c); free(inter); free(g);
            cap = n;
            tgt_c = (double *)malloc(sizeof(double) * (size_t)n);
            inter = (double *)malloc(sizeof(double) * (size_t)n * (size_t)(L + 1));
            g = (double *)malloc(sizeof(double) * (size_t)n);
        }
        embed(tgt, m, canvas, tgt_c);
        effective_weights(wp, w, layout, L, cfg->weight_norm);
        int64_t bs;
        int64_t bad = forward_ir(off, w, layout, L, canvas, inter, &bs);
        if (bad >= 0) { *err_layer = bad; rc = 1; break; }
        const double *ir = inter + L * n;
        double v = 0.0;
        for (int64_t p = 0; p < n; ++p) {
            double d = ir[p] - tgt_c[p];
            v += loss_term(d, cfg->loss_kind, cfg->loss_eps);
            g[p] = loss_grad(d, cfg->loss_kind, cfg->loss_eps);
        }
        trace[step] = v;
        if (v < best_loss) {
            best_loss = v;
            best_step = step;
            memcpy(bo, off, sizeof(double) * (size_t)(2 * P));
            memcpy(bw, w, sizeof(double) * (size_t)P);
        }
        if (step == cfg->steps) break;   /* final forward (optim.py:452-459) */
        backward_pass(off, w, layout, L, canvas, inter, g, g_off, g_w);
        if (cfg->weight_norm == WN_SOFM) {  /* optim.py:266-275 */
            int64_t base = 0;
            for (int64_t l = 0; l < L; ++l) {
                double dot = 0.0;
                for (int64_t i = 0; i < layout[l]; ++i) dot += g_w[base + i] * w[base + i];
                for (int64_t i = 0; i < layout[l]; ++i)
                    g_w[base + i] = w[base + i] * (g_w[base + i] - dot);
                base += layout[l];
            }
        }
        /* adam_step optim.py:338-369 */
        double lr = lr_at(cfg, step);
        double t = (double)(step + 1);
        double c1 = 1.0 - pow(cfg->beta1, t), c2 = 1.0 - pow(cfg->beta2, t);
        for (int64_t q = 0; q < 2 * P; ++q) {
            m_off[q] = m_off[q] * cfg->beta1 + (1 - cfg->beta1) * g_off[q];
            v_off[q] = v_off[q] * cfg->beta2 + (1 - cfg->beta2) * g_off[q] * g_off[q];
            double mh = m_off[q] / c1, vh = v_off[q] / c2;
            off[q] = off[q] - offset_lr_scale * lr * mh / (sqrt(vh) + cfg->eps);
        }
        for (int64_t q = 0; q < P; ++q) {
            m_w[q] = m_w[q] * cfg->beta1 + (1 - cfg->beta1) * g_w[q];
            v_w[q] = v_w[q] * cfg->beta2 + (1 - cfg->beta2) * g_w[q] * g_w[q];
            double mh = m_w[q] / c1, vh = v_w[q] / c2;
            wp[q] = wp[q] - 1.0 * lr * mh / (sqrt(vh) + cfg->eps);
        }
        if (cfg->kws) project_kws(off, wp, layout, L);
        if (cfg->weight_norm == WN_SUM) {
            int64_t b2 = project_sum(wp, layout, L);
            if (b2 >= 0) { *err_layer = b2; rc = 2; break; }
        }
    }
    if (rc == 0) {
        memcpy(best_off, bo, sizeof(double) * (size_t)(2 * P));
        memcpy(best_w, bw, sizeof(double) * (size_t)P);
        *best_loss_out = best_loss;
        info[0] = best_step;
        info[1] = canvas;
    }
    free(tgt_c); free(inter); free(g);
done:
    free(off); free(wp); free(w); free(m_off); free(v_off); free(m_w); free(v_w);
    free(g_off); free(g_w); free(bo); free(bw);
    return rc;
}

/* Batched fits (independent kernels), parallel over the batch -- the CPU
 * baseline for config 4.  tgts (B,m,m); off0 (B,P,2); w0 (B,P); outputs
 * batched likewise; rcs (B,). */
void or_fit_batch(const double *tgts, int64_t B, int64_t m, const double *off0, const double *w0,
                  const int64_t *layout, int64_t L, const or_fit_cfg *cfg, double *trace,
                  double *best_off, double *best_w, double *best_loss, int64_t *info,
                  int64_t *err_layer, int *rcs) {
    int64_t P = 0;
    for (int64_t l = 0; l < L; ++l) P += layout[l];
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < B; ++b) {
        rcs[b] = or_fit(tgts + b * m * m, m, off0 + b * 2 * P, w0 + b * P, layout, L, cfg,
                        trace + b * (cfg->steps + 1), best_off + b * 2 * P, best_w + b * P,
                        best_loss + b, info + 2 * b, err_layer + b);
    }
}
