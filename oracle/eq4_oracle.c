/*
 * eq4_oracle.c -- CPU ORACLE for the row-wise 4-bit clip-search + pack path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is a plain-C restatement of the
 * reference package `embquant` (arXiv 1911.02079 artifact, pure Python/numpy)
 * for the hot path named in BASELINE.json: ASYM, GREEDY and HIST-BRUTE
 * clipping searches, the uniform codec and the packed 4-bit row layout.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load it -- as the checker or as the timed CPU
 * baseline, never as the product path.  The product path is the CUDA
 * library paper_1911_02079_b200/libeq4.so.
 *
 * Arithmetic contract (what makes this a bit-exact restatement):
 *   - every floating-point operation is an IEEE-754 binary64 op in the same
 *     order and association as the numpy expression it restates; the build
 *     uses -ffp-contract=off so no mul+add is fused;
 *   - np.sum over a contiguous float64 vector is numpy's pairwise sum
 *     (numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE=128, 8-way
 *     unrolled leaves) added to the reduction identity 0.0;
 *   - np.float16(x) / np.float32(x) are single round-to-nearest-even
 *     conversions from binary64 (gcc _Float16 / (float) casts);
 *   - x**3 on float64 arrays is libm pow(x, 3.0), as numpy's npy_pow.
 * HIST-BRUTE's np.convolve goes through BLAS ddot in the reference, whose
 * summation order is CPU-kernel specific; here each window norm is a plain
 * ascending-j sum.  Its argmin agrees with the reference except at near-ties
 * (see DESIGN.md "parity"); every other output of this file is bit-exact
 * against the reference (pinned by tests/golden, generated from the
 * reference itself by tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EQO_OK 0
#define EQO_EB 1        /* b < 1                          clipping.py:158-159, histclip.py:54-55 */
#define EQO_ER 2        /* r not in (0, 1]                clipping.py:160-161 */
#define EQO_EEMPTY 3    /* empty vector                   clipping.py:44-48, histclip.py:57-58 */
#define EQO_ERANGE 4    /* ClipRange invalid (xmin>xmax)  table.py:70-74 */
#define EQO_EFINITE 5   /* non-finite input               table.py:28-29 */
#define EQO_ENBITS 6    /* nbits not in {4,8}             table.py:92-93 */
#define EQO_EALLOC 7
#define EQO_EMETHOD 8

#define METHOD_ASYM 0
#define METHOD_GREEDY 1
#define METHOD_HIST_BRUTE 2
#define METHOD_SYM 3
#define METHOD_ACIQ 4
#define METHOD_GSS 5
#define METHOD_TABLE 6
#define METHOD_HIST_APPRX 7

#define DST_NBINS 16 /* histclip.py:31 */

/* numpy pairwise summation (loops_utils.h.src @TYPE@_pairwise_sum). */
static double np_pairwise_sum(const double *a, long n) {
    if (n < 8) {
        double res = 0.;
        for (long i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        long i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        long n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
    }
}

/* np.add.reduce of a 1-D float64 array: identity 0.0 plus the pairwise sum. */
double eqo_np_sum(const double *a, long n) { return 0.0 + np_pairwise_sum(a, n); }

/* np.clip(x, lo, hi) == minimum(maximum(x, lo), hi) for finite inputs. */
static inline double np_clip(double x, double lo, double hi) {
    double t = x > lo ? x : lo;
    return t < hi ? t : hi;
}

/* table.py:81-103 quant_mse: float64 sum of squared reconstruction errors.
 * scratch must hold d doubles. */
int eqo_quant_mse(const float *xf, long d, double xmin, double xmax, int nbits,
                  double *scratch, double *out) {
    if (nbits != 4 && nbits != 8) return EQO_ENBITS;             /* table.py:92-93 */
    if (!(isfinite(xmin) && isfinite(xmax))) return EQO_ERANGE;  /* table.py:71-72 */
    if (xmin > xmax) return EQO_ERANGE;                          /* table.py:73-74 */
    if (xmax == xmin) {                                          /* table.py:96-97 */
        for (long i = 0; i < d; i++) {
            double e = (double)xf[i] - xmin;
            scratch[i] = e * e;
        }
        *out = eqo_np_sum(scratch, d);
        return EQO_OK;
    }
    double qmax = (double)((1 << nbits) - 1);                    /* table.py:98 */
    double scale = (xmax - xmin) / qmax;                         /* table.py:99 */
    for (long i = 0; i < d; i++) {
        double x = (double)xf[i];
        double clamped = np_clip(x, xmin, xmax);                 /* table.py:100 */
        double code = floor((clamped - xmin) / scale + 0.5);     /* table.py:101 */
        code = np_clip(code, 0.0, qmax);
        double recon = scale * code + xmin;                      /* table.py:102 */
        double e = x - recon;                                    /* table.py:103 */
        scratch[i] = e * e;
    }
    *out = eqo_np_sum(scratch, d);
    return EQO_OK;
}

static int check_finite(const float *x, long d) {
    for (long i = 0; i < d; i++)
        if (!isfinite(x[i])) return EQO_EFINITE;
    return EQO_OK;
}

/* np.min / np.max of the row promoted to float64 (clipping.py:46,61,163;
 * histclip.py:57), in numpy's own reduction order: the value is the plain
 * extremum, but WHICH of several equal extrema is returned decides the sign
 * of a zero extremum (+0.0 == -0.0), and that sign reaches the packed bias.
 * numpy 2.x (loops_minmax.dispatch.c.src, AVX-512 dispatch of the host that
 * made tests/golden) reduces a contiguous float64 vector as:
 *   r = x[0]; acc[0..7] = r; over x[1..]: 64-element blocks
 *   acc = OP(acc, OP(OP(OP(v0,v1),OP(v2,v3)), OP(OP(v4,v5),OP(v6,v7)))),
 *   then 8-element vectors acc = OP(acc, v); r = _mm512_reduce (OP(hi4,lo4),
 *   OP(hi2,lo2), OP(v[0],v[1])); then r = OP(r, x[i]) over the scalar tail,
 * with OP(a, b) = a < b ? a : b (max: a > b ? a : b) -- vminpd / vmaxpd
 * return the second operand on equality.  Pinned against np.min/np.max by
 * tests/golden/signed_zero.npz (made by the reference). */
static double np_reduce_ext(const float *x, long d, int is_max) {
#define NP_OP(a, b) (is_max ? ((a) > (b) ? (a) : (b)) : ((a) < (b) ? (a) : (b)))
    double r = (double)x[0];
    const float *ip = x + 1;
    long n = d - 1;
    if (n >= 8) {
        double acc[8];
        for (int k = 0; k < 8; k++) acc[k] = r;
        for (; n >= 64; n -= 64, ip += 64) {
            for (int k = 0; k < 8; k++) {
                double v[8];
                for (int j = 0; j < 8; j++) v[j] = (double)ip[8 * j + k];
                double r01 = NP_OP(v[0], v[1]), r23 = NP_OP(v[2], v[3]);
                double r45 = NP_OP(v[4], v[5]), r67 = NP_OP(v[6], v[7]);
                double t = NP_OP(NP_OP(r01, r23), NP_OP(r45, r67));
                acc[k] = NP_OP(acc[k], t);
            }
        }
        for (; n >= 8; n -= 8, ip += 8)
            for (int k = 0; k < 8; k++) acc[k] = NP_OP(acc[k], (double)ip[k]);
        double t3[4], t6[2];
        for (int k = 0; k < 4; k++) t3[k] = NP_OP(acc[k + 4], acc[k]);
        for (int k = 0; k < 2; k++) t6[k] = NP_OP(t3[k + 2], t3[k]);
        r = NP_OP(t6[0], t6[1]);
    }
    for (; n > 0; n--, ip++) r = NP_OP(r, (double)*ip);
    return r;
#undef NP_OP
}

static void row_minmax(const float *x, long d, double *lo, double *hi) {
    *lo = np_reduce_ext(x, d, 0);
    *hi = np_reduce_ext(x, d, 1);
}

/* Test hook: np.min (is_max = 0) / np.max (1) of a float32 row promoted to float64. */
double eqo_np_extremum(const float *x, long d, int is_max) { return np_reduce_ext(x, d, is_max); }

/* clipping.py:58-61 clip_range_asym. */
int eqo_clip_range_asym(const float *x, long d, double *lo, double *hi) {
    if (d <= 0) return EQO_EEMPTY;
    row_minmax(x, d, lo, hi);
    return EQO_OK;
}

/* clipping.py:51-55 clip_range_sym: xmax = max|x| (float64), range (-xmax, xmax). */
int eqo_clip_range_sym(const float *x, long d, double *lo, double *hi) {
    if (d <= 0) return EQO_EEMPTY;
    double m = fabs((double)x[0]);
    for (long i = 1; i < d; i++) {
        double a = fabs((double)x[i]);
        if (a > m) m = a;
    }
    *lo = -m;
    *hi = m;
    return EQO_OK;
}

/* clipping.py:115-139 clip_range_aciq, laplacian branch (the one row_clip_range uses):
 * mean = np.mean(x) (pairwise sum / n), alpha = 5.03 * np.mean(|x - mean|);
 * alpha == 0 -> the data range.  scratch: d doubles. */
int eqo_clip_range_aciq(const float *x, long d, double *scratch, double *lo, double *hi) {
    if (d <= 0) return EQO_EEMPTY;
    for (long i = 0; i < d; i++) scratch[i] = (double)x[i];
    const double mean = eqo_np_sum(scratch, d) / (double)d;
    for (long i = 0; i < d; i++) scratch[i] = fabs((double)x[i] - mean);
    const double alpha = 5.03 * (eqo_np_sum(scratch, d) / (double)d);
    if (alpha == 0.0) return eqo_clip_range_asym(x, d, lo, hi);
    *lo = mean - alpha;
    *hi = mean + alpha;
    return EQO_OK;
}

/* clipping.py:70-112 clip_range_gss (tol = 1e-4): golden-section search over
 * t in (0, max|x|] of quant_mse(x, (-t, t)), keeping the best point evaluated
 * (strict <, the unclipped endpoint first).  scratch: d doubles. */
int eqo_clip_range_gss(const float *x, long d, int nbits, double *scratch, double *lo, double *hi,
                       int *evals) {
    if (d <= 0) return EQO_EEMPTY;
    const double invphi = (sqrt(5.0) - 1.0) / 2.0;          /* clipping.py:27 */
    const double tol = 1e-4;
    double tmax = 0.0;
    eqo_clip_range_sym(x, d, lo, &tmax);
    int n = 0;
    if (tmax == 0.0) {
        *lo = 0.0;
        *hi = 0.0;
        if (evals) *evals = 0;
        return EQO_OK;
    }
#define GSS_F(t, out) do { n++; int rc_ = eqo_quant_mse(x, d, -(t), (t), nbits, scratch, &(out)); \
                           if (rc_) return rc_; } while (0)
    double best_t = tmax, best_f;
    GSS_F(tmax, best_f);
    double a = 0.0, b = tmax;
    double c = b - invphi * (b - a);
    double e = a + invphi * (b - a);
    double fc, fe;
    GSS_F(c, fc);
    GSS_F(e, fe);
    if (fc < best_f) { best_t = c; best_f = fc; }
    if (fe < best_f) { best_t = e; best_f = fe; }
    while (b - a > tol * tmax) {
        if (fc < fe) {
            b = e; e = c; fe = fc;
            c = b - invphi * (b - a);
            GSS_F(c, fc);
            if (fc < best_f) { best_t = c; best_f = fc; }
        } else {
            a = c; c = e; fc = fe;
            e = a + invphi * (b - a);
            GSS_F(e, fe);
            if (fe < best_f) { best_t = e; best_f = fe; }
        }
    }
#undef GSS_F
    *lo = -best_t;
    *hi = best_t;
    if (evals) *evals = n;
    return EQO_OK;
}

/* clipping.py:142-193 clip_range_greedy (Alg. 1, pair recording).
 * *iters receives the number of while-loop iterations (-1 for a constant
 * row, where the reference returns before evaluating any loss), so the
 * reference's WorkCounters.loss_evals == 1 + 2*iters (0 for constant rows).
 * *best_i / *best_j receive the step counts of the returned pair:
 * (x0 + i*step, x1 - j*step). */
static int greedy_impl(const float *x, long d, int nbits, int b, double r, double *lo, double *hi,
                       int *iters, int *best_i, int *best_j, double *scratch, double *gap_lr,
                       double *gap_best);

int eqo_clip_range_greedy(const float *x, long d, int nbits, int b, double r,
                          double *lo, double *hi, int *iters, int *best_i, int *best_j,
                          double *scratch) {
    return greedy_impl(x, d, nbits, b, r, lo, hi, iters, best_i, best_j, scratch, NULL, NULL);
}

/* Test hook: the walk of clip_range_greedy step by step.  For iteration t (t < *iters):
 * nl[t], nr[t] before the move, loss_l[t], loss_r[t] (clipping.py:181-184).
 * cap = capacity of the arrays.  Returns EQO_* (the walk stops at cap). */
int eqo_greedy_trace(const float *x, long d, int b, double r, int cap, int *iters, int *nl_out,
                     int *nr_out, double *loss_l_out, double *loss_r_out, double *scratch) {
    if (b < 1) return EQO_EB;
    if (!(0.0 < r && r <= 1.0)) return EQO_ER;
    if (d <= 0) return EQO_EEMPTY;
    double x0, x1;
    row_minmax(x, d, &x0, &x1);
    *iters = 0;
    if (x0 == x1) return EQO_OK;
    double stepsize = (x1 - x0) / (double)b;
    double min_steps = (double)b * (1.0 - r) * stepsize;
    long nl = 0, nr = 0;
    int it = 0;
    while ((x0 + (double)nl * stepsize) + min_steps < (x1 - (double)nr * stepsize) && it < cap) {
        double lmin = x0 + (double)(nl + 1) * stepsize, lmax = x1 - (double)nr * stepsize;
        double rmin = x0 + (double)nl * stepsize, rmax = x1 - (double)(nr + 1) * stepsize;
        double loss_l, loss_r;
        int rc = eqo_quant_mse(x, d, lmin, lmax, 4, scratch, &loss_l);
        if (!rc) rc = eqo_quant_mse(x, d, rmin, rmax, 4, scratch, &loss_r);
        if (rc) return rc;
        nl_out[it] = (int)nl; nr_out[it] = (int)nr;
        loss_l_out[it] = loss_l; loss_r_out[it] = loss_r;
        if (loss_l < loss_r) nl += 1; else nr += 1;
        it++;
    }
    *iters = it;
    return EQO_OK;
}

/* Relative gap |a - b| / max(|a|, |b|) of two competing losses (0 when both are 0). */
static double rel_gap(double a, double b) {
    const double m = fmax(fabs(a), fabs(b));
    return m > 0.0 ? fabs(a - b) / m : 0.0;
}

/* The walk of eqo_clip_range_greedy; gap_lr / gap_best (optional) receive the smallest
 * relative gap over the walk between the two competing losses (clipping.py:185) and
 * between the chosen candidate and the best so far (clipping.py:187,191) -- the
 * reference's own near-ties, which north_star asks to count (INFINITY: no iteration). */
static int greedy_impl(const float *x, long d, int nbits, int b, double r, double *lo, double *hi,
                       int *iters, int *best_i, int *best_j, double *scratch, double *gap_lr,
                       double *gap_best) {
    if (gap_lr) *gap_lr = INFINITY;
    if (gap_best) *gap_best = INFINITY;
    if (b < 1) return EQO_EB;                        /* clipping.py:158-159 */
    if (!(0.0 < r && r <= 1.0)) return EQO_ER;       /* clipping.py:160-161 */
    if (d <= 0) return EQO_EEMPTY;                   /* clipping.py:162 */
    double x0, x1;
    row_minmax(x, d, &x0, &x1);                      /* clipping.py:163 */
    if (x0 == x1) {                                  /* clipping.py:164-165 */
        *lo = x0; *hi = x1; *iters = -1; *best_i = 0; *best_j = 0;
        return EQO_OK;
    }
    double stepsize = (x1 - x0) / (double)b;         /* clipping.py:172 */
    double min_steps = (double)b * (1.0 - r) * stepsize; /* clipping.py:173 (left to right) */
    double best_loss;
    int rc = eqo_quant_mse(x, d, x0, x1, nbits, scratch, &best_loss); /* :174 */
    if (rc) return rc;
    double best_min = x0, best_max = x1;
    long nl = 0, nr = 0;
    int bi = 0, bj = 0, it = 0;
    while ((x0 + (double)nl * stepsize) + min_steps < (x1 - (double)nr * stepsize)) { /* :180 */
        double lmin = x0 + (double)(nl + 1) * stepsize, lmax = x1 - (double)nr * stepsize; /* :181 */
        double rmin = x0 + (double)nl * stepsize, rmax = x1 - (double)(nr + 1) * stepsize; /* :182 */
        double loss_l, loss_r;
        rc = eqo_quant_mse(x, d, lmin, lmax, nbits, scratch, &loss_l);   /* :183 */
        if (rc) return rc;
        rc = eqo_quant_mse(x, d, rmin, rmax, nbits, scratch, &loss_r);   /* :184 */
        if (rc) return rc;
        if (gap_lr) {
            const double g1 = rel_gap(loss_l, loss_r);
            const double g2 = rel_gap(loss_l < loss_r ? loss_l : loss_r, best_loss);
            if (g1 < *gap_lr) *gap_lr = g1;
            if (g2 < *gap_best) *gap_best = g2;
        }
        if (loss_l < loss_r) {                                           /* :185 */
            nl += 1;
            if (loss_l < best_loss) {
                best_loss = loss_l; best_min = lmin; best_max = lmax;
                bi = (int)nl; bj = (int)nr;
            }
        } else {                                                         /* :189 */
            nr += 1;
            if (loss_r < best_loss) {
                best_loss = loss_r; best_min = rmin; best_max = rmax;
                bi = (int)nl; bj = (int)nr;
            }
        }
        it++;
    }
    *lo = best_min; *hi = best_max; *iters = it; *best_i = bi; *best_j = bj;
    return EQO_OK;
}

/* histclip.py:52-67 build_histogram. counts has b entries. */
int eqo_build_histogram(const float *x, long d, int b, double *lo, double *hi, int64_t *counts) {
    if (b < 1) return EQO_EB;
    if (d <= 0) return EQO_EEMPTY;
    row_minmax(x, d, lo, hi);
    for (int i = 0; i < b; i++) counts[i] = 0;
    if (*lo == *hi) {
        counts[0] = d;
        return EQO_OK;
    }
    double w = (*hi - *lo) / (double)b;
    for (long i = 0; i < d; i++) {
        double idx = floor(((double)x[i] - *lo) / w);
        long k = (long)np_clip(idx, 0.0, (double)(b - 1));
        counts[k] += 1;
    }
    return EQO_OK;
}

/* histclip.py:70-82 bin_l2_norm: density * (de**3 - db**3) / 3.0 */
double eqo_bin_l2_norm(double db, double de, double density) {
    return density * (pow(de, 3.0) - pow(db, 3.0)) / 3.0;
}

/* histclip.py:85-109 _offset_unit_norms for offsets k[0..n). */
void eqo_offset_unit_norms(const double *k, long n, double bin_width, double dst_bin_width,
                           double *out) {
    double half = 0.5 * dst_bin_width;
    for (long i = 0; i < n; i++) {
        double begin = k[i] * bin_width;
        double end = begin + bin_width;
        double dob = np_clip(floor((begin + half) / dst_bin_width), 0.0, DST_NBINS - 1);
        double doe = np_clip(floor((end + half) / dst_bin_width), 0.0, DST_NBINS - 1);
        double begin_center = dob * dst_bin_width;
        double end_center = doe * dst_bin_width;
        double delta_begin = begin - begin_center;
        double same = eqo_bin_l2_norm(delta_begin, end - begin_center, 1.0);
        double split = eqo_bin_l2_norm(delta_begin, half, 1.0)
                     + (doe - dob - 1.0) * eqo_bin_l2_norm(-half, half, 1.0)
                     + eqo_bin_l2_norm(-half, end - end_center, 1.0);
        out[i] = (dob == doe) ? same : split;
    }
}

/* histclip.py:110-121 window_norm: np.sum(density * _offset_unit_norms(arange(b) - s, w, dst_w)).
 * density/k/contrib scratch: 3b doubles. */
static double window_norm(const double *density, int b, double w, int s, int n, double *kbuf,
                          double *contrib, double *prod) {
    if (w == 0.0) return 0.0;
    double dst_w = w * (double)n / (double)(DST_NBINS - 1);
    for (int j = 0; j < b; j++) kbuf[j] = (double)j - (double)s;
    eqo_offset_unit_norms(kbuf, b, w, dst_w, contrib);
    for (int j = 0; j < b; j++) prod[j] = density[j] * contrib[j];
    return eqo_np_sum(prod, b);
}

/* histclip.py:181-217 hist_apprx_search: from the full window, repeatedly drop
 * NOTE: window norms use libm pow(x, 3); the reference's numpy `**3` dispatches
 * to SIMD (SVML) power on AVX-512 hosts, which differs from libm in the last
 * bit for a few % of inputs, so its norms are host-dependent in the last ulp
 * (window selection agrees except at such near-ties).
 * one bin from the end whose removal scores lower (ties drop from the right),
 * keeping the best window seen.  scratch: >= 4*b doubles. */
static int hist_apprx_impl(const float *x, long d, int b, double *lo, double *hi, int *start,
                           int *nsel, double *norm, long *cand_evals, long *bin_visits,
                           double *scratch, double *min_gap);

int eqo_hist_apprx(const float *x, long d, int b, double *lo, double *hi, int *start, int *nsel,
                   double *norm, long *cand_evals, long *bin_visits, double *scratch) {
    return hist_apprx_impl(x, d, b, lo, hi, start, nsel, norm, cand_evals, bin_visits, scratch, NULL);
}

/* Same walk; *min_gap = min over its decisions of |nl - nr| / max(nl, nr) (test helper:
 * a walk can only diverge from another float64 evaluation order at a near-tie). */
int eqo_hist_apprx_gap(const float *x, long d, int b, double *lo, double *hi, int *start, int *nsel,
                       double *norm, double *scratch, double *min_gap) {
    long ce = 0, bv = 0;
    return hist_apprx_impl(x, d, b, lo, hi, start, nsel, norm, &ce, &bv, scratch, min_gap);
}

static int hist_apprx_impl(const float *x, long d, int b, double *lo, double *hi, int *start,
                           int *nsel, double *norm, long *cand_evals, long *bin_visits,
                           double *scratch, double *min_gap) {
    if (min_gap) *min_gap = INFINITY;
    if (b < 1) return EQO_EB;
    if (d <= 0) return EQO_EEMPTY;
    int64_t *counts = (int64_t *)malloc(sizeof(int64_t) * (size_t)b);
    if (!counts) return EQO_EALLOC;
    double hlo, hhi;
    eqo_build_histogram(x, d, b, &hlo, &hhi, counts);
    if (hlo == hhi) {                                          /* :193-197 */
        *cand_evals += 1;
        *bin_visits += b;
        *lo = hlo; *hi = hhi; *start = 0; *nsel = 1; *norm = 0.0;
        free(counts);
        return EQO_OK;
    }
    double w = (hhi - hlo) / (double)b;
    double *density = scratch, *kbuf = scratch + b, *contrib = scratch + 2 * (long)b,
           *prod = scratch + 3 * (long)b;
    for (int j = 0; j < b; j++) density[j] = (double)counts[j] / w;
    int st = 0, en = b;
    double best = window_norm(density, b, w, st, en - st, kbuf, contrib, prod);
    long evals = 1;
    int bs = st, be = en;
    while (en - st > 1) {                                      /* :201-213 */
        double nl = window_norm(density, b, w, st + 1, en - st - 1, kbuf, contrib, prod);
        double nr = window_norm(density, b, w, st, en - st - 1, kbuf, contrib, prod);
        evals += 2;
        if (min_gap) {
            double m = nl > nr ? nl : nr;
            double g = m > 0 ? fabs(nl - nr) / m : 0.0;
            if (g < *min_gap) *min_gap = g;
        }
        double cur;
        if (nl < nr) { st += 1; cur = nl; } else { en -= 1; cur = nr; }
        if (cur < best) { best = cur; bs = st; be = en; }
    }
    *cand_evals += evals;
    *bin_visits += evals * b;
    *lo = hlo + w * (double)bs;                                /* :214-219 */
    *hi = hlo + w * (double)be;
    *start = bs; *nsel = be - bs; *norm = best;
    free(counts);
    if (!(isfinite(*lo) && isfinite(*hi)) || *lo > *hi) return EQO_ERANGE;
    return EQO_OK;
}

/* histclip.py:136-174 hist_brute_search.  scratch: >= 5*b doubles.
 * Work counters follow histclip.py:148-150,162-164. */
int eqo_hist_brute(const float *x, long d, int b, double *lo, double *hi, int *start, int *nsel,
                   double *norm, long *cand_evals, long *bin_visits, double *scratch) {
    if (b < 1) return EQO_EB;
    if (d <= 0) return EQO_EEMPTY;
    int64_t *counts = (int64_t *)malloc(sizeof(int64_t) * (size_t)b);
    if (!counts) return EQO_EALLOC;
    double hlo, hhi;
    eqo_build_histogram(x, d, b, &hlo, &hhi, counts);
    if (hlo == hhi) {                                         /* histclip.py:147-151 */
        *cand_evals += 1;
        *bin_visits += b;
        *lo = hlo; *hi = hhi; *start = 0; *nsel = 1; *norm = 0.0;
        free(counts);
        return EQO_OK;
    }
    double w = (hhi - hlo) / (double)b;                       /* Histogram.bin_width */
    double *density = scratch;                                /* b */
    double *offsets = scratch + b;                            /* 2b-1 */
    double *contrib = scratch + 3 * (long)b;                  /* 2b-1 */
    for (int j = 0; j < b; j++) density[j] = (double)counts[j] / w;  /* :153 */
    for (int i = 0; i < 2 * b - 1; i++) offsets[i] = (double)(i - (b - 1)); /* :154 */
    double best_norm = INFINITY;
    int best_start = 0, best_n = 1;
    for (int n = 1; n <= b; n++) {                             /* :157 */
        double dst_w = w * (double)n / (double)(DST_NBINS - 1);   /* :158 */
        eqo_offset_unit_norms(offsets, 2 * b - 1, w, dst_w, contrib); /* :159 */
        int ncand = b - n + 1;
        *cand_evals += ncand;                                   /* :162-164 */
        *bin_visits += (long)ncand * b;
        /* :161 norms[s] = sum_j density[j] * contrib[j - s]; first argmin :165 */
        double nmin = INFINITY;
        int smin = 0;
        for (int s = 0; s < ncand; s++) {
            double acc = 0.0;
            for (int j = 0; j < b; j++) acc += density[j] * contrib[(j - s) + (b - 1)];
            if (acc < nmin) { nmin = acc; smin = s; }
        }
        if (nmin < best_norm) {                                 /* :166-168 */
            best_norm = nmin; best_start = smin; best_n = n;
        }
    }
    *lo = hlo + w * (double)best_start;                        /* :170 */
    *hi = hlo + w * (double)(best_start + best_n);
    *start = best_start; *nsel = best_n; *norm = best_norm;
    free(counts);
    if (!(isfinite(*lo) && isfinite(*hi)) || *lo > *hi) return EQO_ERANGE;
    return EQO_OK;
}

/* Norm of one window (start s, width n) as histclip.py:152-161 computes it
 * (plain ascending-j sum in place of BLAS).  Used by tests to classify a
 * differing selection as a norm tie.  scratch: >= 5*b doubles. */
int eqo_hist_window_norm(const float *x, long d, int b, int s, int n, double *out, double *scratch) {
    if (b < 1 || n < 1 || s < 0 || s + n > b) return EQO_EB;
    int64_t *counts = (int64_t *)malloc(sizeof(int64_t) * (size_t)b);
    if (!counts) return EQO_EALLOC;
    double lo, hi;
    eqo_build_histogram(x, d, b, &lo, &hi, counts);
    if (lo == hi) { *out = 0.0; free(counts); return EQO_OK; }
    double w = (hi - lo) / (double)b;
    double *density = scratch, *offsets = scratch + b, *contrib = scratch + 3 * (long)b;
    for (int j = 0; j < b; j++) density[j] = (double)counts[j] / w;
    for (int i = 0; i < 2 * b - 1; i++) offsets[i] = (double)(i - (b - 1));
    double dst_w = w * (double)n / (double)(DST_NBINS - 1);
    eqo_offset_unit_norms(offsets, 2 * b - 1, w, dst_w, contrib);
    double acc = 0.0;
    for (int j = 0; j < b; j++) acc += density[j] * contrib[(j - s) + (b - 1)];
    *out = acc;
    free(counts);
    return EQO_OK;
}

/* uniform.py:60-80 quantize_uniform; aux 0 = fp32, 1 = fp16 (uniform.py:19-35).
 * scale/bias are written as the stored aux value (little-endian bytes). */
int eqo_quantize_uniform(const float *xf, long d, double xmin, double xmax, int nbits, int aux,
                         uint8_t *codes, void *scale_out, void *bias_out) {
    if (nbits != 4 && nbits != 8) return EQO_ENBITS;
    double qmax = (double)((1 << nbits) - 1);
    double scale_d, bias_d = xmin;
    if (xmax == xmin) {                                          /* uniform.py:74-76 */
        for (long i = 0; i < d; i++) codes[i] = 0;
        scale_d = 0.0;
    } else {
        scale_d = (xmax - xmin) / qmax;                           /* uniform.py:77 */
        for (long i = 0; i < d; i++) {
            double c = np_clip((double)xf[i], xmin, xmax);        /* uniform.py:78 */
            double code = np_clip(floor((c - xmin) / scale_d + 0.5), 0.0, qmax); /* :79 */
            codes[i] = (uint8_t)code;
        }
    }
    if (aux == 1) {                                               /* np.float16(x): one RNE rounding */
        _Float16 s = (_Float16)scale_d, bb = (_Float16)bias_d;
        memcpy(scale_out, &s, 2);
        memcpy(bias_out, &bb, 2);
    } else {                                                      /* np.float32(x) */
        float s = (float)scale_d, bb = (float)bias_d;
        memcpy(scale_out, &s, 4);
        memcpy(bias_out, &bb, 4);
    }
    return EQO_OK;
}

/* packed.py:32-33 packed_row_stride */
long eqo_packed_row_stride(long d, int aux) { return (d + 1) / 2 + 2 * (aux == 1 ? 2 : 4); }

/* packed.py:68-83 pack_table4 for one row: nibbles (even j low), scale, bias. */
static void pack_row(const uint8_t *codes, long d, int aux, const void *scale, const void *bias,
                     uint8_t *out) {
    long half = (d + 1) / 2;
    for (long k = 0; k < half; k++) {
        uint8_t lo4 = codes[2 * k];
        uint8_t hi4 = (2 * k + 1 < d) ? codes[2 * k + 1] : 0;   /* packed.py:75-76 odd-d pad */
        out[k] = (uint8_t)(lo4 | (hi4 << 4));                   /* packed.py:77 */
    }
    int ab = aux == 1 ? 2 : 4;
    memcpy(out + half, scale, ab);                              /* packed.py:79-82 */
    memcpy(out + half + ab, bias, ab);
}

int eqo_pack_table4(const uint8_t *codes, long rows, long d, int aux, const void *scales,
                    const void *biases, uint8_t *out) {
    long stride = eqo_packed_row_stride(d, aux);
    int ab = aux == 1 ? 2 : 4;
    for (long i = 0; i < rows; i++)
        pack_row(codes + i * d, d, aux, (const uint8_t *)scales + i * ab,
                 (const uint8_t *)biases + i * ab, out + i * stride);
    return EQO_OK;
}

/* Table driver == pack_table4(quantize_table(EmbeddingTable(x), method, 4, aux, b, r)).
 * methods.py:63-89 (per-row strategy loop) + uniform.py:142-167 + packed.py:68-83.
 * Optional per-row outputs (NULL to skip):
 *   lo/hi      f64 thresholds (ClipRange)
 *   info0/info1  greedy: iterations / -; hist-brute: start_bin / nbins_selected
 *   norm       hist-brute window norm
 * Returns the first error code over rows (rows are independent). */
static int table_impl(const float *x, long rows, long d, long ld, int method, int b, double r,
                      int aux, uint8_t *packed, double *lo_out, double *hi_out, int32_t *info0,
                      int32_t *info1, double *norm_out, double *gap_lr, double *gap_best,
                      int nthreads);

int eqo_quantize_pack_table(const float *x, long rows, long d, long ld, int method, int b,
                            double r, int aux, uint8_t *packed, double *lo_out, double *hi_out,
                            int32_t *info0, int32_t *info1, double *norm_out, int nthreads) {
    return table_impl(x, rows, d, ld, method, b, r, aux, packed, lo_out, hi_out, info0, info1,
                      norm_out, NULL, NULL, nthreads);
}

/* Same, plus GREEDY's per-row smallest near-tie gaps (greedy_impl) -- the parity report. */
int eqo_quantize_pack_table_gaps(const float *x, long rows, long d, long ld, int method, int b,
                                 double r, int aux, uint8_t *packed, double *lo_out,
                                 double *hi_out, int32_t *info0, int32_t *info1, double *norm_out,
                                 double *gap_lr, double *gap_best, int nthreads) {
    return table_impl(x, rows, d, ld, method, b, r, aux, packed, lo_out, hi_out, info0, info1,
                      norm_out, gap_lr, gap_best, nthreads);
}

static int table_impl(const float *x, long rows, long d, long ld, int method, int b, double r,
                      int aux, uint8_t *packed, double *lo_out, double *hi_out, int32_t *info0,
                      int32_t *info1, double *norm_out, double *gap_lr, double *gap_best,
                      int nthreads) {
    if (rows < 1 || d < 1) return EQO_EEMPTY;
    if (method < 0 || method > 7) return EQO_EMETHOD;
    if (method == METHOD_GREEDY) {
        if (b < 1) return EQO_EB;
        if (!(0.0 < r && r <= 1.0)) return EQO_ER;
    }
    if ((method == METHOD_HIST_BRUTE || method == METHOD_HIST_APPRX) && b < 1) return EQO_EB;
    for (long i = 0; i < rows; i++)
        if (check_finite(x + i * ld, d)) return EQO_EFINITE;      /* table.py:28-29 */
    long stride = eqo_packed_row_stride(d, aux);
    int err = 0;
    double tlo = 0.0, thi = 0.0;                                  /* clipping.py:64-67 table range */
    if (method == METHOD_TABLE) {
        float a = x[0], bb = x[0];
        for (long i = 0; i < rows; i++)
            for (long k = 0; k < d; k++) {
                const float v = x[i * ld + k];
                if (v < a) a = v;
                if (v > bb) bb = v;
            }
        tlo = (double)a;
        thi = (double)bb;
    }
    long scratch_n = d > 5 * (long)b ? d : 5 * (long)b;
    if (scratch_n < 16) scratch_n = 16;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        double *scratch = (double *)malloc(sizeof(double) * (size_t)scratch_n);
        uint8_t *codes = (uint8_t *)malloc((size_t)d + 1);
        if (!scratch || !codes) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            err = EQO_EALLOC;
        } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
            for (long i = 0; i < rows; i++) {
                const float *row = x + i * ld;
                double lo = 0, hi = 0, nv = 0;
                int a0 = 0, a1 = 0, rc = 0;
                if (method == METHOD_ASYM) {
                    rc = eqo_clip_range_asym(row, d, &lo, &hi);
                } else if (method == METHOD_GREEDY) {
                    int bi, bj;
                    double g1 = INFINITY, g2 = INFINITY;
                    rc = greedy_impl(row, d, 4, b, r, &lo, &hi, &a0, &bi, &bj, scratch,
                                     gap_lr ? &g1 : NULL, gap_best ? &g2 : NULL);
                    a1 = bi;
                    if (gap_lr) gap_lr[i] = g1;
                    if (gap_best) gap_best[i] = g2;
                } else if (method == METHOD_HIST_BRUTE) {
                    long ce = 0, bv = 0;
                    rc = eqo_hist_brute(row, d, b, &lo, &hi, &a0, &a1, &nv, &ce, &bv, scratch);
                } else if (method == METHOD_HIST_APPRX) {
                    long ce = 0, bv = 0;
                    rc = eqo_hist_apprx(row, d, b, &lo, &hi, &a0, &a1, &nv, &ce, &bv, scratch);
                } else if (method == METHOD_SYM) {
                    rc = eqo_clip_range_sym(row, d, &lo, &hi);
                } else if (method == METHOD_ACIQ) {
                    rc = eqo_clip_range_aciq(row, d, scratch, &lo, &hi);
                } else if (method == METHOD_GSS) {
                    rc = eqo_clip_range_gss(row, d, 4, scratch, &lo, &hi, &a0);
                } else {
                    lo = tlo;
                    hi = thi;
                }
                if (!rc) {
                    uint8_t sb[4], bb[4];
                    rc = eqo_quantize_uniform(row, d, lo, hi, 4, aux, codes, sb, bb);
                    if (!rc) pack_row(codes, d, aux, sb, bb, packed + i * stride);
                }
                if (rc) {
#ifdef _OPENMP
#pragma omp critical
#endif
                    { if (!err) err = rc; }
                }
                if (lo_out) lo_out[i] = lo;
                if (hi_out) hi_out[i] = hi;
                if (info0) info0[i] = a0;
                if (info1) info1[i] = a1;
                if (norm_out) norm_out[i] = nv;
            }
        }
        free(scratch);
        free(codes);
    }
    return err;
}

/* ------------------------------------------------------------------------ */
/* codebook.py:35-137 row-wise KMEANS: kmeans_1d(x, 16, _uniform_grid(x), 100, 1e-7)
 * then _sorted_codebook.  Bit-exact float64 restatement:
 *  - <= 16 distinct values: centers = sorted distinct values padded with the
 *    largest, assignments = searchsorted (codebook.py:55-61);
 *  - Lloyd: argmin |v - c| (ties -> lower index), sse = np.sum((v - c[a])**2)
 *    (pairwise), members.mean() (pairwise sum of the members in index order / m),
 *    empty clusters keep their center, stop when max|new - old| < tol * spread,
 *    keep the best-scoring assignment (strict <), score the final update;
 *  - codebook sorted by a stable argsort, cast to the aux dtype; indices = rank.
 * codebook_out: 16 values at the aux width; idx_out: d bytes; *iters_out =
 * Lloyd rounds run (-1 for the distinct-value shortcut). scratch: 4*d doubles. */
#define KM_K 16

static int km_assign(const double *v, long d, const double *c, uint8_t *a) {
    for (long i = 0; i < d; i++) {
        double best = fabs(v[i] - c[0]);
        int bj = 0;
        for (int j = 1; j < KM_K; j++) {
            double t = fabs(v[i] - c[j]);
            if (t < best) { best = t; bj = j; }
        }
        a[i] = (uint8_t)bj;
    }
    return 0;
}

static double km_sse(const double *v, long d, const double *c, const uint8_t *a, double *tmp) {
    for (long i = 0; i < d; i++) {
        double e = v[i] - c[a[i]];
        tmp[i] = e * e;
    }
    return eqo_np_sum(tmp, d);
}

int eqo_kmeans_row(const float *x, long d, int aux, void *codebook_out, uint8_t *idx_out,
                   int *iters_out, double *scratch) {
    if (d <= 0) return EQO_EEMPTY;
    double *v = scratch, *tmp = scratch + d, *mem = scratch + 2 * d;
    for (long i = 0; i < d; i++) v[i] = (double)x[i];
    double centers[KM_K];
    uint8_t *assign = (uint8_t *)malloc((size_t)d * 2);
    if (!assign) return EQO_EALLOC;
    uint8_t *best_a = assign + d;
    /* distinct values (np.unique) */
    double uniq[KM_K + 1];
    int nu = 0;
    for (long i = 0; i < d && nu <= KM_K; i++) {
        int pos = 0;
        while (pos < nu && uniq[pos] < v[i]) pos++;
        if (pos < nu && uniq[pos] == v[i]) continue;
        if (nu < KM_K + 1) {
            for (int q = nu; q > pos; q--) uniq[q] = uniq[q - 1];
            uniq[pos] = v[i];
            nu++;
        }
    }
    int iters = -1;
    if (nu <= KM_K) {
        for (int j = 0; j < KM_K; j++) centers[j] = j < nu ? uniq[j] : uniq[nu - 1];
        for (long i = 0; i < d; i++) {
            int pos = 0;
            while (uniq[pos] < v[i]) pos++;            /* searchsorted, side='left' */
            best_a[i] = (uint8_t)pos;
        }
    } else {
        double lo = v[0], hi = v[0];
        for (long i = 1; i < d; i++) { if (v[i] < lo) lo = v[i]; if (v[i] > hi) hi = v[i]; }
        const double scale = (hi - lo) / (double)(KM_K - 1);   /* _uniform_grid */
        for (int j = 0; j < KM_K; j++) centers[j] = lo + scale * (double)j;
        const double spread = hi - lo;                          /* uniq[-1] - uniq[0] */
        double best_sse = INFINITY, best_c[KM_K];
        int it = 0;
        for (it = 0; it < 100; it++) {
            km_assign(v, d, centers, assign);
            double sse = km_sse(v, d, centers, assign, tmp);
            if (sse < best_sse) {
                best_sse = sse;
                memcpy(best_c, centers, sizeof centers);
                memcpy(best_a, assign, (size_t)d);
            }
            double nc[KM_K];
            memcpy(nc, centers, sizeof centers);
            for (int j = 0; j < KM_K; j++) {
                long m = 0;
                for (long i = 0; i < d; i++)
                    if (assign[i] == j) mem[m++] = v[i];
                if (m) nc[j] = eqo_np_sum(mem, m) / (double)m;
            }
            double movement = 0.0;
            for (int j = 0; j < KM_K; j++) {
                double t = fabs(nc[j] - centers[j]);
                if (t > movement) movement = t;
            }
            memcpy(centers, nc, sizeof centers);
            if (movement < 1e-7 * spread) break;
        }
        iters = it < 100 ? it + 1 : 100;
        km_assign(v, d, centers, assign);                       /* score the final update */
        double sse = km_sse(v, d, centers, assign, tmp);
        if (sse < best_sse) {
            memcpy(best_a, assign, (size_t)d);
        } else {
            memcpy(centers, best_c, sizeof centers);
        }
    }
    /* _sorted_codebook: stable argsort of the centers */
    int order[KM_K], rank[KM_K];
    for (int j = 0; j < KM_K; j++) order[j] = j;
    for (int j = 1; j < KM_K; j++) {                            /* stable insertion sort */
        int t = order[j], q = j - 1;
        while (q >= 0 && centers[order[q]] > centers[t]) { order[q + 1] = order[q]; q--; }
        order[q + 1] = t;
    }
    for (int j = 0; j < KM_K; j++) rank[order[j]] = j;
    for (int j = 0; j < KM_K; j++) {
        const double c = centers[order[j]];
        if (aux == 1) {
            _Float16 h = (_Float16)c;
            memcpy((uint8_t *)codebook_out + 2 * j, &h, 2);
        } else {
            float f = (float)c;
            memcpy((uint8_t *)codebook_out + 4 * j, &f, 4);
        }
    }
    for (long i = 0; i < d; i++) idx_out[i] = (uint8_t)rank[best_a[i]];
    if (iters_out) *iters_out = iters;
    free(assign);
    return EQO_OK;
}

int eqo_kmeans_table(const float *x, long rows, long d, long ld, int aux, void *codebooks,
                     uint8_t *indices, int32_t *iters, int nthreads) {
    if (rows < 1 || d < 1) return EQO_EEMPTY;
    for (long i = 0; i < rows; i++)
        if (check_finite(x + i * ld, d)) return EQO_EFINITE;
    int err = 0;
    const int ab = aux == 1 ? 2 : 4;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        double *scratch = (double *)malloc(sizeof(double) * (size_t)(4 * d + 16));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
        for (long i = 0; i < rows; i++) {
            int it = 0;
            int rc = scratch ? eqo_kmeans_row(x + i * ld, d, aux, (uint8_t *)codebooks + i * KM_K * ab,
                                              indices + i * d, &it, scratch) : EQO_EALLOC;
            if (iters) iters[i] = it;
            if (rc) {
#ifdef _OPENMP
#pragma omp critical
#endif
                { if (!err) err = rc; }
            }
        }
        free(scratch);
    }
    return err;
}

int eqo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* packed.py:202-221 sparse_lengths_sum_ref for a PackedTable4 source: for each
 * segment s (lengths[s] consecutive entries of indices), out[s, j] accumulates
 * float32(float32(scale) * float32(code) + float32(bias)) in query order,
 * starting from 0.0f (packed.py:185-201 _ref_row_value, nibble decoded from
 * the byte buffer; fp16 aux widened exactly).  PooledQuery validation
 * (packed.py:131-140) and _check_indices (packed.py:147-152) first:
 *   EQO_ELEN   a negative length
 *   EQO_ESUM   lengths do not sum to nidx (*bad_pos = the sum)
 *   EQO_EINDEX first out-of-range index at position *bad_pos
 * out [batch x d] float32.  Float arithmetic is float32 (no contraction). */
#define EQO_ELEN 9
#define EQO_ESUM 10
#define EQO_EINDEX 11

static float aux_to_f32(const uint8_t *p, int aux) {
    if (aux == 1) {
        _Float16 h;
        memcpy(&h, p, 2);
        return (float)h;
    }
    float f;
    memcpy(&f, p, 4);
    return f;
}

int eqo_sls4(const uint8_t *packed, long rows, long d, int aux, const int64_t *indices, long nidx,
             const int64_t *lengths, long batch, float *out, int64_t *bad_pos) {
    int64_t total = 0;
    for (long s = 0; s < batch; s++) {
        if (lengths[s] < 0) return EQO_ELEN;
        total += lengths[s];
    }
    if (total != nidx) {
        if (bad_pos) *bad_pos = total;
        return EQO_ESUM;
    }
    for (long p = 0; p < nidx; p++)
        if (indices[p] < 0 || indices[p] >= rows) {
            if (bad_pos) *bad_pos = p;
            return EQO_EINDEX;
        }
    const long stride = eqo_packed_row_stride(d, aux), half = (d + 1) / 2;
    const int ab = aux == 1 ? 2 : 4;
    long pos = 0;
    for (long s = 0; s < batch; s++) {
        float *o = out + s * d;
        for (long j = 0; j < d; j++) o[j] = 0.0f;
        for (int64_t t = 0; t < lengths[s]; t++, pos++) {
            const uint8_t *row = packed + indices[pos] * stride;
            const float scale = aux_to_f32(row + half, aux);
            const float bias = aux_to_f32(row + half + ab, aux);
            for (long j = 0; j < d; j++) {
                const uint8_t byte = row[j / 2];
                const float code = (float)((j % 2 == 0) ? (byte & 0x0F) : (byte >> 4));
                const float prod = scale * code;          /* rounded to float32 */
                const float v = prod + bias;              /* rounded to float32 */
                o[j] = o[j] + v;
            }
        }
    }
    return EQO_OK;
}
