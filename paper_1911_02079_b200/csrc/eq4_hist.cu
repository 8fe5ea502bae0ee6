// eq4_hist.cu -- HIST-BRUTE (histclip.py:136-178) window search on sm_100a.
//
// Reference: for every width n = 1..b and start s = 0..b-n the window's norm is
//   norm(s, n) = sum_j density[j] * contrib_n[j - s]            (histclip.py:157-161)
// with density = counts / w and contrib_n from _offset_unit_norms
// (histclip.py:85-109), which scales exactly as w^3 * U_n(k) with U_n the
// bin-width-1 table.  So norm = w^2 * sum_j counts[j] U_n(j - s) and the
// argmin does not depend on w.  U_n(k) has closed forms outside the window:
//   k < 0 :  ((k+1)^3 - k^3) / 3                (both ends clip to dst point 0)
//   k >= n:  ((k+1-n)^3 - (k-n)^3) / 3          (both ends clip to dst point 15)
// so the outside part of every window is a prefix/suffix sum over the
// non-empty bins (integer arithmetic, exact in float64), and only the bins
// inside the window need the U table:
//   norm / w^2 = (A3[s] + R3[s + n]) / 3 + sum_{s <= j < s+n} counts[j] U_n(j - s).
// The U table (b(b+1)/2 doubles) is built once per b on the device and cached.
// Work per row: b(b+1)/2 windows x (non-empty bins inside) fused
// multiply-adds instead of the reference's b * b(b+1)/2 bin visits.
//
// Float64 throughout; the first minimum in (n ascending, s ascending) order is
// kept (histclip.py:165-168) with a lexicographic warp reduction.  The
// reference's norms come from BLAS dot products whose summation order is CPU
// specific, so only windows whose norms tie to ~1e-13 relative can select
// differently.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>

#include "../../include/eq4.h"
#include "eq4_device.cuh"
#include "eq4_internal.h"

namespace eq4 {

__device__ __forceinline__ double cube(double x) { return __dmul_rn(__dmul_rn(x, x), x); }

// histclip.py:70-82 bin_l2_norm with density 1
__device__ __forceinline__ double l2unit(double db, double de) {
  return __ddiv_rn(__dsub_rn(cube(de), cube(db)), 3.0);
}

// U[(n-1)n/2 + k] = _offset_unit_norms(k, 1, n/15) for k in [0, n)   (histclip.py:85-109)
__global__ void k_hist_table(int b, double* U) {
  const int n = blockIdx.x + 1;
  if (n > b) return;
  const double dst_w = __ddiv_rn((double)n, 15.0);   // histclip.py:158 (w * n / 15, w = 1)
  const double half = __dmul_rn(0.5, dst_w);
  double* Un = U + (size_t)(n - 1) * n / 2;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double begin = (double)k, end = __dadd_rn(begin, 1.0);
    const double dob = np_clip(floor(__ddiv_rn(__dadd_rn(begin, half), dst_w)), 0.0, 15.0);
    const double doe = np_clip(floor(__ddiv_rn(__dadd_rn(end, half), dst_w)), 0.0, 15.0);
    const double bc = __dmul_rn(dob, dst_w), ec = __dmul_rn(doe, dst_w);
    const double db = __dsub_rn(begin, bc);
    const double same = l2unit(db, __dsub_rn(end, bc));
    const double split = __dadd_rn(__dadd_rn(l2unit(db, half),
                                             __dmul_rn(__dsub_rn(__dsub_rn(doe, dob), 1.0),
                                                       l2unit(-half, half))),
                                   l2unit(-half, __dsub_rn(end, ec)));
    Un[k] = (dob == doe) ? same : split;
  }
}

struct HistParams {
  const float* x;
  int64_t rows, ld;
  int d, b, aux, stride, half;
  uint8_t* packed;
  double *lo_out, *hi_out, *norm_out;
  int32_t *info0, *info1, *status;
  const double* U;
  int wide;   // rows read from global memory (too wide to stage)
};

// codes (uniform.py:60-80) + packed row (packed.py:68-83) + per-row outputs.  Warp-collective.
__device__ __forceinline__ void hist_emit(const HistParams& p, int64_t row, int d, int lane, bool bad,
                                          const float* xs, uint8_t* codes, double wlo, double whi,
                                          int best_s, int best_n, double norm) {
  const bool ok = !bad;
  const CodeParams cp = make_code_params(ok ? wlo : 0.0, ok ? whi : 0.0);
  uint8_t* orow = p.packed + row * (int64_t)p.stride;
  if (p.wide) {   // element pairs straight to packed bytes (no staging)
    for (int m = lane; m < p.half; m += 32) {
      unsigned c0 = 0u, c1 = 0u;
      if (ok) {
        bool ne;
        c0 = code_of(xs[2 * m], cp, ne);
        if (ne) c0 = code_exact(xs[2 * m], cp);
        if (2 * m + 1 < d) {
          c1 = code_of(xs[2 * m + 1], cp, ne);
          if (ne) c1 = code_exact(xs[2 * m + 1], cp);
        }
      }
      orow[m] = (uint8_t)(c0 | (c1 << 4));
    }
  } else {
    for (int k = lane; k < d; k += 32) {
      bool ne;
      unsigned c = code_of(xs[k], cp, ne);
      if (ne) c = code_exact(xs[k], cp);
      codes[k] = ok ? (uint8_t)c : 0;
    }
    __syncwarp();
    for (int m = lane; m < p.half; m += 32) {
      const unsigned c0 = codes[2 * m];
      const unsigned c1 = (2 * m + 1 < d) ? codes[2 * m + 1] : 0u;
      orow[m] = (uint8_t)(c0 | (c1 << 4));
    }
  }
  if (lane == 0) {
    const double sc = (ok && whi != wlo) ? div15(__dsub_rn(whi, wlo)) : 0.0;
    uint8_t* a = orow + p.half;
    if (p.aux == EQ4_AUX_FP16) {
      const uint32_t s16 = aux_bits_f16(sc), b16 = aux_bits_f16(wlo);
      a[0] = s16 & 0xff; a[1] = s16 >> 8; a[2] = b16 & 0xff; a[3] = b16 >> 8;
    } else {
      const uint32_t s32 = aux_bits_f32(sc), b32 = aux_bits_f32(wlo);
      for (int k = 0; k < 4; ++k) { a[k] = (s32 >> (8 * k)) & 0xff; a[4 + k] = (b32 >> (8 * k)) & 0xff; }
    }
    if (p.lo_out) { p.lo_out[row] = wlo; p.hi_out[row] = whi; }
    if (p.info0) p.info0[row] = best_s;
    if (p.info1) p.info1[row] = best_n;
    if (p.norm_out) p.norm_out[row] = norm;
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// k_hist: one warp per row (8 row-warps per block), lanes over start bins.  The
// per-row preparation is warp-parallel: non-empty bins by ballot compaction,
// and the outside-window sums from prefix sums of c, c*j, c*j^2 over the bins:
//   3L(t) = sum_{j<t} c_j (3m^2 - 3m + 1), m = t - j
//         = P0 (3t^2 - 3t + 1) + P1 (3 - 6t) + 3 P2          (P = prefix sums over j < t)
//   3R(t) = sum_{j>=t} c_j (3k^2 + 3k + 1), k = j - t
//         = (T0-P0)(3t^2 - 3t + 1) + (T1-P1)(3 - 6t) + 3(T2-P2)
// all exact integers in float64.  A window's value is one fma of the outside
// part with the inside sum (fma over the non-empty bins inside, ascending).
// The U table stays in global memory (L1/L2): with the pruning below only ~2.5%
// of the windows reach the inside sum, and a shared-memory copy of U (160 KB at
// b = 200) cost more in occupancy than it saved (measured 0.724 vs 0.726 ms at
// d = 64, 1.76 vs 1.68 ms at d = 128).
// ---------------------------------------------------------------------------
// a non-empty bin: index and count (as a double), loaded with one 16-byte access
struct __align__(16) NzBin {
  int j, pad;
  double c;
};

struct HistSlice {
  int b, d, m;   // m = min(b, d): most non-empty bins a row can have
  __host__ __device__ size_t a3_off() const { return 0; }                                   // double[b+1]
  __host__ __device__ size_t r3_off() const { return a3_off() + (size_t)(b + 1) * 8; }      // double[b+1]
  __host__ __device__ size_t tmp_off() const { return r3_off() + (size_t)(b + 1) * 8; }     // double[b] (HIST-APPRX)
  __host__ __device__ size_t nz_off() const { return (tmp_off() + (size_t)b * 8 + 15) & ~(size_t)15; }   // NzBin[m]
  __host__ __device__ size_t cnt_off() const { return nz_off() + (size_t)m * 16; }          // int[b]
  __host__ __device__ size_t lb_off() const { return cnt_off() + (size_t)b * 4; }           // int[b+1]
  __host__ __device__ size_t xs_off() const { return lb_off() + (size_t)(b + 1) * 4; }      // float[d]
  __host__ __device__ size_t codes_off() const { return xs_off() + (wide ? 0 : (size_t)d * 4); }   // u8[d]
  __host__ __device__ size_t wq_off() const {                                                // int[64]
    return (codes_off() + (wide ? 0 : (size_t)d) + 15) & ~(size_t)15;
  }
  __host__ __device__ int leaves() const { return b / 64 + 2; }                             // numpy leaves of b terms
  __host__ __device__ size_t leaf_off() const { return wq_off() + 64 * 4; }                  // double + 2 int per leaf
  __host__ __device__ size_t bytes() const { return leaf_off() + (size_t)leaves() * 16; }
  bool wide;   // the row stays in global memory (xs / codes not staged)
};

__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v = __dadd_rn(v, t);
  }
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

constexpr double APPRX_TOL = 1e-11;   // relative gap below which the walk re-decides exactly

// HIST-APPRX (histclip.py:181-217): from the full window, drop one bin from the
// end whose removal scores lower (ties drop the right end), keeping the first
// best window seen.  Warp-collective, one row.  Each step scores its two
// windows (st + 1, nn) and (st, nn), nn = en - st - 1, with the brute scan's
// formula (outside part from A3/R3, inside sum over the non-empty bins with
// U_nn, lanes over bins, xor-butterfly sum so every lane holds the same value;
// w^2 dropped).  Those values are within ~1e-13 relative of the reference's
// window_norm, so a comparison whose operands differ by more than APPRX_TOL
// relative is the reference's; a closer one is re-decided on the reference's
// own float64 values (apprx_norm_np_warp: its elementwise formula in numpy's
// pairwise order), as is the reported norm of the chosen window.
__device__ __forceinline__ void hist_apprx_walk(const double* Us, const double* A3, const double* R3,
                                                const NzBin* nz, const int* cnt,
                                                double* tmp, int m, int b, double w, int lane, int& best_s,
                                                int& best_n, double& norm, double* leaf_sum, int* leaf_st,
                                                int* leaf_ln, int max_leaves) {
  auto exact = [&](int s0, int n0) -> double {
    return apprx_norm_np_warp(cnt, b, w, s0, n0, tmp, lane, leaf_sum, leaf_st, leaf_ln, max_leaves);
  };
  int st = 0, en = b;
  double bestF;
  {
    const double* Ub = Us + (size_t)(b - 1) * b / 2;
    double a = 0.0;
    for (int i = lane; i < m; i += 32) a = fma(nz[i].c, Ub[nz[i].j], a);
    bestF = __fma_rn(__dadd_rn(A3[0], R3[b]), 1.0 / 3.0, warp_sum_d(a));
  }
  double bestN = 0.0;
  bool have_bestN = false;
  int bs = 0, be = b;
  while (en - st > 1) {                                              // histclip.py:202
    const int nn = en - st - 1;
    const double* Un = Us + (size_t)(nn - 1) * nn / 2;
    double aL = 0.0, aR = 0.0;
    for (int i = lane; i < m; i += 32) {
      const NzBin e = nz[i];
      const int j = e.j;
      const double c = e.c;
      const int kL = j - st - 1, kR = j - st;
      if ((unsigned)kL < (unsigned)nn) aL = fma(c, Un[kL], aL);
      if ((unsigned)kR < (unsigned)nn) aR = fma(c, Un[kR], aR);
    }
    // both sums with one transposing butterfly: the first level trades halves (lanes < 16
    // keep L, the others R), four more levels finish each sum within its half
    const bool upper = lane >= 16;
    double keep = upper ? aR : aL;
    keep = __dadd_rn(keep, __shfl_xor_sync(FULL, upper ? aL : aR, 16));
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) keep = __dadd_rn(keep, __shfl_xor_sync(FULL, keep, o));
    const double FL = __fma_rn(__dadd_rn(A3[st + 1], R3[en]), 1.0 / 3.0, __shfl_sync(FULL, keep, 0));
    const double FR = __fma_rn(__dadd_rn(A3[st], R3[en - 1]), 1.0 / 3.0, __shfl_sync(FULL, keep, 16));
    bool goL, have_cur = false;
    double curN = 0.0;
    if (fabs(FL - FR) > APPRX_TOL * fmax(FL, FR)) {
      goL = FL < FR;
    } else {
      const double NL = exact(st + 1, nn), NR = exact(st, nn);
      goL = NL < NR;                                                 // histclip.py:205-206
      curN = goL ? NL : NR;
      have_cur = true;
    }
    const double curF = goL ? FL : FR;
    if (goL) ++st; else --en;
    bool better;
    if (fabs(curF - bestF) > APPRX_TOL * fmax(curF, bestF)) {
      better = curF < bestF;
    } else {
      if (!have_cur) { curN = exact(st, en - st); have_cur = true; }
      if (!have_bestN) { bestN = exact(bs, be - bs); have_bestN = true; }
      better = curN < bestN;                                         // histclip.py:211-213
    }
    if (better) {
      bestF = curF; bs = st; be = en;
      bestN = curN; have_bestN = have_cur;
    }
  }
  if (!have_bestN) bestN = exact(bs, be - bs);
  best_s = bs;
  best_n = be - bs;
  norm = bestN;
}

constexpr int HIST_NW = 8;   // row-warps per block

template <bool APPRX>
__global__ void __launch_bounds__(32 * HIST_NW) k_hist(const HistParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int b = p.b, d = p.d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const HistSlice S{b, d, min(b, d), p.wide != 0};
  const double* Us = p.U;   // L1/L2-resident (160 KB at b = 200)
  unsigned char* ws = smem + (size_t)warp * S.bytes();
  double* A3 = reinterpret_cast<double*>(ws + S.a3_off());
  double* R3 = reinterpret_cast<double*>(ws + S.r3_off());
  NzBin* nz = reinterpret_cast<NzBin*>(ws + S.nz_off());
  int* cnt = reinterpret_cast<int*>(ws + S.cnt_off());
  int* lb = reinterpret_cast<int*>(ws + S.lb_off());
  float* xs_s = reinterpret_cast<float*>(ws + S.xs_off());
  uint8_t* codes = ws + S.codes_off();
  int* wq = reinterpret_cast<int*>(ws + S.wq_off());
  double* leaf_sum = reinterpret_cast<double*>(ws + S.leaf_off());
  int* leaf_st = reinterpret_cast<int*>(leaf_sum + S.leaves());
  int* leaf_ln = leaf_st + S.leaves();

  for (int64_t row = (int64_t)blockIdx.x * nw + warp; row < p.rows; row += (int64_t)gridDim.x * nw) {
    // ---- row, min/max, finiteness ----
    float mn = INFINITY, mx = -INFINITY;
    bool bad = false;
    // the row: staged in shared memory, or read from global memory when it is too wide
    const float* xs = S.wide ? p.x + row * p.ld : xs_s;
    for (int k = lane; k < d; k += 32) {
      const float v = p.x[row * p.ld + k];
      if (!S.wide) xs_s[k] = v;
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
      bad |= !isfinite(v);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(FULL, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
    }
    bad = __any_sync(FULL, bad);
    if (bad && lane == 0 && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
    if (mn == 0.f || mx == 0.f) {   // rare: numpy's signed-zero choice (histclip.py:57)
      unsigned kz = 0u;
      for (int k = lane; k < d; k += 32) kz = max(kz, np_zero_key(xs[k], k, d));
      np_zero_apply(__reduce_max_sync(FULL, kz), mn, mx);
    }
    const double lo = (double)mn, hi = (double)mx;
    double wlo = lo, whi = hi, norm = 0.0;
    int best_s = 0, best_n = 1;
    if (!bad && lo != hi) {
      // ---- histogram (histclip.py:52-67), float64 bin index ----
      const double w = __ddiv_rn(__dsub_rn(hi, lo), (double)b);
      for (int j = lane; j < b; j += 32) cnt[j] = 0;
      __syncwarp();
      for (int k = lane; k < d; k += 32) {
        const double q = floor(__ddiv_rn(__dsub_rn((double)xs[k], lo), w));
        const int idx = (int)np_clip(q, 0.0, (double)(b - 1));
        atomicAdd(&cnt[idx], 1);
      }
      __syncwarp();
      // ---- non-empty bins by ballot compaction; lb[x] = #non-empty bins below x ----
      int m = 0;
      double t1 = 0.0, t2 = 0.0;
      for (int base = 0; base < b; base += 32) {
        const int j = base + lane;
        const int c = j < b ? cnt[j] : 0;
        const unsigned bal = __ballot_sync(FULL, c != 0);
        const int pos = m + __popc(bal & ((1u << lane) - 1u));
        if (j < b) lb[j] = pos;
        if (c) nz[pos] = NzBin{j, 0, (double)c};
        t1 += (double)c * j;
        t2 += (double)c * j * j;
        m += __popc(bal);
      }
      if (lane == 0) lb[b] = m;
      const double T0 = (double)d, T1 = warp_sum_d(t1), T2 = warp_sum_d(t2);
      // ---- outside-window parts 3L(t), 3R(t) for t = 0..b from prefix sums ----
      double c0 = 0.0, c1 = 0.0, c2 = 0.0;   // carries: sums over bins below the chunk
      for (int base = 0; base <= b; base += 32) {
        const int t = base + lane;
        const double c = (t < b) ? (double)cnt[t] : 0.0;
        const double i0 = warp_incl_scan(c, lane), i1 = warp_incl_scan(c * t, lane),
                     i2 = warp_incl_scan(c * t * t, lane);
        const double P0 = c0 + (i0 - c), P1 = c1 + (i1 - c * t), P2 = c2 + (i2 - c * t * t);
        const double tt = (double)t;
        const double q2 = 3.0 * tt * tt - 3.0 * tt + 1.0, q1 = 3.0 - 6.0 * tt;
        if (t <= b) {
          A3[t] = P0 * q2 + P1 * q1 + 3.0 * P2;
          R3[t] = (T0 - P0) * q2 + (T1 - P1) * q1 + 3.0 * (T2 - P2);
        }
        c0 += __shfl_sync(FULL, i0, 31);
        c1 += __shfl_sync(FULL, i1, 31);
        c2 += __shfl_sync(FULL, i2, 31);
      }
      __syncwarp();
      if constexpr (APPRX) {
        hist_apprx_walk(Us, A3, R3, nz, cnt, reinterpret_cast<double*>(ws + S.tmp_off()), m, b, w, lane,
                        best_s, best_n, norm, leaf_sum, leaf_st, leaf_ln, S.leaves());
        wlo = __dadd_rn(lo, __dmul_rn(w, (double)best_s));          // histclip.py:214-219
        whi = __dadd_rn(lo, __dmul_rn(w, (double)(best_s + best_n)));
      } else {
      // ---- every window, first minimum in (n asc, s asc) order ----
      // Pruning: v = (A3 + R3)/3 + acc with acc >= 0, so a window whose outside
      // part alone exceeds a value some window attains cannot be the minimum
      // (strict >, so equal values -- first-minimum ties -- are still scored).
      // The bound starts at the full window's value (scored exactly as the scan
      // scores it) and tightens to (an upper bound of) the warp's running minimum after
      // every width.
      double bound;
      {
        const double* Ub = Us + (size_t)(b - 1) * b / 2;
        double acc = 0.0;
        if (lane == 0)
          for (int i = 0; i < m; i++) acc = fma(nz[i].c, Ub[nz[i].j], acc);
        bound = __shfl_sync(FULL, __fma_rn(__dadd_rn(A3[0], R3[b]), 1.0 / 3.0, acc), 0);
      }
      // Widths below n0 are skipped whole: the outside part o(s, n) is
      // non-increasing in n (R3 falls as the window's right end moves right), so
      // min_s o(s, n) is too, and n0 = the first width where a lower bound of it
      // (warp minimum of the high words, low word zero) is <= bound.  o(0, b) = 0.
      int n0 = 1;
      {
        int nhi = b;
        while (n0 < nhi) {
          const int mid = (n0 + nhi) >> 1;
          double mo = INFINITY;
          for (int s = lane; s <= b - mid; s += 32)
            mo = fmin(mo, __dmul_rn(__dadd_rn(A3[s], R3[s + mid]), 1.0 / 3.0));
          const unsigned hw = __reduce_min_sync(FULL, (unsigned)__double2hiint(mo));
          if (__hiloint2double((int)hw, 0) > bound) n0 = mid + 1; else nhi = mid;
        }
      }
      // Surviving windows are sparse (a few % of the starts of a width), so they
      // are queued as packed (n << 16 | s) in (n asc, s asc) order and scored 32 at
      // a time, one per lane, instead of idling most lanes of a width's pass.  The
      // bound tightens after every batch.
      double bv = INFINITY;
      int bn = 1 << 30, bs = 1 << 30;
      int qn = 0;   // queued windows (warp-uniform)
      auto score_batch = [&](int count) {
        if (lane < count) {
          const int qe = wq[lane];
          const int n = qe >> 16, s = qe & 0xffff;
          const double* Ub = Us + (size_t)(n - 1) * n / 2 - s;
          double acc = 0.0;
          const int i1 = lb[s + n];
#pragma unroll 4
          for (int i = lb[s]; i < i1; i++) {
            const NzBin nb = nz[i];   // one 16-byte load
            acc = fma(nb.c, Ub[nb.j], acc);
          }
          const double v = __fma_rn(__dadd_rn(A3[s], R3[s + n]), 1.0 / 3.0, acc);   // one rounding
          if (v < bv || (v == bv && (n < bn || (n == bn && s < bs)))) { bv = v; bn = n; bs = s; }
        }
        // values are >= 0, so their high words order like the values: the warp
        // minimum of the high words, low word all ones, bounds the minimum from above
        const unsigned hw = __reduce_min_sync(FULL, (unsigned)__double2hiint(bv));
        bound = fmin(bound, __hiloint2double((int)hw, (int)0xffffffffu));
      };
      for (int n = n0; n <= b; n++) {
        for (int s0 = 0; s0 <= b - n; s0 += 32) {
          const int s = s0 + lane;
          const bool keep = s <= b - n &&
                            !(__dmul_rn(__dadd_rn(A3[s], R3[s + n]), 1.0 / 3.0) > bound);   // o <= v
          const unsigned bal = __ballot_sync(FULL, keep);
          if (keep) wq[qn + __popc(bal & ((1u << lane) - 1u))] = (n << 16) | s;
          qn += __popc(bal);
          __syncwarp();
          if (qn >= 32) {
            score_batch(32);
            const int rest = lane < qn - 32 ? wq[32 + lane] : 0;
            __syncwarp();
            if (lane < qn - 32) wq[lane] = rest;
            qn -= 32;
            __syncwarp();
          }
        }
      }
      if (qn > 0) score_batch(qn);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const double ov = __shfl_xor_sync(FULL, bv, o);
        const int on = __shfl_xor_sync(FULL, bn, o), os = __shfl_xor_sync(FULL, bs, o);
        if (ov < bv || (ov == bv && (on < bn || (on == bn && os < bs)))) { bv = ov; bn = on; bs = os; }
      }
      best_s = bs;
      best_n = bn;
      wlo = __dadd_rn(lo, __dmul_rn(w, (double)bs));                 // histclip.py:170
      whi = __dadd_rn(lo, __dmul_rn(w, (double)(bs + bn)));
      norm = bv * w * w;
      }
    }
    hist_emit(p, row, d, lane, bad, xs, codes, wlo, whi, best_s, best_n, norm);
  }
}

}  // namespace eq4

using namespace eq4;

// U tables cached per (device, b); built once with k_hist_table on the first
// caller's stream.  No host synchronisation: the build is followed by an event,
// and every call (on any stream) waits on that event on the device before its
// k_hist launch -- a no-op once the table exists.
struct UTable {
  double* U = nullptr;
  cudaEvent_t ready = nullptr;
};
static std::mutex g_u_mu;
static std::map<std::pair<int, int>, UTable> g_u_tables;

static const double* hist_table(int b, cudaStream_t s, std::string& err) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_u_mu);
  auto key = std::make_pair(dev, b);
  auto it = g_u_tables.find(key);
  if (it == g_u_tables.end()) {
    UTable t;
    cudaError_t e = cudaMalloc(&t.U, sizeof(double) * (size_t)b * (b + 1) / 2);
    if (e != cudaSuccess) { err = std::string("cudaMalloc U: ") + cudaGetErrorString(e); return nullptr; }
    k_hist_table<<<b, 128, 0, s>>>(b, t.U);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&t.ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(t.ready, s);
    if (e != cudaSuccess) {
      err = std::string("U table: ") + cudaGetErrorString(e);
      cudaFree(t.U);
      if (t.ready) cudaEventDestroy(t.ready);
      return nullptr;
    }
    it = g_u_tables.emplace(key, t).first;
  }
  const cudaError_t e = cudaStreamWaitEvent(s, it->second.ready, 0);
  if (e != cudaSuccess) { err = std::string("U table wait: ") + cudaGetErrorString(e); return nullptr; }
  return it->second.U;
}

int eq4_hist_launch(const float* x, int64_t rows, int64_t dim, int64_t ld, int b, int aux,
                    uint8_t* packed, double* xmin, double* xmax, int32_t* info0, int32_t* info1,
                    double* norm, int32_t* status, cudaStream_t s, std::string& err, bool apprx) {
  if (b > 65535) { err = "hist with b > 65535 is not supported by the B200 path"; return EQ4_EUNSUPPORTED; }
  const double* U = hist_table(b, s, err);
  if (!U) return EQ4_ECUDA;
  HistParams p;
  p.x = x; p.rows = rows; p.ld = ld; p.d = (int)dim; p.b = b; p.aux = aux;
  p.stride = (int)eq4_packed_row_stride(dim, aux);
  p.half = (int)((dim + 1) / 2);
  p.packed = packed; p.lo_out = xmin; p.hi_out = xmax; p.norm_out = norm;
  p.info0 = info0; p.info1 = info1; p.status = status; p.U = U;
  int dev = 0, sms = 148, max_optin = 227 * 1024;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  HistSlice SS{b, (int)dim, (int)std::min<int64_t>(b, dim), false};
  if (SS.bytes() > (size_t)max_optin / 2) SS.wide = true;   // wide rows stay in global memory
  p.wide = SS.wide ? 1 : 0;
  const size_t per = SS.bytes();
  if (per > (size_t)max_optin) {
    err = "hist: the b-bin tables of a row do not fit in shared memory (b too large)";
    return EQ4_EUNSUPPORTED;
  }
  const int nw = (int)std::max<size_t>(1, std::min<size_t>(HIST_NW, max_optin / per));
  const size_t smem = (size_t)nw * per;
  auto kern = apprx ? k_hist<true> : k_hist<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nw * 32, smem);
  if (occ < 1) occ = 1;
  const int64_t need = (rows + nw - 1) / nw;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * occ));
  kern<<<(unsigned)grid, nw * 32, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) { err = std::string("k_hist launch: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  return EQ4_OK;
}
