// eq4_rowrange.cu -- ACIQ and GSS row-range searches fused with the codec and
// the packer (clipping.py:70-139).
//
// Both searches are float64 computations whose every comparison must match the
// reference bit for bit:
//   ACIQ (laplacian, the branch row_clip_range uses): mean = np.mean(x),
//     alpha = 5.03 * np.mean(|x - mean|)  (numpy pairwise sums / n),
//     range (mean - alpha, mean + alpha), or the data range when alpha == 0;
//   GSS (tol 1e-4): golden-section search over t in (0, max|x|] of
//     quant_mse(x, (-t, t), 4), keeping the best point evaluated (strict <),
//     ~23 exact float64 quant_mse evaluations per row.
// So they run lane-per-row: a warp stages 32 rows in shared memory as a
// conflict-free [d][33] column layout and every lane replays numpy's pairwise
// summation order for its own row sequentially (8 accumulator chains per
// <=128-element leaf, recursive halving n2 = n/2 - (n/2 % 8) above), 32 rows
// in flight per warp instead of one warp-cooperative row at a time.  Codes use
// the fp32 estimate of eq4_device.cuh (code_of) and the float64 codec only
// within NEAR of a rounding boundary, so every code is numpy's.
// Rows wider than 256 read their elements straight from global memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/eq4.h"
#include "eq4_device.cuh"
#include "eq4_internal.h"
#include "eq4_np.cuh"

namespace eq4 {

constexpr int RR_THREADS = 128;
constexpr int RR_WARPS = RR_THREADS / 32;
constexpr int RR_MAX_STAGED = 256;   // d above this reads global memory
constexpr int RR_COL = 33;           // padded column stride (floats) of the staged tile
constexpr float MAGIC_F = 8388608.f;  // 2^23: x + 2^23 rounded down leaves floor(x) in the low mantissa bits

struct RRParams {
  const float* x;
  int64_t rows, ld;
  int d, aux, stride, half, method;
  uint8_t* packed;
  double* lo_out;
  double* hi_out;
  int32_t* info0;
  int32_t* status;
  double invphi;     // (sqrt(5) - 1) / 2, clipping.py:27
  double aciq_const; // clipping.py:125-134: 5.03 (laplacian) or the caller's gaussian_constant
  double gss_tol;    // clipping.py:70 tol (default 1e-4)
  int staged;
  int direct;        // wide rows: packed rows written straight to global (no staging tile)
  int vec4;          // rows 16-byte aligned (d % 4 == 0, ld % 4 == 0, aligned base)
  size_t warp_bytes;
};

// Element k of this lane's row (float32 table rows; float64 for the scalar entry points).
template <typename T>
struct RowViewT {
  const T* base;
  int ks;
  __device__ __forceinline__ T operator[](int k) const { return base[(size_t)k * ks]; }
};
using RowView = RowViewT<float>;

// numpy's zero choice (np_zero_key) for an element of either width.
template <typename T>
__device__ __forceinline__ unsigned np_zero_key_t(T v, int p, int d) {
  if (v != (T)0) return 0u;
  return np_zero_key(signbit(v) ? -0.f : 0.f, p, d);
}

// table.py:81-103 quant_mse(x, (lo, hi), 4) of a float64 row, bit-exact (exact codec).
__device__ __forceinline__ double lane_quant_mse(const RowViewT<double>& xr, int d, double lo, double hi) {
  if (hi == lo) {
    return np_sum([&](int k) {
      const double e = __dsub_rn(xr[k], lo);
      return __dmul_rn(e, e);
    }, d);
  }
  const double scale = div15(__dsub_rn(hi, lo));
  return np_sum([&](int k) { return np_err2(xr[k], lo, hi, scale); }, d);
}

// table.py:81-103 quant_mse(x, (lo, hi), 4) of this lane's row, bit-exact.
__device__ __forceinline__ double lane_quant_mse(const RowView& xr, int d, double lo, double hi) {
  if (hi == lo) {
    return np_sum([&](int k) {
      const double e = __dsub_rn((double)xr[k], lo);
      return __dmul_rn(e, e);
    }, d);
  }
  const CodeParams cp = make_code_params(lo, hi);
  if (!cp.slow) {
    // branch-free fp32 codes (as the emit below: saturating scale, round-down add) with the
    // distance to a rounding boundary tracked; if any element came within NEAR of one, the
    // loss is recomputed with the exact codec (rare)
    const float inv1 = cp.inv * (1.f / 15.f);
    float gmax = 0.f;
    const double v = np_sum([&](int k) {
      const float xf = xr[k];
      const float sv = __saturatef(__fmul_rn(__fadd_rn(__fadd_rn(xf, -cp.lo_hi), -cp.lo_lo), inv1));
      const float m = __fadd_rd(__fmaf_rn(sv, 15.f, 0.5f), MAGIC_F);
      gmax = fmaxf(gmax, fabsf(__fmaf_rn(sv, 15.f, -__fadd_rn(m, -MAGIC_F))));
      const double c = (double)(__float_as_uint(m) & 0xFu);
      const double recon = __dadd_rn(__dmul_rn(cp.scale, c), lo);
      const double e = __dsub_rn((double)xf, recon);
      return __dmul_rn(e, e);
    }, d);
    if (!(gmax > 0.5f - NEAR)) return v;
  }
  // codes: fp32 estimate, float64 codec within NEAR of a rounding boundary (exact either way)
  return np_sum([&](int k) {
    const float xf = xr[k];
    bool ne;
    unsigned c = code_of(xf, cp, ne);
    if (ne) c = code_exact(xf, cp);
    const double recon = __dadd_rn(__dmul_rn(cp.scale, (double)c), lo);
    const double e = __dsub_rn((double)xf, recon);
    return __dmul_rn(e, e);
  }, d);
}

// clipping.py:115-139: alpha = constant * mean|x - mean| (5.03 laplacian, :125-126, or
// the caller's gaussian_constant, :127-134).
template <typename T>
__device__ __forceinline__ void lane_aciq(const RowViewT<T>& xr, int d, double mn, double mx,
                                          double constant, double& lo, double& hi) {
  const double n = (double)d;
  const double mean = __ddiv_rn(np_sum([&](int k) { return (double)xr[k]; }, d), n);
  const double mad = __ddiv_rn(np_sum([&](int k) { return fabs(__dsub_rn((double)xr[k], mean)); }, d), n);
  const double alpha = __dmul_rn(constant, mad);
  if (alpha == 0.0) {   // clipping.py:137-138 -> clip_range_asym (numpy's signed-zero choice)
    if (mn == 0.0 || mx == 0.0) {
      unsigned kz = 0u;
      for (int k = 0; k < d; k++) kz = max(kz, np_zero_key_t(xr[k], k, d));
      const double z = (kz & 1u) ? -0.0 : 0.0;
      if (mn == 0.0) mn = z;
      if (mx == 0.0) mx = z;
    }
    lo = mn;
    hi = mx;
  } else {
    lo = __dsub_rn(mean, alpha);
    hi = __dadd_rn(mean, alpha);
  }
}

// clipping.py:70-112; returns the number of quant_mse calls.
template <typename T>
__device__ __forceinline__ int lane_gss(const RowViewT<T>& xr, int d, double mn, double mx, double invphi,
                                        double tol, double& lo_out, double& hi_out) {
  const double tmax = fmax(fabs(mn), fabs(mx));
  if (tmax == 0.0) {
    lo_out = 0.0;
    hi_out = 0.0;
    return 0;
  }
  int n = 0;
  auto f = [&](double t) {
    ++n;
    return lane_quant_mse(xr, d, -t, t);
  };
  double best_t = tmax, best_f = f(tmax);
  double a = 0.0, b = tmax;
  double c = __dsub_rn(b, __dmul_rn(invphi, __dsub_rn(b, a)));
  double e = __dadd_rn(a, __dmul_rn(invphi, __dsub_rn(b, a)));
  double fc = f(c), fe = f(e);
  if (fc < best_f) { best_t = c; best_f = fc; }
  if (fe < best_f) { best_t = e; best_f = fe; }
  const double stop = __dmul_rn(tol, tmax);
  while (__dsub_rn(b, a) > stop) {
    if (fc < fe) {
      b = e; e = c; fe = fc;
      c = __dsub_rn(b, __dmul_rn(invphi, __dsub_rn(b, a)));
      fc = f(c);
      if (fc < best_f) { best_t = c; best_f = fc; }
    } else {
      a = c; c = e; fc = fe;
      e = __dadd_rn(a, __dmul_rn(invphi, __dsub_rn(b, a)));
      fe = f(e);
      if (fe < best_f) { best_t = e; best_f = fe; }
    }
  }
  lo_out = -best_t;
  hi_out = best_t;
  return n;
}

// one instantiation per method: GSS's float64 search state must not shape
// ACIQ's register allocation (ACIQ is a bandwidth-class path)
template <int METHOD>
__global__ void __launch_bounds__(RR_THREADS) k_rowrange(const RRParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ws = smem + (size_t)warp * p.warp_bytes;
  float* xs = reinterpret_cast<float*>(ws);
  const size_t xs_bytes = p.staged ? (size_t)p.d * RR_COL * 4 : 0;
  uint8_t* out_base = ws + ((xs_bytes + 15) & ~(size_t)15);
  const int d = p.d;
  const int64_t nblk = (p.rows + 31) / 32;
  for (int64_t blk = (int64_t)blockIdx.x * RR_WARPS + warp; blk < nblk;
       blk += (int64_t)gridDim.x * RR_WARPS) {
    const int64_t row0 = blk * 32, row = row0 + lane;
    const bool rvalid = row < p.rows;
    const int nrows = (int)min((int64_t)32, p.rows - row0);
    RowView xr;
    if (p.staged) {
      // lane r stages row row0 + r into column r: all of a lane's loads are
      // independent (16-byte loads, 8 in flight per group, when the rows are
      // 16-byte aligned), and the column stores are conflict-free
      if (p.vec4) {
        const float4* src = reinterpret_cast<const float4*>(p.x + (rvalid ? row : row0) * p.ld);
        const int n4 = d >> 2;
        for (int c0 = 0; c0 < n4; c0 += 8) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; u++)
            if (c0 + u < n4) v[u] = __ldcs(src + c0 + u);
#pragma unroll
          for (int u = 0; u < 8; u++)
            if (c0 + u < n4) {
              float* col = xs + (size_t)(4 * (c0 + u)) * RR_COL + lane;
              col[0] = v[u].x; col[RR_COL] = v[u].y; col[2 * RR_COL] = v[u].z; col[3 * RR_COL] = v[u].w;
            }
        }
      } else {
        const float* src = p.x + (rvalid ? row : row0) * p.ld;
        for (int k0 = 0; k0 < d; k0 += 8) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; u++)
            if (k0 + u < d) v[u] = __ldcs(src + k0 + u);
#pragma unroll
          for (int u = 0; u < 8; u++)
            if (k0 + u < d) xs[(size_t)(k0 + u) * RR_COL + lane] = v[u];
        }
      }
      __syncwarp();
      xr.base = xs + lane;
      xr.ks = RR_COL;
    } else {
      xr.base = p.x + (rvalid ? row : row0) * p.ld;
      xr.ks = 1;
    }
    // row min / max / finiteness (table.py:28-29)
    float mn = INFINITY, mx = -INFINITY;
    bool bad = false;
    if (rvalid) {
      for (int k = 0; k < d; k++) {
        const float v = xr[k];
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
        bad |= !isfinite(v);
      }
      if (bad && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
    }
    double lo = 0.0, hi = 0.0;
    int evals = 0;
    if (rvalid && !bad) {
      if constexpr (METHOD == EQ4_METHOD_ACIQ) {
        lane_aciq(xr, d, (double)mn, (double)mx, p.aciq_const, lo, hi);
      } else {
        evals = lane_gss(xr, d, (double)mn, (double)mx, p.invphi, p.gss_tol, lo, hi);
      }
    }
    // codes (uniform.py:60-80) + packed row (packed.py:68-83), staged then copied out
    uint8_t* out_tile = out_base + (((uintptr_t)p.packed + (size_t)row0 * p.stride) & 15);
    if (rvalid) {
      uint8_t* orow = p.direct ? p.packed + (size_t)row * p.stride : out_tile + (size_t)lane * p.stride;
      const bool degenerate = bad || hi == lo;
      const CodeParams cp = make_code_params(degenerate ? 0.0 : lo, degenerate ? 0.0 : hi);
      // Branch-free fp32 codes: s = sat((x - lo) / (hi - lo)) clamps below lo / above hi
      // (codes 0 / 15 there, as numpy's clip), code = floor(15 s + 1/2) by a round-down
      // add of 2^23, and g = 15 s - code tracks the distance to a rounding boundary.
      // A row with any element within NEAR of a boundary (or an extreme range) takes
      // the exact codec for every element (rare).
      bool exact_row = degenerate || cp.slow;
      if (!exact_row) {
        const float inv1 = cp.inv * (1.f / 15.f);
        float gmax = 0.f;
        for (int m = 0; m < p.half; m++) {
          const float x0 = xr[2 * m];
          const float x1 = (2 * m + 1 < d) ? xr[2 * m + 1] : cp.lo_hi;
          const float s0 = __saturatef(__fmul_rn(__fadd_rn(__fadd_rn(x0, -cp.lo_hi), -cp.lo_lo), inv1));
          const float s1 = __saturatef(__fmul_rn(__fadd_rn(__fadd_rn(x1, -cp.lo_hi), -cp.lo_lo), inv1));
          const float m0 = __fadd_rd(__fmaf_rn(s0, 15.f, 0.5f), MAGIC_F), m1 = __fadd_rd(__fmaf_rn(s1, 15.f, 0.5f), MAGIC_F);
          const float g0 = __fmaf_rn(s0, 15.f, -__fadd_rn(m0, -MAGIC_F));
          const float g1 = __fmaf_rn(s1, 15.f, -__fadd_rn(m1, -MAGIC_F));
          gmax = fmaxf(gmax, fmaxf(fabsf(g0), fabsf(g1)));
          const unsigned c0 = __float_as_uint(m0) & 0xFu;
          const unsigned c1 = (2 * m + 1 < d) ? (__float_as_uint(m1) & 0xFu) : 0u;   // packed.py:75-76
          orow[m] = (uint8_t)(c0 | (c1 << 4));
        }
        exact_row = gmax > 0.5f - NEAR;
      }
      if (exact_row) {
        for (int m = 0; m < p.half; m++) {
          unsigned c0 = 0, c1 = 0;
          if (!degenerate) {
            c0 = code_exact(xr[2 * m], cp);
            if (2 * m + 1 < d) c1 = code_exact(xr[2 * m + 1], cp);
          }
          orow[m] = (uint8_t)(c0 | (c1 << 4));
        }
      }
      const double sc = degenerate ? 0.0 : cp.scale;   // uniform.py:74-80
      uint8_t* a = orow + p.half;
      if (p.aux == EQ4_AUX_FP16) {
        const uint32_t s16 = aux_bits_f16(sc), b16 = aux_bits_f16(lo);
        a[0] = s16 & 0xff; a[1] = s16 >> 8; a[2] = b16 & 0xff; a[3] = b16 >> 8;
      } else {
        const uint32_t s32 = aux_bits_f32(sc), b32 = aux_bits_f32(lo);
        for (int k = 0; k < 4; ++k) { a[k] = (s32 >> (8 * k)) & 0xff; a[4 + k] = (b32 >> (8 * k)) & 0xff; }
      }
      if (p.lo_out) { p.lo_out[row] = lo; p.hi_out[row] = hi; }
      if (p.info0) p.info0[row] = evals;
    }
    __syncwarp();
    // warp copy of the staged packed rows (16-byte stores where aligned)
    if (!p.direct) {
      uint8_t* dst = p.packed + (size_t)row0 * p.stride;
      const int nbytes = nrows * p.stride;
      int head = (int)((16 - ((uintptr_t)dst & 15)) & 15);
      if (head > nbytes) head = nbytes;
      const int nvec = (nbytes - head) >> 4;
      const int tail = head + (nvec << 4);
      if (lane < head) dst[lane] = out_tile[lane];
      const uint4* s4 = reinterpret_cast<const uint4*>(out_tile + head);
      uint4* d4 = reinterpret_cast<uint4*>(dst + head);
      for (int i = lane; i < nvec; i += 32) d4[i] = s4[i];
      for (int i = tail + lane; i < nbytes; i += 32) dst[i] = out_tile[i];
    }
    __syncwarp();
  }
}

// ACIQ, cooperative (d % 8 == 0, 8 <= d <= 128: one numpy leaf, no remainder): eight lanes
// per row, four rows per warp.  numpy's leaf sum runs 8 sequential accumulator chains --
// chain j sums elements j, j+8, j+16, ... -- then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7));
// lane j of a row owns chain j (its elements are exactly j + 8k, loaded with 4-byte
// loads whose 8 lanes cover 32 contiguous bytes: every sector is used), and the tree is
// the xor-butterfly over the 8 lanes (IEEE addition commutes, so each level's pairs are
// numpy's).  Elements stay in registers for both sums and the codes; the nibble codes of
// a row are transposed across its 8 lanes (3 butterfly stages on 32-bit words) so lane t
// stores packed bytes 4t..4t+3 (elements 8t..8t+7) with one 32-bit store.
// One row of k_aciq8 (the lane's chain j), elements already loaded.
template <int NCH>
__device__ __forceinline__ void aciq8_row(const RRParams& p, const float (&x)[NCH], int64_t row, bool rvalid,
                                          int j, double n, double rn, bool pow2) {
  constexpr unsigned FULLM = 0xffffffffu;
  double xd[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) xd[k] = (double)x[k];
  // np.mean (clipping.py:135): chain j, then the leaf tree, then np.add.reduce's 0.0 +
  double r = xd[0];
#pragma unroll
  for (int k = 1; k < NCH; ++k) r = __dadd_rn(r, xd[k]);
  r = __dadd_rn(r, __shfl_xor_sync(FULLM, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(FULLM, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(FULLM, r, 4));
  const double sum = __dadd_rn(0.0, r);
  const bool bad = !isfinite(sum);   // a non-finite element (the float64 sum of floats cannot overflow)
  const double mean = pow2 ? __dmul_rn(sum, rn) : __ddiv_rn(sum, n);
  // np.mean(np.abs(x - mean)) (clipping.py:136)
  double a = fabs(__dsub_rn(xd[0], mean));
#pragma unroll
  for (int k = 1; k < NCH; ++k) a = __dadd_rn(a, fabs(__dsub_rn(xd[k], mean)));
  a = __dadd_rn(a, __shfl_xor_sync(FULLM, a, 1));
  a = __dadd_rn(a, __shfl_xor_sync(FULLM, a, 2));
  a = __dadd_rn(a, __shfl_xor_sync(FULLM, a, 4));
  const double sa = __dadd_rn(0.0, a);
  const double alpha = __dmul_rn(p.aciq_const, pow2 ? __dmul_rn(sa, rn) : __ddiv_rn(sa, n));
  double lo = __dsub_rn(mean, alpha), hi = __dadd_rn(mean, alpha);
  const bool flat = rvalid && !bad && alpha == 0.0;
  if (__any_sync(FULLM, flat)) {   // rare: clipping.py:137-138 -> clip_range_asym (numpy's zero choice)
    float mn = x[0], mx = x[0];
#pragma unroll
    for (int k = 1; k < NCH; ++k) { mn = fminf(mn, x[k]); mx = fmaxf(mx, x[k]); }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      mn = fminf(mn, __shfl_xor_sync(FULLM, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(FULLM, mx, o));
    }
    unsigned kz = 0u;
    if (mn == 0.f || mx == 0.f) {
#pragma unroll
      for (int k = 0; k < NCH; ++k) kz = max(kz, np_zero_key_t(x[k], j + 8 * k, p.d));
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) kz = max(kz, __shfl_xor_sync(FULLM, kz, o));
    if (flat) {
      const double z = (kz & 1u) ? -0.0 : 0.0;
      lo = mn == 0.f ? z : (double)mn;
      hi = mx == 0.f ? z : (double)mx;
    }
  }
  if (bad) { lo = 0.0; hi = 0.0; }
  // codes (uniform.py:60-80): branch-free fp32 estimate, the float64 codec for a lane's
  // elements when one of them lies within NEAR of a rounding boundary
  const bool degenerate = bad || hi == lo;
  const double w64 = __dsub_rn(hi, lo);
  const float lo_hi = __double2float_rn(lo), lo_lo = __double2float_rn(__dsub_rn(lo, (double)lo_hi));
  const float wf = __double2float_rn(w64);
  const float inv1 = degenerate ? 0.f : __fdividef(1.f, wf);
  // the estimate needs a normal, finite range (fast_codec's test, on the float copies)
  const bool slow = !degenerate && !(wf > 1e-30f && wf < 1e30f && fabsf(lo_hi) < 1e30f &&
                                     fabsf(__double2float_rn(hi)) < 1e30f);
  unsigned w[(NCH + 7) / 8];
#pragma unroll
  for (int g = 0; g < (NCH + 7) / 8; ++g) w[g] = 0u;
  float gmax = 0.f;
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const float sv = __saturatef(__fmul_rn(__fadd_rn(__fadd_rn(x[k], -lo_hi), -lo_lo), inv1));
    const float m = __fadd_rd(__fmaf_rn(sv, 15.f, 0.5f), 8388608.f);
    gmax = fmaxf(gmax, fabsf(__fmaf_rn(sv, 15.f, -__fadd_rn(m, -8388608.f))));
    w[k >> 3] |= (__float_as_uint(m) & 0xFu) << (4 * (k & 7));
  }
  const bool exact = rvalid && (degenerate || slow || gmax > 0.5f - NEAR);
  if (__any_sync(FULLM, exact) && exact) {
    const CodeParams cp = make_code_params(degenerate ? 0.0 : lo, degenerate ? 0.0 : hi);
#pragma unroll
    for (int g = 0; g < (NCH + 7) / 8; ++g) w[g] = 0u;
#pragma unroll
    for (int k = 0; k < NCH; ++k) w[k >> 3] |= code_exact(x[k], cp) << (4 * (k & 7));
  }
  // 8 x 8 nibble transpose across the row's lanes: lane t ends with nibble t of every lane
#pragma unroll
  for (int g = 0; g < (NCH + 7) / 8; ++g) {
#pragma unroll
    for (int b = 4; b >= 1; b >>= 1) {
      const unsigned msk = b == 4 ? 0x0000FFFFu : (b == 2 ? 0x00FF00FFu : 0x0F0F0F0Fu);
      const unsigned pw = __shfl_xor_sync(FULLM, w[g], b);
      w[g] = (j & b) ? (((pw & ~msk) >> (4 * b)) | (w[g] & ~msk)) : ((w[g] & msk) | ((pw & msk) << (4 * b)));
    }
  }
  if (rvalid) {
    uint8_t* orow = p.packed + (size_t)row * p.stride;
#pragma unroll
    for (int g = 0; g < (NCH + 7) / 8; ++g)
      if (j + 8 * g < NCH) *reinterpret_cast<uint32_t*>(orow + 4 * (j + 8 * g)) = w[g];
    if (j == 0) {
      const double sc = degenerate ? 0.0 : div15(w64);   // uniform.py:74-80
      uint32_t* a4 = reinterpret_cast<uint32_t*>(orow + p.half);
      if (p.aux == EQ4_AUX_FP16) {
        a4[0] = aux_bits_f16(sc) | (aux_bits_f16(lo) << 16);
      } else {
        a4[0] = aux_bits_f32(sc);
        a4[1] = aux_bits_f32(lo);
      }
      if (p.lo_out) { p.lo_out[row] = lo; p.hi_out[row] = hi; }
      if (p.info0) p.info0[row] = 0;
      if (bad && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
    }
  }
}

// occupancy measured on 4M x 64 / 2M x 128 N(0,1): 3 blocks of 256 (d = 64: 0.42 -> 0.415 ms),
// 4 at d = 128 (0.42 -> 0.37 ms)
template <int NCH>
__global__ void __launch_bounds__(256, NCH >= 16 ? 4 : 3) k_aciq8(const RRParams p) {
  const int lane = threadIdx.x & 31, j = lane & 7;
  const int64_t nsets = (p.rows + 3) / 4;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // np.mean divides by n: a power-of-two d makes it an exact scaling (same rounding as the divide)
  const double n = (double)p.d, rn = 1.0 / n;
  const bool pow2 = (p.d & (p.d - 1)) == 0;
  // the next row set's elements are in flight while the current one is computed
  float xn[NCH];
  {
    const int64_t row = wid * 4 + (lane >> 3);
    const float* xr = p.x + (row < p.rows ? row : 0) * p.ld + j;
#pragma unroll
    for (int k = 0; k < NCH; ++k) xn[k] = __ldcs(xr + 8 * k);
  }
  for (int64_t set = wid; set < nsets; set += nw) {
    const int64_t row = set * 4 + (lane >> 3);
    float x[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) x[k] = xn[k];
    if (set + nw < nsets) {
      const int64_t rown = row + 4 * nw;
      const float* xr = p.x + (rown < p.rows ? rown : 0) * p.ld + j;
#pragma unroll
      for (int k = 0; k < NCH; ++k) xn[k] = __ldcs(xr + 8 * k);
    }
    aciq8_row<NCH>(p, x, row, row < p.rows, j, n, rn, pow2);
  }
}

// ACIQ at d = 64, four lanes per row (eight rows per warp): lane q owns numpy's chains 2q and
// 2q+1 (elements 2q + 8k and 2q + 1 + 8k: one 8-byte load per k, the row's four lanes cover
// 32 contiguous bytes), so the leaf tree's first level (r_2q + r_2q+1) is lane-local and the
// other two are xor-shuffles over the four lanes; the per-row work (trees, range, codec
// constants) is shared by 4 lanes instead of 8.  Every lane's element pairs are whole packed
// bytes (byte q + 4k), transposed 4 x 4 across the row's lanes for 32-bit stores.
template <int NPL>   // elements per lane (16 at d = 64)
__device__ __forceinline__ void aciq4_row(const RRParams& p, const float (&x)[NPL], int64_t row, bool rvalid,
                                          int q, double n, double rn) {
  constexpr unsigned FULLM = 0xffffffffu;
  constexpr int NK = NPL / 2;   // elements per chain
  // np.mean (clipping.py:135): chains 2q (even slots) and 2q+1 (odd slots), the tree, 0.0 +
  double ra = (double)x[0], rb = (double)x[1];
#pragma unroll
  for (int k = 1; k < NK; ++k) {
    ra = __dadd_rn(ra, (double)x[2 * k]);
    rb = __dadd_rn(rb, (double)x[2 * k + 1]);
  }
  double r = __dadd_rn(ra, rb);
  r = __dadd_rn(r, __shfl_xor_sync(FULLM, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(FULLM, r, 2));
  const double sum = __dadd_rn(0.0, r);
  const bool bad = !isfinite(sum);
  const double mean = __dmul_rn(sum, rn);   // d = 64: exact scaling
  double aa = fabs(__dsub_rn((double)x[0], mean)), ab = fabs(__dsub_rn((double)x[1], mean));
#pragma unroll
  for (int k = 1; k < NK; ++k) {
    aa = __dadd_rn(aa, fabs(__dsub_rn((double)x[2 * k], mean)));
    ab = __dadd_rn(ab, fabs(__dsub_rn((double)x[2 * k + 1], mean)));
  }
  double a = __dadd_rn(aa, ab);
  a = __dadd_rn(a, __shfl_xor_sync(FULLM, a, 1));
  a = __dadd_rn(a, __shfl_xor_sync(FULLM, a, 2));
  const double alpha = __dmul_rn(p.aciq_const, __dmul_rn(__dadd_rn(0.0, a), rn));
  double lo = __dsub_rn(mean, alpha), hi = __dadd_rn(mean, alpha);
  (void)n;
  const bool flat = rvalid && !bad && alpha == 0.0;
  if (__any_sync(FULLM, flat)) {   // rare: clipping.py:137-138 -> clip_range_asym (numpy's zero choice)
    float mn = x[0], mx = x[0];
#pragma unroll
    for (int k = 1; k < NPL; ++k) { mn = fminf(mn, x[k]); mx = fmaxf(mx, x[k]); }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      mn = fminf(mn, __shfl_xor_sync(FULLM, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(FULLM, mx, o));
    }
    unsigned kz = 0u;
    if (mn == 0.f || mx == 0.f) {
#pragma unroll
      for (int k = 0; k < NPL; ++k) kz = max(kz, np_zero_key_t(x[k], 2 * q + (k & 1) + 8 * (k >> 1), p.d));
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) kz = max(kz, __shfl_xor_sync(FULLM, kz, o));
    if (flat) {
      const double z = (kz & 1u) ? -0.0 : 0.0;
      lo = mn == 0.f ? z : (double)mn;
      hi = mx == 0.f ? z : (double)mx;
    }
  }
  if (bad) { lo = 0.0; hi = 0.0; }
  const bool degenerate = bad || hi == lo;
  const double w64 = __dsub_rn(hi, lo);
  const float lo_hi = __double2float_rn(lo), lo_lo = __double2float_rn(__dsub_rn(lo, (double)lo_hi));
  const float wf = __double2float_rn(w64);
  const float inv1 = degenerate ? 0.f : __fdividef(1.f, wf);
  const bool slow = !degenerate && !(wf > 1e-30f && wf < 1e30f && fabsf(lo_hi) < 1e30f &&
                                     fabsf(__double2float_rn(hi)) < 1e30f);
  // codes: element pairs (2q + 8k, 2q + 1 + 8k) are packed byte q + 4k; bytes k = 0..3 / 4..7
  uint32_t wb[NK / 4];
#pragma unroll
  for (int g = 0; g < NK / 4; ++g) wb[g] = 0u;
  float gmax = 0.f;
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    unsigned cc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float sv = __saturatef(__fmul_rn(__fadd_rn(__fadd_rn(x[2 * k + h], -lo_hi), -lo_lo), inv1));
      const float m = __fadd_rd(__fmaf_rn(sv, 15.f, 0.5f), 8388608.f);
      gmax = fmaxf(gmax, fabsf(__fmaf_rn(sv, 15.f, -__fadd_rn(m, -8388608.f))));
      cc[h] = __float_as_uint(m) & 0xFu;
    }
    wb[k >> 2] |= (cc[0] | (cc[1] << 4)) << (8 * (k & 3));
  }
  const bool exact = rvalid && (degenerate || slow || gmax > 0.5f - NEAR);
  if (__any_sync(FULLM, exact) && exact) {
    const CodeParams cp = make_code_params(degenerate ? 0.0 : lo, degenerate ? 0.0 : hi);
#pragma unroll
    for (int g = 0; g < NK / 4; ++g) wb[g] = 0u;
#pragma unroll
    for (int k = 0; k < NK; ++k)
      wb[k >> 2] |= (code_exact(x[2 * k], cp) | (code_exact(x[2 * k + 1], cp) << 4)) << (8 * (k & 3));
  }
  // 4 x 4 byte transpose across the row's lanes: lane t ends with bytes 4t..4t+3 of each group
#pragma unroll
  for (int g = 0; g < NK / 4; ++g) {
#pragma unroll
    for (int b = 2; b >= 1; b >>= 1) {
      const unsigned msk = b == 2 ? 0x0000FFFFu : 0x00FF00FFu;
      const int sh = 8 * b;
      const unsigned pw = __shfl_xor_sync(FULLM, wb[g], b);
      wb[g] = (q & b) ? (((pw & ~msk) >> sh) | (wb[g] & ~msk)) : ((wb[g] & msk) | ((pw & msk) << sh));
    }
  }
  if (rvalid) {
    uint8_t* orow = p.packed + (size_t)row * p.stride;
#pragma unroll
    for (int g = 0; g < NK / 4; ++g) *reinterpret_cast<uint32_t*>(orow + 16 * g + 4 * q) = wb[g];
    if (q == 0) {
      const double sc = degenerate ? 0.0 : div15(w64);   // uniform.py:74-80
      uint32_t* a4 = reinterpret_cast<uint32_t*>(orow + p.half);
      if (p.aux == EQ4_AUX_FP16) {
        a4[0] = aux_bits_f16(sc) | (aux_bits_f16(lo) << 16);
      } else {
        a4[0] = aux_bits_f32(sc);
        a4[1] = aux_bits_f32(lo);
      }
      if (p.lo_out) { p.lo_out[row] = lo; p.hi_out[row] = hi; }
      if (p.info0) p.info0[row] = 0;
      if (bad && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
    }
  }
}

#ifndef ACIQ4_MINB
#define ACIQ4_MINB 2   // 124 registers: the next row set's 16 floats stay in registers (3: spills, 0.38 ms)
#endif
__global__ void __launch_bounds__(256, ACIQ4_MINB) k_aciq4(const RRParams p) {
  constexpr int NPL = 16;   // d = 64: 2 chains x 8 elements per lane
  const int lane = threadIdx.x & 31, q = lane & 3;
  const int64_t nsets = (p.rows + 7) / 8;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double n = (double)p.d, rn = 1.0 / n;
  float xn[NPL];
  {
    const int64_t row = wid * 8 + (lane >> 2);
    const float2* xr = reinterpret_cast<const float2*>(p.x + (row < p.rows ? row : 0) * p.ld) + q;
#pragma unroll
    for (int k = 0; k < NPL / 2; ++k) {
      const float2 t = __ldcs(xr + 4 * k);
      xn[2 * k] = t.x;
      xn[2 * k + 1] = t.y;
    }
  }
  for (int64_t set = wid; set < nsets; set += nw) {
    const int64_t row = set * 8 + (lane >> 2);
    float x[NPL];
#pragma unroll
    for (int k = 0; k < NPL; ++k) x[k] = xn[k];
    if (set + nw < nsets) {
      const int64_t rown = row + 8 * nw;
      const float2* xr = reinterpret_cast<const float2*>(p.x + (rown < p.rows ? rown : 0) * p.ld) + q;
#pragma unroll
      for (int k = 0; k < NPL / 2; ++k) {
        const float2 t = __ldcs(xr + 4 * k);
        xn[2 * k] = t.x;
        xn[2 * k + 1] = t.y;
      }
    }
    aciq4_row<NPL>(p, x, row, row < p.rows, q, n, rn);
  }
}

// The scalar entry points on float64 rows (clip_range_aciq / clip_range_gss of any array,
// clipping.py:46 promotes it to float64): ranges (and GSS evaluation counts) only, lane
// per row straight from global memory.
template <int METHOD>
__global__ void k_rowrange_f64(const double* x, int64_t rows, int d, int64_t ld, double invphi,
                               double param, double* lo_out, double* hi_out, int32_t* info0,
                               int32_t* status) {
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < rows;
       row += (int64_t)gridDim.x * blockDim.x) {
    RowViewT<double> xr{x + row * ld, 1};
    double mn = INFINITY, mx = -INFINITY;
    bool bad = false;
    for (int k = 0; k < d; k++) {
      const double v = xr[k];
      mn = fmin(mn, v);
      mx = fmax(mx, v);
      bad |= !isfinite(v);
    }
    double lo = 0.0, hi = 0.0;
    int evals = 0;
    if (bad) {
      if (status) atomicOr(status, EQ4_STATUS_NONFINITE);
    } else if constexpr (METHOD == EQ4_METHOD_ACIQ) {
      lane_aciq(xr, d, mn, mx, param, lo, hi);
    } else {
      evals = lane_gss(xr, d, mn, mx, invphi, param, lo, hi);
    }
    lo_out[row] = lo;
    hi_out[row] = hi;
    if (info0) info0[row] = evals;
  }
}

}  // namespace eq4

using namespace eq4;

int eq4_rowrange_f64_launch(const double* x, int64_t rows, int64_t dim, int64_t ld, int method,
                            double param, double* xmin, double* xmax, int32_t* info0, int32_t* status,
                            cudaStream_t s, std::string& err) {
  const double invphi = (std::sqrt(5.0) - 1.0) / 2.0;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 127) / 128, 148 * 8));
  if (method == EQ4_METHOD_ACIQ)
    k_rowrange_f64<EQ4_METHOD_ACIQ><<<grid, 128, 0, s>>>(x, rows, (int)dim, ld, invphi, param, xmin, xmax,
                                                         info0, status);
  else
    k_rowrange_f64<EQ4_METHOD_GSS><<<grid, 128, 0, s>>>(x, rows, (int)dim, ld, invphi, param, xmin, xmax,
                                                        info0, status);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { err = std::string("k_rowrange_f64: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  return EQ4_OK;
}

int eq4_rowrange_launch(const float* x, int64_t rows, int64_t dim, int64_t ld, int method, double param,
                        int aux, uint8_t* packed, double* xmin, double* xmax, int32_t* info0,
                        int32_t* status, cudaStream_t s, std::string& err) {
  RRParams p;
  memset(&p, 0, sizeof(p));
  p.aciq_const = method == EQ4_METHOD_ACIQ ? param : 5.03;
  p.gss_tol = method == EQ4_METHOD_GSS ? param : 1e-4;
  p.x = x; p.rows = rows; p.ld = ld; p.d = (int)dim; p.aux = aux; p.method = method;
  p.half = (int)((dim + 1) / 2);
  p.stride = p.half + 2 * (aux == EQ4_AUX_FP16 ? 2 : 4);
  p.packed = packed; p.lo_out = xmin; p.hi_out = xmax; p.info0 = info0; p.status = status;
  p.invphi = (std::sqrt(5.0) - 1.0) / 2.0;
  if (method == EQ4_METHOD_ACIQ && (dim == 64 || dim == 128) && ((uintptr_t)packed & 3) == 0 &&
      !getenv("EQ4_DEV_ACIQ_LANE")) {   // (env: development A/B only)
    const int nch = (int)(dim / 8);
    // d = 64 with 8-byte aligned rows: four lanes per row (k_aciq4), else eight (k_aciq8)
    const bool four = dim == 64 && (ld % 2) == 0 && (((uintptr_t)x & 7) == 0) && !getenv("EQ4_DEV_ACIQ8");
    auto kern = four ? k_aciq4 : nch == 1 ? k_aciq8<1> : nch == 2 ? k_aciq8<2> : nch == 4 ? k_aciq8<4>
              : nch == 8 ? k_aciq8<8> : nch == 16 ? k_aciq8<16> : nullptr;
    if (kern) {
      int dev = 0, sms = 0, per_sm = 0;
      cudaError_t e = cudaGetDevice(&dev);
      if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
      if (e != cudaSuccess) { err = std::string("k_aciq8 setup: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
      const int64_t nsets = (rows + (four ? 7 : 3)) / (four ? 8 : 4);
      int64_t grid = (nsets + 7) / 8;
      const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
      if (grid > cap) grid = cap;
      kern<<<(unsigned)std::max<int64_t>(1, grid), 256, 0, s>>>(p);
      e = cudaGetLastError();
      if (e != cudaSuccess) { err = std::string("k_aciq8: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
      return EQ4_OK;
    }
  }
  p.staged = dim <= RR_MAX_STAGED;
  p.vec4 = (dim % 4 == 0) && (ld % 4 == 0) && (((uintptr_t)x & 15) == 0);
  const size_t xs_bytes = p.staged ? (size_t)dim * RR_COL * 4 : 0;
  p.direct = (size_t)32 * p.stride > 24 * 1024;   // wide rows: no per-warp staging tile
  p.warp_bytes = ((xs_bytes + 15) & ~(size_t)15) +
                 (p.direct ? 0 : (((size_t)32 * p.stride + 32 + 15) & ~(size_t)15));
  p.warp_bytes = (p.warp_bytes + 15) & ~(size_t)15;
  const size_t smem = p.warp_bytes * RR_WARPS;
  auto kern = method == EQ4_METHOD_ACIQ ? k_rowrange<EQ4_METHOD_ACIQ> : k_rowrange<EQ4_METHOD_GSS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 0, per_sm = 0;
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RR_THREADS, smem);
  if (e != cudaSuccess) { err = std::string("k_rowrange setup: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  const int64_t nblk = (rows + 31) / 32;
  int64_t grid = (nblk + RR_WARPS - 1) / RR_WARPS;
  const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, RR_THREADS, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) { err = std::string("k_rowrange: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  return EQ4_OK;
}
