// eq4_device.cuh -- device-side building blocks for the row-wise 4-bit
// clip-search + pack kernels (sm_100a).
//
// Two arithmetic tiers live here:
//  * "np_*" helpers restate the reference's float64 numpy expressions op by
//    op with explicitly rounded intrinsics (__dadd_rn/__dmul_rn/__ddiv_rn are
//    never contracted into FMAs), so their results are bit-identical to the
//    reference: quant_mse (table.py:81-103), quantize_uniform
//    (uniform.py:60-80) and numpy's pairwise np.sum order.
//  * the search kernels evaluate the same objective approximately in fp32
//    (see eq4.cu, "GREEDY fast path") and only fall back to the np_* tier when
//    two competing values lie inside a proven error band.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

namespace eq4 {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------
// Exact (numpy float64) tier
// ---------------------------------------------------------------------------

// Correctly rounded w / 15 in float64 without a divide: q = RN(w * RN(1/15)),
// r = w - 15 q (exact by FMA), RN(q + r * RN(1/15)) = RN(w / 15) (Markstein's
// correction step; checked against __ddiv_rn by eq4_selftest).
__device__ __forceinline__ double div15(double w) {
  const double y = 0.06666666666666666666;          // RN(1/15)
  const double q = __dmul_rn(w, y);
  const double r = __fma_rn(-q, 15.0, w);
  return __fma_rn(r, y, q);
}

// ---------------------------------------------------------------------------
// numpy's choice among equal extrema (the sign of a zero min / max)
// ---------------------------------------------------------------------------
// np.min / np.max of a row (clipping.py:61,163; histclip.py:57) return one of
// several equal extrema; for a zero extremum that choice is the sign of the
// bias the row is packed with.  numpy's AVX-512 reduction (restated op by op in
// oracle/eq4_oracle.c np_reduce_ext) makes the choice a fixed priority over
// positions p of the row (d elements), the same for min and max:
//   p in 1 .. 8*nv (nv = (d-1)/8 full vectors) by vector lane k = (p-1) % 8 in
//   the order 1 > 5 > 3 > 7 > 0 > 4 > 2 > 6 (the _mm512_reduce tree), the later
//   p within a lane; above all the scalar tail p > 8*nv, the later the higher.
//   x[0] seeds every lane's accumulator, so a zero x[0] stands in lane 1 (the
//   top lane) below lane 1's own elements; with no full vector it is lowest.
//   np_zero_key is 0 for a non-zero element, else a key whose maximum over the
//   row's zeros carries the winner's sign in bit 0.
__device__ __forceinline__ unsigned np_zero_key(float v, int p, int d) {
  if (v != 0.f) return 0u;
  const int nv8 = (d - 1) >> 3;
  unsigned prio;
  if (p == 0) {
    prio = nv8 >= 1 ? (8u << 24) + 1u : 1u;
  } else if (p > 8 * nv8) {
    prio = (1u << 29) + (unsigned)p;
  } else {
    const int k = (p - 1) & 7;
    const unsigned rank = (0x51736284u >> (4 * k)) & 0xFu;   // lane 1 -> 8, 5 -> 7, ..., 6 -> 1
    prio = (rank << 24) + (unsigned)((p - 1) >> 3) + 2u;
  }
  return (prio << 1) | (__float_as_uint(v) >> 31);
}

// Apply the winner of a group's zero keys (already max-reduced) to a zero
// min / max: the row's extremum takes the winning zero's sign.
__device__ __forceinline__ void np_zero_apply(unsigned kz, float& mn, float& mx) {
  const float z = (kz & 1u) ? -0.f : 0.f;
  if (mn == 0.f) mn = z;
  if (mx == 0.f) mx = z;
}

// np.clip(x, lo, hi) == minimum(maximum(x, lo), hi) for finite operands.
__device__ __forceinline__ double np_clip(double x, double lo, double hi) {
  double t = x > lo ? x : lo;
  return t < hi ? t : hi;
}

// uniform.py:78-79 / table.py:100-101: one code, float64, half-up rounding.
__device__ __forceinline__ double np_code(double x, double lo, double hi, double scale) {
  double c = np_clip(x, lo, hi);
  double q = __ddiv_rn(__dsub_rn(c, lo), scale);
  return np_clip(floor(__dadd_rn(q, 0.5)), 0.0, 15.0);
}

// table.py:96-103: squared reconstruction error of one element.
// scale must be (hi - lo) / 15 (float64) unless hi == lo.
__device__ __forceinline__ double np_err2(double x, double lo, double hi, double scale) {
  if (hi == lo) {
    double e = __dsub_rn(x, lo);
    return __dmul_rn(e, e);
  }
  double code = np_code(x, lo, hi, scale);
  double recon = __dadd_rn(__dmul_rn(scale, code), lo);
  double e = __dsub_rn(x, recon);
  return __dmul_rn(e, e);
}

// np_err2 without the divide: q = (c - lo) * RN(1/scale) is within a few ulp of
// numpy's correctly rounded quotient, so floor(q + 0.5) can only differ when
// q + 0.5 lies within ~1e-14 of an integer; inside 1e-12 of one the IEEE
// divide decides (bit-identical to np_err2).
struct NpCodec {
  double lo, hi, scale, inv;
};
__device__ __forceinline__ NpCodec np_codec(double lo, double hi) {
  NpCodec c;
  c.lo = lo;
  c.hi = hi;
  c.scale = (hi == lo) ? 0.0 : div15(__dsub_rn(hi, lo));   // table.py:99
  c.inv = (hi == lo) ? 0.0 : __drcp_rn(c.scale);
  return c;
}
__device__ __forceinline__ double np_err2_fast(double x, const NpCodec& c) {
  if (c.hi == c.lo) {
    const double e = __dsub_rn(x, c.lo);
    return __dmul_rn(e, e);
  }
  const double dl = __dsub_rn(np_clip(x, c.lo, c.hi), c.lo);
  const double t = __dadd_rn(__dmul_rn(dl, c.inv), 0.5);
  const double fl = floor(t);
  const double fr = __dsub_rn(t, fl);
  double q = fl;
  if (!(fr > 1e-12 && fr < 1.0 - 1e-12)) q = floor(__dadd_rn(__ddiv_rn(dl, c.scale), 0.5));
  const double code = np_clip(q, 0.0, 15.0);
  const double e = __dsub_rn(x, __dadd_rn(__dmul_rn(c.scale, code), c.lo));
  return __dmul_rn(e, e);
}

// numpy pairwise-sum leaves: np.add.reduce splits n > 128 into
// n2 = n/2 - (n/2 % 8) and n - n2 recursively; leaves have <= 128 elements.
// Enumerate the leaves of [0, n) in order.  Returns the leaf count.
__device__ __forceinline__ int np_leaves(int n, int* starts, int* lens, int max_leaves) {
  int st_a[32], st_n[32];
  int sp = 0, cnt = 0;
  st_a[sp] = 0; st_n[sp] = n; sp++;
  while (sp > 0) {
    sp--;
    int a = st_a[sp], m = st_n[sp];
    if (m <= 128) {
      if (cnt < max_leaves) { starts[cnt] = a; lens[cnt] = m; }
      cnt++;
    } else {
      int n2 = m / 2;
      n2 -= n2 % 8;
      st_a[sp] = a + n2; st_n[sp] = m - n2; sp++;   // right pushed first
      st_a[sp] = a; st_n[sp] = n2; sp++;            // left popped first
    }
  }
  return cnt;
}

// Combine leaf sums in the recursion's association order.
static __device__ __noinline__ double np_combine(int n, const double* leaf_sum, int* li) {
  if (n <= 128) return leaf_sum[(*li)++];
  int n2 = n / 2;
  n2 -= n2 % 8;
  double left = np_combine(n2, leaf_sum, li);
  double right = np_combine(n - n2, leaf_sum, li);
  return __dadd_rn(left, right);
}

// Warp-cooperative, bit-exact quant_mse (table.py:81-103) of one row whose
// fp32 values sit in shared memory `xs[0..d)`.  All 32 lanes must call it
// with identical arguments; every lane returns the same value.
// Scratch (per warp, shared): e2[e2cap] doubles with e2cap >= min(d, 512),
// leaf_sum/leaf_start/leaf_len[max_leaves].
// Element errors are computed by all 32 lanes into e2, then numpy's
// pairwise order is replayed: per leaf, 8 lanes run the 8 sequential
// accumulator chains, a 3-level butterfly forms ((r0+r1)+(r2+r3))+(...),
// lane 0 adds the leaf's remainder, and lane 0 combines leaf sums in the
// recursion's association order.
// The fp32 code estimates (code_of, fast_code) of x under (lo, hi): the argument
// t' = (x - lo) * 15/(hi-lo) + 0.5 has absolute error < 7e-6 for interior x
// (|t'| < 16, a few roundings of relative 2^-24 each on the range-scaled
// quantities); when frac(t') is within NEAR of an integer the float64 codec
// decides.  x <= lo gives code 0 and x >= hi code 15 exactly in the
// reference (clip then floor(0 + .5) / floor(15 +- 1ulp + .5)).
constexpr float NEAR = 1e-5f;

// Branch-free fp32 code of x under the float64 range [lo, hi] (saturating scale, round-down
// add of 2^23): numpy's code (uniform.py:77-79) unless x lies within NEAR = 1e-5 of a
// rounding boundary, which sets `near` (callers then redo the pass with the float64 codec).
struct FastCodec {
  float lo_hi, lo_lo, inv1;
  bool slow;   // range too extreme for the estimate: always take the float64 codec
};
__device__ __forceinline__ FastCodec fast_codec(double lo, double hi) {
  FastCodec f;
  f.lo_hi = __double2float_rn(lo);
  f.lo_lo = __double2float_rn(__dsub_rn(lo, (double)f.lo_hi));
  const double w = __dsub_rn(hi, lo);
  f.slow = hi != lo && !(w > 1e-30 && w < 1e30 && fabs(lo) < 1e30 && fabs(hi) < 1e30);
  f.inv1 = (hi == lo) ? 0.f : __fdividef(1.f, __double2float_rn(w));
  return f;
}
__device__ __forceinline__ double fast_code(float xf, const FastCodec& f, bool& near) {
  const float sv = __saturatef(__fmul_rn(__fadd_rn(__fadd_rn(xf, -f.lo_hi), -f.lo_lo), f.inv1));
  const float mm = __fadd_rd(__fmaf_rn(sv, 15.f, 0.5f), 8388608.f);
  near |= fabsf(__fmaf_rn(sv, 15.f, -__fadd_rn(mm, -8388608.f))) > 0.5f - NEAR;
  return (double)(__float_as_uint(mm) & 0xFu);
}
// (x - (scale * code + lo))^2 with the reference's float64 operations
__device__ __forceinline__ double np_err2_code(double x, double code, const NpCodec& c) {
  const double e = __dsub_rn(x, __dadd_rn(__dmul_rn(c.scale, code), c.lo));
  return __dmul_rn(e, e);
}

static __device__ __noinline__ double warp_np_loss(const float* xs, int d, double lo, double hi,
                                            double* e2, double* leaf_sum, int* leaf_start,
                                            int* leaf_len, int max_leaves) {
  const int lane = threadIdx.x & 31;
  const NpCodec cd = np_codec(lo, hi);   // table.py:99
  if (d < 8) {  // numpy: res = 0.; res += a[i] sequentially
    double res = 0.0;
    if (lane == 0)
      for (int i = 0; i < d; i++) res = __dadd_rn(res, np_err2_fast((double)xs[i], cd));
    res = __shfl_sync(FULL, res, 0);
    return __dadd_rn(0.0, res);
  }
  const FastCodec fc = fast_codec(lo, hi);
  const int g = lane >> 3, m = lane & 7;
  if (d >= 256 && d <= 16384 && (d & (d - 1)) == 0) {
    // power-of-two rows: numpy's halving is exact down to 128-element leaves, so the leaves are
    // [128 l, 128 l + 128) and they combine as a balanced binary tree -- a shuffle tree over the
    // leaf sums (a + b == b + a bitwise), no leaf table and no recursion
    const int nl = d >> 7;
    for (int base = 0; base < nl; base += 4) {
      const int r0 = base << 7, n4 = (min(base + 4, nl) - base) << 7;
      bool near = fc.slow;
      for (int k = lane; k < n4; k += 32) {
        const float xf = xs[r0 + k];
        e2[k] = np_err2_code((double)xf, fast_code(xf, fc, near), cd);
      }
      if (__any_sync(FULL, near))   // an element near a rounding boundary: the float64 codec
        for (int k = lane; k < n4; k += 32) e2[k] = np_err2_fast((double)xs[r0 + k], cd);
      __syncwarp();
      const int li = base + g;
      double r = 0.0;
      if (li < nl) {
        r = e2[(g << 7) + m];
        for (int i = 8 + m; i < 128; i += 8) r = __dadd_rn(r, e2[(g << 7) + i]);
      }
      r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 1));
      r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 2));
      r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 4));
      if (li < nl && m == 0) leaf_sum[li] = r;
      __syncwarp();
    }
    // balanced tree over the nl = 2..128 leaf sums: up to 4 per lane, then the lane butterfly
    const int per = nl > 32 ? nl / 32 : 1;
    double v = 0.0;
    if (lane * per < nl) {
      v = leaf_sum[lane * per];
      if (per >= 2) v = __dadd_rn(v, leaf_sum[lane * per + 1]);
      if (per == 4) v = __dadd_rn(v, __dadd_rn(leaf_sum[lane * per + 2], leaf_sum[lane * per + 3]));
    }
    const int lanes = nl / per;
    for (int o = 1; o < lanes; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
    __syncwarp();
    return __dadd_rn(0.0, __shfl_sync(FULL, v, 0));
  }
  int nl = 0;
  if (lane == 0) nl = np_leaves(d, leaf_start, leaf_len, max_leaves);
  nl = __shfl_sync(FULL, nl, 0);
  __syncwarp();
  for (int base = 0; base < nl; base += 4) {
    const int last = min(base + 4, nl) - 1;
    const int r0 = leaf_start[base], r1 = leaf_start[last] + leaf_len[last];
    {
      bool near = fc.slow;
      for (int k = lane; k < r1 - r0; k += 32) {
        const float xf = xs[r0 + k];
        e2[k] = np_err2_code((double)xf, fast_code(xf, fc, near), cd);
      }
      if (__any_sync(FULL, near))   // an element near a rounding boundary: the float64 codec
        for (int k = lane; k < r1 - r0; k += 32) e2[k] = np_err2_fast((double)xs[r0 + k], cd);
    }
    __syncwarp();
    const int li = base + g;
    const bool ok = li < nl;
    const int a = ok ? leaf_start[li] - r0 : 0;
    const int len = ok ? leaf_len[li] : 8;
    const int nfull = len - (len % 8);
    // chain m: r[m] = a[m] + a[m+8] + ... sequentially (loops_utils.h.src)
    double r = ok ? e2[a + m] : 0.0;
    for (int i = 8 + m; i < nfull; i += 8) r = __dadd_rn(r, e2[a + i]);
    // ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)); a+b == b+a bitwise
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 4));
    if (ok && m == 0) {
      for (int i = nfull; i < len; i++) r = __dadd_rn(r, e2[a + i]);
      leaf_sum[li] = r;
    }
    __syncwarp();
  }
  double total = 0.0;
  if (lane == 0) {
    int li = 0;
    total = np_combine(d, leaf_sum, &li);
  }
  total = __shfl_sync(FULL, total, 0);
  return __dadd_rn(0.0, total);
}

// Bit-exact quant_mse (table.py:81-103) of up to three clip ranges of one row
// with 8 <= d <= 128, i.e. a single numpy pairwise leaf: the 8 accumulator
// chains r[m] = a[m] + a[m+8] + ... of range k run on lanes 8k..8k+7 (each
// lane computes its own chain's element errors, in order), then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by butterfly and the d % 8 remainder
// on the chain-0 lane -- the same association as warp_np_loss, with the three
// ranges in flight at once and no shared scratch.  Warp-collective; every lane
// returns all values (ranges k >= nr are not evaluated and return 0).
__device__ __forceinline__ void warp_np_loss3_leaf(const float* xs, int d, int nr, double lo0,
                                                   double hi0, double lo1, double hi1, double lo2,
                                                   double hi2, double& v0, double& v1,
                                                   double& v2) {
  const int lane = threadIdx.x & 31;
  const int k = lane >> 3, m = lane & 7;
  const double lo = k == 0 ? lo0 : (k == 1 ? lo1 : lo2);
  const double hi = k == 0 ? hi0 : (k == 1 ? hi1 : hi2);
  const bool act = k < nr;
  const NpCodec cd = np_codec(lo, hi);
  const int nfull = d - (d % 8);
  const int nch = nfull >> 3;   // chain length <= 16
  double r = 0.0;
  // codes from the branch-free fp32 estimate (saturating scale, round-down add); they are
  // numpy's unless an element lies within NEAR of a rounding boundary, in which case the
  // whole pass is redone with the float64 codec.  The errors and sums are the reference's
  // float64 operations either way.
  {
    const FastCodec fc = fast_codec(lo, hi);
    bool flag = act && fc.slow;
    if (act) {
      for (int u = 0; u < nch; u++) {
        const float xf = xs[m + 8 * u];
        const double e2v = np_err2_code((double)xf, fast_code(xf, fc, flag), cd);
        r = u == 0 ? e2v : __dadd_rn(r, e2v);
      }
    }
    if (__any_sync(FULL, flag)) {
      r = 0.0;
      if (act) {
        r = np_err2_fast((double)xs[m], cd);
        for (int u = 1; u < nch; u++) r = __dadd_rn(r, np_err2_fast((double)xs[m + 8 * u], cd));
      }
    }
  }
  r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(FULL, r, 4));
  if (act && m == 0)
    for (int i = nfull; i < d; i++) r = __dadd_rn(r, np_err2_fast((double)xs[i], cd));
  v0 = __dadd_rn(0.0, __shfl_sync(FULL, r, 0));
  v1 = __dadd_rn(0.0, __shfl_sync(FULL, r, 8));
  v2 = __dadd_rn(0.0, __shfl_sync(FULL, r, 16));
}

// Out-of-line copy (keeps the rare path from shaping a big kernel's registers).
static __device__ __noinline__ void warp_np_loss3_leaf_ool(const float* xs, int d, int nr,
                                                           double lo0, double hi0, double lo1,
                                                           double hi1, double lo2, double hi2,
                                                           double& v0, double& v1, double& v2) {
  warp_np_loss3_leaf(xs, d, nr, lo0, hi0, lo1, hi1, lo2, hi2, v0, v1, v2);
}

// ---------------------------------------------------------------------------
// Codes for the final quantize pass (uniform.py:77-79), fast path + exact fix-up
// ---------------------------------------------------------------------------

struct CodeParams {
  double lo, hi, scale;   // float64 range and (hi - lo) / 15
  float lo_rd, hi_ru;     // largest float <= lo, smallest float >= hi
  float lo_hi, lo_lo;     // lo split as float hi + float lo
  float inv;              // ~15 / (hi - lo)
  bool degenerate;        // hi == lo  -> all codes 0 (uniform.py:74-76)
  bool slow;              // range too extreme for the fp32 estimate
};

__device__ __forceinline__ CodeParams make_code_params(double lo, double hi) {
  CodeParams p;
  p.lo = lo;
  p.hi = hi;
  p.degenerate = (hi == lo);
  p.scale = p.degenerate ? 0.0 : div15(__dsub_rn(hi, lo));
  p.lo_rd = __double2float_rd(lo);
  p.hi_ru = __double2float_ru(hi);
  p.lo_hi = __double2float_rn(lo);
  p.lo_lo = __double2float_rn(__dsub_rn(lo, (double)p.lo_hi));
  double w = __dsub_rn(hi, lo);
  p.inv = p.degenerate ? 0.f : __fdividef(15.f, __double2float_rn(w));
  // fp32 estimate needs a normal, finite reciprocal and range
  p.slow = !p.degenerate && !(w > 1e-30 && w < 1e30 && fabs(lo) < 1e30 && fabs(hi) < 1e30);
  return p;
}


// Code of x under (lo, hi), numpy semantics (NEAR above).
__device__ __forceinline__ unsigned code_of(float x, const CodeParams& p, bool& need_exact) {
  // branch-free: every element runs the same instruction stream
  const float dlt = __fadd_rn(__fadd_rn(x, -p.lo_hi), -p.lo_lo);
  const float t = __fmul_rn(dlt, p.inv);
  const float u = __fadd_rn(t, 0.5f);
  const float m = __fadd_rd(u, 8388608.f);          // 2^23 + floor(u)
  const float cf = __fadd_rn(m, -8388608.f);
  const float g = __fadd_rn(t, -cf);                // in [-1/2, 1/2) unless near a boundary
  const bool below = x <= p.lo_rd, above = x >= p.hi_ru;
  const bool interior = !below && !above && !p.degenerate;
  need_exact = interior && (p.slow || fabsf(g) > 0.5f - NEAR || cf < 0.f || cf > 15.f);
  unsigned c = (unsigned)__float_as_uint(m) & 0xFu;
  c = above ? 15u : c;
  return (below || p.degenerate) ? 0u : c;
}

__device__ __forceinline__ unsigned code_exact(float x, const CodeParams& p) {
  if (p.degenerate) return 0u;
  return (unsigned)np_code((double)x, p.lo, p.hi, p.scale);
}

// Stored scale/bias bit patterns (uniform.py:80 dtype(scale), dtype(xmin)):
// np.float16(double) and np.float32(double) both round once, to nearest-even.
// The f16 bits leave the conversion through an opaque move: nvcc 12.9 folds
// "cvt.rn.f16.f64 -> bits -> (uint8_t)(bits & 0xff)" into a numeric
// F2I.U8.F16 conversion, which is wrong for a bit-pattern extraction.
__device__ __forceinline__ uint32_t aux_bits_f16(double v) {
  unsigned short h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(v));
  uint32_t r;
  asm volatile("cvt.u32.u16 %0, %1;" : "=r"(r) : "h"(h));
  return r;
}
__device__ __forceinline__ uint32_t aux_bits_f32(double v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "f"(__double2float_rn(v)));
  return r;
}

// ---- HIST-APPRX exact window norm (histclip.py:110-121), the reference's float64 order ----
// x^3 through a double-double product (the reference's numpy `**3` is SVML /
// libm pow, itself host-dependent in the last bit)
__device__ __forceinline__ double cube_dd(double x) {
  const double h = __dmul_rn(x, x), l = __fma_rn(x, x, -h);
  const double t = __dmul_rn(h, x);
  const double e = __fma_rn(h, x, -t) + __dmul_rn(l, x);
  return __dadd_rn(t, e);
}
// histclip.py:70-82 bin_l2_norm(db, de, 1.0)
__device__ __forceinline__ double l2u(double db, double de) {
  return __ddiv_rn(__dmul_rn(1.0, __dsub_rn(cube_dd(de), cube_dd(db))), 3.0);
}

// histclip.py:85-109 _offset_unit_norms(j - s, w, dst_w) * density for bin j (count c > 0)
__device__ __forceinline__ double apprx_term(int c, int j, double w, int s, double dst_w, double half,
                                             double cw) {
  const double density = __ddiv_rn((double)c, w);
  const double k = __dsub_rn((double)j, (double)s);
  const double begin = __dmul_rn(k, w), end = __dadd_rn(begin, w);
  const double dob = np_clip(floor(__ddiv_rn(__dadd_rn(begin, half), dst_w)), 0.0, 15.0);
  const double doe = np_clip(floor(__ddiv_rn(__dadd_rn(end, half), dst_w)), 0.0, 15.0);
  const double bc = __dmul_rn(dob, dst_w), ec = __dmul_rn(doe, dst_w);
  const double db = __dsub_rn(begin, bc);
  double contrib;
  if (dob == doe) {
    contrib = l2u(db, __dsub_rn(end, bc));
  } else {
    contrib = __dadd_rn(__dadd_rn(l2u(db, half), __dmul_rn(__dsub_rn(__dsub_rn(doe, dob), 1.0), cw)),
                        l2u(-half, __dsub_rn(end, ec)));
  }
  return __dmul_rn(density, contrib);
}

// histclip.py:110-121 window_norm = np.sum over the b bins of density * unit norm, in
// numpy's pairwise order (the leaves of np_leaves, 8 accumulator chains each, the
// fixed ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree, the remainder in order, then the
// leaves combined in the recursion's association, np_combine).  Warp-collective:
// lanes compute the bins' terms into t[0..b) (empty bins give the +0.0 numpy adds,
// which leave every partial sum unchanged), lanes 8l..8l+7 run leaf l's chains.
// Every lane returns the value.
static __device__ __noinline__ double apprx_norm_np_warp(const int* cnt, int b, double w, int s, int n,
                                                  double* t, int lane, double* leaf_sum, int* leaf_st,
                                                  int* leaf_ln, int max_leaves) {
  const double dst_w = __ddiv_rn(__dmul_rn(w, (double)n), 15.0);
  const double half = __dmul_rn(0.5, dst_w);
  const double cw = l2u(-half, half);
  for (int j = lane; j < b; j += 32) {
    const int c = cnt[j];
    t[j] = c ? apprx_term(c, j, w, s, dst_w, half, cw) : 0.0;
  }
  {
    // one leaf (b <= 128) or two (both halves <= 128 elements): lanes 8l..8l+7 run leaf l's
    // chains, the leaves are added once -- no leaf table, no recursion
    int n2 = b;
    if (b > 128) { n2 = b / 2; n2 -= n2 % 8; }
    if (b <= 128 || b - n2 <= 128) {
      __syncwarp();
      const int nleaves = b > 128 ? 2 : 1;
      const int leaf = (lane >> 3) & 1, k = lane & 7;
      const int ls = leaf ? n2 : 0, ln = leaf ? b - n2 : n2;
      const int nfull = ln < 8 ? 0 : ln - (ln % 8);
      double r = 0.0;
      if (lane < 8 * nleaves)
        for (int jj = k; jj < nfull; jj += 8) r = __dadd_rn(r, t[ls + jj]);
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
      double res = ln >= 8 ? r : 0.0;
      for (int jj = nfull; jj < ln; jj++) res = __dadd_rn(res, t[ls + jj]);
      const double leaf1 = __shfl_sync(0xffffffffu, res, 8);
      const double total = nleaves == 2 ? __dadd_rn(res, leaf1) : res;   // lane 0: leaf 0 + leaf 1
      __syncwarp();
      return __shfl_sync(0xffffffffu, __dadd_rn(0.0, total), 0);
    }
  }
  int nl = 0;
  if (lane == 0) nl = np_leaves(b, leaf_st, leaf_ln, max_leaves);
  nl = __shfl_sync(0xffffffffu, nl, 0);
  __syncwarp();
  // four leaves per pass: lanes 8l..8l+7 run leaf l's 8 accumulator chains
  const int g = lane >> 3, m = lane & 7;
  for (int base = 0; base < nl; base += 4) {
    const int li = base + g;
    const bool ok = li < nl;
    const int a = ok ? leaf_st[li] : 0, len = ok ? leaf_ln[li] : 8;
    const int nfull = len - (len % 8);
    double r = (ok && len >= 8) ? t[a + m] : 0.0;
    for (int i = 8 + m; i < nfull; i += 8) r = __dadd_rn(r, t[a + i]);
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (ok && m == 0) {
      if (len < 8) {   // numpy: res = 0.; res += a[i] for n < 8
        r = 0.0;
        for (int i = 0; i < len; i++) r = __dadd_rn(r, t[a + i]);
      } else {
        for (int i = nfull; i < len; i++) r = __dadd_rn(r, t[a + i]);
      }
      leaf_sum[li] = r;
    }
    __syncwarp();
  }
  double total = 0.0;
  if (lane == 0) {
    int li = 0;
    total = np_combine(b, leaf_sum, &li);
  }
  __syncwarp();
  return __shfl_sync(0xffffffffu, __dadd_rn(0.0, total), 0);
}

}  // namespace eq4
