// eq4.cu -- B200 (sm_100a) kernels + C ABI for row-wise 4-bit clip-search + pack.
//
// Reference path (arXiv 1911.02079 artifact `embquant`):
//   methods.py:63-89 quantize_table -> per row methods.py:43-60 row_clip_range
//     -> clipping.py:58-61 clip_range_asym | clipping.py:142-193 clip_range_greedy
//        | histclip.py:136-178 hist_brute_search (eq4_hist.cu)
//   -> uniform.py:142-167 quantize_table_uniform -> packed.py:68-83 pack_table4
// Here one launch does all of it for a whole table: rows are independent, so
// each row is owned by a group of LPR lanes (E elements per lane, row held in
// registers), the packed output of a tile of rows is staged in shared memory
// and leaves as 16-byte stores.
//
// GREEDY fast path (the north-star kernel)
// ----------------------------------------
// The reference evaluates quant_mse (table.py:81-103) in float64 65-67 times
// per row.  Every candidate it visits lies on the grid lo = x0 + i*step,
// hi = x1 - j*step with step = (x1-x0)/b, so in the row coordinate
//     Y = 15 * (x - x0) / step          (Y in [0, 15b])
// candidate (i, j) has base B = 15 i, width W = b - i - j steps and
// reconstruction points B + c*W, c = 0..15 (integers!).  Y is rounded once to
// a float grid of quantum Q = 2^(ceil(log2 15b) - 24) (2^-12 for b=200) so that
//     z = Y - B,   e = z - c*W
// are EXACT fp32 operations; the per element-evaluation cost is 6 fp32
// instructions (FADD, FFMA.SAT, FFMA.RM, FADD, FFMA, FFMA) against the 13
// algorithmic FLOP of table.py:100-103.  The code c = floor(z/W + 1/2) clamped
// to [0,15] comes from one saturating FFMA (s = sat((z/W + 1/2)/alpha)) and
// one round-down FFMA (2^23 + floor(alpha*s)).
// The approximate loss L~ differs from the reference's float64 value by at
// most  tau*L + 2*delta*sqrt(d*L) + d*delta^2 + misround terms  (delta = Q/2;
// fp32 summation), so every comparison whose two sides are
// further apart than that band is decided exactly as the reference decides
// it.  Comparisons inside the band (and every comparison of rows whose
// candidate grid the reference rounds coarsely) are re-decided with the
// bit-exact float64 restatement (eq4_device.cuh warp_np_loss), so the walk --
// and therefore the thresholds, codes and bytes -- match the reference.
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/eq4.h"
#include "eq4_device.cuh"
#include "eq4_internal.h"

namespace eq4 {

constexpr int NTHREADS = 256;
constexpr int NWARPS = NTHREADS / 32;
#ifndef G_THREADS
#define G_THREADS 128
#endif
constexpr int NTHREADS_G = G_THREADS;         // GREEDY blocks (warps are independent)
constexpr int NWARPS_G = NTHREADS_G / 32;
constexpr int MAX_LEAVES = 64;          // numpy pairwise leaves for d <= 4096
constexpr float ALPHA = 15.75f;         // saturation scale for the code FFMA
// |alpha * s - (z/W + 1/2)| <= ETA_CODE for s = RN(z * kw_of(W) + h), |z/W| <= 15.5:
// 15.5 * (2^-24 + 2^-46) (kW rounded once after one Newton step) + 15.75 * 2^-25 (s rounded
// once) + 15.75 * 2^-24 * h (h = 1/(2 alpha) rounded) = 1.43e-6.
constexpr double ETA_CODE = 1.6e-6;
// elements counted as able to take the other code: within ETA_CODE (+ margin) + delta/W
constexpr float NEAR_CNT = 2.2e-6f;
constexpr float MAGIC = 8388608.f;      // 2^23
enum { M_ASYM = 0, M_GREEDY = 1 };
#ifndef GREEDY_MINB
#define GREEDY_MINB 4
#endif
#ifndef G_MINB32
#define G_MINB32 3
#endif
#ifndef G_MINB64
#define G_MINB64 3   // 170 registers: the phase-A loop state stays out of local memory
#endif

// Diagnostic counters of the GREEDY kernel's rare paths (read by eq4_diag_counters):
// [0] rows re-decided with the float64 restatement (one per row and iteration),
// [1] rows whose codes came from the float64 codec (an element near a rounding
// boundary), [2] comparisons resolved by counting near-boundary elements
// (near_escalate), [3] of those, escalated to the exact re-decision (more than
// 2 elements of a side within reach of a boundary).  Only the rare paths touch them.
// [4] rows the screening kernel deferred to the exact kernel (k_greedy_fast).
__device__ unsigned long long g_diag[5];

struct Params {
  const float* x;
  int64_t rows;
  int64_t ld;
  int d;
  int b;
  double r;
  int aux;
  int stride;   // packed row stride (bytes)
  int half;     // ceil(d/2)
  uint8_t* packed;
  double* lo_out;
  double* hi_out;
  int32_t* info0;
  int32_t* info1;
  int32_t* status;
  // ASYM-family range of a row: 0 (min, max) clipping.py:58-61; 1 SYM (-max|x|, max|x|)
  // clipping.py:51-55; 2 TABLE: one (min, max) over the table, clipping.py:64-67
  int range_mode;
  const int* trange;  // TABLE: order-preserving int keys of the table min / max (device)
  // GREEDY constants (host-computed)
  int it_exact_from;  // loop iterations < this have a provably true condition
  double qY, inv_qY;  // Y grid quantum and inverse
  float delta;        // qY / 2
  float tau2;         // relative band coefficient, both sides (incl. reference grid rounding)
  float kmis;         // misround band per W^2, both sides (<= 2 misrounded elements per side)
  float kmisx;        // extra band per W^2 when every element of a side may misround
  float c1;           // Yh quantisation band: 4.2 * delta * sqrt(d)
  float c0;           // 2.1 * d * delta^2
  // GREEDY two-pass scheme (vector rows): the screening kernel appends the rows it
  // defers to dlist (indices into this launch's rows) and counts them in *dcount;
  // k_greedy with list != 0 then runs exactly those rows
  uint32_t* dlist;
  int* dcount;
  int list;          // k_greedy: 0 all rows, 1 the deferred rows (restart list + resume records)
  // resume records (b <= 65535): a row deferred during the walk is stored with its state at
  // the last checkpoint (iteration 8k, k = 1..RG_GROUPS-1) in group k -- {row, nl | bi << 16,
  // bj, Lbest bits} -- and k_greedy (list mode) continues it from iteration 8k
  uint4* drec;
  int* drec_count;   // [RG_GROUPS]; [0] unused
  int drec_cap;      // records per group
  // table walk (k_greedy_table, eq4_gtable.cuh): band = tb_eps mr L + (tb_c1a + tb_c1b mr) sqrt(L) + tb_c0
  // with mr = max(1, max|x| / (max - min)) of the row
  double tb_eps, tb_c1a, tb_c1b, tb_c0;
  int tb_wave;   // blocks per grid wave (the SM count): picks each block's walking warp
  int tb_defer_at;   // tests: the table walk defers every row at this iteration (-1: off)
};
constexpr int RG_GROUPS = 8;   // checkpoints at iterations 8, 16, ..., 56

// Copy nbytes from shared src to global dst; src and dst agree modulo 16.
__device__ __forceinline__ void copy_out(uint8_t* dst, const uint8_t* src, int nbytes) {
  int head = (int)((16 - ((uintptr_t)dst & 15)) & 15);
  if (head > nbytes) head = nbytes;
  int nvec = (nbytes - head) >> 4;
  int tail = head + (nvec << 4);
  for (int i = threadIdx.x; i < head; i += NTHREADS) dst[i] = src[i];
  const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  for (int i = threadIdx.x; i < nvec; i += NTHREADS) d4[i] = s4[i];
  for (int i = tail + threadIdx.x; i < nbytes; i += NTHREADS) dst[i] = src[i];
}

template <int LPR>
__device__ __forceinline__ float group_min(float v) {
#pragma unroll
  for (int o = LPR / 2; o >= 1; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
template <int LPR>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = LPR / 2; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
template <int LPR>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = LPR / 2; o >= 1; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
template <int LPR>
__device__ __forceinline__ unsigned group_umax(unsigned v) {
#pragma unroll
  for (int o = LPR / 2; o >= 1; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
template <int LPR>
__device__ __forceinline__ bool group_any(bool v) {
  unsigned bal = __ballot_sync(FULL, v);
  if (LPR == 32) return bal != 0;
  const int lane = threadIdx.x & 31;
  const unsigned gm = (unsigned)((1ull << LPR) - 1ull) << (lane & ~(LPR - 1));
  return (bal & gm) != 0;
}

// Sum a pair of per-lane partials over the LPR lanes of a group.  Every lane
// of the group ends with bit-identical (SL, SR), so decisions stay uniform.
template <int LPR>
__device__ __forceinline__ void group_sum_pair(float aL, float aR, float& SL, float& SR) {
  if (LPR == 1) {
    SL = aL;
    SR = aR;
    return;
  }
  constexpr int HB = LPR / 2;
  const bool upper = (threadIdx.x & HB) != 0;
  float send = upper ? aL : aR;
  float keep = upper ? aR : aL;
  keep = __fadd_rn(keep, __shfl_xor_sync(FULL, send, HB));
#pragma unroll
  for (int o = HB / 2; o >= 1; o >>= 1) keep = __fadd_rn(keep, __shfl_xor_sync(FULL, keep, o));
  float other = __shfl_xor_sync(FULL, keep, HB);
  SL = upper ? other : keep;
  SR = upper ? keep : other;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// 1 / (W alpha): rcp.approx (1 ulp) refined by one Newton step (W alpha is exact in fp32 for
// W < 2^18): the search's code argument alpha * sat(z * kW + h) is then within
// ETA_CODE of (z / W + 1/2).
__device__ __forceinline__ float kw_of(float Wf) {
  const float x = Wf * ALPHA;            // exact (W < 2^18)
  const float r = rcp_approx(x);         // within 1 ulp
  return __fmaf_rn(r, __fmaf_rn(-x, r, 1.f), r);   // one Newton step: 1/x within 2^-24 + 2^-46
}

__device__ __forceinline__ float sat_fma(float a, float b, float c) {
  float r;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// ---------------------------------------------------------------------------
// shared row helpers (both methods)
// ---------------------------------------------------------------------------

// Number of valid slots of lane q (masked kernels: slot i holds element q + LPR*i).
template <int LPR, int E, bool VEC>
__device__ __forceinline__ int valid_slots(int q, int d) {
  if (VEC) return E;
  int n = (d - q + LPR - 1) / LPR;
  return n < 0 ? 0 : (n > E ? E : n);
}

template <int LPR, int E, bool VEC>
__device__ __forceinline__ void load_row(const Params& p, int64_t row, bool rvalid, int q, int nv,
                                         float (&v)[E]) {
  const float* xrow = p.x + (rvalid ? row : 0) * p.ld;
  if (VEC) {
    const float4* src = reinterpret_cast<const float4*>(xrow);
#pragma unroll
    for (int c = 0; c < E / 4; ++c) {
      float4 t = rvalid ? __ldcs(src + q + LPR * c) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * c] = t.x; v[4 * c + 1] = t.y; v[4 * c + 2] = t.z; v[4 * c + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = (rvalid && i < nv) ? __ldcs(xrow + q + LPR * i) : 0.f;
  }
}

// Row min / max over the group + finiteness (table.py:28-29, clipping.py:58-61).
template <int LPR, int E, bool VEC>
__device__ __forceinline__ void row_minmax(const Params& p, const float (&v)[E], int nv, bool rvalid,
                                           int q, float& mn, float& mx, bool& bad) {
  mn = INFINITY;
  mx = -INFINITY;
  float sm = 0.f;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    if (VEC || i < nv) {
      mn = fminf(mn, v[i]);
      mx = fmaxf(mx, v[i]);
      sm = __fadd_rn(sm, v[i]);   // NaN/Inf propagate; overflow only gives a false alarm
    }
  }
  mn = group_min<LPR>(mn);
  mx = group_max<LPR>(mx);
  sm = group_sum<LPR>(sm);
  if (__any_sync(FULL, rvalid && (mn == 0.f || mx == 0.f))) {   // rare: numpy's signed-zero choice
    unsigned kz = 0u;
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (VEC || i < nv) kz = max(kz, np_zero_key(v[i], VEC ? 4 * (q + LPR * (i >> 2)) + (i & 3) : q + LPR * i, p.d));
    np_zero_apply(group_umax<LPR>(kz), mn, mx);
  }
  bad = false;
  if (__any_sync(FULL, !isfinite(sm) && rvalid)) {
    bool lb = false;
#pragma unroll
    for (int i = 0; i < E; ++i) lb |= (VEC || i < nv) && !isfinite(v[i]);
    bad = group_any<LPR>(lb) && rvalid;
    if (bad && q == 0 && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
  }
}

// Codes (uniform.py:77-79) into the staged row + scale/bias (uniform.py:80,
// packed.py:79-82).  VEC: nibbles straight into the packed row; masked: one
// code byte per element into crow (packed by pack_tile).
// Warp-collective: every lane of the warp must call it (rvalid gates stores).
template <int LPR, int E, bool VEC>
__device__ __forceinline__ void emit_row(const Params& p, const float (&v)[E], int nv, double lo,
                                         double hi, bool range_ok, bool rvalid, int q, uint8_t* orow,
                                         uint8_t* crow) {
  const CodeParams cp = make_code_params(range_ok ? lo : 0.0, range_ok ? hi : 0.0);
  unsigned long long need = 0ull;
  if (VEC) {
#pragma unroll
    for (int c = 0; c < E / 4; ++c) {
      bool n0, n1, n2, n3;
      unsigned c0 = code_of(v[4 * c], cp, n0), c1 = code_of(v[4 * c + 1], cp, n1);
      unsigned c2 = code_of(v[4 * c + 2], cp, n2), c3 = code_of(v[4 * c + 3], cp, n3);
      need |= (unsigned long long)(n0 | (n1 << 1) | (n2 << 2) | (n3 << 3)) << (4 * c);
      const int byte = 2 * (q + LPR * c);
      if (rvalid) {
        orow[byte] = (uint8_t)(c0 | (c1 << 4));
        orow[byte + 1] = (uint8_t)(c2 | (c3 << 4));
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (i < nv) {
        bool ne;
        const uint8_t c = (uint8_t)code_of(v[i], cp, ne);
        if (rvalid) crow[q + LPR * i] = c;
        need |= (unsigned long long)ne << i;
      }
    }
  }
  if (!rvalid) need = 0ull;
  if (__any_sync(FULL, need != 0ull)) {   // rare: float64 codec for near-boundary elements
    for (int i = 0; i < E; ++i) {
      if (!((need >> i) & 1ull)) continue;
      unsigned c = code_exact(v[i], cp);
      if (VEC) {
        const int byte = 2 * (q + LPR * (i >> 2)) + ((i & 3) >> 1);
        const int sh = (i & 1) * 4;
        orow[byte] = (uint8_t)((orow[byte] & ~(0xF << sh)) | (c << sh));
      } else {
        crow[q + LPR * i] = (uint8_t)c;
      }
    }
  }
  if (q == 0 && rvalid) {
    uint8_t* a = orow + p.half;
    const double sc = range_ok ? cp.scale : 0.0;
    if (p.aux == EQ4_AUX_FP16) {
      uint32_t s = aux_bits_f16(sc), bb = aux_bits_f16(lo);
      a[0] = s & 0xff; a[1] = s >> 8; a[2] = bb & 0xff; a[3] = bb >> 8;
    } else {
      uint32_t s = aux_bits_f32(sc), bb = aux_bits_f32(lo);
#pragma unroll
      for (int k = 0; k < 4; ++k) { a[k] = (s >> (8 * k)) & 0xff; a[4 + k] = (bb >> (8 * k)) & 0xff; }
    }
  }
}

// Finish a tile: (masked) nibble packing from the code tile, then 16-byte
// stores of the staged rows.
template <int D, bool VEC>
__device__ __forceinline__ void store_tile(const Params& p, const uint8_t* codes_s, uint8_t* out_tile,
                                           int tile_rows, size_t gofs) {
  if (!VEC) {
    __syncthreads();
    const int nb = tile_rows * p.half;
    for (int t = threadIdx.x; t < nb; t += NTHREADS) {
      int rr = t / p.half, m = t - rr * p.half;
      unsigned c0 = codes_s[rr * D + 2 * m];
      unsigned c1 = (2 * m + 1 < p.d) ? codes_s[rr * D + 2 * m + 1] : 0u;  // packed.py:75-76
      out_tile[rr * p.stride + m] = (uint8_t)(c0 | (c1 << 4));
    }
  }
  __syncthreads();
  copy_out(p.packed + gofs, out_tile, tile_rows * p.stride);
  __syncthreads();
}

// ASYM codes + aux for the vector path: lo = min, hi = max are floats, so
// every element is interior and the code is floor(t + 1/2) with
// t = (x - min) * 15/(max - min) evaluated in fp32 (|error| <= 90u < NEAR,
// see code_of); near-boundary elements (|frac(t) - 1/2| < NEAR) take the float64
// codec.  6 FMA-pipe + 1 ALU instruction per element, 1 ALU per 4 for packing.
template <int LPR, int E>
__device__ __forceinline__ void emit_asym_vec(const Params& p, const float (&v)[E], float mn,
                                              float mx, bool ok, bool rvalid, int q, uint8_t* orow) {
  const float w32 = __fadd_rn(mx, -mn);
  const bool degenerate = !(mn != mx);                 // uniform.py:74-76 (also NaN rows)
  const bool fast = ok && w32 > 1e-30f && w32 < 1e30f;
  const float inv = fast ? __fdividef(15.f, w32) : 0.f;
  float gmax = 0.f;
#pragma unroll
  for (int c = 0; c < E / 4; ++c) {
    uint32_t mb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float t = __fmul_rn(__fadd_rn(v[4 * c + k], -mn), inv);
      const float m = __fadd_rd(__fadd_rn(t, 0.5f), MAGIC);   // 2^23 + floor(t + 1/2)
      const float g = __fadd_rn(t, -__fadd_rn(m, -MAGIC));
      gmax = fmaxf(gmax, fabsf(g));
      mb[k] = __float_as_uint(m);
    }
    const uint32_t lo8 = (mb[0] & 0xFu) | ((mb[1] & 0xFu) << 4);
    const uint32_t hi8 = (mb[2] & 0xFu) | ((mb[3] & 0xFu) << 4);
    if (rvalid) *reinterpret_cast<uint16_t*>(orow + 2 * (q + LPR * c)) = (uint16_t)(lo8 | (hi8 << 8));
  }
  const bool need = rvalid && ok && !degenerate && (!fast || gmax > 0.5f - NEAR);
  if (__any_sync(FULL, need)) {   // rare: float64 codec (uniform.py:77-79) for flagged elements
    if (need) {
      const CodeParams cp = make_code_params((double)mn, (double)mx);
      for (int i = 0; i < E; ++i) {
        const float t = __fmul_rn(__fadd_rn(v[i], -mn), inv);
        const float m = __fadd_rd(__fadd_rn(t, 0.5f), MAGIC);
        const float g = __fadd_rn(t, -__fadd_rn(m, -MAGIC));
        if (fast && !(fabsf(g) > 0.5f - NEAR)) continue;
        const unsigned cc = code_exact(v[i], cp);
        const int byte = 2 * (q + LPR * (i >> 2)) + ((i & 3) >> 1);
        const int sh = (i & 1) * 4;
        orow[byte] = (uint8_t)((orow[byte] & ~(0xF << sh)) | (cc << sh));
      }
    }
  }
  if (degenerate && rvalid) {
#pragma unroll
    for (int c = 0; c < E / 4; ++c) *reinterpret_cast<uint16_t*>(orow + 2 * (q + LPR * c)) = 0;
  }
  if (q == 0 && rvalid) {
    const double sc = (ok && !degenerate) ? div15(__dsub_rn((double)mx, (double)mn)) : 0.0;
    uint8_t* a = orow + p.half;
    if (p.aux == EQ4_AUX_FP16) {
      const uint32_t w = aux_bits_f16(sc) | (aux_bits_f16((double)mn) << 16);
      *reinterpret_cast<uint16_t*>(a) = (uint16_t)w;
      *reinterpret_cast<uint16_t*>(a + 2) = (uint16_t)(w >> 16);
    } else {
      const uint32_t s32 = aux_bits_f32(sc), b32 = aux_bits_f32((double)mn);
      *reinterpret_cast<uint16_t*>(a) = (uint16_t)s32;
      *reinterpret_cast<uint16_t*>(a + 2) = (uint16_t)(s32 >> 16);
      *reinterpret_cast<uint16_t*>(a + 4) = (uint16_t)b32;
      *reinterpret_cast<uint16_t*>(a + 6) = (uint16_t)(b32 >> 16);
    }
  }
}

// Order-preserving float <-> int keys (signed compare), for the TABLE min/max reduction.
__device__ __forceinline__ int float_key(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float key_float(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

// The ASYM family's row range from the row's (min, max): SYM uses (-M, M) with
// M = max|x| (np.max(np.abs(x)), so an all-zero row gives (-0.0, +0.0)); TABLE
// the table-wide range.  Every element then lies inside the range, so the
// fast code path needs no clamping.
template <int RM>
__device__ __forceinline__ void apply_range_mode(const Params& p, float& mn, float& mx) {
  if constexpr (RM == 1) {
    const float m = fmaxf(fabsf(mn), fabsf(mx));
    mn = -m;
    mx = m;
  } else if constexpr (RM == 2) {
    mn = key_float(__ldg(p.trange));
    mx = key_float(__ldg(p.trange + 1));
  }
}

__global__ void k_table_init(int* keys) {
  keys[0] = 0x7fffffff;               // min key
  keys[1] = (int)0x80000000;          // max key
}

// Table-wide min / max (clipping.py:64-67: np.min / np.max over all values):
// warps stride over rows, lanes over the row (float4 when rows are 16-byte
// aligned), then one warp reduction and two atomics per warp.
__global__ void __launch_bounds__(256) k_table_minmax(const float* x, int64_t rows, int d, int64_t ld,
                                                     int* keys) {
  int kmin = 0x7fffffff, kmax = (int)0x80000000;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t wn = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (d % 4 == 0) && (ld % 4 == 0) && (((uintptr_t)x & 15) == 0);
  if (vec && ld == d) {   // contiguous table: one flat float4 stream, 4 loads in flight per thread
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int64_t n4 = rows * (int64_t)d / 4;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, ts = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t0; i < n4; i += 4 * ts) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = i + u * ts < n4 ? __ldcs(x4 + i + u * ts) : x4[t0 < n4 ? t0 : 0];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        kmin = min(kmin, min(min(float_key(v[u].x), float_key(v[u].y)), min(float_key(v[u].z), float_key(v[u].w))));
        kmax = max(kmax, max(max(float_key(v[u].x), float_key(v[u].y)), max(float_key(v[u].z), float_key(v[u].w))));
      }
    }
  } else for (int64_t r = w0; r < rows; r += wn) {
    const float* row = x + r * ld;
    if (vec) {
      const float4* r4 = reinterpret_cast<const float4*>(row);
      for (int k = lane; k < d / 4; k += 32) {
        const float4 v = __ldcs(r4 + k);
        kmin = min(kmin, min(min(float_key(v.x), float_key(v.y)), min(float_key(v.z), float_key(v.w))));
        kmax = max(kmax, max(max(float_key(v.x), float_key(v.y)), max(float_key(v.z), float_key(v.w))));
      }
    } else {
      for (int k = lane; k < d; k += 32) {
        const int key = float_key(__ldcs(row + k));
        kmin = min(kmin, key);
        kmax = max(kmax, key);
      }
    }
  }
  kmin = __reduce_min_sync(FULL, kmin);
  kmax = __reduce_max_sync(FULL, kmax);
  // one pair of atomics per block (not per warp): the two global words are every block's target
  __shared__ int bmin[8], bmax[8];
  const int warp = threadIdx.x >> 5;
  if (lane == 0) { bmin[warp] = kmin; bmax[warp] = kmax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) { kmin = min(kmin, bmin[w]); kmax = max(kmax, bmax[w]); }
    atomicMin(keys, kmin);
    atomicMax(keys + 1, kmax);
  }
}

// ---------------------------------------------------------------------------
// ASYM: min/max -> codes -> pack (HBM-bound streaming kernel)
// ---------------------------------------------------------------------------
template <int LPR, int E, bool VEC>
struct LayoutA {
  static constexpr int RPB = NTHREADS / LPR;
  static constexpr int D = LPR * E;
  __host__ __device__ static size_t out_off() { return VEC ? 0 : (((size_t)RPB * D + 15) & ~(size_t)15); }
  __host__ __device__ static size_t total(int stride) { return out_off() + (size_t)RPB * stride + 32; }
};

template <int LPR, int E, bool VEC, int RM>
__global__ void __launch_bounds__(NTHREADS, E <= 16 ? 4 : (E == 32 ? 3 : 2))
k_asym(const Params p) {
  using L = LayoutA<LPR, E, VEC>;
  constexpr int RPB = L::RPB;
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  const int g = tid / LPR, q = tid % LPR;
  uint8_t* codes_s = smem;
  uint8_t* out_base = smem + L::out_off();
  const int nv = valid_slots<LPR, E, VEC>(q, p.d);
  const int64_t ntiles = (p.rows + RPB - 1) / RPB;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * RPB, row = row0 + g;
    const bool rvalid = row < p.rows;
    const int tile_rows = (int)min((int64_t)RPB, p.rows - row0);
    const size_t gofs = (size_t)row0 * p.stride;
    uint8_t* out_tile = out_base + (((uintptr_t)p.packed + gofs) & 15);
    float v[E];
    load_row<LPR, E, VEC>(p, row, rvalid, q, nv, v);
    float mn, mx;
    bool bad;
    row_minmax<LPR, E, VEC>(p, v, nv, rvalid, q, mn, mx, bad);
    apply_range_mode<RM>(p, mn, mx);
    const double lo = (double)mn, hi = (double)mx;   // clipping.py:61
    if (VEC)
      emit_asym_vec<LPR, E>(p, v, mn, mx, !bad, rvalid, q, out_tile + g * p.stride);
    else
      emit_row<LPR, E, VEC>(p, v, nv, lo, hi, !bad, rvalid, q, out_tile + g * p.stride,
                            codes_s + g * L::D);
    if (rvalid) {
      if (q == 0) {
        if (p.lo_out) { p.lo_out[row] = lo; p.hi_out[row] = hi; }
        if (p.info0) p.info0[row] = 0;
        if (p.info1) p.info1[row] = 0;
      }
    }
    store_tile<L::D, VEC>(p, codes_s, out_tile, tile_rows, gofs);
  }
}

// ---------------------------------------------------------------------------
// GREEDY: clipping.py:142-193, fused with the codec and the packer
// ---------------------------------------------------------------------------

// Rarely-touched float64 state of one row's walk, kept in shared memory so the
// hot loop holds only the row slice (Yh) and a few scalars in registers.
struct RowShared {
  double x0, x1, step, min_steps, kY, kY2, best_ex, elo, ehi;
  int64_t rid;   // list mode: the row's index in the table
};

// Per-warp shared-memory slice of the GREEDY kernel.  Warps run independently
// (no block-wide barrier anywhere), so a warp that stalls on an exact
// re-decision never holds up the others.
template <int LPR, int E, bool VEC>
struct WarpSliceG {
  static constexpr int RPW = 32 / LPR;
  static constexpr int D = LPR * E;
  static constexpr int E2CAP = D < 512 ? D : 512;
  // numpy pairwise leaves of a row of <= D elements (leaves hold 64..128 above 128)
  static constexpr int LEAVES = D / 64 + 2 > MAX_LEAVES ? D / 64 + 2 : MAX_LEAVES;
  __host__ __device__ static size_t ys_off() { return 0; }                            // E/4 x 32 float4
  __host__ __device__ static size_t rs_off() { return ys_off() + (size_t)E * 32 * 4; }
  __host__ __device__ static size_t e2_off() { return rs_off() + RPW * sizeof(RowShared); }
  __host__ __device__ static size_t leaf_off() { return e2_off() + (size_t)E2CAP * 8; }
  __host__ __device__ static size_t codes_off() { return leaf_off() + (size_t)LEAVES * 16; }
  __host__ __device__ static size_t out_off() {
    return (codes_off() + (VEC ? 0 : (size_t)RPW * D) + 15) & ~(size_t)15;
  }
  // per-warp rare-path counters (g_diag), flushed once when the warp exits
  __host__ __device__ static size_t diag_off(int stride) {
    return (out_off() + (size_t)RPW * stride + 32 + 15) & ~(size_t)15;
  }
  __host__ __device__ static size_t bytes(int stride) { return diag_off(stride) + 16; }
};

// Warp-level copy of nbytes from shared src to global dst (equal modulo 16).
__device__ __forceinline__ void warp_copy_out(uint8_t* dst, const uint8_t* src, int nbytes) {
  const int lane = threadIdx.x & 31;
  int head = (int)((16 - ((uintptr_t)dst & 15)) & 15);
  if (head > nbytes) head = nbytes;
  const int nvec = (nbytes - head) >> 4;
  const int tail = head + (nvec << 4);
  if (lane < head) dst[lane] = src[lane];
  const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  for (int i = lane; i < nvec; i += 32) d4[i] = s4[i];
  for (int i = tail + lane; i < nbytes; i += 32) dst[i] = src[i];
}

// ---------------------------------------------------------------------------
// Packed fp32x2 arithmetic (sm_100: one instruction, two IEEE fp32 lanes).
// The FP32 pipe throughput is unchanged, but every packed instruction frees
// an issue slot for the search's bookkeeping.
// ---------------------------------------------------------------------------
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk2(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(f2_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t add2_rm(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t fma2_rm(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

#ifndef G_UNROLL
#define G_UNROLL 16
#endif
constexpr int kGUnroll = G_UNROLL;   // float4 chunks per trip of the element loop

// One fast candidate: approximate loss (Y units) of base B, width W.  The row
// slice is read from shared memory (ys4[c * 32 + lane] holds slots 4c..4c+3)
// so that registers hold one chunk of temporaries, not the whole slice.
template <int E, bool MASKED>
__device__ __forceinline__ float eval_one(const float4* ys4, int nv, float B, float nW, float kW,
                                          float h) {
  const int lane = threadIdx.x & 31;
  float s = 0.f;
#pragma unroll kGUnroll
  for (int c = 0; c < E / 4; ++c) {
    const float4 y4 = ys4[c * 32 + lane];
    const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float z = __fadd_rn(yv[k], -B);
      float t = sat_fma(z, kW, h);
      float m = __fmaf_rd(t, ALPHA, MAGIC);
      float cc = __fadd_rn(m, -MAGIC);
      float e = __fmaf_rn(cc, nW, z);
      if (!MASKED || 4 * c + k < nv) s = __fmaf_rn(e, e, s);
    }
  }
  return s;
}

// The two candidates of one iteration share W: L = (BL, W), R = (BL - 15, W).
// 6 fp32 instructions per element and candidate.
template <int E, bool MASKED>
__device__ __forceinline__ void eval_pair(const float4* ys4, int nv, float BL, float nW, float kW,
                                          float h, float& aL, float& aR) {
  const int lane = threadIdx.x & 31;
  float sL = 0.f, sR = 0.f;
#pragma unroll kGUnroll
  for (int c = 0; c < E / 4; ++c) {
    const float4 y4 = ys4[c * 32 + lane];
    const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float zL = __fadd_rn(yv[k], -BL);
      float zR = __fadd_rn(zL, 15.f);                     // exact
      float tL = sat_fma(zL, kW, h);
      float tR = sat_fma(zR, kW, h);
      float mL = __fmaf_rd(tL, ALPHA, MAGIC);             // 2^23 + floor(alpha * t)
      float mR = __fmaf_rd(tR, ALPHA, MAGIC);
      float cL = __fadd_rn(mL, -MAGIC);
      float cR = __fadd_rn(mR, -MAGIC);
      float eL = __fmaf_rn(cL, nW, zL);                   // exact
      float eR = __fmaf_rn(cR, nW, zR);
      if (!MASKED || 4 * c + k < nv) {
        sL = __fmaf_rn(eL, eL, sL);
        sR = __fmaf_rn(eR, eR, sR);
      }
    }
  }
  aL = sL;
  aR = sR;
}

// Packed variant of eval_pair (vector kernels): element pairs share one
// instruction for z, the round-down code, the code removal, the error and the
// accumulation; only the saturating FFMA stays scalar (no .sat for f32x2).
// 3.5 issue slots per element and candidate instead of 6.
// Accumulator chains per candidate and f32x2 half in the packed evaluations: chunk c adds
// into chain c % NACC, the chains are summed as a tree at the end.  Shorter chains tighten
// the fp32 error band (tau2_for: E/(2 NACC) terms per chain + log2 NACC tree levels), which
// matters for the wide rows (E = 128..512: 64..256-term chains otherwise).
#ifndef G_NACC64
#define G_NACC64 1
#endif
__host__ __device__ constexpr int nacc_for(int E) { return E >= 128 ? 4 : (E == 64 ? G_NACC64 : 1); }

template <int N>
__device__ __forceinline__ float acc_tree(const f2_t (&s)[N]) {
  f2_t t = s[0];
  if constexpr (N == 2) t = add2(s[0], s[1]);
  if constexpr (N == 4) t = add2(add2(s[0], s[1]), add2(s[2], s[3]));
  float a, b;
  upk2(t, a, b);
  return __fadd_rn(a, b);
}

// Packed variant of eval_pair (vector kernels): element pairs share one
// instruction for z, the round-down code, the code removal, the error and the
// accumulation; only the saturating FFMA stays scalar (no .sat for f32x2).
// 3.5 issue slots per element and candidate instead of 6.
template <int E>
__device__ __forceinline__ void eval_pair_x2(const float4* ys4, float BL, float nW, float kW,
                                             float h, float& aL, float& aR) {
  constexpr int NA = nacc_for(E);
  const f2_t nBL2 = pk2(-BL, -BL), c15 = pk2(15.f, 15.f), al2 = pk2(ALPHA, ALPHA);
  const f2_t mg2 = pk2(MAGIC, MAGIC), nmg2 = pk2(-MAGIC, -MAGIC), nW2 = pk2(nW, nW);
  f2_t sL[NA], sR[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) { sL[a] = pk2(0.f, 0.f); sR[a] = pk2(0.f, 0.f); }
#pragma unroll (kGUnroll / NA > 0 ? kGUnroll / NA : 1)
  for (int c0 = 0; c0 < E / 4; c0 += NA) {
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const ulonglong2 yy = *reinterpret_cast<const ulonglong2*>(ys4 + (c0 + a) * 32);
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        const f2_t y2 = hlf ? yy.y : yy.x;
        const f2_t zL = add2(y2, nBL2);
        const f2_t zR = add2(zL, c15);                                   // exact
        float a0, a1, b0, b1;
        upk2(zL, a0, a1);
        upk2(zR, b0, b1);
        const f2_t tL = pk2(sat_fma(a0, kW, h), sat_fma(a1, kW, h));
        const f2_t tR = pk2(sat_fma(b0, kW, h), sat_fma(b1, kW, h));
        const f2_t cL = add2(fma2_rm(tL, al2, mg2), nmg2);              // floor(alpha * t)
        const f2_t cR = add2(fma2_rm(tR, al2, mg2), nmg2);
        const f2_t eL = fma2(cL, nW2, zL);                               // exact
        const f2_t eR = fma2(cR, nW2, zR);
        sL[a] = fma2(eL, eL, sL[a]);
        sR[a] = fma2(eR, eR, sR[a]);
      }
    }
  }
  aL = acc_tree<NA>(sL);
  aR = acc_tree<NA>(sR);
}

// Packed pair evaluation with R derived from L (valid for W > 15): the R grid
// is the L grid shifted by 15 < W, so zR = zL + 15 moves every code by at
// most one:  cR = min(cL + [eL + 15 >= W/2], 15)  (below-window elements have
// eL + 15 < W/2, top-code elements keep 15), hence
//   eR = eL + (15 - W [eL >= W/2 - 15 and cL < 15]),
// all exact in fp32 (eL and the constants are multiples of qY well below
// 2^24 qY).  R costs 2 FMA-pipe instructions per element pair (add, square-
// accumulate) + 3 ALU ones per element, instead of 7 FMA-pipe ones per pair.
// (e >= thr and m < top) ? a : b -- one FSETP, one FSETP with the first
// predicate folded into its boolean combine, one FSEL.
__device__ __forceinline__ float sel_ge_lt(float e, float thr, float m, float top, float a, float b) {
  float r;
  asm("{\n\t.reg .pred p, q;\n\tsetp.lt.f32 p, %2, %3;\n\tsetp.ge.and.f32 q, %1, %4, p;\n\t"
      "selp.f32 %0, %5, %6, q;\n\t}"
      : "=f"(r) : "f"(e), "f"(m), "f"(top), "f"(thr), "f"(a), "f"(b));
  return r;
}

template <int E>
__device__ __forceinline__ void eval_pair_x2_shift(const float4* ys4, float BL, float nW, float kW,
                                                   float h, float& aL, float& aR) {
  constexpr int NA = nacc_for(E);
  const f2_t nBL2 = pk2(-BL, -BL), al2 = pk2(ALPHA, ALPHA);
  const f2_t mg2 = pk2(MAGIC, MAGIC), nmg2 = pk2(-MAGIC, -MAGIC), nW2 = pk2(nW, nW);
  // eR = eL + (15 - W k):  k = [eL + 15 >= W/2] and [cL < 15]
  const float thr = -0.5f * nW - 15.f, cW = 15.f + nW, top = MAGIC + 15.f;   // ulp(2^23) = 1
  f2_t sL[NA], sR[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) { sL[a] = pk2(0.f, 0.f); sR[a] = pk2(0.f, 0.f); }
#pragma unroll (kGUnroll / NA > 0 ? kGUnroll / NA : 1)
  for (int c0 = 0; c0 < E / 4; c0 += NA) {
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const ulonglong2 yy = *reinterpret_cast<const ulonglong2*>(ys4 + (c0 + a) * 32);
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        const f2_t zL = add2(hlf ? yy.y : yy.x, nBL2);
        float a0, a1;
        upk2(zL, a0, a1);
        const f2_t mL = fma2_rm(pk2(sat_fma(a0, kW, h), sat_fma(a1, kW, h)), al2, mg2);   // 2^23 + cL
        const f2_t eL = fma2(add2(mL, nmg2), nW2, zL);                                    // exact
        float e0, e1, m0, m1;
        upk2(eL, e0, e1);
        upk2(mL, m0, m1);
        const float c0v = sel_ge_lt(e0, thr, m0, top, cW, 15.f);
        const float c1v = sel_ge_lt(e1, thr, m1, top, cW, 15.f);
        const f2_t eR = add2(eL, pk2(c0v, c1v));                                          // exact
        sL[a] = fma2(eL, eL, sL[a]);
        sR[a] = fma2(eR, eR, sR[a]);
      }
    }
  }
  aL = acc_tree<NA>(sL);
  aR = acc_tree<NA>(sR);
}

// Packed single-candidate loss (the full range, clipping.py:174).
template <int E>
__device__ __forceinline__ float eval_one_x2(const float4* ys4, float B, float nW, float kW, float h) {
  constexpr int NA = nacc_for(E);
  const f2_t nB2 = pk2(-B, -B), al2 = pk2(ALPHA, ALPHA);
  const f2_t mg2 = pk2(MAGIC, MAGIC), nmg2 = pk2(-MAGIC, -MAGIC), nW2 = pk2(nW, nW);
  f2_t acc[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = pk2(0.f, 0.f);
#pragma unroll (kGUnroll / NA > 0 ? kGUnroll / NA : 1)
  for (int c0 = 0; c0 < E / 4; c0 += NA) {
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const ulonglong2 yy = *reinterpret_cast<const ulonglong2*>(ys4 + (c0 + a) * 32);
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        const f2_t z = add2(hlf ? yy.y : yy.x, nB2);
        float a0, a1;
        upk2(z, a0, a1);
        const f2_t t = pk2(sat_fma(a0, kW, h), sat_fma(a1, kW, h));
        const f2_t e = fma2(add2(fma2_rm(t, al2, mg2), nmg2), nW2, z);
        acc[a] = fma2(e, e, acc[a]);
      }
    }
  }
  return acc_tree<NA>(acc);
}

// Y coordinates on the exact fp32 grid of quantum qY (see file header).
template <int LPR, int E, bool VEC>
__device__ __forceinline__ void make_Y(const Params& p, const float* xr, int q, int nv, double x0,
                                       double kY, bool active, float (&Yh)[E]) {
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const float x = (VEC || i < nv) ? xr[VEC ? 4 * (q + LPR * (i >> 2)) + (i & 3) : q + LPR * i] : 0.f;
    const double Y = __dmul_rn(__dsub_rn((double)x, x0), kY);
    Yh[i] = active ? (float)(rint(Y * p.inv_qY) * p.qY) : 0.f;
  }
}

// Exact (reference) decision of one loop iteration for one row.  Warp-
// collective: every lane passes the owning row's (broadcast) state.
struct ExactOut {
  double vL, vR, vb;
  int flags;  // 1 = range error, 2 = move left, 4 = candidate better than best
};

template <bool INLINE_LEAF, int LEAVES>
__device__ __forceinline__ ExactOut exact_decide(RowShared* R, double nl, double nr, int bi, int bj,
                                                 bool bvalid, const float* xs, int d, double* e2,
                                                 double* leaf_sum, int* leaf_st, int* leaf_ln) {
  ExactOut o;
  const double x0 = R->x0, x1 = R->x1, st = R->step;
  o.vL = o.vR = 0.0;
  o.vb = R->best_ex;
  o.flags = 0;
  // clipping.py:181-184 candidates; ClipRange validation table.py:70-74 (L first)
  const double lmin = __dadd_rn(x0, __dmul_rn(nl + 1.0, st)), lmax = __dsub_rn(x1, __dmul_rn(nr, st));
  const double rmin = __dadd_rn(x0, __dmul_rn(nl, st)), rmax = __dsub_rn(x1, __dmul_rn(nr + 1.0, st));
  const bool errL = !(lmin <= lmax);
  const bool errR = !(rmin <= rmax);
  if (d >= 8 && d <= 128 && !errL && !errR) {   // one pairwise leaf: all ranges at once
    const double blo = bi == 0 ? x0 : __dadd_rn(x0, __dmul_rn((double)bi, st));
    const double bhi = bj == 0 ? x1 : __dsub_rn(x1, __dmul_rn((double)bj, st));
    double vb;
    if constexpr (INLINE_LEAF)   // small kernels: the call overhead outweighs the register cost
      warp_np_loss3_leaf(xs, d, bvalid ? 2 : 3, lmin, lmax, rmin, rmax, blo, bhi, o.vL, o.vR, vb);
    else
      warp_np_loss3_leaf_ool(xs, d, bvalid ? 2 : 3, lmin, lmax, rmin, rmax, blo, bhi, o.vL, o.vR, vb);
    if (!bvalid) o.vb = vb;
    const bool goL = o.vL < o.vR;                           // clipping.py:185
    o.flags = (goL ? 2 : 0) | ((goL ? o.vL : o.vR) < o.vb ? 4 : 0);   // clipping.py:187,191
    return o;
  }
  if (!errL) o.vL = warp_np_loss(xs, d, lmin, lmax, e2, leaf_sum, leaf_st, leaf_ln, LEAVES);
  if (errL || errR) {
    if ((threadIdx.x & 31) == 0) {
      R->elo = errL ? lmin : rmin;
      R->ehi = errL ? lmax : rmax;
    }
    o.flags = 1;
    return o;
  }
  o.vR = warp_np_loss(xs, d, rmin, rmax, e2, leaf_sum, leaf_st, leaf_ln, LEAVES);
  const bool goL = o.vL < o.vR;                             // clipping.py:185
  const double vc = goL ? o.vL : o.vR;
  if (!bvalid) {
    const double blo = bi == 0 ? x0 : __dadd_rn(x0, __dmul_rn((double)bi, st));
    const double bhi = bj == 0 ? x1 : __dsub_rn(x1, __dmul_rn((double)bj, st));
    o.vb = warp_np_loss(xs, d, blo, bhi, e2, leaf_sum, leaf_st, leaf_ln, LEAVES);
  }
  o.flags = (goL ? 2 : 0) | (vc < o.vb ? 4 : 0);            // clipping.py:187,191
  return o;
}

// GREEDY codes from the row slice: with the winning pair (bi, bj) the codes are
// c = clamp(floor((Y - B)/Wb + 1/2), 0, 15), B = 15 bi, Wb = b - bi - bj, i.e.
// the same saturating FFMA + round-down FFMA as the search.  Yh is within
// delta = qY/2 of Y, so when any element's fractional part is within
// NEAR + delta/Wb of a rounding boundary the row slice takes all its codes from
// the float64 codec instead (rare; clamping at lo/hi cannot flip a code: codes
// are continuous there).  ys4 is the lane's column of the slice.
// Warp-collective.
template <int LPR, int E, bool VEC>
__device__ __forceinline__ void emit_greedy(const Params& p, const float4* ys4, int nv, int q,
                                            double lo, double hi, int bi, int bj, bool fast_ok,
                                            bool ok, bool rvalid, const float* xr, uint8_t* orow,
                                            uint8_t* crow, unsigned* wdiag) {
  const int Wb = p.b - bi - bj;
  const float B = (float)(15 * bi);
  const float Wf = (float)(Wb > 0 ? Wb : 1);
  const float kW = __fdividef(1.f, Wf * ALPHA);
  const float h = 0.5f / ALPHA;
  const float nb = NEAR + p.delta / Wf;
  const bool fast = fast_ok && Wb >= 1 && ok;
  bool near = false;
  // streamed chunk by chunk (no per-slot arrays): codes go straight to the
  // staged row; a flagged slice is rewritten below
  const f2_t nB2 = pk2(-B, -B), al2 = pk2(ALPHA, ALPHA);
  const f2_t mg2 = pk2(MAGIC, MAGIC), nmg2 = pk2(-MAGIC, -MAGIC);
#pragma unroll
  for (int c = 0; c < E / 4; ++c) {
    const ulonglong2 yy = *reinterpret_cast<const ulonglong2*>(ys4 + c * 32);
    uint32_t w = 0;
#pragma unroll
    for (int hlf = 0; hlf < 2; ++hlf) {
      const f2_t z = add2(hlf ? yy.y : yy.x, nB2);
      float z0, z1;
      upk2(z, z0, z1);
      const float s0 = sat_fma(z0, kW, h), s1 = sat_fma(z1, kW, h);
      const f2_t sv = pk2(s0, s1);
      const f2_t m = fma2_rm(sv, al2, mg2);
      const f2_t fr = sub2(fma2(sv, al2, pk2(0.f, 0.f)), add2(m, nmg2));   // frac of alpha*s
      float m0, m1, f0, f1;
      upk2(m, m0, m1);
      upk2(fr, f0, f1);
      const int i0 = 4 * c + 2 * hlf;
      // |frac - 1/2| > 1/2 - nb  <=>  frac < nb or frac > 1 - nb (s strictly inside (0, 1))
      const bool n0 = s0 > 0.f && s0 < 1.f && fabsf(f0 - 0.5f) > 0.5f - nb;
      const bool n1 = s1 > 0.f && s1 < 1.f && fabsf(f1 - 0.5f) > 0.5f - nb;
      near |= (n0 && (VEC || i0 < nv)) || (n1 && (VEC || i0 + 1 < nv));
      const uint32_t c0 = ok ? (__float_as_uint(m0) & 0xFu) : 0u;
      const uint32_t c1 = ok ? (__float_as_uint(m1) & 0xFu) : 0u;
      if (VEC) {
        w |= (c0 | (c1 << 4)) << (8 * hlf);
      } else if (rvalid) {
        if (i0 < nv) crow[q + LPR * i0] = (uint8_t)c0;
        if (i0 + 1 < nv) crow[q + LPR * (i0 + 1)] = (uint8_t)c1;
      }
    }
    if (VEC && rvalid) *reinterpret_cast<uint16_t*>(orow + 2 * (q + LPR * c)) = (uint16_t)w;
  }
  if (!fast) near = ok;
  if (!rvalid) near = false;
  if (__any_sync(FULL, near)) {   // rare: float64 codec (uniform.py:77-79) for the whole slice
    if (near) {
      if (fast && q == 0) atomicAdd(&wdiag[1], 1u);
      const CodeParams cp = make_code_params(lo, hi);
      for (int c = 0; c < E / 4; ++c) {
        uint32_t w = 0;
        for (int k = 0; k < 4; ++k) {
          const int i = 4 * c + k;
          if (!VEC && i >= nv) continue;
          const unsigned cc = code_exact(xr[VEC ? 4 * (q + LPR * c) + k : q + LPR * i], cp);
          if (VEC) w |= cc << (4 * k);
          else crow[q + LPR * i] = (uint8_t)cc;
        }
        if (VEC) *reinterpret_cast<uint16_t*>(orow + 2 * (q + LPR * c)) = (uint16_t)w;
      }
    }
  }
  if (rvalid && q == 0) {
    const double sc = (ok && hi != lo) ? div15(__dsub_rn(hi, lo)) : 0.0;   // uniform.py:74-80
    uint8_t* a = orow + p.half;
    if (p.aux == EQ4_AUX_FP16) {
      const uint32_t s16 = aux_bits_f16(sc), b16 = aux_bits_f16(lo);
      a[0] = s16 & 0xff; a[1] = s16 >> 8; a[2] = b16 & 0xff; a[3] = b16 >> 8;
    } else {
      const uint32_t s32 = aux_bits_f32(sc), b32 = aux_bits_f32(lo);
#pragma unroll
      for (int k = 0; k < 4; ++k) { a[k] = (s32 >> (8 * k)) & 0xff; a[4 + k] = (b32 >> (8 * k)) & 0xff; }
    }
  }
}

// 1 if an element at z = Y - B lies within nb of a code rounding boundary of a
// candidate of width W (code argument alpha*s within nb of an integer, strictly
// inside the clamp range), computed with the search's own arithmetic.  Only such
// elements can take a different code in the fp32 loss than in the reference's,
// each moving the loss by <= 2 eta W^2.
__device__ __forceinline__ unsigned near_bnd(float z, float kW, float nb) {
  const float sv = sat_fma(z, kW, 0.5f / ALPHA);
  const float m = __fadd_rn(__fmaf_rd(sv, ALPHA, MAGIC), -MAGIC);
  const float fr = __fmaf_rn(sv, ALPHA, -m);
  return (sv > 0.f && sv < 1.f && fabsf(fr - 0.5f) > 0.5f - nb) ? 1u : 0u;
}

// Elements of group lg's row within reach of a rounding boundary for the two
// candidates of an iteration (L: base BL, R: base BL - 15, width W) and for the
// best pair so far (bi, bj): true when any of the three has more than 2 (the
// error band's allowance per side).  The whole warp counts the row's slice
// columns in one pass (three 10-bit counts packed into one reduction).
// Warp-collective with warp-uniform arguments.
template <int LPR, int E, bool VEC>
__device__ __forceinline__ bool near_over(const Params& p, const float* ysf, int lg, int d, float BL, float W,
                                          int bi, int bj, unsigned* wdiag) {
  const int lane = threadIdx.x & 31;
  const float Wb = (float)(p.b - bi - bj), Bb = (float)(15 * bi);
  const float kW = kw_of(W), kWb = kw_of(Wb);
  const float nb = NEAR_CNT + p.delta / W, nbb = NEAR_CNT + p.delta / Wb;
  unsigned cnt = 0u;
  for (int t = lane; t < LPR * E; t += 32) {
    const int qq = t % LPR, i = t / LPR;
    if (!VEC && i >= valid_slots<LPR, E, VEC>(qq, d)) continue;
    const float y = ysf[((i >> 2) * 32 + lg * LPR + qq) * 4 + (i & 3)];
    const float z = __fadd_rn(y, -BL);
    cnt += near_bnd(z, kW, nb) + (near_bnd(__fadd_rn(z, 15.f), kW, nb) << 10) +
           (near_bnd(__fadd_rn(y, -Bb), kWb, nbb) << 20);
  }
  cnt = __reduce_add_sync(FULL, cnt);
  const bool over = (cnt & 1023u) > 2u || ((cnt >> 10) & 1023u) > 2u || (cnt >> 20) > 2u;
  if (lane == 0) {
    wdiag[2] += 1u;
    wdiag[3] += over ? 1u : 0u;
  }
  return over;
}

// Strict walk: rows whose comparison lies outside the band for <= 2 misrounded
// elements per side but inside the band for all d of them (chk) count the
// elements in reach of a boundary right away; more than 2 on a side sends the
// row to the exact re-decision.  Rows one at a time; returns the lane's row's
// escalation.
template <int LPR, int E, bool VEC>
__device__ __forceinline__ bool near_escalate_body(const Params& p, const float* ysf, bool chk, int q, int gw,
                                                   int d, float BL, float W, int bi, int bj, unsigned* wdiag) {
  unsigned bal = __ballot_sync(FULL, chk && q == 0);
  bool esc = false;
  while (bal) {
    const int leader = __ffs(bal) - 1;
    bal &= bal - 1;
    const int lg = leader / LPR;
    const bool e = near_over<LPR, E, VEC>(p, ysf, lg, d, __shfl_sync(FULL, BL, leader), W,
                                          __shfl_sync(FULL, bi, leader), __shfl_sync(FULL, bj, leader), wdiag);
    if (lg == gw) esc = e;
  }
  return esc;
}
// Out of line for rows of one or two lanes (inlined into the screen's unrolled iteration it cost
// 1.9% of the 20M x 64 launch); inline for wider rows, where the call measured 1% slower.
template <int LPR, int E, bool VEC>
__device__ __noinline__ bool near_escalate_call(const Params& p, const float* ysf, bool chk, int q, int gw,
                                                int d, float BL, float W, int bi, int bj, unsigned* wdiag) {
  return near_escalate_body<LPR, E, VEC>(p, ysf, chk, q, gw, d, BL, W, bi, bj, wdiag);
}
template <int LPR, int E, bool VEC>
__device__ __forceinline__ bool near_escalate(const Params& p, const float* ysf, bool chk, int q, int gw,
                                              int d, float BL, float W, int bi, int bj, unsigned* wdiag) {
  if constexpr (LPR <= 2) return near_escalate_call<LPR, E, VEC>(p, ysf, chk, q, gw, d, BL, W, bi, bj, wdiag);
  else return near_escalate_body<LPR, E, VEC>(p, ysf, chk, q, gw, d, BL, W, bi, bj, wdiag);
}

enum : unsigned { F_ACTIVE = 1, F_EXACT_ONLY = 2, F_BEST_EX = 4, F_ERR = 8 };

// The rare path of one loop iteration: rows flagged need_ex are re-decided one
// at a time by the whole warp with the bit-exact float64 restatement.
template <int LPR, int E, bool VEC>
__device__ __forceinline__ void exact_block(const Params& p, bool need_ex, int q, int gw, int W,
                                            float SL, float SR, RowShared* rs, const float* xr,
                                            int d, double* e2, double* leaf_sum,
                                            int* leaf_st, int* leaf_ln, int& nl, int& nr, int& bi,
                                            int& bj, int& iters, unsigned& flags, float& Lbest,
                                            float& BLf, unsigned* wdiag) {
  unsigned bal = __ballot_sync(FULL, need_ex && q == 0);
  while (bal) {
    const int leader = __ffs(bal) - 1;
    bal &= bal - 1;
    const int lg = leader / LPR;
    if ((threadIdx.x & 31) == 0) wdiag[0] += 1u;
    const ExactOut o = exact_decide<(E <= 16), WarpSliceG<LPR, E, VEC>::LEAVES>(
        &rs[lg], (double)__shfl_sync(FULL, nl, leader), (double)__shfl_sync(FULL, nr, leader),
        __shfl_sync(FULL, bi, leader), __shfl_sync(FULL, bj, leader),
        (__shfl_sync(FULL, flags, leader) & F_BEST_EX) != 0,
        reinterpret_cast<const float*>(__shfl_sync(FULL, reinterpret_cast<unsigned long long>(xr), leader)),
        d, e2, leaf_sum, leaf_st,
        leaf_ln);
    if (lg == gw) {
      if (o.flags & 1) {
        flags = (flags & ~F_ACTIVE) | F_ERR;
      } else {
        const bool goL = (o.flags & 2) != 0;
        const double vc = goL ? o.vL : o.vR;
        if (goL) { ++nl; BLf += 15.f; } else { ++nr; }
        if (o.flags & 4) {
          bi = nl; bj = nr;
          if (q == 0) rs[gw].best_ex = vc;
          Lbest = (W >= 1) ? (goL ? SL : SR) : (float)(vc * rs[gw].kY2);
        } else if (q == 0) {
          rs[gw].best_ex = o.vb;
        }
        flags |= F_BEST_EX;
        ++iters;
      }
    }
    __syncwarp();
  }
}


template <int LPR, int E, bool VEC>
__global__ void __launch_bounds__(NTHREADS_G, E <= 16 ? GREEDY_MINB : (E <= 32 ? G_MINB32 : G_MINB64)) k_greedy(const Params p) {
  using S = WarpSliceG<LPR, E, VEC>;
  constexpr int RPW = S::RPW;
  constexpr int D = S::D;
  static_assert(LPR >= 1 && LPR <= 32 && (LPR & (LPR - 1)) == 0, "LPR");
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = lane / LPR, q = lane % LPR;
  unsigned char* ws = smem + warp * S::bytes(p.stride);
  float4* ys4 = reinterpret_cast<float4*>(ws + S::ys_off());
  const float4* ysl = ys4 + lane;   // this lane's column of the [E/4][32] slice
  RowShared* rs = reinterpret_cast<RowShared*>(ws + S::rs_off());
  double* e2 = reinterpret_cast<double*>(ws + S::e2_off());
  double* leaf_sum = reinterpret_cast<double*>(ws + S::leaf_off());
  int* leaf_st = reinterpret_cast<int*>(leaf_sum + S::LEAVES);
  int* leaf_ln = leaf_st + S::LEAVES;
  uint8_t* codes_w = ws + S::codes_off();
  uint8_t* out_base = ws + S::out_off();
  unsigned* wdiag = reinterpret_cast<unsigned*>(ws + S::diag_off(p.stride));
  if (lane < 4) wdiag[lane] = 0u;
  __syncwarp();
  const int d = p.d;
  const int nv = valid_slots<LPR, E, VEC>(q, d);
  const float hh = 0.5f / ALPHA;
  // list mode: the rows the screening kernel deferred (dlist[0 .. *dcount)), each
  // written on its own; otherwise blocks of RPW consecutive rows
  // list mode: the restart list (group 0) then the resume groups 1.. in one index space of
  // RPW-row units, so every warp's rows start at one iteration (8g) and the longest rows
  // (restarts) are handed out first
  int64_t gcnt[RG_GROUPS], gcum[RG_GROUPS + 1];
  gcum[0] = 0;
#pragma unroll
  for (int g = 0; g < RG_GROUPS; g++) {
    int64_t n = 0;
    if (p.list) {
      if (g == 0) n = *reinterpret_cast<volatile const int*>(p.dcount);
      else if (p.drec) n = min((int64_t)*reinterpret_cast<volatile const int*>(p.drec_count + g), (int64_t)p.drec_cap);
    }
    gcnt[g] = n;
    gcum[g + 1] = gcum[g] + (n + RPW - 1) / RPW;
  }
  const int64_t nblocks = p.list ? gcum[RG_GROUPS] : (p.rows + RPW - 1) / RPW;
  const int nwb = (int)(blockDim.x >> 5);   // warps per block (fewer for wide rows)
  const int64_t wstride = (int64_t)gridDim.x * nwb;

  for (int64_t blk = (int64_t)blockIdx.x * nwb + warp; blk < nblocks; blk += wstride) {
    int grp = 0;
#pragma unroll
    for (int g = 1; g < RG_GROUPS; g++) grp = (p.list && blk >= gcum[g]) ? g : grp;
    const int64_t row0 = p.list ? (blk - gcum[grp]) * RPW : blk * RPW;
    const int64_t nunits = p.list ? gcnt[grp] : p.rows;
    const bool rvalid = row0 + gw < nunits;
    uint4 rec = make_uint4(0u, 0u, 0u, 0u);
    if (grp > 0 && rvalid) rec = p.drec[(size_t)grp * p.drec_cap + row0 + gw];
    const int64_t row = grp > 0 ? (int64_t)rec.x : p.list ? (rvalid ? (int64_t)p.dlist[row0 + gw] : 0) : row0 + gw;
    RowShared& R = rs[gw];
    // the raw rows stay in global memory (L1/L2-resident while the block is
    // searched): only the rare exact decisions and code fix-ups read them
    const float* xr = p.x + (rvalid ? row : (p.list ? 0 : row0)) * p.ld;

    float mn, mx;
    bool bad;
    {
      // Y on the exact fp32 grid of quantum qY: Y + C rounds to a multiple of qY
      // (C = 1.5 * 2^52 * qY, same ties-to-even result as rint(Y / qY) * qY)
      const double cY = 6755399441055744.0 * p.qY;
      double x0, x1, step, kY;
      if constexpr (VEC) {
        // two streaming passes over the row slice (the second hits L1/L2), so
        // no E-element register array is live across the float64 setup
        const float4* src = reinterpret_cast<const float4*>(xr) + q;
        float lmn = INFINITY, lmx = -INFINITY;
        f2_t sm2 = pk2(0.f, 0.f);   // NaN / Inf detector: a packed running sum
#pragma unroll
        for (int c = 0; c < E / 4; ++c) {
          const float4 t = __ldg(src + LPR * c);
          lmn = fminf(lmn, fminf(fminf(t.x, t.y), fminf(t.z, t.w)));
          lmx = fmaxf(lmx, fmaxf(fmaxf(t.x, t.y), fmaxf(t.z, t.w)));
          sm2 = add2(sm2, add2(pk2(t.x, t.y), pk2(t.z, t.w)));
        }
        float s0, s1;
        upk2(sm2, s0, s1);
        float sm = __fadd_rn(s0, s1);
        mn = group_min<LPR>(lmn);
        mx = group_max<LPR>(lmx);
        sm = group_sum<LPR>(sm);
#ifndef G_NOZERO
        if (__any_sync(FULL, rvalid && (mn == 0.f || mx == 0.f))) {   // rare: numpy's signed-zero choice
#else
        if (false) {
#endif
          unsigned kz = 0u;
          for (int c = 0; c < E / 4; ++c) {
            const float4 t = __ldg(src + LPR * c);
            const int p0 = 4 * (q + LPR * c);
            kz = max(max(max(kz, np_zero_key(t.x, p0, d)), np_zero_key(t.y, p0 + 1, d)),
                     max(np_zero_key(t.z, p0 + 2, d), np_zero_key(t.w, p0 + 3, d)));
          }
          np_zero_apply(group_umax<LPR>(kz), mn, mx);
        }
        bad = false;
        if (__any_sync(FULL, !isfinite(sm) && rvalid)) {   // NaN/Inf (or a false alarm on overflow)
          bool lb = false;
          for (int c = 0; c < E / 4; ++c) {
            const float4 t = __ldg(src + LPR * c);
            lb |= !isfinite(t.x) || !isfinite(t.y) || !isfinite(t.z) || !isfinite(t.w);
          }
          bad = group_any<LPR>(lb) && rvalid;
          if (bad && q == 0 && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
        }
        x0 = (double)mn; x1 = (double)mx;
        step = __ddiv_rn(__dsub_rn(x1, x0), (double)p.b);                           // :172
        kY = (x0 != x1) ? __ddiv_rn(15.0, step) : 0.0;
#pragma unroll 4
        for (int c = 0; c < E / 4; ++c) {
          const float4 t = __ldg(src + LPR * c);
          const float tv[4] = {t.x, t.y, t.z, t.w};
          float y[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double Y = __dmul_rn(__dsub_rn((double)tv[k], x0), kY);
            y[k] = (float)__dsub_rn(__dadd_rn(Y, cY), cY);
          }
          ys4[c * 32 + lane] = make_float4(y[0], y[1], y[2], y[3]);
        }
      } else if constexpr (E > 64) {
        // wide masked rows (d > 2048): the lane's slots q + LPR*i are streamed from
        // global memory twice (L1/L2 hits the second time) -- no E-sized register array
        const float* src = xr + q;
        float lmn = INFINITY, lmx = -INFINITY, sm = 0.f;
        for (int i = 0; i < nv; ++i) {
          const float t = rvalid ? __ldg(src + LPR * i) : 0.f;
          lmn = fminf(lmn, t);
          lmx = fmaxf(lmx, t);
          sm = __fadd_rn(sm, t);
        }
        mn = group_min<LPR>(lmn);
        mx = group_max<LPR>(lmx);
        sm = group_sum<LPR>(sm);
        if (__any_sync(FULL, rvalid && (mn == 0.f || mx == 0.f))) {   // rare: numpy's signed-zero choice
          unsigned kz = 0u;
          for (int i = 0; i < nv; ++i)
            kz = max(kz, np_zero_key(rvalid ? __ldg(src + LPR * i) : 1.f, q + LPR * i, d));
          np_zero_apply(group_umax<LPR>(kz), mn, mx);
        }
        bad = false;
        if (__any_sync(FULL, !isfinite(sm) && rvalid)) {
          bool lb = false;
          for (int i = 0; i < nv; ++i) lb |= rvalid && !isfinite(__ldg(src + LPR * i));
          bad = group_any<LPR>(lb) && rvalid;
          if (bad && q == 0 && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
        }
        x0 = (double)mn; x1 = (double)mx;
        step = __ddiv_rn(__dsub_rn(x1, x0), (double)p.b);                           // :172
        kY = (x0 != x1) ? __ddiv_rn(15.0, step) : 0.0;
        for (int c = 0; c < E / 4; ++c) {
          float y[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = 4 * c + k;
            const float t = (rvalid && i < nv) ? __ldg(src + LPR * i) : 0.f;
            const double Y = __dmul_rn(__dsub_rn((double)t, x0), kY);
            y[k] = (float)__dsub_rn(__dadd_rn(Y, cY), cY);
          }
          ys4[c * 32 + lane] = make_float4(y[0], y[1], y[2], y[3]);
        }
      } else {
        float v[E];
        load_row<LPR, E, VEC>(p, row, rvalid, q, nv, v);
        row_minmax<LPR, E, VEC>(p, v, nv, rvalid, q, mn, mx, bad);
        x0 = (double)mn; x1 = (double)mx;
        step = __ddiv_rn(__dsub_rn(x1, x0), (double)p.b);                           // :172
        kY = (x0 != x1) ? __ddiv_rn(15.0, step) : 0.0;
#pragma unroll
        for (int c = 0; c < E / 4; ++c) {
          float y[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double Y = __dmul_rn(__dsub_rn((double)v[4 * c + k], x0), kY);
            y[k] = (float)__dsub_rn(__dadd_rn(Y, cY), cY);
          }
          ys4[c * 32 + lane] = make_float4(y[0], y[1], y[2], y[3]);
        }
      }
      if (q == 0) {
        R.x0 = x0; R.x1 = x1; R.step = step;
        R.min_steps = __dmul_rn(__dmul_rn((double)p.b, __dsub_rn(1.0, p.r)), step);  // :173
        R.kY = kY; R.kY2 = kY * kY; R.best_ex = 0.0; R.elo = 0.0; R.ehi = 0.0; R.rid = row;
      }
    }
    __syncwarp();
    unsigned flags = 0;
    if (rvalid && !bad && mn != mx) {                                                // :164-165
      flags = F_ACTIVE;
      const float M = fmaxf(fabsf(mn), fabsf(mx)), Dwf = mx - mn;
      if (!(M <= 1e6f * Dwf)) flags |= F_EXACT_ONLY;   // reference grid rounds coarsely
    }
    float Lbest;
    int nl = 0, nr = 0, bi = 0, bj = 0, iters = 0;
    float BLf = 15.f;                       // base of the L candidate, 15 * (nl + 1)
    int it = 0;
    if (grp > 0) {
      // resume where the screening kernel's checkpoint left the row: its fp32 walk up to
      // iteration 8 grp is this kernel's own (same evaluations, all outside the band)
      Lbest = __uint_as_float(rec.w);
      nl = (int)(rec.y & 0xFFFFu);
      bi = (int)(rec.y >> 16);
      bj = (int)rec.z;
      it = 8 * grp;
      nr = it - nl;
      iters = it;
      BLf = 15.f * (float)(nl + 1);
    } else {
      const float Wf = (float)p.b;                                                   // :174
      float a0;
      if constexpr (VEC)
        a0 = eval_one_x2<E>(ysl, 0.f, -Wf, kw_of(Wf), hh);
      else
        a0 = eval_one<E, true>(ys4, nv, 0.f, -Wf, kw_of(Wf), hh);
      Lbest = group_sum<LPR>(a0);
    }
    // Phase A: for it < it_exact_from every active row provably stays in the
    // loop (its float64 condition holds by >= 2 steps) and W >= 1, so the body
    // is straight-line: evaluate, reduce, decide.  An iteration that needs an
    // exact re-decision leaves the inner loop; the rare path runs outside it so
    // the hot loop's registers are not shaped by the calls it makes.
    const int itA = __any_sync(FULL, flags & F_EXACT_ONLY) ? 0 : min(p.it_exact_from, p.b - 1);
    while (it < itA) {
      bool need_ex = false, goL = false, chk = false;
      float SL = 0.f, SR = 0.f, cand = 0.f;
      for (; it < itA; ++it) {
        const float Wf = (float)(p.b - it - 1);
        float aL, aR;
        if constexpr (VEC) {
          if (Wf >= 17.f)   // codes move by at most one under the 15-shift
            eval_pair_x2_shift<E>(ysl, BLf, -Wf, kw_of(Wf), hh, aL, aR);
          else
            eval_pair_x2<E>(ysl, BLf, -Wf, kw_of(Wf), hh, aL, aR);
        } else {
          eval_pair<E, true>(ys4, nv, BLf, -Wf, kw_of(Wf), hh, aL, aR);
        }
        group_sum_pair<LPR>(aL, aR, SL, SR);
        goL = SL < SR;                                                   // clipping.py:185
        cand = goL ? SL : SR;
        const float mall = fmaxf(fmaxf(SL, SR), Lbest);
        const float band = p.tau2 * mall + p.c1 * sqrt_approx(mall) + (p.c0 + p.kmis * Wf * Wf);
        const float gap = fminf(fabsf(SL - SR), fabsf(cand - Lbest));
        need_ex = (flags & F_ACTIVE) && gap <= band;
        chk = (flags & F_ACTIVE) && !need_ex && gap <= __fmaf_rn(p.kmisx * Wf, Wf, band);
        if (__any_sync(FULL, need_ex || chk)) break;
        const bool upd = (flags & F_ACTIVE) != 0;
        const bool mvL = upd && goL;
        nl += mvL;
        nr += upd && !goL;
        BLf += mvL ? 15.f : 0.f;
        const bool better = upd && cand < Lbest;                         // clipping.py:187,191
        Lbest = better ? cand : Lbest;
        bi = better ? nl : bi;
        bj = better ? nr : bj;
        flags = better ? (flags & ~F_BEST_EX) : flags;
        iters += upd;
      }
      if (it >= itA) break;
      if (__any_sync(FULL, chk))
        need_ex |= near_escalate<LPR, E, VEC>(p, reinterpret_cast<const float*>(ys4), chk, q, gw, d, BLf,
                                              (float)(p.b - it - 1), bi, bj, wdiag);
      // iteration `it` has rows to re-decide exactly; the others apply the fast decision
      const bool upd = (flags & F_ACTIVE) && !need_ex;
      if (upd) {
        if (goL) { ++nl; BLf += 15.f; } else { ++nr; }
        if (cand < Lbest) { Lbest = cand; bi = nl; bj = nr; flags &= ~F_BEST_EX; }
        ++iters;
      }
      exact_block<LPR, E, VEC>(p, need_ex, q, gw, p.b - it - 1, SL, SR, rs, xr, d, e2, leaf_sum,
                               leaf_st, leaf_ln, nl, nr, bi, bj, iters, flags, Lbest, BLf, wdiag);
      ++it;
    }
    // Phase B: the remaining iterations, with the float64 loop condition
    // (clipping.py:180) and widths down to W <= 0 (exact decisions only).
    for (;; ++it) {
      if ((flags & F_ACTIVE) && (it >= p.it_exact_from || (flags & F_EXACT_ONLY))) {   // :180
        const double lhs = __dadd_rn(__dadd_rn(R.x0, __dmul_rn((double)nl, R.step)), R.min_steps);
        const double rhs = __dsub_rn(R.x1, __dmul_rn((double)nr, R.step));
        if (!(lhs < rhs)) flags &= ~F_ACTIVE;
      }
      if (!__any_sync(FULL, flags & F_ACTIVE)) break;
      const int W = p.b - it - 1;
      float SL = 0.f, SR = 0.f;
      bool need_ex = (flags & F_ACTIVE) != 0;
      if (W >= 1) {
        const float Wf = (float)W;
        float aL, aR;
        if constexpr (VEC)
          eval_pair_x2<E>(ysl, BLf, -Wf, kw_of(Wf), hh, aL, aR);
        else
          eval_pair<E, true>(ys4, nv, BLf, -Wf, kw_of(Wf), hh, aL, aR);
        group_sum_pair<LPR>(aL, aR, SL, SR);
        const bool goL = SL < SR;
        const float cand = goL ? SL : SR;
        const float mall = fmaxf(fmaxf(SL, SR), Lbest);
        const float band = p.tau2 * mall + p.c1 * sqrt_approx(mall) + (p.c0 + p.kmis * Wf * Wf);
        const float gap = fminf(fabsf(SL - SR), fabsf(cand - Lbest));
        need_ex = (flags & F_ACTIVE) && ((flags & F_EXACT_ONLY) || gap <= band);
        const bool chk = (flags & F_ACTIVE) && !need_ex && gap <= __fmaf_rn(p.kmisx * Wf, Wf, band);
        if (__any_sync(FULL, chk))
          need_ex |= near_escalate<LPR, E, VEC>(p, reinterpret_cast<const float*>(ys4), chk, q, gw, d, BLf,
                                                Wf, bi, bj, wdiag);
        if ((flags & F_ACTIVE) && !need_ex) {
          if (goL) { ++nl; BLf += 15.f; } else { ++nr; }
          if (cand < Lbest) {
            Lbest = cand; bi = nl; bj = nr;
            flags &= ~F_BEST_EX;
          }
          ++iters;
        }
      }
      if (__any_sync(FULL, need_ex))
        exact_block<LPR, E, VEC>(p, need_ex, q, gw, W, SL, SR, rs, xr, d, e2, leaf_sum, leaf_st,
                                 leaf_ln, nl, nr, bi, bj, iters, flags, Lbest, BLf, wdiag);
    }

    // ---- result, codes, pack ----
    double lo, hi;
    int info0 = -1, info1 = 0;
    if (flags & F_ERR) {
      lo = R.elo; hi = R.ehi; info0 = -2;
      if (q == 0 && p.status) atomicOr(p.status, EQ4_STATUS_RANGE);
    } else {
      // clipping.py:175,182: the start pair is (x0, x1) itself; any recorded
      // candidate's xmin is x0 + nl*step, which is +0.0 for nl = 0 and x0 = -0.0
      lo = (bi == 0 && bj == 0) ? R.x0 : __dadd_rn(R.x0, __dmul_rn((double)bi, R.step));
      hi = bj == 0 ? R.x1 : __dsub_rn(R.x1, __dmul_rn((double)bj, R.step));
      // (best_i << 16) | best_j; best_i alone when b > 65535 (it would not fit)
      if (rvalid && !bad && mn != mx) { info0 = iters; info1 = p.b > 65535 ? bi : ((bi << 16) | bj); }
    }
    const int blk_rows = (int)min((int64_t)RPW, nunits - row0);
    const size_t gofs = (size_t)row0 * p.stride;
    uint8_t* out_tile = p.list ? out_base : out_base + (((uintptr_t)p.packed + gofs) & 15);
    emit_greedy<LPR, E, VEC>(p, ysl, nv, q, lo, hi, bi, bj, mn != mx,
                             rvalid && !bad && !(flags & F_ERR), rvalid, xr,
                             out_tile + gw * p.stride, codes_w + gw * D, wdiag);
    if (rvalid && q == 0) {
      if (p.lo_out) { p.lo_out[row] = lo; p.hi_out[row] = hi; }
      if (p.info0) p.info0[row] = info0;
      if (p.info1) p.info1[row] = info1;
    }
    __syncwarp();
    if (!VEC) {
      const int nb = blk_rows * p.half;
      for (int t = lane; t < nb; t += 32) {
        const int rr = t / p.half, m = t - rr * p.half;
        const unsigned c0b = codes_w[rr * D + 2 * m];
        const unsigned c1b = (2 * m + 1 < d) ? codes_w[rr * D + 2 * m + 1] : 0u;  // packed.py:75-76
        out_tile[rr * p.stride + m] = (uint8_t)(c0b | (c1b << 4));
      }
      __syncwarp();
    }
    if (p.list) {   // scattered rows: each row's bytes to its own place
      for (int t = lane; t < blk_rows * p.stride; t += 32) {
        const int rr = t / p.stride;
        p.packed[(size_t)rs[rr].rid * p.stride + (t - rr * p.stride)] = out_tile[t];
      }
    } else {
      warp_copy_out(p.packed + gofs, out_tile, blk_rows * p.stride);
    }
    __syncwarp();
  }
  if (lane < 4 && wdiag[lane]) atomicAdd(&g_diag[lane], (unsigned long long)wdiag[lane]);
}

// ---------------------------------------------------------------------------
// GREEDY screening kernel (vector rows: d % 4 == 0, 16-byte aligned).
// The same fp32 walk as k_greedy's phase A/B -- Y slice in shared memory,
// packed pair evaluation, the error band on both sides of every comparison --
// but without the float64 tier: a row whose walk meets a comparison inside the
// band (after the near-boundary count of near_escalate), whose codes need the
// float64 codec, or that the fast walk does not take at all (non-finite values,
// a zero at its min or max -- numpy's signed-zero choice --, constant rows, rows
// the reference's grid rounds coarsely, W < 1) is DEFERRED: its index goes to
// p.dlist and k_greedy (list mode) redoes the whole row with the exact tier
// right after on the same stream.  About 2% of the rows of the bench tables
// are deferred.  Without the exact tier's calls, stack and float64 state the
// kernel fits 4 warps per SMSP (k_greedy: 3 at 168 registers).
// ---------------------------------------------------------------------------
struct RowFast {
  double x0, x1, step, min_steps;
};

template <int LPR, int E>
struct FastSlice {
  static constexpr int RPW = 32 / LPR;
  __host__ __device__ static size_t rf_off() { return (size_t)E * 32 * 4; }   // after the E/4 x 32 float4 slice
  __host__ __device__ static size_t out_off() { return (rf_off() + RPW * sizeof(RowFast) + 15) & ~(size_t)15; }
  __host__ __device__ static size_t diag_off(int stride) {
    return (out_off() + (size_t)RPW * stride + 32 + 15) & ~(size_t)15;
  }
  __host__ __device__ static size_t bytes(int stride) { return diag_off(stride) + 16; }
};

#ifdef EQ4_DBG
#define GF_CHECK(cond, tag, v)                                                                  \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("GF_CHECK %s failed: blk %d thr %d val %lld\n", tag, blockIdx.x, threadIdx.x, (long long)(v)); \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define GF_CHECK(cond, tag, v) do {} while (0)
#endif

#ifndef GF_MINB
#define GF_MINB 5
#endif
#ifndef GF_MINB_SMALL   // E <= 16 (d <= 16): 72 registers, 7 blocks of 4 warps per SM (d = 16: 4.58 ms at 5, 4.46 at 6, 4.42 at 7)
#define GF_MINB_SMALL 7
#endif

// k_greedy_fast's emit, rare path: the elements of one lane's slice that lie within nb of a
// rounding boundary of the winning pair take numpy's float64 codec; their nibbles are patched
// into the staged packed row (orow_q: the lane's first byte).
template <int LPR, int E>
__device__ __noinline__ void fast_emit_patch(const RowFast& R, int bi, int bj, const float* src, const float4* ysl,
                                             uint8_t* orow_q, float B, float kW, float hh, float nb) {
  const double lo = (bi == 0 && bj == 0) ? R.x0 : __dadd_rn(R.x0, __dmul_rn((double)bi, R.step));
  const double hi = bj == 0 ? R.x1 : __dsub_rn(R.x1, __dmul_rn((double)bj, R.step));
  const CodeParams cp = make_code_params(lo, hi);
  for (int c = 0; c < E / 4; ++c) {
    const float4 yv = ysl[c * 32];
    const float yk[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float sv = sat_fma(__fadd_rn(yk[k], -B), kW, hh);
      const float mm = __fadd_rn(__fmaf_rd(sv, ALPHA, MAGIC), -MAGIC);
      const float fr = __fmaf_rn(sv, ALPHA, -mm);
      if (sv > 0.f && sv < 1.f && fabsf(fr - 0.5f) > 0.5f - nb) {
        const unsigned cc = code_exact(src[4 * LPR * c + k], cp);
        uint8_t* by = orow_q + 2 * LPR * c + (k >> 1);
        const int sh = (k & 1) * 4;
        *by = (uint8_t)((*by & ~(0xF << sh)) | (cc << sh));
      }
    }
  }
}

template <int LPR, int E>
__global__ void __launch_bounds__(NTHREADS_G, E <= 16 ? GF_MINB_SMALL : (E <= 32 ? 5 : GF_MINB)) k_greedy_fast(const Params p) {
  using S = FastSlice<LPR, E>;
  constexpr int RPW = S::RPW;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = lane / LPR, q = lane % LPR;
  unsigned char* ws = smem + warp * S::bytes(p.stride);
  float4* ys4 = reinterpret_cast<float4*>(ws);
  const float4* ysl = ys4 + lane;
  RowFast* rf = reinterpret_cast<RowFast*>(ws + S::rf_off());
  uint8_t* out_base = ws + S::out_off();
  unsigned* wdiag = reinterpret_cast<unsigned*>(ws + S::diag_off(p.stride));
  if (lane < 4) wdiag[lane] = 0u;
  __syncwarp();
  const float hh = 0.5f / ALPHA;
  const int64_t nblocks = (p.rows + RPW - 1) / RPW;
  const int nwb = (int)(blockDim.x >> 5);
  const int64_t wstride = (int64_t)gridDim.x * nwb;
  unsigned ndefer = 0u;

  for (int64_t blk = (int64_t)blockIdx.x * nwb + warp; blk < nblocks; blk += wstride) {
    const int64_t row0 = blk * RPW, row = row0 + gw;
    const bool rvalid = row < p.rows;
    const float* xr = p.x + (row0 + (rvalid ? gw : 0)) * p.ld;
    bool defer, active;
    {
      const float4* src = reinterpret_cast<const float4*>(xr) + q;
      float lmn = INFINITY, lmx = -INFINITY;
      f2_t sm2 = pk2(0.f, 0.f);   // NaN / Inf detector: a packed running sum
#pragma unroll
      for (int c = 0; c < E / 4; ++c) {
        const float4 t = __ldg(src + LPR * c);
        lmn = fminf(lmn, fminf(fminf(t.x, t.y), fminf(t.z, t.w)));
        lmx = fmaxf(lmx, fmaxf(fmaxf(t.x, t.y), fmaxf(t.z, t.w)));
        sm2 = add2(sm2, add2(pk2(t.x, t.y), pk2(t.z, t.w)));
      }
      float s0, s1;
      upk2(sm2, s0, s1);
      const float mn = group_min<LPR>(lmn), mx = group_max<LPR>(lmx);
      const float sm = group_sum<LPR>(__fadd_rn(s0, s1));
      // rows the fp32 walk does not take (clipping.py:163-165 and the band's premises)
      const float M = fmaxf(fabsf(mn), fabsf(mx));
      defer = rvalid && (!isfinite(sm) || mn == 0.f || mx == 0.f || !(mn < mx) || !(M <= 1e6f * (mx - mn)));
      active = rvalid && !defer;
      const double x0 = (double)mn, x1 = (double)mx;
      const double step = __ddiv_rn(__dsub_rn(x1, x0), (double)p.b);                  // clipping.py:172
      const double kY = active ? __ddiv_rn(15.0, step) : 0.0;
      const double cY = 6755399441055744.0 * p.qY;   // Y + cY rounds Y to the qY grid
#pragma unroll 4
      for (int c = 0; c < E / 4; ++c) {
        const float4 t = __ldg(src + LPR * c);
        const float tv[4] = {t.x, t.y, t.z, t.w};
        float y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double Y = __dmul_rn(__dsub_rn((double)tv[k], x0), kY);
          y[k] = (float)__dsub_rn(__dadd_rn(Y, cY), cY);
        }
        ys4[c * 32 + lane] = make_float4(y[0], y[1], y[2], y[3]);
      }
      GF_CHECK(S::diag_off(p.stride) + 16 <= S::bytes(p.stride), "bytes", S::bytes(p.stride));
      GF_CHECK(row0 * p.ld + (int64_t)LPR * E <= p.rows * p.ld, "xread", row0);
      if (q == 0) {
        rf[gw].x0 = x0; rf[gw].x1 = x1; rf[gw].step = step;
        rf[gw].min_steps = __dmul_rn(__dmul_rn((double)p.b, __dsub_rn(1.0, p.r)), step);   // :173
      }
    }
    __syncwarp();
    // the next row block's rows towards L2 while this one is walked (its setup then waits on
    // L2, not HBM: -0.7% at 20M x 64, -2.3% at d = 16)
    {
      const int64_t nrow = row + wstride * RPW;
      if (nrow < p.rows) {
        const char* np = reinterpret_cast<const char*>(p.x + nrow * p.ld) + q * 128;
        for (int o = 0; o < E * 4 * LPR; o += 128 * LPR)
          asm volatile("prefetch.global.L2 [%0];" :: "l"(np + o));
      }
    }
    const float Wf0 = (float)p.b;                                                     // :174
    float Lbest = group_sum<LPR>(eval_one_x2<E>(ysl, 0.f, -Wf0, kw_of(Wf0), hh));
    int nl = 0, nr = 0, bi = 0, bj = 0;
    float BLf = 15.f;                      // base of the L candidate, 15 * (nl + 1)
    int it = 0;
    // the walk's state at the last checkpoint (iteration 8k) before a deferral: the exact kernel
    // resumes the row from there (resume records, Params::drec)
    int cp_it = 0, cp_nl = 0, cp_bi = 0, cp_bj = 0;
    float cp_L = 0.f;
    auto checkpoint = [&](int at) {
      if ((at & 7) == 0 && at > 0 && at < 8 * RG_GROUPS && !defer) {
        cp_it = at; cp_nl = nl; cp_bi = bi; cp_bj = bj; cp_L = Lbest;
      }
    };
    {
      // Phase A: iterations whose loop condition provably holds (it < it_exact_from) and
      // whose width takes the shift evaluation (W >= 17): straight-line body, no float64
      // test, no per-iteration vote but the near-boundary one.  kW of the next width and
      // the square-root term of the band come off the decision's critical path:
      // c1 sqrt(m) <= c1 (m / sqrt(S0) + sqrt(S0)) / 2 for any S0 > 0 (AM-GM), with S0 the
      // row's starting loss -- an upper bound, so the band stays sound (the losses of a walk
      // stay within a factor ~2 of it: a few % on that term; refreshing S0 every iteration
      // cost 2.3% at d = 16 and bought nothing measurable; a shared-memory table of
      // 1 / (alpha W) in place of kw_of measured no gain either).
      const int itA = max(0, min(p.it_exact_from, p.b - 17));
      const float c1h = 0.5f * p.c1;
      float kWn = kw_of((float)(p.b - 1));
      float sq = sqrt_approx(fmaxf(Lbest, 1e-30f));
      float rsq = rcp_approx(sq) * 1.000001f;   // any sq > 0 gives an upper bound; rcp.approx is within 1 ulp
      for (; it < itA;) {
      checkpoint(it);   // once per 8 iterations
      const int itE = min(itA, (it & ~7) + 8);
      for (; it < itE; ++it) {
        const float Wf = (float)(p.b - it - 1);
        const float kW = kWn;
        kWn = kw_of(Wf - 1.f);
        float aL, aR;
        eval_pair_x2_shift<E>(ysl, BLf, -Wf, kW, hh, aL, aR);
        float SL, SR;
        group_sum_pair<LPR>(aL, aR, SL, SR);
        const bool goL = SL < SR;                                                 // clipping.py:185
        const float cand = goL ? SL : SR;
        const float mall = fmaxf(fmaxf(SL, SR), Lbest);
        const float band = __fmaf_rn(p.tau2, mall, __fmaf_rn(c1h, __fmaf_rn(mall, rsq, sq),
                                                             __fmaf_rn(p.kmis * Wf, Wf, p.c0)));
        const float gap = fminf(fabsf(SL - SR), fabsf(cand - Lbest));
#ifdef G_NODECIDE   // development: timing without the band test
        bool need = false;
        const bool chk = false;
        (void)gap; (void)band;
#else
        bool need = active && gap <= band;
        const bool chk = active && !need && gap <= __fmaf_rn(p.kmisx * Wf, Wf, band);
#endif
        if (__any_sync(FULL, chk))
          need |= near_escalate<LPR, E, true>(p, reinterpret_cast<const float*>(ys4), chk, q, gw, p.d, BLf,
                                              Wf, bi, bj, wdiag);
        defer |= need;
        active = active && !need;
        const bool mv = active && goL;
        nl += mv;
        nr += active && !goL;
        BLf += mv ? 15.f : 0.f;
        const bool better = active && cand < Lbest;                               // clipping.py:187,191
        Lbest = better ? cand : Lbest;
        bi = better ? nl : bi;
        bj = better ? nr : bj;
      }
      }
    }
    for (;; ++it) {
      checkpoint(it);
      if (active && it >= p.it_exact_from) {   // clipping.py:180 in float64 (earlier: provably true)
        const RowFast& R = rf[gw];
        const double lhs = __dadd_rn(__dadd_rn(R.x0, __dmul_rn((double)nl, R.step)), R.min_steps);
        const double rhs = __dsub_rn(R.x1, __dmul_rn((double)nr, R.step));
        active = lhs < rhs;
      }
      if (!__any_sync(FULL, active)) break;
      const int W = p.b - it - 1;
      if (W < 1) {   // widths the fp32 grid cannot take: the exact kernel walks on
        defer |= active;
        break;
      }
      const float Wf = (float)W;
      float aL, aR;
      if (W >= 17)   // codes move by at most one under the 15-shift
        eval_pair_x2_shift<E>(ysl, BLf, -Wf, kw_of(Wf), hh, aL, aR);
      else
        eval_pair_x2<E>(ysl, BLf, -Wf, kw_of(Wf), hh, aL, aR);
      float SL, SR;
      group_sum_pair<LPR>(aL, aR, SL, SR);
      const bool goL = SL < SR;                                                   // clipping.py:185
      const float cand = goL ? SL : SR;
      const float mall = fmaxf(fmaxf(SL, SR), Lbest);
      const float band = p.tau2 * mall + p.c1 * sqrt_approx(mall) + (p.c0 + p.kmis * Wf * Wf);
      const float gap = fminf(fabsf(SL - SR), fabsf(cand - Lbest));
      bool need = active && gap <= band;
      const bool chk = active && !need && gap <= __fmaf_rn(p.kmisx * Wf, Wf, band);
      if (__any_sync(FULL, chk))
        need |= near_escalate<LPR, E, true>(p, reinterpret_cast<const float*>(ys4), chk, q, gw, p.d, BLf,
                                            Wf, bi, bj, wdiag);
      if (need) {
        defer = true;
        active = false;
      }
      if (active) {
        nl += goL;
        nr += !goL;
        BLf += goL ? 15.f : 0.f;
        if (cand < Lbest) {                                                       // clipping.py:187,191
          Lbest = cand;
          bi = nl;
          bj = nr;
        }
      }
    }

    // ---- result, codes, pack ----
    const size_t gofs = (size_t)row0 * p.stride;
    uint8_t* out_tile = out_base + (((uintptr_t)p.packed + gofs) & 15);
    uint8_t* orow = out_tile + gw * p.stride;
    const bool ok = rvalid && !defer;
    {
      const int Wb = p.b - bi - bj;
      const float B = (float)(15 * bi);
      const float Wbf = (float)(Wb > 0 ? Wb : 1);
      const float kW = __fdividef(1.f, Wbf * ALPHA);
      const float nb = NEAR + p.delta / Wbf;
      bool near = false;
      const f2_t nB2 = pk2(-B, -B), al2 = pk2(ALPHA, ALPHA);
      const f2_t mg2 = pk2(MAGIC, MAGIC), nmg2 = pk2(-MAGIC, -MAGIC);
#pragma unroll 4
      for (int c = 0; c < E / 4; ++c) {
        const ulonglong2 yy = *reinterpret_cast<const ulonglong2*>(ysl + c * 32);
        uint32_t w = 0;
#pragma unroll
        for (int hlf = 0; hlf < 2; ++hlf) {
          const f2_t z = add2(hlf ? yy.y : yy.x, nB2);
          float z0, z1;
          upk2(z, z0, z1);
          const float s0 = sat_fma(z0, kW, hh), s1 = sat_fma(z1, kW, hh);
          const f2_t sv = pk2(s0, s1);
          const f2_t m = fma2_rm(sv, al2, mg2);
          const f2_t fr = sub2(fma2(sv, al2, pk2(0.f, 0.f)), add2(m, nmg2));   // frac of alpha*s
          float m0, m1, f0, f1;
          upk2(m, m0, m1);
          upk2(fr, f0, f1);
          // an element within nb of a rounding boundary (strictly inside the clamp
          // range) may take another code in the reference: the float64 codec below
          near |= (s0 > 0.f && s0 < 1.f && fabsf(f0 - 0.5f) > 0.5f - nb) ||
                  (s1 > 0.f && s1 < 1.f && fabsf(f1 - 0.5f) > 0.5f - nb);
          w |= ((__float_as_uint(m0) & 0xFu) | ((__float_as_uint(m1) & 0xFu) << 4)) << (8 * hlf);
        }
        if (rvalid) *reinterpret_cast<uint16_t*>(orow + 2 * (q + LPR * c)) = (uint16_t)w;
      }
      // rare (a few % of the rows at d >= 2048): the lane's flagged elements take numpy's
      // float64 codec (uniform.py:77-79), patched into the staged nibbles (out of line)
      if (__any_sync(FULL, near && ok) && near && ok) {
        fast_emit_patch<LPR, E>(rf[gw], bi, bj, xr + 4 * q, ysl, orow + 2 * q, B, kW, hh, nb);
        atomicAdd(&wdiag[1], 1u);   // per lane with flagged elements
      }
    }
    if (rvalid && !defer && q == 0) {
      const RowFast& R = rf[gw];
      // clipping.py:175,182: x0 + bi*step (x0 itself for the start pair), x1 - bj*step
      const double lo = (bi == 0 && bj == 0) ? R.x0 : __dadd_rn(R.x0, __dmul_rn((double)bi, R.step));
      const double hi = bj == 0 ? R.x1 : __dsub_rn(R.x1, __dmul_rn((double)bj, R.step));
      const double sc = div15(__dsub_rn(hi, lo));                                  // uniform.py:74-80
      uint8_t* a = orow + p.half;
      if (p.aux == EQ4_AUX_FP16) {
        const uint32_t s16 = aux_bits_f16(sc), b16 = aux_bits_f16(lo);
        *reinterpret_cast<uint16_t*>(a) = (uint16_t)s16;
        *reinterpret_cast<uint16_t*>(a + 2) = (uint16_t)b16;
      } else {
        const uint32_t s32 = aux_bits_f32(sc), b32 = aux_bits_f32(lo);
        *reinterpret_cast<uint16_t*>(a) = (uint16_t)s32;
        *reinterpret_cast<uint16_t*>(a + 2) = (uint16_t)(s32 >> 16);
        *reinterpret_cast<uint16_t*>(a + 4) = (uint16_t)b32;
        *reinterpret_cast<uint16_t*>(a + 6) = (uint16_t)(b32 >> 16);
      }
      if (p.lo_out) { p.lo_out[row] = lo; p.hi_out[row] = hi; }
      if (p.info0) p.info0[row] = nl + nr;
      if (p.info1) p.info1[row] = p.b > 65535 ? bi : ((bi << 16) | bj);
    }
    // deferred rows (about 2% of the rows): a resume record when the walk passed a checkpoint,
    // else (or when the group is full) a slot of the restart list
    if (rvalid && defer && q == 0) {
      bool stored = false;
      if (p.drec && cp_it > 0) {
        const int k = cp_it >> 3;
        const int slot = atomicAdd(&p.drec_count[k], 1);
        if (slot < p.drec_cap) {
          p.drec[(size_t)k * p.drec_cap + slot] =
              make_uint4((unsigned)row, (unsigned)cp_nl | ((unsigned)cp_bi << 16), (unsigned)cp_bj,
                         __float_as_uint(cp_L));
          stored = true;
        }
      }
      if (!stored) {
        const unsigned slot = (unsigned)atomicAdd(p.dcount, 1);
        GF_CHECK(slot < p.rows, "dlist", slot);
        p.dlist[slot] = (uint32_t)row;
      }
      ++ndefer;
    }
    __syncwarp();
    GF_CHECK(gofs + (size_t)min((int64_t)RPW, p.rows - row0) * p.stride <= (size_t)p.rows * p.stride, "out", gofs);
    GF_CHECK(out_tile - out_base < 16, "tile", out_tile - out_base);
    warp_copy_out(p.packed + gofs, out_tile, (int)min((int64_t)RPW, p.rows - row0) * p.stride);
    __syncwarp();
  }
  if (lane < 4 && wdiag[lane]) atomicAdd(&g_diag[lane], (unsigned long long)wdiag[lane]);
  if (ndefer) atomicAdd(&g_diag[4], (unsigned long long)ndefer);
}

#include "eq4_gtable.cuh"

// ---------------------------------------------------------------------------
// ASYM vector kernel: warp-autonomous (per-warp staging, no block barriers),
// the next row block's loads in flight while the current one is coded, and
// the per-element code arithmetic on packed fp32x2.
// ---------------------------------------------------------------------------

template <int LPR, int E>
struct SliceA {
  static constexpr int RPW = 32 / LPR;
  __host__ __device__ static size_t bytes(int) { return 0; }
};

template <int LPR, int E>
__device__ __forceinline__ void asym_load(const float* rowp, bool ok, int q, float4 (&v)[E / 4]) {
  const float4* src = reinterpret_cast<const float4*>(rowp);
#pragma unroll
  for (int c = 0; c < E / 4; ++c)
    if (ok) v[c] = __ldcs(src + q + LPR * c);
}

// Code + pack one row slice (E elements of lane q) straight to the packed row
// in global memory (2-byte stores; L2 merges a row's partial sectors).
// The winning zero key (np_zero_key) over a whole row, by one lane (rare path of asym_row).
__device__ __noinline__ unsigned asym_zero_key_row(const float* rowp, int d) {
  unsigned kz = 0u;
  for (int i = 0; i < d; i += 4) {
    const float4 t = *reinterpret_cast<const float4*>(rowp + i);
    kz = max(max(max(kz, np_zero_key(t.x, i, d)), np_zero_key(t.y, i + 1, d)),
             max(np_zero_key(t.z, i + 2, d), np_zero_key(t.w, i + 3, d)));
  }
  return kz;
}

template <int LPR, int E, int RM>
__device__ __forceinline__ void asym_row(const Params& p, const float4 (&cur)[E / 4], int64_t row,
                                         int q) {
  const bool rvalid = row < p.rows;
  // ---- min / max / finiteness (clipping.py:58-61, table.py:28-29) ----
  float mn = INFINITY, mx = -INFINITY, sm = 0.f;
#pragma unroll
  for (int c = 0; c < E / 4; ++c) {
    mn = fminf(mn, fminf(fminf(cur[c].x, cur[c].y), fminf(cur[c].z, cur[c].w)));
    mx = fmaxf(mx, fmaxf(fmaxf(cur[c].x, cur[c].y), fmaxf(cur[c].z, cur[c].w)));
    sm = __fadd_rn(sm, __fadd_rn(__fadd_rn(cur[c].x, cur[c].y), __fadd_rn(cur[c].z, cur[c].w)));
  }
  mn = group_min<LPR>(mn);
  mx = group_max<LPR>(mx);
  sm = group_sum<LPR>(sm);
  bool bad = false;
  if (__any_sync(FULL, !isfinite(sm) && rvalid)) {
    bool lb = false;
#pragma unroll
    for (int c = 0; c < E / 4; ++c)
      lb |= !isfinite(cur[c].x) || !isfinite(cur[c].y) || !isfinite(cur[c].z) || !isfinite(cur[c].w);
    bad = group_any<LPR>(lb) && rvalid;
    if (bad && q == 0 && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
  }
  apply_range_mode<RM>(p, mn, mx);
  // ---- codes: u = (x - min) * 15/(max - min) + 1/2, code = floor(u) ----
  const float w32 = __fadd_rn(mx, -mn);
  const bool degenerate = !(mn != mx);                     // uniform.py:74-76: all codes 0
  const bool fast = !bad && w32 > 1e-30f && w32 < 1e30f;
  const float inv = fast ? __fdividef(15.f, w32) : 0.f;    // 0 -> u = 1/2 -> code 0
  const f2_t nmn2 = pk2(-mn, -mn), inv2 = pk2(inv, inv), h2 = pk2(0.5f, 0.5f);
  const f2_t mg2 = pk2(MAGIC, MAGIC), nmg2 = pk2(-MAGIC, -MAGIC);
  float gmin = 0.5f, gmax = 0.5f;
  uint8_t* orow = p.packed + (rvalid ? row : 0) * (int64_t)p.stride;
  uint32_t w16[E / 4];
#pragma unroll
  for (int c = 0; c < E / 4; ++c) {
    const f2_t xa = pk2(cur[c].x, cur[c].y), xb = pk2(cur[c].z, cur[c].w);
    const f2_t ua = fma2(add2(xa, nmn2), inv2, h2), ub = fma2(add2(xb, nmn2), inv2, h2);
    const f2_t ma = add2_rm(ua, mg2), mb = add2_rm(ub, mg2);            // 2^23 + floor(u)
    const f2_t ga = sub2(ua, add2(ma, nmg2)), gb = sub2(ub, add2(mb, nmg2));   // frac(u), exact
    float g0, g1, g2, g3;
    upk2(ga, g0, g1);
    upk2(gb, g2, g3);
    gmin = fminf(gmin, fminf(fminf(g0, g1), fminf(g2, g3)));
    gmax = fmaxf(gmax, fmaxf(fmaxf(g0, g1), fmaxf(g2, g3)));
    float m0, m1, m2, m3;
    upk2(ma, m0, m1);
    upk2(mb, m2, m3);
    // low nibbles of the four 2^23 + code bit patterns -> one 16-bit word
    w16[c] = __byte_perm(__float_as_uint(m0) | (__float_as_uint(m1) << 4),
                         __float_as_uint(m2) | (__float_as_uint(m3) << 4), 0x40) & 0xFFFFu;
  }
  const bool need = rvalid && !bad && !degenerate && (!fast || gmin < NEAR || gmax > 1.f - NEAR);
  if (__any_sync(FULL, need)) {   // rare: float64 codec (uniform.py:77-79) for flagged elements
    if (need) {
      const CodeParams cp = make_code_params((double)mn, (double)mx);
      for (int i = 0; i < E; ++i) {
        const float4 v4 = cur[i >> 2];
        const float x = (i & 3) == 0 ? v4.x : (i & 3) == 1 ? v4.y : (i & 3) == 2 ? v4.z : v4.w;
        const float u = __fmaf_rn(__fadd_rn(x, -mn), inv, 0.5f);
        const float g = __fadd_rn(u, -__fadd_rn(__fadd_rd(u, MAGIC), -MAGIC));
        if (fast && g >= NEAR && g <= 1.f - NEAR) continue;
        const uint32_t cc = code_exact(x, cp);
        const int sh = 4 * (i & 3);
        w16[i >> 2] = (w16[i >> 2] & ~(0xFu << sh)) | (cc << sh);
      }
    }
  }
  if (rvalid) {
#pragma unroll
    for (int c = 0; c < E / 4; ++c)
      *reinterpret_cast<uint16_t*>(orow + 2 * (q + LPR * c)) = (uint16_t)(bad ? 0u : w16[c]);
    if (q == 0) {
      // rare: numpy's signed-zero choice for a zero min / max (np_zero_key).  Only the stored
      // bias and the reported range carry the sign -- codes and scale do not -- so the row's
      // first lane settles it here, out of line and from global memory (inline in the main
      // path, with a warp vote, it cost 4% of the launch).  SYM / TABLE ranges do not use it.
      if constexpr (RM == 0) {
        if (mn == 0.f || mx == 0.f) np_zero_apply(asym_zero_key_row(p.x + row * p.ld, p.d), mn, mx);
      }
      const double sc = (!bad && !degenerate) ? div15(__dsub_rn((double)mx, (double)mn)) : 0.0;
      uint8_t* a = orow + p.half;
      if (p.aux == EQ4_AUX_FP16) {
        *reinterpret_cast<uint16_t*>(a) = (uint16_t)aux_bits_f16(sc);
        *reinterpret_cast<uint16_t*>(a + 2) = (uint16_t)aux_bits_f16((double)mn);
      } else {
        const uint32_t s32 = aux_bits_f32(sc), b32 = aux_bits_f32((double)mn);
        *reinterpret_cast<uint16_t*>(a) = (uint16_t)s32;
        *reinterpret_cast<uint16_t*>(a + 2) = (uint16_t)(s32 >> 16);
        *reinterpret_cast<uint16_t*>(a + 4) = (uint16_t)b32;
        *reinterpret_cast<uint16_t*>(a + 6) = (uint16_t)(b32 >> 16);
      }
      if (p.lo_out) { p.lo_out[row] = (double)mn; p.hi_out[row] = (double)mx; }
      if (p.info0) p.info0[row] = 0;
      if (p.info1) p.info1[row] = 0;
    }
  }
}

// ASYM vector kernel: warps are independent; each warp keeps the next row
// block's loads in flight (double buffer A/B) while it codes the current one.
template <int LPR, int E, int RM>
__global__ void __launch_bounds__(NTHREADS, 3) k_asym_vec(const Params p) {
  constexpr int RPW = 32 / LPR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = lane / LPR, q = lane % LPR;
  const int64_t nblocks = (p.rows + RPW - 1) / RPW;
  const int64_t wstride = (int64_t)gridDim.x * NWARPS;
  int64_t blk = (int64_t)blockIdx.x * NWARPS + warp;
  const int64_t rstep = wstride * RPW * p.ld;               // floats between a warp's blocks
  const float* xp = p.x + (blk * RPW + gw) * p.ld;
  float4 a[E / 4], b[E / 4];
  if (blk < nblocks) asym_load<LPR, E>(xp, blk * RPW + gw < p.rows, q, a);
  while (blk < nblocks) {
    if (blk + wstride < nblocks) asym_load<LPR, E>(xp + rstep, (blk + wstride) * RPW + gw < p.rows, q, b);
    asym_row<LPR, E, RM>(p, a, blk * RPW + gw, q);
    blk += wstride;
    xp += rstep;
    if (blk >= nblocks) break;
    if (blk + wstride < nblocks) asym_load<LPR, E>(xp + rstep, (blk + wstride) * RPW + gw < p.rows, q, a);
    asym_row<LPR, E, RM>(p, b, blk * RPW + gw, q);
    blk += wstride;
    xp += rstep;
  }
}

// ASYM-family kernel fed by the bulk-copy (TMA) engine: each warp owns a ring
// of ASTAGES shared-memory stages; lane 0 keeps the next ASTAGES-1 row blocks
// (RPW contiguous rows, <= 2 KB) in flight with cp.async.bulk + mbarrier
// transaction counts, so the bytes in flight per SM no longer depend on
// registers.  Rows must be contiguous (ld == d) and 16-byte aligned.
#ifndef ASTAGES
#define ASTAGES 4
#endif
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
               "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}"
      ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(parity) : "memory");
}

template <int LPR, int E>
struct SliceB {
  static constexpr int RPW = 32 / LPR;
  static constexpr int BLK = RPW * LPR * E * 4;                      // bytes per row block
  static constexpr int NST = (ASTAGES * 2048) / BLK;                // ~8 KB of stages per warp
  static constexpr size_t bytes() { return (size_t)NST * BLK + 128; }   // + barriers
};

template <int LPR, int E, int RM>
__global__ void __launch_bounds__(NTHREADS, 2) k_asym_bulk(const Params p) {
  using S = SliceB<LPR, E>;
  constexpr int RPW = S::RPW;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = lane / LPR, q = lane % LPR;
  unsigned char* ws = smem + (size_t)warp * S::bytes();
  uint64_t* bar = reinterpret_cast<uint64_t*>(ws + (size_t)S::NST * S::BLK);
  const int64_t nblocks = (p.rows + RPW - 1) / RPW;
  const int64_t wstride = (int64_t)gridDim.x * NWARPS;
  const int64_t blk0 = (int64_t)blockIdx.x * NWARPS + warp;
  const size_t row_bytes = (size_t)p.d * 4;
  if (lane == 0) {
    for (int st = 0; st < S::NST; st++) mbar_init(bar + st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int64_t blk, int st) {
    const int64_t r0 = blk * RPW;
    const unsigned nb = (unsigned)(min((int64_t)RPW, p.rows - r0) * row_bytes);
    mbar_expect_tx(bar + st, nb);
    bulk_g2s(ws + (size_t)st * S::BLK, p.x + r0 * p.d, nb, bar + st);
  };
  if (lane == 0)
    for (int st = 0; st < S::NST - 1; st++)
      if (blk0 + st * wstride < nblocks) issue(blk0 + st * wstride, st);
  int64_t it = 0;
  for (int64_t blk = blk0; blk < nblocks; blk += wstride, ++it) {
    const int st = (int)(it % S::NST);
    if (lane == 0) {   // keep S::NST - 1 blocks ahead in flight
      const int64_t ahead = blk + (int64_t)(S::NST - 1) * wstride;
      if (ahead < nblocks) issue(ahead, (int)((it + S::NST - 1) % S::NST));
    }
    mbar_wait(bar + st, (unsigned)((it / S::NST) & 1));
    const float4* rs = reinterpret_cast<const float4*>(ws + (size_t)st * S::BLK + (size_t)gw * row_bytes);
    float4 cur[E / 4];
#pragma unroll
    for (int c = 0; c < E / 4; ++c) cur[c] = rs[q + LPR * c];
    __syncwarp();   // the stage is refilled only after every lane has read it
    asym_row<LPR, E, RM>(p, cur, blk * RPW + gw, q);
  }
}

// ---------------------------------------------------------------------------
// ASYM family on wide rows (d > 2048): one warp per row, two streaming passes
// (min / max / finiteness, then codes; the second pass hits L1/L2), nibbles
// written straight to the packed row.  Bandwidth-class like k_asym; no
// E-sized register arrays, so any d.
// ---------------------------------------------------------------------------
template <int RM>
__global__ void __launch_bounds__(256) k_asym_wide(const Params p) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int d = p.d;
  const bool vec = (d % 4 == 0) && (p.ld % 4 == 0) && (((uintptr_t)p.x & 15) == 0);
  for (int64_t row = w0; row < p.rows; row += ws) {
    const float* xr = p.x + row * p.ld;
    float mn = INFINITY, mx = -INFINITY, sm = 0.f;
    if (vec) {
      const float4* x4 = reinterpret_cast<const float4*>(xr);
      for (int c = lane; c < d / 4; c += 32) {
        const float4 t = __ldcs(x4 + c);
        mn = fminf(mn, fminf(fminf(t.x, t.y), fminf(t.z, t.w)));
        mx = fmaxf(mx, fmaxf(fmaxf(t.x, t.y), fmaxf(t.z, t.w)));
        sm = __fadd_rn(sm, __fadd_rn(__fadd_rn(t.x, t.y), __fadd_rn(t.z, t.w)));
      }
    } else {
      for (int k = lane; k < d; k += 32) {
        const float t = __ldcs(xr + k);
        mn = fminf(mn, t);
        mx = fmaxf(mx, t);
        sm = __fadd_rn(sm, t);
      }
    }
    mn = group_min<32>(mn);
    mx = group_max<32>(mx);
    sm = group_sum<32>(sm);
    if (mn == 0.f || mx == 0.f) {   // rare: numpy's signed-zero choice
      unsigned kz = 0u;
      for (int k = lane; k < d; k += 32) kz = max(kz, np_zero_key(xr[k], k, d));
      np_zero_apply(__reduce_max_sync(FULL, kz), mn, mx);
    }
    bool bad = false;
    if (!isfinite(sm)) {
      bool lb = false;
      for (int k = lane; k < d; k += 32) lb |= !isfinite(xr[k]);
      bad = __any_sync(FULL, lb);
      if (bad && lane == 0 && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
    }
    apply_range_mode<RM>(p, mn, mx);
    const double lo = (double)mn, hi = (double)mx;          // clipping.py:51-67
    const CodeParams cp = make_code_params(bad ? 0.0 : lo, bad ? 0.0 : hi);
    uint8_t* orow = p.packed + row * (int64_t)p.stride;
    // codes (uniform.py:77-79) of element pairs -> packed bytes (packed.py:75-77)
    for (int m = lane; m < p.half; m += 32) {
      unsigned c0 = 0u, c1 = 0u;
      if (!bad) {
        bool n0, n1 = false;
        const float a = xr[2 * m];
        c0 = code_of(a, cp, n0);
        if (n0) c0 = code_exact(a, cp);
        if (2 * m + 1 < d) {
          const float bb = xr[2 * m + 1];
          c1 = code_of(bb, cp, n1);
          if (n1) c1 = code_exact(bb, cp);
        }
      }
      orow[m] = (uint8_t)(c0 | (c1 << 4));
    }
    if (lane == 0) {
      const double sc = (!bad && hi != lo) ? cp.scale : 0.0;   // uniform.py:74-80
      uint8_t* a = orow + p.half;
      if (p.aux == EQ4_AUX_FP16) {
        const uint32_t s16 = aux_bits_f16(sc), b16 = aux_bits_f16(lo);
        a[0] = s16 & 0xff; a[1] = s16 >> 8; a[2] = b16 & 0xff; a[3] = b16 >> 8;
      } else {
        const uint32_t s32 = aux_bits_f32(sc), b32 = aux_bits_f32(lo);
        for (int k = 0; k < 4; ++k) { a[k] = (s32 >> (8 * k)) & 0xff; a[4 + k] = (b32 >> (8 * k)) & 0xff; }
      }
      if (p.lo_out) { p.lo_out[row] = lo; p.hi_out[row] = hi; }
      if (p.info0) p.info0[row] = 0;
      if (p.info1) p.info1[row] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// pack / unpack / quant_mse utility kernels
// ---------------------------------------------------------------------------
__global__ void k_pack(const uint8_t* codes, int64_t rows, int d, int aux, const uint8_t* sc,
                       const uint8_t* bi, uint8_t* out, int stride) {
  const int half = (d + 1) / 2, ab = aux == EQ4_AUX_FP16 ? 2 : 4;
  int64_t n = rows * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / stride;
    int k = (int)(t - r * stride);
    uint8_t v;
    if (k < half) {
      unsigned c0 = codes[r * d + 2 * k] & 0xF;
      unsigned c1 = (2 * k + 1 < d) ? (codes[r * d + 2 * k + 1] & 0xF) : 0u;
      v = (uint8_t)(c0 | (c1 << 4));
    } else if (k < half + ab) {
      v = sc[r * ab + (k - half)];
    } else {
      v = bi[r * ab + (k - half - ab)];
    }
    out[t] = v;
  }
}

__global__ void k_unpack(const uint8_t* packed, int64_t rows, int d, int aux, uint8_t* codes,
                         uint8_t* sc, uint8_t* bi, int stride) {
  const int half = (d + 1) / 2, ab = aux == EQ4_AUX_FP16 ? 2 : 4;
  int64_t n = rows * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / stride;
    int k = (int)(t - r * stride);
    uint8_t v = packed[t];
    if (k < half) {
      codes[r * d + 2 * k] = v & 0xF;
      if (2 * k + 1 < d) codes[r * d + 2 * k + 1] = v >> 4;
    } else if (k < half + ab) {
      sc[r * ab + (k - half)] = v;
    } else {
      bi[r * ab + (k - half - ab)] = v;
    }
  }
}

// One warp per row: bit-exact quant_mse (table.py:81-103).
__global__ void __launch_bounds__(NTHREADS) k_quant_mse(const float* x, int64_t rows, int d,
                                                        int64_t ld, const double* lo,
                                                        const double* hi, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = (size_t)MAX_LEAVES * 16 + 512 * 8 + (((size_t)d * 4 + 15) & ~(size_t)15);
  unsigned char* ws = smem + warp * per_warp;
  double* leaf_sum = reinterpret_cast<double*>(ws);
  int* leaf_st = reinterpret_cast<int*>(leaf_sum + MAX_LEAVES);
  int* leaf_ln = leaf_st + MAX_LEAVES;
  double* e2 = reinterpret_cast<double*>(ws + MAX_LEAVES * 16);
  float* xs = reinterpret_cast<float*>(ws + MAX_LEAVES * 16 + 512 * 8);
  for (int64_t row = blockIdx.x * (int64_t)NWARPS + warp; row < rows;
       row += (int64_t)gridDim.x * NWARPS) {
    for (int k = lane; k < d; k += 32) xs[k] = x[row * ld + k];
    __syncwarp();
    double v = warp_np_loss(xs, d, lo[row], hi[row], e2, leaf_sum, leaf_st, leaf_ln, MAX_LEAVES);
    if (lane == 0) out[row] = v;
    __syncwarp();
  }
}

// Self-test kernel: div15 (Markstein) against the IEEE divide on n values.
// which = 0: w = |f1 - f0| of random floats (the values div15 sees);
// which = 1: random doubles over the whole normal exponent range.
__global__ void k_selftest_div15(int which, int64_t n, uint64_t seed, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    double w;
    if (which == 0) {
      float a = __uint_as_float((uint32_t)z & 0xBFFFFFFFu);   // finite floats, both signs
      float b = __uint_as_float((uint32_t)(z >> 32) & 0xBFFFFFFFu);
      w = fabs((double)a - (double)b);
    } else {
      w = __longlong_as_double((long long)((z & 0x000FFFFFFFFFFFFFull) |
                                           ((uint64_t)(1 + (z >> 52) % 2045) << 52)));
    }
    if (__double_as_longlong(div15(w)) != __double_as_longlong(__ddiv_rn(w, 15.0))) local++;
  }
  if (local) atomicAdd(bad, local);
}

}  // namespace eq4

// ===========================================================================
// Host side
// ===========================================================================
using namespace eq4;

static thread_local std::string g_err;

// Python's repr(float) (shortest round-trip digits; fixed notation for decimal
// exponents -4..15 with at least one fractional digit, else d.ddde+XX), so the
// C ABI's messages carry the reference's exact ValueError texts (table.py:73-74
// formats the floats with str()).
std::string py_float_repr(double v) {
  if (v != v) return "nan";
  if (v == INFINITY) return "inf";
  if (v == -INFINITY) return "-inf";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
    if (strtod(buf, nullptr) == v) break;
  }
  // buf = [-]d.ddde[+-]XX with prec significant digits
  std::string m(buf);
  const size_t epos = m.find('e');
  const int exp10 = atoi(m.c_str() + epos + 1);
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (m[i] >= '0' && m[i] <= '9') digits += m[i];
  const bool neg = v < 0 || (v == 0 && std::signbit(v));
  std::string out = neg ? "-" : "";
  if (exp10 >= -4 && exp10 < 16) {
    if (exp10 < 0) {
      out += "0." + std::string(-exp10 - 1, '0') + digits;
    } else {
      if ((int)digits.size() <= exp10 + 1) {
        out += digits + std::string(exp10 + 1 - digits.size(), '0') + ".0";
      } else {
        out += digits.substr(0, exp10 + 1) + "." + digits.substr(exp10 + 1);
      }
    }
  } else {
    out += digits.substr(0, 1);
    if (digits.size() > 1) out += "." + digits.substr(1);
    char e[16];
    snprintf(e, sizeof e, "e%c%02d", exp10 < 0 ? '-' : '+', exp10 < 0 ? -exp10 : exp10);
    out += e;
  }
  return out;
}
static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
static int cuda_fail(cudaError_t e, const char* where) {
  return fail(EQ4_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

static int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

template <typename Kern>
static int launch_persistent(Kern kern, size_t smem, int64_t ntiles, const Params& p, cudaStream_t s,
                             const char* name, int nthreads = NTHREADS) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  }
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nthreads, smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy");
  if (occ < 1) occ = 1;
  int64_t grid = std::min<int64_t>(ntiles, (int64_t)sm_count() * occ);
  kern<<<(unsigned)grid, nthreads, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, name);
  return EQ4_OK;
}

// The device's default memory pool keeps what it has (stream-ordered scratch of
// the GREEDY deferral list is then recycled, not remapped, call after call).
static void keep_pool_memory() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

// GREEDY on vector rows: k_greedy_fast screens every row, then k_greedy (list mode)
// redoes the deferred ones with the exact tier.  Both on stream s, no host sync;
// the deferral list (4 bytes per row) is stream-ordered scratch.
// Rows the table walk takes (eq4_gtable.cuh): wide vector rows whose table fits a warp's
// share of shared memory and whose integer sums fit 64 bits (d * 15 b < 2^27).
static bool table_walk_applies(const Params& p) {
  // measured crossover against the per-element screen on 1 GiB N(0,1) tables (K2)
  int min_d = 2048;
  if (const char* ev = getenv("EQ4_DEV_TABLE_MIN_D")) min_d = atoi(ev);   // development A/B only
  return p.d >= min_d && p.d <= 16384 && p.b <= 400 && (int64_t)p.d * 15 * p.b < ((int64_t)1 << 27) &&
         p.rows < ((int64_t)1 << 32);
}

template <int LPR, int E>
static int greedy_two_pass(Params p, cudaStream_t s, int nw_exact) {
  keep_pool_memory();
  using F = FastSlice<LPR, E>;
  using S = WarpSliceG<LPR, E, true>;
  const int64_t chunk = (int64_t)1 << 30;   // list entries are 32-bit row offsets
  uint32_t* buf = nullptr;
  const int64_t cap = std::min<int64_t>(p.rows, chunk);
  // restart list (4 B per row) + resume records (16 B, groups 1..RG_GROUPS-1, b <= 65535)
  const bool resume = p.b <= 65535 && !getenv("EQ4_DEV_NO_RESUME");   // (env: development A/B only)
  int64_t rcap = resume ? std::min<int64_t>(cap, (int64_t)1 << 18) : 0;
  if (const char* ev = getenv("EQ4_DEV_RCAP")) rcap = resume ? std::min<int64_t>(rcap, atoll(ev)) : 0;   // tests: overflow
  const size_t list_bytes = ((size_t)(cap + 4) * 4 + 255) & ~(size_t)255;
  const size_t rec_bytes = (size_t)rcap * RG_GROUPS * 16;
  cudaError_t e = cudaMallocAsync((void**)&buf, list_bytes + rec_bytes + 64, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  int* rcount = reinterpret_cast<int*>(reinterpret_cast<char*>(buf) + list_bytes + rec_bytes);
  uint4* recs = resume ? reinterpret_cast<uint4*>(reinterpret_cast<char*>(buf) + list_bytes) : nullptr;
  // warps per block: as many as pack the most resident warps per SM (wide rows: 17-33 KB slices)
  int nwf = NWARPS_G;
  {
    int best = 0;
    for (int w = NWARPS_G; w >= 1; w >>= 1) {
      const int per_sm = (int)((227 * 1024) / ((size_t)w * F::bytes(p.stride))) * w;
      if (per_sm > best) { best = per_sm; nwf = w; }
    }
  }
  int rc = EQ4_OK;
  const int64_t rows = p.rows;
  for (int64_t r0 = 0; r0 < rows && rc == EQ4_OK; r0 += chunk) {
    Params c = p;
    c.rows = std::min<int64_t>(chunk, rows - r0);
    c.x = p.x + r0 * p.ld;
    c.packed = p.packed + r0 * p.stride;
    if (p.lo_out) { c.lo_out = p.lo_out + r0; c.hi_out = p.hi_out + r0; }
    if (p.info0) c.info0 = p.info0 + r0;
    if (p.info1) c.info1 = p.info1 + r0;
    c.dcount = reinterpret_cast<int*>(buf);
    c.dlist = buf + 4;
    c.drec = recs;
    c.drec_count = rcount;
    c.drec_cap = (int)rcap;
    e = cudaMemsetAsync(c.dcount, 0, 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(rcount, 0, RG_GROUPS * sizeof(int), s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "cudaMemsetAsync"); break; }
    c.list = 0;
    if (table_walk_applies(p)) {
      // one block per row, the table in its shared memory (4 blocks per SM at b = 200)
      // 128 threads per row (256 measured slower at every d: 3 blocks per SM)
      c.tb_wave = sm_count();
      c.tb_defer_at = -1;
      if (const char* ev = getenv("EQ4_DEV_TABLE_DEFER_AT")) c.tb_defer_at = atoi(ev);   // tests: resume records
      rc = launch_persistent(k_greedy_table<128>, TableSlice::bytes(p.b, 128), c.rows, c, s, "k_greedy_table", 128);
    } else {
      rc = launch_persistent(k_greedy_fast<LPR, E>, nwf * F::bytes(p.stride),
                             (c.rows + F::RPW * nwf - 1) / (F::RPW * nwf), c, s, "k_greedy_fast", 32 * nwf);
    }
    if (rc != EQ4_OK) break;
    if (getenv("EQ4_DEV_SKIP_EXACT")) continue;   // development only
    c.list = 1;
    // wide rows: as few warps per block as packs the most resident warps per SM (the
    // per-warp slices of k_greedy are 20-43 KB at E >= 128)
    int nwe = nw_exact, best = 0;
    for (int w = nw_exact; w >= 1; w >>= 1) {
      const int per_sm = (int)((227 * 1024) / ((size_t)w * S::bytes(p.stride))) * w;
      if (per_sm > best) { best = per_sm; nwe = w; }
    }
    nw_exact = nwe;
    rc = launch_persistent(k_greedy<LPR, E, true>, nw_exact * S::bytes(p.stride),
                           (c.rows + S::RPW * nw_exact - 1) / (S::RPW * nw_exact), c, s, "k_greedy", 32 * nw_exact);
  }
  cudaFreeAsync(buf, s);
  return rc;
}

template <int METHOD, int LPR, int E, bool VEC>
static int launch_rq(const Params& p, cudaStream_t s) {
  if constexpr (METHOD == M_ASYM) {
    if constexpr (VEC && E <= 16) {
      // contiguous rows of >= 32 floats: bulk-copy ring (d = 16 rows make 1 KB blocks,
      // where the register double buffer measured faster)
      if (LPR * E >= 32 && p.ld == p.d) {
        using B = SliceB<LPR, E>;
        const int64_t nt = (p.rows + B::RPW * NWARPS - 1) / (B::RPW * NWARPS);
        const size_t sm = NWARPS * B::bytes();
        if (p.range_mode == 1) return launch_persistent(k_asym_bulk<LPR, E, 1>, sm, nt, p, s, "k_asym_bulk");
        if (p.range_mode == 2) return launch_persistent(k_asym_bulk<LPR, E, 2>, sm, nt, p, s, "k_asym_bulk");
        return launch_persistent(k_asym_bulk<LPR, E, 0>, sm, nt, p, s, "k_asym_bulk");
      }
      using S = SliceA<LPR, E>;
      const int64_t nt = (p.rows + S::RPW * NWARPS - 1) / (S::RPW * NWARPS);
      if (p.range_mode == 1) return launch_persistent(k_asym_vec<LPR, E, 1>, 0, nt, p, s, "k_asym_vec");
      if (p.range_mode == 2) return launch_persistent(k_asym_vec<LPR, E, 2>, 0, nt, p, s, "k_asym_vec");
      return launch_persistent(k_asym_vec<LPR, E, 0>, 0, nt, p, s, "k_asym_vec");
    }
    using L = LayoutA<LPR, E, VEC>;
    const int64_t nt = (p.rows + L::RPB - 1) / L::RPB;
    if (p.range_mode == 1) return launch_persistent(k_asym<LPR, E, VEC, 1>, L::total(p.stride), nt, p, s, "k_asym");
    if (p.range_mode == 2) return launch_persistent(k_asym<LPR, E, VEC, 2>, L::total(p.stride), nt, p, s, "k_asym");
    return launch_persistent(k_asym<LPR, E, VEC, 0>, L::total(p.stride), nt, p, s, "k_asym");
  } else {
    using S = WarpSliceG<LPR, E, VEC>;
    // wide rows: as many warps per block as the per-warp slices fit in shared memory
    int nw = NWARPS_G;
    while (nw > 1 && (size_t)nw * S::bytes(p.stride) > 220 * 1024) nw >>= 1;
    if (S::bytes(p.stride) > 220 * 1024) return fail(EQ4_EUNSUPPORTED, "GREEDY row does not fit in shared memory");
    if constexpr (VEC) {
      if (!getenv("EQ4_DEV_ONE_PASS")) return greedy_two_pass<LPR, E>(p, s, nw);   // (env: development A/B only)
    }
    return launch_persistent(k_greedy<LPR, E, VEC>, nw * S::bytes(p.stride),
                             (p.rows + S::RPW * nw - 1) / (S::RPW * nw), p, s, "k_greedy", 32 * nw);
  }
}

template <int METHOD>
static int dispatch_rq(const Params& p, bool vec, cudaStream_t s) {
  const int d = p.d;
  if constexpr (METHOD == M_ASYM) {
    if (vec) {
      switch (d) {
        case 16: return launch_rq<METHOD, 2, 8, true>(p, s);
        case 32: return launch_rq<METHOD, 2, 16, true>(p, s);
        case 64: return launch_rq<METHOD, 4, 16, true>(p, s);
        case 128: return launch_rq<METHOD, 8, 16, true>(p, s);
        case 256: return launch_rq<METHOD, 16, 16, true>(p, s);
        case 512: return launch_rq<METHOD, 32, 16, true>(p, s);
        case 1024: return launch_rq<METHOD, 32, 32, true>(p, s);
        case 2048: return launch_rq<METHOD, 32, 64, true>(p, s);
        default: break;
      }
    }
    if (d <= 8) return launch_rq<METHOD, 1, 8, false>(p, s);
    if (d <= 16) return launch_rq<METHOD, 1, 16, false>(p, s);
    if (d <= 32) return launch_rq<METHOD, 2, 16, false>(p, s);
    if (d <= 64) return launch_rq<METHOD, 4, 16, false>(p, s);
    if (d <= 128) return launch_rq<METHOD, 8, 16, false>(p, s);
    if (d <= 256) return launch_rq<METHOD, 16, 16, false>(p, s);
    if (d <= 512) return launch_rq<METHOD, 32, 16, false>(p, s);
    if (d <= 1024) return launch_rq<METHOD, 32, 32, false>(p, s);
    if (d <= 2048) return launch_rq<METHOD, 32, 64, false>(p, s);
    // wide rows: warp per row, two streaming passes
    const int64_t nt = (p.rows + 7) / 8;
    if (p.range_mode == 1) return launch_persistent(k_asym_wide<1>, 0, nt, p, s, "k_asym_wide");
    if (p.range_mode == 2) return launch_persistent(k_asym_wide<2>, 0, nt, p, s, "k_asym_wide");
    return launch_persistent(k_asym_wide<0>, 0, nt, p, s, "k_asym_wide");
  } else {
  // GREEDY: 64 elements per lane amortise the per-iteration decision work best
  // (measured on 20M x 64 and the 1 GiB d-sweep against 32 per lane; the row
  // slice lives in shared memory)
  if (vec) {
    switch (d) {
      case 16: return launch_rq<METHOD, 1, 16, true>(p, s);
      case 32: return launch_rq<METHOD, 1, 32, true>(p, s);
      case 64: return launch_rq<METHOD, 1, 64, true>(p, s);
      case 128: return launch_rq<METHOD, 2, 64, true>(p, s);
      case 256: return launch_rq<METHOD, 4, 64, true>(p, s);
      case 512: return launch_rq<METHOD, 8, 64, true>(p, s);
      case 1024: return launch_rq<METHOD, 16, 64, true>(p, s);
      case 2048: return launch_rq<METHOD, 32, 64, true>(p, s);
      case 4096: return launch_rq<METHOD, 32, 128, true>(p, s);
      case 8192: return launch_rq<METHOD, 32, 256, true>(p, s);
      case 16384: return launch_rq<METHOD, 32, 512, true>(p, s);
      default: break;
    }
  }
  if (d <= 8) return launch_rq<METHOD, 1, 8, false>(p, s);
  if (d <= 16) return launch_rq<METHOD, 1, 16, false>(p, s);
  if (d <= 32) return launch_rq<METHOD, 1, 32, false>(p, s);
  if (d <= 64) return launch_rq<METHOD, 1, 64, false>(p, s);
  if (d <= 128) return launch_rq<METHOD, 2, 64, false>(p, s);
  if (d <= 256) return launch_rq<METHOD, 4, 64, false>(p, s);
  if (d <= 512) return launch_rq<METHOD, 8, 64, false>(p, s);
  if (d <= 1024) return launch_rq<METHOD, 16, 64, false>(p, s);
  if (d <= 2048) return launch_rq<METHOD, 32, 64, false>(p, s);
  // wide rows: one warp per row, 128..512 elements per lane (row slice in shared memory)
  if (d <= 4096) return launch_rq<METHOD, 32, 128, false>(p, s);
  if (d <= 8192) return launch_rq<METHOD, 32, 256, false>(p, s);
  if (d <= 16384) return launch_rq<METHOD, 32, 512, false>(p, s);
  return fail(EQ4_EUNSUPPORTED, "GREEDY with dim > 16384 is not supported by the B200 path");
  }
}

// GREEDY error-band constants.  The fp32 loss of one
// candidate is a sum of exactly computed squares (each squared and added by one
// FMA), so its error is <= gamma_h * S with h the most roundings any term passes
// through: the packed kernels (d a power of two, 16-byte rows) accumulate E/2
// terms per f32x2 half, add the halves and reduce LPR lanes (E/2 + 1 + log2 LPR);
// the masked kernels run one chain of up to E terms per lane (E + log2 LPR).
// (LPR, E) must follow dispatch_rq's GREEDY table.  Both sides -> x2; one extra
// rounding and 5% margin.
static float tau2_for(int d, bool vec) {
  int lpr, e;
  if (d <= 8) { lpr = 1; e = 8; }
  else if (d <= 16) { lpr = 1; e = 16; }
  else if (d <= 32) { lpr = 1; e = 32; }
  else if (d <= 2048) { lpr = 1; while (lpr * 64 < d) lpr *= 2; e = 64; }
  else { lpr = 32; e = d <= 4096 ? 128 : (d <= 8192 ? 256 : 512); }
  const bool packed = vec && (d == 16 || d == 32 || d == 64 || d == 128 || d == 256 || d == 512 ||
                              d == 1024 || d == 2048 || d == 4096 || d == 8192 || d == 16384);
  int lg = 0;
  while ((1 << lg) < lpr) lg++;
  // packed: chains of e / (2 nacc) terms, log2(nacc) tree levels, the two halves added
  const int na = nacc_for(e);
  const int lna = na == 4 ? 2 : (na == 2 ? 1 : 0);
  const int h = (packed ? e / 2 / na + lna + 1 : e) + lg + 1;
  return (float)(2.0 * 1.05 * h * 5.9604645e-8);
}

// Streams, chunk buffers and the pinned status words of the host pipeline are kept
// per device and reused by later calls (grow-only): creating / freeing them per call
// (stream create/destroy, cudaMallocHost/cudaFreeHost, pool allocations released at
// every synchronisation) cost 0.1-0.5 s on some calls.  Calls on one device are
// serialised by the context's mutex.
namespace {
constexpr int HP_NS = 3;   // chunk c's H2D overlaps chunk c-1's kernel and chunk c-2's D2H
struct HostBuf {
  float* x = nullptr; uint8_t* out = nullptr; double* lo = nullptr; double* hi = nullptr;
  int32_t* i0 = nullptr; int32_t* i1 = nullptr; int32_t* status = nullptr; double* nrm = nullptr;
};
struct HostPipe {
  std::mutex mu;
  bool init = false;
  cudaStream_t st[HP_NS] = {};
  HostBuf bf[HP_NS];
  size_t x_bytes = 0, out_bytes = 0, i0_rows = 0, i1_rows = 0, lohi_rows = 0, nrm_rows = 0;   // capacities
  int32_t* hstatus = nullptr;
  int64_t hstatus_n = 0;
};
HostPipe g_pipes[64];

template <class T>
cudaError_t grow(T** p, size_t have, size_t want) {
  if (*p && have >= want) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  return cudaMalloc((void**)p, want);
}

// capacity for chunks of `chunk` rows (grow-only); returns a cudaError_t
cudaError_t pipe_reserve(HostPipe& hp, int64_t chunk, int64_t dim, int64_t stride, bool want_i1,
                         bool want_lohi, bool want_norm, int64_t nchunks) {
  cudaError_t e = cudaSuccess;
  if (!hp.init) {
    for (int i = 0; i < HP_NS && e == cudaSuccess; i++)
      e = cudaStreamCreateWithFlags(&hp.st[i], cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
    hp.init = true;
  }
  const size_t xb = (size_t)chunk * dim * 4, ob = (size_t)chunk * stride, rows = (size_t)chunk;
  for (int i = 0; i < HP_NS && e == cudaSuccess; i++) {
    HostBuf& B = hp.bf[i];
    e = grow(&B.x, hp.x_bytes, xb);
    if (e == cudaSuccess) e = grow(&B.out, hp.out_bytes, ob);
    if (e == cudaSuccess) e = grow(&B.i0, hp.i0_rows * 4, rows * 4);
    if (e == cudaSuccess && !B.status) e = cudaMalloc((void**)&B.status, 4);
    if (e == cudaSuccess && want_i1) e = grow(&B.i1, hp.i1_rows * 4, rows * 4);
    if (e == cudaSuccess && want_lohi) e = grow(&B.lo, hp.lohi_rows * 8, rows * 8);
    if (e == cudaSuccess && want_lohi) e = grow(&B.hi, hp.lohi_rows * 8, rows * 8);
    if (e == cudaSuccess && want_norm) e = grow(&B.nrm, hp.nrm_rows * 8, rows * 8);
  }
  if (e != cudaSuccess) {   // partially grown: forget every capacity, the next call reallocates
    hp.x_bytes = hp.out_bytes = hp.i0_rows = hp.i1_rows = hp.lohi_rows = hp.nrm_rows = 0;
    return e;
  }
  hp.x_bytes = std::max(hp.x_bytes, xb);
  hp.out_bytes = std::max(hp.out_bytes, ob);
  hp.i0_rows = std::max(hp.i0_rows, rows);
  if (want_i1) hp.i1_rows = std::max(hp.i1_rows, rows);
  if (want_lohi) hp.lohi_rows = std::max(hp.lohi_rows, rows);
  if (want_norm) hp.nrm_rows = std::max(hp.nrm_rows, rows);
  if (hp.hstatus_n < nchunks) {
    if (hp.hstatus) cudaFreeHost(hp.hstatus);
    hp.hstatus = nullptr;
    hp.hstatus_n = 0;
    e = cudaMallocHost((void**)&hp.hstatus, sizeof(int32_t) * nchunks);
    if (e != cudaSuccess) return e;
    hp.hstatus_n = nchunks;
  }
  return cudaSuccess;
}
}  // namespace

extern "C" {

const char* eq4_version(void) { return "eq4 0.1.0 (sm_100a)"; }

const char* eq4_last_error(void) { return g_err.c_str(); }

int64_t eq4_kmeans_row_stride(int64_t dim, int aux) {
  return 16 * (aux == EQ4_AUX_FP16 ? 2 : 4) + (dim + 1) / 2;
}

int eq4_kmeans_rows(const float* x, int64_t rows, int64_t dim, int64_t ld, int aux, uint8_t* out,
                    int32_t* iters, int32_t* status, void* stream) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "table must be at least 1x1");
  if (ld < dim) return fail(EQ4_EINVAL, "ld must be >= dim");
  if (!x || !out) return fail(EQ4_EINVAL, "null buffer");
  if (aux != EQ4_AUX_FP16 && aux != EQ4_AUX_FP32) return fail(EQ4_EINVAL, "aux must be fp32 or fp16");
  std::string err;
  const int rc = eq4_kmeans_launch(x, rows, dim, ld, aux, out, iters, status, (cudaStream_t)stream, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

int eq4_quantize_file(const char* in_path, const char* out_path, int method, int b, double r,
                      int aux, int64_t chunk_rows, int64_t* bad_row, double* bad_lohi) {
  if (!in_path || !out_path) return fail(EQ4_EINVAL, "null path");
  if (aux != EQ4_AUX_FP16 && aux != EQ4_AUX_FP32) return fail(EQ4_EINVAL, "aux must be fp32 or fp16");
  if (method < EQ4_METHOD_ASYM || method > EQ4_METHOD_HIST_APPRX)
    return fail(EQ4_EINVAL, "unknown method " + std::to_string(method));
  std::string err;
  const int rc = eq4_io_quantize_file(in_path, out_path, method, b, r, aux, chunk_rows, bad_row,
                                      bad_lohi, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

int eq4_write_embq(const char* path, const uint8_t* packed, int64_t rows, int64_t dim, int aux,
                   int on_device) {
  if (!path || !packed) return fail(EQ4_EINVAL, "null buffer");
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "packed table must be at least 1x1");
  if (aux != EQ4_AUX_FP16 && aux != EQ4_AUX_FP32) return fail(EQ4_EINVAL, "aux must be fp32 or fp16");
  std::string err;
  const int rc = eq4_io_write_embq(path, packed, rows, dim, aux, on_device, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

int eq4_sparse_lengths_sum4(const uint8_t* packed, int64_t rows, int64_t dim, int aux,
                            const int64_t* indices, int64_t nidx, const int64_t* lengths,
                            int64_t batch, float* out, int32_t* status, int64_t* bad_pos,
                            void* stream) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "packed table must be at least 1x1");
  if (batch < 0 || nidx < 0) return fail(EQ4_EINVAL, "batch and nidx must be non-negative");
  if (aux != EQ4_AUX_FP16 && aux != EQ4_AUX_FP32) return fail(EQ4_EINVAL, "aux must be fp32 or fp16");
  if (!packed || (batch > 0 && (!lengths || !out)) || (nidx > 0 && !indices))
    return fail(EQ4_EINVAL, "null buffer");
  std::string err;
  const int rc = eq4_sls_launch(packed, rows, dim, aux, indices, nidx, lengths, batch, out, status,
                                bad_pos, (cudaStream_t)stream, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

int64_t eq4_packed_row_stride(int64_t dim, int aux) {
  return (dim + 1) / 2 + 2 * (aux == EQ4_AUX_FP16 ? 2 : 4);
}

static int quantize_pack_impl(const float* x, int64_t rows, int64_t dim, int64_t ld, int method,
                              int b, double r, int aux, uint8_t* packed, double* xmin, double* xmax,
                              int32_t* info0, int32_t* info1, double* norm, int32_t* status,
                              void* stream, const int* table_keys, double param = 0.0);

int eq4_quantize_pack(const float* x, int64_t rows, int64_t dim, int64_t ld, int method, int b,
                      double r, int aux, uint8_t* packed, double* xmin, double* xmax,
                      int32_t* info0, int32_t* info1, double* norm, int32_t* status,
                      void* stream) {
  return eq4_quantize_pack_p(x, rows, dim, ld, method, b, r, 0.0, aux, packed, xmin, xmax, info0, info1,
                             norm, status, stream);
}

int eq4_quantize_pack_p(const float* x, int64_t rows, int64_t dim, int64_t ld, int method, int b,
                        double r, double param, int aux, uint8_t* packed, double* xmin, double* xmax,
                        int32_t* info0, int32_t* info1, double* norm, int32_t* status, void* stream) {
  if (!(param >= 0.0) || !std::isfinite(param))
    return fail(EQ4_EINVAL, "param must be finite and >= 0 (0 = the reference default)");
  // the status word describes this call: cleared on the stream before the kernels OR into it
  if (status) {
    const cudaError_t e = cudaMemsetAsync(status, 0, 4, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "status reset");
  }
  return quantize_pack_impl(x, rows, dim, ld, method, b, r, aux, packed, xmin, xmax, info0, info1,
                            norm, status, stream, nullptr, param);
}

int eq4_row_range_f64(const double* x, int64_t rows, int64_t dim, int64_t ld, int method, double param,
                      double* xmin, double* xmax, int32_t* info0, int32_t* status, void* stream) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "input vector is empty");
  if (ld < dim) return fail(EQ4_EINVAL, "ld must be >= dim");
  if (!x || !xmin || !xmax) return fail(EQ4_EINVAL, "null buffer");
  if (method != EQ4_METHOD_ACIQ && method != EQ4_METHOD_GSS)
    return fail(EQ4_EUNSUPPORTED, "float64 rows: only aciq and gss ranges are computed here");
  if (!(param >= 0.0) || !std::isfinite(param)) return fail(EQ4_EINVAL, "param must be finite and >= 0");
  if (param == 0.0) param = method == EQ4_METHOD_ACIQ ? 5.03 : 1e-4;
  cudaStream_t s = (cudaStream_t)stream;
  if (status) {
    const cudaError_t e = cudaMemsetAsync(status, 0, 4, s);
    if (e != cudaSuccess) return cuda_fail(e, "status reset");
  }
  std::string err;
  const int rc = eq4_rowrange_f64_launch(x, rows, dim, ld, method, param, xmin, xmax, info0, status, s, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

// TABLE range keys of rows [0, rows) accumulated into keys[0..1] (k_table_init first).
static int table_keys_accumulate(const float* x, int64_t rows, int64_t dim, int64_t ld, int* keys,
                                 cudaStream_t s) {
  int64_t blocks = (rows + 7) / 8;                       // 8 warps per block, >= 1 row each
  const int64_t cap = (int64_t)sm_count() * 4;
  if (blocks > cap) blocks = cap;
  k_table_minmax<<<(unsigned)std::max<int64_t>(1, blocks), 256, 0, s>>>(x, rows, (int)dim, ld, keys);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EQ4_OK : cuda_fail(e, "k_table_minmax");
}

static int quantize_pack_impl(const float* x, int64_t rows, int64_t dim, int64_t ld, int method,
                              int b, double r, int aux, uint8_t* packed, double* xmin, double* xmax,
                              int32_t* info0, int32_t* info1, double* norm, int32_t* status,
                              void* stream, const int* table_keys, double param) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "table must be at least 1x1");
  if (ld < dim) return fail(EQ4_EINVAL, "ld must be >= dim");
  if (!x || !packed) return fail(EQ4_EINVAL, "null buffer");
  if (aux != EQ4_AUX_FP16 && aux != EQ4_AUX_FP32) return fail(EQ4_EINVAL, "aux must be fp32 or fp16");
  if ((xmin == nullptr) != (xmax == nullptr)) return fail(EQ4_EINVAL, "xmin/xmax must be given together");
  if (method == EQ4_METHOD_GREEDY || method == EQ4_METHOD_HIST_BRUTE ||
      method == EQ4_METHOD_HIST_APPRX) {
    if (b < 1) return fail(EQ4_EINVAL, "b must be >= " "1, got " + std::to_string(b));
  }
  if (method == EQ4_METHOD_GREEDY && !(0.0 < r && r <= 1.0))
    return fail(EQ4_EINVAL, "r must be in (0, 1], got " + std::to_string(r));
  cudaStream_t s = (cudaStream_t)stream;
  Params p;
  memset(&p, 0, sizeof(p));
  p.x = x; p.rows = rows; p.ld = ld; p.d = (int)dim; p.b = b; p.r = r; p.aux = aux;
  p.stride = (int)eq4_packed_row_stride(dim, aux);
  p.half = (int)((dim + 1) / 2);
  p.packed = packed; p.lo_out = xmin; p.hi_out = xmax; p.info0 = info0; p.info1 = info1;
  p.status = status;
  // vector path: 16-byte aligned rows in, 2-byte aligned packed rows out
  const bool vec = (dim % 4 == 0) && (ld % 4 == 0) && (((uintptr_t)x & 15) == 0) &&
                   (((uintptr_t)packed & 1) == 0);
  if (method == EQ4_METHOD_ASYM) return dispatch_rq<M_ASYM>(p, vec, s);
  if (method == EQ4_METHOD_SYM) {
    p.range_mode = 1;
    return dispatch_rq<M_ASYM>(p, vec, s);
  }
  if (method == EQ4_METHOD_TABLE) {
    p.range_mode = 2;
    if (table_keys) {   // range computed by the caller (chunked host path)
      p.trange = table_keys;
      return dispatch_rq<M_ASYM>(p, vec, s);
    }
    int* keys = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&keys, 8, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    k_table_init<<<1, 1, 0, s>>>(keys);
    int rc = table_keys_accumulate(x, rows, dim, ld, keys, s);
    p.trange = keys;
    if (rc == EQ4_OK) rc = dispatch_rq<M_ASYM>(p, vec, s);
    cudaFreeAsync(keys, s);
    return rc;
  }
  if (method == EQ4_METHOD_ACIQ || method == EQ4_METHOD_GSS) {
    std::string err;
    if (param == 0.0) param = method == EQ4_METHOD_ACIQ ? 5.03 : 1e-4;   // clipping.py:70,125-126
    const int rc = eq4_rowrange_launch(x, rows, dim, ld, method, param, aux, packed, xmin, xmax, info0,
                                       status, s, err);
    return rc == EQ4_OK ? rc : fail(rc, err);
  }
  if (method == EQ4_METHOD_HIST_APPRX) {
    std::string err;
    const int rc = eq4_hist_launch(x, rows, dim, ld, b, aux, packed, xmin, xmax, info0, info1, norm,
                                   status, s, err, true);
    return rc == EQ4_OK ? rc : fail(rc, err);
  }
  if (method == EQ4_METHOD_GREEDY) {
    // W * alpha must stay exact in fp32 (kw_of) and 15 b representable on the Y grid
    if (b > 262143) return fail(EQ4_EUNSUPPORTED, "GREEDY with b > 262143 is not supported by the B200 path");
    // Loop condition (clipping.py:180) at iteration it, i.e. after it moves
    // (nl + nr == it): exactly  (it + b(1-r)) * step < x1 - x0  <=>  it < T with
    // T = b - b(1-r).  For it <= T - 1 the two sides differ by >= one step,
    // far beyond the float64 rounding of a row with max|x| <= 1e6 (max - min)
    // (wider-magnitude rows run exact_only and always evaluate it), so the
    // first iteration that needs the float64 test is floor(T).
    const double B1 = (double)b * (1.0 - r);
    const double T = (double)b - B1;
    p.it_exact_from = T >= 1.0 ? (int)std::floor(T) : 0;
    int ey = 0;
    while (std::ldexp(1.0, ey) <= 15.0 * b) ey++;
    p.qY = std::ldexp(1.0, ey - 24);
    p.inv_qY = 1.0 / p.qY;
    p.delta = (float)(p.qY * 0.5);
    p.tau2 = tau2_for((int)dim, vec);
    // misround: the code argument alpha*s carries |error| <= eta = ETA_CODE
    // (kW within 1 ulp, s rounded once), so a code can differ from the reference's
    // only for elements within eta of a rounding boundary, each adding
    // <= 2*eta*W^2 to the loss; the band allows 2 per side, both sides.
    p.kmis = (float)(2.0 * 2.0 * 2.0 * ETA_CODE);
    // ... and when more than 2 elements of a side could misround (repeated values
    // parked next to a boundary), the comparison is only trusted after counting
    // them (near_escalate): up to all d elements per side
    p.kmisx = p.kmis * (float)std::max<int64_t>(0, dim - 2) * 0.5f;
    if (const char* ev = getenv("EQ4_DEV_KMISX_SCALE")) p.kmisx *= (float)atof(ev);   // development A/B only
    // rows with max|x| <= 1e6 (max - min) (others run exact_only): the
    // reference's rounded grid moves its losses by <= 3e-14 * 1e6 relative
    p.tau2 += (float)(2.0 * 3e-14 * 1e6);
    p.c1 = (float)(4.2 * p.delta * std::sqrt((double)dim));
    p.c0 = (float)(2.1 * (double)dim * p.delta * p.delta);
    {
      // table walk (eq4_gtable.cuh): y on the 2^-33 grid (plus the float64 rounding of Y itself);
      // the reference's reconstruction rounds at 2^-53 max|x| per element -- in Y units
      // 2^-52 * 15 b * mr over both roundings -- and its sums and squares at a few 2^-53 relative
      // (3e-14 mr with the candidate grid, as above); the polynomial's float64 evaluation and the
      // conversions of P1 and the chi sum move a candidate by <= 17 * 2^-53 * d (15 b)^2.
      const double Yb = 15.0 * b, u = std::ldexp(1.0, -53);
      const double dl = std::ldexp(1.0, -34) + 8.0 * u * Yb;
      p.tb_eps = 2.1 * 3e-14;
      p.tb_c1a = 4.2 * dl * std::sqrt((double)dim);
      p.tb_c1b = 4.2 * 2.0 * u * Yb * std::sqrt((double)dim);
      p.tb_c0 = 2.1 * (double)dim * dl * dl + 40.0 * u * (double)dim * Yb * Yb + 1e-9 * (double)dim;
    }
    return dispatch_rq<M_GREEDY>(p, vec, s);
  }
  if (method == EQ4_METHOD_HIST_BRUTE) {
    std::string err;
    const int rc = eq4_hist_launch(x, rows, dim, ld, b, aux, packed, xmin, xmax, info0, info1, norm,
                                   status, s, err, false);
    return rc == EQ4_OK ? rc : fail(rc, err);
  }
  return fail(EQ4_EINVAL, "unknown method " + std::to_string(method));
}

int eq4_pack(const uint8_t* codes, int64_t rows, int64_t dim, int aux, const void* scales,
             const void* biases, uint8_t* packed, void* stream) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "bad shape");
  int stride = (int)eq4_packed_row_stride(dim, aux);
  int64_t n = rows * stride;
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
  k_pack<<<grid, 256, 0, (cudaStream_t)stream>>>(codes, rows, (int)dim, aux,
                                                 (const uint8_t*)scales, (const uint8_t*)biases,
                                                 packed, stride);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EQ4_OK : cuda_fail(e, "k_pack");
}

int eq4_unpack(const uint8_t* packed, int64_t rows, int64_t dim, int aux, uint8_t* codes,
               void* scales, void* biases, void* stream) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "bad shape");
  int stride = (int)eq4_packed_row_stride(dim, aux);
  int64_t n = rows * stride;
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
  k_unpack<<<grid, 256, 0, (cudaStream_t)stream>>>(packed, rows, (int)dim, aux, codes,
                                                   (uint8_t*)scales, (uint8_t*)biases, stride);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EQ4_OK : cuda_fail(e, "k_unpack");
}

int eq4_quant_mse(const float* x, int64_t rows, int64_t dim, int64_t ld, const double* xmin,
                  const double* xmax, double* out, void* stream) {
  if (rows < 1 || dim < 1 || ld < dim) return fail(EQ4_EINVAL, "bad shape");
  if (dim > 4096) return fail(EQ4_EUNSUPPORTED, "quant_mse: dim > 4096");
  size_t smem = (size_t)NWARPS * ((size_t)MAX_LEAVES * 16 + 512 * 8 + (((size_t)dim * 4 + 15) & ~(size_t)15));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_quant_mse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  }
  int64_t grid = std::min<int64_t>((rows + NWARPS - 1) / NWARPS, (int64_t)sm_count() * 8);
  k_quant_mse<<<(unsigned)grid, NTHREADS, smem, (cudaStream_t)stream>>>(x, rows, (int)dim, ld, xmin,
                                                                     xmax, out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EQ4_OK : cuda_fail(e, "k_quant_mse");
}

// Host-buffer entry point: chunks of rows are staged through device memory on
// two streams so that the H2D copy of chunk i+1, the kernel of chunk i and
// the D2H copy of chunk i-1 overlap (copy engines run beside the SMs).
// nr rows of a host table (row pitch ld floats) into a dense device chunk: one
// linear copy when the rows are contiguous, a pitched copy otherwise
static cudaError_t h2d_rows(float* dst, const float* src, int64_t nr, int64_t dim, int64_t ld,
                            cudaStream_t s) {
  if (ld == dim) return cudaMemcpyAsync(dst, src, (size_t)nr * dim * 4, cudaMemcpyHostToDevice, s);
  return cudaMemcpy2DAsync(dst, dim * 4, src, ld * 4, dim * 4, nr, cudaMemcpyHostToDevice, s);
}


int eq4_quantize_pack_host(const float* x, int64_t rows, int64_t dim, int64_t ld, int method,
                           int b, double r, int aux, uint8_t* packed, double* xmin, double* xmax,
                           int32_t* info0, int32_t* info1, double* norm, int64_t chunk_rows,
                           int64_t* bad_row, double* bad_lohi) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "table must be at least 1x1");
  if (ld < dim) return fail(EQ4_EINVAL, "ld must be >= dim");
  if (!x || !packed) return fail(EQ4_EINVAL, "null buffer");
  const int64_t stride = eq4_packed_row_stride(dim, aux);
  int64_t chunk = chunk_rows > 0 ? chunk_rows : std::max<int64_t>(1024, (16ll << 20) / (dim * 4));
  chunk = std::min(chunk, rows);
  const int64_t nchunks = (rows + chunk - 1) / chunk;
  const int NS = HP_NS;
  const bool want_lohi = xmin != nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(EQ4_EUNSUPPORTED, "device index out of range");
  HostPipe& hp = g_pipes[dev];
  std::lock_guard<std::mutex> lk(hp.mu);
  int rc = EQ4_OK;
  cudaError_t e = pipe_reserve(hp, chunk, dim, stride, info1 != nullptr, want_lohi, norm != nullptr,
                               nchunks);
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline buffers");
  cudaStream_t* st = hp.st;
  HostBuf* bf = hp.bf;
  int32_t* hstatus = hp.hstatus;
  // TABLE: one range over the whole table -> a first streaming pass for the min / max keys
  int* tkeys = nullptr;
  if (rc == EQ4_OK && method == EQ4_METHOD_TABLE) {
    e = cudaMallocAsync((void**)&tkeys, 8, st[0]);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMallocAsync");
    if (rc == EQ4_OK) k_table_init<<<1, 1, 0, st[0]>>>(tkeys);
    if (rc == EQ4_OK) e = cudaStreamSynchronize(st[0]);
    for (int64_t c = 0; c < nchunks && rc == EQ4_OK; c++) {
      const int si = (int)(c % NS);
      const int64_t r0 = c * chunk, nr = std::min(chunk, rows - r0);
      e = h2d_rows(bf[si].x, x + r0 * ld, nr, dim, ld, st[si]);
      if (e != cudaSuccess) { rc = cuda_fail(e, "H2D"); break; }
      rc = table_keys_accumulate(bf[si].x, nr, dim, dim, tkeys, st[si]);
    }
    for (int i = 0; i < NS && rc == EQ4_OK; i++) {
      e = cudaStreamSynchronize(st[i]);
      if (e != cudaSuccess) rc = cuda_fail(e, "stream sync");
    }
  }
  for (int64_t c = 0; c < nchunks && rc == EQ4_OK; c++) {
    const int si = (int)(c % NS);
    cudaStream_t s = st[si];
    HostBuf& B = bf[si];
    const int64_t r0 = c * chunk, nr = std::min(chunk, rows - r0);
    e = h2d_rows(B.x, x + r0 * ld, nr, dim, ld, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(B.status, 0, 4, s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "H2D"); break; }
    rc = quantize_pack_impl(B.x, nr, dim, dim, method, b, r, aux, B.out, want_lohi ? B.lo : nullptr,
                            want_lohi ? B.hi : nullptr, B.i0, info1 ? B.i1 : nullptr, norm ? B.nrm : nullptr,
                            B.status, s, tkeys);
    if (rc) break;
    e = cudaMemcpyAsync(packed + r0 * stride, B.out, nr * stride, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && info0) e = cudaMemcpyAsync(info0 + r0, B.i0, nr * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && info1) e = cudaMemcpyAsync(info1 + r0, B.i1, nr * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && want_lohi) e = cudaMemcpyAsync(xmin + r0, B.lo, nr * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && want_lohi) e = cudaMemcpyAsync(xmax + r0, B.hi, nr * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && norm) e = cudaMemcpyAsync(norm + r0, B.nrm, nr * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hstatus + c, B.status, 4, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "D2H"); break; }
  }
  for (int i = 0; i < NS; i++) {
    e = cudaStreamSynchronize(st[i]);
    if (e != cudaSuccess && rc == EQ4_OK) rc = cuda_fail(e, "stream sync");
  }
  // data-dependent failures: report the first failing row, like the reference's row loop
  if (rc == EQ4_OK) {
    for (int64_t c = 0; c < nchunks && rc == EQ4_OK; c++) {
      if (!hstatus[c]) continue;
      const int64_t r0 = c * chunk, nr = std::min(chunk, rows - r0);
      int64_t first_nf = -1, first_rg = -1;
      if (hstatus[c] & EQ4_STATUS_NONFINITE)
        for (int64_t i = 0; i < nr && first_nf < 0; i++)
          for (int64_t k = 0; k < dim; k++)
            if (!std::isfinite(x[(r0 + i) * ld + k])) { first_nf = i; break; }
      double elo = 0, ehi = 0;
      if (hstatus[c] & EQ4_STATUS_RANGE) {
        // re-run this chunk with per-row outputs to locate the row
        HostBuf& B = bf[0];
        double *dlo = nullptr, *dhi = nullptr;
        cudaMallocAsync(&dlo, nr * 8, st[0]);
        cudaMallocAsync(&dhi, nr * 8, st[0]);
        cudaMemcpy2DAsync(B.x, dim * 4, x + r0 * ld, ld * 4, dim * 4, nr, cudaMemcpyHostToDevice, st[0]);
        rc = eq4_quantize_pack(B.x, nr, dim, dim, method, b, r, aux, B.out, dlo, dhi, B.i0, nullptr,
                               nullptr, nullptr, st[0]);
        int32_t* hi0 = (int32_t*)malloc(nr * 4);
        cudaMemcpyAsync(hi0, B.i0, nr * 4, cudaMemcpyDeviceToHost, st[0]);
        cudaStreamSynchronize(st[0]);
        for (int64_t i = 0; i < nr; i++)
          if (hi0[i] == -2) { first_rg = i; break; }
        if (first_rg >= 0) {
          cudaMemcpy(&elo, dlo + first_rg, 8, cudaMemcpyDeviceToHost);
          cudaMemcpy(&ehi, dhi + first_rg, 8, cudaMemcpyDeviceToHost);
        }
        free(hi0);
        cudaFreeAsync(dlo, st[0]);
        cudaFreeAsync(dhi, st[0]);
      }
      int64_t first = -1;
      int code = EQ4_OK;
      if (first_nf >= 0) { first = first_nf; code = EQ4_EDATA; }
      if (first_rg >= 0 && (first < 0 || first_rg < first)) { first = first_rg; code = EQ4_ERANGE; }
      if (code == EQ4_EDATA) {
        rc = fail(EQ4_EDATA, "table contains non-finite values (NaN/Inf)");
      } else if (code == EQ4_ERANGE) {
        rc = fail(EQ4_ERANGE, "xmin " + py_float_repr(elo) + " exceeds xmax " + py_float_repr(ehi));
        if (bad_lohi) { bad_lohi[0] = elo; bad_lohi[1] = ehi; }
      }
      if (bad_row && first >= 0) *bad_row = r0 + first;
    }
  }
  if (tkeys) cudaFreeAsync(tkeys, st[0]);
  for (int i = 0; i < NS; i++) cudaStreamSynchronize(st[i]);
  return rc;
}

int eq4_quantize_rows(const void* x, int x_is_f64, int64_t rows, int64_t dim, int64_t ld,
                      const double* xmin, const double* xmax, int64_t range_stride, int nbits, int aux,
                      uint8_t* codes, void* scales, void* biases, void* stream) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "table must be at least 1x1");
  if (ld < dim) return fail(EQ4_EINVAL, "ld must be >= dim");
  if (nbits != 4 && nbits != 8) return fail(EQ4_EINVAL, "nbits must be 4 or 8, got " + std::to_string(nbits));
  if (aux != EQ4_AUX_FP16 && aux != EQ4_AUX_FP32) return fail(EQ4_EINVAL, "aux must be fp32 or fp16");
  if (range_stride < 0) return fail(EQ4_EINVAL, "range_stride must be >= 0");
  if (!x || !xmin || !xmax || !codes || !scales || !biases) return fail(EQ4_EINVAL, "null buffer");
  std::string err;
  const int rc = eq4_codec_quantize_rows(x, x_is_f64, rows, dim, ld, xmin, xmax, range_stride, nbits, aux,
                                         codes, scales, biases, (cudaStream_t)stream, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

int eq4_dequantize_rows(const uint8_t* codes, int64_t rows, int64_t dim, const void* scales,
                        const void* biases, int aux, float* out, void* stream) {
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "table must be at least 1x1");
  if (aux != EQ4_AUX_FP16 && aux != EQ4_AUX_FP32) return fail(EQ4_EINVAL, "aux must be fp32 or fp16");
  if (!codes || !scales || !biases || !out) return fail(EQ4_EINVAL, "null buffer");
  std::string err;
  const int rc = eq4_codec_dequantize_rows(codes, rows, dim, scales, biases, aux, out, (cudaStream_t)stream, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

int eq4_build_histogram(const void* x, int x_is_f64, int64_t rows, int64_t dim, int64_t ld, int b,
                        double* lo, double* hi, int64_t* counts, void* stream) {
  if (b < 1) return fail(EQ4_EINVAL, "b must be >= 1, got " + std::to_string(b));   // histclip.py:54-55
  if (rows < 1 || dim < 1) return fail(EQ4_EINVAL, "input vector is empty");          // histclip.py:57-58
  if (ld < dim) return fail(EQ4_EINVAL, "ld must be >= dim");
  if (!x || !lo || !hi || !counts) return fail(EQ4_EINVAL, "null buffer");
  std::string err;
  const int rc = eq4_codec_build_histogram(x, x_is_f64, rows, dim, ld, b, lo, hi, counts, (cudaStream_t)stream, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

int eq4_bin_l2_norm(const double* delta_begin, const double* delta_end, const double* density, int64_t n,
                    double* out, void* stream) {
  if (n < 0) return fail(EQ4_EINVAL, "n must be >= 0");
  if (n == 0) return EQ4_OK;
  if (!delta_begin || !delta_end || !density || !out) return fail(EQ4_EINVAL, "null buffer");
  std::string err;
  const int rc = eq4_codec_bin_l2_norm(delta_begin, delta_end, density, n, out, (cudaStream_t)stream, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

int eq4_quant_mse_rows(const void* x, int x_is_f64, int64_t rows, int64_t dim, int64_t ld,
                       const double* xmin, const double* xmax, int nbits, double* out, void* stream) {
  if (nbits != 4 && nbits != 8) return fail(EQ4_EINVAL, "nbits must be 4 or 8, got " + std::to_string(nbits));
  if (rows < 1 || dim < 1 || ld < dim) return fail(EQ4_EINVAL, "bad shape");
  if (!x || !xmin || !xmax || !out) return fail(EQ4_EINVAL, "null buffer");
  std::string err;
  const int rc = eq4_codec_quant_mse_rows(x, x_is_f64, rows, dim, ld, xmin, xmax, nbits, out, (cudaStream_t)stream, err);
  return rc == EQ4_OK ? rc : fail(rc, err);
}

// Diagnostics: the GREEDY rare-path counters (g_diag) of the current device;
// reset != 0 zeroes them after the read.  Synchronous.
int eq4_diag_counters(int64_t* out, int reset) {
  unsigned long long h[5] = {0, 0, 0, 0, 0};
  cudaError_t e = cudaMemcpyFromSymbol(h, g_diag, sizeof h);
  if (e == cudaSuccess && reset) {
    const unsigned long long z[5] = {0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_diag, z, sizeof z);
  }
  if (e != cudaSuccess) return cuda_fail(e, "diag counters");
  for (int i = 0; i < 5; i++) out[i] = (int64_t)h[i];
  return EQ4_OK;
}

// Diagnostics: run an internal arithmetic self-test on the current device and
// return the mismatch count (-1 on CUDA error).  which: 0/1 = div15 vs IEEE
// divide on float-difference / full-range doubles.
long long eq4_selftest(int which, int64_t n, uint64_t seed) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 8) != cudaSuccess) return -1;
  cudaMemset(d, 0, 8);
  k_selftest_div15<<<sm_count() * 8, 256>>>(which, n, seed, d);
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) { cuda_fail(e, "selftest"); return -1; }
  return (long long)h;
}

}  // extern "C"

// Internal entry points for the streaming file pipeline (eq4_io.cu): the TABLE
// range must cover the whole file, so it is accumulated over a first pass.
int eq4_internal_table_init(int* keys, cudaStream_t s) {
  k_table_init<<<1, 1, 0, s>>>(keys);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EQ4_OK : cuda_fail(e, "k_table_init");
}
int eq4_internal_table_accumulate(const float* x, int64_t rows, int64_t dim, int* keys,
                                  cudaStream_t s) {
  return table_keys_accumulate(x, rows, dim, dim, keys, s);
}
int eq4_internal_quantize_pack_keys(const float* x, int64_t rows, int64_t dim, int method, int b,
                                    double r, int aux, uint8_t* packed, int32_t* info0,
                                    int32_t* status, cudaStream_t s, const int* keys) {
  return quantize_pack_impl(x, rows, dim, dim, method, b, r, aux, packed, nullptr, nullptr, info0,
                            nullptr, nullptr, status, s, keys);
}


