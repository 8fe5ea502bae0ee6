// eq4_gtable.cuh -- GREEDY screening on wide rows by a per-row threshold table
// (included by eq4.cu inside namespace eq4, after Params and the code helpers).
//
// clip_range_greedy (clipping.py:142-193) evaluates 2 candidates per iteration, each a
// quant_mse over the whole row (table.py:81-103): O(d) per candidate, ~131 candidates.
// In row coordinates Y = 15 (x - x0) / step a candidate (nl, nr) has base B = 15 nl and
// width W = b - nl - nr, reconstruction points B + c W (c = 0..15) and rounding
// thresholds T_c = B + (c - 1/2) W, c = 1..15 -- always multiples of 1/2.  With the
// nearest (clamped) code the squared error of an element telescopes over the thresholds
// it lies above,
//     (y - r_code)^2 = (y - B)^2 - 2 W * sum_{c : y >= T_c} (y - T_c),
// so the candidate's loss is
//     L(B, W) = P2 - 2 B P1 + d B^2 - 2 W * sum_{c=1..15} chi(T_c),
//     chi(T) = sum_t max(y_t - T, 0),  P1 = sum y,  P2 = sum y^2.
// chi is one function per row and every T the walk can visit is m/2 with m in 0..30 b:
// the kernel histograms the row once into the 30 b + 1 half-unit bins, turns the bins
// into the table chi[m] with one suffix scan, and then every candidate costs 15 table
// reads -- O(d + b) per row instead of O(d * iterations).
//
// Arithmetic.  y is rounded to the 2^-33 grid (yi = rint(Y * 2^33), a 64-bit integer whose
// high word is the bin and whose low word the offset inside the bin); counts, offset sums,
// chi and P1 are exact integers, the polynomial above is evaluated in float64.  What the
// value can differ from the reference's float64 loss by is bounded per row (band below,
// DESIGN.md "table walk"): the grid rounding (delta = 2^-34), the float64 evaluation of the
// polynomial (cancellation against d (15 b)^2), and the reference's own rounding.  A
// comparison whose operands are closer than the band defers the row to k_greedy in list
// mode (resume record at the last checkpoint), exactly like k_greedy_fast; so do rows the
// walk does not take (non-finite values, a zero min or max, constant rows, coarse grids).
//
// One warp per row; the table (8 B x (30 b + 2), 48 KB at b = 200) lives in the warp's
// shared memory, the row itself is read three times (range; histogram; codes), twice from
// L2.
#pragma once

struct TableSlice {
  __host__ __device__ static int nbins(int b) { return 30 * b + 2; }
  // entries per lane in the scan; odd, so the lanes' 8-byte columns fall in distinct banks
  __host__ __device__ static int chunk(int b) { return ((nbins(b) + 31) / 32) | 1; }
  __host__ __device__ static size_t bytes(int b) { return (size_t)chunk(b) * 32 * 8 + 16; }
};

__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int o) {
  const unsigned lo = __shfl_xor_sync(FULL, (unsigned)v, o);
  const unsigned hi = __shfl_xor_sync(FULL, (unsigned)(v >> 32), o);
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long shfl_down_u64(unsigned long long v, int o) {
  const unsigned lo = __shfl_down_sync(FULL, (unsigned)v, o);
  const unsigned hi = __shfl_down_sync(FULL, (unsigned)(v >> 32), o);
  return ((unsigned long long)hi << 32) | lo;
}

// chi sums of two candidates of width W (bases B0, B1): lanes 0..14 read the 15
// thresholds of the first, lanes 16..30 of the second; every lane returns both sums.
__device__ __forceinline__ void table_pair(const unsigned long long* tab, int lane, int B0, int B1, int W,
                                           unsigned long long& s0, unsigned long long& s1) {
  const int c = (lane & 15) + 1;
  const int Bx = (lane & 16) ? B1 : B0;
  const int idx = 2 * Bx + (2 * c - 1) * W;
  unsigned long long v = c <= 15 ? tab[idx] : 0ull;
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) v += shfl_xor_u64(v, o);
  const unsigned long long w = shfl_xor_u64(v, 16);
  s0 = (lane & 16) ? w : v;
  s1 = (lane & 16) ? v : w;
}

__global__ void __launch_bounds__(128) k_greedy_table(const Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = TableSlice::chunk(p.b);
  unsigned long long* tab = reinterpret_cast<unsigned long long*>(smem + warp * TableSlice::bytes(p.b));
  unsigned* tab32 = reinterpret_cast<unsigned*>(tab);
  const int nwb = (int)(blockDim.x >> 5);
  const int64_t wstride = (int64_t)gridDim.x * nwb;
  const int d4 = p.d >> 2;
  const double dd = (double)p.d;
  unsigned ndefer = 0u, nexact = 0u;

  for (int64_t row = (int64_t)blockIdx.x * nwb + warp; row < p.rows; row += wstride) {
    const float4* src = reinterpret_cast<const float4*>(p.x + row * p.ld);
    // ---- range and finiteness (clipping.py:163-165) ----
    float mn = INFINITY, mx = -INFINITY, sm = 0.f;
#pragma unroll 4
    for (int i = lane; i < d4; i += 32) {
      const float4 t = __ldg(src + i);
      mn = fminf(mn, fminf(fminf(t.x, t.y), fminf(t.z, t.w)));
      mx = fmaxf(mx, fmaxf(fmaxf(t.x, t.y), fmaxf(t.z, t.w)));
      sm = __fadd_rn(sm, __fadd_rn(__fadd_rn(t.x, t.y), __fadd_rn(t.z, t.w)));
    }
    mn = group_min<32>(mn);
    mx = group_max<32>(mx);
    sm = group_sum<32>(sm);
    const float M = fmaxf(fabsf(mn), fabsf(mx));
    // rows the table walk does not take (the band's premises; numpy's signed-zero choice)
    bool defer = !isfinite(sm) || mn == 0.f || mx == 0.f || !(mn < mx) || !(M <= 1e6f * (mx - mn));
    // the next row towards L2 while this one is walked
    {
      const int64_t nrow = row + wstride;
      if (nrow < p.rows) {
        const char* np = reinterpret_cast<const char*>(p.x + nrow * p.ld);
        for (int o = lane * 128; o < p.d * 4; o += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(np + o));
      }
    }
    const double x0 = (double)mn, x1 = (double)mx;
    const double step = __ddiv_rn(__dsub_rn(x1, x0), (double)p.b);                    // clipping.py:172
    int nl = 0, nr = 0, bi = 0, bj = 0;
    int cp_it = 0, cp_nl = 0, cp_bi = 0, cp_bj = 0;
    float cp_L = 0.f;
    if (!defer) {
      // ---- histogram: bin = floor(2 y), offset sums with carries, exact P1 ----
      for (int i = lane; i < L * 32; i += 32) tab[i] = 0ull;
      __syncwarp();
      const double kY = __ddiv_rn(15.0, step);
      const double C = 786432.0;   // 1.5 * 2^19: Y + C is Y rounded to the 2^-33 grid
      unsigned long long p1i = 0ull;
      double p2 = 0.0;
#pragma unroll 2
      for (int i = lane; i < d4; i += 32) {
        const float4 t = __ldg(src + i);
        const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double Y = __dmul_rn(__dsub_rn((double)tv[k], x0), kY);
          const double yc = __dadd_rn(Y, C);
          const unsigned long long v =
              (unsigned long long)(__double_as_longlong(yc) - __double_as_longlong(C));   // rint(Y 2^33)
          const double yh = __dsub_rn(yc, C);
          p2 = __fma_rn(yh, yh, p2);
          p1i += v;
          const unsigned m = (unsigned)(v >> 32), o = (unsigned)v;
          const unsigned old = atomicAdd(&tab32[2 * m], o);
          const unsigned carry = (unsigned)(old + o < old);
          atomicAdd(&tab32[2 * m + 1], (1u << 17) + carry);
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        p1i += shfl_xor_u64(p1i, o);
        p2 = __dadd_rn(p2, __shfl_xor_sync(FULL, p2, o));
      }
      const double p1 = __dmul_rn(__ull2double_rn(p1i), 0x1p-33);
      __syncwarp();
      // ---- chi[m] = chi[m+1] + (count above m) / 2 + (offset sum of bin m), top-down ----
      {
        unsigned long long* mine = tab + lane * L;
        unsigned cl = 0u;
        unsigned long long xl = 0ull;
        for (int t = L - 1; t >= 0; --t) {
          const uint2 e = *reinterpret_cast<const uint2*>(mine + t);
          xl += ((unsigned long long)(cl + (e.y & 0x1FFFFu)) << 32) + e.x;
          cl += e.y >> 17;
        }
        unsigned cin = cl;   // counts in the lanes above
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_down_sync(FULL, cin, o);
          if (lane + o < 32) cin += v;
        }
        cin -= cl;
        const unsigned long long tl = xl + ((unsigned long long)(cin * (unsigned)L) << 32);
        unsigned long long xin = tl;   // chi entering this lane's chunk from above
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long v = shfl_down_u64(xin, o);
          if (lane + o < 32) xin += v;
        }
        xin -= tl;
        for (int t = L - 1; t >= 0; --t) {
          const uint2 e = *reinterpret_cast<const uint2*>(mine + t);
          xin += ((unsigned long long)(cin + (e.y & 0x1FFFFu)) << 32) + e.x;
          cin += e.y >> 17;
          mine[t] = xin;
        }
      }
      __syncwarp();
      // ---- the walk (clipping.py:174-192), every lane with the same values ----
      const double mr = fmax(1.0, (double)M / ((double)mx - (double)mn));
      const double eps = p.tb_eps * mr, c1 = p.tb_c1a + p.tb_c1b * mr;
      auto loss_of = [&](int B, int W, unsigned long long sx) {
        const double Bd = (double)B;
        double a = __fma_rn(-2.0 * Bd, p1, p2);
        a = __fma_rn(dd * Bd, Bd, a);
        return __fma_rn(-0x1p-32 * (double)W, __ull2double_rn(sx), a);
      };
      double Lbest;
      {
        unsigned long long s0, s1;
        table_pair(tab, lane, 0, 0, p.b, s0, s1);
        Lbest = loss_of(0, p.b, s0);                                                  // :174
      }
      const double min_steps = __dmul_rn(__dmul_rn((double)p.b, __dsub_rn(1.0, p.r)), step);   // :173
      for (int it = 0;; ++it) {
        if ((it & 7) == 0 && it > 0 && it < 8 * RG_GROUPS) {
          cp_it = it; cp_nl = nl; cp_bi = bi; cp_bj = bj; cp_L = (float)Lbest;
        }
        if (it >= p.it_exact_from) {   // clipping.py:180 in float64 (earlier: provably true)
          const double lhs = __dadd_rn(__dadd_rn(x0, __dmul_rn((double)nl, step)), min_steps);
          const double rhs = __dsub_rn(x1, __dmul_rn((double)nr, step));
          if (!(lhs < rhs)) break;
        }
        const int W = p.b - it - 1;
        if (W < 1) { defer = true; break; }   // widths below 1: the exact kernel walks on
        unsigned long long sL, sR;
        table_pair(tab, lane, 15 * (nl + 1), 15 * nl, W, sL, sR);
        const double SL = loss_of(15 * (nl + 1), W, sL), SR = loss_of(15 * nl, W, sR);
        const bool goL = SL < SR;                                                     // :185
        const double cand = goL ? SL : SR;
        const double mall = fmax(fmax(SL, SR), Lbest);
        const double band = __fma_rn(eps, mall, __fma_rn(c1, (double)sqrt_approx(fmaxf((float)mall, 0.f)) * 1.001, p.tb_c0));
        const double gap = fmin(fabs(SL - SR), fabs(cand - Lbest));
        if (gap <= band) { defer = true; break; }
        nl += goL;
        nr += !goL;
        if (cand < Lbest) { Lbest = cand; bi = nl; bj = nr; }                         // :187,191
      }
    }
    if (!defer) {
      // ---- result, codes (uniform.py:77-79), pack ----
      const double lo = (bi == 0 && bj == 0) ? x0 : __dadd_rn(x0, __dmul_rn((double)bi, step));   // :175,182
      const double hi = bj == 0 ? x1 : __dsub_rn(x1, __dmul_rn((double)bj, step));
      const CodeParams cp = make_code_params(lo, hi);
      uint8_t* orow = p.packed + (size_t)row * p.stride;
      bool any_exact = false;
#pragma unroll 2
      for (int i = lane; i < d4; i += 32) {
        const float4 t = __ldg(src + i);
        bool n0, n1, n2, n3;
        unsigned c0 = code_of(t.x, cp, n0), c1 = code_of(t.y, cp, n1);
        unsigned c2 = code_of(t.z, cp, n2), c3 = code_of(t.w, cp, n3);
        if (n0 | n1 | n2 | n3) {   // rare: numpy's float64 codec for an element next to a boundary
          if (n0) c0 = code_exact(t.x, cp);
          if (n1) c1 = code_exact(t.y, cp);
          if (n2) c2 = code_exact(t.z, cp);
          if (n3) c3 = code_exact(t.w, cp);
          any_exact = true;
        }
        *reinterpret_cast<uint16_t*>(orow + 2 * i) = (uint16_t)(c0 | (c1 << 4) | (c2 << 8) | (c3 << 12));
      }
      nexact += __any_sync(FULL, any_exact) ? 1u : 0u;
      if (lane == 0) {
        const double sc = div15(__dsub_rn(hi, lo));                                   // uniform.py:74-80
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
    } else if (lane == 0) {
      // deferred: a resume record when the walk passed a checkpoint, else the restart list
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
      if (!stored) p.dlist[(unsigned)atomicAdd(p.dcount, 1)] = (uint32_t)row;
      ++ndefer;
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (nexact) atomicAdd(&g_diag[1], (unsigned long long)nexact);
    if (ndefer) atomicAdd(&g_diag[4], (unsigned long long)ndefer);
  }
}
