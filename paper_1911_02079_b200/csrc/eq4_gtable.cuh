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
// polynomial (cancellation against d (15 b)^2), and the reference's own rounding.  (P2 is a
// rounded float64 sum whose error shifts every candidate of the row by the same amount, so
// it moves no comparison.)  A comparison whose operands are closer than the band defers the
// row to k_greedy in list mode (resume record at the last checkpoint), exactly like
// k_greedy_fast; so do rows the walk does not take (non-finite values, a zero min or max,
// constant rows, coarse grids).
//
// One block of NT threads per row (round 2, second version; the first ran one warp per row
// and was latency-bound at one warp per SM sub-partition): the table (8 B x (30 b + 2),
// 48 KB at b = 200) lives in the block's shared memory, four blocks per SM.  Range,
// histogram, scan and codes are spread over the block's threads; the walk itself is a
// chain of dependent decisions and runs on one warp, SPECULATIVELY: lane q evaluates one
// of the 27 candidates the next six iterations can reach (level l = 1..6 has the l + 1
// candidates with l moves, a of them to the left) with 15 table reads of its own, and the
// six decisions are then settled at once: each lane compares its candidate with its neighbour's
// (two ballots: decision bits, in-band bits), the path through the masks is integer work, and
// lane = level evaluates the loop test, the band against the running best loss and the
// checkpoint -- 6 iterations per table round trip instead of one.  Rows are pipelined through
// the block: while one warp walks row r, the others write the codes of row r - 1 and take the
// range of row r + 1 (neither touches the table) from a shared-memory work queue.  The row
// itself is read three times (range; histogram; codes), twice from L2.
#pragma once

constexpr int TB_K = 6;                          // iterations settled per table round trip
constexpr int TB_NC = TB_K * (TB_K + 3) / 2;     // candidates those iterations can reach (27)
static_assert(TB_NC <= 32, "one candidate per lane");

// per-block scratch behind the table
struct TableScratch {
  float mn[8], mx[8], sm[8];
  unsigned long long p1[8];
  double p2[8];
  unsigned cw[8];
  unsigned long long tw[8];
  int res[8];   // nl, nr, bi, bj, defer, checkpoint it / nl / (bi | bj << 16)
  float cpL;
  int q;        // next item of the codes / range queue
};

struct TableSlice {
  __host__ __device__ static int nbins(int b) { return 30 * b + 2; }
  // entries per thread in the scan; odd, so the threads' 8-byte columns fall in distinct banks
  __host__ __device__ static int chunk(int b, int nt) { return ((nbins(b) + nt - 1) / nt) | 1; }
  __host__ __device__ static size_t tab_bytes(int b, int nt) { return (size_t)chunk(b, nt) * nt * 8; }
  __host__ __device__ static size_t bytes(int b, int nt) { return tab_bytes(b, nt) + sizeof(TableScratch) + 16; }
};

__device__ __forceinline__ unsigned long long shfl_down_u64(unsigned long long v, int o) {
  const unsigned lo = __shfl_down_sync(FULL, (unsigned)v, o);
  const unsigned hi = __shfl_down_sync(FULL, (unsigned)(v >> 32), o);
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int o) {
  const unsigned lo = __shfl_xor_sync(FULL, (unsigned)v, o);
  const unsigned hi = __shfl_xor_sync(FULL, (unsigned)(v >> 32), o);
  return ((unsigned long long)hi << 32) | lo;
}

// sum of the 15 chi entries of candidate (base B, width W >= 1): thresholds 2 B + (2 c - 1) W
__device__ __forceinline__ unsigned long long table_sum15(const unsigned long long* tab, int B, int W) {
  const unsigned long long* t = tab + 2 * B + W;
  unsigned long long s0 = 0ull, s1 = 0ull, s2 = 0ull;
#pragma unroll
  for (int c = 0; c < 15; c += 3) {
    s0 += t[(2 * c) * W];
    s1 += t[(2 * c + 2) * W];
    s2 += t[(2 * c + 4) * W];
  }
  return s0 + s1 + s2;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_greedy_table(const Params p) {
  constexpr int NW = NT / 32;
  static_assert(NW >= 1 && NW <= 8, "scratch arrays hold 8 warps");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int L = TableSlice::chunk(p.b, NT);
  unsigned long long* tab = reinterpret_cast<unsigned long long*>(smem);
  unsigned* tab32 = reinterpret_cast<unsigned*>(tab);
  TableScratch* sc = reinterpret_cast<TableScratch*>(smem + TableSlice::tab_bytes(p.b, NT));
  // the walking warp: blocks that share an SM (ids one grid wave apart) use different ones,
  // so the walks spread over the SM's sub-partitions
  const int walker = (int)((blockIdx.x / (unsigned)max(p.tb_wave, 1)) % NW);
  const int d4 = p.d >> 2;
  const double dd = (double)p.d;
  unsigned ndefer = 0u, nexact = 0u;
  // this lane's candidate of a speculative round: level lv (moves made), la of them to the left
  int lv = 0, la = 0;
  {
    int q = lane;
    for (int l = 1; l <= TB_K; ++l) {
      if (lv == 0 && q <= l) { lv = l; la = q; }
      q -= l + 1;
    }
  }

#ifdef TB_PROF   // development: cycles per phase on the walking warp's lane 0 (block 0 prints)
  long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#define TBP(i) do { if (tid == walker * 32) { const long long t_ = clock64(); tp[i] += t_ - tq; tq = t_; } } while (0)
#else
#define TBP(i) do {} while (0)
#endif
  // Rows are pipelined through the block: while one warp walks row r (the only phase that is a
  // chain of dependent steps), the others write the codes of row r - 1 and take the range of row
  // r + 1 -- neither touches the table -- from a queue of 128-float4 items; the walking warp
  // joins the queue when its walk is done.
  const int nit = (d4 + 127) >> 7;   // queue items per row pass
  auto range_item = [&](const float4* src, int item, float& mn, float& mx, float& sm) {
    float4 t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = (item * 4 + k) * 32 + lane;
      t[k] = i < d4 ? __ldg(src + i) : make_float4(INFINITY, -INFINITY, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = (item * 4 + k) * 32 + lane;
      if (i < d4) {
        mn = fminf(mn, fminf(fminf(t[k].x, t[k].y), fminf(t[k].z, t[k].w)));
        mx = fmaxf(mx, fmaxf(fmaxf(t[k].x, t[k].y), fmaxf(t[k].z, t[k].w)));
        sm = __fadd_rn(sm, __fadd_rn(__fadd_rn(t[k].x, t[k].y), __fadd_rn(t[k].z, t[k].w)));
      }
    }
  };
  auto emit_item = [&](const float4* src, uint8_t* orow, const CodeParams& cp, int item, bool& any_exact) {
    float4 t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = (item * 4 + k) * 32 + lane;
      t[k] = i < d4 ? __ldg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = (item * 4 + k) * 32 + lane;
      bool n0, n1, n2, n3;
      unsigned c0 = code_of(t[k].x, cp, n0), c1 = code_of(t[k].y, cp, n1);
      unsigned c2 = code_of(t[k].z, cp, n2), c3 = code_of(t[k].w, cp, n3);
      if ((n0 | n1 | n2 | n3) && i < d4) {   // rare: numpy's float64 codec for an element next to a boundary
        if (n0) c0 = code_exact(t[k].x, cp);
        if (n1) c1 = code_exact(t[k].y, cp);
        if (n2) c2 = code_exact(t[k].z, cp);
        if (n3) c3 = code_exact(t[k].w, cp);
        any_exact = true;
      }
      if (i < d4) *reinterpret_cast<uint16_t*>(orow + 2 * i) = (uint16_t)(c0 | (c1 << 4) | (c2 << 8) | (c3 << 12));
    }
  };
  // block-wide range from the warps' partial values in the scratch (after a barrier)
  auto block_range = [&](float& mn, float& mx, float& sm) {
    mn = INFINITY; mx = -INFINITY; sm = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      mn = fminf(mn, sc->mn[w]);
      mx = fmaxf(mx, sc->mx[w]);
      sm = __fadd_rn(sm, sc->sm[w]);
    }
  };

  float mn, mx, sm;
  {   // prologue: the first row's range (clipping.py:163-165)
    float wmn = INFINITY, wmx = -INFINITY, wsm = 0.f;
    if ((int64_t)blockIdx.x < p.rows) {
      const float4* src = reinterpret_cast<const float4*>(p.x + (int64_t)blockIdx.x * p.ld);
      for (int item = warp; item < nit; item += NW) range_item(src, item, wmn, wmx, wsm);
    }
    wmn = group_min<32>(wmn); wmx = group_max<32>(wmx); wsm = group_sum<32>(wsm);
    if (lane == 0) { sc->mn[warp] = wmn; sc->mx[warp] = wmx; sc->sm[warp] = wsm; }
    __syncthreads();
    block_range(mn, mx, sm);
  }
  // the previous row, whose codes are still to be written
  bool pv = false;
  int64_t pv_row = 0;
  double pv_lo = 0.0, pv_hi = 0.0;

  for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
    const float4* src = reinterpret_cast<const float4*>(p.x + row * p.ld);
    const int64_t nrow = row + gridDim.x;
    const bool has_next = nrow < p.rows;
    // ---- clear the table ----
    for (int i = tid; i < L * NT; i += NT) tab[i] = 0ull;
    if (tid == 0) sc->q = 0;
    const float M = fmaxf(fabsf(mn), fabsf(mx));
    // rows the table walk does not take (the band's premises; numpy's signed-zero choice)
    const bool skip = !isfinite(sm) || mn == 0.f || mx == 0.f || !(mn < mx) || !(M <= 1e6f * (mx - mn));
    const double x0 = (double)mn, x1 = (double)mx;
    const double step = __ddiv_rn(__dsub_rn(x1, x0), (double)p.b);                    // clipping.py:172
    bool defer = skip;
    int nl = 0, nr = 0, bi = 0, bj = 0;
    TBP(0);
    __syncthreads();   // the table is clear; the scratch of the last row has been read
    TBP(1);
    if (!skip) {
      // ---- histogram: bin = floor(2 y), offset sums with carries, exact P1 ----
      const double kY = __ddiv_rn(15.0, step);
      const double C = 786432.0;   // 1.5 * 2^19: Y + C is Y rounded to the 2^-33 grid
      unsigned long long p1i = 0ull;
      double p2 = 0.0;
#pragma unroll 4
      for (int i = tid; i < d4; i += NT) {
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
      if (lane == 0) { sc->p1[warp] = p1i; sc->p2[warp] = p2; }
      TBP(2);
      __syncthreads();
      TBP(1);
      // ---- chi[m] = chi[m+1] + (count above m) / 2 + (offset sum of bin m), top-down ----
      {
        unsigned long long* mine = tab + tid * L;
        unsigned cl = 0u;
        unsigned long long xl = 0ull;
#pragma unroll 8
        for (int t = L - 1; t >= 0; --t) {
          const uint2 e = *reinterpret_cast<const uint2*>(mine + t);
          xl += ((unsigned long long)(cl + (e.y & 0x1FFFFu)) << 32) + e.x;
          cl += e.y >> 17;
        }
        // suffix sums over the threads above, within the warp first and with ONE block barrier:
        // counts (cin) and chi (xin).  A thread's chunk adds tl = xl + cin_total * L half-units
        // to everything below it; cin_total = (counts above in the warp) + (counts of the warps
        // above, Ca, known only after the barrier), so the warp-level sums are taken with Ca = 0
        // and the Ca terms -- (lanes above in the warp) * Ca * L -- are added afterwards.
        unsigned cin = cl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_down_sync(FULL, cin, o);
          if (lane + o < 32) cin += v;
        }
        const unsigned cw = __shfl_sync(FULL, cin, 0);   // this warp's count
        cin -= cl;                                       // counts above, inside the warp
        const unsigned long long tl0 = xl + ((unsigned long long)(cin * (unsigned)L) << 32);
        unsigned long long xin = tl0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long v = shfl_down_u64(xin, o);
          if (lane + o < 32) xin += v;
        }
        if (lane == 0) { sc->cw[warp] = cw; sc->tw[warp] = xin; }
        __syncthreads();
        xin -= tl0;                                      // chi from the lanes above, Ca = 0
        unsigned Ca = 0u;                                // counts of the warps above
        unsigned long long Xa = 0ull;                    // chi entering this warp from above
        for (int w = NW - 1; w > warp; --w) {
          // warp w as a whole: its Ca = 0 total plus 32 chunks of L bins under the counts above it
          Xa += sc->tw[w] + ((unsigned long long)(Ca * (unsigned)(32 * L)) << 32);
          Ca += sc->cw[w];
        }
        xin += Xa + ((unsigned long long)(Ca * (unsigned)((31 - lane) * L)) << 32);
        cin += Ca;
#pragma unroll 8
        for (int t = L - 1; t >= 0; --t) {
          const uint2 e = *reinterpret_cast<const uint2*>(mine + t);
          xin += ((unsigned long long)(cin + (e.y & 0x1FFFFu)) << 32) + e.x;
          cin += e.y >> 17;
          mine[t] = xin;
        }
      }
      TBP(3);
      __syncthreads();
      TBP(1);
      if (warp == walker) {
        // ---- the walk (clipping.py:174-192), every lane with the same state ----
        unsigned long long p1s = 0ull;
        p2 = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          p1s += sc->p1[w];
          p2 = __dadd_rn(p2, sc->p2[w]);
        }
        const double p1 = __dmul_rn(__ull2double_rn(p1s), 0x1p-33);
        auto loss_of = [&](int B, int W, unsigned long long sx) {
          const double Bd = (double)B;
          double a = __fma_rn(-2.0 * Bd, p1, p2);
          a = __fma_rn(dd * Bd, Bd, a);
          return __fma_rn(-0x1p-32 * (double)W, __ull2double_rn(sx), a);
        };
        double Lbest = loss_of(0, p.b, table_sum15(tab, 0, p.b));                     // :174
        // band = eps m + c1 sqrt(m) + c0 over m = max(SL, SR, Lbest), with
        // sqrt(m) <= (m / s0 + s0) / 2 for any s0 > 0 (AM-GM): one fma per comparison
        const double mr = fmax(1.0, (double)M / ((double)mx - (double)mn));
        const double c1 = p.tb_c1a + p.tb_c1b * mr;
        const double s0 = (double)sqrt_approx(fmaxf((float)Lbest, 1e-30f));
        const double kA = __fma_rn(0.5 * c1, 1.0 / s0, p.tb_eps * mr) * 1.000001;
        const double kB = __fma_rn(0.5 * c1, s0, p.tb_c0) * 1.000001;
        const double min_steps = __dmul_rn(__dmul_rn((double)p.b, __dsub_rn(1.0, p.r)), step);   // :173
        int cp_it = 0, cp_nl = 0, cp_bi = 0, cp_bj = 0;
        float cp_L = 0.f;
        bool done = false;
        int it = 0;
        const double INF = __longlong_as_double(0x7ff0000000000000ll);
        constexpr unsigned KM = (1u << TB_K) - 1u;
        while (!done && !defer) {
          // (1) this lane's candidate of the next TB_K iterations: lv moves, la of them left
          double mine = INF;
          {
            const int W = p.b - it - lv;
            if (lane < TB_NC && W >= 1) {
              const int B = 15 * (nl + la);
              mine = loss_of(B, W, table_sum15(tab, B, W));
            }
          }
          // (2) every L/R comparison those iterations could make (clipping.py:185), at once: the
          // pair (l, a - 1) | (l, a) sits in lanes q - 1 | q.  The band takes the round's
          // starting best loss -- an upper bound of every later one.
          const double left = __shfl_up_sync(FULL, mine, 1);
          const bool pair = lane < TB_NC && la >= 1;
          const double bandp = __fma_rn(fmax(fmax(mine, left), Lbest), kA, kB);
          const unsigned G = __ballot_sync(FULL, pair && mine < left);
          const unsigned NLR = __ballot_sync(FULL, pair && fabs(mine - left) <= bandp);
          // (3) the path through them: integer work on the two masks; lane l - 1 keeps level l
          unsigned P = 0u, A = 0u;   // per level: the move (1 bit) and the left moves before it (4 bits)
          {
            int a = 0;
#pragma unroll
            for (int l = 1; l <= TB_K; ++l) {
              const unsigned g = (G >> (l * (l + 1) / 2 + a)) & 1u;   // lane of the L candidate (l, a + 1)
              A |= (unsigned)a << (4 * (l - 1));
              P |= g << (l - 1);
              a += (int)g;
            }
          }
          const int lq = min(lane, TB_K - 1);
          const int mya = (int)((A >> (4 * lq)) & 15u);
          const int mypos = (lq + 1) * (lq + 2) / 2 + mya;
          const int mysel = mypos - 1 + (int)((P >> lq) & 1u);
          // (4) level l = lane + 1: the chosen candidate, the best loss before it, the tests
          const bool lvl = lane < TB_K;
          const double cands = __shfl_sync(FULL, mine, mysel);   // (every lane takes part)
          const double candl = lvl ? cands : INF;
          const double bandl = __shfl_sync(FULL, bandp, mypos);
          double pm = candl;   // inclusive running minimum over the levels
#pragma unroll
          for (int o = 1; o < TB_K; o <<= 1) {
            const double t = __shfl_up_sync(FULL, pm, o);
            if (lane >= o) pm = fmin(pm, t);
          }
          const double prev = __shfl_up_sync(FULL, pm, 1);
          const double before = lane == 0 ? Lbest : fmin(Lbest, prev);
          const bool improved = lvl && candl < before;                                // :187,191
          const int itl = it + lane, nlb = nl + mya, nrb = nr + lane - mya;
          bool exitl = false;
          if (itl >= p.it_exact_from) {   // clipping.py:180 in float64 (earlier: provably true)
            const double lhs = __dadd_rn(__dadd_rn(x0, __dmul_rn((double)nlb, step)), min_steps);
            const double rhs = __dsub_rn(x1, __dmul_rn((double)nrb, step));
            exitl = !(lhs < rhs);
          }
          // widths below 1 (the exact kernel walks on) and comparisons inside the band
          // (tb_defer_at: development / tests -- hand every row over at that iteration)
          const bool deferl = (p.b - itl - 1 < 1) || ((NLR >> mypos) & 1u) || fabs(candl - before) <= bandl ||
                              itl == p.tb_defer_at;
          const unsigned E = __ballot_sync(FULL, lvl && exitl) & KM;
          const unsigned D = __ballot_sync(FULL, lvl && deferl) & KM;
          const unsigned I = __ballot_sync(FULL, improved) & KM;
          const int ncommit = (E | D) ? __ffs(E | D) - 1 : TB_K;   // levels settled this round
          if (ncommit < TB_K) {
            if ((E >> ncommit) & 1u) done = true;   // the loop test comes first
            else defer = true;
          }
          // checkpoint: the level whose iteration index is a multiple of 8, if the walk reaches it
          {
            const int lc = ((8 - (it & 7)) & 7) + 1;   // level with (it + lc - 1) % 8 == 0
            const int itc = it + lc - 1;
            if (lc <= TB_K && lc <= ncommit + 1 && itc > 0 && itc < 8 * RG_GROUPS) {
              const unsigned Ic = I & ((1u << (lc - 1)) - 1u);
              const unsigned Pc = P & ((1u << (lc - 1)) - 1u);
              cp_it = itc;
              cp_nl = nl + __popc(Pc);
              if (Ic) {
                const int ls = 31 - __clz(Ic);   // last improving level before lc (0-based)
                const int al = __popc(P & ((2u << ls) - 1u));
                cp_L = (float)__shfl_sync(FULL, candl, ls);
                cp_bi = nl + al;
                cp_bj = nr + (ls + 1) - al;
              } else {
                cp_L = (float)Lbest; cp_bi = bi; cp_bj = bj;
              }
            }
          }
          // commit
          {
            const unsigned Im = I & ((1u << ncommit) - 1u);
            if (Im) {
              const int ls = 31 - __clz(Im);
              const int al = __popc(P & ((2u << ls) - 1u));
              Lbest = __shfl_sync(FULL, candl, ls);
              bi = nl + al;
              bj = nr + (ls + 1) - al;
            }
            const int an = __popc(P & ((1u << ncommit) - 1u));
            nl += an;
            nr += ncommit - an;
            it += ncommit;
          }
        }
        if (lane == 0) {
          sc->res[0] = nl; sc->res[1] = nr; sc->res[2] = bi; sc->res[3] = bj; sc->res[4] = defer;
          sc->res[5] = cp_it; sc->res[6] = cp_nl; sc->res[7] = cp_bi | (cp_bj << 16);
          sc->cpL = cp_L;
        }
        TBP(4);
      }
    }
    // ---- the queue: codes of the previous row, then the range of the next one ----
    bool any_exact = false;
    {
      float wmn = INFINITY, wmx = -INFINITY, wsm = 0.f;
      const int n_emit = pv ? nit : 0, n_items = n_emit + (has_next ? nit : 0);
      const float4* psrc = reinterpret_cast<const float4*>(p.x + pv_row * p.ld);
      const float4* nsrc = reinterpret_cast<const float4*>(p.x + (has_next ? nrow : row) * p.ld);
      uint8_t* porow = p.packed + (size_t)pv_row * p.stride;
      CodeParams cp;
      if (pv) cp = make_code_params(pv_lo, pv_hi);
      for (;;) {
        int item = 0;
        if (lane == 0) item = atomicAdd(&sc->q, 1);
        item = __shfl_sync(FULL, item, 0);
        if (item >= n_items) break;
        if (item < n_emit) emit_item(psrc, porow, cp, item, any_exact);
        else range_item(nsrc, item - n_emit, wmn, wmx, wsm);
      }
      wmn = group_min<32>(wmn); wmx = group_max<32>(wmx); wsm = group_sum<32>(wsm);
      if (lane == 0) { sc->mn[warp] = wmn; sc->mx[warp] = wmx; sc->sm[warp] = wsm; }
    }
    TBP(5);
    nexact += __syncthreads_or(any_exact) ? 1u : 0u;
    TBP(1);
    block_range(mn, mx, sm);   // the next row's
    if (!skip) {
      nl = sc->res[0]; nr = sc->res[1]; bi = sc->res[2]; bj = sc->res[3]; defer = sc->res[4] != 0;
    }
    pv = !defer;
    if (!defer) {
      // ---- result (the codes follow from the queue of the next round) ----
      const double lo = (bi == 0 && bj == 0) ? x0 : __dadd_rn(x0, __dmul_rn((double)bi, step));   // :175,182
      const double hi = bj == 0 ? x1 : __dsub_rn(x1, __dmul_rn((double)bj, step));
      pv_row = row; pv_lo = lo; pv_hi = hi;
      if (tid == 0) {
        uint8_t* orow = p.packed + (size_t)row * p.stride;
        const double scl = div15(__dsub_rn(hi, lo));                                  // uniform.py:74-80
        uint8_t* a = orow + p.half;
        if (p.aux == EQ4_AUX_FP16) {
          const uint32_t s16 = aux_bits_f16(scl), b16 = aux_bits_f16(lo);
          *reinterpret_cast<uint16_t*>(a) = (uint16_t)s16;
          *reinterpret_cast<uint16_t*>(a + 2) = (uint16_t)b16;
        } else {
          const uint32_t s32 = aux_bits_f32(scl), b32 = aux_bits_f32(lo);
          *reinterpret_cast<uint16_t*>(a) = (uint16_t)s32;
          *reinterpret_cast<uint16_t*>(a + 2) = (uint16_t)(s32 >> 16);
          *reinterpret_cast<uint16_t*>(a + 4) = (uint16_t)b32;
          *reinterpret_cast<uint16_t*>(a + 6) = (uint16_t)(b32 >> 16);
        }
        if (p.lo_out) { p.lo_out[row] = lo; p.hi_out[row] = hi; }
        if (p.info0) p.info0[row] = nl + nr;
        if (p.info1) p.info1[row] = p.b > 65535 ? bi : ((bi << 16) | bj);
      }
    } else if (tid == 0) {
      // deferred: a resume record when the walk passed a checkpoint, else the restart list
      bool stored = false;
      const int cp_it = skip ? 0 : sc->res[5];
      if (p.drec && cp_it > 0) {
        const int k = cp_it >> 3;
        const int slot = atomicAdd(&p.drec_count[k], 1);
        if (slot < p.drec_cap) {
          const unsigned bb = (unsigned)sc->res[7];
          p.drec[(size_t)k * p.drec_cap + slot] =
              make_uint4((unsigned)row, (unsigned)sc->res[6] | ((bb & 0xFFFFu) << 16), bb >> 16,
                         __float_as_uint(sc->cpL));
          stored = true;
        }
      }
      if (!stored) p.dlist[(unsigned)atomicAdd(p.dcount, 1)] = (uint32_t)row;
      ++ndefer;
    }
  }
  // epilogue: the last row's codes
  {
    bool any_exact = false;
    if (pv) {
      const CodeParams cp = make_code_params(pv_lo, pv_hi);
      const float4* psrc = reinterpret_cast<const float4*>(p.x + pv_row * p.ld);
      uint8_t* porow = p.packed + (size_t)pv_row * p.stride;
      for (int item = warp; item < nit; item += NW) emit_item(psrc, porow, cp, item, any_exact);
    }
    nexact += __syncthreads_or(any_exact) ? 1u : 0u;
  }
#ifdef TB_PROF
  if (blockIdx.x == 0 && tid == walker * 32)
    printf("TB_PROF cycles: clear %lld barrier-waits %lld hist %lld scan %lld walk %lld queue %lld\n", tp[0], tp[1], tp[2],
           tp[3], tp[4], tp[5]);
#endif
  if (tid == 0) {
    if (nexact) atomicAdd(&g_diag[1], (unsigned long long)nexact);
    if (ndefer) atomicAdd(&g_diag[4], (unsigned long long)ndefer);
  }
}
