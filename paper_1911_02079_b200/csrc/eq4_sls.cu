// eq4_sls.cu -- pooled lookup over packed 4-bit rows:
// sparse_lengths_sum_4bit (packed.py:167-177) on sm_100a.
//
// Contract (packed.py:155-164, test_acceptance.py:222-252): out[s, j] is the
// float32 sum, strictly in query order and starting from 0.0f, of
//   float32(scale) * float32(code) + float32(bias)
// over the rows listed by segment s; the product and the sum are separately
// rounded float32 operations (numpy evaluates scales[:, None] * codes + biases
// as two ufuncs), so there is no FMA contraction here.  fp16 scale/bias widen
// exactly to float32.
//
// Decoupling the gather from the ordered sum: the flattened index list is cut
// into tiles of T positions (T rows of the packed table fit in ~24 KB of
// shared memory).  A CTA takes the next tile (tile ids come from an atomic
// counter, so they are handed out in scheduling order), stages the tile's
// indices, and gathers all T rows into shared memory with 4-byte cp.async
// copies -- every row of the tile in flight at once, independent of how the
// positions split into segments.  Then each warp walks the segments that
// intersect the tile (segment k of the tile -> warp k mod 8), lanes over the
// row's bytes (2 codes each), summing the staged rows in query order.  A
// segment that continues into the next tile publishes its partial sums
// (carry[tile], then a release flag); the next tile's warp 0 starts that
// segment from them after an acquire spin, so the association is exactly the
// reference's ((0 + v0) + v1) + ... for any segment length.  Segment offsets
// come from a three-kernel scan of the lengths (tile sums, scan of the sums,
// per-tile downsweep), which also writes the zero rows of empty segments.
//
// Validation (PooledQuery.__post_init__, packed.py:131-140, and _check_indices,
// packed.py:147-152) runs on the device: a negative length or a length sum
// different from the index count zeroes the output and sets EQ4_STATUS_QUERY;
// an out-of-range index is skipped, sets EQ4_STATUS_INDEX and its position is
// min-reduced into *bad_pos so the host can raise the reference's IndexError
// for the first one.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/eq4.h"
#include "eq4_internal.h"

namespace eq4 {

constexpr int LT = 2048;            // lengths per scan tile (256 threads x 8)
#ifndef SLS_NTHREADS
#define SLS_NTHREADS 256
#endif
#ifndef SLS_TILE_ROWS
#define SLS_TILE_ROWS 512
#endif
#ifndef SLS_L2HINT
#define SLS_L2HINT ""
#endif
constexpr int SLS_THREADS = SLS_NTHREADS;
#ifndef SLS_MINB
#define SLS_MINB 6
#endif
constexpr int SLS_WARPS = SLS_THREADS / 32;
constexpr int SLS_BUF_BYTES = 20 * 1024;   // gathered rows of one tile
constexpr int MAX_TILE_ROWS = SLS_TILE_ROWS;

struct SlsParams {
  const uint8_t* packed;
  int64_t rows;
  int dim, half, stride, aux;
  const int64_t* indices;
  int64_t nidx;
  const int64_t* lengths;
  int64_t batch;
  float* out;
  int64_t* offsets;       // [batch] exclusive prefix sums of lengths
  int64_t* partial;       // [nlt] scan-tile sums, then their exclusive prefixes
  int64_t nlt;
  int32_t* q_ok;          // 1 = lengths valid (set by k_len_scan)
  int32_t* neg;           // a negative length was seen
  uint32_t* tile_counter;
  float* carry;           // [ntiles x dim] partial sums of a segment crossing a tile end
  int32_t* carry_flag;    // [ntiles]
  int32_t* status;
  unsigned long long* bad_pos;
  int tile_rows;
  int64_t ntiles;
  int64_t* tile_seg;      // [ntiles] first segment intersecting each tile
};

__device__ __forceinline__ void flag_index(const SlsParams& p, int64_t pos) {
  atomicMin(p.bad_pos, (unsigned long long)pos);
  if (p.status) atomicOr(p.status, EQ4_STATUS_INDEX);
}

// Programmatic dependent launch: a kernel may start while its predecessor in
// the stream is still running; griddep_wait() blocks until the predecessor
// has completed and its writes are visible.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- lengths -> offsets (PooledQuery validation, packed.py:131-140) ----

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[w] = v;
  __syncthreads();
  T t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (int)(blockDim.x >> 5) ? sh[threadIdx.x] : 0;
    for (int o = 16; o >= 1; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;   // valid in thread 0
}

__global__ void __launch_bounds__(256) k_len_partials(const SlsParams p) {
  __shared__ int64_t sh[8];
  griddep_launch();
  const int64_t base = (int64_t)blockIdx.x * LT;
  int64_t sum = 0;
  bool bad = false;
#pragma unroll
  for (int k = 0; k < LT / 256; ++k) {
    const int64_t s = base + threadIdx.x + 256 * k;
    if (s < p.batch) {
      const int64_t l = p.lengths[s];
      bad |= l < 0;
      sum += l;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *p.neg = 1;
  const int64_t t = block_sum(sum, sh);
  if (threadIdx.x == 0) p.partial[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) k_len_scan(const SlsParams p) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry_in;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  griddep_launch();
  griddep_wait();   // partial sums of k_len_partials
  if (threadIdx.x == 0) carry_in = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < p.nlt; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    const int64_t v = i < p.nlt ? p.partial[i] : 0;
    int64_t x = v;   // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t z = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      wsum[lane] = z;   // inclusive over warps
    }
    __syncthreads();
    const int64_t excl = carry_in + (w ? wsum[w - 1] : 0) + x - v;
    if (i < p.nlt) p.partial[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry_in = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const bool ok = (*p.neg == 0) && carry_in == p.nidx;
    *p.q_ok = ok ? 1 : 0;
    if (!ok && p.status) atomicOr(p.status, EQ4_STATUS_QUERY);
  }
}

__device__ void zero_row(const SlsParams& p, int64_t s) {
  float* o = p.out + s * (int64_t)p.dim;
  for (int j = 0; j < p.dim; ++j) o[j] = 0.f;
}

// Per scan tile: offsets = tile prefix + in-tile exclusive scan; zero rows for
// empty segments (no tile of the lookup kernel touches them) or, when the
// query is invalid, for every segment.
__global__ void __launch_bounds__(256) k_len_offsets(const SlsParams p) {
  __shared__ int64_t wsum[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t s0 = (int64_t)blockIdx.x * LT + 8 * threadIdx.x;
  griddep_launch();
  int64_t l[8], tsum = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    l[k] = s0 + k < p.batch ? p.lengths[s0 + k] : 0;
    tsum += l[k];
  }
  int64_t x = tsum;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  int64_t wpre = 0;
  for (int k = 0; k < w; ++k) wpre += wsum[k];
  griddep_wait();   // scanned partials and q_ok of k_len_scan
  int64_t run = p.partial[blockIdx.x] + wpre + x - tsum;
  const bool ok = *p.q_ok != 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (s0 + k < p.batch) {
      p.offsets[s0 + k] = run;
      if (!ok || l[k] == 0) zero_row(p, s0 + k);
      // tiles whose first position falls in this segment start with it
      if (ok && l[k] > 0) {
        const int64_t T = p.tile_rows;
        for (int64_t t = (run + T - 1) / T; t * T < run + l[k]; ++t) p.tile_seg[t] = s0 + k;
      }
    }
    run += l[k];
  }
}

// ---- the lookup ----

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global" SLS_L2HINT " [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ int ld_acquire(const int32_t* f) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int32_t* f) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* f, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(f), "r"(v) : "memory");
}

namespace sls {
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(f2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 add(f2 a, f2 b) {   // two separately rounded float32 adds
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
}  // namespace sls

__device__ __forceinline__ float aux_at(const uint8_t* a, int aux) {
  if (aux == EQ4_AUX_FP16)
    return __half2float(__ushort_as_half((unsigned short)(a[0] | (a[1] << 8))));
  return __uint_as_float((uint32_t)a[0] | ((uint32_t)a[1] << 8) | ((uint32_t)a[2] << 16) |
                         ((uint32_t)a[3] << 24));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Stage tile `tile`'s indices in shared memory (one coalesced pass; out-of-range
// indices, packed.py:147-152, are reported and become -1), then issue the copies
// of its rows into `buf` (row-major, the packed stride).  An out-of-range row is
// staged as zeros (scale 0, bias 0), which adds nothing to a sum.
__device__ __forceinline__ void gather_tile(const SlsParams& p, int64_t tile, uint8_t* buf,
                                            int64_t* idx_s, bool words) {
  const int T = p.tile_rows, stride = p.stride;
  const int64_t P0 = tile * T;
  const int n = (int)(min(p.nidx, P0 + T) - P0);
  for (int r = threadIdx.x; r < n; r += SLS_THREADS) {
    int64_t i = __ldg(p.indices + P0 + r);
    if (i < 0 || i >= p.rows) {
      flag_index(p, P0 + r);
      i = -1;
    }
    idx_s[r] = i;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (words) {
    const int wpr = stride >> 2;
    if (wpr <= 32) {   // a warp moves floor(32 / wpr) whole rows per step, lane -> (row, word)
      const int rpw = 32 / wpr, rr = lane / wpr, k = lane - rr * wpr;
      if (rr < rpw) {
        for (int r = warp * rpw + rr; r < n; r += SLS_WARPS * rpw) {
          const int64_t i = idx_s[r];
          uint32_t* dst = reinterpret_cast<uint32_t*>(buf + (size_t)r * stride) + k;
          if (i >= 0) cp_async4(dst, p.packed + i * stride + 4 * k);
          else *dst = 0u;
        }
      }
    } else {           // wide rows: one warp per row
      for (int r = warp; r < n; r += SLS_WARPS) {
        const int64_t i = idx_s[r];
        uint32_t* dst = reinterpret_cast<uint32_t*>(buf + (size_t)r * stride);
        for (int k = lane; k < wpr; k += 32) {
          if (i >= 0) cp_async4(dst + k, p.packed + i * stride + 4 * k);
          else dst[k] = 0u;
        }
      }
    }
  } else {             // unaligned rows: plain byte copies
    for (int r = warp; r < n; r += SLS_WARPS) {
      const int64_t i = idx_s[r];
      for (int k = lane; k < stride; k += 32)
        buf[(size_t)r * stride + k] = i >= 0 ? p.packed[i * stride + k] : (uint8_t)0;
    }
  }
  cp_async_commit();
}

// Ordered sums of the segments intersecting tile `tile` (staged in buf): segment
// k of the tile goes to warp k mod 8, lanes over the row bytes (M per lane).
template <int M>
__device__ __forceinline__ void accumulate_tile(const SlsParams& p, int64_t tile, const uint8_t* buf,
                                                bool words) {
  const int T = p.tile_rows, stride = p.stride;
  const int64_t P0 = tile * T, P1 = min(p.nidx, P0 + T);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = p.half, d = p.dim;
  const int ab = p.aux == EQ4_AUX_FP16 ? 2 : 4;
  const sls::f2 magic2 = sls::pk(-8388608.f, -8388608.f);
  const int64_t seg_first = p.tile_seg[tile];
  for (int64_t s = seg_first + warp; s < p.batch; s += SLS_WARPS) {
    const int64_t off = p.offsets[s];
    if (off >= P1) break;
    const int64_t end = off + p.lengths[s];
    if (end <= P0) continue;   // empty segments sharing the offset
    const bool before = off < P0, after = end > P1;
    const int r0 = (int)(max(off, P0) - P0), r1 = (int)(min(end, P1) - P0);
    if (before) {              // the previous tile's carry for this segment
      // poll with relaxed loads (an acquire load invalidates L1 on every poll), then
      // one acquire to order the carry reads after the flag
      while (ld_relaxed(p.carry_flag + tile - 1) == 0) __nanosleep(32);
      (void)ld_acquire(p.carry_flag + tile - 1);
    }
    for (int b0 = 0; b0 < half; b0 += 32 * M) {
      sls::f2 acc[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int j = 2 * (b0 + lane + 32 * m);
        acc[m] = sls::pk((before && j < d) ? p.carry[(tile - 1) * d + j] : 0.f,
                         (before && j + 1 < d) ? p.carry[(tile - 1) * d + j + 1] : 0.f);
      }
      int rbeg = r0;
      if (words && M == 1 && b0 + lane < half) {
        // aligned rows, one byte (two codes) per lane: 8 rows' values are formed
        // independently, then added to the running sum in query order
        sls::f2 a = acc[0];
        const int b = b0 + lane;
        for (; rbeg + 8 <= r1; rbeg += 8) {
          sls::f2 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint8_t* row = buf + (size_t)(rbeg + u) * stride;
            const uint32_t* aw = reinterpret_cast<const uint32_t*>(row + half);
            float sc, bi;
            if (ab == 2) {
              const uint32_t w = aw[0];
              sc = __half2float(__ushort_as_half((unsigned short)(w & 0xffffu)));
              bi = __half2float(__ushort_as_half((unsigned short)(w >> 16)));
            } else {
              sc = __uint_as_float(aw[0]);
              bi = __uint_as_float(aw[1]);
            }
            const uint32_t c = row[b];
            const float c0 = __fadd_rn(__uint_as_float((c & 0xFu) | 0x4B000000u), -8388608.f);
            const float c1 = __fadd_rn(__uint_as_float((c >> 4) | 0x4B000000u), -8388608.f);
            v[u] = sls::add(sls::pk(__fmul_rn(sc, c0), __fmul_rn(sc, c1)), sls::pk(bi, bi));
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) a = sls::add(a, v[u]);
        }
        acc[0] = a;
      }
#pragma unroll 8
      for (int r = rbeg; r < r1; ++r) {   // unrolled: the shared-memory loads of 8 rows in flight
        const uint8_t* row = buf + (size_t)r * stride;
        float sc, bi;
        if (words) {
          const uint32_t* aw = reinterpret_cast<const uint32_t*>(row + half);
          if (ab == 2) {
            const uint32_t w = aw[0];
            sc = __half2float(__ushort_as_half((unsigned short)(w & 0xffffu)));
            bi = __half2float(__ushort_as_half((unsigned short)(w >> 16)));
          } else {
            sc = __uint_as_float(aw[0]);
            bi = __uint_as_float(aw[1]);
          }
        } else {
          sc = aux_at(row + half, p.aux);
          bi = aux_at(row + half + ab, p.aux);
        }
        const sls::f2 bi2 = sls::pk(bi, bi);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int b = b0 + lane + 32 * m;
          if (b < half) {
            const uint32_t v = row[b];
            // codes as exact floats: 2^23 + c reinterpreted, minus 2^23
            const sls::f2 c2 = sls::add(sls::pk(__uint_as_float((v & 0xFu) | 0x4B000000u),
                                                __uint_as_float((v >> 4) | 0x4B000000u)), magic2);
            // float32(scale * code) + bias, then the running sum (packed.py:174-176).  The
            // products are scalar __fmul_rn: ptxas contracts mul.rn.f32x2 + add.rn.f32x2
            // into FFMA2, which would skip the product's rounding.
            float c0, c1;
            sls::upk(c2, c0, c1);
            const sls::f2 pr = sls::pk(__fmul_rn(sc, c0), __fmul_rn(sc, c1));
            acc[m] = sls::add(acc[m], sls::add(pr, bi2));
          }
        }
      }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const int j = 2 * (b0 + lane + 32 * m);
        float a0, a1;
        sls::upk(acc[m], a0, a1);
        float* dst = after ? p.carry + tile * d : p.out + s * (int64_t)d;
        if (j < d) dst[j] = a0;
        if (j + 1 < d) dst[j + 1] = a1;
      }
    }
    if (after) {               // publish the carry for the next tile
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release(p.carry_flag + tile, 1);
    }
  }
}

// One tile per CTA (tile ids from an atomic counter, so they are handed out in
// scheduling order and a CTA waiting for the previous tile's carry always waits
// on a resident or finished CTA).
template <int M>
__global__ void __launch_bounds__(SLS_THREADS, M <= 1 ? SLS_MINB : (M <= 4 ? 4 : 2)) k_sls_tiles(const SlsParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t claim_sh;
  const bool words = (p.stride & 3) == 0 && (p.half & 3) == 0 && (((uintptr_t)p.packed) & 3) == 0;
  if (threadIdx.x == 0) claim_sh = atomicAdd(p.tile_counter, 1u);
  __syncthreads();
  const int64_t tile = claim_sh;
  int64_t* idx_s = reinterpret_cast<int64_t*>(smem);
  uint8_t* rows_s = smem + (size_t)p.tile_rows * 8;
  gather_tile(p, tile, rows_s, idx_s, words);
  // the gather only needs the indices; segment offsets and the query check
  // come from the scan kernels that may still be finishing
  griddep_wait();
  cp_async_wait_group<0>();
  __syncthreads();
  if (*p.q_ok == 0) return;
  accumulate_tile<M>(p, tile, rows_s, words);
}

template <typename Kern>
static cudaError_t launch_pdl(Kern k, unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                              const SlsParams& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, p);
}

}  // namespace eq4

using namespace eq4;

int eq4_sls_launch(const uint8_t* packed, int64_t rows, int64_t dim, int aux,
                   const int64_t* indices, int64_t nidx, const int64_t* lengths, int64_t batch,
                   float* out, int32_t* status, int64_t* bad_pos, cudaStream_t s, std::string& err) {
  SlsParams p;
  memset(&p, 0, sizeof(p));
  p.packed = packed; p.rows = rows; p.dim = (int)dim; p.half = (int)((dim + 1) / 2);
  p.aux = aux;
  p.stride = p.half + 2 * (aux == EQ4_AUX_FP16 ? 2 : 4);
  p.indices = indices; p.nidx = nidx; p.lengths = lengths; p.batch = batch; p.out = out;
  p.status = status;
  int T = SLS_BUF_BYTES / p.stride;
  if (T > MAX_TILE_ROWS) T = MAX_TILE_ROWS;
  if (T < 1) T = 1;
  p.tile_rows = T;
  p.ntiles = (nidx + T - 1) / T;
  p.nlt = (batch + LT - 1) / LT;
  // scratch: offsets | partial | tile_seg | carry | carry_flag | q_ok, neg, tile_counter, pad | bad_pos
  const size_t off_b = 0;
  const size_t part_b = off_b + (size_t)batch * 8;
  const size_t tseg_b = part_b + (size_t)p.nlt * 8;
  const size_t carry_b = tseg_b + (size_t)p.ntiles * 8;
  const size_t flag_b = carry_b + (((size_t)p.ntiles * dim * 4 + 15) & ~(size_t)15);
  const size_t misc_b = flag_b + (((size_t)p.ntiles * 4 + 15) & ~(size_t)15);
  const size_t bad_b = misc_b + 16;
  const size_t bytes = bad_b + 8;
  uint8_t* scratch = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&scratch, bytes, s);
  if (e != cudaSuccess) { err = std::string("cudaMallocAsync: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  p.offsets = reinterpret_cast<int64_t*>(scratch + off_b);
  p.partial = reinterpret_cast<int64_t*>(scratch + part_b);
  p.tile_seg = reinterpret_cast<int64_t*>(scratch + tseg_b);
  p.carry = reinterpret_cast<float*>(scratch + carry_b);
  p.carry_flag = reinterpret_cast<int32_t*>(scratch + flag_b);
  p.q_ok = reinterpret_cast<int32_t*>(scratch + misc_b);
  p.neg = p.q_ok + 1;
  p.tile_counter = reinterpret_cast<uint32_t*>(p.q_ok + 2);
  p.bad_pos = bad_pos ? reinterpret_cast<unsigned long long*>(bad_pos)
                      : reinterpret_cast<unsigned long long*>(scratch + bad_b);
  e = cudaMemsetAsync(scratch + flag_b, 0, bad_b - flag_b, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.bad_pos, 0x7f, 8, s);   // 0x7f7f... = none
  if (e == cudaSuccess) {
    if (p.nlt > 0) k_len_partials<<<(unsigned)p.nlt, 256, 0, s>>>(p);
    e = cudaGetLastError();
    // the rest chain with programmatic dependent launch (each waits in-kernel)
    if (e == cudaSuccess) e = launch_pdl(k_len_scan, 1, 1024, 0, s, p);   // batch 0: ok iff nidx 0
    if (e == cudaSuccess && p.nlt > 0) e = launch_pdl(k_len_offsets, (unsigned)p.nlt, 256, 0, s, p);
  }
  if (e == cudaSuccess && p.ntiles > 0) {
    const size_t sm = (size_t)T * 8 + (((size_t)T * p.stride + 15) & ~(size_t)15);
    const int M = p.half <= 32 ? 1 : p.half <= 64 ? 2 : p.half <= 128 ? 4 : p.half <= 256 ? 8 : 16;
    const unsigned g = (unsigned)p.ntiles;
    switch (M) {
      case 1: e = launch_pdl(k_sls_tiles<1>, g, SLS_THREADS, sm, s, p); break;
      case 2: e = launch_pdl(k_sls_tiles<2>, g, SLS_THREADS, sm, s, p); break;
      case 4: e = launch_pdl(k_sls_tiles<4>, g, SLS_THREADS, sm, s, p); break;
      case 8: e = launch_pdl(k_sls_tiles<8>, g, SLS_THREADS, sm, s, p); break;
      default: e = launch_pdl(k_sls_tiles<16>, g, SLS_THREADS, sm, s, p); break;
    }
  }
  cudaFreeAsync(scratch, s);
  if (e != cudaSuccess) {
    err = std::string("pooled lookup launch: ") + cudaGetErrorString(e);
    return EQ4_ECUDA;
  }
  return EQ4_OK;
}
