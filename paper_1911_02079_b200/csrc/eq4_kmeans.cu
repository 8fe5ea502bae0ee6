// eq4_kmeans.cu -- row-wise KMEANS codebooks (
// codebook.py:35-172): per row, scalar Lloyd iterations seeded at the 16
// points of the row's uniform grid, float64, then a stable sort of the
// codebook.  Output is the EMBQ kmeans_row payload (fileio.py:105-110): per
// row 16 codebook values at the aux width, then the ceil(d/2) nibble bytes of
// the indices (element 2k in the low nibble).
//
// Lane-per-row: every comparison and every float64 sum of the reference must
// be replayed in order (argmin |v - c| with ties to the lower index, numpy
// pairwise sums for the SSE and for each cluster mean, strict improvements of
// the best SSE, movement < 1e-7 * spread), so each lane runs its own row's
// Lloyd loop while the warp stages 32 rows as a [d][33] column tile.  The 16
// centers live in registers (fully unrolled cluster loops); assignments are a
// per-lane byte column in shared memory; each round's cluster means run over a
// stable counting sort of the element indices by cluster (a byte column too).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/eq4.h"
#include "eq4_device.cuh"
#include "eq4_internal.h"
#include "eq4_np.cuh"

namespace eq4 {

constexpr int KM_THREADS = 128;
constexpr int KM_WARPS = KM_THREADS / 32;
constexpr int KM_K = 16;
constexpr int KM_COL = 33;

struct KMParams {
  const float* x;
  int64_t rows, ld;
  int d, aux, stride, half;
  uint8_t* out;
  int32_t* iters;
  int32_t* status;
  size_t warp_bytes;
  int staged;   // rows staged in shared memory as a [d][33] tile
};

// This lane's row: a staged [d][33] column (STAGED) or the row in global memory (wide
// rows); the stride is a compile-time constant either way.
template <bool STAGED>
struct KMLane {
  const float* xs;   // element k at xs[k * KM_COL] (staged) or xs[k]
  uint8_t* a;        // assignments, element k at a[k * 32]
  __device__ __forceinline__ float f(int k) const { return xs[STAGED ? k * KM_COL : k]; }
  __device__ __forceinline__ double v(int k) const { return (double)f(k); }
};

// members.mean() of the m members at perm[s0 ..] (perm holds each cluster's members in
// element order: a stable counting sort): 0.0 + numpy pairwise sum / m (eq4_np.cuh)
template <class Lane, typename PermT>
__device__ __forceinline__ double km_sorted_mean(const Lane& L, const PermT* perm, int s0, int m) {
  const double s = np_pw([&](int i) { return L.v(perm[(s0 + i) * 32]); }, 0, m);
  return __ddiv_rn(__dadd_rn(0.0, s), (double)m);
}

// np.sum((v - c[a])**2): numpy's pairwise order over the d squared errors (eq4_np.cuh)
template <class Lane>
__device__ __forceinline__ double km_sse(const Lane& L, const double* cl, int d) {
  return np_sum([&](int k) {
    const double e = __dsub_rn(L.v(k), cl[L.a[k * 32]]);
    return __dmul_rn(e, e);
  }, d);
}

// argmin_j |v - c_j| (first minimum), assignments to L.a, per-cluster counts (counted in
// the lane's shared-memory column hist[j * 32], then read back: one increment per
// element instead of a 16-way compare-and-add)
template <class Lane>
__device__ __forceinline__ void km_assign(const Lane& L, const double (&c)[KM_K], int d,
                                          int (&cnt)[KM_K], int* hist) {
#pragma unroll
  for (int j = 0; j < KM_K; j++) hist[j * 32] = 0;
  for (int k = 0; k < d; k++) {
    const double x = L.v(k);
    double best = fabs(__dsub_rn(x, c[0]));
    int bj = 0;
#pragma unroll
    for (int j = 1; j < KM_K; j++) {
      const double t = fabs(__dsub_rn(x, c[j]));
      if (t < best) { best = t; bj = j; }
    }
    L.a[k * 32] = (uint8_t)bj;
    hist[bj * 32] += 1;
  }
#pragma unroll
  for (int j = 0; j < KM_K; j++) cnt[j] = hist[j * 32];
}

// PermT: the cluster-sorted element indices (bytes while d <= 256: half the shared memory)
template <bool STAGED, typename PermT>
__global__ void __launch_bounds__(KM_THREADS) k_kmeans_rows(const KMParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ws = smem + (size_t)warp * p.warp_bytes;
  const int d = p.d;
  float* xs = reinterpret_cast<float*>(ws);
  uint8_t* abuf = ws + (STAGED ? (((size_t)d * KM_COL * 4 + 15) & ~(size_t)15) : 0);
  PermT* pbuf = reinterpret_cast<PermT*>(abuf + (((size_t)d * 32 + 15) & ~(size_t)15));   // sorted indices
  int* obuf = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(pbuf) +
                                     (((size_t)d * 32 * sizeof(PermT) + 15) & ~(size_t)15));   // [16][32] offsets
  uint8_t* out_base = reinterpret_cast<uint8_t*>(obuf + KM_K * 32);
  const int ab = p.aux == EQ4_AUX_FP16 ? 2 : 4;
  const int64_t nblk = (p.rows + 31) / 32;
  const int nw = blockDim.x >> 5;
  for (int64_t blk = (int64_t)blockIdx.x * nw + warp; blk < nblk; blk += (int64_t)gridDim.x * nw) {
    const int64_t row0 = blk * 32, row = row0 + lane;
    const bool rvalid = row < p.rows;
    const int nrows = (int)min((int64_t)32, p.rows - row0);
    for (int r = 0; r < nrows; r++) {
      const float* src = p.x + (row0 + r) * p.ld;
      if (STAGED)
        for (int k = lane; k < d; k += 32) xs[k * KM_COL + r] = __ldcs(src + k);
    }
    __syncwarp();
    KMLane<STAGED> L;
    // wide rows: read the row from global memory (L1/L2)
    L.xs = STAGED ? xs + lane : p.x + (rvalid ? row : row0) * p.ld;
    L.a = abuf + lane;
    PermT* perm = pbuf + lane;
    int* offs = obuf + lane;
    double c[KM_K];
    int iters = -1;
    bool bad = false;
    if (rvalid) {
      double lo = L.v(0), hi = lo;
      for (int k = 0; k < d; k++) {
        const float f = L.f(k);
        bad |= !isfinite(f);
        const double x = (double)f;
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
      }
      if (bad && p.status) atomicOr(p.status, EQ4_STATUS_NONFINITE);
      // np.unique(values).size <= 16: exact codebook (codebook.py:55-61)
      double uq[KM_K + 1];
      int nu = 0;
      for (int k = 0; k < d && nu <= KM_K && !bad; k++) {
        const double x = L.v(k);
        int pos = 0;
        while (pos < nu && uq[pos] < x) pos++;
        if (pos < nu && uq[pos] == x) continue;
        for (int q = nu; q > pos; q--) uq[q] = uq[q - 1];
        uq[pos] = x;
        nu++;
      }
      if (bad) {
#pragma unroll
        for (int j = 0; j < KM_K; j++) c[j] = 0.0;
        for (int k = 0; k < d; k++) L.a[k * 32] = 0;
      } else if (nu <= KM_K) {
#pragma unroll
        for (int j = 0; j < KM_K; j++) c[j] = j < nu ? uq[j] : uq[nu - 1];
        for (int k = 0; k < d; k++) {
          const double x = L.v(k);
          int pos = 0;
          while (uq[pos] < x) pos++;   // searchsorted(side='left')
          L.a[k * 32] = (uint8_t)pos;
        }
      } else {
        const double scale = __ddiv_rn(__dsub_rn(hi, lo), 15.0);   // _uniform_grid
#pragma unroll
        for (int j = 0; j < KM_K; j++) c[j] = __dadd_rn(lo, __dmul_rn(scale, (double)j));
        const double stop = __dmul_rn(1e-7, __dsub_rn(hi, lo));   // tol * spread
        double best_sse = INFINITY, bc[KM_K];
        double cl[KM_K];   // dynamically indexed copy of the centers (sse)
        int cnt[KM_K];
        int it = 0;
        for (it = 0; it < 100; it++) {
          km_assign(L, c, d, cnt, offs);
#pragma unroll
          for (int j = 0; j < KM_K; j++) cl[j] = c[j];
          const double sse = km_sse(L, cl, d);
          if (sse < best_sse) {
            best_sse = sse;
#pragma unroll
            for (int j = 0; j < KM_K; j++) bc[j] = c[j];
          }
          // stable counting sort of the element indices by cluster (O(d), instead of a
          // members scan per cluster), then each cluster's mean over its contiguous run
          {
            int o = 0;
#pragma unroll
            for (int j = 0; j < KM_K; j++) { offs[j * 32] = o; o += cnt[j]; }
            for (int k = 0; k < d; k++) {
              const int j = L.a[k * 32];
              const int pos = offs[j * 32];
              perm[pos * 32] = (PermT)k;
              offs[j * 32] = pos + 1;
            }
          }
          double movement = 0.0;
          int s0 = 0;
#pragma unroll
          for (int j = 0; j < KM_K; j++) {
            if (cnt[j]) {
              const double nc = km_sorted_mean(L, perm, s0, cnt[j]);
              const double t = fabs(__dsub_rn(nc, c[j]));
              movement = t > movement ? t : movement;
              c[j] = nc;
            }
            s0 += cnt[j];
          }
          if (movement < stop) break;
        }
        iters = it < 100 ? it + 1 : 100;
        km_assign(L, c, d, cnt, offs);   // score the final center update
#pragma unroll
        for (int j = 0; j < KM_K; j++) cl[j] = c[j];
        const double sse = km_sse(L, cl, d);
        if (!(sse < best_sse)) {
          // the best scored assignment is argmin |v - c| under the best centers, a function of
          // the centers alone: recompute it instead of keeping a copy per improvement
#pragma unroll
          for (int j = 0; j < KM_K; j++) c[j] = bc[j];
          km_assign(L, c, d, cnt, offs);
        }
      }
    }
    // _sorted_codebook: stable argsort of the 16 centers, rank of each center
    uint8_t* out_tile = out_base + (((uintptr_t)p.out + (size_t)row0 * p.stride) & 15);
    if (rvalid) {
      int rank[KM_K];
#pragma unroll
      for (int j = 0; j < KM_K; j++) {
        int rj = 0;
#pragma unroll
        for (int i = 0; i < KM_K; i++) rj += (c[i] < c[j]) || (c[i] == c[j] && i < j);
        rank[j] = rj;
      }
      uint8_t* orow = out_tile + (size_t)lane * p.stride;
#pragma unroll
      for (int j = 0; j < KM_K; j++) {
        // position rank[j] holds center j, cast once from float64 (astype)
        if (ab == 2) {
          const uint32_t h = aux_bits_f16(c[j]);
          orow[2 * rank[j]] = h & 0xff;
          orow[2 * rank[j] + 1] = h >> 8;
        } else {
          const uint32_t f = aux_bits_f32(c[j]);
          for (int b = 0; b < 4; b++) orow[4 * rank[j] + b] = (f >> (8 * b)) & 0xff;
        }
      }
      uint8_t* nib = orow + KM_K * ab;
      for (int m = 0; m < p.half; m++) {
        const int a0 = L.a[(2 * m) * 32];
        const int a1 = 2 * m + 1 < d ? L.a[(2 * m + 1) * 32] : -1;
        unsigned c0 = 0, c1 = 0;
#pragma unroll
        for (int j = 0; j < KM_K; j++) {
          c0 = a0 == j ? (unsigned)rank[j] : c0;
          c1 = a1 == j ? (unsigned)rank[j] : c1;
        }
        nib[m] = (uint8_t)(c0 | (c1 << 4));
      }
      if (p.iters) p.iters[row] = iters;
    }
    __syncwarp();
    {
      uint8_t* dst = p.out + (size_t)row0 * p.stride;
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

}  // namespace eq4

using namespace eq4;

int eq4_kmeans_launch(const float* x, int64_t rows, int64_t dim, int64_t ld, int aux, uint8_t* out,
                      int32_t* iters, int32_t* status, cudaStream_t s, std::string& err) {
  KMParams p;
  p.x = x; p.rows = rows; p.ld = ld; p.d = (int)dim; p.aux = aux;
  p.half = (int)((dim + 1) / 2);
  p.stride = KM_K * (aux == EQ4_AUX_FP16 ? 2 : 4) + p.half;
  p.out = out; p.iters = iters; p.status = status;
  // staged rows, assignments, cluster-sorted indices, offsets, packed tile
  // rows whose staged [d][33] tile would take more than half the shared memory are read
  // from global memory instead
  p.staged = (size_t)dim * KM_COL * 4 <= 96 * 1024;
  const size_t pbytes = dim <= 256 ? 1 : 2;
  size_t wb = (p.staged ? (((size_t)dim * KM_COL * 4 + 15) & ~(size_t)15) : 0) + (((size_t)dim * 32 + 15) & ~(size_t)15) +
              (((size_t)dim * 32 * pbytes + 15) & ~(size_t)15) + (size_t)KM_K * 32 * 4 + (size_t)32 * p.stride + 32;
  p.warp_bytes = (wb + 15) & ~(size_t)15;
  auto kern = p.staged ? (dim <= 256 ? k_kmeans_rows<true, uint8_t> : k_kmeans_rows<true, uint16_t>)
                       : (dim <= 256 ? k_kmeans_rows<false, uint8_t> : k_kmeans_rows<false, uint16_t>);
  int dev = 0, sms = 0, per_sm = 0, max_optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) { err = std::string("k_kmeans_rows setup: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  // The per-warp slice (staged rows, assignment columns) makes shared memory the
  // occupancy limit: pick the block width (1..KM_WARPS row-warps) that keeps the
  // most warps resident per SM (the Lloyd loops are latency chains).
  int nw = 1, best_warps = 0;
  for (int w = 1; w <= KM_WARPS; w++) {
    const size_t sm_w = p.warp_bytes * w;
    if (sm_w > (size_t)max_optin) break;
    int blocks = 0;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_w);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, w * 32, sm_w);
    if (e != cudaSuccess) { err = std::string("k_kmeans_rows setup: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
    if (blocks * w > best_warps) { best_warps = blocks * w; nw = w; per_sm = blocks; }
  }
  if (best_warps == 0) {
    err = "kmeans: a warp's 32 staged rows of dim " + std::to_string(dim) + " do not fit in shared memory";
    return EQ4_EUNSUPPORTED;
  }
  const size_t smem = p.warp_bytes * nw;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) { err = std::string("k_kmeans_rows setup: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  const int64_t nblk = (rows + 31) / 32;
  int64_t grid = (nblk + nw - 1) / nw;
  const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, nw * 32, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) { err = std::string("k_kmeans_rows: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  return EQ4_OK;
}
