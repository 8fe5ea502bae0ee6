// eq4_codec.cu -- the reference's standalone codec and histogram entry points on the GPU:
//   uniform.py:60-80   quantize_uniform / uniform.py:142-167 quantize_table_uniform
//                      (codes of rows against GIVEN float64 ranges, nbits 4 or 8)
//   uniform.py:83-91   dequantize_uniform (float32 scale * code + bias, two roundings)
//   histclip.py:52-67  build_histogram (np.min / np.max incl. numpy's signed-zero choice,
//                      float64 bin index, int64 counts)
//   histclip.py:70-82  bin_l2_norm (density * (de**3 - db**3) / 3.0)
//   table.py:81-103    quant_mse of float32 or float64 rows, nbits 4 or 8
// Rows may be float32 (EmbeddingTable rows) or float64 (the reference's functions take any
// array and promote it to float64).  These are element-parallel or lane-per-row kernels:
// bandwidth-class work next to the fused search kernels, exact float64 arithmetic in the
// reference's operation order (explicitly rounded intrinsics, numpy pairwise sums).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "../../include/eq4.h"
#include "eq4_device.cuh"
#include "eq4_internal.h"
#include "eq4_np.cuh"

namespace eq4 {

template <typename T>
__device__ __forceinline__ double ld_elem(const T* x, int64_t i) {
  return (double)x[i];
}

// uniform.py:77-79 / table.py:100-101 with qmax = 2^nbits - 1: one code, float64.
__device__ __forceinline__ double np_code_q(double x, double lo, double hi, double scale, double qmax) {
  const double c = np_clip(x, lo, hi);
  const double q = __ddiv_rn(__dsub_rn(c, lo), scale);
  return np_clip(floor(__dadd_rn(q, 0.5)), 0.0, qmax);
}

template <typename T>
__global__ void k_quantize_rows(const T* x, int64_t rows, int d, int64_t ld, const double* lo,
                                const double* hi, int64_t rstride, int qmax, int aux, uint8_t* codes,
                                uint8_t* scales, uint8_t* biases) {
  const int64_t n = rows * (int64_t)d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int k = (int)(e - r * d);
    const double l = lo[r * rstride], h = hi[r * rstride];
    double scale = 0.0;
    unsigned c = 0;
    if (h != l) {                                                   // uniform.py:74-76
      scale = __ddiv_rn(__dsub_rn(h, l), (double)qmax);             // uniform.py:77
      c = (unsigned)np_code_q(ld_elem(x, r * ld + k), l, h, scale, (double)qmax);
    }
    codes[e] = (uint8_t)c;
    if (k == 0) {                                                   // uniform.py:80
      if (aux == EQ4_AUX_FP16) {
        reinterpret_cast<uint16_t*>(scales)[r] = (uint16_t)aux_bits_f16(scale);
        reinterpret_cast<uint16_t*>(biases)[r] = (uint16_t)aux_bits_f16(l);
      } else {
        reinterpret_cast<uint32_t*>(scales)[r] = aux_bits_f32(scale);
        reinterpret_cast<uint32_t*>(biases)[r] = aux_bits_f32(l);
      }
    }
  }
}

// uniform.py:83-91: np.float32(scale) * codes.astype(float32) + np.float32(bias).
__global__ void k_dequantize_rows(const uint8_t* codes, int64_t rows, int d, const uint8_t* scales,
                                  const uint8_t* biases, int aux, float* out) {
  const int64_t n = rows * (int64_t)d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    float s, b;
    if (aux == EQ4_AUX_FP16) {
      s = __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(scales)[r]));
      b = __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(biases)[r]));
    } else {
      s = __uint_as_float(reinterpret_cast<const uint32_t*>(scales)[r]);
      b = __uint_as_float(reinterpret_cast<const uint32_t*>(biases)[r]);
    }
    out[e] = __fadd_rn(__fmul_rn(s, (float)codes[e]), b);
  }
}

// numpy's zero choice (np_zero_key) for a float64 element.
__device__ __forceinline__ unsigned np_zero_key_d(double v, int p, int d) {
  if (v != 0.0) return 0u;
  return np_zero_key(0.f, p, d) | (unsigned)((unsigned long long)__double_as_longlong(v) >> 63);
}

// histclip.py:52-67, one warp per row.
template <typename T>
__global__ void k_build_histogram(const T* x, int64_t rows, int d, int64_t ld, int b, double* lo_out,
                                  double* hi_out, unsigned long long* counts) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < rows; r += ws) {
    const T* xr = x + r * ld;
    double mn = INFINITY, mx = -INFINITY;
    for (int k = lane; k < d; k += 32) {
      const double v = ld_elem(xr, k);
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
    for (int o = 16; o >= 1; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
      mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    }
    if (mn == 0.0 || mx == 0.0) {   // numpy's signed-zero choice
      unsigned kz = 0u;
      for (int k = lane; k < d; k += 32) kz = max(kz, np_zero_key_d(ld_elem(xr, k), k, d));
      kz = __reduce_max_sync(FULL, kz);
      const double z = (kz & 1u) ? -0.0 : 0.0;
      if (mn == 0.0) mn = z;
      if (mx == 0.0) mx = z;
    }
    unsigned long long* cr = counts + r * b;
    if (lane == 0) { lo_out[r] = mn; hi_out[r] = mx; }
    if (mn == mx) {                                                 // histclip.py:61-63
      if (lane == 0) cr[0] = (unsigned long long)d;
      continue;
    }
    const double w = __ddiv_rn(__dsub_rn(mx, mn), (double)b);      // histclip.py:64
    for (int k = lane; k < d; k += 32) {
      const double q = floor(__ddiv_rn(__dsub_rn(ld_elem(xr, k), mn), w));
      const int idx = (int)np_clip(q, 0.0, (double)(b - 1));        // histclip.py:65
      atomicAdd(cr + idx, 1ull);
    }
  }
}

// x^3 rounded once (double-double product, then one rounding).
__device__ __forceinline__ double cube_rn(double x) {
  const double p = __dmul_rn(x, x);
  const double pe = __fma_rn(x, x, -p);            // x^2 = p + pe exactly
  const double c = __dmul_rn(p, x);
  const double ce = __fma_rn(p, x, -c);            // p*x = c + ce exactly
  return __dadd_rn(c, __fma_rn(pe, x, ce));
}

// histclip.py:70-82: density * (delta_end**3 - delta_begin**3) / 3.0.
__global__ void k_bin_l2_norm(const double* db, const double* de, const double* rho, int64_t n,
                              double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double diff = __dsub_rn(cube_rn(de[i]), cube_rn(db[i]));
    out[i] = __ddiv_rn(__dmul_rn(rho[i], diff), 3.0);
  }
}

// table.py:81-103, lane per row, any d, nbits 4 or 8, float32 or float64 rows.
template <typename T>
__global__ void k_quant_mse_rows(const T* x, int64_t rows, int d, int64_t ld, const double* lo,
                                 const double* hi, int qmax, double* out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const T* xr = x + r * ld;
    const double l = lo[r], h = hi[r];
    double v;
    if (h == l) {                                                   // table.py:96-97
      v = np_sum([&](int k) {
        const double e = __dsub_rn(ld_elem(xr, k), l);
        return __dmul_rn(e, e);
      }, d);
    } else {
      const double scale = __ddiv_rn(__dsub_rn(h, l), (double)qmax);   // table.py:99
      v = np_sum([&](int k) {
        const double xv = ld_elem(xr, k);
        const double code = np_code_q(xv, l, h, scale, (double)qmax);
        const double e = __dsub_rn(xv, __dadd_rn(__dmul_rn(scale, code), l));
        return __dmul_rn(e, e);
      }, d);
    }
    out[r] = v;
  }
}

}  // namespace eq4

using namespace eq4;

namespace {
int grid_for(int64_t n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)sms * 16));
}
int launched(const char* what, std::string& err) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return EQ4_OK;
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return EQ4_ECUDA;
}
}  // namespace

int eq4_codec_quantize_rows(const void* x, int x_f64, int64_t rows, int64_t dim, int64_t ld,
                            const double* xmin, const double* xmax, int64_t range_stride, int nbits,
                            int aux, uint8_t* codes, void* scales, void* biases, cudaStream_t s,
                            std::string& err) {
  const int qmax = (1 << nbits) - 1;
  const int grid = grid_for(rows * dim, 256);
  if (x_f64)
    k_quantize_rows<double><<<grid, 256, 0, s>>>((const double*)x, rows, (int)dim, ld, xmin, xmax,
                                                 range_stride, qmax, aux, codes, (uint8_t*)scales,
                                                 (uint8_t*)biases);
  else
    k_quantize_rows<float><<<grid, 256, 0, s>>>((const float*)x, rows, (int)dim, ld, xmin, xmax,
                                                range_stride, qmax, aux, codes, (uint8_t*)scales,
                                                (uint8_t*)biases);
  return launched("k_quantize_rows", err);
}

int eq4_codec_dequantize_rows(const uint8_t* codes, int64_t rows, int64_t dim, const void* scales,
                              const void* biases, int aux, float* out, cudaStream_t s, std::string& err) {
  k_dequantize_rows<<<grid_for(rows * dim, 256), 256, 0, s>>>(codes, rows, (int)dim, (const uint8_t*)scales,
                                                              (const uint8_t*)biases, aux, out);
  return launched("k_dequantize_rows", err);
}

int eq4_codec_build_histogram(const void* x, int x_f64, int64_t rows, int64_t dim, int64_t ld, int b,
                              double* lo, double* hi, int64_t* counts, cudaStream_t s, std::string& err) {
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)rows * (size_t)b, s);
  if (e != cudaSuccess) { err = std::string("counts reset: ") + cudaGetErrorString(e); return EQ4_ECUDA; }
  const int grid = grid_for(rows * 32, 256);
  if (x_f64)
    k_build_histogram<double><<<grid, 256, 0, s>>>((const double*)x, rows, (int)dim, ld, b, lo, hi,
                                                   (unsigned long long*)counts);
  else
    k_build_histogram<float><<<grid, 256, 0, s>>>((const float*)x, rows, (int)dim, ld, b, lo, hi,
                                                  (unsigned long long*)counts);
  return launched("k_build_histogram", err);
}

int eq4_codec_bin_l2_norm(const double* db, const double* de, const double* rho, int64_t n, double* out,
                          cudaStream_t s, std::string& err) {
  k_bin_l2_norm<<<grid_for(n, 256), 256, 0, s>>>(db, de, rho, n, out);
  return launched("k_bin_l2_norm", err);
}

int eq4_codec_quant_mse_rows(const void* x, int x_f64, int64_t rows, int64_t dim, int64_t ld,
                             const double* xmin, const double* xmax, int nbits, double* out,
                             cudaStream_t s, std::string& err) {
  const int qmax = (1 << nbits) - 1;
  const int grid = grid_for(rows, 128);
  if (x_f64)
    k_quant_mse_rows<double><<<grid, 128, 0, s>>>((const double*)x, rows, (int)dim, ld, xmin, xmax, qmax, out);
  else
    k_quant_mse_rows<float><<<grid, 128, 0, s>>>((const float*)x, rows, (int)dim, ld, xmin, xmax, qmax, out);
  return launched("k_quant_mse_rows", err);
}
