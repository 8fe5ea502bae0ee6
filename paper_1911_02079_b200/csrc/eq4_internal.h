// eq4_internal.h -- launchers shared between the translation units of libeq4.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

// HIST-BRUTE (apprx = false) / HIST-APPRX (apprx = true) fused search + quantize +
// pack (eq4_hist.cu).  Returns an EQ4_* code; on failure err holds the message.
int eq4_hist_launch(const float* x, int64_t rows, int64_t dim, int64_t ld, int b, int aux,
                    uint8_t* packed, double* xmin, double* xmax, int32_t* info0, int32_t* info1,
                    double* norm, int32_t* status, cudaStream_t s, std::string& err, bool apprx);

// Pooled lookup over packed rows (eq4_sls.cu).  Returns an EQ4_* code.
int eq4_sls_launch(const uint8_t* packed, int64_t rows, int64_t dim, int aux,
                   const int64_t* indices, int64_t nidx, const int64_t* lengths, int64_t batch,
                   float* out, int32_t* status, int64_t* bad_pos, cudaStream_t s, std::string& err);

// EMBT -> EMBQ uniform4 streaming pipeline and the EMBQ writer (eq4_io.cu).
int eq4_io_quantize_file(const char* in_path, const char* out_path, int method, int b, double r,
                         int aux, int64_t chunk_rows, int64_t* bad_row, double* bad_lohi,
                         std::string& err);
int eq4_io_write_embq(const char* path, const uint8_t* packed, int64_t rows, int64_t dim, int aux,
                      int on_device, std::string& err);

// ACIQ / GSS row-range searches + quantize + pack (eq4_rowrange.cu).
// param: ACIQ's constant (5.03 laplacian or a gaussian_constant), GSS's tol.
int eq4_rowrange_launch(const float* x, int64_t rows, int64_t dim, int64_t ld, int method, double param,
                        int aux, uint8_t* packed, double* xmin, double* xmax, int32_t* info0,
                        int32_t* status, cudaStream_t s, std::string& err);
// ACIQ / GSS ranges of float64 rows (the scalar entry points), no packing.
int eq4_rowrange_f64_launch(const double* x, int64_t rows, int64_t dim, int64_t ld, int method,
                            double param, double* xmin, double* xmax, int32_t* info0, int32_t* status,
                            cudaStream_t s, std::string& err);

// Row-wise KMEANS codebooks (eq4_kmeans.cu).
int eq4_kmeans_launch(const float* x, int64_t rows, int64_t dim, int64_t ld, int aux, uint8_t* out,
                      int32_t* iters, int32_t* status, cudaStream_t s, std::string& err);

// TABLE-range helpers for the file pipeline (eq4.cu).
int eq4_internal_table_init(int* keys, cudaStream_t s);
int eq4_internal_table_accumulate(const float* x, int64_t rows, int64_t dim, int* keys,
                                  cudaStream_t s);
int eq4_internal_quantize_pack_keys(const float* x, int64_t rows, int64_t dim, int method, int b,
                                    double r, int aux, uint8_t* packed, int32_t* info0,
                                    int32_t* status, cudaStream_t s, const int* keys);

// Standalone codec / histogram helpers (eq4_codec.cu).  x_f64: rows are float64.
int eq4_codec_quantize_rows(const void* x, int x_f64, int64_t rows, int64_t dim, int64_t ld,
                            const double* xmin, const double* xmax, int64_t range_stride, int nbits,
                            int aux, uint8_t* codes, void* scales, void* biases, cudaStream_t s,
                            std::string& err);
int eq4_codec_dequantize_rows(const uint8_t* codes, int64_t rows, int64_t dim, const void* scales,
                              const void* biases, int aux, float* out, cudaStream_t s, std::string& err);
int eq4_codec_build_histogram(const void* x, int x_f64, int64_t rows, int64_t dim, int64_t ld, int b,
                              double* lo, double* hi, int64_t* counts, cudaStream_t s, std::string& err);
int eq4_codec_bin_l2_norm(const double* db, const double* de, const double* rho, int64_t n, double* out,
                          cudaStream_t s, std::string& err);
int eq4_codec_quant_mse_rows(const void* x, int x_f64, int64_t rows, int64_t dim, int64_t ld,
                             const double* xmin, const double* xmax, int nbits, double* out,
                             cudaStream_t s, std::string& err);

// Python's repr(float) text (eq4.cu), for the reference's ValueError messages.
std::string py_float_repr(double v);
