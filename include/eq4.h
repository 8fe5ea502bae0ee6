/*
 * eq4.h -- C ABI of the B200-native row-wise 4-bit clip-search + pack library
 * (libeq4.so, paper_1911_02079_b200/).  Plain pointers and sizes only.
 *
 * The reference (`embquant`, pure Python/numpy) has no FFI layer; its
 * operator API for this path is the Python functions listed against each
 * entry point below.  paper_1911_02079_b200/api.py binds this header with
 * ctypes and re-exposes the reference's Python names; INTEGRATION.md shows
 * the binding a maintainer would add to the reference itself.
 *
 * Conventions
 *   - Device entry points (eq4_quantize_pack, eq4_pack, eq4_unpack,
 *     eq4_quant_mse) take DEVICE pointers and a cudaStream_t passed as void*;
 *     they are stream-ordered and never synchronize the host.  GREEDY on
 *     vector rows (d % 4 == 0, 16-byte aligned) runs two kernels on the
 *     stream -- an fp32 screening kernel, then the exact kernel over the rows
 *     it deferred -- with stream-ordered scratch from the device's default
 *     memory pool (cudaMallocAsync: 4 bytes per row + 28 MB of resume
 *     records); the first such call raises that pool's release threshold so
 *     the scratch is recycled, not remapped, by later calls.
 *   - Return 0 on success, an EQ4_E* code otherwise (argument errors are
 *     detected synchronously, before any launch); eq4_last_error() returns a
 *     thread-local message for the last failure on the calling thread.
 *   - Data-dependent failures (non-finite input, a search producing
 *     xmin > xmax) are reported through the optional device status word
 *     `status` (EQ4_STATUS_* bits, OR-ed) and per-row info0 == -2.
 *   - Row layout of `packed` is the reference's PackedTable4 layout
 *     (packed.py:3-6,68-83): ceil(d/2) nibble bytes (element 2k in the low
 *     nibble of byte k), then scale, then bias, little-endian, at the aux
 *     width; row stride = eq4_packed_row_stride(d, aux).
 */
#ifndef EQ4_H
#define EQ4_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EQ4_OK 0
#define EQ4_EINVAL 1      /* bad argument                                  -> ValueError */
#define EQ4_ECUDA 2       /* CUDA runtime failure                          -> RuntimeError */
#define EQ4_EDATA 3       /* host path: non-finite input (table.py:28-29)  -> ValueError */
#define EQ4_ERANGE 4      /* host path: xmin > xmax (table.py:73-74)       -> ValueError */
#define EQ4_EUNSUPPORTED 5 /* valid for the reference, not on this path    -> ValueError */

#define EQ4_METHOD_ASYM 0       /* clipping.py:58-61   clip_range_asym */
#define EQ4_METHOD_GREEDY 1     /* clipping.py:142-193 clip_range_greedy */
#define EQ4_METHOD_HIST_BRUTE 2 /* histclip.py:136-178 hist_brute_search */
#define EQ4_METHOD_SYM 3        /* clipping.py:51-55   clip_range_sym */
#define EQ4_METHOD_ACIQ 4       /* clipping.py:115-139 clip_range_aciq (constant: eq4_quantize_pack_p) */
#define EQ4_METHOD_GSS 5        /* clipping.py:70-112  clip_range_gss (tol: eq4_quantize_pack_p) */
#define EQ4_METHOD_TABLE 6      /* clipping.py:64-67   clip_range_table (one range per table) */
#define EQ4_METHOD_HIST_APPRX 7 /* histclip.py:181-217 hist_apprx_search (b <= 256) */

#define EQ4_AUX_FP32 0 /* uniform.py:19-35 aux_precision="fp32" */
#define EQ4_AUX_FP16 1 /* aux_precision="fp16" */

#define EQ4_STATUS_NONFINITE 1 /* a row holds NaN/Inf */
#define EQ4_STATUS_RANGE 2     /* a GREEDY candidate had xmin > xmax (ClipRange ValueError) */
#define EQ4_STATUS_QUERY 4     /* pooled lookup: negative length / lengths do not sum to nidx */
#define EQ4_STATUS_INDEX 8     /* pooled lookup: a query index is out of range */

/* Version string of the library build. */
const char *eq4_version(void);

/* Thread-local description of the last error returned on this thread. */
const char *eq4_last_error(void);

/* packed.py:32-33 packed_row_stride(dim, aux_precision). */
int64_t eq4_packed_row_stride(int64_t dim, int aux);

/*
 * Fused clip-range search + quantize + pack of a whole table:
 *   packed = pack_table4(quantize_table(table, method, 4, aux, b, r))
 * replacing methods.py:63-89 quantize_table (per-row loop over
 * methods.py:43-60 row_clip_range -> clipping.py / histclip.py strategies),
 * uniform.py:142-167 quantize_table_uniform and packed.py:68-83 pack_table4.
 *   x        [rows x ld] fp32, row-major, device; only the first `dim`
 *            columns of each row are read
 *   b, r     GREEDY bins / ratio (clipping.py:142-148); HIST-BRUTE bins
 *   packed   [rows x eq4_packed_row_stride(dim, aux)] bytes, device
 * Optional per-row device outputs (NULL to skip):
 *   xmin, xmax  float64 ClipRange of the row (the reference's row_clip_range)
 *   info0       GREEDY: while-loop iterations (loss_evals = 1 + 2*iters),
 *               -1 constant row, -2 range error; HIST-BRUTE: start_bin;
 *               GSS: quant_mse evaluations (WorkCounters.loss_evals);
 *               HIST-APPRX: start_bin (info1 nbins_selected, norm the window norm)
 *   info1       GREEDY: (best_i << 16) | best_j (best_i alone for b > 65535);
 *               HIST-BRUTE: nbins_selected
 *   norm        HIST-BRUTE window norm (HistWindow.norm); unused otherwise
 *   status      device int32, EQ4_STATUS_* bits OR-ed in by the kernels
 */
int eq4_quantize_pack(const float *x, int64_t rows, int64_t dim, int64_t ld, int method, int b,
                      double r, int aux, uint8_t *packed, double *xmin, double *xmax,
                      int32_t *info0, int32_t *info1, double *norm, int32_t *status,
                      void *stream);

/*
 * eq4_quantize_pack with the method's real parameter the reference takes beside b and r:
 *   ACIQ  param = the clipping constant (clipping.py:115-134: 5.03 for the laplacian
 *         assumption, or the caller's gaussian_constant);
 *   GSS   param = tol (clipping.py:70, the bracket stops below tol * max|x|);
 *   param = 0 selects the reference default (5.03, 1e-4); other methods ignore it.
 * eq4_quantize_pack(...) == eq4_quantize_pack_p(..., param = 0, ...).
 */
int eq4_quantize_pack_p(const float *x, int64_t rows, int64_t dim, int64_t ld, int method, int b,
                        double r, double param, int aux, uint8_t *packed, double *xmin, double *xmax,
                        int32_t *info0, int32_t *info1, double *norm, int32_t *status, void *stream);

/*
 * clip_range_aciq / clip_range_gss (clipping.py:70-139) of FLOAT64 rows -- the scalar entry
 * points promote any input to float64 (clipping.py:46), which need not be float32 values.
 * Ranges only (no packing): xmin/xmax [rows] float64, info0 (optional) GSS quant_mse
 * evaluations.  method EQ4_METHOD_ACIQ or EQ4_METHOD_GSS; param as eq4_quantize_pack_p.
 * Device pointers, stream-ordered; non-finite rows set EQ4_STATUS_NONFINITE.
 */
int eq4_row_range_f64(const double *x, int64_t rows, int64_t dim, int64_t ld, int method, double param,
                      double *xmin, double *xmax, int32_t *info0, int32_t *status, void *stream);

/*
 * Same operation on HOST buffers (pinned or pageable), the call a
 * reference-side binding makes: chunks of rows are staged through device
 * memory with H2D copy / kernel / D2H copy overlapped on internal streams.
 * Synchronous; data-dependent failures return EQ4_EDATA / EQ4_ERANGE with the
 * first failing row in *bad_row and, for EQ4_ERANGE, the offending
 * (xmin, xmax) pair in bad_lohi[0..1] (both optional).  xmin/xmax/info0/
 * info1/norm are optional host arrays of length rows.  chunk_rows = 0 picks
 * a default (16 MiB of input per chunk).  The internal streams, device chunk
 * buffers and pinned status words are created on the first call per device
 * and reused (grown as needed) by later calls, which are serialised per
 * device; they stay allocated for the life of the process (do not call
 * cudaDeviceReset while the library is in use).  Pinned (page-locked) host
 * buffers give full PCIe bandwidth; pageable ones are staged by the driver.
 */
int eq4_quantize_pack_host(const float *x, int64_t rows, int64_t dim, int64_t ld, int method,
                           int b, double r, int aux, uint8_t *packed, double *xmin, double *xmax,
                           int32_t *info0, int32_t *info1, double *norm, int64_t chunk_rows,
                           int64_t *bad_row, double *bad_lohi);

/* packed.py:68-83 pack_table4 of an existing UniformQuantTable:
 * codes [rows x dim] uint8 (values 0..15), scales/biases [rows] at the aux
 * dtype (fp32 or fp16 bit patterns), all device. */
int eq4_pack(const uint8_t *codes, int64_t rows, int64_t dim, int aux, const void *scales,
             const void *biases, uint8_t *packed, void *stream);

/* packed.py:86-99 _decode_rows inverse of eq4_pack: packed -> codes,
 * scales, biases (aux-width bit patterns), all device. */
int eq4_unpack(const uint8_t *packed, int64_t rows, int64_t dim, int aux, uint8_t *codes,
               void *scales, void *biases, void *stream);

/* table.py:81-103 quant_mse per row, bit-exact float64 (numpy pairwise sum):
 * out[i] = quant_mse(x[i, :dim], ClipRange(xmin[i], xmax[i]), 4).  Device. */
int eq4_quant_mse(const float *x, int64_t rows, int64_t dim, int64_t ld, const double *xmin,
                  const double *xmax, double *out, void *stream);

/*
 * packed.py:167-177 sparse_lengths_sum_4bit: pooled lookup over packed rows.
 *   out[s, :] = sum over segment s's rows (lengths[s] consecutive entries of
 *   indices), strictly in query order from 0.0f, of the dequantized row
 *   float32(scale) * float32(code) + float32(bias) (two rounded float32 ops,
 *   packed.py:174-176; fp16 aux widened exactly), i.e. the bit-exact contract
 *   of sparse_lengths_sum_ref (packed.py:202-221).
 *   packed  [rows x eq4_packed_row_stride(dim, aux)] bytes, device
 *   indices [nidx] int64, lengths [batch] int64, out [batch x dim] fp32, device
 * Validation on the device (PooledQuery, packed.py:131-140; _check_indices,
 * packed.py:147-152): a negative length or sum(lengths) != nidx sets
 * EQ4_STATUS_QUERY and zeroes out; an out-of-range index sets
 * EQ4_STATUS_INDEX, is skipped, and the first such position is written to
 * *bad_pos (optional device int64; INT64-large when none).  Stream-ordered.
 */
int eq4_sparse_lengths_sum4(const uint8_t *packed, int64_t rows, int64_t dim, int aux,
                            const int64_t *indices, int64_t nidx, const int64_t *lengths,
                            int64_t batch, float *out, int32_t *status, int64_t *bad_pos,
                            void *stream);

/*
 * EMBT file -> EMBQ uniform4 file (fileio.py:40-70 read_embt, methods.py:63-89,
 * packed.py:68-83, fileio.py:87-101 write_embq), streamed: chunks of the EMBT
 * payload are read into pinned memory, quantized on the GPU and written as the
 * reference's EMBQ header + PackedTable4 bytes while the next chunk is read.
 * Synchronous.  EQ4_EDATA for a malformed input or non-finite values
 * (read_embt's DataError), EQ4_ERANGE with *bad_row / bad_lohi for a GREEDY
 * candidate with xmin > xmax; on failure no output file is left behind.
 * chunk_rows = 0 picks ~64 MiB of input per chunk.
 */
int eq4_quantize_file(const char *in_path, const char *out_path, int method, int b, double r,
                      int aux, int64_t chunk_rows, int64_t *bad_row, double *bad_lohi);

/* fileio.py:87-101 write_embq of a PackedTable4: the EMBQ uniform4 header then
 * the packed rows verbatim.  on_device != 0: `packed` is a device pointer and
 * is streamed out through pinned buffers (no host repack).  Synchronous. */
int eq4_write_embq(const char *path, const uint8_t *packed, int64_t rows, int64_t dim, int aux,
                   int on_device);

/* fileio.py:105-110 kmeans_row payload stride: 16 codebook values at the aux
 * width, then ceil(d/2) nibble bytes. */
int64_t eq4_kmeans_row_stride(int64_t dim, int aux);

/*
 * codebook.py:164-172 quantize_table_kmeans (row-wise 16-value codebooks,
 * k-means seeded at the row's uniform grid, codebook.py:35-137), bit-exact
 * float64.  out [rows x eq4_kmeans_row_stride(dim, aux)] receives each row's
 * sorted codebook (aux width) followed by its packed indices -- the EMBQ
 * kmeans_row payload (fileio.py:105-110).  iters (optional): Lloyd rounds
 * per row, -1 for the <= 16 distinct values shortcut.  dim <= 256.  Device
 * pointers, stream-ordered; non-finite rows set EQ4_STATUS_NONFINITE.
 */
int eq4_kmeans_rows(const float *x, int64_t rows, int64_t dim, int64_t ld, int aux, uint8_t *out,
                    int32_t *iters, int32_t *status, void *stream);

/*
 * Standalone codec and histogram entry points (device pointers, stream-ordered).
 * x_is_f64 != 0: the rows are float64 (the reference promotes any input to
 * float64, uniform.py:72 / histclip.py:56 / table.py:94); else float32.
 *
 * uniform.py:60-80 quantize_uniform per row / uniform.py:142-167
 * quantize_table_uniform: codes [rows x dim] (one byte per code, 0..2^nbits-1)
 * of each row against the float64 range (xmin[i*range_stride],
 * xmax[i*range_stride]) -- range_stride 0 applies one range to every row --
 * with scales/biases [rows] written as aux-width bit patterns.  The ranges
 * must be valid ClipRanges (finite, xmin <= xmax; table.py:70-74).  nbits 4 or 8.
 */
int eq4_quantize_rows(const void *x, int x_is_f64, int64_t rows, int64_t dim, int64_t ld,
                      const double *xmin, const double *xmax, int64_t range_stride, int nbits, int aux,
                      uint8_t *codes, void *scales, void *biases, void *stream);

/* uniform.py:83-91 dequantize_uniform: out = float32(scale) * float32(code) + float32(bias),
 * two rounded float32 operations per element. */
int eq4_dequantize_rows(const uint8_t *codes, int64_t rows, int64_t dim, const void *scales,
                        const void *biases, int aux, float *out, void *stream);

/* histclip.py:52-67 build_histogram of every row: lo/hi [rows] = np.min / np.max (numpy's
 * choice among equal extrema included), counts [rows x b] int64 (bins of width
 * (hi - lo)/b, index clip(floor((x - lo)/w), 0, b-1); a constant row puts d in bin 0). */
int eq4_build_histogram(const void *x, int x_is_f64, int64_t rows, int64_t dim, int64_t ld, int b,
                        double *lo, double *hi, int64_t *counts, void *stream);

/* histclip.py:70-82 bin_l2_norm elementwise: density * (de**3 - db**3) / 3.0 with each cube
 * rounded once (numpy's power may differ in the last bit: host SIMD pow). */
int eq4_bin_l2_norm(const double *delta_begin, const double *delta_end, const double *density,
                    int64_t n, double *out, void *stream);

/* table.py:81-103 quant_mse per row for nbits 4 or 8 and float32 or float64 rows (one
 * lane per row, numpy pairwise sum, bit-exact). */
int eq4_quant_mse_rows(const void *x, int x_is_f64, int64_t rows, int64_t dim, int64_t ld,
                       const double *xmin, const double *xmax, int nbits, double *out, void *stream);

/* Diagnostics: counters of the GREEDY kernel's rare paths on the current device,
 * accumulated over launches since the last reset: out[0] = float64 re-decisions
 * (one per row and loop iteration whose fp32 comparison fell inside the error
 * band), out[1] = rows whose codes took the float64 codec, out[2] = comparisons
 * settled by counting the elements within reach of a rounding boundary (inside
 * the band for d misrounded elements, outside the one for 2), out[3] = of those,
 * escalated to a float64 re-decision (more than 2 such elements on a side),
 * out[4] = rows the GREEDY screening kernel deferred to the exact kernel
 * (vector rows: d % 4 == 0 and 16-byte aligned).  out holds 5 entries.
 * reset != 0 zeroes them after the read.  Synchronous (device-wide). */
int eq4_diag_counters(int64_t *out, int reset);

/* Diagnostics: internal arithmetic self-test on the current device (mismatch
 * count, -1 on CUDA error).  which 0/1: the divide-free float64 w/15 used for
 * scales against the IEEE divide, on float differences / full-range doubles. */
long long eq4_selftest(int which, int64_t n, uint64_t seed);

#ifdef __cplusplus
}
#endif

#endif /* EQ4_H */
