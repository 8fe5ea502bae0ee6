// eq4_io.cu -- EMBT -> EMBQ (uniform4) streaming pipeline and the device-side
// EMBQ writer (reference fileio.py:40-127).
//
// EMBT: "<4sIQQB" header (magic "EMBT", version 1, rows u64, dim u64, dtype 0)
// followed by rows x dim little-endian fp32 (fileio.py:40-70).
// EMBQ uniform4: "<4sIBBQQ" header (magic "EMBQ", version 1, scheme 0, aux
// code, rows u64, dim u64) followed by the PackedTable4 bytes verbatim
// (fileio.py:87-101).
//
// quantize_file: the table never exists whole in host or device memory.  A
// host loop reads chunk c of the EMBT payload straight into a pinned buffer
// while the GPU (one stream per buffer pair) runs H2D copy -> fused
// search/quantize/pack kernel -> D2H copy of chunk c-1, and the packed bytes
// of chunk c-2 go to the EMBQ file -- disk read, PCIe both ways, the kernel
// and the disk write all overlap.  Header validation (with the reference's
// DataError texts) is done by the Python layer before this is called; here
// the header is re-checked for consistency only.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/eq4.h"
#include "eq4_internal.h"

namespace {

constexpr size_t EMBT_HEADER = 25;   // struct "<4sIQQB"
constexpr size_t EMBQ_HEADER = 26;   // struct "<4sIBBQQ"

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

bool read_full(int fd, void* buf, size_t n, off_t off) {
  uint8_t* p = static_cast<uint8_t*>(buf);
  while (n) {
    const ssize_t k = pread(fd, p, n, off);
    if (k <= 0) {
      if (k < 0 && errno == EINTR) continue;
      return false;
    }
    p += k; n -= (size_t)k; off += k;
  }
  return true;
}

// pread of a large span split across threads: a single copying thread reads the
// page cache at ~5 GB/s, far below PCIe; 8-16 threads keep the pipeline on the GPU side
bool read_parallel(int fd, void* buf, size_t n, off_t off) {
  constexpr size_t SLICE = 8u << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>(std::min<size_t>(hw, 16), (n + SLICE - 1) / SLICE);
  if (nt <= 1) return read_full(fd, buf, n, off);
  std::vector<std::thread> th;
  std::vector<char> ok(nt, 1);
  const size_t per = (n + nt - 1) / nt;
  for (size_t t = 0; t < nt; t++) {
    const size_t a = t * per, len = a >= n ? 0 : std::min(per, n - a);
    th.emplace_back([&, t, a, len] {
      ok[t] = read_full(fd, static_cast<uint8_t*>(buf) + a, len, off + (off_t)a) ? 1 : 0;
    });
  }
  bool good = true;
  for (size_t t = 0; t < nt; t++) {
    th[t].join();
    good = good && ok[t];
  }
  return good;
}

bool write_full(int fd, const void* buf, size_t n) {
  const uint8_t* p = static_cast<const uint8_t*>(buf);
  while (n) {
    const ssize_t k = write(fd, p, n);
    if (k <= 0) {
      if (k < 0 && errno == EINTR) continue;
      return false;
    }
    p += k; n -= (size_t)k;
  }
  return true;
}

void embq_header(uint8_t* h, int aux, int64_t rows, int64_t dim) {
  memcpy(h, "EMBQ", 4);
  const uint32_t version = 1;
  memcpy(h + 4, &version, 4);
  h[8] = 0;                                        // scheme uniform4 (fileio.py:29)
  h[9] = aux == EQ4_AUX_FP16 ? 1 : 0;              // aux code (fileio.py:31)
  const uint64_t r = (uint64_t)rows, d = (uint64_t)dim;
  memcpy(h + 10, &r, 8);
  memcpy(h + 18, &d, 8);
}

std::string sys_err(const char* what, const char* path) {
  return std::string(what) + " " + path + ": " + strerror(errno);
}

}  // namespace

int eq4_io_quantize_file(const char* in_path, const char* out_path, int method, int b, double r,
                         int aux, int64_t chunk_rows, int64_t* bad_row, double* bad_lohi,
                         std::string& err) {
  Fd in;
  in.fd = open(in_path, O_RDONLY);
  if (in.fd < 0) { err = sys_err("cannot open", in_path); return EQ4_EINVAL; }
  uint8_t h[EMBT_HEADER];
  if (!read_full(in.fd, h, EMBT_HEADER, 0) || memcmp(h, "EMBT", 4) != 0) {
    err = std::string(in_path) + ": not an EMBT file";
    return EQ4_EDATA;
  }
  uint32_t version;
  uint64_t rows_u, dim_u;
  memcpy(&version, h + 4, 4);
  memcpy(&rows_u, h + 8, 8);
  memcpy(&dim_u, h + 16, 8);
  if (version != 1 || h[24] != 0 || rows_u < 1 || dim_u < 1) {
    err = std::string(in_path) + ": unsupported EMBT header";
    return EQ4_EDATA;
  }
  const int64_t rows = (int64_t)rows_u, dim = (int64_t)dim_u;
  const off_t size = lseek(in.fd, 0, SEEK_END);
  if (size != (off_t)(EMBT_HEADER + (uint64_t)rows * dim * 4)) {
    err = std::string(in_path) + ": payload size does not match the header";
    return EQ4_EDATA;
  }
  const int64_t stride = eq4_packed_row_stride(dim, aux);
  int64_t chunk = chunk_rows > 0 ? chunk_rows : std::max<int64_t>(1024, (64ll << 20) / (dim * 4));
  chunk = std::min(chunk, rows);
  const int64_t nchunks = (rows + chunk - 1) / chunk;

  Fd out;
  out.fd = open(out_path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (out.fd < 0) { err = sys_err("cannot create", out_path); return EQ4_EINVAL; }
  uint8_t qh[EMBQ_HEADER];
  embq_header(qh, aux, rows, dim);
  if (!write_full(out.fd, qh, EMBQ_HEADER)) { err = sys_err("write", out_path); return EQ4_EINVAL; }

  constexpr int NS = 2;
  cudaStream_t st[NS] = {nullptr, nullptr};
  float* hin[NS] = {nullptr, nullptr};
  uint8_t* hout[NS] = {nullptr, nullptr};
  float* dx[NS] = {nullptr, nullptr};
  uint8_t* dq[NS] = {nullptr, nullptr};
  int32_t* dst[NS] = {nullptr, nullptr};
  int32_t* di0[NS] = {nullptr, nullptr};
  int32_t* hstatus = nullptr;
  int rc = EQ4_OK;
  auto cuda_check = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == EQ4_OK) {
      err = std::string(what) + ": " + cudaGetErrorString(e);
      rc = EQ4_ECUDA;
    }
    return rc == EQ4_OK;
  };
  cuda_check(cudaMallocHost(&hstatus, sizeof(int32_t) * nchunks), "cudaMallocHost");
  for (int i = 0; i < NS && rc == EQ4_OK; i++) {
    cuda_check(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking), "stream");
    cuda_check(cudaMallocHost(&hin[i], chunk * dim * 4), "cudaMallocHost");
    cuda_check(cudaMallocHost(&hout[i], chunk * stride), "cudaMallocHost");
    cuda_check(cudaMalloc(&dx[i], chunk * dim * 4), "cudaMalloc");
    cuda_check(cudaMalloc(&dq[i], chunk * stride), "cudaMalloc");
    cuda_check(cudaMalloc(&dst[i], 4), "cudaMalloc");
    cuda_check(cudaMalloc(&di0[i], chunk * 4), "cudaMalloc");
  }
  // TABLE (clipping.py:64-67): one range over the whole file -> a first streaming pass
  int* tkeys = nullptr;
  if (rc == EQ4_OK && method == EQ4_METHOD_TABLE) {
    cuda_check(cudaMalloc(&tkeys, 8), "cudaMalloc");
    if (rc == EQ4_OK) rc = eq4_internal_table_init(tkeys, st[0]);
    for (int64_t c = 0; c < nchunks && rc == EQ4_OK; c++) {
      const int i = (int)(c % NS);
      if (!cuda_check(cudaStreamSynchronize(st[i]), "stream sync")) break;   // hin[i] free again
      const int64_t r0 = c * chunk, nr = std::min(chunk, rows - r0);
      if (!read_parallel(in.fd, hin[i], (size_t)(nr * dim * 4), (off_t)(EMBT_HEADER + r0 * dim * 4))) {
        err = sys_err("read", in_path);
        rc = EQ4_EINVAL;
        break;
      }
      if (!cuda_check(cudaMemcpyAsync(dx[i], hin[i], nr * dim * 4, cudaMemcpyHostToDevice, st[i]), "H2D"))
        break;
      if (i != 0 && !cuda_check(cudaStreamSynchronize(st[0]), "stream sync")) break;  // keys init
      rc = eq4_internal_table_accumulate(dx[i], nr, dim, tkeys, st[i]);
    }
    for (int i = 0; i < NS && rc == EQ4_OK; i++) cuda_check(cudaStreamSynchronize(st[i]), "stream sync");
  }
  // c: read + enqueue chunk c; before reusing buffer pair c % NS, drain chunk c - NS
  int64_t pending[NS] = {-1, -1};
  auto drain = [&](int i) {
    if (pending[i] < 0 || rc != EQ4_OK) return;
    if (!cuda_check(cudaStreamSynchronize(st[i]), "stream sync")) return;
    const int64_t c = pending[i];
    const int64_t nr = std::min(chunk, rows - c * chunk);
    if (!write_full(out.fd, hout[i], (size_t)(nr * stride)) && rc == EQ4_OK) {
      err = sys_err("write", out_path);
      rc = EQ4_EINVAL;
    }
    pending[i] = -1;
  };
  for (int64_t c = 0; c < nchunks && rc == EQ4_OK; c++) {
    const int i = (int)(c % NS);
    drain(i);
    if (rc != EQ4_OK) break;
    const int64_t r0 = c * chunk, nr = std::min(chunk, rows - r0);
    if (!read_parallel(in.fd, hin[i], (size_t)(nr * dim * 4), (off_t)(EMBT_HEADER + r0 * dim * 4))) {
      err = sys_err("read", in_path);
      rc = EQ4_EINVAL;
      break;
    }
    if (!cuda_check(cudaMemcpyAsync(dx[i], hin[i], nr * dim * 4, cudaMemcpyHostToDevice, st[i]), "H2D"))
      break;
    if (!cuda_check(cudaMemsetAsync(dst[i], 0, 4, st[i]), "memset")) break;
    const int krc = eq4_internal_quantize_pack_keys(dx[i], nr, dim, method, b, r, aux, dq[i], di0[i],
                                                    dst[i], st[i], tkeys);
    if (krc != EQ4_OK) {
      err = eq4_last_error();
      rc = krc;
      break;
    }
    if (!cuda_check(cudaMemcpyAsync(hout[i], dq[i], nr * stride, cudaMemcpyDeviceToHost, st[i]), "D2H"))
      break;
    if (!cuda_check(cudaMemcpyAsync(hstatus + c, dst[i], 4, cudaMemcpyDeviceToHost, st[i]), "D2H"))
      break;
    pending[i] = c;
  }
  for (int64_t k = 0; k < NS; k++) drain((int)((nchunks + k) % NS));
  for (int i = 0; i < NS; i++)
    if (st[i]) cudaStreamSynchronize(st[i]);
  // data-dependent failures, first failing row first (like the reference's row loop)
  if (rc == EQ4_OK) {
    for (int64_t c = 0; c < nchunks; c++) {
      if (!hstatus[c]) continue;
      if (hstatus[c] & EQ4_STATUS_NONFINITE) {
        // read_embt rejects the whole file (fileio.py:68-69) before quantizing
        err = std::string(in_path) + ": payload contains non-finite values";
        rc = EQ4_EDATA;
      } else {
        // a GREEDY candidate with xmin > xmax: locate the row by re-running the chunk
        const int64_t r0 = c * chunk, nr = std::min(chunk, rows - r0);
        double *dlo = nullptr, *dhi = nullptr;
        int64_t found = -1;
        double lohi[2] = {0.0, 0.0};
        if (read_full(in.fd, hin[0], (size_t)(nr * dim * 4), (off_t)(EMBT_HEADER + r0 * dim * 4)) &&
            cudaMalloc(&dlo, nr * 8) == cudaSuccess && cudaMalloc(&dhi, nr * 8) == cudaSuccess &&
            cudaMemcpy(dx[0], hin[0], nr * dim * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
            eq4_quantize_pack(dx[0], nr, dim, dim, method, b, r, aux, dq[0], dlo, dhi, di0[0],
                              nullptr, nullptr, nullptr, st[0]) == EQ4_OK &&
            cudaStreamSynchronize(st[0]) == cudaSuccess) {
          int32_t* hi0 = reinterpret_cast<int32_t*>(hout[0]);   // reuse (>= nr * 4 bytes)
          cudaMemcpy(hi0, di0[0], nr * 4, cudaMemcpyDeviceToHost);
          for (int64_t k = 0; k < nr; k++)
            if (hi0[k] == -2) { found = k; break; }
          if (found >= 0) {
            cudaMemcpy(&lohi[0], dlo + found, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&lohi[1], dhi + found, 8, cudaMemcpyDeviceToHost);
          }
        }
        if (dlo) cudaFree(dlo);
        if (dhi) cudaFree(dhi);
        if (bad_row) *bad_row = found >= 0 ? r0 + found : -1;
        if (bad_lohi) { bad_lohi[0] = lohi[0]; bad_lohi[1] = lohi[1]; }
        err = "xmin " + py_float_repr(lohi[0]) + " exceeds xmax " + py_float_repr(lohi[1]);
        rc = EQ4_ERANGE;
      }
      break;
    }
  }
  for (int i = 0; i < NS; i++) {
    if (hin[i]) cudaFreeHost(hin[i]);
    if (hout[i]) cudaFreeHost(hout[i]);
    if (dx[i]) cudaFree(dx[i]);
    if (dq[i]) cudaFree(dq[i]);
    if (dst[i]) cudaFree(dst[i]);
    if (di0[i]) cudaFree(di0[i]);
    if (st[i]) cudaStreamDestroy(st[i]);
  }
  if (hstatus) cudaFreeHost(hstatus);
  if (tkeys) cudaFree(tkeys);
  if (rc != EQ4_OK) unlink(out_path);   // no partial container on failure
  return rc;
}

int eq4_io_write_embq(const char* path, const uint8_t* packed, int64_t rows, int64_t dim, int aux,
                      int on_device, std::string& err) {
  const int64_t stride = eq4_packed_row_stride(dim, aux);
  Fd out;
  out.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (out.fd < 0) { err = sys_err("cannot create", path); return EQ4_EINVAL; }
  uint8_t qh[EMBQ_HEADER];
  embq_header(qh, aux, rows, dim);
  if (!write_full(out.fd, qh, EMBQ_HEADER)) { err = sys_err("write", path); return EQ4_EINVAL; }
  if (!on_device) {
    if (!write_full(out.fd, packed, (size_t)(rows * stride))) { err = sys_err("write", path); return EQ4_EINVAL; }
    return EQ4_OK;
  }
  // device buffer: 64 MiB D2H chunks into two pinned buffers, the write of one
  // overlapping the copy of the next
  const size_t total = (size_t)(rows * stride);
  const size_t cb = std::min<size_t>(total, 64u << 20);
  uint8_t* hb[2] = {nullptr, nullptr};
  cudaStream_t st[2] = {nullptr, nullptr};
  int rc = EQ4_OK;
  for (int i = 0; i < 2 && rc == EQ4_OK; i++) {
    if (cudaMallocHost(&hb[i], cb) != cudaSuccess || cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking) != cudaSuccess) {
      err = "cudaMallocHost/stream";
      rc = EQ4_ECUDA;
    }
  }
  size_t off = 0;
  int k = 0;
  size_t inflight[2] = {0, 0};
  while (rc == EQ4_OK && (off < total || inflight[0] || inflight[1])) {
    const int i = k & 1;
    if (inflight[i]) {
      if (cudaStreamSynchronize(st[i]) != cudaSuccess) { err = "D2H"; rc = EQ4_ECUDA; break; }
      if (!write_full(out.fd, hb[i], inflight[i])) { err = sys_err("write", path); rc = EQ4_EINVAL; break; }
      inflight[i] = 0;
    }
    if (off < total) {
      const size_t n = std::min(cb, total - off);
      if (cudaMemcpyAsync(hb[i], packed + off, n, cudaMemcpyDeviceToHost, st[i]) != cudaSuccess) {
        err = "D2H";
        rc = EQ4_ECUDA;
        break;
      }
      inflight[i] = n;
      off += n;
    }
    k++;
  }
  for (int i = 0; i < 2; i++) {
    if (st[i]) { cudaStreamSynchronize(st[i]); cudaStreamDestroy(st[i]); }
    if (hb[i]) cudaFreeHost(hb[i]);
  }
  if (rc != EQ4_OK) unlink(path);
  return rc;
}
