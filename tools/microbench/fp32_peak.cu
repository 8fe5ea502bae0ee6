// Measured FP32 FMA throughput of the whole GPU (the GREEDY roofline denominator):
// scalar FFMA and packed FFMA2 (fma.rn.f32x2), 8 independent chains per thread, every SM
// busy (148 x 8 blocks of 256 threads).  Prints JSON: TFLOP/s counting 2 FLOP per FMA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp32_peak fp32_peak.cu && ./fp32_peak
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 8192
#define CH 8

__global__ void k_ffma(float* out, float a) {
  float v[CH], w[CH];
  for (int i = 0; i < CH; i++) { v[i] = threadIdx.x * 1e-3f + i; w[i] = 0.999f - i * 1e-4f; }
  for (int it = 0; it < N_IT; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) v[i] = __fmaf_rn(v[i], w[i], a);
  }
  float s = 0.f;
  for (int i = 0; i < CH; i++) s += v[i];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a) {
  unsigned long long v[CH], w[CH], c;
  asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(a));
  for (int i = 0; i < CH; i++) {
    const float x = threadIdx.x * 1e-3f + i, y = 0.999f - i * 1e-4f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(v[i]) : "f"(x), "f"(x + 1.f));
    asm("mov.b64 %0, {%1, %2};" : "=l"(w[i]) : "f"(y), "f"(y));
  }
  for (int it = 0; it < N_IT; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[i]) : "l"(w[i]), "l"(c));
  }
  float s = 0.f;
  for (int i = 0; i < CH; i++) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v[i]));
    s += x + y;
  }
  if (s == 1234.5f) out[0] = s;
}

template <class K>
static double run(K kern, int lanes_per_fma, float* out, int sms) {
  const int blocks = sms * 8, threads = 256;
  kern<<<blocks, threads>>>(out, 0.5f);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, 0.5f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)blocks * threads * N_IT * CH * lanes_per_fma;
    const double tflops = 2.0 * fmas / (ms * 1e-3) / 1e12;
    if (tflops > best) best = tflops;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4);
  const double ffma = run(k_ffma, 1, out, sms);
  const double ffma2 = run(k_ffma2, 2, out, sms);
  printf("{\"ffma_tflops\": %.3f, \"ffma2_tflops\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d, "
         "\"derived_tflops_at_attr_clock\": %.3f}\n",
         ffma, ffma2, sms, clk, sms * 128 * 2.0 * clk * 1e3 / 1e12);
  return 0;
}
