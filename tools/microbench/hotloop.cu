// Throughput of the GREEDY hot loop alone (eval_pair_x2 over a 32-slot row
// slice in shared memory), to separate the FMA-pipe bound from the rest.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk2(float a, float b) { f2_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk2(f2_t v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) { f2_t r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) { f2_t r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ f2_t fma2_rm(f2_t a, f2_t b, f2_t c) { f2_t r; asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float sat_fma(float a, float b, float c) { float r; asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
constexpr float ALPHA = 15.75f, MAGIC = 8388608.f;

template <int MODE>
__global__ void __launch_bounds__(128, 4) k(float* out, int iters) {
  __shared__ float4 ys[8 * 32 * 4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* ys4 = ys + warp * 256;
  for (int c = 0; c < 8; c++) ys4[c * 32 + lane] = make_float4(lane * 3.1f + c, lane * 7.7f + c * 11, 1000.f + lane, 2000.f - c * lane);
  __syncwarp();
  float accs = 0.f;
  for (int it = 0; it < iters; it++) {
    const float Wf = 199.f - (it & 31), BL = 15.f * (it & 7);
    const float kW = 1.f / (Wf * ALPHA), h = 0.5f / ALPHA, nW = -Wf;
    const f2_t nBL2 = pk2(-BL, -BL), c15 = pk2(15.f, 15.f), al2 = pk2(ALPHA, ALPHA);
    const f2_t mg2 = pk2(MAGIC, MAGIC), nmg2 = pk2(-MAGIC, -MAGIC), nW2 = pk2(nW, nW);
    f2_t sL = pk2(0.f, 0.f), sR = pk2(0.f, 0.f);
#pragma unroll 4
    for (int c = 0; c < 8; ++c) {
      const ulonglong2 yy = *reinterpret_cast<const ulonglong2*>(ys4 + c * 32 + lane);
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        const f2_t y2 = hlf ? yy.y : yy.x;
        const f2_t zL = add2(y2, nBL2);
        const f2_t zR = add2(zL, c15);
        float a0, a1, b0, b1; upk2(zL, a0, a1); upk2(zR, b0, b1);
        const f2_t tL = pk2(sat_fma(a0, kW, h), sat_fma(a1, kW, h));
        const f2_t tR = pk2(sat_fma(b0, kW, h), sat_fma(b1, kW, h));
        const f2_t cL = add2(fma2_rm(tL, al2, mg2), nmg2);
        const f2_t cR = add2(fma2_rm(tR, al2, mg2), nmg2);
        f2_t eL, eR;
        if (MODE == 2) { eL = fma2(cL, pk2(-199.f, -199.f), zL); eR = fma2(cR, pk2(-199.f, -199.f), zR); }
        else if (MODE == 3) { eL = add2(zL, cL); eR = add2(zR, cR); }
        else { eL = fma2(cL, nW2, zL); eR = fma2(cR, nW2, zR); }
        sL = fma2(eL, eL, sL);
        sR = fma2(eR, eR, sR);
      }
    }
    float l0, l1, r0, r1; upk2(sL, l0, l1); upk2(sR, r0, r1);
    float SL = l0 + l1, SR = r0 + r1;
    if (MODE == 1) { SL += __shfl_xor_sync(0xffffffff, SL, 1); SR += __shfl_xor_sync(0xffffffff, SR, 1); }
    accs += (SL < SR) ? SL : SR;
  }
  if (accs == 1234.5f) out[0] = accs;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096;
  for (int mode = 0; mode < 4; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 4, 128>>>(d, iters); else if (mode == 1) k<1><<<148 * 4, 128>>>(d, iters);
      else if (mode == 2) k<2><<<148 * 4, 128>>>(d, iters); else k<3><<<148 * 4, 128>>>(d, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double evals = 148.0 * 4 * 128 * (double)iters * 32 * 2;   // element-candidate evals
      if (rep) printf("mode %d: %.3f ms  %.2f elem-cand evals/clk/SM (1.965 GHz); FMA bound 21.3\n", mode, ms, evals / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
