// eq4_np.cuh -- numpy's pairwise float64 summation replayed by ONE thread
// (numpy/_core/src/umath/loops_utils.h.src @TYPE@_pairwise_sum: 8 accumulator
// chains per <= 128-element leaf, the fixed ((r0+r1)+(r2+r3))+... tree, the
// remainder, and n2 = n/2 - (n/2 % 8) halving above 128), for the lane-per-row
// kernels (ACIQ/GSS, the codec and histogram helpers).  Every add is an
// explicitly rounded __dadd_rn, so results are bit-identical to np.sum.
#pragma once
#include <cuda_runtime.h>

namespace eq4 {

// numpy pairwise summation of f(a .. a+n-1) (loops_utils.h.src), one thread.
template <class F>
__device__ __forceinline__ double np_leaf(const F& f, int a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res = __dadd_rn(res, f(a + i));
    return res;
  }
  double r0 = f(a), r1 = f(a + 1), r2 = f(a + 2), r3 = f(a + 3);
  double r4 = f(a + 4), r5 = f(a + 5), r6 = f(a + 6), r7 = f(a + 7);
  const int nf = n - (n % 8);
  int i = 8;
  for (; i < nf; i += 8) {
    r0 = __dadd_rn(r0, f(a + i));     r1 = __dadd_rn(r1, f(a + i + 1));
    r2 = __dadd_rn(r2, f(a + i + 2)); r3 = __dadd_rn(r3, f(a + i + 3));
    r4 = __dadd_rn(r4, f(a + i + 4)); r5 = __dadd_rn(r5, f(a + i + 5));
    r6 = __dadd_rn(r6, f(a + i + 6)); r7 = __dadd_rn(r7, f(a + i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; i++) res = __dadd_rn(res, f(a + i));
  return res;
}

// pw(a, n) = pw(a, n2) + pw(a + n2, n - n2) for n > 128, n2 = n/2 - (n/2 % 8),
// evaluated with an explicit stack (leaves left to right, the same association).
template <class F>
__device__ __forceinline__ double np_pw(const F& f, int a0, int n0) {
  if (n0 <= 128) return np_leaf(f, a0, n0);
  int sa[24], sn[24], sstage[24];
  double sleft[24];
  int sp = 0;
  sa[0] = a0; sn[0] = n0; sstage[0] = 0;
  double ret = 0.0;
  while (true) {
    const int a = sa[sp], n = sn[sp];
    if (n <= 128) {
      ret = np_leaf(f, a, n);
      // return up the stack until a node still needs its right half
      while (true) {
        if (sp == 0) return ret;
        --sp;
        if (sstage[sp] == 1) {
          sleft[sp] = ret;
          sstage[sp] = 2;
          int n2 = sn[sp] / 2;
          n2 -= n2 % 8;
          ++sp;
          sa[sp] = sa[sp - 1] + n2; sn[sp] = sn[sp - 1] - n2; sstage[sp] = 0;
          break;
        }
        ret = __dadd_rn(sleft[sp], ret);
      }
    } else {
      int n2 = n / 2;
      n2 -= n2 % 8;
      sstage[sp] = 1;
      ++sp;
      sa[sp] = a; sn[sp] = n2; sstage[sp] = 0;
    }
  }
}

// np.add.reduce: identity 0.0 plus the pairwise sum.
template <class F>
__device__ __forceinline__ double np_sum(const F& f, int n) {
  return __dadd_rn(0.0, np_pw(f, 0, n));
}

}  // namespace eq4
