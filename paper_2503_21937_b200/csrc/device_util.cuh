// device_util.cuh — small device helpers shared by the kernels of this library.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace lob {

__device__ __forceinline__ uint64_t bmask(int bits) { return bits >= 64 ? ~0ull : ((1ull << bits) - 1ull); }

__device__ __forceinline__ uint64_t apply_moves(const Move* mv, int n, uint64_t a, uint64_t b) {
  uint64_t o = 0;
#pragma unroll
  for (int i = 0; i < MAXM; ++i) {
    if (i < n) {
      const Move m = mv[i];
      const uint64_t s = m.src ? b : a;
      o |= ((s >> m.sshift) & bmask(m.bits)) << m.dshift;
    }
  }
  return o;
}

__device__ __forceinline__ int64_t operand_value(const Operand& o, uint64_t a, uint64_t b) {
  if (o.src == 2) return (int64_t)o.base;
  const uint64_t s = o.src ? b : a;
  return (int64_t)((s >> o.shift) & bmask(o.bits)) + (int64_t)o.base;
}

// first index in [0, n) with key[idx] >= x (n if none)
__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* __restrict__ key, int64_t n, uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(key + mid) < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// largest i in [0, n) with a[i] <= x  (a non-decreasing, a[0] <= x)
__device__ __forceinline__ int64_t upper_bound_m1_i64(const int64_t* __restrict__ a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) <= x) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

__device__ __forceinline__ float u2f(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }

// ⊗: one IEEE fp32 op, no contraction (reading 9)
__device__ __forceinline__ float otimes(int semi, float a, float b) {
  if (semi == S_MAXMIN) return a < b ? a : b;
  return __fmul_rn(a, b);
}

inline int grid_for(int64_t n, int threads, int cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace lob
