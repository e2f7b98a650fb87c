// device_util.cuh — small device helpers shared by the kernels of this library.
#pragma once
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace lob {

__device__ __forceinline__ uint64_t bmask(int bits) { return bits >= 64 ? ~0ull : ((1ull << bits) - 1ull); }

template <typename K>
__device__ __forceinline__ constexpr K dead() { return ~K(0); }

// Moves are merged host-side (adjacent fields with the same shift delta become
// one move), so the common case has <= 4 moves: a short predicated unrolled
// loop; longer lists take a rolled loop (keeps the kernels' code small: the
// unrolled MAXM path blew join_write_k up to 17.7k SASS instructions).
__device__ __forceinline__ uint64_t apply_moves(const Move* mv, int n, uint64_t a, uint64_t b) {
  uint64_t o = 0;
  if (n <= 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < n) {
        const Move m = mv[i];
        const uint64_t s = m.src ? b : a;
        o |= ((s >> m.sshift) & ((1ull << m.bits) - 1ull)) << m.dshift;
      }
    }
    return o;
  }
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const Move m = mv[i];
    const uint64_t s = m.src ? b : a;
    o |= ((s >> m.sshift) & ((1ull << m.bits) - 1ull)) << m.dshift;
  }
  return o;
}

__device__ __forceinline__ int64_t operand_value(const Operand& o, uint64_t a, uint64_t b) {
  if (o.src == 2) return (int64_t)o.base;
  const uint64_t s = o.src ? b : a;
  return (int64_t)((s >> o.shift) & bmask(o.bits)) + (int64_t)o.base;
}

// Stale reads of slot words that other threads of the same launch update with
// atomics: relaxed loads at GPU scope, so the read and the atomics are morally
// strong and the race is defined behaviour (PTX memory model).  The value is
// any version of the word between the launch start and now — a lower bound of
// the final value, which is all the fused ⊕ needs (kernels.cuh Direct).
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

#ifndef PEEK_SLOT
#define PEEK_SLOT ld_relaxed  // A/B: -DPEEK_SLOT=__ldca (plain L1 read, formally racy)
#endif

// relation encoded as Cmp::neq: 0 ==, 1 !=, 2 <, 3 <=, 4 >, 5 >=
__device__ __forceinline__ bool cmp_holds(int rel, int64_t a, int64_t b) {
  switch (rel) {
    case 0: return a == b;
    case 1: return a != b;
    case 2: return a < b;
    case 3: return a <= b;
    case 4: return a > b;
    default: return a >= b;
  }
}

// The eval stack machine (kernels.cuh Bc): false if the program fails
// (division / remainder by zero, INT32_MIN / -1).  Fixed 8-entry stack.
__device__ __forceinline__ bool bc_eval(const Bc& b, uint64_t key, int32_t& out) {
  int32_t st[8];
  int sp = 0;
  for (int i = 0; i < b.n; ++i) {
    const BcIns in = b.ins[i];
    if (in.op == BC_FIELD) {
      st[sp++] = (int32_t)((uint32_t)((key >> in.shift) & bmask(in.bits)) + (uint32_t)in.v);
    } else if (in.op == BC_CONST) {
      st[sp++] = in.v;
    } else if (in.op == BC_NEG) {
      st[sp - 1] = (int32_t)(0u - (uint32_t)st[sp - 1]);
    } else {
      const int32_t y = st[--sp], x = st[sp - 1];
      int32_t r;
      switch (in.op) {
        case BC_ADD: r = (int32_t)((uint32_t)x + (uint32_t)y); break;
        case BC_SUB: r = (int32_t)((uint32_t)x - (uint32_t)y); break;
        case BC_MUL: r = (int32_t)((uint32_t)x * (uint32_t)y); break;
        default:
          if (y == 0 || (x == INT32_MIN && y == -1)) return false;
          r = in.op == BC_DIV ? x / y : x % y;
      }
      st[sp - 1] = r;
    }
  }
  out = st[0];
  return true;
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

// max-min direct-store word: fp32 bits of p (p >= 0: order-preserving) + 1, 0 =
// absent.  No settled bit: an equal p is never an improvement (no witness to
// tie-break), so a slot is only rewritten when p strictly grows.
__device__ __forceinline__ uint32_t mm_word(float p) { return f2u(p) + 1u; }
__device__ __forceinline__ float mm_p(uint32_t v) { return u2f(v - 1u); }

// max-mult direct-store word (kernels.cuh MxEnc)
__device__ __forceinline__ unsigned long long mx_word(float p, uint32_t w, const MxEnc& e) {
  return ((unsigned long long)(f2u(p) + 1u) << 34) | e.stamp | ((unsigned long long)(~w) & e.wmask);
}
__device__ __forceinline__ float mx_p(unsigned long long v) { return u2f((uint32_t)(v >> 34) - 1u); }

// ⊗: one IEEE fp32 op, no contraction (reading 9)
__device__ __forceinline__ float otimes(int semi, float a, float b) {
  if (semi == S_MAXMIN) return a < b ? a : b;
  return __fmul_rn(a, b);
}

// Direct ⊕ of one live candidate into a dense store (see kernels.cuh Direct).
// Called by the threads that hold a live candidate (any divergence).  With
// `aggregate` (narrow heads, e.g. endpoints_connected() sends ~1M candidates
// to each of 64 slots) lanes of a warp aiming at the same slot are pre-reduced
// (match + shuffle tree) so one atomic per (warp, slot) reaches L2.
__device__ __forceinline__ void direct_oplus(int semi, void* f, uint32_t slot, float p, uint32_t w, uint32_t* dirty,
                                             int aggregate, const MxEnc& mx) {
  namespace cg = cooperative_groups;
  bool app = false;
  if (semi == S_UNIT) {
    const uint32_t bit = 1u << (slot & 31u);
    const uint32_t old = atomicOr(reinterpret_cast<uint32_t*>(f) + (slot >> 5), bit);
    app = !(old & bit);
  } else if (semi == S_MAXMIN) {
    uint32_t v = mm_word(p);
    bool lead = true;
    if (aggregate) {
      cg::coalesced_group part = cg::labeled_partition(cg::coalesced_threads(), (int)slot);
      v = cg::reduce(part, v, cg::greater<uint32_t>());
      lead = part.thread_rank() == 0;
    }
    if (lead) {
      const uint32_t old = atomicMax(reinterpret_cast<uint32_t*>(f) + slot, v);
      app = old < v;  // any improvement marks the slot (idempotent OR)
    }
  } else {
    unsigned long long v = mx_word(p, w, mx);
    bool lead = true;
    if (aggregate) {
      cg::coalesced_group part = cg::labeled_partition(cg::coalesced_threads(), (int)slot);
      v = cg::reduce(part, v, cg::greater<unsigned long long>());
      lead = part.thread_rank() == 0;
    }
    if (lead) {
      const unsigned long long old = atomicMax(reinterpret_cast<unsigned long long*>(f) + slot, v);
      app = old < v;
    }
  }
  if (app) atomicOr(dirty + (slot >> 5), 1u << (slot & 31u));
}

// Batched direct ⊕ for a thread's independent candidates (no pre-reduction).
// direct_pack: the candidate's value in the store's packed word (unit: the bit
// within its 32-bit bitmap word).  direct_peek: a plain L2 read of the word —
// the store only grows (atomicMax / OR), so a stale read is a lower bound and
// a candidate not above it can never improve the slot.  direct_commit issues
// the remaining updates and dirty bits as fire-and-forget reductions.
__device__ __forceinline__ unsigned long long direct_pack(int semi, uint32_t slot, float t, uint32_t w,
                                                          const MxEnc& mx) {
  if (semi == S_UNIT) return 1ull << (slot & 31u);
  if (semi == S_MAXMIN) return (unsigned long long)mm_word(t);
  return mx_word(t, w, mx);
}

__device__ __forceinline__ unsigned long long direct_peek(int semi, const void* f, uint32_t slot) {
  // through L1 (ld.ca): L1 holds no line from before this launch, so a hit is
  // still a lower bound of the slot's round-start value
  if (semi == S_UNIT) return PEEK_SLOT(reinterpret_cast<const uint32_t*>(f) + (slot >> 5));
  if (semi == S_MAXMIN) return PEEK_SLOT(reinterpret_cast<const uint32_t*>(f) + slot);
  return PEEK_SLOT(reinterpret_cast<const unsigned long long*>(f) + slot);
}

template <int N>
__device__ __forceinline__ void direct_commit(int semi, void* f, uint32_t* dirty, const uint32_t* slotv,
                                              const unsigned long long* newv, const unsigned long long* oldv,
                                              const bool* live) {
  // v > the (stale) read >= the slot's round-start value: the slot ends the
  // round strictly above its settled value, so it is in Δ' — RED the value and
  // the dirty bit without waiting for the atomic's old value.
#pragma unroll
  for (int d = 0; d < N; ++d) {
    if (!live[d]) continue;
    const unsigned long long v = newv[d];
    if (semi == S_UNIT) {
      if (oldv[d] & v) continue;
      atomicOr(reinterpret_cast<uint32_t*>(f) + (slotv[d] >> 5), (uint32_t)v);
    } else if (semi == S_MAXMIN) {
      if (v <= oldv[d]) continue;
      atomicMax(reinterpret_cast<uint32_t*>(f) + slotv[d], (uint32_t)v);
    } else {
      if (v <= oldv[d]) continue;
      atomicMax(reinterpret_cast<unsigned long long*>(f) + slotv[d], v);
    }
    atomicOr(dirty + (slotv[d] >> 5), 1u << (slotv[d] & 31u));
  }
}

// Per-CTA candidate count -> one global atomic per CTA (blockDim <= 1024, every
// thread of the CTA calls it at the end of the kernel).  Per-warp atomics on
// the single counter (~6k per fused-join launch) serialised in L2 at the tail.
__device__ __forceinline__ void cta_count_add(unsigned long long* ctr, uint32_t mine) {
  __shared__ uint32_t s_cnt[32];
  mine = __reduce_add_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_cnt[w];
    if (t) atomicAdd(ctr, t);
  }
}

inline int grid_for(int64_t n, int threads, int cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace lob
