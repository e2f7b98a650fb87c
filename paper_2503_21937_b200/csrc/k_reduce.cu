// k_reduce.cu — ingest (A0), segmented ⊕ dedup (A7), diff / apply / merge into
// the relation (A8) and the change count that ends the fixpoint (A9).
//
//   unique⟨σ⟩  PAPER.md:364 (Table 1), :1297 (Fig. 10 Stratum)  -> seg_reduce
//   merge      PAPER.md:365, :1294                             -> merge
//   promote    PAPER.md:606-609 (§3.4)                         -> diff + apply
// Semantics (SURVEY §8(c) points 1, 5, 8, 9): Δ' = {(t,b) in U : t not in F or
// bits(F[t] ⊕ b) != bits(F[t])}; ⊕ within a round in canonical (sorted) order:
// add-mult accumulates in fp64 and rounds once; max-mult keeps the larger p and,
// on equal p, the smaller witness (rule, non-head variables); across rounds a
// tie keeps the existing tag.
//
// Two relation stores: sorted (keys + SoA tags, merged each round) and dense
// (a direct-mapped tag array over the packed-key domain,
// so A8 is an O(|U|) in-place update instead of an O(|F|) merge).
#include <cstdlib>

#include "device_util.cuh"

namespace lob {
namespace {

// ---------------------------------------------------------------- ingest ----
__global__ void minmax_k(const int32_t* __restrict__ col, int64_t n, int32_t* __restrict__ out2) {
  int32_t lo = INT32_MAX, hi = INT32_MIN;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = col[i];
    lo = min(lo, v);
    hi = max(hi, v);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out2, lo);
    atomicMax(out2 + 1, hi);
  }
}

__global__ void pack_k(const PackPlan pp, int64_t n, uint64_t* __restrict__ key, uint32_t* __restrict__ rowid) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = 0ull;
    bool live = true;
    if (pp.sample) {
      const int32_t s = pp.sample[i];
      live = s >= pp.s_lo && s < pp.s_hi;
      k = (uint64_t)(uint32_t)(s - pp.s_lo) << pp.sshift;
    }
    for (int c = 0; c < pp.ncols; ++c) k |= (uint64_t)(uint32_t)(pp.col[c][i] - pp.min[c]) << pp.shift[c];
    key[i] = live ? k : KEY_DEAD;
    rowid[i] = (uint32_t)i;
  }
}

__global__ void gather_f32_k(const float* __restrict__ s, const uint32_t* __restrict__ idx, float* __restrict__ d,
                             int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[idx[i]];
}
__global__ void gather_i32_k(const int32_t* __restrict__ s, const uint32_t* __restrict__ idx,
                             int32_t* __restrict__ d, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[idx[i]];
}
__global__ void iota_k(int32_t* d, int64_t n, int32_t first) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = first + (int32_t)i;
}
__global__ void fill_k(float* d, int64_t n, float v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = v;
}
__global__ void validate_k(const float* __restrict__ p, const int32_t* __restrict__ s, int64_t n, int32_t batch,
                           uint32_t* flags) {
  uint32_t f = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (p) {
      const float x = p[i];
      if (!(x >= 0.0f && x <= 1.0f)) f |= 1u;
    }
    if (s) {
      const int32_t v = s[i];
      if (v < 0 || v >= batch) f |= 2u;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// -------------------------------------------------------- heads / dedup ----
template <typename K>
__global__ void heads_k(const K* __restrict__ key, int64_t n, uint32_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const K k = key[i];
    flag[i] = (k != dead<K>() && (i == 0 || key[i - 1] != k)) ? 1u : 0u;
  }
}

// Duplicate input tuples: ⊕-merge in push order (reading 16).
__global__ void edb_reduce_k(const uint64_t* __restrict__ key, const float* __restrict__ p,
                             const int32_t* __restrict__ fid, const uint32_t* __restrict__ pos, int64_t n, int semi,
                             uint64_t* __restrict__ okey, float* __restrict__ op, int32_t* __restrict__ ofid) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    if (k == KEY_DEAD || (i > 0 && key[i - 1] == k)) continue;  // dead: outside the micro-batch
    float bp = p[i];
    int32_t bf = fid[i];
    double acc = (double)bp;
    for (int64_t j = i + 1; j < n && key[j] == k; ++j) {
      const float q = p[j];
      if (semi == S_ADDMULT) acc = __dadd_rn(acc, (double)q);
      else if (semi == S_MAXMIN) { if (q > bp) bp = q; }
      else if (semi == S_MAXMULT) {
        const int32_t g = fid[j];
        if (q > bp || (q == bp && g < bf)) { bp = q; bf = g; }
      }
    }
    if (semi == S_ADDMULT) bp = (float)acc;
    const uint32_t u = pos[i];
    okey[u] = k;
    op[u] = bp;
    ofid[u] = bf;
  }
}

// U = segmented ⊕ of sorted candidates (A7).  Segment boundaries come from
// the head flags' scan (pos); uend[u] = one past the last element of segment u.
// Short segments: one thread each, left-to-right.  Long segments (> LONG_SEG,
// e.g. a C3 kinship head's per-round contributions): one warp each.  Huge
// segments (> HUGE_SEG, e.g. the per-sample `endpoints_connected()` groups of
// ~1M candidates): one CTA each.  Warp/CTA partials are strided folds combined
// by a fixed-shape tree, so the result is deterministic.
constexpr int LONG_SEG = 64;
constexpr int HUGE_SEG = 4096;

template <typename K>
__global__ void seg_ends_k(const K* __restrict__ key, const uint32_t* __restrict__ pos, int64_t n,
                           uint32_t* __restrict__ uend) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const K k = key[i];
    if (k == dead<K>()) continue;
    if (i == n - 1 || key[i + 1] != k) {
      const bool head = i == 0 || key[i - 1] != k;  // pos = exclusive count of heads
      uend[pos[i] - (head ? 0u : 1u)] = (uint32_t)(i + 1);
    }
  }
}

struct Acc {
  double s;    // add-mult sum
  float p;     // max
  uint32_t w;  // witness (max-mult)
};

template <int SEMI>
__device__ __forceinline__ Acc acc_load(const void* valv, int64_t j) {
  Acc a{0.0, 0.0f, 0u};
  if constexpr (SEMI == S_MAXMULT) {
    const uint64_t c = ((const uint64_t*)valv)[j];
    a.p = u2f((uint32_t)c);
    a.w = (uint32_t)(c >> 32);
  } else if constexpr (SEMI == S_ADDMULT) {
    a.s = (double)u2f(((const uint32_t*)valv)[j]);
  } else if constexpr (SEMI == S_MAXMIN) {
    a.p = u2f(((const uint32_t*)valv)[j]);
  }
  return a;
}

// b follows a in canonical order
template <int SEMI>
__device__ __forceinline__ Acc acc_join(Acc a, Acc b) {
  if constexpr (SEMI == S_ADDMULT) {
    a.s = __dadd_rn(a.s, b.s);
  } else if constexpr (SEMI == S_MAXMULT) {
    if (b.p > a.p || (b.p == a.p && b.w < a.w)) { a.p = b.p; a.w = b.w; }
  } else if constexpr (SEMI == S_MAXMIN) {
    if (b.p > a.p) a.p = b.p;
  }
  return a;
}

template <int SEMI>
__device__ __forceinline__ void acc_store(Acc a, int64_t u, float* up, uint32_t* uw) {
  if constexpr (SEMI == S_ADDMULT) up[u] = (float)a.s;
  if constexpr (SEMI == S_MAXMIN || SEMI == S_MAXMULT) up[u] = a.p;
  if constexpr (SEMI == S_MAXMULT) uw[u] = a.w;
}

template <typename K, int SEMI>
__global__ void seg_reduce_short_k(const K* __restrict__ key, const void* __restrict__ valv,
                                   const uint32_t* __restrict__ uend, int64_t nu, K* __restrict__ ukey,
                                   float* __restrict__ up, uint32_t* __restrict__ uw, uint32_t* __restrict__ nlong,
                                   uint32_t* __restrict__ longs) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = u ? (int64_t)uend[u - 1] : 0, e = uend[u];
    ukey[u] = key[s];
    if constexpr (SEMI == S_UNIT) continue;
    if (e - s > LONG_SEG) {  // warp list from the front, CTA list from the back
      if (e - s > HUGE_SEG) longs[nu - 1 - atomicAdd(nlong + 1, 1u)] = (uint32_t)u;
      else longs[atomicAdd(nlong, 1u)] = (uint32_t)u;
      continue;
    }
    Acc a = acc_load<SEMI>(valv, s);
    for (int64_t j = s + 1; j < e; ++j) a = acc_join<SEMI>(a, acc_load<SEMI>(valv, j));
    acc_store<SEMI>(a, u, up, uw);
  }
}

template <int SEMI>
__device__ __forceinline__ Acc acc_shfl_down(Acc a, int off) {
  Acc b;
  b.s = __shfl_down_sync(0xffffffffu, a.s, off);
  b.p = __shfl_down_sync(0xffffffffu, a.p, off);
  b.w = __shfl_down_sync(0xffffffffu, a.w, off);
  return b;
}

template <int SEMI>
__global__ void __launch_bounds__(256) seg_reduce_warp_k(const void* __restrict__ valv,
                                                         const uint32_t* __restrict__ uend,
                                                         const uint32_t* __restrict__ nlong,
                                                         const uint32_t* __restrict__ longs, float* __restrict__ up,
                                                         uint32_t* __restrict__ uw) {
  const uint32_t nl = nlong[0];
  const int lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < nl; q += nw) {
    const uint32_t u = longs[q];
    const int64_t s = u ? (int64_t)uend[u - 1] : 0, e = uend[u];
    // lane t folds s+t, s+t+32, ... in order (e - s > LONG_SEG >= 32)
    Acc a = acc_load<SEMI>(valv, s + lane);
    for (int64_t j = s + lane + 32; j < e; j += 32) a = acc_join<SEMI>(a, acc_load<SEMI>(valv, j));
#pragma unroll
    for (int off = 16; off; off >>= 1) a = acc_join<SEMI>(a, acc_shfl_down<SEMI>(a, off));
    if (lane == 0) acc_store<SEMI>(a, u, up, uw);
  }
}

template <int SEMI>
__global__ void __launch_bounds__(256) seg_reduce_long_k(const void* __restrict__ valv,
                                                         const uint32_t* __restrict__ uend,
                                                         const uint32_t* __restrict__ nlong, int64_t nu,
                                                         const uint32_t* __restrict__ longs, float* __restrict__ up,
                                                         uint32_t* __restrict__ uw) {
  __shared__ Acc part[256];
  const uint32_t nl = nlong[1];
  for (uint32_t q = blockIdx.x; q < nl; q += gridDim.x) {
    const uint32_t u = longs[nu - 1 - q];
    const int64_t s = u ? (int64_t)uend[u - 1] : 0, e = uend[u];
    // thread t folds elements s+t, s+t+256, ... in order (e - s > HUGE_SEG >= 256)
    Acc a = acc_load<SEMI>(valv, s + threadIdx.x);
    for (int64_t j = s + threadIdx.x + 256; j < e; j += 256) a = acc_join<SEMI>(a, acc_load<SEMI>(valv, j));
    part[threadIdx.x] = a;
    __syncthreads();
    for (int d = 1; d < 256; d <<= 1) {  // fixed pairwise tree over the thread partials
      if ((threadIdx.x % (2 * d)) == 0)
        part[threadIdx.x] = acc_join<SEMI>(part[threadIdx.x], part[threadIdx.x + d]);
      __syncthreads();
    }
    if (threadIdx.x == 0) acc_store<SEMI>(part[0], u, up, uw);
    __syncthreads();
  }
}

// ------------------------------------------------------------ diff/apply ----
__device__ __forceinline__ float state_oplus(int semi, float s, float b) {
  if (semi == S_ADDMULT) return (float)__dadd_rn((double)s, (double)b);
  return b > s ? b : s;
}

__global__ void diff_k(const uint64_t* __restrict__ ukey, const float* __restrict__ up, int64_t nu,
                       const uint64_t* __restrict__ fkey, const float* __restrict__ fp, int64_t nf, int semi,
                       uint64_t* __restrict__ flags, int64_t* __restrict__ pos) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = ukey[i];
    const int64_t p = lower_bound_u64(fkey, nf, k);
    uint64_t fl;
    if (p >= nf || fkey[p] != k) {
      fl = (1ull << 32) | 1ull;  // new tuple: in Δ' and inserted
      pos[i] = -1;
    } else {
      bool changed = false;
      if (semi != S_UNIT) {
        const float s = fp[p];
        changed = f2u(state_oplus(semi, s, up[i])) != f2u(s);
      }
      fl = changed ? 1ull : 0ull;
      pos[i] = p;
    }
    flags[i] = fl;
  }
}

__global__ void apply_k(const uint64_t* __restrict__ ukey, const float* __restrict__ up,
                        const uint32_t* __restrict__ uw, int64_t nu, const uint64_t* __restrict__ flags,
                        const uint64_t* __restrict__ offs, const int64_t* __restrict__ pos, int semi,
                        float* __restrict__ fp, uint32_t* __restrict__ fw, uint64_t* __restrict__ dkey,
                        float* __restrict__ dp, uint32_t* __restrict__ dw, uint64_t* __restrict__ nkey,
                        float* __restrict__ np_, uint32_t* __restrict__ nw) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nu; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t fl = flags[i];
    if (!(fl & 1ull)) continue;
    const uint64_t o = offs[i];
    const uint32_t di = (uint32_t)o;
    const uint64_t k = ukey[i];
    dkey[di] = k;
    const float b = semi != S_UNIT ? up[i] : 0.0f;
    const uint32_t bw = semi == S_MAXMULT ? uw[i] : 0u;
    if (semi != S_UNIT) dp[di] = b;
    if (semi == S_MAXMULT) dw[di] = bw;
    if (fl >> 32) {
      const uint32_t ni = (uint32_t)(o >> 32);
      nkey[ni] = k;
      if (semi != S_UNIT) np_[ni] = b;
      if (semi == S_MAXMULT) nw[ni] = bw;
    } else {
      const int64_t p = pos[i];
      fp[p] = state_oplus(semi, fp[p], b);
      if (semi == S_MAXMULT) fw[p] = bw;  // strict improvement: witness follows p
    }
  }
}

// ----------------------------------------------------------------- merge ----
constexpr int MITEMS = 8;
__global__ void merge_k(const uint64_t* __restrict__ ak, const float* __restrict__ ap,
                        const uint32_t* __restrict__ aw, int64_t na, const uint64_t* __restrict__ bk,
                        const float* __restrict__ bp, const uint32_t* __restrict__ bw, int64_t nb,
                        uint64_t* __restrict__ ok, float* __restrict__ op, uint32_t* __restrict__ ow) {
  const int64_t total = na + nb;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t * MITEMS < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = t * MITEMS;
    int64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
    while (lo < hi) {  // merge path: number of A elements among the first d outputs
      const int64_t mid = (lo + hi) >> 1;
      if (ak[mid] < bk[d - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    int64_t i = lo, j = d - lo;
    const int64_t end = d + MITEMS < total ? d + MITEMS : total;
    for (int64_t o = d; o < end; ++o) {
      const bool takeA = i < na && (j >= nb || ak[i] < bk[j]);
      if (takeA) {
        ok[o] = ak[i];
        if (op) op[o] = ap[i];
        if (ow) ow[o] = aw[i];
        ++i;
      } else {
        ok[o] = bk[j];
        if (op) op[o] = bp[j];
        if (ow) ow[o] = bw[j];
        ++j;
      }
    }
  }
}

// ----------------------------------------------------------- dense store ----
__global__ void dense_fill_k(uint32_t* __restrict__ a, int64_t n, uint32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

template <int SEMI>
__global__ void dense_diff_k(const uint32_t* __restrict__ ukey, const float* __restrict__ up,
                             const uint32_t* __restrict__ uw, int64_t nu, float* __restrict__ fp,
                             uint32_t* __restrict__ fw, uint32_t* __restrict__ fbits, uint64_t* __restrict__ flags) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t slot = ukey[u];
    uint64_t fl = 0;
    if constexpr (SEMI == S_UNIT) {
      const uint32_t bit = 1u << (slot & 31u);
      const uint32_t old = atomicOr(fbits + (slot >> 5), bit);  // other bits of the word belong to other U rows
      if (!(old & bit)) fl = (1ull << 32) | 1ull;
    } else {
      const float s = fp[slot];
      const float b = up[u];
      if (f2u(s) == DENSE_ABSENT) {
        fl = (1ull << 32) | 1ull;
        fp[slot] = b;
        if constexpr (SEMI == S_MAXMULT) fw[slot] = uw[u];
      } else {
        const float nv = state_oplus(SEMI, s, b);
        if (f2u(nv) != f2u(s)) {
          fl = 1ull;
          fp[slot] = nv;
          if constexpr (SEMI == S_MAXMULT) fw[slot] = uw[u];  // strict improvement: witness follows p
        }
      }
    }
    flags[u] = fl;
  }
}

__global__ void dense_delta_k(const uint32_t* __restrict__ ukey, const float* __restrict__ up,
                              const uint32_t* __restrict__ uw, int64_t nu, const uint64_t* __restrict__ flags,
                              const uint64_t* __restrict__ offs, int semi, uint32_t* __restrict__ dkey,
                              float* __restrict__ dp, uint32_t* __restrict__ dw) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    if (!(flags[u] & 1ull)) continue;
    const uint32_t d = (uint32_t)offs[u];
    dkey[d] = ukey[u];
    if (semi != S_UNIT) dp[d] = up[u];  // Δ carries the increment b (reading 5)
    if (semi == S_MAXMULT) dw[d] = uw[u];
  }
}

__global__ void dense_present_k(const float* __restrict__ fp, const uint32_t* __restrict__ fbits, int64_t n,
                                int semi, uint32_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (semi == S_UNIT) flag[i] = (fbits[i >> 5] >> (i & 31)) & 1u;
    else flag[i] = f2u(fp[i]) != DENSE_ABSENT ? 1u : 0u;
  }
}

__global__ void dense_compact_k(const float* __restrict__ fp, const uint32_t* __restrict__ fw,
                                const uint32_t* __restrict__ fbits, const uint32_t* __restrict__ pos, int64_t n,
                                int semi, uint64_t* __restrict__ key, float* __restrict__ p,
                                uint32_t* __restrict__ w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool present;
    if (semi == S_UNIT) present = (fbits[i >> 5] >> (i & 31)) & 1u;
    else present = f2u(fp[i]) != DENSE_ABSENT;
    if (!present) continue;
    const uint32_t o = pos[i];
    key[o] = (uint64_t)i;
    if (semi != S_UNIT) p[o] = fp[i];
    if (semi == S_MAXMULT) w[o] = fw[i];
  }
}

__global__ void widen_u32_k(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint64_t)in[i];
}

// ------------------------------------------------------ direct ⊕ store ----
// wmask / wT / wrb: max-mult witness field and its decompression (kernels.cuh MxEnc):
// wc = rule << wT | vars  ->  w = rule << (32 - wrb) | vars
__device__ __forceinline__ void direct_decode(const void* f, int semi, int64_t slot, bool& present, float& p,
                                              uint32_t& w, unsigned long long wmask = 0, int wT = 0, int wrb = 0) {
  present = false;
  p = 0.0f;
  w = 0;
  if (semi == S_UNIT) {
    present = (reinterpret_cast<const uint32_t*>(f)[slot >> 5] >> (slot & 31)) & 1u;
  } else if (semi == S_MAXMIN) {
    const uint32_t v = reinterpret_cast<const uint32_t*>(f)[slot];
    present = v != 0u;
    p = mm_p(v);
  } else {
    const unsigned long long v = reinterpret_cast<const unsigned long long*>(f)[slot];
    present = v != 0ull;
    p = mx_p(v);
    const unsigned long long wc = ~v & wmask;
    const unsigned long long vars = wc & ((1ull << wT) - 1ull);
    w = (uint32_t)(wrb ? (((wc >> wT) << (32 - wrb)) | vars) : vars);
  }
}

// Dirty bitmap -> Δ' in slot order in two launches (replaces the per-chunk
// count, scan and extraction above: three plus the scan's).  CTA tile = 2048
// bitmap words, 8 per lane in warp-strided chunks of 32 (each chunk load is one
// 128-B line per warp).  Launch 1 counts the set bits of every tile and of every
// group of 8 tiles; launch 2 gives each tile its base as the sum of the group
// counts before it plus the tile counts of its own group before it (a parallel
// block reduction: no serial chain across tiles, unlike a decoupled look-back
// when every tile of a small grid is resident at once), then writes the tile's
// Δ' rows.
constexpr int LB_WPT = 8;   // bitmap words per lane
constexpr int LB_U = 4;     // Δ' rows per lane in flight
constexpr int LB_TILE = 256 * LB_WPT;
constexpr int LB_GROUP = 8;  // tiles per group (one counting CTA, one tile per warp)

__global__ void __launch_bounds__(256) dirty_group_count_k(const uint32_t* __restrict__ dirty, int64_t nw,
                                                           int64_t nt, uint32_t* __restrict__ tcnt,
                                                           uint32_t* __restrict__ gsum) {
  __shared__ uint32_t wt[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tile = (int64_t)blockIdx.x * LB_GROUP + warp;
  uint32_t c = 0;
  if (tile < nt) {
    const int64_t w0 = tile * LB_TILE;
    if (w0 + LB_TILE <= nw) {
#pragma unroll
      for (int i = 0; i < LB_TILE / 128; ++i) {  // 16 B per lane, 512 B per warp load
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(dirty + w0) + i * 32 + lane);
        c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
      }
    } else {
      for (int64_t w = w0 + lane; w < nw; w += 32) c += __popc(__ldcg(dirty + w));
    }
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane == 0) {
    wt[warp] = c;
    if (tile < nt) tcnt[tile] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t g = 0;
    for (int k = 0; k < 8; ++k) g += wt[k];
    gsum[blockIdx.x] = g;
  }
}

// ATOMIC: one launch, no counting pass — each warp claims its output range with
// one atomicAdd (Δ' = runs sorted within each warp's 8192 slots, runs in any
// order; joins over idempotent ⊕ do not depend on Δ order) and the last CTA to
// claim publishes |Δ'| (ctr[0] = rows, ctr[1] = CTAs that claimed; both reset).
template <int SEMI, bool ATOMIC, int WPT>
__global__ void __launch_bounds__(256) direct_extract2_k(void* __restrict__ f, uint32_t* __restrict__ dirty,
                                                         int64_t nw, uint32_t* __restrict__ dkey,
                                                         float* __restrict__ dp, uint32_t* __restrict__ dw,
                                                         const uint32_t* __restrict__ tcnt,
                                                         const uint32_t* __restrict__ gsum,
                                                         uint32_t* __restrict__ total, unsigned long long restamp,
                                                         unsigned long long wmask, unsigned long long* ring,
                                                         uint32_t seq, uint32_t* __restrict__ ctr) {
  __shared__ uint32_t wtot[8];
  __shared__ uint32_t wpre[8];
  __shared__ uint32_t s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // ATOMIC: grid-stride over tiles (the launcher caps the grid) with ONE
  // claim atomic per CTA tile and one completion atomic per CTA: per-warp
  // claims plus a completion atomic from each of C2's 4096 CTAs serialised on
  // the two counters (a ~12 µs floor per round even when Δ' is tiny)
  const int64_t ntiles = ATOMIC ? (nw + 256 * WPT - 1) / (256 * WPT) : (int64_t)gridDim.x;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  const int64_t w0 = tile * (256 * WPT) + (int64_t)warp * (32 * WPT);
  uint32_t m[WPT];
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < WPT; ++j) {
    const int64_t w = w0 + j * 32 + lane;
    m[j] = w < nw ? __ldcg(dirty + w) : 0u;
    c += __popc(m[j]);
  }
  const uint32_t wsum = __reduce_add_sync(0xffffffffu, c);
  uint32_t base;
  if constexpr (ATOMIC) {
    if (lane == 0) wtot[warp] = wsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int k = 0; k < 8; ++k) {
        wpre[k] = t;
        t += wtot[k];
      }
      s_base = t ? atomicAdd(ctr, t) : 0u;
    }
    __syncthreads();
    base = s_base + wpre[warp];
  } else {
  // tile base: groups before this tile's group + this group's earlier tiles
  const int64_t grp = tile / LB_GROUP;
  uint32_t pre = 0;
  for (int64_t i = threadIdx.x; i < grp; i += 256) pre += gsum[i];
  if (threadIdx.x < (unsigned)(tile - grp * LB_GROUP)) pre += tcnt[grp * LB_GROUP + threadIdx.x];
  pre = __reduce_add_sync(0xffffffffu, pre);
  if (lane == 0) {
    wtot[warp] = wsum;
    wpre[warp] = pre;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t own = lane < 8 ? wtot[lane] : 0u;
    uint32_t inc = own;
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += u;
    }
    const uint32_t prefix = __reduce_add_sync(0xffffffffu, lane < 8 ? wpre[lane] : 0u);
    const uint32_t agg = __shfl_sync(0xffffffffu, inc, 7);
    if (lane == 0) {
      s_base = prefix;
      if (tile == (int64_t)gridDim.x - 1) {
        *total = prefix + agg;
        if (ring) {  // zero-copy report to the host (async rounds)
          *reinterpret_cast<volatile unsigned long long*>(ring) = ((unsigned long long)seq << 32) | (prefix + agg);
          __threadfence_system();
        }
      }
    }
    __syncwarp();
    if (lane < 8) wtot[lane] = inc - own;
  }
  __syncthreads();
  base = s_base + wtot[warp];
  }
#pragma unroll 1
  for (int j = 0; j < (wsum ? WPT : 0); ++j) {  // a warp whose words are all clean has nothing to do
    const uint32_t mm = m[j];
    const uint32_t cnt = __popc(mm);
    uint32_t inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += u;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    if (!tot) continue;
    const int64_t wbase = w0 + j * 32;
    if (mm) dirty[wbase + lane] = 0u;
    // bits spread evenly over the lanes, LB_U per lane per batch: every slot
    // read of a batch is issued before any dependent store (memory-level
    // parallelism; the loop is latency-bound otherwise)
    for (uint32_t kb = 0; kb < tot; kb += 32 * LB_U) {
      uint32_t slotv[LB_U];
      bool act[LB_U];
#pragma unroll
      for (int u = 0; u < LB_U; ++u) {
        const uint32_t k = kb + u * 32 + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const uint32_t v = __shfl_sync(0xffffffffu, inc, lo + step - 1);
          if (v <= k) lo += step;
        }
        const uint32_t wm = __shfl_sync(0xffffffffu, mm, lo);
        const uint32_t wex = __shfl_sync(0xffffffffu, inc - cnt, lo);
        act[u] = k < tot;
        slotv[u] = act[u] ? (uint32_t)((wbase + lo) * 32 + __fns(wm, 0, (int)(k - wex) + 1)) : 0u;
      }
      if (SEMI == S_MAXMIN) {
        uint32_t v[LB_U];
#pragma unroll
        for (int u = 0; u < LB_U; ++u)
          if (act[u]) v[u] = __ldcg(reinterpret_cast<const uint32_t*>(f) + slotv[u]);
#pragma unroll
        for (int u = 0; u < LB_U; ++u) {
          if (!act[u]) continue;
          const uint32_t o = base + kb + u * 32 + lane;
          dkey[o] = slotv[u];  // no settle: max-min words carry no tie state
          dp[o] = mm_p(v[u]);
        }
      } else if (SEMI == S_MAXMULT) {
        unsigned long long v[LB_U];
#pragma unroll
        for (int u = 0; u < LB_U; ++u)
          if (act[u]) v[u] = __ldcg(reinterpret_cast<const unsigned long long*>(f) + slotv[u]);
#pragma unroll
        for (int u = 0; u < LB_U; ++u) {
          if (!act[u]) continue;
          const uint32_t o = base + kb + u * 32 + lane;
          if (restamp) __stcg(reinterpret_cast<unsigned long long*>(f) + slotv[u], v[u] | restamp);
          dkey[o] = slotv[u];
          dp[o] = mx_p(v[u]);
          if (dw) dw[o] = (uint32_t)(~v[u] & wmask);
        }
      } else {
#pragma unroll
        for (int u = 0; u < LB_U; ++u)
          if (act[u]) dkey[base + kb + u * 32 + lane] = slotv[u];
      }
    }
    base += tot;
  }
  __syncthreads();  // wtot / wpre / s_base are rewritten by the next tile
  }
  if constexpr (ATOMIC) {
    // |Δ'| is final once every CTA has claimed (writes may still be in flight:
    // the next kernel is stream-ordered after them), so the last CTA to finish
    // claiming publishes it and resets the counters
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
        __threadfence();
        const uint32_t n = *reinterpret_cast<volatile uint32_t*>(ctr);
        *total = n;
        ctr[0] = 0u;
        ctr[1] = 0u;
        if (ring) {  // zero-copy report to the host (async rounds)
          *reinterpret_cast<volatile unsigned long long*>(ring) = ((unsigned long long)seq << 32) | n;
          __threadfence_system();
        }
      }
    }
  }
}


__global__ void direct_present_k(const void* __restrict__ f, int64_t n, int semi, uint32_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool pr;
    float p;
    uint32_t w;
    direct_decode(f, semi, i, pr, p, w);
    flag[i] = pr ? 1u : 0u;
  }
}

__global__ void direct_count_k(const void* __restrict__ f, int64_t n, int semi, unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  if (semi == S_UNIT) {  // bitmap words (bits past n are never set)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n + 31) / 32; i += S)
      c += __popc(reinterpret_cast<const uint32_t*>(f)[i]);
  } else if (semi == S_MAXMIN) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += S)
      c += reinterpret_cast<const uint32_t*>(f)[i] != 0u;
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += S)
      c += reinterpret_cast<const unsigned long long*>(f)[i] != 0ull;
  }
  c = __reduce_add_sync(0xffffffffu, (unsigned)c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void direct_compact_k(const void* __restrict__ f, const uint32_t* __restrict__ pos, int64_t n, int semi,
                                 uint64_t* __restrict__ key, float* __restrict__ p, uint32_t* __restrict__ w,
                                 unsigned long long wmask, int wT, int wrb) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool pr;
    float pp;
    uint32_t ww;
    direct_decode(f, semi, i, pr, pp, ww, wmask, wT, wrb);
    if (!pr) continue;
    const uint32_t o = pos[i];
    key[o] = (uint64_t)i;
    if (semi != S_UNIT) p[o] = pp;
    if (semi == S_MAXMULT) w[o] = ww;
  }
}

template <typename K>
void seg_reduce_impl(const K* key, const void* val, const uint32_t* pos, int64_t n, int64_t nu, int semi, K* ukey,
                     float* up, uint32_t* uw, uint32_t* scratch, cudaStream_t st) {
  if (n <= 0 || nu <= 0) return;
  uint32_t* uend = scratch;            // nu
  uint32_t* nlong = scratch + nu;      // 2: [0] warp list, [1] CTA list
  uint32_t* longs = scratch + nu + 2;  // nu: warp list from the front, CTA list from the back
  cudaMemsetAsync(nlong, 0, 8, st);
  note_launch();
  seg_ends_k<K><<<grid_for(n, 256), 256, 0, st>>>(key, pos, n, uend);
  const int g = grid_for(nu, 256);
  note_launch();
  switch (semi) {
    case S_UNIT:
      seg_reduce_short_k<K, S_UNIT><<<g, 256, 0, st>>>(key, val, uend, nu, ukey, up, uw, nlong, longs);
      return;
    case S_MAXMIN:
      seg_reduce_short_k<K, S_MAXMIN><<<g, 256, 0, st>>>(key, val, uend, nu, ukey, up, uw, nlong, longs);
      break;
    case S_ADDMULT:
      seg_reduce_short_k<K, S_ADDMULT><<<g, 256, 0, st>>>(key, val, uend, nu, ukey, up, uw, nlong, longs);
      break;
    default:
      seg_reduce_short_k<K, S_MAXMULT><<<g, 256, 0, st>>>(key, val, uend, nu, ukey, up, uw, nlong, longs);
      break;
  }
  const int gw = grid_for((nu + 7) / 8, 1, 148 * 8), gl = 148 * 4;
  note_launch();
  note_launch();
  switch (semi) {
    case S_MAXMIN:
      seg_reduce_warp_k<S_MAXMIN><<<gw, 256, 0, st>>>(val, uend, nlong, longs, up, uw);
      seg_reduce_long_k<S_MAXMIN><<<gl, 256, 0, st>>>(val, uend, nlong, nu, longs, up, uw);
      break;
    case S_ADDMULT:
      seg_reduce_warp_k<S_ADDMULT><<<gw, 256, 0, st>>>(val, uend, nlong, longs, up, uw);
      seg_reduce_long_k<S_ADDMULT><<<gl, 256, 0, st>>>(val, uend, nlong, nu, longs, up, uw);
      break;
    default:
      seg_reduce_warp_k<S_MAXMULT><<<gw, 256, 0, st>>>(val, uend, nlong, longs, up, uw);
      seg_reduce_long_k<S_MAXMULT><<<gl, 256, 0, st>>>(val, uend, nlong, nu, longs, up, uw);
      break;
  }
}

}  // namespace

void launch_minmax(const int32_t* col, int64_t n, int32_t* out2, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  minmax_k<<<grid_for(n, 256, 148 * 4), 256, 0, st>>>(col, n, out2);
}
void launch_pack(const PackPlan& pp, int64_t n, uint64_t* key, uint32_t* rowid, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  pack_k<<<grid_for(n, 256), 256, 0, st>>>(pp, n, key, rowid);
}
void launch_gather_f32(const float* s, const uint32_t* idx, float* d, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  gather_f32_k<<<grid_for(n, 256), 256, 0, st>>>(s, idx, d, n);
}
void launch_gather_i32(const int32_t* s, const uint32_t* idx, int32_t* d, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  gather_i32_k<<<grid_for(n, 256), 256, 0, st>>>(s, idx, d, n);
}
void launch_iota_i32(int32_t* d, int64_t n, int32_t first, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  iota_k<<<grid_for(n, 256), 256, 0, st>>>(d, n, first);
}
void launch_fill_f32(float* d, int64_t n, float v, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  fill_k<<<grid_for(n, 256), 256, 0, st>>>(d, n, v);
}
void launch_validate(const float* p, const int32_t* s, int64_t n, int32_t batch, uint32_t* flags, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  validate_k<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(p, s, n, batch, flags);
}
void launch_heads(const uint64_t* key, int64_t n, uint32_t* flag, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  heads_k<uint64_t><<<grid_for(n, 256), 256, 0, st>>>(key, n, flag);
}
void launch_heads(const uint32_t* key, int64_t n, uint32_t* flag, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  heads_k<uint32_t><<<grid_for(n, 256), 256, 0, st>>>(key, n, flag);
}
void launch_edb_reduce(const uint64_t* key, const float* p, const int32_t* fid, const uint32_t* pos, int64_t n,
                       int semi, uint64_t* okey, float* op, int32_t* ofid, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  edb_reduce_k<<<grid_for(n, 256), 256, 0, st>>>(key, p, fid, pos, n, semi, okey, op, ofid);
}
void launch_seg_reduce(const uint64_t* key, const void* val, const uint32_t* pos, int64_t n, int64_t nu, int semi,
                       uint64_t* ukey, float* up, uint32_t* uw, uint32_t* scratch, cudaStream_t st) {
  seg_reduce_impl<uint64_t>(key, val, pos, n, nu, semi, ukey, up, uw, scratch, st);
}
void launch_seg_reduce(const uint32_t* key, const void* val, const uint32_t* pos, int64_t n, int64_t nu, int semi,
                       uint32_t* ukey, float* up, uint32_t* uw, uint32_t* scratch, cudaStream_t st) {
  seg_reduce_impl<uint32_t>(key, val, pos, n, nu, semi, ukey, up, uw, scratch, st);
}
void launch_diff(const uint64_t* ukey, const float* up, const uint32_t* uw, int64_t nu, const uint64_t* fkey,
                 const float* fp, int64_t nf, int semi, uint64_t* flags, int64_t* pos, cudaStream_t st) {
  (void)uw;
  if (nu <= 0) return;
  note_launch();
  diff_k<<<grid_for(nu, 256), 256, 0, st>>>(ukey, up, nu, fkey, fp, nf, semi, flags, pos);
}
void launch_apply(const uint64_t* ukey, const float* up, const uint32_t* uw, int64_t nu, const uint64_t* flags,
                  const uint64_t* offs, const int64_t* pos, int semi, float* fp, uint32_t* fw, uint64_t* dkey,
                  float* dp, uint32_t* dw, uint64_t* nkey, float* np_, uint32_t* nw, cudaStream_t st) {
  if (nu <= 0) return;
  note_launch();
  apply_k<<<grid_for(nu, 256), 256, 0, st>>>(ukey, up, uw, nu, flags, offs, pos, semi, fp, fw, dkey, dp, dw, nkey,
                                             np_, nw);
}
void launch_merge(const uint64_t* akey, const float* ap, const uint32_t* aw, int64_t na, const uint64_t* bkey,
                  const float* bp, const uint32_t* bw, int64_t nb, uint64_t* okey, float* op, uint32_t* ow,
                  cudaStream_t st) {
  const int64_t total = na + nb;
  if (total <= 0) return;
  const int64_t threads = (total + MITEMS - 1) / MITEMS;
  note_launch();
  merge_k<<<grid_for(threads, 256), 256, 0, st>>>(akey, ap, aw, na, bkey, bp, bw, nb, okey, op, ow);
}
void launch_dense_fill(float* fp, uint32_t* fbits, int64_t nslots, int semi, cudaStream_t st) {
  note_launch();
  if (semi == S_UNIT) dense_fill_k<<<grid_for((nslots + 31) / 32, 256), 256, 0, st>>>(fbits, (nslots + 31) / 32, 0u);
  else dense_fill_k<<<grid_for(nslots, 256), 256, 0, st>>>(reinterpret_cast<uint32_t*>(fp), nslots, DENSE_ABSENT);
}
void launch_dense_diff(const uint32_t* ukey, const float* up, const uint32_t* uw, int64_t nu, int semi, float* fp,
                       uint32_t* fw, uint32_t* fbits, uint64_t* flags, cudaStream_t st) {
  if (nu <= 0) return;
  const int g = grid_for(nu, 256);
  note_launch();
  switch (semi) {
    case S_UNIT: dense_diff_k<S_UNIT><<<g, 256, 0, st>>>(ukey, up, uw, nu, fp, fw, fbits, flags); break;
    case S_MAXMIN: dense_diff_k<S_MAXMIN><<<g, 256, 0, st>>>(ukey, up, uw, nu, fp, fw, fbits, flags); break;
    case S_ADDMULT: dense_diff_k<S_ADDMULT><<<g, 256, 0, st>>>(ukey, up, uw, nu, fp, fw, fbits, flags); break;
    default: dense_diff_k<S_MAXMULT><<<g, 256, 0, st>>>(ukey, up, uw, nu, fp, fw, fbits, flags); break;
  }
}
void launch_dense_delta(const uint32_t* ukey, const float* up, const uint32_t* uw, int64_t nu, const uint64_t* flags,
                        const uint64_t* offs, int semi, uint32_t* dkey, float* dp, uint32_t* dw, cudaStream_t st) {
  if (nu <= 0) return;
  note_launch();
  dense_delta_k<<<grid_for(nu, 256), 256, 0, st>>>(ukey, up, uw, nu, flags, offs, semi, dkey, dp, dw);
}
void launch_direct_fill(void* f, int64_t nslots, int semi, cudaStream_t st) {
  const size_t bytes = semi == S_UNIT ? (size_t)((nslots + 31) / 32) * 4
                                      : (size_t)nslots * (semi == S_MAXMULT ? 8 : 4);
  cudaMemsetAsync(f, 0, bytes, st);
}
void launch_widen_u32(const uint32_t* in, int64_t n, uint64_t* out, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  widen_u32_k<<<grid_for(n, 256), 256, 0, st>>>(in, n, out);
}

int64_t direct_extract2_scratch(int64_t nwords) {
  const int64_t nt = (nwords + LB_TILE - 1) / LB_TILE;
  return nt + (nt + LB_GROUP - 1) / LB_GROUP;
}
// LOBSTER_EX_CTAS: CTAs per SM of the atomic extraction's grid (A/B; default 8;
// 12 and 8 are equal within noise on C2, 4 is +3.5%; 4 words per lane equal to 2)
static int ex_ctas_per_sm() {
  static const int v = [] {
    const char* e = getenv("LOBSTER_EX_CTAS");
    const int x = e ? atoi(e) : 8;
    return x < 1 ? 1 : (x > 64 ? 64 : x);
  }();
  return v;
}

void launch_direct_extract2(void* f, uint32_t* dirty, int64_t nwords, int semi, uint32_t* dkey, float* dp,
                            uint32_t* dw, uint32_t* scratch, uint32_t* total, unsigned long long restamp,
                            unsigned long long wmask, unsigned long long* ring, uint32_t seq, uint32_t* ctr,
                            cudaStream_t st) {
  if (nwords <= 0) return;
  const int64_t nt = (nwords + LB_TILE - 1) / LB_TILE;
  const int64_t ng = (nt + LB_GROUP - 1) / LB_GROUP;
  uint32_t* tcnt = scratch;
  uint32_t* gsum = scratch ? scratch + nt : nullptr;
  if (!ctr) {  // slot-ordered Δ': counting pass first
    note_launch();
    dirty_group_count_k<<<(unsigned)ng, 256, 0, st>>>(dirty, nwords, nt, tcnt, gsum);
  }
  note_launch();
  // atomic runs: 2 (or 4) words per lane (more CTAs, shorter per-warp chains) up to
  // C2-sized bitmaps; 8 beyond, where the per-CTA claim / completion atomics on
  // one counter would otherwise serialise (C5: 32M words per micro-batch)
  const bool small = ctr && nwords <= (int64_t(1) << 22);
  // words per lane on C2-sized bitmaps: 2 (measured 1% faster than 4 on C2, equal on C4)
  // (LOBSTER_EX_WPT=4 selects the other instantiated width; read once, anything else = 2)
  static const int swpt = [] {
    const char* e = getenv("LOBSTER_EX_WPT");
    return (e && atoi(e) == 4) ? 4 : 2;
  }();
  // ATOMIC on C2-sized bitmaps: a grid-stride grid of at most 148 x 8 CTAs (one
  // completion atomic each; C2 23.9 -> 23.1 ms).  Larger bitmaps keep one CTA
  // per tile of 8 words per lane: capping C5's 16k tiles measured +9%.
  const int64_t tiles = small ? (nwords + 256 * swpt - 1) / (256 * swpt) : nt;
  const unsigned g = (unsigned)(small ? std::min<int64_t>(tiles, 148 * ex_ctas_per_sm()) : tiles);
#define LOB_EX(S, A, W) direct_extract2_k<S, A, W><<<g, 256, 0, st>>>(f, dirty, nwords, dkey, dp, dw, tcnt, gsum, \
                                                                  total, restamp, wmask, ring, seq, ctr)
#define LOB_EXS(S) if (!ctr) LOB_EX(S, false, LB_WPT); else if (small && swpt == 2) LOB_EX(S, true, 2); \
  else if (small) LOB_EX(S, true, 4); else LOB_EX(S, true, LB_WPT)
  switch (semi) {
    case S_UNIT: LOB_EXS(S_UNIT); break;
    case S_MAXMIN: LOB_EXS(S_MAXMIN); break;
    default: LOB_EXS(S_MAXMULT); break;
  }
#undef LOB_EXS
#undef LOB_EX
}
void launch_direct_present(const void* f, int64_t nslots, int semi, uint32_t* flag, cudaStream_t st) {
  if (nslots <= 0) return;
  note_launch();
  direct_present_k<<<grid_for(nslots, 256), 256, 0, st>>>(f, nslots, semi, flag);
}
void launch_direct_count(const void* f, int64_t nslots, int semi, unsigned long long* out, cudaStream_t st) {
  if (nslots <= 0) return;
  note_launch();
  direct_count_k<<<148 * 8, 256, 0, st>>>(f, nslots, semi, out);
}
void launch_direct_compact(const void* f, const uint32_t* pos, int64_t nslots, int semi, uint64_t* key, float* p,
                           uint32_t* w, unsigned long long wmask, int wT, int wrb, cudaStream_t st) {
  if (nslots <= 0) return;
  note_launch();
  direct_compact_k<<<grid_for(nslots, 256), 256, 0, st>>>(f, pos, nslots, semi, key, p, w, wmask, wT, wrb);
}
void launch_dense_present(const float* fp, const uint32_t* fbits, int64_t nslots, int semi, uint32_t* flag,
                          cudaStream_t st) {
  if (nslots <= 0) return;
  note_launch();
  dense_present_k<<<grid_for(nslots, 256), 256, 0, st>>>(fp, fbits, nslots, semi, flag);
}
void launch_dense_compact(const float* fp, const uint32_t* fw, const uint32_t* fbits, const uint32_t* pos,
                          int64_t nslots, int semi, uint64_t* key, float* p, uint32_t* w, cudaStream_t st) {
  if (nslots <= 0) return;
  note_launch();
  dense_compact_k<<<grid_for(nslots, 256), 256, 0, st>>>(fp, fw, fbits, pos, nslots, semi, key, p, w);
}

}  // namespace lob
