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
    uint64_t k = pp.sample ? ((uint64_t)(uint32_t)pp.sample[i] << pp.sshift) : 0ull;
    for (int c = 0; c < pp.ncols; ++c) k |= (uint64_t)(uint32_t)(pp.col[c][i] - pp.min[c]) << pp.shift[c];
    key[i] = k;
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
__global__ void heads_k(const uint64_t* __restrict__ key, int64_t n, uint32_t* __restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    flag[i] = (k != KEY_DEAD && (i == 0 || key[i - 1] != k)) ? 1u : 0u;
  }
}

// Duplicate input tuples: ⊕-merge in push order (reading 16).
__global__ void edb_reduce_k(const uint64_t* __restrict__ key, const float* __restrict__ p,
                             const int32_t* __restrict__ fid, const uint32_t* __restrict__ pos, int64_t n, int semi,
                             uint64_t* __restrict__ okey, float* __restrict__ op, int32_t* __restrict__ ofid) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    if (i > 0 && key[i - 1] == k) continue;
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
// e.g. the per-sample `endpoints_connected()` groups of ~1M candidates): one
// CTA each, strided partials combined by a fixed-shape tree (deterministic).
constexpr int LONG_SEG = 64;

__global__ void seg_ends_k(const uint64_t* __restrict__ key, const uint32_t* __restrict__ pos, int64_t n,
                           uint32_t* __restrict__ uend) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    if (k == KEY_DEAD) continue;
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

template <int SEMI>
__global__ void seg_reduce_short_k(const uint64_t* __restrict__ key, const void* __restrict__ valv,
                                   const uint32_t* __restrict__ uend, int64_t nu, uint64_t* __restrict__ ukey,
                                   float* __restrict__ up, uint32_t* __restrict__ uw, uint32_t* __restrict__ nlong,
                                   uint32_t* __restrict__ longs) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = u ? (int64_t)uend[u - 1] : 0, e = uend[u];
    ukey[u] = key[s];
    if constexpr (SEMI == S_UNIT) continue;
    if (e - s > LONG_SEG) {
      longs[atomicAdd(nlong, 1u)] = (uint32_t)u;
      continue;
    }
    Acc a = acc_load<SEMI>(valv, s);
    for (int64_t j = s + 1; j < e; ++j) a = acc_join<SEMI>(a, acc_load<SEMI>(valv, j));
    acc_store<SEMI>(a, u, up, uw);
  }
}

template <int SEMI>
__global__ void __launch_bounds__(256) seg_reduce_long_k(const void* __restrict__ valv,
                                                         const uint32_t* __restrict__ uend,
                                                         const uint32_t* __restrict__ nlong,
                                                         const uint32_t* __restrict__ longs, float* __restrict__ up,
                                                         uint32_t* __restrict__ uw) {
  __shared__ Acc part[256];
  const uint32_t nl = *nlong;
  for (uint32_t q = blockIdx.x; q < nl; q += gridDim.x) {
    const uint32_t u = longs[q];
    const int64_t s = u ? (int64_t)uend[u - 1] : 0, e = uend[u];
    // thread t folds elements s+t, s+t+256, ... (in order)
    Acc a = acc_load<SEMI>(valv, s + threadIdx.x < e ? s + threadIdx.x : s);
    bool have = s + threadIdx.x < e;
    for (int64_t j = s + threadIdx.x + 256; j < e; j += 256) a = acc_join<SEMI>(a, acc_load<SEMI>(valv, j));
    part[threadIdx.x] = a;
    __syncthreads();
    // fixed pairwise tree over thread partials (every segment here has > 64 elements,
    // so partials 0..63 always exist; missing partials only occur above e - s)
    const int cnt = (int)((e - s) < 256 ? (e - s) : 256);
    for (int d = 1; d < 256; d <<= 1) {
      if ((threadIdx.x % (2 * d)) == 0 && threadIdx.x + d < cnt) part[threadIdx.x] = acc_join<SEMI>(part[threadIdx.x], part[threadIdx.x + d]);
      __syncthreads();
    }
    if (threadIdx.x == 0) acc_store<SEMI>(part[0], u, up, uw);
    __syncthreads();
    (void)have;
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
  if (n > 0) {
    note_launch();
    gather_f32_k<<<grid_for(n, 256), 256, 0, st>>>(s, idx, d, n);
  }
}
void launch_gather_i32(const int32_t* s, const uint32_t* idx, int32_t* d, int64_t n, cudaStream_t st) {
  if (n > 0) {
    note_launch();
    gather_i32_k<<<grid_for(n, 256), 256, 0, st>>>(s, idx, d, n);
  }
}
void launch_iota_i32(int32_t* d, int64_t n, int32_t first, cudaStream_t st) {
  if (n > 0) {
    note_launch();
    iota_k<<<grid_for(n, 256), 256, 0, st>>>(d, n, first);
  }
}
void launch_fill_f32(float* d, int64_t n, float v, cudaStream_t st) {
  if (n > 0) {
    note_launch();
    fill_k<<<grid_for(n, 256), 256, 0, st>>>(d, n, v);
  }
}
void launch_validate(const float* p, const int32_t* s, int64_t n, int32_t batch, uint32_t* flags, cudaStream_t st) {
  if (n > 0) {
    note_launch();
    validate_k<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(p, s, n, batch, flags);
  }
}
void launch_heads(const uint64_t* key, int64_t n, uint32_t* flag, cudaStream_t st) {
  if (n > 0) {
    note_launch();
    heads_k<<<grid_for(n, 256), 256, 0, st>>>(key, n, flag);
  }
}
void launch_edb_reduce(const uint64_t* key, const float* p, const int32_t* fid, const uint32_t* pos, int64_t n,
                       int semi, uint64_t* okey, float* op, int32_t* ofid, cudaStream_t st) {
  if (n > 0) {
    note_launch();
    edb_reduce_k<<<grid_for(n, 256), 256, 0, st>>>(key, p, fid, pos, n, semi, okey, op, ofid);
  }
}
void launch_seg_reduce(const uint64_t* key, const void* val, const uint32_t* pos, int64_t n, int64_t nu, int semi,
                       uint64_t* ukey, float* up, uint32_t* uw, uint32_t* scratch, cudaStream_t st) {
  if (n <= 0 || nu <= 0) return;
  uint32_t* uend = scratch;            // nu
  uint32_t* nlong = scratch + nu;      // 1
  uint32_t* longs = scratch + nu + 1;  // nu
  cudaMemsetAsync(nlong, 0, 4, st);
  note_launch();
  seg_ends_k<<<grid_for(n, 256), 256, 0, st>>>(key, pos, n, uend);
  const int g = grid_for(nu, 256);
  note_launch();
  switch (semi) {
    case S_UNIT: seg_reduce_short_k<S_UNIT><<<g, 256, 0, st>>>(key, val, uend, nu, ukey, up, uw, nlong, longs); return;
    case S_MAXMIN: seg_reduce_short_k<S_MAXMIN><<<g, 256, 0, st>>>(key, val, uend, nu, ukey, up, uw, nlong, longs); break;
    case S_ADDMULT: seg_reduce_short_k<S_ADDMULT><<<g, 256, 0, st>>>(key, val, uend, nu, ukey, up, uw, nlong, longs); break;
    default: seg_reduce_short_k<S_MAXMULT><<<g, 256, 0, st>>>(key, val, uend, nu, ukey, up, uw, nlong, longs); break;
  }
  const int gl = 148 * 4;
  note_launch();
  switch (semi) {
    case S_MAXMIN: seg_reduce_long_k<S_MAXMIN><<<gl, 256, 0, st>>>(val, uend, nlong, longs, up, uw); break;
    case S_ADDMULT: seg_reduce_long_k<S_ADDMULT><<<gl, 256, 0, st>>>(val, uend, nlong, longs, up, uw); break;
    default: seg_reduce_long_k<S_MAXMULT><<<gl, 256, 0, st>>>(val, uend, nlong, longs, up, uw); break;
  }
}
void launch_diff(const uint64_t* ukey, const float* up, const uint32_t* uw, int64_t nu, const uint64_t* fkey,
                 const float* fp, int64_t nf, int semi, uint64_t* flags, int64_t* pos, cudaStream_t st) {
  (void)uw;
  if (nu > 0) {
    note_launch();
    diff_k<<<grid_for(nu, 256), 256, 0, st>>>(ukey, up, nu, fkey, fp, nf, semi, flags, pos);
  }
}
void launch_apply(const uint64_t* ukey, const float* up, const uint32_t* uw, int64_t nu, const uint64_t* flags,
                  const uint64_t* offs, const int64_t* pos, int semi, float* fp, uint32_t* fw, uint64_t* dkey,
                  float* dp, uint32_t* dw, uint64_t* nkey, float* np_, uint32_t* nw, cudaStream_t st) {
  if (nu > 0)
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

}  // namespace lob
