// k_walk.cu — witness walk + gradient (A11), output extract (A12) and the
// optional dense backward contraction.
//
// diff-max-mult (SURVEY §8(c) point 7): every IDB tuple stores (p, w) where w =
// rule index | packed non-head variable values of the winning derivation.  From
// an output tuple, the head values + w determine every body atom's tuple; input
// atoms are leaves (fact ids), IDB atoms are walked recursively.  The leaf
// multiset {f: m_f} gives ∂p/∂p_f = m_f p_f^{m_f-1} Π_{g≠f} p_g^{m_g} in fp64
// (§1: gradients for the input facts; §2).
// Output disaggregation per sample: PAPER.md:685 (§4.3).
#include "device_util.cuh"

namespace lob {
namespace {

// Pending IDB atoms of the walk.  Input atoms are leaves and are emitted the
// moment their key is known, so only IDB atoms are pushed: linear recursion
// (path :- path, edge) keeps one entry whatever the proof length, and a tree of
// height h with b IDB atoms per rule needs at most h·(b−1)+1.  The bottom STACK
// entries live in registers / local memory; deeper entries spill to a global
// per-thread region (gstack, gcap entries per thread) when the host provides
// one — the retry after a pass reports err bit 2.
constexpr int STACK = 32;

__device__ int64_t find_key(const WalkRel& R, uint64_t k) {
  if (R.off) {
    const uint64_t pre = k >> R.pshift;
    if (pre >= (uint64_t)R.nprefix) return -1;
    for (int64_t i = R.off[pre], e = R.off[pre + 1]; i < e; ++i)
      if (R.key[i] == k) return i;
    return -1;
  }
  const int64_t i = lower_bound_u64(R.key, R.n, k);
  return (i < R.n && R.key[i] == k) ? i : -1;
}

__device__ __forceinline__ int64_t emit_leaf(const WalkRel& A, uint64_t key, int pass, int64_t* leaves,
                                             int64_t out, int64_t count, int* err) {
  const int64_t idx = find_key(A, key);
  if (idx < 0) { atomicOr(err, 1); return -1; }
  if (pass) leaves[out + count] = (int64_t)A.fid[idx];
  return count + 1;
}

__global__ void walk_k(const WalkTables T, int rel0, int64_t n, int pass, const int64_t* __restrict__ offs,
                       int64_t* __restrict__ cnt, int64_t* __restrict__ leaves, int* __restrict__ err,
                       uint64_t* __restrict__ gkey, int* __restrict__ grel, int64_t gcap) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // without a spill region: one thread per tuple; with one: grid-stride, the
  // region indexed by the thread
  const int64_t step = gkey ? (int64_t)gridDim.x * blockDim.x : n;
  for (int64_t t = tid; t < n; t += step) {
    int srel[STACK];
    uint64_t skey[STACK];
    int64_t sp = 0;
    auto push = [&](int r, uint64_t k) -> bool {
      if (sp < STACK) { srel[sp] = r; skey[sp] = k; }
      else if (gkey && sp - STACK < gcap) { gkey[tid * gcap + sp - STACK] = k; grel[tid * gcap + sp - STACK] = r; }
      else return false;
      ++sp;
      return true;
    };
    int64_t count = 0;
    const int64_t out = pass ? offs[t] : 0;
    bool ok = push(rel0, T.rels[rel0].key[t]);
    int32_t val[16];
    while (ok && sp > 0) {
      --sp;
      int r;
      uint64_t k;
      if (sp < STACK) { r = srel[sp]; k = skey[sp]; }
      else { r = grel[tid * gcap + sp - STACK]; k = gkey[tid * gcap + sp - STACK]; }
      const WalkRel& R = T.rels[r];
      uint32_t w;
      if (R.dir && !R.input) {  // direct store still holds the final words: slot = packed key
        const unsigned long long word = R.dir[k];
        if (!word) { atomicOr(err, 1); return; }
        const unsigned long long wc = ~word & R.wmask;
        const unsigned long long vars = wc & ((1ull << R.wT) - 1ull);
        w = (uint32_t)(R.wrb ? (((wc >> R.wT) << (32 - R.wrb)) | vars) : vars);
      } else {
        const int64_t idx = find_key(R, k);
        if (idx < 0) { atomicOr(err, 1); return; }
        w = R.w[idx];
      }
      const int rb = T.rule_bits[r];
      const int lr = rb ? (int)(w >> (32 - rb)) : 0;
      const WalkRule& ru = T.rules[T.rule_base[r] + lr];
      const uint64_t sample = R.has_sample ? (k >> R.sshift) : 0ull;
      for (int v = 0; v < ru.nvars && v < 16; ++v) {
        const int hc = ru.head_col[v];
        if (hc >= 0) {
          val[v] = (int32_t)((k >> R.shift[hc]) & bmask(R.bits[hc])) + R.min[hc];
        } else {
          val[v] = (int32_t)((w >> ru.wshift[v]) & bmask(ru.wbits[v])) + ru.wmin[v];
        }
      }
      for (int a = ru.natoms - 1; a >= 0; --a) {
        const WalkAtom& at = ru.atom[a];
        const WalkRel& A = T.rels[at.rel];
        uint64_t key = A.has_sample ? (sample << A.sshift) : 0ull;
        for (int c = 0; c < at.ncols; ++c) {
          const int32_t x = at.var[c] >= 0 ? val[at.var[c]] : at.cst[c];
          const int64_t f = (int64_t)x - (int64_t)A.min[c];
          if (f < 0 || f > (int64_t)bmask(A.bits[c])) { atomicOr(err, 4); return; }
          key |= (uint64_t)f << A.shift[c];
        }
        if (A.input) {
          count = emit_leaf(A, key, pass, leaves, out, count, err);
          if (count < 0) return;
        } else if (!push(at.rel, key)) {
          ok = false;
          break;
        }
      }
    }
    if (!ok) { atomicOr(err, 2); if (!pass) cnt[t] = 0; continue; }
    if (!pass) cnt[t] = count;
  }
}

// One thread per output tuple: leaves sorted by (tuple << 32 | fact); unique
// (tuple, fact) runs give multiplicities; prefix / suffix products in fp64.
__global__ void grad_k(const uint64_t* __restrict__ tf, const uint32_t* __restrict__ pos, int64_t nleaf,
                       int64_t nuniq, const float* __restrict__ fact_p, int64_t ntup, const int64_t* __restrict__ loff,
                       int64_t* __restrict__ goff, int64_t* __restrict__ gfid, float* __restrict__ gval,
                       double* __restrict__ scratch) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntup) return;
  if (t == ntup) { goff[ntup] = nuniq; return; }
  const int64_t a = loff[t], b = loff[t + 1];
  const int64_t u0 = a < nleaf ? (int64_t)pos[a] : nuniq;
  goff[t] = u0;
  // pass 1: unique facts, multiplicity, prefix products (exclusive) into scratch
  double pre = 1.0;
  int64_t u = u0;
  for (int64_t i = a; i < b;) {
    const uint32_t f = (uint32_t)(tf[i] & 0xffffffffu);
    int64_t j = i;
    while (j < b && (uint32_t)(tf[j] & 0xffffffffu) == f) ++j;
    const int m = (int)(j - i);
    const double p = (double)fact_p[f];
    double pm = 1.0;
    for (int q = 0; q < m; ++q) pm *= p;
    gfid[u] = (int64_t)f;
    gval[u] = (float)m;  // temporarily the multiplicity
    scratch[u] = pre;
    pre *= pm;
    ++u;
    i = j;
  }
  // pass 2: backward with suffix products
  double suf = 1.0;
  for (int64_t v = u - 1; v >= u0; --v) {
    const int m = (int)gval[v];
    const double p = (double)fact_p[gfid[v]];
    double pm1 = 1.0;
    for (int q = 0; q < m - 1; ++q) pm1 *= p;
    gval[v] = (float)((double)m * pm1 * scratch[v] * suf);
    suf *= pm1 * p;
  }
}

// diff-max-min-prob: p = min over the derivation's leaves, so ∂p/∂p_f is one-hot
// on the leaf holding the minimum; leaves are sorted by (tuple, fact), so a
// strict < keeps the smallest fact id among equal minima.
__global__ void grad_onehot_k(const uint64_t* __restrict__ tf, int64_t nleaf, const float* __restrict__ fact_p,
                              int64_t ntup, const int64_t* __restrict__ loff, int64_t* __restrict__ goff,
                              int64_t* __restrict__ gfid, float* __restrict__ gval) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntup) return;
  goff[t] = t;
  if (t == ntup) return;
  uint32_t best = 0;
  float bp = 0.0f;
  for (int64_t i = loff[t], e = loff[t + 1]; i < e && i < nleaf; ++i) {
    const uint32_t f = (uint32_t)(tf[i] & 0xffffffffu);
    const float p = fact_p[f];
    if (i == loff[t] || p < bp) { best = f; bp = p; }
  }
  gfid[t] = (int64_t)best;
  gval[t] = 1.0f;
}

__global__ void unpack_k(const uint64_t* __restrict__ key, int64_t n, int has_sample, int sshift, int ncols,
                         const uint8_t* __restrict__ shift, const uint8_t* __restrict__ bits,
                         const int32_t* __restrict__ mins, int32_t* __restrict__ sample, int32_t* __restrict__ cols) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    sample[i] = has_sample ? (int32_t)(k >> sshift) : 0;
    for (int c = 0; c < ncols; ++c) cols[(int64_t)c * n + i] = (int32_t)((k >> shift[c]) & bmask(bits[c])) + mins[c];
  }
}

__global__ void sample_offsets_k(const uint64_t* __restrict__ key, int64_t n, int32_t batch, int sshift,
                                 int has_sample, int64_t* __restrict__ off) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > batch) return;
  if (!has_sample) { off[s] = s == 0 ? 0 : n; return; }
  off[s] = lower_bound_u64(key, n, (uint64_t)s << sshift);
}

__global__ void grad_contrib_k(const int64_t* __restrict__ goff, const int64_t* __restrict__ gfid,
                               const float* __restrict__ gval, const float* __restrict__ up, int64_t n,
                               uint64_t* __restrict__ key, uint32_t* __restrict__ val) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const float u = up[r];
    for (int64_t g = goff[r]; g < goff[r + 1]; ++g) {
      key[g] = (uint64_t)gfid[g];
      val[g] = f2u(__fmul_rn(u, gval[g]));
    }
  }
}

__global__ void dense_sum_k(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val, int64_t n,
                            float* __restrict__ dense) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    if (i > 0 && key[i - 1] == k) continue;
    double acc = 0.0;
    for (int64_t j = i; j < n && key[j] == k; ++j) acc = __dadd_rn(acc, (double)u2f(val[j]));
    dense[k] = (float)acc;
  }
}

__global__ void add_i32_k(int32_t* __restrict__ a, int64_t n, int32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] += v;
}
__global__ void add_i64_k(const int64_t* __restrict__ s, int64_t n, int64_t v, int64_t* __restrict__ d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i] + v;
}
__global__ void sample_offsets_i32_k(const int32_t* __restrict__ sid, int64_t n, int32_t batch,
                                     int64_t* __restrict__ off) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > batch) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sid[mid] < s) lo = mid + 1; else hi = mid;
  }
  off[s] = lo;
}


// diff-add-mult: per output row i (sorted by (sample, cols)), the first row of
// the adjoint's __grad relation (sorted by (sample, cols, fact)) with the same
// (sample, cols) prefix; goff[n] = ng.  Columns are SoA (column c at c * rows).
__global__ void grad_rows_k(const int32_t* __restrict__ osid, const int32_t* __restrict__ ocols, int64_t n, int k,
                            const int32_t* __restrict__ gsid, const int32_t* __restrict__ gcols, int64_t ng,
                            int64_t* __restrict__ goff) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) {
      goff[n] = ng;
      continue;
    }
    int64_t lo = 0, hi = ng;
    while (lo < hi) {  // first g with (gsid, gcols[0..k)) >= (osid, ocols)
      const int64_t mid = (lo + hi) >> 1;
      int cmp = gsid[mid] < osid[i] ? -1 : (gsid[mid] > osid[i] ? 1 : 0);
      for (int c = 0; c < k && cmp == 0; ++c) {
        const int32_t a = gcols[(int64_t)c * ng + mid], b = ocols[(int64_t)c * n + i];
        cmp = a < b ? -1 : (a > b ? 1 : 0);
      }
      if (cmp < 0) lo = mid + 1; else hi = mid;
    }
    goff[i] = lo;
  }
}

__global__ void widen_i32_k(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

}  // namespace

void launch_add_i32(int32_t* a, int64_t n, int32_t v, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  add_i32_k<<<grid_for(n, 256), 256, 0, st>>>(a, n, v);
}
void launch_add_i64(const int64_t* s, int64_t n, int64_t v, int64_t* d, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  add_i64_k<<<grid_for(n, 256), 256, 0, st>>>(s, n, v, d);
}
void launch_sample_offsets_i32(const int32_t* sid, int64_t n, int32_t batch, int64_t* off, cudaStream_t st) {
  note_launch();
  sample_offsets_i32_k<<<(unsigned)((batch + 1 + 255) / 256), 256, 0, st>>>(sid, n, batch, off);
}

void launch_walk(const WalkTables& T, int rel, int64_t n, int pass, const int64_t* offs, int64_t* cnt,
                 int64_t* leaves, int* err, uint64_t* gkey, int* grel, int64_t gcap, int64_t gthreads,
                 cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  const int64_t thr = gkey ? std::min<int64_t>(n, gthreads) : n;
  walk_k<<<(unsigned)((thr + 127) / 128), 128, 0, st>>>(T, rel, n, pass, offs, cnt, leaves, err, gkey, grel, gcap);
}

void launch_leaf_heads(const uint64_t* k, int64_t n, uint32_t* flag, cudaStream_t st) { launch_heads(k, n, flag, st); }

void launch_grad(const uint64_t* sorted_tf, const uint32_t* pos, int64_t nleaf, int64_t nuniq, const float* fact_p,
                  int64_t ntup, const int64_t* loff, int64_t* goff, int64_t* gfid, float* gval, double* scratch,
                  cudaStream_t st) {
  note_launch();
  grad_k<<<(unsigned)((ntup + 1 + 127) / 128), 128, 0, st>>>(sorted_tf, pos, nleaf, nuniq, fact_p, ntup, loff, goff,
                                                            gfid, gval, scratch);
}

void launch_grad_onehot(const uint64_t* sorted_tf, int64_t nleaf, const float* fact_p, int64_t ntup,
                        const int64_t* loff, int64_t* goff, int64_t* gfid, float* gval, cudaStream_t st) {
  note_launch();
  grad_onehot_k<<<(unsigned)((ntup + 1 + 127) / 128), 128, 0, st>>>(sorted_tf, nleaf, fact_p, ntup, loff, goff, gfid,
                                                                   gval);
}

void launch_unpack(const uint64_t* key, int64_t n, int has_sample, uint8_t sshift, int ncols, const uint8_t* shift,
                   const uint8_t* bits, const int32_t* mins, int32_t* sample, int32_t* cols, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  unpack_k<<<grid_for(n, 256), 256, 0, st>>>(key, n, has_sample, sshift, ncols, shift, bits, mins, sample, cols);
}

void launch_sample_offsets(const uint64_t* key, int64_t n, int32_t batch, uint8_t sshift, int has_sample,
                           int64_t* off, cudaStream_t st) {
  note_launch();
  sample_offsets_k<<<(unsigned)((batch + 1 + 255) / 256), 256, 0, st>>>(key, n, batch, sshift, has_sample, off);
}

void launch_grad_contrib(const int64_t* goff, const int64_t* gfid, const float* gval, const float* upstream,
                         int64_t n, int64_t ng, uint64_t* key, uint32_t* val, cudaStream_t st) {
  (void)ng;
  if (n > 0) {
    note_launch();
    grad_contrib_k<<<grid_for(n, 256), 256, 0, st>>>(goff, gfid, gval, upstream, n, key, val);
  }
}

void launch_dense_sum(const uint64_t* key, const uint32_t* val, const uint32_t* pos, int64_t n, float* dense,
                      cudaStream_t st) {
  (void)pos;
  if (n > 0) {
    note_launch();
    dense_sum_k<<<grid_for(n, 256), 256, 0, st>>>(key, val, n, dense);
  }
}

void launch_grad_rows(const int32_t* osid, const int32_t* ocols, int64_t n, int k, const int32_t* gsid,
                      const int32_t* gcols, int64_t ng, int64_t* goff, cudaStream_t st) {
  note_launch();
  grad_rows_k<<<grid_for(n + 1, 256), 256, 0, st>>>(osid, ocols, n, k, gsid, gcols, ng, goff);
}

void launch_widen_i32(const int32_t* in, int64_t n, int64_t* out, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  widen_i32_k<<<grid_for(n, 256), 256, 0, st>>>(in, n, out);
}

}  // namespace lob
