// k_top1.cu — diff-top-1-proofs tags (§2,
// 617-628 §3.5 "Limitations").
//
// A tag is ONE proof: a sorted set of input-fact ids, at most 300 of them
// (P:628).  ⊗ is the union of the body proofs and fails on a conflict (two
// facts of one exclusion group); ⊕ keeps the more likely proof
// with the diff-max-mult tie rules; p(proof) = Π_{f in proof} p_f in
// fp64 over ascending ids, rounded once (reading "top-1-proof").
//
// Proofs live in a per-relation pool of u32 fact ids; a relation's proof
// index (sorted keys = its stored tuples, offset + length into the pool) is
// updated once per round with the round's Δ'.  The fixpoint itself runs the
// diff-max-mult sorted-store pipeline: a candidate (head key, rule | non-head
// variables) names its body tuples, whose proofs give the union; the union's
// p replaces the candidate's ⊗ before the segmented ⊕, so the standard
// winner selection (max p, then the smallest witness) applies unchanged.
#include "device_util.cuh"

namespace lob {
namespace {

__device__ int64_t pfind(const uint64_t* __restrict__ key, int64_t n, uint64_t k) {
  const int64_t i = lower_bound_u64(key, n, k);
  return (i < n && key[i] == k) ? i : -1;
}

// the body proofs of one candidate (key, witness): up to MAXT sorted lists
struct Lists {
  const uint32_t* p[MAXT];
  int n[MAXT];
  int k;
};

// 0: ok; 1: a body tuple is missing (engine bug); 4: a field outside its domain
__device__ int body_lists(const ProofTables& T, int hrel, uint64_t key, uint32_t w, Lists& L, uint32_t* one) {
  const ProofRel& H = T.rels[hrel];
  const int rb = T.rule_bits[hrel];
  const int lr = rb ? (int)(w >> (32 - rb)) : 0;
  const WalkRule& ru = T.rules[T.rule_base[hrel] + lr];
  const uint64_t sample = H.has_sample ? (key >> H.sshift) : 0ull;
  int32_t val[16];
  for (int v = 0; v < ru.nvars && v < 16; ++v) {
    const int hc = ru.head_col[v];
    val[v] = hc >= 0 ? (int32_t)((key >> H.shift[hc]) & bmask(H.bits[hc])) + H.min[hc]
                     : (int32_t)((w >> ru.wshift[v]) & bmask(ru.wbits[v])) + ru.wmin[v];
  }
  L.k = ru.natoms;
  for (int a = 0; a < ru.natoms; ++a) {
    const WalkAtom& at = ru.atom[a];
    const ProofRel& A = T.rels[at.rel];
    uint64_t k = A.has_sample ? (sample << A.sshift) : 0ull;
    for (int c = 0; c < at.ncols; ++c) {
      const int32_t x = at.var[c] >= 0 ? val[at.var[c]] : at.cst[c];
      const int64_t f = (int64_t)x - (int64_t)A.min[c];
      if (f < 0 || f > (int64_t)bmask(A.bits[c])) return 4;
      k |= (uint64_t)f << A.shift[c];
    }
    const int64_t i = pfind(A.key, A.n, k);
    if (i < 0) return 1;
    if (A.fid) {  // input relation: the proof is the fact itself
      one[a] = (uint32_t)A.fid[i];
      L.p[a] = one + a;
      L.n[a] = 1;
    } else {
      L.p[a] = A.pool + A.pof[i];
      L.n[a] = (int)A.pln[i];
    }
  }
  return 0;
}

// k-way union of the lists in ascending order; MODE 0: length, fp64 product,
// conflict test; MODE 1: also write the ids.  Returns the length, or -1 on a
// conflict.
template <int MODE>
__device__ int union_lists(const ProofTables& T, Lists& L, double& prod, uint32_t* out) {
  int pos[MAXT] = {0, 0, 0, 0, 0, 0};
  int len = 0;
  prod = 1.0;
  uint32_t last = 0xffffffffu;
  for (;;) {
    uint32_t m = 0xffffffffu;
    for (int a = 0; a < L.k; ++a)
      if (pos[a] < L.n[a] && L.p[a][pos[a]] < m) m = L.p[a][pos[a]];
    if (m == 0xffffffffu) break;
    for (int a = 0; a < L.k; ++a)
      if (pos[a] < L.n[a] && L.p[a][pos[a]] == m) ++pos[a];
    if (m == last) continue;
    last = m;
    if (MODE == 0 && T.group) {  // a conflict needs two facts of one group in different lists
      const int32_t g = T.group[m];
      if (g >= 0) {
        for (int a = 0; a < L.k; ++a)
          for (int q = 0; q < L.n[a]; ++q) {
            const uint32_t f = L.p[a][q];
            if (f != m && T.group[f] == g) return -1;
          }
      }
    }
    if (MODE == 0) prod *= (double)T.fact_p[m];
    if (MODE == 1) out[len] = m;
    ++len;
  }
  return len;
}

// candidates (unsorted): p := the union's p (low 32 bits of val), conflicts
// become dead keys, proofs above the cap raise err bit 8
__global__ void top1_cand_k(const ProofTables T, int hrel, uint64_t* __restrict__ key, uint64_t* __restrict__ val,
                            int64_t n, int* __restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    if (k == KEY_DEAD) continue;
    const uint64_t v = val[i];
    Lists L;
    uint32_t one[MAXT];
    const int e = body_lists(T, hrel, k, (uint32_t)(v >> 32), L, one);
    if (e) { atomicOr(err, e); continue; }
    double prod;
    const int len = union_lists<0>(T, L, prod, nullptr);
    if (len < 0) { key[i] = KEY_DEAD; continue; }
    if (len > T.cap) { atomicOr(err, 8); continue; }
    val[i] = (v & 0xffffffff00000000ull) | (uint64_t)__float_as_uint((float)prod);
  }
}

// Δ' rows (key, witness): proof lengths (MODE 0) / ids at offs (MODE 1)
template <int MODE>
__global__ void top1_delta_k(const ProofTables T, int hrel, const uint64_t* __restrict__ key,
                             const uint32_t* __restrict__ w, int64_t n, uint32_t* __restrict__ len,
                             const uint64_t* __restrict__ offs, uint32_t* __restrict__ pool, int* __restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Lists L;
    uint32_t one[MAXT];
    const int e = body_lists(T, hrel, key[i], w[i], L, one);
    if (e) { atomicOr(err, e); if (MODE == 0) len[i] = 0; continue; }
    double prod;
    if (MODE == 0) len[i] = (uint32_t)union_lists<0>(T, L, prod, nullptr);
    else union_lists<1>(T, L, prod, pool + offs[i]);
  }
}

// Δ' rows already in the index (improved tuples) overwrite their handle in
// place; the others are flagged new (isnew = 1)
__global__ void top1_update_k(const uint64_t* __restrict__ pkey, int64_t np, uint64_t* __restrict__ pof,
                              uint32_t* __restrict__ pln, const uint64_t* __restrict__ dkey,
                              const uint64_t* __restrict__ dof, const uint32_t* __restrict__ dln, int64_t nd,
                              uint32_t* __restrict__ isnew) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nd; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = pfind(pkey, np, dkey[j]);
    if (i >= 0) {
      pof[i] = dof[j];
      pln[i] = dln[j];
    }
    isnew[j] = i < 0 ? 1u : 0u;
  }
}

// compaction of the new rows (pos = exclusive scan of isnew)
__global__ void top1_compact_k(const uint64_t* __restrict__ dkey, const uint64_t* __restrict__ dof,
                               const uint32_t* __restrict__ dln, const uint32_t* __restrict__ isnew,
                               const uint32_t* __restrict__ pos, int64_t nd, uint64_t* __restrict__ nkey,
                               uint64_t* __restrict__ nof, uint32_t* __restrict__ nln) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nd; j += (int64_t)gridDim.x * blockDim.x) {
    if (!isnew[j]) continue;
    const uint32_t o = pos[j];
    nkey[o] = dkey[j];
    nof[o] = dof[j];
    nln[o] = dln[j];
  }
}

// merge of two sorted, disjoint indexes by rank: A[i] lands at i + #B keys
// below it, B[j] at j + #A keys below it
__global__ void top1_merge_k(const uint64_t* __restrict__ akey, const uint64_t* __restrict__ aof,
                             const uint32_t* __restrict__ aln, int64_t na, const uint64_t* __restrict__ bkey,
                             const uint64_t* __restrict__ bof, const uint32_t* __restrict__ bln, int64_t nb,
                             uint64_t* __restrict__ okey, uint64_t* __restrict__ oof, uint32_t* __restrict__ oln) {
  const int64_t tot = na + nb;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < na) {
      const int64_t o = t + lower_bound_u64(bkey, nb, akey[t]);
      okey[o] = akey[t];
      oof[o] = aof[t];
      oln[o] = aln[t];
    } else {
      const int64_t j = t - na;
      const int64_t o = j + lower_bound_u64(akey, na, bkey[j]);
      okey[o] = bkey[j];
      oof[o] = bof[j];
      oln[o] = bln[j];
    }
  }
}

// pool compaction: live proofs gathered in index order (offs = scan of pln)
__global__ void top1_gather_k(const uint32_t* __restrict__ pool, const uint64_t* __restrict__ pof,
                              const uint32_t* __restrict__ pln, const uint64_t* __restrict__ noff, int64_t n,
                              uint32_t* __restrict__ npool) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = pof[i], b = noff[i];
    for (uint32_t q = 0; q < pln[i]; ++q) npool[b + q] = pool[a + q];
  }
}

// gradients of an output relation: ∂p/∂p_f = Π_{g in proof, g != f} p_g in
// fp64 (prefix / suffix products over the sorted proof); goff = noff
__global__ void top1_grad_k(const uint32_t* __restrict__ pool, const uint64_t* __restrict__ pof,
                            const uint32_t* __restrict__ pln, const uint64_t* __restrict__ noff, int64_t n,
                            const float* __restrict__ fact_p, int64_t* __restrict__ goff, int64_t* __restrict__ gfid,
                            float* __restrict__ gval, double* __restrict__ scratch) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { goff[n] = n ? (int64_t)(noff[n - 1] + pln[n - 1]) : 0; continue; }
    const uint64_t a = pof[i], o = noff[i];
    const uint32_t m = pln[i];
    goff[i] = (int64_t)o;
    double pre = 1.0;
    for (uint32_t q = 0; q < m; ++q) {
      const uint32_t f = pool[a + q];
      gfid[o + q] = (int64_t)f;
      scratch[o + q] = pre;
      pre *= (double)fact_p[f];
    }
    double suf = 1.0;
    for (int64_t q = (int64_t)m - 1; q >= 0; --q) {
      const uint32_t f = pool[a + q];
      gval[o + q] = (float)(scratch[o + q] * suf);
      suf *= (double)fact_p[f];
    }
  }
}

}  // namespace

void launch_top1_cand(const ProofTables& T, int hrel, uint64_t* key, uint64_t* val, int64_t n, int* err,
                      cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  top1_cand_k<<<grid_for(n, 128), 128, 0, st>>>(T, hrel, key, val, n, err);
}
void launch_top1_delta(const ProofTables& T, int hrel, const uint64_t* key, const uint32_t* w, int64_t n,
                       uint32_t* len, const uint64_t* offs, uint32_t* pool, int* err, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  if (!offs) top1_delta_k<0><<<grid_for(n, 128), 128, 0, st>>>(T, hrel, key, w, n, len, offs, pool, err);
  else top1_delta_k<1><<<grid_for(n, 128), 128, 0, st>>>(T, hrel, key, w, n, len, offs, pool, err);
}
void launch_top1_update(const uint64_t* pkey, int64_t np, uint64_t* pof, uint32_t* pln, const uint64_t* dkey,
                        const uint64_t* dof, const uint32_t* dln, int64_t nd, uint32_t* isnew, cudaStream_t st) {
  if (nd <= 0) return;
  note_launch();
  top1_update_k<<<grid_for(nd, 256), 256, 0, st>>>(pkey, np, pof, pln, dkey, dof, dln, nd, isnew);
}
void launch_top1_compact(const uint64_t* dkey, const uint64_t* dof, const uint32_t* dln, const uint32_t* isnew,
                         const uint32_t* pos, int64_t nd, uint64_t* nkey, uint64_t* nof, uint32_t* nln,
                         cudaStream_t st) {
  if (nd <= 0) return;
  note_launch();
  top1_compact_k<<<grid_for(nd, 256), 256, 0, st>>>(dkey, dof, dln, isnew, pos, nd, nkey, nof, nln);
}
void launch_top1_merge(const uint64_t* akey, const uint64_t* aof, const uint32_t* aln, int64_t na,
                       const uint64_t* bkey, const uint64_t* bof, const uint32_t* bln, int64_t nb, uint64_t* okey,
                       uint64_t* oof, uint32_t* oln, cudaStream_t st) {
  if (na + nb <= 0) return;
  note_launch();
  top1_merge_k<<<grid_for(na + nb, 256), 256, 0, st>>>(akey, aof, aln, na, bkey, bof, bln, nb, okey, oof, oln);
}
void launch_top1_gather(const uint32_t* pool, const uint64_t* pof, const uint32_t* pln, const uint64_t* noff,
                        int64_t n, uint32_t* npool, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  top1_gather_k<<<grid_for(n, 256), 256, 0, st>>>(pool, pof, pln, noff, n, npool);
}
void launch_top1_grad(const uint32_t* pool, const uint64_t* pof, const uint32_t* pln, const uint64_t* noff, int64_t n,
                      const float* fact_p, int64_t* goff, int64_t* gfid, float* gval, double* scratch,
                      cudaStream_t st) {
  note_launch();
  top1_grad_k<<<grid_for(n + 1, 128), 128, 0, st>>>(pool, pof, pln, noff, n, fact_p, goff, gfid, gval, scratch);
}

}  // namespace lob
