// k_join.cu — count-then-write join with fused gather, ⊗, projection, filters
// (A3-A5): the `count` / `join` / `gather` / `gather⟨⊗⟩` instructions of
// PAPER.md:359-361 (Table 1), lowered as in Fig. 5 and
// Fig. 10 join_impl, and projection.
//
// Build sides are sorted index keys [prefix | free fields] (static EDB indexes
// are built once per run, §4.2) with optional CSR offsets
// over the dense prefix domain; otherwise binary search.  The write stage is
// balanced over OUTPUT slots (skew-proof for power-law hubs): each slot finds
// its probe row by binary search on the scanned offsets.
#include "device_util.cuh"

namespace lob {
namespace {

__device__ __forceinline__ uint64_t probe_prefix(const JoinPlan& jp, uint64_t pk) {
  uint64_t pre = jp.cprefix;
#pragma unroll
  for (int i = 0; i < MAXM; ++i) {
    if (i < jp.nprem) {
      const Move m = jp.prem[i];
      pre |= ((pk >> m.sshift) & bmask(m.bits)) << m.dshift;
    }
  }
  return pre;
}

__global__ void __launch_bounds__(256) join_count_k(const JoinPlan jp, int64_t* __restrict__ count,
                                                    int64_t* __restrict__ start) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < jp.np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t pk = jp.pkey[i];
    int64_t lo = 0, hi = 0;
    if (pk != KEY_DEAD) {
      const uint64_t pre = probe_prefix(jp, pk);
      if (jp.boff) {
        if (pre < (uint64_t)jp.nprefix) {
          lo = jp.boff[pre];
          hi = jp.boff[pre + 1];
        }
      } else {
        const uint64_t a = pre << jp.free_bits;
        const uint64_t b = (pre + 1) << jp.free_bits;
        lo = lower_bound_u64(jp.bkey, jp.nb, a);  // prefix + free bits <= 63: no overflow
        hi = lower_bound_u64(jp.bkey, jp.nb, b);
      }
    }
    count[i] = hi - lo;
    start[i] = lo;
  }
}

__device__ __forceinline__ float tag_at(const JoinPlan& jp, int idx, int64_t row, int64_t j) {
  float t = 1.0f;
#pragma unroll
  for (int k = 0; k < MAXT; ++k)
    if (k == idx) t = (k < jp.npt) ? jp.ptag[k][row] : 1.0f;
  if (idx == jp.npt) t = jp.btag ? jp.btag[j] : 1.0f;
  return t;
}

// Output-slot tiles: CTA b owns slots [b*WT, (b+1)*WT).  Thread 0 finds the
// tile's probe-row range by binary search on the scanned offsets; when the
// range is small its offsets are staged in shared memory and each slot's row
// is found there (load-balanced expansion, skew-proof).
constexpr int WT = 2048;
constexpr int WROWS = 2048;

__device__ __forceinline__ int64_t smem_row(const int64_t* s, int n, int64_t o) {
  int lo = 0, hi = n;  // largest i with s[i] <= o
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s[mid] <= o) lo = mid + 1; else hi = mid;
  }
  return lo - 1;
}

__global__ void __launch_bounds__(256) join_write_k(const JoinPlan jp, const int64_t* __restrict__ offs,
                                                    const int64_t* __restrict__ start, int64_t total) {
  __shared__ int64_t soff[WROWS];
  __shared__ int64_t r0s, r1s;
  const int64_t o0 = (int64_t)blockIdx.x * WT;
  if (o0 >= total) return;
  const int64_t o1 = (o0 + WT < total ? o0 + WT : total) - 1;
  if (threadIdx.x == 0) {
    r0s = upper_bound_m1_i64(offs, jp.np, o0);
    r1s = upper_bound_m1_i64(offs, jp.np, o1);
  }
  __syncthreads();
  const int64_t r0 = r0s, r1 = r1s;
  const int nrows = (int)(r1 - r0 + 1);
  const bool staged = r1 - r0 + 1 <= WROWS;
  if (staged)
    for (int i = threadIdx.x; i < nrows; i += blockDim.x) soff[i] = offs[r0 + i];
  __syncthreads();
  for (int64_t o = o0 + threadIdx.x; o <= o1; o += blockDim.x) {
    int64_t row;
    if (staged) {
      row = r0 + smem_row(soff, nrows, o);
    } else {
      int64_t lo = r0, hi = r1 + 1;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (offs[mid] <= o) lo = mid + 1; else hi = mid;
      }
      row = lo - 1;
    }
    const int64_t j = start[row] + (o - (staged ? soff[row - r0] : offs[row]));
    const uint64_t pk = jp.pkey[row];
    const uint64_t bk = jp.bkey[j];
    bool ok = true;
    for (int e = 0; e < jp.nfeq; ++e) {
      const Move m = jp.feq[e];
      ok &= ((bk >> m.sshift) & bmask(m.bits)) == ((bk >> m.dshift) & bmask(m.bits));
    }
    for (int c = 0; c < jp.ncmp; ++c) {
      const int64_t a = operand_value(jp.cmp[c].a, pk, bk);
      const int64_t b = operand_value(jp.cmp[c].b, pk, bk);
      ok &= jp.cmp[c].neq ? (a != b) : (a == b);
    }
    const uint64_t key = ok ? (jp.cout | apply_moves(jp.om, jp.nom, pk, bk)) : KEY_DEAD;
    jp.okey[o] = key;
    if (jp.final_step) {
      if (jp.semi == S_UNIT) continue;
      // ⊗ left-deep in body order (reading 9)
      float t = tag_at(jp, jp.tag_order[0], row, j);
      for (int k = 1; k < jp.ntag; ++k) t = otimes(jp.semi, t, tag_at(jp, jp.tag_order[k], row, j));
      if (jp.semi == S_MAXMULT) {
        const uint32_t w = jp.wconst | (uint32_t)apply_moves(jp.wm, jp.nwm, pk, bk);
        jp.oval64[o] = (uint64_t)f2u(t) | ((uint64_t)w << 32);
      } else {
        jp.oval32[o] = f2u(t);
      }
    } else if (jp.semi != S_UNIT) {
      for (int k = 0; k < jp.npt; ++k) jp.otag[k][o] = jp.ptag[k][row];
      jp.otag[jp.npt][o] = jp.btag ? jp.btag[j] : 1.0f;
    }
  }
}

__global__ void __launch_bounds__(256) project_k(const ProjectPlan pp) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pp.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = pp.key[i];
    bool ok = k != KEY_DEAD;
    for (int c = 0; c < pp.ncmp; ++c) {
      const int64_t a = operand_value(pp.cmp[c].a, k, 0);
      const int64_t b = operand_value(pp.cmp[c].b, k, 0);
      ok &= pp.cmp[c].neq ? (a != b) : (a == b);
    }
    pp.okey[i] = ok ? (pp.cout | apply_moves(pp.om, pp.nom, k, 0)) : KEY_DEAD;
    if (pp.semi == S_UNIT) continue;
    const float t = pp.tag ? pp.tag[i] : 1.0f;
    if (pp.semi == S_MAXMULT) {
      const uint32_t w = pp.wconst | (uint32_t)apply_moves(pp.wm, pp.nwm, k, 0);
      pp.oval64[i] = (uint64_t)f2u(t) | ((uint64_t)w << 32);
    } else {
      pp.oval32[i] = f2u(t);
    }
  }
}

struct MoveList {
  Move m[MAXM];
  int n;
};

__global__ void rekey_k(const uint64_t* __restrict__ key, int64_t n, const MoveList ml, uint64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    uint64_t o = 0;
#pragma unroll
    for (int t = 0; t < MAXM; ++t)
      if (t < ml.n) o |= ((k >> ml.m[t].sshift) & bmask(ml.m[t].bits)) << ml.m[t].dshift;
    out[i] = k == KEY_DEAD ? KEY_DEAD : o;
  }
}

__global__ void build_offsets_k(const uint64_t* __restrict__ key, int64_t n, int free_bits, int64_t nprefix,
                                int64_t* __restrict__ off) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p <= nprefix;
       p += (int64_t)gridDim.x * blockDim.x) {
    off[p] = lower_bound_u64(key, n, (uint64_t)p << free_bits);
  }
}

}  // namespace

void launch_join_count(const JoinPlan& jp, int64_t* count, int64_t* start, cudaStream_t st) {
  if (jp.np <= 0) return;
  note_launch();
  join_count_k<<<grid_for(jp.np, 256), 256, 0, st>>>(jp, count, start);
}

void launch_join_write(const JoinPlan& jp, const int64_t* offs, const int64_t* start, int64_t total,
                       cudaStream_t st) {
  if (total <= 0) return;
  note_launch();
  join_write_k<<<(unsigned)((total + WT - 1) / WT), 256, 0, st>>>(jp, offs, start, total);
}

void launch_project(const ProjectPlan& pp, cudaStream_t st) {
  if (pp.n <= 0) return;
  note_launch();
  project_k<<<grid_for(pp.n, 256), 256, 0, st>>>(pp);
}

void launch_rekey(const uint64_t* key, int64_t n, const Move* mv, int nmv, uint64_t* out, cudaStream_t st) {
  if (n <= 0) return;
  MoveList ml = {};
  ml.n = nmv < MAXM ? nmv : MAXM;
  for (int i = 0; i < ml.n; ++i) ml.m[i] = mv[i];
  note_launch();
  rekey_k<<<grid_for(n, 256), 256, 0, st>>>(key, n, ml, out);
}

void launch_build_offsets(const uint64_t* key, int64_t n, int free_bits, int64_t nprefix, int64_t* off,
                          cudaStream_t st) {
  note_launch();
  build_offsets_k<<<grid_for(nprefix + 1, 256), 256, 0, st>>>(key, n, free_bits, nprefix, off);
}

}  // namespace lob
