// k_join.cu — count-then-write join with fused gather, ⊗, projection, filters
// (A3-A5): the `count` / `join` / `gather` / `gather⟨⊗⟩` instructions of
// PAPER.md:359-361 (Table 1), lowered as in Fig. 5 and
// Fig. 10 join_impl, and projection.
//
// Build sides are sorted index keys [prefix | free fields] (static EDB indexes
// are built once per run, §4.2) with optional CSR offsets
// over the dense prefix domain; otherwise binary search.  The write stage is
// balanced over OUTPUT slots (skew-proof for power-law hubs): each CTA owns a
// tile of output slots, finds its probe-row range once, stages those offsets
// in shared memory and resolves each slot's row there.
//
// Probe / output keys are u32 or u64 (template PK / OK): relations whose
// packed key fits 31 bits move half the key bytes.
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "device_util.cuh"

namespace lob {
namespace {

__device__ __forceinline__ uint64_t probe_prefix(const JoinPlan& jp, uint64_t pk) {
  return jp.cprefix | apply_moves(jp.prem, jp.nprem, pk, 0);
}

template <typename PK>
__global__ void __launch_bounds__(256) join_count_k(const JoinPlan jp, int64_t* __restrict__ count,
                                                    int64_t* __restrict__ start) {
  const PK* __restrict__ pkey = reinterpret_cast<const PK*>(jp.pkey);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < jp.np;
       i += (int64_t)gridDim.x * blockDim.x) {
    const PK pk = pkey[i];
    int64_t lo = 0, hi = 0;
    if (pk != dead<PK>()) {
      const uint64_t pre = probe_prefix(jp, (uint64_t)pk);
      if (jp.boff) {
        if (pre < (uint64_t)jp.nprefix) {
          lo = jp.boff[pre];
          hi = jp.boff[pre + 1];
        }
      } else {
        const uint64_t a = pre << jp.free_bits;  // prefix + free bits <= 63: no overflow
        const uint64_t b = (pre + 1) << jp.free_bits;
        lo = lower_bound_u64(jp.bkey, jp.nb, a);
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

constexpr int WT = 2048;    // output slots per CTA (8 per thread)
constexpr int WROWS = 2048; // probe-row offsets staged in shared memory
constexpr int SPT = WT / 256;

// ⊗ in body order over T = [ptag[0..npt-1], btag] (reading 9).  Fast path:
// one probe tag followed by the build tag (every linear TC-shaped rule).
__device__ __forceinline__ float candidate_tag(const JoinPlan& jp, int semi, int64_t row, int64_t j) {
  if (jp.omin) semi = S_MAXMIN;  // diff-max-min: ⊗ = min
  if (jp.npt == 1 && jp.ntag == 2) {
    const float a = jp.ptag[0][row], b = jp.btag[j];
    return jp.tag_order[0] == 0 ? otimes(semi, a, b) : otimes(semi, b, a);
  }
  if (jp.npt == 2 && jp.ntag == 3) {  // three-atom rules (e.g. C3's composition): 3 loads, no scan
    const float v0 = jp.ptag[0][row], v1 = jp.ptag[1][row], v2 = jp.btag ? jp.btag[j] : 1.0f;
    auto pick = [&](int idx) { return idx == 0 ? v0 : (idx == 1 ? v1 : v2); };
    return otimes(semi, otimes(semi, pick(jp.tag_order[0]), pick(jp.tag_order[1])), pick(jp.tag_order[2]));
  }
  float t = tag_at(jp, jp.tag_order[0], row, j);
#pragma unroll 1
  for (int k = 1; k < jp.ntag; ++k) t = otimes(semi, t, tag_at(jp, jp.tag_order[k], row, j));
  return t;
}

// MODE (compile time, keeps each variant's code small): JW_INTER = intermediate
// rows (final_step 0), JW_CAND = candidates (semiring at run time), JW_DIRECT +
// semiring = direct ⊕ into the dense store.
constexpr int JW_INTER = 0, JW_CAND = 1, JW_DIRECT = 2;

// Tile -> first probe row: row i owns output slots [offs[i], offs[i+1]); every
// tile whose first slot t*WT falls in that range starts at row i.  One pass
// over the offsets (coalesced) instead of a per-CTA search of them.
__global__ void tile_rows_k(const int64_t* __restrict__ offs, int64_t np, int64_t total, int64_t ntiles,
                            int64_t* __restrict__ tile_row) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = offs[i], b = i + 1 < np ? offs[i + 1] : total;
    for (int64_t t = (a + WT - 1) / WT; t * WT < b; ++t) tile_row[t] = i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) tile_row[ntiles] = np - 1;
}

template <typename PK, typename OK, int MODE>
__global__ void __launch_bounds__(256) join_write_k(const JoinPlan jp, const int64_t* __restrict__ offs,
                                                    const int64_t* __restrict__ start, int64_t total,
                                                    const int64_t* __restrict__ tile_row) {
  constexpr bool FINAL = MODE != JW_INTER;
  constexpr bool DIRECT = MODE >= JW_DIRECT;
  const int semi = DIRECT ? MODE - JW_DIRECT : jp.semi;
  // the tile's probe rows, staged: build-index delta start - offs (so a slot's
  // build row is j = sdel + o) and the probe key; srow[k] = the tile-local row
  // of output slot o0 + k, by scattering each row's index to its first slot
  // and an inclusive max-scan over the tile (no per-slot binary search)
  __shared__ int32_t srow[WT];
  __shared__ int64_t sdel[WROWS];
  __shared__ PK spk[WROWS];
  __shared__ int32_t wmax[8];
  const PK* __restrict__ pkey = reinterpret_cast<const PK*>(jp.pkey);
  OK* __restrict__ okey = reinterpret_cast<OK*>(jp.okey);
  const int64_t o0 = (int64_t)blockIdx.x * WT;
  if (o0 >= total) return;
  const int64_t o1 = (o0 + WT < total ? o0 + WT : total) - 1;
  // r1 may overshoot by rows that start after the tile (harmless: they own no slot here)
  const int64_t r0 = tile_row[blockIdx.x];
  const int64_t r1 = tile_row[blockIdx.x + 1];
  const int nrows = (int)(r1 - r0 + 1);
  const bool staged = r1 - r0 + 1 <= WROWS;
  if (staged) {
#pragma unroll
    for (int q = 0; q < SPT; ++q) srow[threadIdx.x + q * 256] = (threadIdx.x + q * 256) == 0 ? 0 : -1;
    __syncthreads();
    for (int i = threadIdx.x; i < nrows; i += blockDim.x) {
      const int64_t of = offs[r0 + i];
      if (of >= o0 && of - o0 < WT) atomicMax(&srow[of - o0], i);  // equal offsets: the last row owns the slots
      sdel[i] = start[r0 + i] - of;
      spk[i] = pkey[r0 + i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int v[SPT];
    int m = -1;
#pragma unroll
    for (int q = 0; q < SPT; ++q) {
      m = max(m, srow[threadIdx.x * SPT + q]);
      v[q] = m;
    }
    int inc = m;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) inc = max(inc, __shfl_up_sync(0xffffffffu, inc, d));
    if (lane == 31) wmax[warp] = inc;
    int ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = -1;
    __syncthreads();
    for (int q = 0; q < warp; ++q) ex = max(ex, wmax[q]);
#pragma unroll
    for (int q = 0; q < SPT; ++q) srow[threadIdx.x * SPT + q] = max(v[q], ex);
  }
  __syncthreads();
  // phase 1: resolve every slot of this thread (independent loads in flight)
  int64_t rowv[SPT], jv[SPT];
  PK pkv[SPT];
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    const int64_t o = o0 + threadIdx.x + k * 256;
    rowv[k] = -1;
    if (o > o1) continue;
    if (staged) {
      const int li = srow[threadIdx.x + k * 256];
      rowv[k] = r0 + li;
      jv[k] = sdel[li] + o;
      pkv[k] = spk[li];
    } else {
      int64_t lo = r0, hi = r1 + 1;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (offs[mid] <= o) lo = mid + 1; else hi = mid;
      }
      const int64_t row = lo - 1;
      rowv[k] = row;
      jv[k] = start[row] + (o - offs[row]);
      pkv[k] = pkey[row];
    }
  }
  uint64_t keyv[SPT];
  float tv[SPT];
  uint32_t wv[SPT];
  bool okv[SPT];
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    okv[k] = false;
    if (rowv[k] < 0) continue;
    const int64_t row = rowv[k];
    const int64_t j = jv[k];
    const uint64_t pk = (uint64_t)pkv[k];
    const uint64_t bk = jp.bkey[j];
    bool ok = true;
    for (int e = 0; e < jp.nfeq; ++e) {
      const Move m = jp.feq[e];
      ok &= ((bk >> m.sshift) & bmask(m.bits)) == ((bk >> m.dshift) & bmask(m.bits));
    }
    for (int c = 0; c < jp.ncmp; ++c) {
      const int64_t a = operand_value(jp.cmp[c].a, pk, bk);
      const int64_t b = operand_value(jp.cmp[c].b, pk, bk);
      ok &= cmp_holds(jp.cmp[c].neq, a, b);
    }
    okv[k] = ok;
    keyv[k] = jp.cout | apply_moves(jp.om, jp.nom, pk, bk);
    tv[k] = 1.0f;
    wv[k] = 0;
    if (FINAL && semi != S_UNIT) {
      tv[k] = candidate_tag(jp, semi, row, j);
      if (semi == S_MAXMULT) wv[k] = jp.wconst | (uint32_t)apply_moves(jp.wm, jp.nwm, pk, bk);
    }
  }
  // phase 2: emit
  if constexpr (DIRECT) {  // fused A5-A8: ⊕ straight into the direct-mapped store
    if (!jp.aggregate) {
      // stale-read filter, then this thread's remaining atomics back to back
      unsigned long long oldv[SPT], newv[SPT];
      uint32_t slotv[SPT];
      bool live[SPT];
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        live[k] = rowv[k] >= 0 && okv[k];
        if (!live[k]) continue;
        slotv[k] = (uint32_t)keyv[k];
        newv[k] = direct_pack(semi, slotv[k], tv[k], wv[k], jp.mx);
        oldv[k] = direct_peek(semi, jp.fdir, slotv[k]);
      }
      direct_commit<SPT>(semi, jp.fdir, jp.dirty, slotv, newv, oldv, live);
    } else {  // narrow heads (rare): warp pre-aggregation, rolled to keep the code small
#pragma unroll 1
      for (int k = 0; k < SPT; ++k)
        if (rowv[k] >= 0 && okv[k])
          direct_oplus(semi, jp.fdir, (uint32_t)keyv[k], tv[k], wv[k], jp.dirty, jp.aggregate, jp.mx);
    }
  } else {
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      if (rowv[k] < 0) continue;
      const int64_t o = o0 + threadIdx.x + k * 256;
      okey[o] = okv[k] ? (OK)keyv[k] : dead<OK>();
      if (semi == S_UNIT) continue;
      if constexpr (FINAL) {
        if (semi == S_MAXMULT) jp.oval64[o] = (uint64_t)f2u(tv[k]) | ((uint64_t)wv[k] << 32);
        else jp.oval32[o] = f2u(tv[k]);
      } else {
        const int64_t row = rowv[k];
#pragma unroll 1
        for (int q = 0; q < jp.npt; ++q) jp.otag[q][o] = jp.ptag[q][row];
        jp.otag[jp.npt][o] = jp.btag ? jp.btag[jv[k]] : 1.0f;
      }
    }
  }
}

template <typename PK, typename OK>
__global__ void __launch_bounds__(256) project_k(const ProjectPlan pp) {
  const PK* __restrict__ key = reinterpret_cast<const PK*>(pp.key);
  OK* __restrict__ okey = reinterpret_cast<OK*>(pp.okey);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pp.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const PK kk = key[i];
    const uint64_t k = (uint64_t)kk;
    bool ok = kk != dead<PK>();
    for (int c = 0; c < pp.ncmp; ++c) {
      const int64_t a = operand_value(pp.cmp[c].a, k, 0);
      const int64_t b = operand_value(pp.cmp[c].b, k, 0);
      ok &= cmp_holds(pp.cmp[c].neq, a, b);
    }
    uint64_t hk = pp.cout | apply_moves(pp.om, pp.nom, k, 0);
    for (int f = 0; f < pp.nbf && ok; ++f) {  // expression comparisons (bytecode)
      int32_t a, b;
      ok = bc_eval(pp.bf[f].lhs, k, a) && bc_eval(pp.bf[f].rhs, k, b) && cmp_holds(pp.bf[f].rel, a, b);
    }
    for (int e = 0; e < pp.nbh && ok; ++e) {  // computed head columns (bytecode)
      int32_t v;
      ok = bc_eval(pp.bh[e].e, k, v);
      const int64_t f = (int64_t)v - pp.bh[e].base;
      ok = ok && f >= 0 && f < ((int64_t)1 << pp.bh[e].bits);
      if (ok) hk |= (uint64_t)f << pp.bh[e].dshift;
    }
    if (pp.direct) {
      if (ok) {
        const float t = (pp.semi != S_UNIT && pp.tag) ? pp.tag[i] : 1.0f;
        const uint32_t w = pp.semi == S_MAXMULT ? (pp.wconst | (uint32_t)apply_moves(pp.wm, pp.nwm, k, 0)) : 0u;
        direct_oplus(pp.semi, pp.fdir, (uint32_t)hk, t, w, pp.dirty, pp.aggregate, pp.mx);
      }
      continue;
    }
    okey[i] = ok ? (OK)hk : dead<OK>();
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

// Row-centric fused join + direct ⊕ for bounded fan-out (every prefix of the
// static CSR index has <= MAXDEG rows, e.g. lattice edges: 4).  One thread per
// probe row: coalesced probe key / tag loads, its matches unrolled, all
// updates issued before any result is consumed.  No count / scan / host sync.
// Specialised on the semiring and on the longest move list (NM: 2, 4 or MAXM
// bit moves for prefix / slot / witness) — the generic kernel was 3.7k SASS
// instructions and stalled on instruction fetch (ncu: 21% no_instruction).
// Measured on C2 and rejected: two rows per thread (152 vs 101 us per launch:
// fewer resident warps for the same requests in flight; re-measured with the
// specialised kernel, 8-B paired key/tag loads and all 8 peeks in flight:
// +30%, 48 registers with spills), a fixed-width ELL
// copy of the build index replacing boff -> bkey (+3%: boff hits L1), a
// software pipeline prefetching row i+stride's key and CSR range (+22%),
// grids other than one wave of resident CTAs in async rounds (2 or 4 waves:
// +7% / +15%; 4 or 3 CTAs per SM: +8% / +24%),
// warp-merged dirty-bit updates (__match_any_sync + __reduce_or_sync per
// direction: +29%, the warp collectives cost more than the REDs they save),
// and (for join_write_k too) u32 copies of the build keys' free bits (no
// change on C4, +1% on C2/C3: build rows are L2-resident already), and a
// window variant for TC-shaped heads (the CTA's 256 rows max-reduce their
// candidates over two 1024-slot shared-memory windows, one global update per
// touched slot: +49% — the zero / flush passes and two barriers per 256 rows
// cost more than the global operations saved).
#ifndef FJ_MINB
#define FJ_MINB 6
#endif
template <int NM>
__device__ __forceinline__ uint64_t moves_n(const Move* mv, int n, uint64_t a, uint64_t b) {
  uint64_t o = 0;
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    if (i < n) {
      const Move m = mv[i];
      const uint64_t s = m.src ? b : a;
      o |= ((s >> m.sshift) & ((1ull << m.bits) - 1ull)) << m.dshift;
    }
  }
  return o;
}

// resident CTAs per SM: 6 (40 registers) except max-mult, whose 64-bit words
// need 48 registers to stay out of local memory (5).  Re-measured after the
// per-CTA candidate counters (scripts/ab.sh, same box): 7 or 8 / 6 CTAs per SM
// spill 24-32 B and run 4-6% slower on C2 (23.1-23.5 vs 22.0-22.3 ms), 2-3% on C5.
#ifndef FJ_MINB_MX
#define FJ_MINB_MX 5
#endif
// The stale read is a relaxed GPU-scope load (device_util.cuh ld_relaxed):
// slots only grow, so any value it returns is a lower bound of the slot and
// >= its round-start value.  (A plain ld.ca through L1 was 1% faster but
// formally a data race with the other threads' atomics.)
#define PEEK PEEK_SLOT
template <typename PK, int MAXDEG, int SEMI, int NM, bool REC>
__global__ void __launch_bounds__(256, (MAXDEG <= 4) ? (SEMI == S_MAXMULT ? FJ_MINB_MX : FJ_MINB) : 4)
    join_rows_direct_k(const JoinPlan jp,
                                                          unsigned long long* __restrict__ ncand) {
  const PK* __restrict__ pkey = reinterpret_cast<const PK*>(jp.pkey);
  uint32_t mycount = 0;
  int64_t np = jp.np;
  if (jp.np_dev) {
    const int64_t nd = (int64_t)*jp.np_dev;
    np = nd < np ? nd : np;
  }
  const int ncmp = jp.ncmp;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
    // the next grid-stride row's key and tag into L2 (no registers held): the
    // chain key -> record -> slot peek then starts from an L2 hit
    if (jp.prefetch && i + stride < np) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pkey + i + stride));
      if (SEMI != S_UNIT) asm volatile("prefetch.global.L2 [%0];" ::"l"(jp.ptag[0] + i + stride));
    }
    const PK pkr = pkey[i];
    if (pkr == dead<PK>()) continue;
    const uint64_t pk = (uint64_t)pkr;
    const uint64_t pre = jp.cprefix | moves_n<NM>(jp.prem, jp.nprem, pk, 0);
    if (pre >= (uint64_t)jp.nprefix) continue;
    // build rows of the prefix: CSR range, or (REC) one 32-B record = one sector
    int64_t lo = 0;
    int n = 0;
    uint32_t rk[REC ? 4 : 1];
    float rt[REC ? 4 : 1];
    if constexpr (REC) {
      const uint4 kk = __ldg(jp.brec + 2 * pre);
      rk[0] = kk.x; rk[1] = kk.y; rk[2] = kk.z; rk[3] = kk.w;
      n = (kk.x != ~0u) + (kk.y != ~0u) + (kk.z != ~0u) + (kk.w != ~0u);
      if (SEMI != S_UNIT) {
        const uint4 tt = __ldg(jp.brec + 2 * pre + 1);
        rt[0] = u2f(tt.x); rt[1] = u2f(tt.y); rt[2] = u2f(tt.z); rt[3] = u2f(tt.w);
      }
    } else {
      lo = jp.boff[pre];
      n = (int)(jp.boff[pre + 1] - lo);
    }
    mycount += (uint32_t)n;
    const float pt = SEMI != S_UNIT ? jp.ptag[0][i] : 1.0f;
    // word-sized values (u32 for unit / max-min): no wasted registers
    using VW = typename std::conditional<SEMI == S_MAXMULT, unsigned long long, uint32_t>::type;
    VW oldv[MAXDEG], newv[MAXDEG];
    uint32_t slotv[MAXDEG];
    bool live[MAXDEG];
    // phase A: candidate slot + packed value, and a plain (possibly stale) read
    // of the slot.  The store is monotone (atomicMax / OR only), so a stale
    // read is a lower bound: a candidate not above it can never improve the
    // slot and needs no atomic.
#pragma unroll
    for (int d = 0; d < MAXDEG; ++d) {
      live[d] = false;
      if (d >= n) continue;
      uint64_t bk;
      float bt = 1.0f;
      if constexpr (REC) {
        bk = rk[d];
        if (SEMI != S_UNIT) bt = rt[d];
      } else {
        bk = jp.bkey[lo + d];
        if (SEMI != S_UNIT) bt = jp.btag[lo + d];
      }
      bool ok = true;
      for (int c = 0; c < ncmp; ++c) {
        const int64_t a = operand_value(jp.cmp[c].a, pk, bk);
        const int64_t b = operand_value(jp.cmp[c].b, pk, bk);
        ok &= cmp_holds(jp.cmp[c].neq, a, b);
      }
      if (!ok) continue;
      const uint32_t slot = (uint32_t)(jp.cout | moves_n<NM>(jp.om, jp.nom, pk, bk));
      slotv[d] = slot;
      live[d] = true;
      if (SEMI == S_UNIT) {
        newv[d] = 1u << (slot & 31u);
        oldv[d] = PEEK(reinterpret_cast<const uint32_t*>(jp.fdir) + (slot >> 5));
        continue;
      }
      const int osemi = (SEMI == S_MAXMULT && jp.omin) ? S_MAXMIN : SEMI;  // diff-max-min: ⊗ = min
      const float t = jp.tag_order[0] == 0 ? otimes(osemi, pt, bt) : otimes(osemi, bt, pt);
      if (SEMI == S_MAXMIN) {
        newv[d] = mm_word(t);
        oldv[d] = PEEK(reinterpret_cast<const uint32_t*>(jp.fdir) + slot);
      } else {
        const uint32_t w = jp.wconst | (uint32_t)moves_n<NM>(jp.wm, jp.nwm, pk, bk);
        newv[d] = mx_word(t, w, jp.mx);
        oldv[d] = PEEK(reinterpret_cast<const unsigned long long*>(jp.fdir) + slot);
      }
    }
    // phase B: fire-and-forget reductions (RED, no return) for candidates above
    // the stale bound.  The read is >= the slot's value at round start (slots
    // only grow; earlier kernels' writes are visible), so v > read means the
    // slot ends the round strictly above its settled value: it IS in Δ' and
    // its dirty bit is set unconditionally (idempotent OR) — no need to learn
    // from the atomic's old value who improved first.
#pragma unroll
    for (int d = 0; d < MAXDEG; ++d) {
      if (!live[d]) continue;
      const VW v = newv[d];
      if (SEMI == S_UNIT) {
        if (oldv[d] & v) continue;
        atomicOr(reinterpret_cast<uint32_t*>(jp.fdir) + (slotv[d] >> 5), (uint32_t)v);
      } else if (SEMI == S_MAXMIN) {
        if (v <= oldv[d]) continue;
        atomicMax(reinterpret_cast<uint32_t*>(jp.fdir) + slotv[d], (uint32_t)v);
      } else {
        if (v <= oldv[d]) continue;
        atomicMax(reinterpret_cast<unsigned long long*>(jp.fdir) + slotv[d], (unsigned long long)v);
      }
      atomicOr(jp.dirty + (slotv[d] >> 5), 1u << (slotv[d] & 31u));
    }
  }
  cta_count_add(ncand, mycount);
}

// 32-bit fast path of the fused join (the C2 / C5 hot kernel): probe keys,
// record keys, slots and witnesses all fit 32 bits, the rule has no filter
// and no repeated free variable, every move list has <= 2 moves.  The plan is
// pre-split on the host into the probe row's part (prefix, slot and witness
// bits taken from the probe key: once per row) and the build side's part
// (once per candidate), each move as ((x >> r) & m) << l with unused moves
// masked to 0, so no loop over move descriptors and no 64-bit bit moves run
// per candidate (the generic kernel spent ~430 instructions per probe row,
// 19% of them parameter loads: ncu, profiles/ncu_full_r02_fj_before.txt).
struct Mv32 {
  uint32_t r[2], m[2], l[2];
};
struct Fast32 {
  Mv32 pre, slot_a, slot_b, w_a, w_b;
  uint32_t cprefix, cout, wconst;
  int tag_first_probe;  // ⊗ order: probe tag first (1) or build tag first (0)
};
__device__ __forceinline__ uint32_t mv32(const Mv32& v, uint32_t x) {
  return (((x >> v.r[0]) & v.m[0]) << v.l[0]) | (((x >> v.r[1]) & v.m[1]) << v.l[1]);
}

template <int SEMI>
__global__ void __launch_bounds__(256, SEMI == S_MAXMULT ? FJ_MINB_MX : FJ_MINB)
    join_rows_rec32_k(const JoinPlan jp, const Fast32 f, unsigned long long* __restrict__ ncand) {
  const uint32_t* __restrict__ pkey = reinterpret_cast<const uint32_t*>(jp.pkey);
  const float* __restrict__ ptag = jp.ptag[0];
  const uint4* __restrict__ brec = jp.brec;
  uint32_t* __restrict__ dirty = jp.dirty;
  const uint32_t nprefix = (uint32_t)jp.nprefix;
  const bool omin = jp.omin;
  const unsigned long long stamp = jp.mx.stamp, wmask = jp.mx.wmask;
  uint32_t mycount = 0;
  int64_t np = jp.np;
  if (jp.np_dev) {
    const int64_t nd = (int64_t)*jp.np_dev;
    np = nd < np ? nd : np;
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
    if (jp.prefetch && i + stride < np) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pkey + i + stride));
      if (SEMI != S_UNIT) asm volatile("prefetch.global.L2 [%0];" ::"l"(ptag + i + stride));
    }
    const uint32_t pk = pkey[i];
    if (pk == 0xffffffffu) continue;
    const uint32_t pre = f.cprefix | mv32(f.pre, pk);
    if (pre >= nprefix) continue;
    const uint4 kk = __ldg(brec + 2 * (size_t)pre);
    uint4 tt = make_uint4(0, 0, 0, 0);
    if (SEMI != S_UNIT) tt = __ldg(brec + 2 * (size_t)pre + 1);
    const float pt = SEMI != S_UNIT ? ptag[i] : 1.0f;
    const uint32_t slot_row = f.cout | mv32(f.slot_a, pk);
    const uint32_t w_row = f.wconst | mv32(f.w_a, pk);
    const uint32_t rk[4] = {kk.x, kk.y, kk.z, kk.w};
    const uint32_t rt[4] = {tt.x, tt.y, tt.z, tt.w};
    using VW = typename std::conditional<SEMI == S_MAXMULT, unsigned long long, uint32_t>::type;
    VW oldv[4], newv[4];
    uint32_t slotv[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const uint32_t bk = rk[d];
      if (bk == 0xffffffffu) { slotv[d] = 0xffffffffu; continue; }
      ++mycount;
      const uint32_t slot = slot_row | mv32(f.slot_b, bk);
      slotv[d] = slot;
      if (SEMI == S_UNIT) {
        newv[d] = 1u << (slot & 31u);
        oldv[d] = PEEK(reinterpret_cast<const uint32_t*>(jp.fdir) + (slot >> 5));
        continue;
      }
      const float bt = __uint_as_float(rt[d]);
      float t;
      if (SEMI == S_MAXMIN || omin) t = pt < bt ? pt : bt;
      else t = f.tag_first_probe ? __fmul_rn(pt, bt) : __fmul_rn(bt, pt);
      if (SEMI == S_MAXMIN) {
        newv[d] = mm_word(t);
        oldv[d] = PEEK(reinterpret_cast<const uint32_t*>(jp.fdir) + slot);
      } else {
        const uint32_t w = w_row | mv32(f.w_b, bk);
        newv[d] = ((unsigned long long)(__float_as_uint(t) + 1u) << 34) | stamp | ((unsigned long long)(~w) & wmask);
        oldv[d] = PEEK(reinterpret_cast<const unsigned long long*>(jp.fdir) + slot);
      }
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      if (slotv[d] == 0xffffffffu) continue;
      const VW v = newv[d];
      if (SEMI == S_UNIT) {
        if (oldv[d] & v) continue;
        atomicOr(reinterpret_cast<uint32_t*>(jp.fdir) + (slotv[d] >> 5), (uint32_t)v);
      } else if (SEMI == S_MAXMIN) {
        if (v <= oldv[d]) continue;
        atomicMax(reinterpret_cast<uint32_t*>(jp.fdir) + slotv[d], (uint32_t)v);
      } else {
        if (v <= oldv[d]) continue;
        atomicMax(reinterpret_cast<unsigned long long*>(jp.fdir) + slotv[d], (unsigned long long)v);
      }
      atomicOr(dirty + (slotv[d] >> 5), 1u << (slotv[d] & 31u));
    }
  }
  cta_count_add(ncand, mycount);
}

// host: split a move list by source into two 32-bit move pairs; false when a
// list needs more than two moves per source or a field leaves 32 bits
static bool split_moves32(const Move* mv, int n, Mv32& a, Mv32& b) {
  int na = 0, nb = 0;
  a = Mv32{{0, 0}, {0, 0}, {0, 0}};
  b = a;
  for (int i = 0; i < n; ++i) {
    const Move& m = mv[i];
    if (m.sshift + m.bits > 32 || m.dshift + m.bits > 32 || m.bits == 0) return false;
    Mv32& t = m.src ? b : a;
    int& k = m.src ? nb : na;
    if (k >= 2) return false;
    t.r[k] = m.sshift;
    t.m[k] = m.bits >= 32 ? 0xffffffffu : ((1u << m.bits) - 1u);
    t.l[k] = m.dshift;
    ++k;
  }
  return true;
}

static bool fast32_plan(const JoinPlan& jp, Fast32& f) {
  if (!jp.pk32 || !jp.brec || jp.ncmp || jp.nfeq || jp.npt != 1) return false;
  if (jp.cprefix >> 32 || jp.cout >> 32 || jp.nprefix > 0xffffffffll) return false;
  Mv32 dummy;
  if (!split_moves32(jp.prem, jp.nprem, f.pre, dummy)) return false;
  for (int k = 0; k < 2; ++k)
    if (dummy.m[k]) return false;  // the prefix is built from the probe key only
  if (!split_moves32(jp.om, jp.nom, f.slot_a, f.slot_b)) return false;
  if (jp.semi == S_MAXMULT && !split_moves32(jp.wm, jp.nwm, f.w_a, f.w_b)) return false;
  if (jp.semi != S_MAXMULT) f.w_a = f.w_b = Mv32{{0, 0}, {0, 0}, {0, 0}};
  if (jp.ntag != 2 && jp.semi != S_UNIT) return false;
  f.cprefix = (uint32_t)jp.cprefix;
  f.cout = (uint32_t)jp.cout;
  f.wconst = jp.wconst;
  f.tag_first_probe = jp.tag_order[0] == 0 ? 1 : 0;
  return true;
}

// MODE: LC_CAND = candidates (semiring at run time), LC_DIRECT + semiring =
// direct ⊕ into the dense store (compile time: small code, no semiring branches).
constexpr int LC_CAND = 0, LC_DIRECT = 1;

// One probe row of a lookup chain: filters, point lookups, ⊗ in body order,
// witness and head key.  Returns whether the row yields a candidate.  (A
// per-prefix tag table replacing the offsets -> tag loads of a point lookup
// was measured on C2's endpoints_connected: no change — not load-bound.)
// probe row i: its key and tag, from the probe arrays or (pdir) a direct store's
// slot word (slot i present <=> row exists; key = slot)
template <typename PK>
__device__ __forceinline__ PK lookup_probe(const LookupPlan& lp, int semi, int64_t i, float& p0) {
  p0 = 1.0f;
  if (lp.pdir) {
    if (semi == S_UNIT) {
      const uint32_t wd = reinterpret_cast<const uint32_t*>(lp.pdir)[i >> 5];
      return ((wd >> (i & 31)) & 1u) ? (PK)i : dead<PK>();
    }
    if (semi == S_MAXMIN) {
      const uint32_t v = reinterpret_cast<const uint32_t*>(lp.pdir)[i];
      p0 = mm_p(v);
      return v ? (PK)i : dead<PK>();
    }
    const unsigned long long v = reinterpret_cast<const unsigned long long*>(lp.pdir)[i];
    p0 = mx_p(v);
    return v ? (PK)i : dead<PK>();
  }
  const PK k = reinterpret_cast<const PK*>(lp.pkey)[i];
  if (semi != S_UNIT && lp.ptag && k != dead<PK>()) p0 = lp.ptag[i];
  return k;
}

template <typename PK, int NM>
__device__ __forceinline__ bool lookup_row(const LookupPlan& lp, int semi, PK pkr, float p0, float& t, uint32_t& w,
                                           uint64_t& key) {
  bool ok = pkr != dead<PK>();
  const uint64_t pk = (uint64_t)pkr;
#pragma unroll 1
  for (int c = 0; c < lp.ncmp; ++c) {
    const int64_t a = operand_value(lp.cmp[c].a, pk, 0);
    const int64_t b = operand_value(lp.cmp[c].b, pk, 0);
    ok &= cmp_holds(lp.cmp[c].neq, a, b);
  }
  float tags[MAXL + 1];
  tags[0] = p0;
#pragma unroll
  for (int l = 0; l < MAXL; ++l) {
    tags[l + 1] = 1.0f;
    if (l >= lp.nlk || !ok) continue;
    const Lookup& L = lp.lk[l];
    const uint64_t pre = L.cprefix | (NM ? moves_n<NM>(L.prem, L.nprem, pk, 0) : apply_moves(L.prem, L.nprem, pk, 0));
    int64_t j = -1;
    if (L.boff) {
      if (pre < (uint64_t)L.nprefix) {
        const int64_t b0 = L.boff[pre];
        if (L.boff[pre + 1] > b0) j = b0;
      }
    } else {
      const int64_t q = lower_bound_u64(L.bkey, L.nb, pre);
      if (q < L.nb && L.bkey[q] == pre) j = q;
    }
    if (j < 0) ok = false;
    else if (semi != S_UNIT && L.btag) tags[l + 1] = L.btag[j];
  }
  t = 1.0f;
  w = 0;
  if (ok && semi != S_UNIT) {
    auto pick = [&](int idx) {
      float r = tags[0];
#pragma unroll
      for (int k = 1; k <= MAXL; ++k)
        if (k == idx) r = tags[k];
      return r;
    };
    t = pick(lp.tag_order[0]);
#pragma unroll 1
    for (int k = 1; k < lp.ntag; ++k) t = otimes(lp.omin ? S_MAXMIN : semi, t, pick(lp.tag_order[k]));
    if (semi == S_MAXMULT)
      w = lp.wconst | (uint32_t)(NM ? moves_n<NM>(lp.wm, lp.nwm, pk, 0) : apply_moves(lp.wm, lp.nwm, pk, 0));
  }
  key = lp.cout | (NM ? moves_n<NM>(lp.om, lp.nom, pk, 0) : apply_moves(lp.om, lp.nom, pk, 0));
  return ok;
}

template <int SEMI>
__device__ __forceinline__ unsigned long long agg_pack(float p, uint32_t w, const MxEnc& mx) {
  if (SEMI == S_MAXMIN) return (unsigned long long)mm_word(p);
  if (SEMI == S_MAXMULT) return mx_word(p, w, mx);
  return 1ull;
}

// warp max of the lanes' packed values, one atomic for the warp's slot
template <int SEMI>
__device__ __forceinline__ void agg_flush(void* f, uint32_t* dirty, uint32_t slot, unsigned long long v) {
  if (SEMI == S_MAXMIN) {
    const uint32_t m = __reduce_max_sync(0xffffffffu, (uint32_t)v);
    if ((threadIdx.x & 31) == 0 && m) {
      const uint32_t old = atomicMax(reinterpret_cast<uint32_t*>(f) + slot, m);
      if (old < m) atomicOr(dirty + (slot >> 5), 1u << (slot & 31u));
    }
  } else if (SEMI == S_MAXMULT) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long u = __shfl_xor_sync(0xffffffffu, v, d);
      v = u > v ? u : v;
    }
    if ((threadIdx.x & 31) == 0 && v) {
      const unsigned long long old = atomicMax(reinterpret_cast<unsigned long long*>(f) + slot, v);
      if (old < v) atomicOr(dirty + (slot >> 5), 1u << (slot & 31u));
    }
  } else {
    if (__any_sync(0xffffffffu, v != 0ull) && (threadIdx.x & 31) == 0) {
      const uint32_t bit = 1u << (slot & 31u);
      const uint32_t old = atomicOr(reinterpret_cast<uint32_t*>(f) + (slot >> 5), bit);
      if (!(old & bit)) atomicOr(dirty + (slot >> 5), bit);
    }
  }
}

// NM: 2 when every move list (prefixes, head, witness) has <= 2 moves, else 0 (generic)
template <typename PK, typename OK, int MODE, int NM>
__global__ void __launch_bounds__(256) lookup_chain_k(const LookupPlan lp, unsigned long long* __restrict__ ncand) {
  constexpr bool DIRECT = MODE >= LC_DIRECT;
  constexpr int SEMI_C = DIRECT ? MODE - LC_DIRECT : -1;
  const int semi = DIRECT ? SEMI_C : lp.semi;
  OK* __restrict__ okey = reinterpret_cast<OK*>(lp.okey);
  uint32_t mycount = 0;
  if (DIRECT && lp.aggregate) {
    // Narrow head (e.g. endpoints_connected(): ~1M candidates per slot, rows
    // sorted by sample): each warp walks a contiguous chunk 32 rows at a time
    // and keeps a per-lane running max while all its live rows aim at one
    // slot; one warp reduction + one atomic per (warp, slot) segment instead
    // of one per 32 rows (same-address atomics serialise in L2).
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t chunk = ((lp.np + nwarps - 1) / nwarps + 31) & ~(int64_t)31;
    const int64_t r0 = wid * chunk, r1 = r0 + chunk < lp.np ? r0 + chunk : lp.np;
    uint32_t cur = 0xffffffffu;
    unsigned long long run = 0;
    for (int64_t base = r0; base < r1; base += 32) {
      const int64_t i = base + (threadIdx.x & 31);
      float p0 = 1.0f;
      const PK pkr = i < r1 ? lookup_probe<PK>(lp, SEMI_C, i, p0) : dead<PK>();
      float t;
      uint32_t w;
      uint64_t key;
      const bool ok = lookup_row<PK, NM>(lp, SEMI_C, pkr, p0, t, w, key);
      if (ok) ++mycount;
      const uint32_t slot = (uint32_t)key;
      const unsigned act = __ballot_sync(0xffffffffu, ok);
      if (!act) continue;
      const uint32_t s0 = __shfl_sync(0xffffffffu, slot, __ffs(act) - 1);
      const bool uniform = __all_sync(0xffffffffu, !ok || slot == s0);
      if (uniform && s0 == cur) {
        const unsigned long long v = ok ? agg_pack<SEMI_C>(t, w, lp.mx) : 0ull;
        run = v > run ? v : run;
        continue;
      }
      if (cur != 0xffffffffu) agg_flush<SEMI_C>(lp.fdir, lp.dirty, cur, run);
      run = 0;
      cur = 0xffffffffu;
      if (uniform) {
        cur = s0;
        run = ok ? agg_pack<SEMI_C>(t, w, lp.mx) : 0ull;
      } else if (ok) {
        direct_oplus(SEMI_C, lp.fdir, slot, t, w, lp.dirty, 1, lp.mx);
      }
    }
    if (cur != 0xffffffffu) agg_flush<SEMI_C>(lp.fdir, lp.dirty, cur, run);
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < lp.np;
         i += (int64_t)gridDim.x * blockDim.x) {
      float t, p0;
      uint32_t w;
      uint64_t key;
      const PK pkr = lookup_probe<PK>(lp, semi, i, p0);
      const bool ok = lookup_row<PK, NM>(lp, semi, pkr, p0, t, w, key);
      if (ok) ++mycount;
      if constexpr (DIRECT) {
        if (ok) direct_oplus(SEMI_C, lp.fdir, (uint32_t)key, t, w, lp.dirty, 0, lp.mx);
      } else {
        okey[i] = ok ? (OK)key : dead<OK>();
        if (semi == S_MAXMULT) lp.oval64[i] = (uint64_t)f2u(t) | ((uint64_t)w << 32);
        else if (semi != S_UNIT) lp.oval32[i] = f2u(t);
      }
    }
  }
  cta_count_add(ncand, mycount);
}

// (ncu of this kernel on C2: 0.57 ms per fixpoint, issue-bound — 71% issue
// slots busy, IPC 2.8, all lanes active; issuing four rows' loads before
// folding them measured no faster, so the single-row loop stays.)
// 32-bit fast path of an aggregating lookup chain over a direct store (C2 /
// C5 `endpoints_connected() :- is_endpoint(x), is_endpoint(y), path(x, y),
// x != y`: every path slot probes two point lookups into a narrow head).  The
// generic row (64-bit operands, move-list loops, run-time ⊗ order, a binary
// search compiled in) spent ~500 thread instructions per probe row; here the
// plan is pre-split on the host into 32-bit single-source move pairs, field
// comparisons and a fixed ⊗ order.  Same filters, lookups, ⊗ order, witness
// and head key as lookup_row.
struct LOpnd32 {
  uint32_t shift, mask;  // field = (pk >> shift) & mask (mask 0: constant)
  int64_t base;          // field min or the constant
};
struct LFast32 {
  int nlk, ncmp, ntag;
  Mv32 pre[MAXL];
  uint32_t cprefix[MAXL], nprefix[MAXL];
  LOpnd32 ca[MAXC], cb[MAXC];
  int8_t neq[MAXC];
  int8_t tag_order[MAXT];
  Mv32 out, wm;
  uint32_t cout, wconst;
};

__device__ __forceinline__ int64_t lopnd(const LOpnd32& o, uint32_t pk) {
  return (int64_t)((pk >> o.shift) & o.mask) + o.base;
}

template <int SEMI>
__global__ void __launch_bounds__(256) lookup_agg32_k(const LookupPlan lp, const LFast32 f,
                                                      unsigned long long* __restrict__ ncand) {
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t chunk = ((lp.np + nwarps - 1) / nwarps + 31) & ~(int64_t)31;
  const int64_t r0 = wid * chunk, r1 = r0 + chunk < lp.np ? r0 + chunk : lp.np;
  uint32_t mycount = 0, cur = 0xffffffffu;
  unsigned long long run = 0;
  for (int64_t base = r0; base < r1; base += 32) {
    const int64_t i = base + (threadIdx.x & 31);
    const uint32_t pk = (uint32_t)i;
    bool ok = i < r1;
    float tags[MAXL + 1];
    tags[0] = 1.0f;
    if (ok) {
      if (SEMI == S_UNIT) {
        ok = (reinterpret_cast<const uint32_t*>(lp.pdir)[i >> 5] >> (i & 31)) & 1u;
      } else if (SEMI == S_MAXMIN) {
        const uint32_t v = reinterpret_cast<const uint32_t*>(lp.pdir)[i];
        ok = v != 0u;
        tags[0] = mm_p(v);
      } else {
        const unsigned long long v = reinterpret_cast<const unsigned long long*>(lp.pdir)[i];
        ok = v != 0ull;
        tags[0] = mx_p(v);
      }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < f.ncmp) ok = ok && cmp_holds(f.neq[c], lopnd(f.ca[c], pk), lopnd(f.cb[c], pk));
#pragma unroll
    for (int l = 0; l < MAXL; ++l) {
      tags[l + 1] = 1.0f;
      if (l >= f.nlk || !ok) continue;
      const uint32_t pre = f.cprefix[l] | mv32(f.pre[l], pk);
      if (pre >= f.nprefix[l]) {
        ok = false;
        continue;
      }
      const int64_t b0 = __ldg(lp.lk[l].boff + pre), b1 = __ldg(lp.lk[l].boff + pre + 1);
      ok = b1 > b0;
      if (ok && SEMI != S_UNIT && lp.lk[l].btag) tags[l + 1] = __ldg(lp.lk[l].btag + b0);
    }
    float t = 1.0f;
    uint32_t w = 0;
    if (ok && SEMI != S_UNIT) {
      auto pick = [&](int idx) {
        float r = tags[0];
#pragma unroll
        for (int k = 1; k <= MAXL; ++k)
          if (k == idx) r = tags[k];
        return r;
      };
      t = pick(f.tag_order[0]);
#pragma unroll
      for (int k = 1; k < MAXT; ++k)
        if (k < f.ntag) t = otimes(lp.omin ? S_MAXMIN : SEMI, t, pick(f.tag_order[k]));
      if (SEMI == S_MAXMULT) w = f.wconst | mv32(f.wm, pk);
    }
    if (ok) ++mycount;
    const uint32_t slot = f.cout | mv32(f.out, pk);
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (!act) continue;
    const uint32_t s0 = __shfl_sync(0xffffffffu, slot, __ffs(act) - 1);
    const bool uniform = __all_sync(0xffffffffu, !ok || slot == s0);
    if (uniform && s0 == cur) {
      const unsigned long long v = ok ? agg_pack<SEMI>(t, w, lp.mx) : 0ull;
      run = v > run ? v : run;
      continue;
    }
    if (cur != 0xffffffffu) agg_flush<SEMI>(lp.fdir, lp.dirty, cur, run);
    run = 0;
    cur = 0xffffffffu;
    if (uniform) {
      cur = s0;
      run = ok ? agg_pack<SEMI>(t, w, lp.mx) : 0ull;
    } else if (ok) {
      direct_oplus(SEMI, lp.fdir, slot, t, w, lp.dirty, 1, lp.mx);
    }
  }
  if (cur != 0xffffffffu) agg_flush<SEMI>(lp.fdir, lp.dirty, cur, run);
  cta_count_add(ncand, mycount);
}

// host: the 32-bit plan, or false (then the generic kernel runs)
static bool split_src0_32(const Move* mv, int n, Mv32& a) {
  Mv32 b;
  for (int i = 0; i < n; ++i)
    if (mv[i].src != 0) return false;
  return split_moves32(mv, n, a, b);
}
static bool lookup_fast32_plan(const LookupPlan& lp, LFast32& f) {
  if (!lp.pdir || !lp.direct || !lp.aggregate || lp.np > 0xffffffffll || lp.cout >> 32) return false;
  if (lp.nlk > MAXL || lp.ncmp > MAXC || lp.ntag > MAXT || lp.ntag < 1) return false;
  std::memset(&f, 0, sizeof(f));
  f.nlk = lp.nlk;
  f.ncmp = lp.ncmp;
  f.ntag = lp.ntag;
  for (int l = 0; l < lp.nlk; ++l) {
    const Lookup& L = lp.lk[l];
    if (!L.boff || L.cprefix >> 32 || L.nprefix > 0xffffffffll || !split_src0_32(L.prem, L.nprem, f.pre[l]))
      return false;
    f.cprefix[l] = (uint32_t)L.cprefix;
    f.nprefix[l] = (uint32_t)L.nprefix;
  }
  for (int c = 0; c < lp.ncmp; ++c) {
    const Operand* o[2] = {&lp.cmp[c].a, &lp.cmp[c].b};
    LOpnd32* d[2] = {&f.ca[c], &f.cb[c]};
    for (int k = 0; k < 2; ++k) {
      if (o[k]->src == 1) return false;
      if (o[k]->src == 2) {
        *d[k] = LOpnd32{0, 0, (int64_t)o[k]->base};
      } else {
        if (o[k]->shift + o[k]->bits > 32) return false;
        *d[k] = LOpnd32{o[k]->shift, o[k]->bits >= 32 ? 0xffffffffu : ((1u << o[k]->bits) - 1u), (int64_t)o[k]->base};
      }
    }
    f.neq[c] = lp.cmp[c].neq;
  }
  for (int k = 0; k < lp.ntag; ++k) f.tag_order[k] = lp.tag_order[k];
  if (!split_src0_32(lp.om, lp.nom, f.out)) return false;
  f.cout = (uint32_t)lp.cout;
  if (lp.semi == S_MAXMULT && !split_src0_32(lp.wm, lp.nwm, f.wm)) return false;
  f.wconst = lp.wconst;
  return true;
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
  if (jp.pk32) join_count_k<uint32_t><<<grid_for(jp.np, 256), 256, 0, st>>>(jp, count, start);
  else join_count_k<uint64_t><<<grid_for(jp.np, 256), 256, 0, st>>>(jp, count, start);
}

template <typename PK, typename OK>
static void launch_join_write_t(const JoinPlan& jp, const int64_t* offs, const int64_t* start, int64_t total,
                                unsigned g, int64_t* tile_row, cudaStream_t st) {
  int64_t* tr = tile_row;
  if (!jp.final_step) join_write_k<PK, OK, JW_INTER><<<g, 256, 0, st>>>(jp, offs, start, total, tr);
  else if (!jp.direct) join_write_k<PK, OK, JW_CAND><<<g, 256, 0, st>>>(jp, offs, start, total, tr);
  else if (jp.semi == S_UNIT) join_write_k<PK, OK, JW_DIRECT + S_UNIT><<<g, 256, 0, st>>>(jp, offs, start, total, tr);
  else if (jp.semi == S_MAXMIN) join_write_k<PK, OK, JW_DIRECT + S_MAXMIN><<<g, 256, 0, st>>>(jp, offs, start, total, tr);
  else join_write_k<PK, OK, JW_DIRECT + S_MAXMULT><<<g, 256, 0, st>>>(jp, offs, start, total, tr);
}

int64_t join_write_tiles(int64_t total) { return (total + WT - 1) / WT; }

void launch_join_write(const JoinPlan& jp, const int64_t* offs, const int64_t* start, int64_t total,
                       int64_t* tile_row, cudaStream_t st) {
  if (total <= 0) return;
  const int64_t nt = join_write_tiles(total);
  const unsigned g = (unsigned)nt;
  note_launch();
  tile_rows_k<<<grid_for(jp.np, 256), 256, 0, st>>>(offs, jp.np, total, nt, tile_row);
  note_launch();
  if (jp.pk32 && jp.ok32) launch_join_write_t<uint32_t, uint32_t>(jp, offs, start, total, g, tile_row, st);
  else if (jp.pk32) launch_join_write_t<uint32_t, uint64_t>(jp, offs, start, total, g, tile_row, st);
  else if (jp.ok32) launch_join_write_t<uint64_t, uint32_t>(jp, offs, start, total, g, tile_row, st);
  else launch_join_write_t<uint64_t, uint64_t>(jp, offs, start, total, g, tile_row, st);
}

// LOBSTER_FAST32=0: the generic fused kernel only (A/B)
static bool getenv_fast32_off() {
  static const bool off = getenv("LOBSTER_FAST32") && atoi(getenv("LOBSTER_FAST32")) == 0;
  return off;
}

template <typename PK, int SEMI, int NM>
static void launch_rows_direct_t(const JoinPlan& jp, int maxdeg, unsigned long long* ncand, cudaStream_t st, int g) {
  if (maxdeg <= 4 && jp.brec) join_rows_direct_k<PK, 4, SEMI, NM, true><<<g, 256, 0, st>>>(jp, ncand);
  else if (maxdeg <= 4) join_rows_direct_k<PK, 4, SEMI, NM, false><<<g, 256, 0, st>>>(jp, ncand);
  else join_rows_direct_k<PK, 8, SEMI, NM, false><<<g, 256, 0, st>>>(jp, ncand);
}
template <int SEMI>
static void launch_rows_direct_s(const JoinPlan& jp, int maxdeg, unsigned long long* ncand, cudaStream_t st, int g) {
  const int nm = std::max(jp.nprem, std::max(jp.nom, jp.nwm));
  if (!jp.pk32) launch_rows_direct_t<uint64_t, SEMI, MAXM>(jp, maxdeg, ncand, st, g);
  else if (nm <= 2) launch_rows_direct_t<uint32_t, SEMI, 2>(jp, maxdeg, ncand, st, g);
  else if (nm <= 4) launch_rows_direct_t<uint32_t, SEMI, 4>(jp, maxdeg, ncand, st, g);
  else launch_rows_direct_t<uint32_t, SEMI, MAXM>(jp, maxdeg, ncand, st, g);
}

void launch_join_rows_direct(const JoinPlan& jp, int maxdeg, unsigned long long* ncand, cudaStream_t st,
                             int64_t np_hint) {
  if (jp.np <= 0) return;
  // device-sized Δ: at most one wave of resident CTAs (grid-stride), at least 2 per SM
  int g = grid_for(np_hint, 256);
  if (jp.np_dev)
    g = std::max(148 * 2, std::min(g, 148 * ((maxdeg <= 4) ? (jp.semi == S_MAXMULT ? FJ_MINB_MX : FJ_MINB) : 4)));
  note_launch();
  Fast32 f;
  if (maxdeg <= 4 && !getenv_fast32_off() && fast32_plan(jp, f)) {
    switch (jp.semi) {
      case S_UNIT: join_rows_rec32_k<S_UNIT><<<g, 256, 0, st>>>(jp, f, ncand); break;
      case S_MAXMIN: join_rows_rec32_k<S_MAXMIN><<<g, 256, 0, st>>>(jp, f, ncand); break;
      default: join_rows_rec32_k<S_MAXMULT><<<g, 256, 0, st>>>(jp, f, ncand); break;
    }
    return;
  }
  switch (jp.semi) {
    case S_UNIT: launch_rows_direct_s<S_UNIT>(jp, maxdeg, ncand, st, g); break;
    case S_MAXMIN: launch_rows_direct_s<S_MAXMIN>(jp, maxdeg, ncand, st, g); break;
    default: launch_rows_direct_s<S_MAXMULT>(jp, maxdeg, ncand, st, g); break;
  }
}

template <typename PK, typename OK, int NM>
static void launch_lookup_chain_m(const LookupPlan& lp, unsigned long long* ncand, int g, cudaStream_t st) {
  if (!lp.direct) lookup_chain_k<PK, OK, LC_CAND, NM><<<g, 256, 0, st>>>(lp, ncand);
  else if (lp.semi == S_UNIT) lookup_chain_k<PK, OK, LC_DIRECT + S_UNIT, NM><<<g, 256, 0, st>>>(lp, ncand);
  else if (lp.semi == S_MAXMIN) lookup_chain_k<PK, OK, LC_DIRECT + S_MAXMIN, NM><<<g, 256, 0, st>>>(lp, ncand);
  else lookup_chain_k<PK, OK, LC_DIRECT + S_MAXMULT, NM><<<g, 256, 0, st>>>(lp, ncand);
}
template <typename PK, typename OK>
static void launch_lookup_chain_t(const LookupPlan& lp, unsigned long long* ncand, int g, cudaStream_t st) {
  int nm = std::max(lp.nom, lp.nwm);
  for (int l = 0; l < lp.nlk; ++l) nm = std::max(nm, lp.lk[l].nprem);
  if (nm <= 2) launch_lookup_chain_m<PK, OK, 2>(lp, ncand, g, st);
  else launch_lookup_chain_m<PK, OK, 0>(lp, ncand, g, st);
}

void launch_lookup_chain(const LookupPlan& lp, unsigned long long* ncand, cudaStream_t st) {
  if (lp.np <= 0) return;
  const int g = grid_for(lp.np, 256);
  note_launch();
  static const bool fast_off = getenv("LOBSTER_LOOKUP_FAST32") && atoi(getenv("LOBSTER_LOOKUP_FAST32")) == 0;
  LFast32 f;
  if (!fast_off && lookup_fast32_plan(lp, f)) {
    switch (lp.semi) {
      case S_UNIT: lookup_agg32_k<S_UNIT><<<g, 256, 0, st>>>(lp, f, ncand); break;
      case S_MAXMIN: lookup_agg32_k<S_MAXMIN><<<g, 256, 0, st>>>(lp, f, ncand); break;
      default: lookup_agg32_k<S_MAXMULT><<<g, 256, 0, st>>>(lp, f, ncand); break;
    }
    return;
  }
  if (lp.pk32 && lp.ok32) launch_lookup_chain_t<uint32_t, uint32_t>(lp, ncand, g, st);
  else if (lp.pk32) launch_lookup_chain_t<uint32_t, uint64_t>(lp, ncand, g, st);
  else if (lp.ok32) launch_lookup_chain_t<uint64_t, uint32_t>(lp, ncand, g, st);
  else launch_lookup_chain_t<uint64_t, uint64_t>(lp, ncand, g, st);
}

__global__ void build_rec4_k(const int64_t* __restrict__ off, const uint64_t* __restrict__ key,
                             const float* __restrict__ tag, int64_t np, uint4* __restrict__ rec) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = off[p];
    const int n = (int)(off[p + 1] - lo);
    uint32_t k[4], t[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      k[d] = d < n ? (uint32_t)key[lo + d] : ~0u;
      t[d] = d < n && tag ? __float_as_uint(tag[lo + d]) : 0u;
    }
    rec[2 * p] = make_uint4(k[0], k[1], k[2], k[3]);
    rec[2 * p + 1] = make_uint4(t[0], t[1], t[2], t[3]);
  }
}

void launch_build_rec4(const int64_t* off, const uint64_t* key, const float* tag, int64_t nprefix, uint4* rec,
                       cudaStream_t st) {
  if (nprefix <= 0) return;
  note_launch();
  build_rec4_k<<<grid_for(nprefix, 256), 256, 0, st>>>(off, key, tag, nprefix, rec);
}

__global__ void max_degree_k(const int64_t* __restrict__ off, int64_t np, unsigned long long* __restrict__ out) {
  unsigned long long m = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = (unsigned long long)(off[p + 1] - off[p]);
    m = d > m ? d : m;
  }
  m = __reduce_max_sync(0xffffffffu, (unsigned)m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

void launch_max_degree(const int64_t* off, int64_t nprefix, unsigned long long* out, cudaStream_t st) {
  if (nprefix <= 0) return;
  note_launch();
  max_degree_k<<<grid_for(nprefix, 256, 148 * 8), 256, 0, st>>>(off, nprefix, out);
}

void launch_project(const ProjectPlan& pp, cudaStream_t st) {
  if (pp.n <= 0) return;
  const int g = grid_for(pp.n, 256);
  note_launch();
  if (pp.pk32 && pp.ok32) project_k<uint32_t, uint32_t><<<g, 256, 0, st>>>(pp);
  else if (pp.pk32) project_k<uint32_t, uint64_t><<<g, 256, 0, st>>>(pp);
  else if (pp.ok32) project_k<uint64_t, uint32_t><<<g, 256, 0, st>>>(pp);
  else project_k<uint64_t, uint64_t><<<g, 256, 0, st>>>(pp);
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
