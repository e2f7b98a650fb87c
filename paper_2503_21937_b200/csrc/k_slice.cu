// k_slice.cu — bit-sliced multi-source frontier (unit semiring).
//
// C4-shaped strata: one batched unary relation R
// whose recursive rules join it with SHARED binary relations,
//     reach(y) :- reach(x), edge(x, y).        edge shared, one source per sample
// Every sample runs the same semi-naive rounds (Alg. 1) over the
// same graph, so the sample becomes the fastest-varying bit: node t owns
// W = ceil(B/32) words and bit j of word wi is sample 32·wi + j.  One Δ entry
// (t, wi, bits) then joins edge(t, ·) once for up to 32 samples — one
// coalesced-ish word update per (edge, word) instead of one bitmap atomic per
// (edge, sample).  Per sample the rounds are exactly the per-sample
// semi-naive rounds: bit (t, s) is in Δ of round r iff R(t) is new for sample
// s in round r-1 (the bits never interact).
//
// State: Rb (relation bits), Nb (bits derived this round), a dirty bitmap over
// the T·W words, and Δ as (t, wi, bits) triples.  Rb changes only in the
// extraction, so the join's read of Rb is exact; a stale read of Nb is a
// lower bound (Nb only gains bits within a round).
#include "device_util.cuh"

namespace lob {
namespace {

__global__ void slice_hist_k(const uint64_t* __restrict__ key, int64_t n, int ssrc, uint64_t msk,
                             uint32_t* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + ((key[i] >> ssrc) & msk), 1u);
}

__global__ void slice_fill_k(const uint64_t* __restrict__ key, int64_t n, int ssrc, int sdst, uint64_t msk,
                             uint32_t* __restrict__ cursor, uint32_t* __restrict__ nbr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    const uint32_t pos = atomicAdd(cursor + ((k >> ssrc) & msk), 1u);
    nbr[pos] = (uint32_t)((k >> sdst) & msk);
  }
}

// bit (s, t) of the direct unit store: slot = s << tbits | t
__device__ __forceinline__ uint32_t bm_row_bits(const uint32_t* __restrict__ bm, int tbits, int64_t s, int64_t t0,
                                                int64_t T) {
  if (tbits >= 5) return bm[((s << tbits) | t0) >> 5];
  uint32_t w = 0;
  for (int i = 0; i < 32 && t0 + i < T; ++i) {
    const int64_t slot = (s << tbits) | (t0 + i);
    w |= ((bm[slot >> 5] >> (slot & 31)) & 1u) << i;
  }
  return w;
}

// (s, t) bitmap -> Nb words (t, wi) with dirty bits: one warp per 32x32 tile
// (32 nodes x 32 samples), transposed with 32 ballots.
__global__ void slice_from_bitmap_k(const uint32_t* __restrict__ bm, int tbits, int B, int64_t T, int W,
                                    uint32_t* __restrict__ Nb, uint32_t* __restrict__ dirty) {
  const int lane = threadIdx.x & 31;
  const int64_t ntb = (T + 31) / 32;
  const int64_t ntiles = ntb * W;
  for (int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile < ntiles;
       tile += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t tb = tile / W;
    const int wi = (int)(tile % W);
    const int64_t s = (int64_t)wi * 32 + lane;
    const uint32_t w = s < B ? bm_row_bits(bm, tbits, s, tb * 32, T) : 0u;
    uint32_t out = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint32_t b = __ballot_sync(0xffffffffu, (w >> i) & 1u);
      if (lane == i) out = b;
    }
    const int64_t t = tb * 32 + lane;
    if (t < T) {
      const int64_t idx = t * W + wi;
      Nb[idx] = out;
      if (out) atomicOr(dirty + (idx >> 5), 1u << (idx & 31));
    }
  }
}

// Rb words -> the (s, t) bitmap of the direct unit store (all words of the
// first B samples are written; smaller domains OR single bits)
__global__ void slice_to_bitmap_k(const uint32_t* __restrict__ Rb, int tbits, int B, int64_t T, int W,
                                  uint32_t* __restrict__ bm) {
  const int lane = threadIdx.x & 31;
  const int64_t ntb = (T + 31) / 32;
  const int64_t ntiles = ntb * W;
  for (int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile < ntiles;
       tile += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t tb = tile / W;
    const int wi = (int)(tile % W);
    const int64_t t = tb * 32 + lane;
    const uint32_t w = t < T ? Rb[t * W + wi] : 0u;  // bits over samples
    uint32_t out = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t b = __ballot_sync(0xffffffffu, (w >> j) & 1u);
      if (lane == j) out = b;  // bits over the tile's nodes for sample 32 wi + j
    }
    const int64_t s = (int64_t)wi * 32 + lane;
    if (s >= B) continue;
    if (tbits >= 5) {
      bm[((s << tbits) | (tb * 32)) >> 5] = out;
    } else {
      for (int i = 0; i < 32 && tb * 32 + i < T; ++i)
        if ((out >> i) & 1u) {
          const int64_t slot = (s << tbits) | (tb * 32 + i);
          atomicOr(bm + (slot >> 5), 1u << (slot & 31));
        }
    }
  }
}

// Δ' extraction: a CTA takes 32 dirty-bitmap words per step (4 per warp, one
// lane per word slot).  d = Nb & ~Rb; Rb |= d; Nb = 0; nonzero d -> Δ' entry
// (t, wi, d).  Positions come from ONE global atomic per CTA step (a per-warp
// atomic on the single counter serialised in L2: 81 µs per C4 round).
constexpr int SX_WPW = 4;  // dirty words per warp per step
__global__ void __launch_bounds__(256) slice_extract_k(uint32_t* __restrict__ dirty, int64_t ndw,
                                                       uint32_t* __restrict__ Nb, uint32_t* __restrict__ Rb, int W,
                                                       uint32_t* __restrict__ dt, uint32_t* __restrict__ dwi,
                                                       uint32_t* __restrict__ dbits, uint32_t* __restrict__ count,
                                                       unsigned long long* __restrict__ tuples) {
  __shared__ uint32_t wcnt[8], wpre[8], cbase;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long mytup = 0;
  const int64_t per = (int64_t)(blockDim.x >> 5) * SX_WPW;
  for (int64_t q0 = (int64_t)blockIdx.x * per; q0 < ndw; q0 += (int64_t)gridDim.x * per) {
    uint32_t d[SX_WPW], act[SX_WPW];
    int64_t idxv[SX_WPW];
    uint32_t n = 0;
#pragma unroll
    for (int j = 0; j < SX_WPW; ++j) {
      const int64_t q = q0 + (int64_t)warp * SX_WPW + j;
      const uint32_t m = q < ndw ? dirty[q] : 0u;
      idxv[j] = q * 32 + lane;
      d[j] = 0;
      if ((m >> lane) & 1u) {
        const uint32_t r = Rb[idxv[j]];
        d[j] = Nb[idxv[j]] & ~r;
        Nb[idxv[j]] = 0;
        if (d[j]) Rb[idxv[j]] = r | d[j];
      }
      act[j] = __ballot_sync(0xffffffffu, d[j] != 0);
      if (lane == 0 && m) dirty[q] = 0;
      n += __popc(act[j]);
    }
    if (lane == 0) wcnt[warp] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        wpre[w] = t;
        t += wcnt[w];
      }
      cbase = t ? atomicAdd(count, t) : 0u;
    }
    __syncthreads();
    uint32_t base = cbase + wpre[warp];
#pragma unroll
    for (int j = 0; j < SX_WPW; ++j) {
      if (d[j]) {
        const uint32_t pos = base + __popc(act[j] & ((1u << lane) - 1u));
        dt[pos] = (uint32_t)(idxv[j] / W);
        dwi[pos] = (uint32_t)(idxv[j] % W);
        dbits[pos] = d[j];
        mytup += (unsigned long long)__popc(d[j]);
      }
      base += __popc(act[j]);
    }
    __syncthreads();  // wcnt / wpre / cbase are rewritten by the next step
  }
  cta_count_add(tuples, (uint32_t)mytup);
}

__global__ void slice_deg_k(const uint32_t* __restrict__ dt, int64_t nd, const uint32_t* __restrict__ off,
                            uint32_t* __restrict__ deg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = dt[i];
    deg[i] = off[t + 1] - off[t];
  }
}

// Join: items k in [0, Σ deg) = (Δ entry i, its e-th neighbour y); the new
// bits of word (y, wi) are bits & ~Rb; ORed into Nb (fire-and-forget) when a
// peek of Nb does not already hold them, with the word's dirty bit.
constexpr int SLICE_IPT = 8;  // consecutive items per thread (one binary search)
__global__ void __launch_bounds__(256) slice_expand_k(const uint32_t* __restrict__ dt, const uint32_t* __restrict__ dwi,
                                                      const uint32_t* __restrict__ dbits,
                                                      const uint32_t* __restrict__ pos, int64_t nd,
                                                      const uint32_t* __restrict__ total_dev,
                                                      const uint32_t* __restrict__ off,
                                                      const uint32_t* __restrict__ nbr,
                                                      const uint32_t* __restrict__ Rb, uint32_t* __restrict__ Nb,
                                                      int W, uint32_t* __restrict__ dirty,
                                                      unsigned long long* __restrict__ cands) {
  const int64_t total = *total_dev;
  unsigned long long mycand = 0;
  for (int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * SLICE_IPT; k0 < total;
       k0 += (int64_t)gridDim.x * blockDim.x * SLICE_IPT) {
    int64_t lo = 0, hi = nd;  // last i with pos[i] <= k0
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (pos[mid] <= (uint32_t)k0) lo = mid; else hi = mid;
    }
    int64_t i = lo;
    uint32_t p_i = pos[i], p_next = i + 1 < nd ? pos[i + 1] : (uint32_t)total;
    uint32_t base = off[dt[i]], wi = dwi[i], bits = dbits[i];
    const int64_t k1 = k0 + SLICE_IPT < total ? k0 + SLICE_IPT : total;
    for (int64_t k = k0; k < k1; ++k) {
      while ((uint32_t)k >= p_next) {  // next Δ entry (zero-degree entries are skipped)
        ++i;
        p_i = p_next;
        p_next = i + 1 < nd ? pos[i + 1] : (uint32_t)total;
        base = off[dt[i]];
        wi = dwi[i];
        bits = dbits[i];
      }
      const uint32_t y = nbr[base + ((uint32_t)k - p_i)];
      const int64_t idx = (int64_t)y * W + wi;
      mycand += (unsigned long long)__popc(bits);
      const uint32_t nb = bits & ~Rb[idx];
      if (!nb) continue;
      if (!(nb & ~PEEK_SLOT(Nb + idx))) continue;  // stale lower bound (relaxed load; Nb only gains bits)
      atomicOr(Nb + idx, nb);
      atomicOr(dirty + (idx >> 5), 1u << (idx & 31));
    }
  }
  cta_count_add(cands, (uint32_t)mycand);
}

__global__ void add_u32_dev_k(uint32_t* dst, const uint32_t* src, int assign) {
  *dst = assign ? *src : *dst + *src;
}

}  // namespace

void launch_add_u32_dev(uint32_t* dst, const uint32_t* src, bool assign, cudaStream_t st) {
  note_launch();
  add_u32_dev_k<<<1, 1, 0, st>>>(dst, src, assign ? 1 : 0);
}

void launch_slice_csr(const uint64_t* key, int64_t n, int ssrc, int sdst, int bits, int64_t T, uint32_t* off,
                      uint32_t* cursor, uint32_t* nbr, void* scan_tmp, cudaStream_t st) {
  const uint64_t msk = bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
  cudaMemsetAsync(cursor, 0, (size_t)(T + 1) * 4, st);
  if (n > 0) {
    note_launch();
    slice_hist_k<<<grid_for(n, 256), 256, 0, st>>>(key, n, ssrc, msk, cursor);
  }
  exclusive_scan<uint32_t>(cursor, off, T + 1, nullptr, scan_tmp, st);
  cudaMemcpyAsync(cursor, off, (size_t)(T + 1) * 4, cudaMemcpyDeviceToDevice, st);
  if (n > 0) {
    note_launch();
    slice_fill_k<<<grid_for(n, 256), 256, 0, st>>>(key, n, ssrc, sdst, msk, cursor, nbr);
  }
}

void launch_slice_from_bitmap(const uint32_t* bm, int tbits, int B, int64_t T, int W, uint32_t* Nb, uint32_t* dirty,
                              cudaStream_t st) {
  const int64_t tiles = (T + 31) / 32 * W;
  note_launch();
  slice_from_bitmap_k<<<grid_for(tiles * 32, 256), 256, 0, st>>>(bm, tbits, B, T, W, Nb, dirty);
}

void launch_slice_to_bitmap(const uint32_t* Rb, int tbits, int B, int64_t T, int W, uint32_t* bm, cudaStream_t st) {
  const int64_t tiles = (T + 31) / 32 * W;
  note_launch();
  slice_to_bitmap_k<<<grid_for(tiles * 32, 256), 256, 0, st>>>(Rb, tbits, B, T, W, bm);
}

void launch_slice_extract(uint32_t* dirty, int64_t ndw, uint32_t* Nb, uint32_t* Rb, int W, uint32_t* dt, uint32_t* dwi,
                          uint32_t* dbits, uint32_t* count, unsigned long long* tuples, cudaStream_t st) {
  note_launch();
  slice_extract_k<<<grid_for(ndw, 8 * SX_WPW, 148 * 16), 256, 0, st>>>(dirty, ndw, Nb, Rb, W, dt, dwi, dbits, count, tuples);
}

void launch_slice_deg(const uint32_t* dt, int64_t nd, const uint32_t* off, uint32_t* deg, cudaStream_t st) {
  if (nd <= 0) return;
  note_launch();
  slice_deg_k<<<grid_for(nd, 256), 256, 0, st>>>(dt, nd, off, deg);
}

void launch_slice_expand(const uint32_t* dt, const uint32_t* dwi, const uint32_t* dbits, const uint32_t* pos,
                         int64_t nd, const uint32_t* total_dev, const uint32_t* off, const uint32_t* nbr,
                         const uint32_t* Rb, uint32_t* Nb, int W, uint32_t* dirty, unsigned long long* cands,
                         cudaStream_t st) {
  if (nd <= 0) return;
  note_launch();
  // one wave of resident CTAs, grid-stride over the device-side item count
  slice_expand_k<<<148 * 8, 256, 0, st>>>(dt, dwi, dbits, pos, nd, total_dev, off, nbr, Rb, Nb, W, dirty, cands);
}

}  // namespace lob
