// k_sort.cu — stable LSD radix sort of packed keys (A6; the `sort`
// instruction, Table 1, run every round by the Stratum rule,
// PAPER.md:1296).  Only the significant bits of the key are sorted (keys are
// packed with per-column domain widths), 8 bits per pass; u32 keys are used
// whenever the relation's packed key fits, halving the bytes moved.
//
// Per pass: (1) per-tile digit histogram in shared memory, written digit-major
// so (2) one exclusive scan yields every (digit, tile) global base; (3) scatter:
// each CTA ranks its 4096 keys stably with warp __match_any_sync + per-warp
// digit counters and writes them at base + rank.  Keys (and values) of a tile
// are loaded once into registers (16 in flight per thread).  The scatter is
// shared-memory-instruction bound (ncu on C3: MIO 41%, barrier 17%; 2.7 TB/s).
// Measured and rejected on C3: staging the ranked tile in shared memory for
// run-contiguous writes (11.4 -> 17.4 ms) and warp-blocked ranks with
// warp-private running counters (10.0 -> 13.6 ms): both raise registers to
// 104-145 per thread and halve the resident CTAs, which costs more than the
// coalescing / fewer shared-memory operations gain.
#include <type_traits>

#include "device_util.cuh"

namespace lob {
namespace {

constexpr int NT = 256;
constexpr int IPT = 16;
constexpr int TILE = NT * IPT;
constexpr int NW = NT / 32;

template <typename K>
__global__ void __launch_bounds__(NT) radix_hist_k(const K* __restrict__ key, int64_t n, int shift,
                                                   uint32_t* __restrict__ hist, int64_t ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * TILE;
#pragma unroll 4
  for (int k = 0; k < IPT; ++k) {
    int64_t i = base + k * NT + threadIdx.x;
    if (i < n) atomicAdd(&h[(uint32_t)(key[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <typename K, typename V, bool HASV>
__global__ void __launch_bounds__(NT) radix_scatter_k(const K* __restrict__ kin, const V* __restrict__ vin,
                                                      K* __restrict__ kout, V* __restrict__ vout, int64_t n,
                                                      int shift, const uint32_t* __restrict__ base_off,
                                                      int64_t ntiles) {
  __shared__ uint32_t wcnt[NW][256];
  __shared__ uint32_t run[256];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  run[tid] = base_off[(int64_t)tid * ntiles + blockIdx.x];
  const int64_t base = (int64_t)blockIdx.x * TILE;
  K k[IPT];
  V v[HASV ? IPT : 1];
#pragma unroll
  for (int s = 0; s < IPT; ++s) {
    int64_t i = base + s * NT + tid;
    if (i < n) {
      k[s] = kin[i];
      if constexpr (HASV) v[s] = vin[i];
    }
  }
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int s = 0; s < IPT; ++s) {
    const int64_t i = base + s * NT + tid;
    const bool valid = i < n;
    const uint32_t d = valid ? ((uint32_t)(k[s] >> shift) & 255u) : 256u;
#pragma unroll
    for (int j = 0; j < 8; ++j) wcnt[w][lane * 8 + j] = 0;
    __syncwarp();
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) wcnt[w][d] = __popc(peers);
    __syncthreads();
    {
      uint32_t sum = run[tid];
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) {
        uint32_t c = wcnt[ww][tid];
        wcnt[ww][tid] = sum;
        sum += c;
      }
      run[tid] = sum;
    }
    __syncthreads();
    if (valid) {
      const uint32_t dst = wcnt[w][d] + rank;
      kout[dst] = k[s];
      if constexpr (HASV) vout[dst] = v[s];
    }
    __syncthreads();
  }
}

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Tiny inputs (C1-sized relations): one CTA ranks every key against all others
// on the same low bits the LSD passes would sort, ties by index — the same
// stable permutation as the passes, in one launch instead of ~5 per 8-bit
// pass (hist, scan, scatter).
constexpr int SMALL_SORT = 256;
template <typename K, typename V, bool HASV>
__global__ void __launch_bounds__(SMALL_SORT) radix_small_k(const K* __restrict__ ki, const V* __restrict__ vi,
                                                            K* __restrict__ ko, V* __restrict__ vo, int n, K mask) {
  __shared__ K sk[SMALL_SORT];
  const int i = threadIdx.x;
  if (i < n) sk[i] = ki[i] & mask;
  __syncthreads();
  if (i >= n) return;
  const K x = sk[i];
  int r = 0;
  for (int j = 0; j < n; ++j) {
    const K y = sk[j];
    r += (y < x) || (y == x && j < i);
  }
  ko[r] = ki[i];
  if (HASV) vo[r] = vi[i];
}

template <typename K, typename V, bool HASV>
int radix_sort_impl(K* k0, V* v0, K* k1, V* v1, int64_t n, int bits, void* tmp, cudaStream_t st) {
  if (n <= 1 || bits <= 0) return 0;
  if (n <= SMALL_SORT) {
    const int sb = ((bits + 7) / 8) * 8;  // the bits the passes would sort
    const K mask = sb >= (int)(8 * sizeof(K)) ? ~K(0) : (K)((K(1) << sb) - 1);
    note_launch();
    radix_small_k<K, V, HASV><<<1, SMALL_SORT, 0, st>>>(k0, v0, k1, v1, (int)n, mask);
    return 1;
  }
  const int64_t ntiles = (n + TILE - 1) / TILE;
  uint32_t* hist = reinterpret_cast<uint32_t*>(tmp);
  void* stmp = reinterpret_cast<char*>(tmp) + align_up((size_t)ntiles * 256 * sizeof(uint32_t));
  const int passes = (bits + 7) / 8;
  int cur = 0;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    const K* ki = cur ? k1 : k0;
    const V* vi = cur ? v1 : v0;
    K* ko = cur ? k0 : k1;
    V* vo = cur ? v0 : v1;
    note_launch();
    radix_hist_k<K><<<(unsigned)ntiles, NT, 0, st>>>(ki, n, shift, hist, ntiles);
    exclusive_scan<uint32_t>(hist, hist, ntiles * 256, nullptr, stmp, st);
    note_launch();
    radix_scatter_k<K, V, HASV><<<(unsigned)ntiles, NT, 0, st>>>(ki, vi, ko, vo, n, shift, hist, ntiles);
    cur ^= 1;
  }
  return cur;
}

}  // namespace

size_t sort_tmp_bytes(int64_t n) {
  const int64_t ntiles = (n + TILE - 1) / TILE;
  return align_up((size_t)ntiles * 256 * sizeof(uint32_t)) + scan_tmp_bytes<uint32_t>(ntiles * 256) + 256;
}

template <typename K, typename V>
int radix_sort(K* k0, V* v0, K* k1, V* v1, int64_t n, int bits, void* tmp, cudaStream_t st) {
  if constexpr (std::is_void_v<V>)
    return radix_sort_impl<K, uint32_t, false>(k0, (uint32_t*)v0, k1, (uint32_t*)v1, n, bits, tmp, st);
  else
    return radix_sort_impl<K, V, true>(k0, v0, k1, v1, n, bits, tmp, st);
}

template int radix_sort<uint64_t, void>(uint64_t*, void*, uint64_t*, void*, int64_t, int, void*, cudaStream_t);
template int radix_sort<uint64_t, uint32_t>(uint64_t*, uint32_t*, uint64_t*, uint32_t*, int64_t, int, void*,
                                            cudaStream_t);
template int radix_sort<uint64_t, uint64_t>(uint64_t*, uint64_t*, uint64_t*, uint64_t*, int64_t, int, void*,
                                            cudaStream_t);
template int radix_sort<uint32_t, void>(uint32_t*, void*, uint32_t*, void*, int64_t, int, void*, cudaStream_t);
template int radix_sort<uint32_t, uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, int64_t, int, void*,
                                            cudaStream_t);
template int radix_sort<uint32_t, uint64_t>(uint32_t*, uint64_t*, uint32_t*, uint64_t*, int64_t, int, void*,
                                            cudaStream_t);

}  // namespace lob
