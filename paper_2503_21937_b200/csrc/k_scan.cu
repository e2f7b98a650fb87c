// k_scan.cu — exclusive prefix sum (A4: "scan", PAPER.md:360 Table 1, :508).
//
// Reduce-then-scan over 2048-item tiles (256 threads x 8 items, coalesced loads
// staged through shared memory), recursing on the tile partials.  The total is
// written to device memory so no host read is implied by the scan itself.
#include "device_util.cuh"

namespace lob {
namespace {

constexpr int NT = 256;
constexpr int IPT = 8;
constexpr int TILE = NT * IPT;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  return v;
}

// exclusive block scan of one value per thread; returns the block total via *tot
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* tot) {
  __shared__ T wsum[NT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane < NT / 32 ? wsum[lane] : T(0);
    T xi = warp_incl_scan(x);
    if (lane < NT / 32) wsum[lane] = xi - x;
    if (lane == NT / 32 - 1) *tot = xi;
  }
  __syncthreads();
  T r = inc - v + wsum[w];
  __syncthreads();
  return r;
}

template <typename T>
__global__ void __launch_bounds__(NT) scan_reduce_k(const T* __restrict__ in, int64_t n, T* __restrict__ partial) {
  const int64_t base = (int64_t)blockIdx.x * TILE;
  T s = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int64_t i = base + k * NT + threadIdx.x;
    if (i < n) s += in[i];
  }
  __shared__ T tot;
  block_excl_scan<T>(s, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(NT) scan_tile_k(const T* in, T* out, int64_t n,
                                                  const T* __restrict__ carry, T* __restrict__ total) {
  __shared__ T sm[TILE + TILE / 32];
  auto at = [](int i) { return i + (i >> 5); };  // pad one slot per 32 to soften bank conflicts
  const int64_t base = (int64_t)blockIdx.x * TILE;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int64_t i = base + k * NT + threadIdx.x;
    sm[at(k * NT + threadIdx.x)] = i < n ? in[i] : T(0);
  }
  __syncthreads();
  T v[IPT];
  T run = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    T x = sm[at(threadIdx.x * IPT + k)];
    v[k] = run;
    run += x;
  }
  __shared__ T btot;
  T pre = block_excl_scan<T>(run, &btot);
  const T c = carry ? carry[blockIdx.x] : T(0);
#pragma unroll
  for (int k = 0; k < IPT; ++k) sm[at(threadIdx.x * IPT + k)] = v[k] + pre + c;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int64_t i = base + k * NT + threadIdx.x;
    if (i < n) out[i] = sm[at(k * NT + threadIdx.x)];
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = c + btot;
}

template <typename T>
__global__ void zero_total_k(T* total) { *total = T(0); }

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

template <typename T>
size_t scan_tmp_bytes(int64_t n) {
  size_t b = 0;
  int64_t m = n;
  while (m > TILE) {
    m = (m + TILE - 1) / TILE;
    b += align_up((size_t)m * sizeof(T));
  }
  return b + 256;
}

template <typename T>
void exclusive_scan(const T* in, T* out, int64_t n, T* total_dev, void* tmp, cudaStream_t st) {
  if (n <= 0) {
    if (total_dev) {
      note_launch();
      zero_total_k<T><<<1, 1, 0, st>>>(total_dev);
    }
    return;
  }
  const int64_t ntiles = (n + TILE - 1) / TILE;
  if (ntiles == 1) {
    note_launch();
    scan_tile_k<T><<<1, NT, 0, st>>>(in, out, n, nullptr, total_dev);
    return;
  }
  T* partial = reinterpret_cast<T*>(tmp);
  void* rest = reinterpret_cast<char*>(tmp) + align_up((size_t)ntiles * sizeof(T));
  note_launch();
  scan_reduce_k<T><<<(unsigned)ntiles, NT, 0, st>>>(in, n, partial);
  exclusive_scan<T>(partial, partial, ntiles, nullptr, rest, st);
  note_launch();
  scan_tile_k<T><<<(unsigned)ntiles, NT, 0, st>>>(in, out, n, partial, total_dev);
}

template size_t scan_tmp_bytes<uint32_t>(int64_t);
template size_t scan_tmp_bytes<int64_t>(int64_t);
template size_t scan_tmp_bytes<uint64_t>(int64_t);
template void exclusive_scan<uint32_t>(const uint32_t*, uint32_t*, int64_t, uint32_t*, void*, cudaStream_t);
template void exclusive_scan<int64_t>(const int64_t*, int64_t*, int64_t, int64_t*, void*, cudaStream_t);
template void exclusive_scan<uint64_t>(const uint64_t*, uint64_t*, int64_t, uint64_t*, void*, cudaStream_t);

}  // namespace lob
