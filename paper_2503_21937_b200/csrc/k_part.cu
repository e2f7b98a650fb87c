// k_part.cu — key-partitioned evaluation: the owner of a
// tuple is a hash of its packed key; candidates are bucketed by owner (stable,
// so every receiver sees them in a deterministic order) before the all-to-all.
#include "device_util.cuh"

namespace lob {
namespace {

__device__ __forceinline__ uint32_t owner_of(uint64_t key, uint32_t world) {
  uint64_t h = key + 0x9E3779B97F4A7C15ull;  // splitmix64 finaliser
  h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
  h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
  h ^= h >> 31;
  return (uint32_t)(((h >> 32) * (uint64_t)world) >> 32);
}

template <typename K>
__global__ void part_dest_k(const K* __restrict__ key, int64_t n, uint32_t world, uint32_t* __restrict__ dest,
                            uint32_t* __restrict__ idx, unsigned long long* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const K k = key[i];
    const uint32_t d = k == dead<K>() ? world : owner_of((uint64_t)k, world);  // dead rows: dropped
    dest[i] = d;
    idx[i] = (uint32_t)i;
    atomicAdd(cnt + d, 1ull);
  }
}

template <typename K>
__global__ void part_keep_k(K* __restrict__ key, int64_t n, uint32_t world, uint32_t rank) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const K k = key[i];
    if (k != dead<K>() && owner_of((uint64_t)k, world) != rank) key[i] = dead<K>();
  }
}

template <typename T>
__global__ void part_gather_k(const T* __restrict__ s, const uint32_t* __restrict__ idx, T* __restrict__ d, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[idx[i]];
}

}  // namespace

void launch_part_dest(const void* key, bool k32, int64_t n, uint32_t world, uint32_t* dest, uint32_t* idx,
                      unsigned long long* cnt, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  if (k32)
    part_dest_k<uint32_t><<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint32_t*>(key), n, world, dest, idx, cnt);
  else
    part_dest_k<uint64_t><<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint64_t*>(key), n, world, dest, idx, cnt);
}

void launch_part_keep(void* key, bool k32, int64_t n, uint32_t world, uint32_t rank, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  if (k32) part_keep_k<uint32_t><<<grid_for(n, 256), 256, 0, st>>>(static_cast<uint32_t*>(key), n, world, rank);
  else part_keep_k<uint64_t><<<grid_for(n, 256), 256, 0, st>>>(static_cast<uint64_t*>(key), n, world, rank);
}

void launch_part_gather(const void* src, const uint32_t* idx, void* dst, int64_t n, int elem_bytes, cudaStream_t st) {
  if (n <= 0) return;
  note_launch();
  if (elem_bytes == 8)
    part_gather_k<uint64_t><<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint64_t*>(src), idx,
                                                               static_cast<uint64_t*>(dst), n);
  else
    part_gather_k<uint32_t><<<grid_for(n, 256), 256, 0, st>>>(static_cast<const uint32_t*>(src), idx,
                                                               static_cast<uint32_t*>(dst), n);
}

}  // namespace lob
