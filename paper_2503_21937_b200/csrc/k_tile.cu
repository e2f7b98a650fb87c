// k_tile.cu — small dense per-sample strata: the whole fixpoint in one launch.
//
// CLUTRR-shaped kinship and C1-sized
// problems have tiny per-sample domains (20 entities × 20 relation types): the
// general path spends its time on per-round launches, host syncs and sorting
// candidates that a head receives hundreds of times.  Here one CTA owns one
// sample (grid-stride over samples) and keeps every relation of the stratum
// dense in shared memory:
//
//   S (state), Δ (increments, reading 5) and U (this round's ⊕ per head)
//   as fp32 tags + presence bitmaps over compact slots (row-major over the
//   columns' true domain sizes), and 64-bit presence FIBERS of S and Δ along
//   every column that closes an atom during enumeration.
//
// A round (Alg. 1; the oracle's steps i-v):
//   (i)+(iii) every thread pulls its head slots: for each rule in program order
//     it enumerates the non-head variables in order of first appearance (the
//     canonical tie / summation order, reading 8b), each level's candidate
//     values = OR over variants of AND of the fibers of the atoms that variable
//     closes (variant j: local atoms before j read NEW = S ⊕ Δ, atom j reads Δ,
//     later ones OLD = S), and at a leaf forms every alive
//     variant's ⊗ left-deep in body order.  add-mult accumulates those terms
//     in fp64 in exactly the oracle's sorted-candidate order and rounds once
//     (reading 9), so tags are bit-exact, not just within 1 ulp.
//   (ii)+(iv) per slot: S ← S ⊕ Δ, then Δ' = U where the tuple is new or
//     fp32 bits of S ⊕ U differ from S (reading 1); fibers rebuilt from bits.
//   (v) __syncthreads_or(Δ' non-empty) ends the sample's fixpoint.
// No host round trip, no candidate buffer, no sort.  External atoms read dense
// per-sample arrays built once per stratum by tile_scatter_k.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "devmem.hpp"
#include "device_util.cuh"
#include "tile_device.cuh"

namespace lob {
namespace {

constexpr int TILE_THREADS = TILE_THREADS_N;

template <int SEMI, int NT>
__global__ void __launch_bounds__(NT, 1) tile_fixpoint_k(const TilePlan* __restrict__ Pg, int* rounds_out,
                                                         unsigned long long* ncand, int* cap_hit) {
  extern __shared__ __align__(16) uint8_t sm[];
  // The plan (~5.5 KB) is copied to shared memory: every enumeration step
  // indexes it.  (Reading it through a pointer to a > 4 KB __grid_constant__
  // parameter returned garbage under load on sm_100a: out-of-range fiber
  // indexes with >= 8 warps per CTA, found by compute-sanitizer memcheck.)
  __shared__ __align__(16) TilePlan Q;
  for (int i = threadIdx.x; i < (int)(sizeof(TilePlan) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(&Q)[i] = reinterpret_cast<const uint32_t*>(Pg)[i];
  __syncthreads();
  tile_body<SEMI, (NT > 512 ? 2 : TILE_MAXLEV)>(Q, sm, rounds_out, ncand, cap_hit);
}

__global__ void tile_scatter_k(const __grid_constant__ TileScatter S) {
  const TileRel& T = S.rel;
  const int nbw = (T.D + 31) >> 5;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S.n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = S.key[i];
    if (k == KEY_DEAD) continue;
    const int64_t s = S.has_sample ? (int64_t)((k >> S.sshift) & ((1ull << S.sbits) - 1ull)) : 0;
    int32_t coord[TILE_MAXCOL];
    int slot = 0;
    for (int c = 0; c < S.ncols; ++c) {
      coord[c] = (int32_t)((k >> S.shift[c]) & ((1ull << S.bits[c]) - 1ull));
      slot += coord[c] * T.stride[c];
    }
    if (T.tag) const_cast<float*>(T.tag)[s * T.D + slot] = S.p ? S.p[i] : 1.0f;
    atomicOr(const_cast<uint32_t*>(T.bits) + s * nbw + (slot >> 5), 1u << (slot & 31));
    for (int c = 0; c < S.ncols; ++c) {
      if (!T.nfib[c]) continue;
      int f = 0;
      for (int q = 0; q < S.ncols; ++q)
        if (q != c) f += coord[q] * T.fstride[c][q];
      atomicOr(const_cast<unsigned long long*>(T.fib[c]) + s * T.nfib[c] + f, 1ull << coord[c]);
    }
  }
}

__global__ void max_i32_k(const int* __restrict__ a, int n, int* __restrict__ out) {
  int m = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = max(m, a[i]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_down_sync(~0u, m, o));
  __shared__ int wm[32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, wm[w]);
    *out = max(m, wm[0]);
  }
}

template <int SEMI, int NT>
void launch_tile_t(const TilePlan& P, const TilePlan* dplan, int* rounds_out, unsigned long long* ncand, int* cap_hit,
                   cudaStream_t st) {
  static int configured_bytes = -1;  // per template: opt in to > 48 KB of dynamic shared memory once
  if (configured_bytes < P.smem_bytes) {
    const int dyn = 227 * 1024 - (int)((sizeof(TilePlan) + 255) & ~size_t(255));  // static plan copy + dynamic <= 227 KB
    cuda_check(cudaFuncSetAttribute(tile_fixpoint_k<SEMI, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn),
               "tile smem attribute");
    configured_bytes = dyn;
  }
  // occupancy per shared-memory size, SM count: host queries cached (microseconds each)
  static std::mutex mu;
  static std::map<int, int> occ;
  static int sms = 0;
  int per_sm = 1;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    auto it = occ.find(P.smem_bytes);
    if (it == occ.end()) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_fixpoint_k<SEMI, NT>, NT, P.smem_bytes);
      occ[P.smem_bytes] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  const int threads = NT;
  int grid = std::max(1, std::min(P.nsamples, std::max(1, per_sm) * sms));
  if (const char* e = getenv("LOBSTER_TILE_GRID")) grid = std::max(1, std::min(grid, atoi(e)));
  tile_fixpoint_k<SEMI, NT><<<grid, threads, P.smem_bytes, st>>>(dplan, rounds_out, ncand, cap_hit);
}

}  // namespace

void launch_tile_fixpoint(const TilePlan& P, TilePlan* dplan, int* rounds_out, unsigned long long* ncand,
                          int* cap_hit, cudaStream_t st) {
  if (P.nsamples <= 0) return;
  // P should live in pinned host memory (the engine's staging copy): an async copy
  cuda_check(cudaMemcpyAsync(dplan, &P, sizeof(TilePlan), cudaMemcpyHostToDevice, st), "tile plan");
  note_launch();
  // compacted composition plans: the recursive rounds need few registers, so
  // a 1024-thread CTA (64 registers) doubles the warps hiding shared-memory
  // latency (LOBSTER_TILE_THREADS=512 for A/B)
  static const int nt_env = getenv("LOBSTER_TILE_THREADS") ? atoi(getenv("LOBSTER_TILE_THREADS")) : 1024;
  bool wide = P.cm_rule >= 0 && nt_env >= 1024;
  for (int i = 0; i < P.nrule && wide; ++i) wide = i == P.cm_rule || P.rule[i].nlev <= 2;
  switch (P.semi) {
    case S_UNIT:
      if (wide) launch_tile_t<S_UNIT, 1024>(P, dplan, rounds_out, ncand, cap_hit, st);
      else launch_tile_t<S_UNIT, TILE_THREADS>(P, dplan, rounds_out, ncand, cap_hit, st);
      break;
    case S_MAXMIN:
      if (wide) launch_tile_t<S_MAXMIN, 1024>(P, dplan, rounds_out, ncand, cap_hit, st);
      else launch_tile_t<S_MAXMIN, TILE_THREADS>(P, dplan, rounds_out, ncand, cap_hit, st);
      break;
    default:
      if (wide) launch_tile_t<S_ADDMULT, 1024>(P, dplan, rounds_out, ncand, cap_hit, st);
      else launch_tile_t<S_ADDMULT, TILE_THREADS>(P, dplan, rounds_out, ncand, cap_hit, st);
      break;
  }
}

void launch_tile_scatter(const TileScatter& S, cudaStream_t st) {
  if (S.n <= 0) return;
  note_launch();
  tile_scatter_k<<<grid_for(S.n, 256), 256, 0, st>>>(S);
}

void launch_max_i32(const int* a, int n, int* out, cudaStream_t st) {
  note_launch();
  max_i32_k<<<1, 1024, 0, st>>>(a, n, out);
}

}  // namespace lob
