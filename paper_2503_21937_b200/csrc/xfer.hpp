// xfer.hpp — the exchange step of key-partitioned evaluation (SURVEY §8(f)
// NEXT-3; the paper's TC / SG inputs outgrow one GPU).
//
// One database, W ranks: every IDB tuple is owned by one rank (a hash of its
// packed key), inputs are replicated, and each round ends with an all-to-all
// of the candidates to their owners plus an all-reduce of |Δ'| (the fixpoint
// test, Alg. 1, over all ranks).  Two transports:
//   NcclXfer  — one process per GPU: grouped ncclSend / ncclRecv (NVLink /
//               NVSwitch), NCCL loaded at run time from libnccl.so.2.
//   LocalXfer — W contexts of one process (one thread each, any devices):
//               peers copy their chunks out of each other's send buffers with
//               cudaMemcpyAsync between two host barriers.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace lob {

struct Xfer {
  int world = 1;
  virtual ~Xfer() = default;
  // host int64 per peer: recv[d] = the value rank d sent to `rank`
  virtual void counts(int rank, const int64_t* send, int64_t* recv, cudaStream_t st) = 0;
  // device buffers; element counts per peer (host); chunks laid out by peer rank
  virtual void alltoallv(int rank, const void* send, const int64_t* scnt, void* recv, const int64_t* rcnt,
                         size_t elem, cudaStream_t st) = 0;
};

// W contexts in one process
struct LocalXfer : Xfer {
  explicit LocalXfer(int w);
  void counts(int rank, const int64_t* send, int64_t* recv, cudaStream_t st) override;
  void alltoallv(int rank, const void* send, const int64_t* scnt, void* recv, const int64_t* rcnt, size_t elem,
                 cudaStream_t st) override;

 private:
  void barrier();
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  uint64_t gen_ = 0;
  std::vector<const void*> sbuf_;
  std::vector<std::vector<int64_t>> cnt_;  // [sender][peer]
  std::vector<int> dev_;
};

// one process per GPU over NCCL
struct NcclXfer : Xfer {
  NcclXfer(const uint8_t id[128], int rank, int w, int device);
  ~NcclXfer() override;
  void counts(int rank, const int64_t* send, int64_t* recv, cudaStream_t st) override;
  void alltoallv(int rank, const void* send, const int64_t* scnt, void* recv, const int64_t* rcnt, size_t elem,
                 cudaStream_t st) override;
  static void unique_id(uint8_t id[128]);

 private:
  void* comm_ = nullptr;
  int64_t* dcnt_ = nullptr;  // 2 * world int64 (device)
  int64_t* hcnt_ = nullptr;  // pinned
};

}  // namespace lob
