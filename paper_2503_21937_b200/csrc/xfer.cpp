// xfer.cpp — transports of the key-partitioned exchange (see xfer.hpp).
#include "xfer.hpp"

#include <dlfcn.h>

#include <cstring>

#include "devmem.hpp"
#include "program.hpp"
#include "lobster.h"

namespace lob {

// ------------------------------------------------------------------ local
LocalXfer::LocalXfer(int w) {
  world = w;
  sbuf_.assign(w, nullptr);
  cnt_.assign(w, std::vector<int64_t>(w, 0));
  dev_.assign(w, 0);
}

void LocalXfer::barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  const uint64_t g = gen_;
  if (++arrived_ == world) {
    arrived_ = 0;
    ++gen_;
    cv_.notify_all();
    return;
  }
  cv_.wait(lk, [&] { return gen_ != g; });
}

void LocalXfer::counts(int rank, const int64_t* send, int64_t* recv, cudaStream_t) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    cnt_[rank].assign(send, send + world);
  }
  barrier();
  {
    std::lock_guard<std::mutex> lk(mu_);
    for (int d = 0; d < world; ++d) recv[d] = cnt_[d][rank];
  }
  barrier();  // nobody overwrites cnt_ before every peer has read it
}

void LocalXfer::alltoallv(int rank, const void* send, const int64_t* scnt, void* recv, const int64_t* rcnt,
                          size_t elem, cudaStream_t st) {
  cuda_check(cudaStreamSynchronize(st), "xfer: send buffer ready");
  {
    std::lock_guard<std::mutex> lk(mu_);
    sbuf_[rank] = send;
    cnt_[rank].assign(scnt, scnt + world);
  }
  barrier();
  int64_t roff = 0;
  for (int d = 0; d < world; ++d) {
    int64_t soff = 0;
    for (int k = 0; k < rank; ++k) soff += cnt_[d][k];
    const int64_t n = cnt_[d][rank];
    if (n != rcnt[d]) throw Failure(LOBSTER_E_INVALID_ARG, "xfer: receive count mismatch");
    if (n)
      cuda_check(cudaMemcpyAsync(static_cast<char*>(recv) + roff * elem, static_cast<const char*>(sbuf_[d]) + soff * elem,
                                 (size_t)n * elem, cudaMemcpyDefault, st),
                 "xfer: peer copy");
    roff += n;
  }
  cuda_check(cudaStreamSynchronize(st), "xfer: copies done");
  barrier();  // every peer finished reading this rank's send buffer
}

// ------------------------------------------------------------------- NCCL
namespace {
// the few NCCL entry points used, resolved from libnccl.so.2 at run time
// (RTLD_LOCAL: no clash with another NCCL a host framework may have loaded)
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*errstr)(int) = nullptr;
  void* initRank = nullptr;
};
struct Id128 {
  char b[128];
};
constexpr int NCCL_INT8 = 0, NCCL_INT64 = 4;

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclGetUniqueId"));
    api.initRank = dlsym(api.h, "ncclCommInitRank");
    api.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclCommDestroy"));
    api.groupStart = reinterpret_cast<int (*)()>(dlsym(api.h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<int (*)()>(dlsym(api.h, "ncclGroupEnd"));
    api.send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(dlsym(api.h, "ncclSend"));
    api.recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(dlsym(api.h, "ncclRecv"));
    api.errstr = reinterpret_cast<const char* (*)(int)>(dlsym(api.h, "ncclGetErrorString"));
  });
  if (!api.h || !api.getUniqueId || !api.initRank || !api.send || !api.recv || !api.groupStart || !api.groupEnd)
    throw Failure(LOBSTER_E_NCCL, "libnccl.so.2 could not be loaded");
  return api;
}

void nccl_check(int r, const char* what) {
  if (r == 0) return;
  const char* s = nccl().errstr ? nccl().errstr(r) : "?";
  throw Failure(LOBSTER_E_NCCL, std::string(what) + ": " + s);
}
}  // namespace

void NcclXfer::unique_id(uint8_t id[128]) { nccl_check(nccl().getUniqueId(id), "ncclGetUniqueId"); }

NcclXfer::NcclXfer(const uint8_t id[128], int rank, int w, int device) {
  world = w;
  NcclApi& A = nccl();
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  Id128 uid;
  std::memcpy(uid.b, id, 128);
  auto init = reinterpret_cast<int (*)(void**, int, Id128, int)>(A.initRank);
  nccl_check(init(&comm_, w, uid, rank), "ncclCommInitRank");
  cuda_check(cudaMalloc(&dcnt_, 2 * (size_t)w * 8), "cudaMalloc");
  cuda_check(cudaMallocHost(&hcnt_, 2 * (size_t)w * 8), "cudaMallocHost");
}

NcclXfer::~NcclXfer() {
  if (comm_ && nccl().commDestroy) nccl().commDestroy(comm_);
  if (dcnt_) cudaFree(dcnt_);
  if (hcnt_) cudaFreeHost(hcnt_);
}

void NcclXfer::counts(int, const int64_t* send, int64_t* recv, cudaStream_t st) {
  NcclApi& A = nccl();
  std::memcpy(hcnt_, send, (size_t)world * 8);
  cuda_check(cudaMemcpyAsync(dcnt_, hcnt_, (size_t)world * 8, cudaMemcpyHostToDevice, st), "H2D");
  nccl_check(A.groupStart(), "ncclGroupStart");
  for (int d = 0; d < world; ++d) {
    nccl_check(A.send(dcnt_ + d, 1, NCCL_INT64, d, comm_, st), "ncclSend");
    nccl_check(A.recv(dcnt_ + world + d, 1, NCCL_INT64, d, comm_, st), "ncclRecv");
  }
  nccl_check(A.groupEnd(), "ncclGroupEnd");
  cuda_check(cudaMemcpyAsync(hcnt_ + world, dcnt_ + world, (size_t)world * 8, cudaMemcpyDeviceToHost, st), "D2H");
  cuda_check(cudaStreamSynchronize(st), "xfer counts");
  std::memcpy(recv, hcnt_ + world, (size_t)world * 8);
}

void NcclXfer::alltoallv(int, const void* send, const int64_t* scnt, void* recv, const int64_t* rcnt, size_t elem,
                         cudaStream_t st) {
  NcclApi& A = nccl();
  nccl_check(A.groupStart(), "ncclGroupStart");
  int64_t so = 0, ro = 0;
  for (int d = 0; d < world; ++d) {
    if (scnt[d])
      nccl_check(A.send(static_cast<const char*>(send) + so * elem, (size_t)scnt[d] * elem, NCCL_INT8, d, comm_, st),
                 "ncclSend");
    if (rcnt[d])
      nccl_check(A.recv(static_cast<char*>(recv) + ro * elem, (size_t)rcnt[d] * elem, NCCL_INT8, d, comm_, st),
                 "ncclRecv");
    so += scnt[d];
    ro += rcnt[d];
  }
  nccl_check(A.groupEnd(), "ncclGroupEnd");
}

}  // namespace lob
