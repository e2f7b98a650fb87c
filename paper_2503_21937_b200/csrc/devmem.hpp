// devmem.hpp — device buffers with capacity reuse (§4.1 buffer
// reuse: over-allocate, keep across iterations, grow x1.5) and the per-round
// bump arena (§4.1 arena allocation: alloc = pointer bump,
// free = no-op, reset every round).  Backed by the stream-ordered allocator.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "lobster.h"
#include "program.hpp"

namespace lob {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Failure(LOBSTER_E_OOM, std::string(what) + ": out of device memory");
  }
  throw Failure(LOBSTER_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

class DevMem {
 public:
  DevMem() = default;
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  ~DevMem() { release(); }
  void bind(cudaStream_t st) { st_ = st; }
  // ensure capacity >= bytes; keep=true preserves the first `keep_bytes`
  void reserve(size_t bytes, size_t keep_bytes = 0) {
    if (bytes <= cap_) return;
    size_t ncap = cap_ ? cap_ + cap_ / 2 : 0;
    if (ncap < bytes) ncap = bytes;
    ncap = (ncap + 255) & ~size_t(255);
    void* np = nullptr;
    cuda_check(cudaMallocAsync(&np, ncap, st_), "cudaMallocAsync");
    if (keep_bytes && p_) cuda_check(cudaMemcpyAsync(np, p_, keep_bytes, cudaMemcpyDeviceToDevice, st_), "grow copy");
    if (p_) cudaFreeAsync(p_, st_);
    p_ = np;
    cap_ = ncap;
  }
  void release() {
    if (p_) cudaFreeAsync(p_, st_);
    p_ = nullptr;
    cap_ = 0;
  }
  void swap(DevMem& o) {
    std::swap(p_, o.p_);
    std::swap(cap_, o.cap_);
  }
  void* get() const { return p_; }
  size_t capacity() const { return cap_; }

 private:
  void* p_ = nullptr;
  size_t cap_ = 0;
  cudaStream_t st_ = nullptr;
};

template <typename T>
class DBuf {
 public:
  void bind(cudaStream_t st) { m_.bind(st); }
  void reserve(int64_t n, int64_t keep = 0) { m_.reserve((size_t)(n > 0 ? n : 1) * sizeof(T), (size_t)keep * sizeof(T)); }
  T* ptr() const { return reinterpret_cast<T*>(m_.get()); }
  void release() { m_.release(); }
  void swap(DBuf& o) { m_.swap(o.m_); }
  size_t bytes() const { return m_.capacity(); }

 private:
  DevMem m_;
};

// Pinned host buffer for output_get(where=0) copies: page-locked so the D2H
// runs at full link speed, grown x1.5 and kept across runs (no zero-fill,
// no first-touch faults on the next read-back).
template <typename T>
class HBuf {
 public:
  HBuf() = default;
  HBuf(const HBuf&) = delete;
  HBuf& operator=(const HBuf&) = delete;
  ~HBuf() { if (p_) cudaFreeHost(p_); }
  void resize(size_t n) {
    n_ = n;
    if (n <= cap_) return;
    size_t ncap = cap_ + cap_ / 2;
    if (ncap < n) ncap = n;
    void* np = nullptr;
    cuda_check(cudaHostAlloc(&np, (ncap ? ncap : 1) * sizeof(T), cudaHostAllocDefault), "cudaHostAlloc");
    if (p_) cudaFreeHost(p_);
    p_ = reinterpret_cast<T*>(np);
    cap_ = ncap;
  }
  T* data() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t cap_ = 0, n_ = 0;
};

class Arena {
 public:
  void bind(cudaStream_t st) { st_ = st; }
  ~Arena() { free_all(); }
  void* alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    if (off_ + bytes <= cap_) {
      void* p = base_ + off_;
      off_ += bytes;
      high_ = off_ > high_ ? off_ : high_;
      return p;
    }
    void* p = nullptr;  // overflow: served separately, folded into the next reset's capacity
    cuda_check(cudaMallocAsync(&p, bytes, st_), "arena overflow");
    overflow_.push_back(p);
    over_bytes_ += bytes;
    return p;
  }
  template <typename T>
  T* get(int64_t n) { return reinterpret_cast<T*>(alloc((size_t)(n > 0 ? n : 1) * sizeof(T))); }
  void reset() {
    for (void* p : overflow_) cudaFreeAsync(p, st_);
    overflow_.clear();
    size_t want = high_ + over_bytes_;
    over_bytes_ = 0;
    if (want > cap_) {
      if (base_) cudaFreeAsync(base_, st_);
      cap_ = want + want / 2;
      cap_ = (cap_ + 4095) & ~size_t(4095);
      void* p = nullptr;
      cuda_check(cudaMallocAsync(&p, cap_, st_), "arena grow");
      base_ = reinterpret_cast<char*>(p);
    }
    off_ = 0;
    high_ = 0;
  }
  void reserve_initial(size_t bytes) {
    if (bytes > cap_) {
      high_ = bytes;
      reset();
    }
  }
  void free_all() {
    for (void* p : overflow_) cudaFreeAsync(p, st_);
    overflow_.clear();
    if (base_) cudaFreeAsync(base_, st_);
    base_ = nullptr;
    cap_ = off_ = high_ = over_bytes_ = 0;
  }
  size_t capacity() const { return cap_; }

 private:
  cudaStream_t st_ = nullptr;
  char* base_ = nullptr;
  size_t cap_ = 0, off_ = 0, high_ = 0, over_bytes_ = 0;
  std::vector<void*> overflow_;
};

}  // namespace lob
