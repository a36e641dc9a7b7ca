// Pageable host memory <-> device at PCIe speed (kmb_capi.cu host-input batches).
//
// A copy from pageable memory is staged by the driver through its own small
// pinned buffers, one piece at a time and blocking the calling thread: config 3
// from numpy arrays or std::vectors moved 256 MiB in 28.9 ms (9.3 GB/s, against
// 55 GB/s from pinned memory).  HostStager copies through a ring of pinned
// slots instead, the pageable -> pinned memcpy split over a small pool of host
// threads, each slot's H2D enqueued as soon as it is full, so the host copy of
// slot k+1 overlaps the DMA of slot k.  Results go the other way through a
// pinned buffer the caller's pageable arrays are filled from after the solve.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace kmb {

// A fixed set of worker threads running parts of one job at a time.
class CopyPool {
 public:
  explicit CopyPool(int workers) {
    for (int k = 0; k < workers; ++k) th_.emplace_back([this, k] { loop(k + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int threads() const { return static_cast<int>(th_.size()) + 1; }
  // job(part) for part in [0, parts): part 0 on the caller, the rest on workers
  void run(int parts, const std::function<void(int)>& job) {
    parts = std::max(1, std::min(parts, threads()));
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = &job;
      parts_ = parts;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    job(0);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int idx) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job = nullptr;
      int parts = 0;
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
        parts = parts_;
      }
      if (idx < parts && job) {
        (*job)(idx);
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int parts_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

class HostStager {
 public:
  static constexpr int kSlots = 4;
  static constexpr size_t kSlot = size_t{8} << 20;

  HostStager() : pool_(std::max(1u, std::min(7u, std::thread::hardware_concurrency() / 2))) {}
  ~HostStager() {
    for (int k = 0; k < kSlots; ++k)
      if (ev_[k]) cudaEventDestroy(ev_[k]);
    if (ring_) cudaFreeHost(ring_);
    if (out_) cudaFreeHost(out_);
  }

  // host -> host with the pool (pieces of at least 1 MiB)
  void memcpy_par(void* dst, const void* src, size_t bytes) {
    const size_t kMin = size_t{1} << 20;
    const int parts = static_cast<int>(std::min<size_t>(pool_.threads(), (bytes + kMin - 1) / kMin));
    if (parts <= 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const size_t per = (bytes + parts - 1) / parts;
    pool_.run(parts, [&](int k) {
      const size_t lo = per * k, hi = std::min(bytes, lo + per);
      if (lo < hi) std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, hi - lo);
    });
  }

  // pageable src -> device dst, enqueued on s; returns once src has been read
  cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    cudaError_t e = ensure_ring();
    if (e != cudaSuccess) return e;
    for (size_t off = 0; off < bytes; off += kSlot) {
      const size_t len = std::min(kSlot, bytes - off);
      const int k = next_++ % kSlots;
      if ((e = cudaEventSynchronize(ev_[k])) != cudaSuccess) return e;  // slot's last DMA done
      unsigned char* slot = ring_ + static_cast<size_t>(k) * kSlot;
      memcpy_par(slot, static_cast<const char*>(src) + off, len);
      if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + off, slot, len, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return e;
      if ((e = cudaEventRecord(ev_[k], s)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }

  // a pinned buffer of at least `bytes` for results bound for pageable memory
  cudaError_t out_buffer(size_t bytes, unsigned char** p) {
    if (bytes > out_bytes_) {
      if (out_) cudaFreeHost(out_);
      out_ = nullptr;
      out_bytes_ = 0;
      cudaError_t e = cudaMallocHost(&out_, bytes);
      if (e != cudaSuccess) return e;
      out_bytes_ = bytes;
    }
    *p = out_;
    return cudaSuccess;
  }

 private:
  cudaError_t ensure_ring() {
    if (ring_) return cudaSuccess;
    cudaError_t e = cudaMallocHost(&ring_, kSlot * kSlots);
    if (e != cudaSuccess) {
      ring_ = nullptr;
      return e;
    }
    for (int k = 0; k < kSlots; ++k)
      if ((e = cudaEventCreateWithFlags(&ev_[k], cudaEventDisableTiming)) != cudaSuccess) return e;
    return cudaSuccess;
  }
  CopyPool pool_;
  unsigned char* ring_ = nullptr;
  cudaEvent_t ev_[kSlots] = {};
  uint64_t next_ = 0;
  unsigned char* out_ = nullptr;
  size_t out_bytes_ = 0;
};

// pinned (page-locked / registered) host memory?
inline bool is_pinned_host(const void* p) {
  cudaPointerAttributes at;
  if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

}  // namespace kmb
