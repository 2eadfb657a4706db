// host_copy.h — host threads that move bytes between a caller's pageable
// arrays and the pipeline's page-locked staging ring (internal to capi.cu).
//
// The reference's callers hand over ordinary numpy arrays (codec.py:144-155:
// numpy in, numpy out).  Copying them into page-locked memory is host-memory
// bandwidth work that one thread cannot do at PCIe speed, so each batch of
// segments is cut into <= 2 MiB pieces shared by a few persistent workers
// and the calling thread.  run() returns when every piece is copied.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include <emmintrin.h>  // SSE2 (baseline x86-64): non-temporal 16-byte stores

namespace adct {

// memcpy with non-temporal (streaming) stores: the destination lines are not
// read for ownership first and do not evict the source from the caches.  The
// staging copies are pure bandwidth (each byte is touched once), and on the
// B200 hosts measured the host memory bandwidth, not the PCIe link, bounds
// the pageable path, so avoiding the read-for-ownership traffic matters.
inline void stream_copy(uint8_t* dst, const uint8_t* src, size_t n) {
  if (n < 256) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();  // streaming stores are weakly ordered: complete them before the piece counts as done
}

class HostCopyPool {
 public:
  struct Seg {
    uint8_t* dst;
    const uint8_t* src;
    size_t n;
  };

  // ADCT_PIPELINE_THREADS (1..64) or min(16, hardware threads), at least 1
  // (tools/e2e_pageable.py on a 16-core B200 host: 2 threads 10, 8 threads
  // 21, 16 threads 26 Gpixel/s for config-3 images in and out).
  static int default_threads() {
    if (const char* e = std::getenv("ADCT_PIPELINE_THREADS")) {
      const int v = std::atoi(e);
      if (v >= 1 && v <= 64) return v;
    }
    const int hw = (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(16, hw));
  }

  explicit HostCopyPool(int threads) {
    for (int t = 1; t < threads; ++t) workers_.emplace_back([this] { loop(); });
  }

  ~HostCopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

  HostCopyPool(const HostCopyPool&) = delete;
  HostCopyPool& operator=(const HostCopyPool&) = delete;

  void run(const std::vector<Seg>& segs) {
    if (workers_.empty()) {
      for (const Seg& s : segs) stream_copy(s.dst, s.src, s.n);
      return;
    }
    {
      // A worker woken late for the previous batch may still be inside
      // work(): wait for it to leave before the piece list changes.  Workers
      // only enter work() after counting themselves in under this lock.
      std::unique_lock<std::mutex> lk(mu_);
      idle_cv_.wait(lk, [this] { return active_ == 0; });
      pieces_.clear();
      for (const Seg& s : segs)
        for (size_t o = 0; o < s.n; o += kPiece) pieces_.push_back({s.dst + o, s.src + o, std::min(kPiece, s.n - o)});
      if (pieces_.empty()) return;
      next_.store(0);
      left_.store(pieces_.size());
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return left_.load() == 0; });
  }

 private:
  static constexpr size_t kPiece = 2u << 20;

  void work() {
    for (;;) {
      const size_t i = next_.fetch_add(1);
      if (i >= pieces_.size()) return;
      stream_copy(pieces_[i].dst, pieces_[i].src, pieces_[i].n);
      if (left_.fetch_sub(1) == 1) {
        std::lock_guard<std::mutex> g(mu_);
        done_cv_.notify_all();
      }
    }
  }

  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        ++active_;
      }
      work();
      {
        std::lock_guard<std::mutex> g(mu_);
        if (--active_ == 0) idle_cv_.notify_all();
      }
    }
  }

  std::vector<std::thread> workers_;
  std::vector<Seg> pieces_;
  std::atomic<size_t> next_{0}, left_{0};
  std::mutex mu_;
  std::condition_variable cv_, done_cv_, idle_cv_;
  uint64_t gen_ = 0;
  int active_ = 0;
  bool stop_ = false;
};

}  // namespace adct
