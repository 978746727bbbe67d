// Host worker pool of the host-tier streamer: the pageable -> pinned bounce
// copies (pageable data is first copied to pinned memory) and the disk
// tier's reads are split across the workers so they keep up with the DMA.
//
// A bounce copy of one 16.5 MiB item takes ~0.2 ms on 16 threads, so waking the
// workers through a condition variable (tens of microseconds per round trip)
// would cost a large share of it: workers spin on a generation counter for a
// while after each job (they are about to get the next piece) and only then
// sleep; the caller spins on the pending count.  Worker threads can be pinned to
// the CPUs local to the store's GPU (set_affinity).
#pragma once

#include <immintrin.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace harag {

// Non-temporal (streaming-store) copy: the bounce destination is written once and read only by the
// DMA engine, so write-allocate reads of it are wasted host DRAM traffic — and the bounce copy shares
// host DRAM bandwidth with the very DMA it feeds.
__attribute__((target("avx2"))) inline void copy_nt(void* dst, const void* src, size_t n) {
  uint8_t* d = (uint8_t*)dst;
  const uint8_t* s = (const uint8_t*)src;
  const size_t head = (32 - ((uintptr_t)d & 31)) & 31;
  if (n < head + 128) {
    std::memcpy(d, s, n);
    return;
  }
  std::memcpy(d, s, head);
  d += head, s += head, n -= head;
  const size_t body = n & ~size_t(127);
  for (size_t i = 0; i < body; i += 128) {
    const __m256i a = _mm256_loadu_si256((const __m256i*)(s + i));
    const __m256i b = _mm256_loadu_si256((const __m256i*)(s + i + 32));
    const __m256i c = _mm256_loadu_si256((const __m256i*)(s + i + 64));
    const __m256i e = _mm256_loadu_si256((const __m256i*)(s + i + 96));
    _mm256_stream_si256((__m256i*)(d + i), a);
    _mm256_stream_si256((__m256i*)(d + i + 32), b);
    _mm256_stream_si256((__m256i*)(d + i + 64), c);
    _mm256_stream_si256((__m256i*)(d + i + 96), e);
  }
  _mm_sfence();
  std::memcpy(d + body, s + body, n - body);
}

class CopyPool {
 public:
  explicit CopyPool(unsigned n, int spin = 2000, bool nt = true)
      : spin_(spin), nt_(nt && __builtin_cpu_supports("avx2")) {
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_.store(true);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // Pin every worker (and nothing else) to the given CPUs; empty = leave as is.
  void set_affinity(const std::vector<int>& cpus) {
    if (cpus.empty()) return;
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int c : cpus) CPU_SET(c, &set);
    for (auto& t : workers_) pthread_setaffinity_np(t.native_handle(), sizeof(set), &set);
  }
  // memcpy(dst, src, n) over the calling thread and the workers; returns when done.  The range is cut
  // into 256 KiB chunks claimed through an atomic counter, so a worker that is descheduled or shares a
  // core with another busy thread takes fewer chunks instead of holding up the whole copy (a static
  // split of a 16.5 MiB item over 10 threads ran the pageable leg at 0.61-0.88 of the link, bimodally).
  void copy(void* dst, const void* src, size_t n) {
    if (n < (1u << 20) || workers_.empty()) {
      std::memcpy(dst, src, n);
      return;
    }
    uint8_t* d = (uint8_t*)dst;
    const uint8_t* s = (const uint8_t*)src;
    constexpr size_t kChunk = size_t(1) << 18;
    const size_t n_chunks = (n + kChunk - 1) / kChunk;
    const unsigned parts = std::min<unsigned>(size(), (unsigned)n_chunks);
    std::atomic<size_t> next{0};
    parallel_for(parts, [&](unsigned) {
      for (size_t c = next.fetch_add(1, std::memory_order_relaxed); c < n_chunks;
           c = next.fetch_add(1, std::memory_order_relaxed)) {
        const size_t b = c * kChunk, len = std::min(kChunk, n - b);
        if (nt_)
          copy_nt(d + b, s + b, len);
        else
          std::memcpy(d + b, s + b, len);
      }
    });
  }
  // fn(0..parts-1) over the calling thread (part 0) and the workers; returns when all are done.
  void parallel_for(unsigned parts, const std::function<void(unsigned)>& fn) {
    parts = std::min(parts, size());
    if (parts <= 1) {
      fn(0);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      parts_ = parts;
      pending_.store((unsigned)workers_.size());
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    fn(0);
    while (pending_.load(std::memory_order_acquire) != 0) cpu_relax();
  }
  unsigned size() const { return (unsigned)workers_.size() + 1; }

 private:
  static void cpu_relax() {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#else
    std::this_thread::yield();
#endif
  }
  void run(unsigned i) {
    uint64_t seen = 0;
    for (;;) {
      // spin for the next job (spin_ PAUSEs, ~0.1 ms), then sleep
      uint64_t g = gen_.load(std::memory_order_acquire);
      for (int spin = 0; g == seen && spin < spin_; ++spin) {
        cpu_relax();
        g = gen_.load(std::memory_order_acquire);
      }
      if (g == seen) {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
        g = gen_.load();
      }
      if (stop_.load()) return;
      seen = g;
      const std::function<void(unsigned)>* fn;
      unsigned parts;
      {
        std::lock_guard<std::mutex> lk(m_);
        fn = fn_;
        parts = parts_;
      }
      if (i + 1 < parts) (*fn)(i + 1);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  const int spin_;
  const bool nt_;
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_;
  std::atomic<bool> stop_{false};
  std::atomic<uint64_t> gen_{0};
  std::atomic<unsigned> pending_{0};
  unsigned parts_ = 0;
  const std::function<void(unsigned)>* fn_ = nullptr;
};

}  // namespace harag
