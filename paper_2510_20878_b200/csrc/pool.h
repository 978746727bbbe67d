// Host worker pool of the host-tier streamer: the pageable -> pinned bounce
// copies (pageable data is first copied to pinned memory) and the disk
// tier's reads are split across the workers so they keep up with the DMA.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace harag {

class CopyPool {
 public:
  explicit CopyPool(unsigned n) {
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  // memcpy(dst, src, n) split over the calling thread and the workers; returns when done.
  void copy(void* dst, const void* src, size_t n) {
    if (n < (4u << 20) || workers_.empty()) {
      std::memcpy(dst, src, n);
      return;
    }
    uint8_t* d = (uint8_t*)dst;
    const uint8_t* s = (const uint8_t*)src;
    const size_t chunk = (n / (workers_.size() + 1) + 4095) & ~size_t(4095);
    parallel_for((unsigned)workers_.size() + 1, [&](unsigned p) {
      const size_t b = (size_t)p * chunk;
      if (b < n) std::memcpy(d + b, s + b, std::min(chunk, n - b));
    });
  }
  // fn(0..parts-1) over the calling thread (part 0) and the workers; returns when all are done.
  void parallel_for(unsigned parts, const std::function<void(unsigned)>& fn) {
    parts = std::min(parts, (unsigned)workers_.size() + 1);
    if (parts <= 1) {
      fn(0);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      parts_ = parts;
      pending_ = (unsigned)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }
  unsigned size() const { return (unsigned)workers_.size() + 1; }

 private:
  void run(unsigned i) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(unsigned)>* fn;
      unsigned parts;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        fn = fn_;
        parts = parts_;
      }
      if (i + 1 < parts) (*fn)(i + 1);
      {
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  bool stop_ = false;
  uint64_t gen_ = 0;
  unsigned pending_ = 0, parts_ = 0;
  const std::function<void(unsigned)>* fn_ = nullptr;
};

}  // namespace harag
