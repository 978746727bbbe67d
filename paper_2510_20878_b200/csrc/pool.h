// Host worker pool for the pageable -> pinned bounce copies of the host-tier
// streamer (pageable data is first copied to pinned memory).  One
// memcpy is split across the workers so the bounce keeps up with the DMA.
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
    const unsigned parts = (unsigned)workers_.size() + 1;
    if (n < (4u << 20) || parts == 1) {
      std::memcpy(dst, src, n);
      return;
    }
    const size_t chunk = (n / parts + 4095) & ~size_t(4095);
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = (uint8_t*)dst, src_ = (const uint8_t*)src, n_ = n, chunk_ = chunk;
      pending_ = (unsigned)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    part(0);  // the caller takes chunk 0
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void part(unsigned p) {
    const size_t b = (size_t)p * chunk_;
    if (b < n_) std::memcpy(dst_ + b, src_ + b, std::min(chunk_, n_ - b));
  }
  void run(unsigned i) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      part(i + 1);
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
  unsigned pending_ = 0;
  uint8_t* dst_ = nullptr;
  const uint8_t* src_ = nullptr;
  size_t n_ = 0, chunk_ = 0;
};

}  // namespace harag
