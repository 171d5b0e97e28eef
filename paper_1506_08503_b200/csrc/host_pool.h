// host_pool.h -- host-side parallel byte work for the staging pipeline
// (pageable <-> pinned copies, shared-IV detection).  Internal to
// libgaes_b200.so.
#pragma once
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace gaes {
namespace host {

// --------------------------------------------------------------------------
// Host-side parallel byte work (staging copies, shared-IV detection).  Large
// pageable buffers are copied by several threads: one core's memcpy (~10 GB/s)
// is slower than a PCIe Gen5 DMA, so a single-threaded staging copy would
// bound the drop-in path.
inline int host_threads() {
  static int t = [] {
    int hw = (int)std::thread::hardware_concurrency();
    const char* e = std::getenv("GAES_HOST_THREADS");
    int v = (e && *e) ? std::atoi(e) : std::max(1, std::min(12, hw - 4));
    return std::max(1, v);
  }();
  return t;
}

// Persistent workers (spawning threads per staging copy costs ~50 us).
class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 0; i < n; i++) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  // Runs fn(i) for i in [0, parts) on the workers plus the calling thread.
  void run(size_t parts, const std::function<void(size_t)>& fn) {
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel region at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      parts_ = parts;
      next_.store(0);
      pending_ = parts;
      gen_++;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      const size_t i = next_.fetch_add(1);
      if (i >= parts_) return;
      (*fn_)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && fn_ != nullptr); });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* fn_ = nullptr;
  size_t parts_ = 0, pending_ = 0;
  std::atomic<size_t> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

inline HostPool& host_pool() {
  static HostPool* pool = new HostPool(std::max(0, host_threads() - 1));  // leaked: lives until exit
  return *pool;
}

template <typename F>
void parallel_ranges(size_t n, size_t min_per_thread, F&& fn) {
  const size_t want = std::min<size_t>((size_t)host_threads(), std::max<size_t>(1, n / min_per_thread));
  if (want <= 1) {
    fn(0, n);
    return;
  }
  const size_t step = (n + want - 1) / want;
  const std::function<void(size_t)> part = [&](size_t t) {
    const size_t lo = t * step, hi = std::min(n, lo + step);
    if (lo < hi) fn(lo, hi);
  };
  host_pool().run(want, part);
}

inline void par_memcpy(void* dst, const void* src, size_t bytes) {
  parallel_ranges(bytes, (size_t)512 << 10, [&](size_t lo, size_t hi) {
    std::memcpy((uint8_t*)dst + lo, (const uint8_t*)src + lo, hi - lo);
  });
}

}  // namespace host
}  // namespace gaes
