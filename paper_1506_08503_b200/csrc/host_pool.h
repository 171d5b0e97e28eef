// host_pool.h -- host-side parallel byte work for the staging pipeline
// (pageable <-> pinned copies, shared-IV detection).  Internal to
// libgaes_b200.so.
#pragma once
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "runtime.h"

namespace gaes {
namespace host {

// --------------------------------------------------------------------------
// Host-side parallel byte work (staging copies, shared-IV detection).  Large
// pageable buffers are copied by several threads: one core's memcpy (~10 GB/s)
// is slower than a PCIe Gen5 DMA, so a single-threaded staging copy would
// bound the drop-in path.
// Default: every CPU this process may run on (its affinity mask -- one
// NUMA node per rank under bench.py's binding), at most 32.  Measured on the
// 16-CPU GPU box (scripts/exp/dropin_probe.py, 64 MiB pageable drop-in):
// 11.9 / 14.6 / 16.3 GB/s with 8 / 12 / 16 threads.
inline int host_threads() {
  static int t = [] {
    int cpus = (int)std::thread::hardware_concurrency();
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) cpus = CPU_COUNT(&set);
    const char* e = std::getenv("GAES_HOST_THREADS");
    int v = (e && *e) ? std::atoi(e) : std::min(32, cpus);
    return std::max(1, v);
  }();
  return t;
}

inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#else
  std::this_thread::yield();
#endif
}

// Counters behind gaes_host_stats() (measurement / tests).
struct PoolStats {
  std::atomic<int64_t> pools{0};           // pools created (the process pool + one per device in sharded use)
  std::atomic<int64_t> regions{0};         // parallel regions run on a pool
  std::atomic<int64_t> active{0};          // regions running right now
  std::atomic<int64_t> max_active{0};      // most regions ever running at once (across pools)
  std::atomic<int64_t> busy_fallbacks{0};  // regions run on the caller's thread because its pool was busy
};
inline PoolStats& pool_stats() {
  static PoolStats* s = new PoolStats();
  return *s;
}

// Persistent workers (spawning threads per staging copy costs ~50 us).  A
// worker woken from a condition-variable sleep can take a few hundred
// microseconds to run on the GPU box (scripts/exp/dropin_probe.py: 1 MiB
// drop-in calls were slower with the pool than on one thread), so after each
// region workers spin for a short window before sleeping, and warm() lets a
// caller wake them ahead of a burst of regions (a staged pipeline).
//
// Parts are claimed through one 64-bit ticket, (region generation << 32) |
// next part, advanced only by compare-and-swap against the generation the
// claimant joined: a worker descheduled across the end of a region can never
// claim (and run a second time) a part of the next region -- its CAS sees a
// different generation and it leaves.
class HostPool {
 public:
  // n workers (plus the calling thread); cpus: CPU ids to pin them to (empty:
  // the process's affinity mask).
  explicit HostPool(int n, std::vector<int> cpus = {}) : cpus_(std::move(cpus)) {
    pool_stats().pools.fetch_add(1);
    for (int i = 0; i < n; i++) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return (int)workers_.size() + 1; }
  // Runs fn(i) for i in [0, parts) on the workers plus the calling thread
  // and returns true -- or returns false at once if another caller's region
  // is running (concurrent host-API calls then copy on their own threads
  // instead of queueing for the pool).
  bool try_run(size_t parts, const std::function<void(size_t)>& fn) {
    std::unique_lock<std::mutex> call(call_mu_, std::try_to_lock);  // one parallel region at a time
    if (!call.owns_lock()) {
      pool_stats().busy_fallbacks.fetch_add(1);
      return false;
    }
    PoolStats& st = pool_stats();
    st.regions.fetch_add(1);
    const int64_t now = st.active.fetch_add(1) + 1;
    for (int64_t m = st.max_active.load(); now > m && !st.max_active.compare_exchange_weak(m, now);) {
    }
    uint32_t g;
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      parts_ = parts;
      pending_ = parts;
      g = (uint32_t)(gen_.load() + 1);
      ticket_.store((uint64_t)g << 32, std::memory_order_release);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work(g, &fn, parts);
    {
      std::unique_lock<std::mutex> lk(mu_);
      done_cv_.wait(lk, [this] { return pending_ == 0; });
      fn_ = nullptr;
    }
    st.active.fetch_sub(1);
    return true;
  }
  // Wakes sleeping workers into their spin window (no work).
  void warm() {
    if (workers_.empty()) return;
    {
      std::lock_guard<std::mutex> lk(mu_);
      wake_++;
    }
    cv_.notify_all();
  }

 private:
  static constexpr auto kSpin = std::chrono::microseconds(400);
  // Claims and runs parts of region g until none is left (or the region is
  // no longer g).
  void work(uint32_t g, const std::function<void(size_t)>* fn, size_t parts) {
    for (;;) {
      uint64_t t = ticket_.load(std::memory_order_acquire);
      do {
        if ((uint32_t)(t >> 32) != g || (t & 0xFFFFFFFFull) >= parts) return;
      } while (!ticket_.compare_exchange_weak(t, t + 1, std::memory_order_acq_rel));
      (*fn)((size_t)(t & 0xFFFFFFFFull));
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void pin_self() {
    if (cpus_.empty()) return;
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int c : cpus_) CPU_SET(c, &set);
    pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
  }
  void loop() {
    pin_self();
    uint64_t seen = 0, seen_wake = 0;
    for (;;) {
      const auto t0 = std::chrono::steady_clock::now();
      for (int k = 0; gen_.load(std::memory_order_acquire) == seen && !stop_.load(); k++) {
        if ((k & 63) == 0 && std::chrono::steady_clock::now() - t0 > kSpin) break;
        cpu_relax();
      }
      uint32_t g = 0;
      const std::function<void(size_t)>* fn = nullptr;
      size_t parts = 0;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] {
          return stop_.load() || (gen_.load() != seen && fn_ != nullptr) || wake_ != seen_wake;
        });
        if (stop_.load()) return;
        seen_wake = wake_;
        seen = gen_.load();
        if (fn_ == nullptr) continue;  // warm-up only (or the region already ended): spin for the next one
        // join the current region: its generation, body and size, read together
        g = (uint32_t)seen;
        fn = fn_;
        parts = parts_;
      }
      work(g, fn, parts);
    }
  }
  std::vector<int> cpus_;
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* fn_ = nullptr;
  size_t parts_ = 0, pending_ = 0;
  std::atomic<uint64_t> ticket_{0};
  std::atomic<uint64_t> gen_{0};
  uint64_t wake_ = 0;
  std::atomic<bool> stop_{false};
};

// The process-wide pool: every CPU of the affinity mask (host_threads()).
inline HostPool& host_pool() {
  static HostPool* pool = new HostPool(std::max(0, host_threads() - 1));  // leaked: lives until exit
  return *pool;
}

// The pool parallel_ranges uses on this thread: a device's own pool while a
// sharded job runs on it (see PoolScope), else the process pool.
inline HostPool*& current_pool_slot() {
  static thread_local HostPool* p = nullptr;
  return p;
}
inline HostPool& current_pool() {
  HostPool* p = current_pool_slot();
  return p ? *p : host_pool();
}
struct PoolScope {
  HostPool* prev;
  explicit PoolScope(HostPool* p) : prev(current_pool_slot()) { current_pool_slot() = p; }
  ~PoolScope() { current_pool_slot() = prev; }
};

template <typename F>
void parallel_ranges(size_t n, size_t min_per_thread, F&& fn) {
  HostPool& pool = current_pool();
  const size_t want = std::min<size_t>((size_t)pool.size(), std::max<size_t>(1, n / min_per_thread));
  if (want <= 1) {
    fn(0, n);
    return;
  }
  const size_t step = (n + want - 1) / want;
  const std::function<void(size_t)> part = [&](size_t t) {
    const size_t lo = t * step, hi = std::min(n, lo + step);
    if (lo < hi) fn(lo, hi);
  };
  if (!pool.try_run(want, part)) fn(0, n);
}

// Copy with non-temporal (streaming) stores: the destination lines are
// written without first being read into the cache (no read-for-ownership),
// which on a staging copy saves one of the host-DRAM crossings that bound the
// pageable drop-in path (the pinned staging buffer is read next by the DMA
// engine, the caller's output buffer is not re-read by this call).  glibc's
// memcpy only streams above a size threshold far larger than the per-thread
// pieces here.  Ends with sfence: the stores are weakly ordered and must be
// globally visible before the DMA that reads them is issued.
#if defined(__x86_64__)
__attribute__((target("avx2"))) inline void nt_copy_avx2(uint8_t* dst, const uint8_t* src, size_t n) {
  const size_t head = std::min(n, (size_t)((32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31));
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}
#endif

inline bool nt_copies() {
#if defined(__x86_64__)
  static const bool on = rt::tune_int("NT", 1) != 0 && __builtin_cpu_supports("avx2");
  return on;
#else
  return false;
#endif
}

// Single-threaded piece of a staging copy (streaming stores when available).
inline void stage_copy(void* dst, const void* src, size_t bytes) {
#if defined(__x86_64__)
  // (small pieces -- a small job's whole staging copy -- stay in the cache:
  // measured faster for 16-160 KB jobs, scripts/r2/host_floor.cu)
  if (nt_copies() && bytes >= ((size_t)64 << 10)) {
    nt_copy_avx2(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), bytes);
    return;
  }
#endif
  std::memcpy(dst, src, bytes);
}

// Minimum bytes per copy thread of a parallel staging copy.
inline size_t copy_grain() {
  static const size_t grain = (size_t)std::max(4, rt::tune_int("MEMCPY_GRAIN_KB", 128)) << 10;
  return grain;
}

inline void par_memcpy(void* dst, const void* src, size_t bytes) {
  parallel_ranges(bytes, copy_grain(), [&](size_t lo, size_t hi) {
    stage_copy((uint8_t*)dst + lo, (const uint8_t*)src + lo, hi - lo);
  });
}

}  // namespace host
}  // namespace gaes
