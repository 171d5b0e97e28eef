// device_ctx.h -- per-device state of libgaes_b200.so (internal): contexts
// with their GF-layer tables, the lanes of staging slots / streams that
// host-buffer jobs run on, the caller-table cache and the texture cache
// behind the texture-path input loads.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "host_pool.h"
#include "kernels.h"
#include "runtime.h"
#include "types.h"

namespace gaes {
namespace rt {

// --------------------------------------------------------------------------
// Per-device context.
struct Slot {
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  uint8_t *h_in = nullptr, *h_out = nullptr, *h_iv = nullptr;  // pinned staging
  uint8_t *dv_in = nullptr, *dv_out = nullptr, *dv_iv = nullptr;  // their device views (small zero-copy jobs)
  uint8_t *d_in = nullptr, *d_out = nullptr, *d_iv = nullptr;
  size_t cap = 0, iv_cap = 0;
  // pending D2H copy-out (pageable destination)
  uint8_t* pending_dst = nullptr;
  size_t pending_bytes = 0;
};

constexpr int kSlots = 4;
constexpr int kLanes = 4;

// One host-buffer job at a time runs on a lane: its staging slots and
// streams plus the per-job device scratch.  Several lanes per device let
// concurrent callers (the reference's parallel._run_chunks worker threads,
// parallel.py:66-75) overlap their host copies, transfers and kernels
// instead of queueing behind one device mutex.
struct Lane {
  std::mutex mu;
  Slot slots[kSlots];
  uint8_t* d_scratch = nullptr;  // generic path: box(256) lut(4096) perm(16) rk(176)
  uint8_t* d_mk = nullptr;       // many-key: keys | rk_enc | rk_dec | ivs
  size_t mk_cap = 0;
  uint32_t* d_tables = nullptr;  // caller tables built here once the per-device cache is full
};

// Persistent threads that run one device's shards of in-process multi-GPU
// host jobs (gaes_set_num_gpus > 1): up to kLanes of them, created on demand
// and kept for the process, so a sharded call spawns no threads.
class ShardRunner {
 public:
  void post(std::function<void()> f) {
    std::lock_guard<std::mutex> lk(mu_);
    q_.push_back(std::move(f));
    if (idle_ == 0 && threads_ < kLanes) {
      threads_++;
      std::thread([this] { loop(); }).detach();  // lives as long as the (never destroyed) context
    }
    cv_.notify_one();
  }
  int threads() {
    std::lock_guard<std::mutex> lk(mu_);
    return threads_;
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        idle_++;
        cv_.wait(lk, [this] { return !q_.empty(); });
        idle_--;
        f = std::move(q_.front());
        q_.pop_front();
      }
      f();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  int threads_ = 0, idle_ = 0;
};

struct DevCtx {
  int dev = 0;
  int sms = 148;
  uint32_t* d_std_enc = nullptr;  // compact 5x256 (GF layer)
  uint32_t* d_std_dec = nullptr;
  uint8_t std_sbox[256], std_inv[256];
  uint32_t std_te[1024], std_td[1024];
  uint8_t std_mix_fwd[4096], std_mix_inv[4096];  // mix_lut[r][j][x] = M[r][j] * x
  std::mutex cache_mu;
  std::unordered_map<std::string, uint32_t*> cache;  // (box || lut) -> compact tables; never evicted
  uint8_t* d_tmp = nullptr;      // GF-build outputs + error flag
  // S-box / inverse S-box bytes (256 B each) and u8 textures over them: the
  // last round's lookups for the standard tables go through the TEX pipe
  // (0 = unavailable or GAES_TUNE=TEXS=0: read the replicated S table in smem)
  uint8_t* d_sbox = nullptr;
  uint8_t* d_inv = nullptr;
  cudaTextureObject_t tex_s_enc = 0, tex_s_dec = 0;
  // linear textures over input buffers (texture-path loads, see k_blocks),
  // least-recently-used first; see tex_for
  struct Tex {
    const void* ptr = nullptr;
    size_t bytes = 0;
    unsigned long long buffer_id = 0;  // CU_POINTER_ATTRIBUTE_BUFFER_ID of the allocation it views (0: unknown)
    cudaTextureObject_t tex = 0;
    // One event per stream whose launches read this texture, re-recorded
    // after each such launch; eviction waits on all of them.  Past
    // kMaxStreams distinct streams, `overflow` makes eviction wait for the
    // whole device instead.
    static constexpr size_t kMaxStreams = 8;
    std::mutex mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> evs;
    bool overflow = false;
    std::atomic<int> users{0};  // leases not yet enqueued
    uint64_t stamp = 0;
    void record(cudaStream_t s) {
      std::lock_guard<std::mutex> lk(mu);
      for (auto& e : evs)
        if (e.first == s) {
          cudaEventRecord(e.second, s);
          return;
        }
      cudaEvent_t ev = nullptr;
      if (evs.size() < kMaxStreams && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(ev, s);
        evs.emplace_back(s, ev);
      } else {
        cudaGetLastError();
        overflow = true;
      }
    }
    // Blocks until every launch that read the texture has finished.
    bool drain() {
      std::lock_guard<std::mutex> lk(mu);
      bool ok = true;
      for (auto& e : evs) ok &= cudaEventSynchronize(e.second) == cudaSuccess;
      if (overflow) ok &= cudaDeviceSynchronize() == cudaSuccess;
      if (!ok) cudaGetLastError();
      return ok;
    }
    ~Tex() {
      for (auto& e : evs) cudaEventDestroy(e.second);
      if (tex) cudaDestroyTextureObject(tex);
    }
  };
  std::mutex tex_mu;
  std::vector<std::unique_ptr<Tex>> tex_cache;
  uint64_t tex_clock = 0;
  uint64_t tex_created = 0;  // texture objects created over caller / slot buffers (gaes_debug_counters)
  int tex_align = 0;
  size_t tex_max_texels = 0;
  Lane lanes[kLanes];
  // In-process multi-GPU (gaes_set_num_gpus > 1): this device's own host copy
  // pool, its threads pinned to the CPUs local to the GPU's PCIe root
  // (created on first sharded use, see device_pool()), and its shard runners.
  std::once_flag pool_once;
  host::HostPool* pool = nullptr;
  ShardRunner runner;
  // Only runs when initialisation fails (live contexts are never destroyed:
  // freeing after the CUDA runtime has shut down at exit is not allowed).
  ~DevCtx() {
    for (cudaTextureObject_t t : {tex_s_enc, tex_s_dec})
      if (t) cudaDestroyTextureObject(t);
    for (void* p : {(void*)d_std_enc, (void*)d_std_dec, (void*)d_tmp, (void*)d_sbox, (void*)d_inv})
      if (p) cudaFree(p);
    for (auto& L : lanes) {
      for (void* p : {(void*)L.d_scratch, (void*)L.d_mk, (void*)L.d_tables})
        if (p) cudaFree(p);
      for (auto& s : L.slots) {
        if (s.stream) cudaStreamDestroy(s.stream);
        if (s.done) cudaEventDestroy(s.done);
      }
    }
    for (auto& kv : cache) cudaFree(kv.second);
  }
};

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int dev;
  explicit DeviceGuard(int d) : dev(d) {}
  ~DeviceGuard() { cudaSetDevice(dev); }
};

// A texture object lent to one launch.  It converts to the handle the
// launcher takes; when the lease ends -- the end of the full expression that
// enqueued the launch -- the entry's event for the launch stream is recorded,
// so the entry can later be evicted once exactly the kernels that read it,
// on every stream, are done.
class TexLease {
 public:
  TexLease() = default;
  TexLease(DevCtx::Tex* e, cudaStream_t s) : e_(e), s_(s) {}
  TexLease(const TexLease&) = delete;
  TexLease& operator=(const TexLease&) = delete;
  ~TexLease() {
    if (!e_) return;
    e_->record(s_);
    e_->users.fetch_sub(1, std::memory_order_release);
  }
  operator cudaTextureObject_t() const { return e_ ? e_->tex : 0; }

 private:
  DevCtx::Tex* e_ = nullptr;
  cudaStream_t s_ = nullptr;
};

struct PrivateInput {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  ~PrivateInput() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

// A caller output the kernels cannot write directly (not 16-byte aligned:
// they store whole 16-byte blocks): the launches write a private aligned
// buffer and finish() copies it to the caller's pointer, stream-ordered.
struct PrivateOutput {
  void* ptr = nullptr;
  void* dst = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  int finish() {
    if (ptr) GAES_CK(cudaMemcpyAsync(dst, ptr, bytes, cudaMemcpyDeviceToDevice, stream));
    return GAES_OK;
  }
  ~PrivateOutput() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Logical device -> context table (device_ctx.cpp); g_ctx_mu guards it.
extern std::mutex g_ctx_mu;
extern std::vector<DevCtx*>& g_ctx;

// The host copy pool of c for sharded jobs (see DevCtx::pool).
host::HostPool* device_pool(DevCtx* c);
// CPU ids local to CUDA device `dev` (sysfs local_cpulist of its PCI
// function) that this process may run on; empty if unknown.
std::vector<int> device_local_cpus(int dev);
// Number of logical devices (GAES_DEVICE_MAP-aware), -1 before the first query.
int device_count();
// Context of logical device `dev`, created on first use (GF layer built on
// the device and cross-checked against the host restatement).
int get_ctx(int dev, DevCtx** out);
// Context of the caller's current CUDA device.
int current_ctx(DevCtx** out);
// True if the caller's tables equal the device GF layer's.
bool is_standard(const DevCtx* c, bool dec, const uint8_t* box, const uint8_t* lut, const uint8_t* perm);
// Compact T tables for caller-supplied (box, lut); see device_ctx.cpp.
int tables_for(DevCtx* c, Lane* lane, cudaStream_t stream, const uint8_t* box, const uint8_t* lut,
               uint32_t** out);
TexLease tex_for(DevCtx* c, const void* ptr, size_t bytes, cudaStream_t stream);
size_t tex_segment_blocks(DevCtx* c);
int private_input_if_aliased(const void* in, const void* out, size_t bytes, bool identical_is_unsafe,
                             cudaStream_t stream, const void** src, PrivateInput* tmp);
// `p` itself if 16-byte aligned (or null), else a stream-ordered aligned copy
// of its `bytes` (kernels read 16-byte blocks).
int aligned_input(const void* p, size_t bytes, cudaStream_t stream, const void** src, PrivateInput* tmp);
// `out` itself if 16-byte aligned, else a private buffer that tmp->finish()
// copies to `out` after the launches.
int aligned_output(void* out, size_t bytes, cudaStream_t stream, void** dst, PrivateOutput* tmp);
int ilp_default();
// S-box texture matching the compact tables `compact` (standard tables only).
cudaTextureObject_t sbox_tex(const DevCtx* c, const uint32_t* compact);
// M = 16 shared-IV encrypt: the formulation chosen by measurement
// (profiles/): T-table unless gaes_set_variant(2) selects the bitsliced kernel.
// host_job: a synchronous host-buffer job (see launch_blocks_small's `early`).
cudaError_t launch_enc_folded(DevCtx* c, const void* in, void* out, uint64_t n, const uint32_t* compact,
                              const RoundKeys& k, int ilp, cudaStream_t s, cudaTextureObject_t tin,
                              bool host_job = false);

// M = 16 with the IV folded into the key (either direction): the small-batch
// kernel for standard tables and n <= small_blocks_max, else k_blocks.
cudaError_t launch_folded(DevCtx* c, bool dec, const void* in, void* out, uint64_t n, const uint32_t* compact,
                          const RoundKeys& k, cudaStream_t s, cudaTextureObject_t tin, bool host_job = false);

// Runs fn(offset, count) over [0, n) in texture-sized segments.
template <typename F>
int for_segments(DevCtx* c, size_t n, F&& fn) {
  size_t seg = tex_segment_blocks(c);
  if (seg == 0 || n <= seg) return fn((size_t)0, n);
  for (size_t off = 0; off < n; off += seg) {
    int rc = fn(off, std::min(seg, n - off));
    if (rc) return rc;
  }
  return GAES_OK;
}

}  // namespace rt
}  // namespace gaes
