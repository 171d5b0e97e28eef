// device_ctx.h -- per-device state of libgaes_b200.so (internal): contexts
// with their GF-layer tables, the lanes of staging slots / streams that
// host-buffer jobs run on, the caller-table cache and the texture cache
// behind the texture-path input loads.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

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
  // (0 = unavailable or GAES_TEXS=0: read the replicated S table in smem)
  uint8_t* d_sbox = nullptr;
  uint8_t* d_inv = nullptr;
  cudaTextureObject_t tex_s_enc = 0, tex_s_dec = 0;
  // linear textures over input buffers (texture-path loads, see k_blocks),
  // least-recently-used first; see tex_for
  struct Tex {
    const void* ptr = nullptr;
    size_t bytes = 0;
    cudaTextureObject_t tex = 0;
    cudaEvent_t last = nullptr;  // recorded after every launch that reads it
    std::atomic<int> users{0};   // leases not yet enqueued
    uint64_t stamp = 0;
  };
  std::mutex tex_mu;
  std::vector<std::unique_ptr<Tex>> tex_cache;
  uint64_t tex_clock = 0;
  int tex_align = 0;
  size_t tex_max_texels = 0;
  Lane lanes[kLanes];
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
    for (auto& t : tex_cache) {
      cudaDestroyTextureObject(t->tex);
      if (t->last) cudaEventDestroy(t->last);
    }
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
// enqueued the launch -- an event is recorded on the launch stream, so the
// entry can later be evicted once exactly the kernels that read it are done.
class TexLease {
 public:
  TexLease() = default;
  TexLease(DevCtx::Tex* e, cudaStream_t s) : e_(e), s_(s) {}
  TexLease(const TexLease&) = delete;
  TexLease& operator=(const TexLease&) = delete;
  ~TexLease() {
    if (!e_) return;
    cudaEventRecord(e_->last, s_);
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
int ilp_default();
// S-box texture matching the compact tables `compact` (standard tables only).
cudaTextureObject_t sbox_tex(const DevCtx* c, const uint32_t* compact);
// M = 16 shared-IV encrypt: the formulation chosen by measurement
// (profiles/): T-table unless gaes_set_variant(2) selects the bitsliced kernel.
cudaError_t launch_enc_folded(DevCtx* c, const void* in, void* out, uint64_t n, const uint32_t* compact,
                              const RoundKeys& k, int ilp, cudaStream_t s, cudaTextureObject_t tin);

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
