// dispatch.cpp -- host side of libgaes_b200.so: the C ABI (include/gaes_b200.h),
// per-device contexts, table caching, the H2D -> kernel -> D2H pipeline and
// the multi-GPU row sharding.
//
// Reference boundary replaced: pkg/src/gaes/backend.py:56-61 forwards
// cbc_encrypt / cbc_decrypt (7 arguments) to the active kernel module;
// _kernel.pyx:12-101 is the kernel.  parallel.py:37-50 (plan) and :66-75
// (thread fan-out over contiguous row ranges) become the GPU shard plan.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/gaes_b200.h"
#include "aes_bitslice.cuh"
#include "gf.cuh"
#include "host_pool.h"
#include "kernels.h"
#include "round_keys.h"

using namespace gaes;
using namespace gaes::host;

namespace {

constexpr int kVersion = 10000;  // 1.0.0
constexpr uint8_t kShiftRowsSrc[16] = {0, 5, 10, 15, 4, 9, 14, 3, 8, 13, 2, 7, 12, 1, 6, 11};  // aes_cbc.py:41
constexpr uint8_t kInvShiftRowsSrc[16] = {0, 13, 10, 7, 4, 1, 14, 11, 8, 5, 2, 15, 12, 9, 6, 3};  // :42

thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};
std::mutex g_name_mu;
std::string g_last_kernel = "";
std::atomic<int> g_num_gpus{0};
std::atomic<int> g_variant{0};

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

#define GAES_CK(expr)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(GAES_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

void note_kernel(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  std::lock_guard<std::mutex> lk(g_name_mu);
  g_last_kernel = name;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atoi(v);
}

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
    for (void* p : {(void*)d_std_enc, (void*)d_std_dec, (void*)d_tmp})
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

std::mutex g_ctx_mu;
// Contexts live for the process (never destroyed, see ~DevCtx).
std::vector<DevCtx*>& g_ctx = *new std::vector<DevCtx*>();
int g_ndev = -1;

// Logical device i -> physical CUDA device g_phys[i].  Identity unless
// GAES_DEVICE_MAP="a,b,..." is set (e.g. "0,0" runs the multi-GPU shard path
// as two contexts on one GPU -- used to test the sharding on a 1-GPU box; the
// shards never wait on each other, so sharing a GPU is safe).
std::vector<int>& g_phys = *new std::vector<int>();

int device_count() {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if (g_ndev < 0) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    g_phys.clear();
    const char* map = std::getenv("GAES_DEVICE_MAP");
    if (n > 0 && map && *map) {
      for (const char* p = map; *p;) {
        char* end = nullptr;
        const long d = std::strtol(p, &end, 10);
        if (end == p) break;
        if (d >= 0 && d < n) g_phys.push_back((int)d);
        p = (*end == ',') ? end + 1 : end;
        if (*end != ',' && *end) break;
      }
    }
    if (g_phys.empty())
      for (int i = 0; i < n; i++) g_phys.push_back(i);
    g_ndev = (int)g_phys.size();
    g_ctx.resize(g_ndev);
  }
  return g_ndev;
}

// Creates the context on first use: GF-layer tables built on the device.
int get_ctx(int dev, DevCtx** out) {
  const int n = device_count();
  if (n <= 0) return fail(GAES_ENODEV, "no CUDA device visible");
  if (dev < 0 || dev >= n) return fail(GAES_EINVAL, "device index out of range");
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if (g_ctx[dev]) {
    *out = g_ctx[dev];
    return GAES_OK;
  }
  auto c = std::make_unique<DevCtx>();
  c->dev = g_phys[dev];
  int prev = 0;
  GAES_CK(cudaGetDevice(&prev));
  DeviceGuard guard(prev);
  GAES_CK(cudaSetDevice(c->dev));
  GAES_CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->dev));
  GAES_CK(cudaMalloc(&c->d_std_enc, kCompactWords * 4));
  GAES_CK(cudaMalloc(&c->d_std_dec, kCompactWords * 4));
  GAES_CK(cudaMalloc(&c->d_tmp, 512 + sizeof(int)));
  uint8_t* d_box = c->d_tmp;
  int* d_err = reinterpret_cast<int*>(c->d_tmp + 512);
  GAES_CK(cudaMemset(d_err, 0, sizeof(int)));
  GAES_CK(launch_gf_build(c->d_std_enc, c->d_std_dec, d_box, d_box + 256, d_err, 0));
  note_kernel("k_gf_build");
  int err = 0;
  GAES_CK(cudaMemcpy(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
  GAES_CK(cudaMemcpy(c->std_sbox, d_box, 256, cudaMemcpyDeviceToHost));
  GAES_CK(cudaMemcpy(c->std_inv, d_box + 256, 256, cudaMemcpyDeviceToHost));
  uint32_t tmp[kCompactWords];
  GAES_CK(cudaMemcpy(tmp, c->d_std_enc, sizeof(tmp), cudaMemcpyDeviceToHost));
  std::memcpy(c->std_te, tmp, sizeof(c->std_te));
  GAES_CK(cudaMemcpy(tmp, c->d_std_dec, sizeof(tmp), cudaMemcpyDeviceToHost));
  std::memcpy(c->std_td, tmp, sizeof(c->std_td));
  for (auto& L : c->lanes) {
    GAES_CK(cudaMalloc(&L.d_scratch, 256 + 4096 + 16 + 176 + 512));
    for (auto& s : L.slots) {
      GAES_CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
      GAES_CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    }
  }
  if (err) return fail(GAES_ETABLE, "GF layer self check failed (S^-1 o S != id or M.M^-1 != I)");
  // The device-built S-box must equal the host restatement of the same
  // field arithmetic (gf.cuh is compiled for both sides).
  for (int v = 0; v < 256; v++)
    if (c->std_sbox[v] != sbox_forward((uint8_t)v) || c->std_inv[v] != sbox_inverse((uint8_t)v))
      return fail(GAES_ETABLE, "device GF tables disagree with the host field arithmetic");
  for (int r = 0; r < 4; r++)
    for (int j = 0; j < 4; j++)
      for (int x = 0; x < 256; x++) {
        c->std_mix_fwd[(r * 4 + j) * 256 + x] = gf_mul(mix_coef(false, r, j), (uint8_t)x);
        c->std_mix_inv[(r * 4 + j) * 256 + x] = gf_mul(mix_coef(true, r, j), (uint8_t)x);
      }
  g_ctx[dev] = c.release();
  *out = g_ctx[dev];
  return GAES_OK;
}

// True if the caller's tables equal the device GF layer's (the usual drop-in
// case: aes_cbc._encrypt_tables / _decrypt_tables build exactly these).
bool is_standard(const DevCtx* c, bool dec, const uint8_t* box, const uint8_t* lut, const uint8_t* perm) {
  static const uint8_t kShift[16] = {0, 5, 10, 15, 4, 9, 14, 3, 8, 13, 2, 7, 12, 1, 6, 11};
  static const uint8_t kInvShift[16] = {0, 13, 10, 7, 4, 1, 14, 11, 8, 5, 2, 15, 12, 9, 6, 3};
  return std::memcmp(box, dec ? c->std_inv : c->std_sbox, 256) == 0 &&
         std::memcmp(lut, dec ? c->std_mix_inv : c->std_mix_fwd, 4096) == 0 &&
         std::memcmp(perm, dec ? kInvShift : kShift, 16) == 0;
}

// Context of the caller's current CUDA device (first logical device mapped
// to it).
int current_ctx(DevCtx** out) {
  int dev = 0;
  if (device_count() <= 0) return fail(GAES_ENODEV, "no CUDA device visible");
  GAES_CK(cudaGetDevice(&dev));
  for (size_t i = 0; i < g_phys.size(); i++)
    if (g_phys[i] == dev) return get_ctx((int)i, out);
  return fail(GAES_EINVAL, "current device is not in GAES_DEVICE_MAP");
}

// Compact T tables for caller-supplied (box, lut), cached per device (up to
// 64 sets, never evicted: a concurrent job may be about to launch with any
// cached pointer).  Past that, the tables are built into the lane's own
// buffer for this job.  `stream` is the lane's stream.
int tables_for(DevCtx* c, Lane* lane, cudaStream_t stream, const uint8_t* box, const uint8_t* lut,
               uint32_t** out) {
  std::string key(reinterpret_cast<const char*>(box), 256);
  key.append(reinterpret_cast<const char*>(lut), 4096);
  std::lock_guard<std::mutex> lk(c->cache_mu);
  auto it = c->cache.find(key);
  if (it != c->cache.end()) {
    *out = it->second;
    return GAES_OK;
  }
  const bool cache_it = c->cache.size() < 64;
  struct DevBuf {  // freed on every exit path unless released
    void* p = nullptr;
    ~DevBuf() {
      if (p) cudaFree(p);
    }
  } d, d_in;
  uint32_t* tables = nullptr;
  if (cache_it) {
    GAES_CK(cudaMalloc(&d.p, kCompactWords * 4));
    tables = static_cast<uint32_t*>(d.p);
  } else {
    if (!lane->d_tables) GAES_CK(cudaMalloc(&lane->d_tables, kCompactWords * 4));
    tables = lane->d_tables;
  }
  GAES_CK(cudaMalloc(&d_in.p, 256 + 4096));
  uint8_t* in8 = static_cast<uint8_t*>(d_in.p);
  GAES_CK(cudaMemcpyAsync(in8, box, 256, cudaMemcpyHostToDevice, stream));
  GAES_CK(cudaMemcpyAsync(in8 + 256, lut, 4096, cudaMemcpyHostToDevice, stream));
  GAES_CK(launch_build_tables(in8, in8 + 256, tables, stream));
  note_kernel("k_build_tables");
  GAES_CK(cudaStreamSynchronize(stream));
  if (cache_it) {
    d.p = nullptr;
    c->cache.emplace(key, tables);
  }
  *out = tables;
  return GAES_OK;
}

// Texture limits of c->dev, queried once.  Must be called with c->tex_mu held.
void query_tex_limits(DevCtx* c) {
  if (c->tex_align != 0) return;
  int align = 0, maxw = 0;
  if (cudaDeviceGetAttribute(&align, cudaDevAttrTextureAlignment, c->dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxTexture1DLinearWidth, c->dev) != cudaSuccess) {
    cudaGetLastError();
    c->tex_align = -1;
  } else {
    c->tex_align = std::max(align, 16);
    c->tex_max_texels = (size_t)maxw;
  }
}

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

// A linear uint4 texture over [ptr, ptr + bytes) for the texture-path input
// loads, cached per device by pointer (callers and the staging slots reuse
// buffers).  Empty (handle 0) when disabled (GAES_TEXIN=0), misaligned, too
// large or unavailable -- the kernels then use LDG.  Must be called with
// c->dev current and the lease used for one launch on `stream`.  At 64
// entries the least recently used idle entry is evicted after waiting for
// the launches that read it (its `last` event); entries lent out right now
// are never evicted.
TexLease tex_for(DevCtx* c, const void* ptr, size_t bytes, cudaStream_t stream) {
  static const bool enabled = env_int("GAES_TEXIN", 1) != 0;
  if (!enabled || !ptr || bytes < 16) return {};
  // A launch captured into a CUDA graph may be replayed long after this
  // cache evicted (destroyed) the texture object; captured launches use LDG.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cap) != cudaSuccess) {
    cudaGetLastError();
    return {};
  }
  if (cap != cudaStreamCaptureStatusNone) return {};
  std::lock_guard<std::mutex> lk(c->tex_mu);
  query_tex_limits(c);
  if (c->tex_align < 0 || reinterpret_cast<uintptr_t>(ptr) % (uintptr_t)c->tex_align != 0) return {};
  if (bytes / 16 > c->tex_max_texels || bytes / 16 > 0x7FFFFFFFull) return {};
  for (auto& t : c->tex_cache)
    if (t->ptr == ptr && t->bytes >= bytes) {
      t->users.fetch_add(1, std::memory_order_acquire);
      t->stamp = ++c->tex_clock;
      return TexLease(t.get(), stream);
    }
  if (c->tex_cache.size() >= 64) {
    // users only grows under tex_mu, so an idle entry seen here stays idle
    size_t victim = c->tex_cache.size();
    for (size_t i = 0; i < c->tex_cache.size(); i++)
      if (c->tex_cache[i]->users.load(std::memory_order_acquire) == 0 &&
          (victim == c->tex_cache.size() || c->tex_cache[i]->stamp < c->tex_cache[victim]->stamp))
        victim = i;
    if (victim == c->tex_cache.size()) return {};
    auto& v = c->tex_cache[victim];
    if (cudaEventSynchronize(v->last) != cudaSuccess) {
      cudaGetLastError();
      return {};
    }
    cudaDestroyTextureObject(v->tex);
    cudaEventDestroy(v->last);
    c->tex_cache.erase(c->tex_cache.begin() + victim);
  }
  auto e = std::make_unique<DevCtx::Tex>();
  if (cudaEventCreateWithFlags(&e->last, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return {};
  }
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = const_cast<void*>(ptr);
  rd.res.linear.desc = cudaCreateChannelDesc<uint4>();
  rd.res.linear.sizeInBytes = bytes / 16 * 16;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  if (cudaCreateTextureObject(&e->tex, &rd, &td, nullptr) != cudaSuccess) {
    cudaGetLastError();
    cudaEventDestroy(e->last);
    return {};
  }
  e->ptr = ptr;
  e->bytes = bytes;
  e->stamp = ++c->tex_clock;
  e->users.store(1, std::memory_order_relaxed);
  c->tex_cache.push_back(std::move(e));
  return TexLease(c->tex_cache.back().get(), stream);
}

// Largest launch (in 16-byte blocks) that a texture can cover on this
// device; device-API calls above it are cut into segments so every segment
// keeps the texture-path loads.  0 = textures unavailable.
size_t tex_segment_blocks(DevCtx* c) {
  std::lock_guard<std::mutex> lk(c->tex_mu);
  query_tex_limits(c);
  if (c->tex_align < 0) return 0;
  size_t seg = std::min<size_t>(c->tex_max_texels, 0x7FFFFFFFull);
  return seg & ~((size_t)(1 << 20) - 1);
}

// Device-API aliasing.  Every kernel reads a block before writing the same
// block, so out == in is safe -- except block-parallel CBC decrypt, where the
// first lane of each warp reads its chain value in[b-1] from a block another
// warp may already have overwritten.  Partially overlapping ranges are unsafe
// for every kernel.  In those cases the input is first copied to a
// stream-ordered private buffer (freed on the same stream after the launch).
struct PrivateInput {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  ~PrivateInput() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

int private_input_if_aliased(const void* in, const void* out, size_t bytes, bool identical_is_unsafe,
                             cudaStream_t stream, const void** src, PrivateInput* tmp) {
  *src = in;
  const uintptr_t a = reinterpret_cast<uintptr_t>(in), b = reinterpret_cast<uintptr_t>(out);
  const bool overlap = a < b + bytes && b < a + bytes;
  if (!overlap || (a == b && !identical_is_unsafe)) return GAES_OK;
  GAES_CK(cudaMallocAsync(&tmp->ptr, bytes, stream));
  tmp->stream = stream;
  GAES_CK(cudaMemcpyAsync(tmp->ptr, in, bytes, cudaMemcpyDeviceToDevice, stream));
  *src = tmp->ptr;
  return GAES_OK;
}

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

// M = 16 shared-IV encrypt: the formulation chosen by measurement
// (profiles/): T-table unless gaes_set_variant(2) selects the bitsliced kernel.
cudaError_t launch_enc_folded(DevCtx* c, const void* in, void* out, uint64_t n, const uint32_t* compact,
                              const RoundKeys& k, int ilp, cudaStream_t s, cudaTextureObject_t tin);

int ilp_default() {
  // ILP 1 measured ~1% faster than 2 at configs 2 and 3 (finer tail, 40 regs)
  static int ilp = std::max(1, std::min(2, env_int("GAES_ILP", 1)));
  return ilp;
}

cudaError_t launch_enc_folded(DevCtx* c, const void* in, void* out, uint64_t n, const uint32_t* compact,
                              const RoundKeys& k, int ilp, cudaStream_t s, cudaTextureObject_t tin) {
  if (g_variant.load() == 2) {
    static thread_local BitsliceKeys bk;
    bs_make_keys(k.w, bk);
    note_kernel("k_bs_blocks");
    return launch_bs_blocks(in, out, n, bk, c->sms, s);
  }
  note_kernel("k_blocks_enc_folded");
  return launch_blocks(false, kIvFolded, ilp, in, out, n, compact, k, nullptr, 1, c->sms, s, tin);
}

// --------------------------------------------------------------------------
// Host-buffer pipeline.
enum class Mode { kFolded, kChain, kEncRows, kGeneric, kManyKey };

struct Job {
  bool dec = false;
  Mode mode = Mode::kFolded;
  const uint8_t* data = nullptr;
  const uint8_t* ivs = nullptr;  // per-row IVs (kChain with rows, kEncRows, kGeneric) or nullptr
  uint8_t* out = nullptr;
  size_t n = 0, m = 16;
  RoundKeys rk;
  const uint8_t* raw_rk = nullptr;  // generic path
  const uint8_t *box = nullptr, *lut = nullptr, *perm = nullptr;
  bool standard = true;  // use the device GF tables
  // kManyKey: key i owns global blocks [i*bpk, (i+1)*bpk); this job's rows
  // start at global block `first`; keys / per-key IVs are host arrays.
  size_t bpk = 0, first = 0, n_keys = 0;
  const uint8_t* mk_keys = nullptr;
  const uint8_t* mk_ivs = nullptr;
  // auto_iv (pageable drop-in calls): `ivs` may be IVSet.rows' tiling of one
  // IV.  Each staged chunk checks its rows against iv0 while it is copied;
  // chunks that match run the shared variant (mode_shared / rk_shared, no IV
  // rows cross PCIe), the others the per-row variant (mode / rk / ivs).
  bool auto_iv = false;
  const uint8_t* iv0 = nullptr;
  Mode mode_shared = Mode::kFolded;
  RoundKeys rk_shared;
};

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Device address of a pinned (page-locked, mapped) host pointer, or nullptr.
const uint8_t* host_dev_view(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? static_cast<const uint8_t*>(a.devicePointer) : nullptr;
}

// Jobs up to this size on pinned caller buffers run as one zero-copy launch.
size_t zero_copy_bytes() {
  static size_t b = (size_t)std::max(0, env_int("GAES_ZEROCOPY_MB", 64)) << 20;
  return b;
}

size_t chunk_bytes() {
  static size_t b = (size_t)std::max(1, env_int("GAES_CHUNK_MB", 32)) << 20;
  return b;
}

int ensure_slot(Slot& s, size_t bytes, size_t iv_bytes, bool staged_in, bool staged_out) {
  if (s.cap < bytes) {
    if (s.d_in) cudaFree(s.d_in);
    if (s.d_out) cudaFree(s.d_out);
    if (s.h_in) cudaFreeHost(s.h_in);
    if (s.h_out) cudaFreeHost(s.h_out);
    s.d_in = s.d_out = s.h_in = s.h_out = nullptr;
    s.cap = 0;
    GAES_CK(cudaMalloc(&s.d_in, bytes));
    GAES_CK(cudaMalloc(&s.d_out, bytes));
    s.cap = bytes;
  }
  if (staged_in && !s.h_in) GAES_CK(cudaMallocHost(&s.h_in, s.cap));
  if (staged_out && !s.h_out) GAES_CK(cudaMallocHost(&s.h_out, s.cap));
  if (iv_bytes && s.iv_cap < iv_bytes) {
    if (s.d_iv) cudaFree(s.d_iv);
    if (s.h_iv) cudaFreeHost(s.h_iv);
    s.d_iv = s.h_iv = nullptr;
    s.iv_cap = 0;
    GAES_CK(cudaMalloc(&s.d_iv, iv_bytes));
    GAES_CK(cudaMallocHost(&s.h_iv, iv_bytes));
    s.iv_cap = iv_bytes;
  }
  return GAES_OK;
}

int finish_slot(Slot& s) {
  GAES_CK(cudaEventSynchronize(s.done));
  if (s.pending_dst) {
    par_memcpy(s.pending_dst, s.h_out, s.pending_bytes);
    s.pending_dst = nullptr;
    s.pending_bytes = 0;
  }
  return GAES_OK;
}

// One kernel launch over rows [r0, r0 + rows) of job j: `in` / `out` / `ivs`
// hold exactly those rows (device staging buffers, or the caller's pinned
// host buffers for a zero-copy launch); `tin` is a texture over `in` or 0.
int launch_chunk(DevCtx* c, Lane* lane, const Job& j, cudaStream_t stream, const uint8_t* in, uint8_t* out,
                 const uint8_t* ivs, size_t r0, size_t rows, const uint32_t* compact, cudaTextureObject_t tin,
                 cudaTextureObject_t tiv = 0) {
  const uint64_t bpr = j.m / 16;
  const uint64_t nblk = rows * bpr;
  switch (j.mode) {
    case Mode::kFolded:
      if (j.dec) {
        GAES_CK(launch_blocks(true, kIvFolded, ilp_default(), in, out, nblk, compact, j.rk, nullptr, 1,
                              c->sms, stream, tin));
        note_kernel("k_blocks_dec_folded");
      } else if (j.standard || g_variant.load() < 2) {
        GAES_CK(launch_enc_folded(c, in, out, nblk, compact, j.rk, ilp_default(), stream,
                                  tin));
      } else {  // bitsliced kernel has the standard S-box built in; caller tables -> T-table
        GAES_CK(launch_blocks(false, kIvFolded, ilp_default(), in, out, nblk, compact, j.rk, nullptr, 1,
                              c->sms, stream));
        note_kernel("k_blocks_enc_folded");
      }
      break;
    case Mode::kChain:
      GAES_CK(launch_blocks(j.dec, kIvChain, ilp_default(), in, out, nblk, compact, j.rk,
                            j.ivs ? ivs : nullptr, bpr, c->sms, stream, tin, j.ivs ? tiv : 0));
      note_kernel(j.dec ? "k_blocks_dec_chain" : "k_blocks_enc_chain");
      break;
    case Mode::kEncRows:
      GAES_CK(launch_cbc_enc_rows(in, out, rows, bpr, compact, j.rk, j.ivs ? ivs : nullptr, c->sms,
                                  stream, tin));
      note_kernel("k_cbc_enc_rows");
      break;
    case Mode::kManyKey: {
      const size_t kb = j.n_keys * 16, rkb = j.n_keys * 176;
      GAES_CK(launch_many_key(j.dec, in, out, nblk, j.first + r0, j.bpk, compact,
                              lane->d_mk + kb + (j.dec ? rkb : 0), j.mk_ivs ? lane->d_mk + kb + 2 * rkb : nullptr, c->sms,
                              stream, tin));
      note_kernel(j.dec ? "k_many_key_dec" : "k_many_key_enc");
      break;
    }
    case Mode::kGeneric: {
      uint8_t* sc = lane->d_scratch;
      GAES_CK(launch_generic(j.dec, in, ivs, rows, j.m, sc + 256 + 4096 + 16, sc, sc + 256, sc + 256 + 4096,
                             out, c->sms, stream));
      note_kernel("k_generic_cbc");
      break;
    }
  }
  return GAES_OK;
}

// One parallel pass over a staged chunk: copy rows [0, rows) of width m to
// the pinned staging buffer and check that their IV rows all equal iv0
// (IVSet.rows tiles a shared IV, aes_cbc.py:107-115).  Fusing the check into
// the copy keeps the IV grid off the critical path: no whole-grid pre-scan
// before the first chunk.
bool stage_and_check_iv(uint8_t* dst, const uint8_t* src, size_t m, const uint8_t* ivs, size_t rows,
                        const uint8_t* iv0) {
  std::atomic<bool> same{true};
  uint64_t a0, a1;
  std::memcpy(&a0, iv0, 8);
  std::memcpy(&a1, iv0 + 8, 8);
  parallel_ranges(rows, std::max<size_t>(1, ((size_t)128 << 10) / m), [&](size_t lo, size_t hi) {
    std::memcpy(dst + lo * m, src + lo * m, (hi - lo) * m);
    if (!same.load(std::memory_order_relaxed)) return;
    uint64_t diff = 0;
    for (size_t i = lo; i < hi; i++) {
      uint64_t b0, b1;
      std::memcpy(&b0, ivs + 16 * i, 8);
      std::memcpy(&b1, ivs + 16 * i + 8, 8);
      diff |= (a0 ^ b0) | (a1 ^ b1);
    }
    if (diff) same.store(false, std::memory_order_relaxed);
  });
  return same.load();
}

// Runs rows [0, j.n) of `j` on device context c (one shard).
// Locks the first free lane of c (lane 0 for a lone caller, so its staging
// buffers -- allocated on first use, cudaMallocHost costs milliseconds -- are
// reused call after call; lanes 1.. only for concurrent callers); if all
// are busy, waits on one chosen by thread.
std::unique_lock<std::mutex> lock_lane(DevCtx* c, Lane** out) {
  static const int lanes = std::max(1, std::min(kLanes, env_int("GAES_LANES", kLanes)));
  for (int k = 0; k < lanes; k++) {
    std::unique_lock<std::mutex> lk(c->lanes[k].mu, std::try_to_lock);
    if (lk.owns_lock()) {
      *out = &c->lanes[k];
      return lk;
    }
  }
  const size_t k = std::hash<std::thread::id>{}(std::this_thread::get_id()) % lanes;
  *out = &c->lanes[k];
  return std::unique_lock<std::mutex>(c->lanes[k].mu);
}

int run_job(DevCtx* c, const Job& j) {
  if (j.n == 0) return GAES_OK;
  Lane* lane = nullptr;
  std::unique_lock<std::mutex> lk = lock_lane(c, &lane);
  int prev = 0;
  GAES_CK(cudaGetDevice(&prev));
  DeviceGuard guard(prev);
  GAES_CK(cudaSetDevice(c->dev));
  // On any early return: wait for whatever was issued and drop pending
  // copy-outs, so the next call never writes into this call's buffers.
  struct Drain {
    Lane* lane;
    bool armed = true;
    ~Drain() {
      if (!armed) return;
      for (auto& s : lane->slots) {
        if (s.stream) cudaStreamSynchronize(s.stream);
        s.pending_dst = nullptr;
        s.pending_bytes = 0;
      }
    }
  } drain{lane};

  const uint32_t* compact = nullptr;
  if (j.mode != Mode::kGeneric) {
    if (j.standard) {
      compact = j.dec ? c->d_std_dec : c->d_std_enc;
    } else {
      uint32_t* t = nullptr;
      int rc = tables_for(c, lane, lane->slots[0].stream, j.box, j.lut, &t);
      if (rc) return rc;
      compact = t;
    }
  } else {
    uint8_t* sc = lane->d_scratch;
    GAES_CK(cudaMemcpy(sc, j.box, 256, cudaMemcpyHostToDevice));
    GAES_CK(cudaMemcpy(sc + 256, j.lut, 4096, cudaMemcpyHostToDevice));
    GAES_CK(cudaMemcpy(sc + 256 + 4096, j.perm, 16, cudaMemcpyHostToDevice));
    GAES_CK(cudaMemcpy(sc + 256 + 4096 + 16, j.raw_rk, 176, cudaMemcpyHostToDevice));
  }

  if (j.mode == Mode::kManyKey) {
    // keys (and per-key IVs) to the device, batched key schedule there
    // layout: keys (K x 16) | rk_enc (K x 176) | rk_dec (K x 176) | ivs (K x 16)
    const size_t need = j.n_keys * (16 + 176 + 176 + 16);
    if (lane->mk_cap < need) {
      if (lane->d_mk) cudaFree(lane->d_mk);
      lane->d_mk = nullptr;
      lane->mk_cap = 0;
      GAES_CK(cudaMalloc(&lane->d_mk, need));
      lane->mk_cap = need;
    }
    const size_t kb = j.n_keys * 16;
    cudaStream_t s0 = lane->slots[0].stream;
    GAES_CK(cudaMemcpyAsync(lane->d_mk, j.mk_keys, kb, cudaMemcpyHostToDevice, s0));
    if (j.mk_ivs)
      GAES_CK(cudaMemcpyAsync(lane->d_mk + kb + 2 * j.n_keys * 176, j.mk_ivs, kb, cudaMemcpyHostToDevice, s0));
    // encrypt and equivalent-inverse-cipher (decrypt) schedules
    GAES_CK(launch_expand_keys(lane->d_mk, j.n_keys, c->d_std_enc, lane->d_mk + kb,
                               j.dec ? lane->d_mk + kb + j.n_keys * 176 : nullptr, s0));
    note_kernel("k_expand_keys");
    GAES_CK(cudaStreamSynchronize(s0));
  }

  const bool in_pinned = is_pinned(j.data);
  const bool out_pinned = is_pinned(j.out);
  if (!(in_pinned && out_pinned) && j.n * j.m >= ((size_t)256 << 10)) host_pool().warm();
  const bool need_iv = j.ivs != nullptr;
  const bool iv_pinned = need_iv && is_pinned(j.ivs);

  // Pinned caller buffers and a job small enough that the staged pipeline's
  // ramp dominates: one zero-copy launch -- the kernel reads and writes the
  // caller's host memory over PCIe itself, no staging copies
  // (scripts/exp/zerocopy_probe.py: 21 vs 15 GB/s at 1 MiB, 34 vs 32 at
  // 16 MiB, 38.6 vs 37.9 at 64 MiB; the staged pipeline leads from 256 MiB).
  // Not for byte-level generic tables (byte loads over PCIe) nor for
  // overlapping in/out (the kernels assume distinct buffers).
  const size_t total = j.n * j.m;
  const uintptr_t ia = reinterpret_cast<uintptr_t>(j.data), oa = reinterpret_cast<uintptr_t>(j.out);
  if (in_pinned && out_pinned && (!need_iv || iv_pinned) && j.mode != Mode::kGeneric && total <= zero_copy_bytes() &&
      !(ia < oa + total && oa < ia + total)) {
    const uint8_t* din = host_dev_view(j.data);
    uint8_t* dout = const_cast<uint8_t*>(host_dev_view(j.out));
    const uint8_t* div = need_iv ? host_dev_view(j.ivs) : nullptr;
    if (din && dout && (!need_iv || div)) {
      cudaStream_t st = lane->slots[0].stream;
      int rc = launch_chunk(c, lane, j, st, din, dout, div, 0, j.n, compact, 0);
      if (rc) return rc;
      GAES_CK(cudaStreamSynchronize(st));
      drain.armed = false;
      return GAES_OK;
    }
  }
  // Chunk schedule: ramp up from base/8 so the first H2D is short (nothing
  // overlaps it), run at `base`, ramp down at the end so the last D2H is
  // short too.  All chunks are whole rows.
  // Pageable buffers are staged by host copies: smaller chunks let the copy
  // of chunk c+1 overlap the DMA of chunk c.
  // pageable callers: 16 MiB (17.0 vs 16.3 / 15.2 GB/s with 8 / 4 MiB, 16 threads)
  static const size_t pageable_chunk = (size_t)std::max(1, env_int("GAES_PAGEABLE_CHUNK_MB", 16)) << 20;
  const size_t base_bytes = (in_pinned && out_pinned) ? chunk_bytes() : std::min<size_t>(chunk_bytes(), pageable_chunk);
  const size_t base_rows = std::max<size_t>(1, base_bytes / j.m);
  const size_t min_rows = std::max<size_t>(1, base_rows / 8);
  std::vector<std::pair<size_t, size_t>> chunks;  // (first row, rows)
  {
    size_t r0 = 0, cur = min_rows;
    while (r0 < j.n) {
      const size_t left = j.n - r0;
      size_t take = std::min(cur, left);
      if (left <= 2 * base_rows) take = std::min(take, std::max(min_rows, (left + 1) / 2));
      if (left - take < min_rows / 2) take = left;
      chunks.emplace_back(r0, take);
      r0 += take;
      cur = std::min(base_rows, cur * 2);
    }
  }
  size_t max_rows = 0;
  for (auto& ch : chunks) max_rows = std::max(max_rows, ch.second);
  const size_t nchunks = chunks.size();
  const int used_slots = (int)std::min<size_t>(kSlots, nchunks);
  for (int k = 0; k < used_slots; k++) {
    int rc = ensure_slot(lane->slots[k], max_rows * j.m, need_iv ? max_rows * 16 : 0, !in_pinned, !out_pinned);
    if (rc) return rc;
  }
  int rc_final = GAES_OK;
  for (size_t ci = 0; ci < nchunks; ci++) {
    Slot& s = lane->slots[ci % kSlots];
    if (ci >= (size_t)kSlots) {
      int rc = finish_slot(s);
      if (rc) return rc;
    }
    const size_t r0 = chunks[ci].first;
    const size_t rows = chunks[ci].second;
    const size_t off = r0 * j.m, bytes = rows * j.m;
    const uint8_t* src = j.data + off;
    bool chunk_shared = false;
    if (!in_pinned) {
      if (j.auto_iv)
        chunk_shared = stage_and_check_iv(s.h_in, src, j.m, j.ivs + r0 * 16, rows, j.iv0);
      else
        par_memcpy(s.h_in, src, bytes);
      src = s.h_in;
    }
    GAES_CK(cudaMemcpyAsync(s.d_in, src, bytes, cudaMemcpyHostToDevice, s.stream));
    Job shared_view;
    const Job* jc = &j;
    if (chunk_shared) {
      shared_view = j;
      shared_view.mode = j.mode_shared;
      shared_view.rk = j.rk_shared;
      shared_view.ivs = nullptr;
      jc = &shared_view;
    }
    if (need_iv && !chunk_shared) {
      const uint8_t* ivsrc = j.ivs + r0 * 16;
      if (!iv_pinned) {
        par_memcpy(s.h_iv, ivsrc, rows * 16);
        ivsrc = s.h_iv;
      }
      GAES_CK(cudaMemcpyAsync(s.d_iv, ivsrc, rows * 16, cudaMemcpyHostToDevice, s.stream));
    }
    const bool iv_tex = jc->ivs && jc->mode == Mode::kChain && j.m == 16;
    int rc = launch_chunk(c, lane, *jc, s.stream, s.d_in, s.d_out, s.d_iv, r0, rows, compact,
                          tex_for(c, s.d_in, s.cap, s.stream),
                          iv_tex ? tex_for(c, s.d_iv, s.iv_cap, s.stream) : TexLease());
    if (rc) return rc;
    if (out_pinned) {
      GAES_CK(cudaMemcpyAsync(j.out + off, s.d_out, bytes, cudaMemcpyDeviceToHost, s.stream));
    } else {
      GAES_CK(cudaMemcpyAsync(s.h_out, s.d_out, bytes, cudaMemcpyDeviceToHost, s.stream));
      s.pending_dst = j.out + off;
      s.pending_bytes = bytes;
    }
    GAES_CK(cudaEventRecord(s.done, s.stream));
  }
  // drain in issue order
  for (size_t ci = (nchunks > (size_t)kSlots ? nchunks - kSlots : 0); ci < nchunks; ci++) {
    int rc = finish_slot(lane->slots[ci % kSlots]);
    if (rc && !rc_final) rc_final = rc;
  }
  drain.armed = rc_final != GAES_OK;
  return rc_final;
}

// parallel.py:37-50 applied to GPUs: contiguous, sizes differ by <= 1.
std::vector<std::pair<size_t, size_t>> plan_rows(size_t n, int workers) {
  std::vector<std::pair<size_t, size_t>> out;
  const size_t used = std::min<size_t>((size_t)workers, n);
  size_t start = 0;
  for (size_t i = 0; i < used; i++) {
    const size_t size = n / used + (i < n % used ? 1 : 0);
    out.emplace_back(start, start + size);
    start += size;
  }
  return out;
}

int gpus_in_use() {
  const int n = device_count();
  const int want = g_num_gpus.load();
  if (want <= 0 || want > n) return n;
  return want;
}

// Shard rows across devices; one host thread per device when > 1.
int run_sharded(const Job& j) {
  if (j.n == 0) return GAES_OK;
  const int ndev = device_count();
  if (ndev <= 0) return fail(GAES_ENODEV, "no CUDA device visible");
  const int g = gpus_in_use();
  auto chunks = plan_rows(j.n, g);
  std::vector<DevCtx*> ctxs(chunks.size());
  // One GPU: the caller's current device (one process per GPU under
  // torchrun).  Several: devices 0 .. g-1 (one process driving the box).
  for (size_t i = 0; i < chunks.size(); i++) {
    int rc = chunks.size() == 1 ? current_ctx(&ctxs[i]) : get_ctx((int)i, &ctxs[i]);
    if (rc) return rc;
  }
  auto shard_job = [&](size_t i) {
    Job s = j;
    s.data = j.data + chunks[i].first * j.m;
    s.out = j.out + chunks[i].first * j.m;
    if (j.ivs) s.ivs = j.ivs + chunks[i].first * 16;
    s.first = j.first + chunks[i].first;
    s.n = chunks[i].second - chunks[i].first;
    return s;
  };
  if (chunks.size() == 1) return run_job(ctxs[0], shard_job(0));
  std::vector<int> rcs(chunks.size(), GAES_OK);
  std::vector<std::string> errs(chunks.size());
  std::vector<std::thread> th;
  for (size_t i = 0; i < chunks.size(); i++)
    th.emplace_back([&, i] {
      rcs[i] = run_job(ctxs[i], shard_job(i));
      if (rcs[i]) errs[i] = t_err;
    });
  for (auto& t : th) t.join();
  for (size_t i = 0; i < chunks.size(); i++)
    if (rcs[i]) return fail(rcs[i], "gpu " + std::to_string(i) + ": " + errs[i]);
  return GAES_OK;
}

// IVSet.rows tiles a shared IV into N x 16 (aes_cbc.py:107-115); detect it so
// the IV folds into the key and the grid never crosses PCIe.
bool rows_share_iv(const uint8_t* ivs, size_t n) {
  std::atomic<bool> same{true};
  parallel_ranges(n, (size_t)1 << 13, [&](size_t lo, size_t hi) {
    uint64_t a0, a1;
    std::memcpy(&a0, ivs, 8);
    std::memcpy(&a1, ivs + 8, 8);
    for (size_t i = std::max<size_t>(lo, 1); i < hi; i++) {
      uint64_t b0, b1;
      std::memcpy(&b0, ivs + 16 * i, 8);
      std::memcpy(&b1, ivs + 16 * i + 8, 8);
      if ((a0 ^ b0) | (a1 ^ b1)) {
        same.store(false, std::memory_order_relaxed);
        return;
      }
      if ((i & 4095) == 0 && !same.load(std::memory_order_relaxed)) return;
    }
  });
  return same.load();
}

int check_grid(const void* data, const void* out, size_t n, size_t m) {
  if (n == 0) return GAES_OK;
  if (!data || !out) return fail(GAES_EINVAL, "null data/out pointer");
  if (m == 0 || m % 16 != 0) return fail(GAES_EINVAL, "padded width must be a positive multiple of 16");
  return GAES_OK;
}

// The 7-argument backend contract (both directions).
int cbc_host(bool dec, const uint8_t* data, const uint8_t* ivs, size_t n, size_t m, const uint8_t* rk,
             const uint8_t* box, const uint8_t* lut, const uint8_t* perm, uint8_t* out) {
  int rc = check_grid(data, out, n, m);
  if (rc || n == 0) return rc;
  if (!ivs || !rk || !box || !lut || !perm) return fail(GAES_EINVAL, "null table / IV pointer");
  const uint8_t* std_perm = dec ? kInvShiftRowsSrc : kShiftRowsSrc;
  const bool std_shift = std::memcmp(perm, std_perm, 16) == 0;
  const bool linear = !dec || lut_is_linear(lut);
  Job j;
  j.dec = dec;
  j.data = data;
  j.out = out;
  j.n = n;
  j.m = m;
  j.box = box;
  j.lut = lut;
  j.perm = perm;
  j.raw_rk = rk;
  {
    DevCtx* c0 = nullptr;
    int rc0 = current_ctx(&c0);
    if (rc0) return rc0;
    j.standard = is_standard(c0, dec, box, lut, perm);
  }
  if (!std_shift || !linear) {
    j.mode = Mode::kGeneric;
    j.ivs = ivs;
    return run_sharded(j);
  }
  const size_t bpr = m / 16;
  if (n >= ((size_t)1 << 14)) host_pool().warm();  // parallel IV checks + staging copies follow
  if (!is_pinned(data)) {
    // staged input: the shared-IV check rides along with each chunk's copy
    j.auto_iv = true;
    j.iv0 = ivs;
    j.ivs = ivs;
    if (dec || bpr == 1) {
      j.mode = Mode::kChain;
      j.rk = dec ? make_dec_keys(rk, ivs, false, lut) : make_enc_keys(rk, ivs, false);
    } else {
      j.mode = Mode::kEncRows;
      j.rk = make_enc_keys(rk, ivs, false);
    }
    j.mode_shared = bpr == 1 ? Mode::kFolded : j.mode;
    j.rk_shared = bpr != 1 ? j.rk : dec ? make_dec_keys(rk, ivs, true, lut) : make_enc_keys(rk, ivs, true);
    return run_sharded(j);
  }
  const bool shared = rows_share_iv(ivs, n);
  if (bpr == 1 && shared) {
    j.mode = Mode::kFolded;
    j.rk = dec ? make_dec_keys(rk, ivs, true, lut) : make_enc_keys(rk, ivs, true);
  } else if (dec || bpr == 1) {
    j.mode = Mode::kChain;
    j.ivs = shared ? nullptr : ivs;
    j.rk = dec ? make_dec_keys(rk, ivs, false, lut) : make_enc_keys(rk, ivs, false);
  } else {
    j.mode = Mode::kEncRows;
    j.ivs = shared ? nullptr : ivs;
    j.rk = make_enc_keys(rk, ivs, false);
  }
  return run_sharded(j);
}

int shared_iv_host(bool dec, const uint8_t* data, size_t n, size_t m, const uint8_t* iv, const uint8_t* rk,
                   uint8_t* out) {
  int rc = check_grid(data, out, n, m);
  if (rc || n == 0) return rc;
  if (!rk) return fail(GAES_EINVAL, "null round keys");
  static const uint8_t zero_iv[16] = {0};
  if (!iv) iv = zero_iv;
  Job j;
  j.dec = dec;
  j.data = data;
  j.out = out;
  j.n = n;
  j.m = m;
  j.standard = true;
  const size_t bpr = m / 16;
  if (bpr == 1) {
    j.mode = Mode::kFolded;
    j.rk = dec ? make_dec_keys(rk, iv, true, nullptr) : make_enc_keys(rk, iv, true);
  } else if (dec) {
    j.mode = Mode::kChain;
    j.rk = make_dec_keys(rk, iv, false, nullptr);
  } else {
    j.mode = Mode::kEncRows;
    j.rk = make_enc_keys(rk, iv, false);
  }
  return run_sharded(j);
}

}  // namespace

// ==========================================================================
// C ABI
extern "C" {

GAES_API int gaes_version(void) { return kVersion; }

GAES_API const char* gaes_last_error(void) { return t_err.c_str(); }

GAES_API int gaes_device_count(void) { return device_count(); }

GAES_API int gaes_set_num_gpus(int n) {
  g_num_gpus.store(n);
  return gpus_in_use();
}

GAES_API int gaes_get_num_gpus(void) { return gpus_in_use(); }

GAES_API uint64_t gaes_launch_count(void) { return g_launches.load(); }

GAES_API const char* gaes_last_kernel(void) {
  static thread_local std::string copy;
  std::lock_guard<std::mutex> lk(g_name_mu);
  copy = g_last_kernel;
  return copy.c_str();
}

GAES_API int gaes_set_variant(int variant) {
  if (variant < 0 || variant > 2)
    return fail(GAES_EINVAL, "unknown variant (0 = auto, 1 = T-table, 2 = bitsliced)");
  g_variant.store(variant);
  return variant;
}

GAES_API int gaes_probe_round_rate(int device, uint32_t iters, double* lookups_per_sec, double* ms) {
  DevCtx* c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  int prev = 0;
  GAES_CK(cudaGetDevice(&prev));
  DeviceGuard guard(prev);
  GAES_CK(cudaSetDevice(c->dev));
  struct Res {
    uint32_t* sink = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    ~Res() {
      if (sink) cudaFree(sink);
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } r;
  GAES_CK(cudaMalloc(&r.sink, 4));
  uint8_t rk[176] = {0};
  const RoundKeys k = make_enc_keys(rk, nullptr, false);
  GAES_CK(cudaEventCreate(&r.a));
  GAES_CK(cudaEventCreate(&r.b));
  GAES_CK(launch_round_probe(c->d_std_enc, k, 16, r.sink, c->sms, 0));  // warm-up
  GAES_CK(cudaEventRecord(r.a, 0));
  GAES_CK(launch_round_probe(c->d_std_enc, k, iters, r.sink, c->sms, 0));
  GAES_CK(cudaEventRecord(r.b, 0));
  GAES_CK(cudaEventSynchronize(r.b));
  note_kernel("k_round_probe");
  note_kernel("k_round_probe");
  float t = 0;
  GAES_CK(cudaEventElapsedTime(&t, r.a, r.b));
  const double lookups = (double)c->sms * kBlockThreads * (double)iters * 160.0;
  if (lookups_per_sec) *lookups_per_sec = lookups / (t / 1e3);
  if (ms) *ms = t;
  return GAES_OK;
}

GAES_API int gaes_probe_lds_peak(int device, uint32_t iters, double* lookups_per_sec, double* ms) {
  DevCtx* c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  int prev = 0;
  GAES_CK(cudaGetDevice(&prev));
  DeviceGuard guard(prev);
  GAES_CK(cudaSetDevice(c->dev));
  struct Res {
    uint32_t* sink = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    ~Res() {
      if (sink) cudaFree(sink);
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } r;
  GAES_CK(cudaMalloc(&r.sink, 4));
  GAES_CK(cudaEventCreate(&r.a));
  GAES_CK(cudaEventCreate(&r.b));
  GAES_CK(launch_lds_peak(64, r.sink, c->sms, 0));  // warm-up
  GAES_CK(cudaEventRecord(r.a, 0));
  GAES_CK(launch_lds_peak(iters, r.sink, c->sms, 0));
  GAES_CK(cudaEventRecord(r.b, 0));
  GAES_CK(cudaEventSynchronize(r.b));
  note_kernel("k_lds_peak");
  note_kernel("k_lds_peak");
  float t = 0;
  GAES_CK(cudaEventElapsedTime(&t, r.a, r.b));
  const double lookups = (double)c->sms * kBlockThreads * (double)iters * 16.0;
  if (lookups_per_sec) *lookups_per_sec = lookups / (t / 1e3);
  if (ms) *ms = t;
  return GAES_OK;
}

GAES_API int gaes_gf_tables(int device, uint8_t sbox[256], uint8_t inv_sbox[256], uint32_t te[1024],
                            uint32_t td[1024]) {
  DevCtx* c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  if (sbox) std::memcpy(sbox, c->std_sbox, 256);
  if (inv_sbox) std::memcpy(inv_sbox, c->std_inv, 256);
  if (te) std::memcpy(te, c->std_te, sizeof(c->std_te));
  if (td) std::memcpy(td, c->std_td, sizeof(c->std_td));
  return GAES_OK;
}

GAES_API int gaes_std_tables(int decrypt, uint8_t sbox[256], uint8_t mix_lut[4096], uint8_t shift_src[16]) {
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  if (sbox) std::memcpy(sbox, decrypt ? c->std_inv : c->std_sbox, 256);
  if (mix_lut) std::memcpy(mix_lut, decrypt ? c->std_mix_inv : c->std_mix_fwd, 4096);
  if (shift_src) std::memcpy(shift_src, decrypt ? kInvShiftRowsSrc : kShiftRowsSrc, 16);
  return GAES_OK;
}

GAES_API int gaes_tables_are_standard(const uint8_t sbox[256], const uint8_t mix_lut[4096],
                                      const uint8_t shift_src[16], int decrypt) {
  if (!sbox || !mix_lut || !shift_src) return fail(GAES_EINVAL, "null table pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  const uint8_t* box = decrypt ? c->std_inv : c->std_sbox;
  if (std::memcmp(box, sbox, 256) != 0) return 0;
  if (std::memcmp(shift_src, decrypt ? kInvShiftRowsSrc : kShiftRowsSrc, 16) != 0) return 0;
  for (int r = 0; r < 4; r++)
    for (int j = 0; j < 4; j++)
      for (int x = 0; x < 256; x++)
        if (mix_lut[(r * 4 + j) * 256 + x] != gf_mul(mix_coef(decrypt != 0, r, j), (uint8_t)x)) return 0;
  return 1;
}

GAES_API int gaes_cbc_encrypt(const uint8_t* data, const uint8_t* ivs, size_t n, size_t m,
                              const uint8_t round_keys[176], const uint8_t sbox[256], const uint8_t mix_lut[4096],
                              const uint8_t shift_src[16], uint8_t* out) {
  return cbc_host(false, data, ivs, n, m, round_keys, sbox, mix_lut, shift_src, out);
}

GAES_API int gaes_cbc_decrypt(const uint8_t* data, const uint8_t* ivs, size_t n, size_t m,
                              const uint8_t round_keys[176], const uint8_t inv_sbox[256],
                              const uint8_t inv_mix_lut[4096], const uint8_t inv_shift_src[16], uint8_t* out) {
  return cbc_host(true, data, ivs, n, m, round_keys, inv_sbox, inv_mix_lut, inv_shift_src, out);
}

GAES_API int gaes_cbc_encrypt_std(const uint8_t* data, const uint8_t* ivs, size_t n, size_t m,
                                  const uint8_t round_keys[176], uint8_t* out) {
  if (n == 0) return GAES_OK;
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  return cbc_host(false, data, ivs, n, m, round_keys, c->std_sbox, c->std_mix_fwd, kShiftRowsSrc, out);
}

GAES_API int gaes_cbc_decrypt_std(const uint8_t* data, const uint8_t* ivs, size_t n, size_t m,
                                  const uint8_t round_keys[176], uint8_t* out) {
  if (n == 0) return GAES_OK;
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  return cbc_host(true, data, ivs, n, m, round_keys, c->std_inv, c->std_mix_inv, kInvShiftRowsSrc, out);
}

static int many_key_host(bool dec, const uint8_t* data, size_t bpk, size_t k, const uint8_t* keys,
                         const uint8_t* ivs, uint8_t* out) {
  if (bpk == 0 || k == 0) return GAES_OK;
  if (!data || !out || !keys) return fail(GAES_EINVAL, "null pointer");
  Job j;
  j.dec = dec;
  j.mode = Mode::kManyKey;
  j.data = data;
  j.out = out;
  j.n = bpk * k;
  j.m = 16;
  j.bpk = bpk;
  j.n_keys = k;
  j.mk_keys = keys;
  j.mk_ivs = ivs;
  j.standard = true;
  return run_sharded(j);
}

GAES_API int gaes_many_key_encrypt(const uint8_t* data, size_t blocks_per_key, size_t k, const uint8_t* keys,
                                   const uint8_t* ivs, uint8_t* out) {
  return many_key_host(false, data, blocks_per_key, k, keys, ivs, out);
}

GAES_API int gaes_many_key_decrypt(const uint8_t* data, size_t blocks_per_key, size_t k, const uint8_t* keys,
                                   const uint8_t* ivs, uint8_t* out) {
  return many_key_host(true, data, blocks_per_key, k, keys, ivs, out);
}

GAES_API int gaes_encrypt_shared_iv(const uint8_t* data, size_t n, size_t m, const uint8_t iv[16],
                                    const uint8_t round_keys[176], uint8_t* out) {
  return shared_iv_host(false, data, n, m, iv, round_keys, out);
}

GAES_API int gaes_decrypt_shared_iv(const uint8_t* data, size_t n, size_t m, const uint8_t iv[16],
                                    const uint8_t round_keys[176], uint8_t* out) {
  return shared_iv_host(true, data, n, m, iv, round_keys, out);
}

GAES_API int gaes_encrypt_blocks_dev(const void* in, void* out, size_t n_blocks, const uint8_t round_keys[176],
                                     const uint8_t iv[16], void* stream) {
  if (n_blocks == 0) return GAES_OK;
  if (!in || !out || !round_keys) return fail(GAES_EINVAL, "null pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  const RoundKeys k = make_enc_keys(round_keys, iv, true);
  const void* src = nullptr;
  PrivateInput tmp;
  rc = private_input_if_aliased(in, out, n_blocks * 16, false, (cudaStream_t)stream, &src, &tmp);
  if (rc) return rc;
  return for_segments(c, n_blocks, [&](size_t off, size_t cnt) {
    const uint4* i = static_cast<const uint4*>(src) + off;
    GAES_CK(launch_enc_folded(c, i, static_cast<uint4*>(out) + off, cnt, c->d_std_enc, k, ilp_default(),
                              (cudaStream_t)stream, tex_for(c, i, cnt * 16, (cudaStream_t)stream)));
    return GAES_OK;
  });
}

GAES_API int gaes_decrypt_blocks_dev(const void* in, void* out, size_t n_blocks, const uint8_t round_keys[176],
                                     const uint8_t iv[16], void* stream) {
  if (n_blocks == 0) return GAES_OK;
  if (!in || !out || !round_keys) return fail(GAES_EINVAL, "null pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  const RoundKeys k = make_dec_keys(round_keys, iv, true, nullptr);
  const void* src = nullptr;
  PrivateInput tmp;
  rc = private_input_if_aliased(in, out, n_blocks * 16, false, (cudaStream_t)stream, &src, &tmp);
  if (rc) return rc;
  return for_segments(c, n_blocks, [&](size_t off, size_t cnt) {
    const uint4* i = static_cast<const uint4*>(src) + off;
    GAES_CK(launch_blocks(true, kIvFolded, ilp_default(), i, static_cast<uint4*>(out) + off, cnt, c->d_std_dec, k,
                          nullptr, 1, c->sms, (cudaStream_t)stream, tex_for(c, i, cnt * 16, (cudaStream_t)stream)));
    note_kernel("k_blocks_dec_folded");
    return GAES_OK;
  });
}

GAES_API int gaes_cbc_encrypt_dev(const void* in, void* out, size_t n, size_t m, const void* ivs_dev,
                                  const uint8_t iv[16], const uint8_t round_keys[176], void* stream) {
  int rc = check_grid(in, out, n, m);
  if (rc || n == 0) return rc;
  if (!round_keys) return fail(GAES_EINVAL, "null round keys");
  DevCtx* c = nullptr;
  rc = current_ctx(&c);
  if (rc) return rc;
  const uint64_t bpr = m / 16;
  if (bpr == 1 && !ivs_dev) return gaes_encrypt_blocks_dev(in, out, n, round_keys, iv, stream);
  const RoundKeys k = make_enc_keys(round_keys, iv, false);
  const void* src = nullptr;
  PrivateInput tmp;
  rc = private_input_if_aliased(in, out, n * m, false, (cudaStream_t)stream, &src, &tmp);
  if (rc) return rc;
  if (bpr == 1) {
    GAES_CK(launch_blocks(false, kIvChain, ilp_default(), src, out, n, c->d_std_enc, k, ivs_dev, 1, c->sms,
                          (cudaStream_t)stream, tex_for(c, src, n * 16, (cudaStream_t)stream),
                          tex_for(c, ivs_dev, n * 16, (cudaStream_t)stream)));
    note_kernel("k_blocks_enc_chain");
  } else {
    // segments of whole rows, each inside one texture
    const size_t seg_blocks = tex_segment_blocks(c);
    const size_t seg_rows = seg_blocks >= bpr ? seg_blocks / bpr : n;
    const uint8_t* i8 = static_cast<const uint8_t*>(src);
    uint8_t* o8 = static_cast<uint8_t*>(out);
    const uint8_t* v8 = static_cast<const uint8_t*>(ivs_dev);
    for (size_t r = 0; r < n; r += seg_rows) {
      const size_t cnt = std::min(seg_rows, n - r);
      GAES_CK(launch_cbc_enc_rows(i8 + r * m, o8 + r * m, cnt, bpr, c->d_std_enc, k, v8 ? v8 + r * 16 : nullptr,
                                  c->sms, (cudaStream_t)stream, tex_for(c, i8 + r * m, cnt * m, (cudaStream_t)stream)));
    }
    note_kernel("k_cbc_enc_rows");
  }
  return GAES_OK;
}

GAES_API int gaes_cbc_decrypt_dev(const void* in, void* out, size_t n, size_t m, const void* ivs_dev,
                                  const uint8_t iv[16], const uint8_t round_keys[176], void* stream) {
  int rc = check_grid(in, out, n, m);
  if (rc || n == 0) return rc;
  if (!round_keys) return fail(GAES_EINVAL, "null round keys");
  DevCtx* c = nullptr;
  rc = current_ctx(&c);
  if (rc) return rc;
  const uint64_t bpr = m / 16;
  if (bpr == 1 && !ivs_dev) return gaes_decrypt_blocks_dev(in, out, n, round_keys, iv, stream);
  const RoundKeys k = make_dec_keys(round_keys, iv, false, nullptr);
  const void* src = nullptr;
  PrivateInput tmp;
  rc = private_input_if_aliased(in, out, n * m, bpr > 1, (cudaStream_t)stream, &src, &tmp);
  if (rc) return rc;
  GAES_CK(launch_blocks(true, kIvChain, ilp_default(), src, out, n * bpr, c->d_std_dec, k, ivs_dev, bpr, c->sms,
                        (cudaStream_t)stream, tex_for(c, src, n * bpr * 16, (cudaStream_t)stream),
                        bpr == 1 && ivs_dev ? tex_for(c, ivs_dev, n * 16, (cudaStream_t)stream) : TexLease()));
  note_kernel("k_blocks_dec_chain");
  return GAES_OK;
}

GAES_API int gaes_expand_keys_dev(const void* keys, size_t k, void* rk_enc, void* rk_dec, void* stream) {
  if (k == 0) return GAES_OK;
  if (!keys || !rk_enc) return fail(GAES_EINVAL, "null pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  GAES_CK(launch_expand_keys((const uint8_t*)keys, k, c->d_std_enc, (uint8_t*)rk_enc, (uint8_t*)rk_dec,
                             (cudaStream_t)stream));
  note_kernel("k_expand_keys");
  return GAES_OK;
}

GAES_API int gaes_many_key_encrypt_dev(const void* in, void* out, size_t blocks_per_key, size_t k,
                                       const void* rk_enc, const void* ivs_dev, void* stream) {
  if (k == 0 || blocks_per_key == 0) return GAES_OK;
  if (!in || !out || !rk_enc) return fail(GAES_EINVAL, "null pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  const void* src = nullptr;
  PrivateInput tmp;
  rc = private_input_if_aliased(in, out, blocks_per_key * k * 16, false, (cudaStream_t)stream, &src, &tmp);
  if (rc) return rc;
  return for_segments(c, blocks_per_key * k, [&](size_t off, size_t cnt) {
    const uint4* i = static_cast<const uint4*>(src) + off;
    GAES_CK(launch_many_key(false, i, static_cast<uint4*>(out) + off, cnt, off, blocks_per_key, c->d_std_enc, rk_enc,
                            ivs_dev, c->sms, (cudaStream_t)stream, tex_for(c, i, cnt * 16, (cudaStream_t)stream)));
    note_kernel("k_many_key_enc");
    return GAES_OK;
  });
}

GAES_API int gaes_many_key_decrypt_dev(const void* in, void* out, size_t blocks_per_key, size_t k,
                                       const void* rk_dec, const void* ivs_dev, void* stream) {
  if (k == 0 || blocks_per_key == 0) return GAES_OK;
  if (!in || !out || !rk_dec) return fail(GAES_EINVAL, "null pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  const void* src = nullptr;
  PrivateInput tmp;
  rc = private_input_if_aliased(in, out, blocks_per_key * k * 16, false, (cudaStream_t)stream, &src, &tmp);
  if (rc) return rc;
  return for_segments(c, blocks_per_key * k, [&](size_t off, size_t cnt) {
    const uint4* i = static_cast<const uint4*>(src) + off;
    GAES_CK(launch_many_key(true, i, static_cast<uint4*>(out) + off, cnt, off, blocks_per_key, c->d_std_dec, rk_dec,
                            ivs_dev, c->sms, (cudaStream_t)stream, tex_for(c, i, cnt * 16, (cudaStream_t)stream)));
    note_kernel("k_many_key_dec");
    return GAES_OK;
  });
}

}  // extern "C"
