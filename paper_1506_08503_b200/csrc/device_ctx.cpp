// device_ctx.cpp -- see device_ctx.h.
#include "device_ctx.h"

#include <cuda.h>
#include <sched.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "aes_bitslice.cuh"
#include "gf.cuh"

namespace gaes {
namespace rt {

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

// A u8 linear texture over 256 bytes (0 if unavailable).
cudaTextureObject_t make_byte_texture(const uint8_t* p) {
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = const_cast<uint8_t*>(p);
  rd.res.linear.desc = cudaCreateChannelDesc<unsigned char>();
  rd.res.linear.sizeInBytes = 256;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t t = 0;
  if (cudaCreateTextureObject(&t, &rd, &td, nullptr) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return t;
}

cudaTextureObject_t sbox_tex(const DevCtx* c, const uint32_t* compact) {
  if (compact == c->d_std_enc) return c->tex_s_enc;
  if (compact == c->d_std_dec) return c->tex_s_dec;
  return 0;
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
  // S-box textures for round 10 (standard tables); optional
  GAES_CK(cudaMalloc(&c->d_sbox, 256));
  GAES_CK(cudaMalloc(&c->d_inv, 256));
  GAES_CK(cudaMemcpy(c->d_sbox, d_box, 256, cudaMemcpyDeviceToDevice));
  GAES_CK(cudaMemcpy(c->d_inv, d_box + 256, 256, cudaMemcpyDeviceToDevice));
  if (tune_int("TEXS", 1) != 0) {
    c->tex_s_enc = make_byte_texture(c->d_sbox);
    c->tex_s_dec = make_byte_texture(c->d_inv);
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


// Identity of the allocation `p` lies in (CU_POINTER_ATTRIBUTE_BUFFER_ID:
// unique per allocation for the life of the process, so a buffer freed and
// re-allocated at the same address gets a new id), through the runtime's
// driver entry point (no libcuda link dependency).  0 if unavailable.
unsigned long long buffer_id(const void* p) {
  using GetAttrFn = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
  static GetAttrFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (GetAttrFn) nullptr;
    }
    return reinterpret_cast<GetAttrFn>(f);
  }();
  unsigned long long id = 0;
  if (!fn || fn(&id, CU_POINTER_ATTRIBUTE_BUFFER_ID, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return 0;
  return id;
}

// A linear uint4 texture over [ptr, ptr + bytes) for the texture-path input
// loads, cached per device by (pointer, allocation id): callers and the
// staging slots reuse buffers, and a buffer freed and re-allocated at the
// same address is a different allocation, whose old texture object must not
// be reused (it was created over memory that no longer exists).  Empty
// (handle 0) when disabled (GAES_TUNE=TEXIN=0), misaligned, too large or
// unavailable -- the kernels then use LDG.  Must be called with c->dev
// current and the lease used for one launch on `stream`.  At 64 entries the
// least recently used idle entry is evicted after waiting for the launches
// that read it (its per-stream events); entries lent out right now are never
// evicted.
TexLease tex_for(DevCtx* c, const void* ptr, size_t bytes, cudaStream_t stream) {
  static const bool enabled = tune_int("TEXIN", 1) != 0;
  if (!enabled || !ptr || bytes < 16) return {};
  // A launch captured into a CUDA graph may be replayed long after this
  // cache evicted (destroyed) the texture object; captured launches use LDG.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cap) != cudaSuccess) {
    cudaGetLastError();
    return {};
  }
  if (cap != cudaStreamCaptureStatusNone) return {};
  const unsigned long long id = buffer_id(ptr);
  std::lock_guard<std::mutex> lk(c->tex_mu);
  query_tex_limits(c);
  if (c->tex_align < 0 || reinterpret_cast<uintptr_t>(ptr) % (uintptr_t)c->tex_align != 0) return {};
  if (bytes / 16 > c->tex_max_texels || bytes / 16 > 0x7FFFFFFFull) return {};
  auto evict = [&](size_t i) {  // users == 0 (checked by the caller, under tex_mu)
    if (!c->tex_cache[i]->drain()) return false;
    c->tex_cache.erase(c->tex_cache.begin() + i);
    return true;
  };
  for (size_t i = 0; i < c->tex_cache.size(); i++) {
    auto& t = c->tex_cache[i];
    if (t->ptr != ptr) continue;
    if (t->buffer_id == id && t->bytes >= bytes) {
      t->users.fetch_add(1, std::memory_order_acquire);
      t->stamp = ++c->tex_clock;
      return TexLease(t.get(), stream);
    }
    // same address, another allocation (or a shorter view): drop the stale entry
    if (t->buffer_id != id && t->users.load(std::memory_order_acquire) == 0) {
      if (!evict(i)) return {};
      break;
    }
  }
  if (c->tex_cache.size() >= 64) {
    // users only grows under tex_mu, so an idle entry seen here stays idle
    size_t victim = c->tex_cache.size();
    for (size_t i = 0; i < c->tex_cache.size(); i++)
      if (c->tex_cache[i]->users.load(std::memory_order_acquire) == 0 &&
          (victim == c->tex_cache.size() || c->tex_cache[i]->stamp < c->tex_cache[victim]->stamp))
        victim = i;
    if (victim == c->tex_cache.size() || !evict(victim)) return {};
  }
  auto e = std::make_unique<DevCtx::Tex>();
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = const_cast<void*>(ptr);
  rd.res.linear.desc = cudaCreateChannelDesc<uint4>();
  rd.res.linear.sizeInBytes = bytes / 16 * 16;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  if (cudaCreateTextureObject(&e->tex, &rd, &td, nullptr) != cudaSuccess) {
    cudaGetLastError();
    e->tex = 0;
    return {};
  }
  e->ptr = ptr;
  e->bytes = bytes;
  e->buffer_id = id;
  e->stamp = ++c->tex_clock;
  e->users.store(1, std::memory_order_relaxed);
  c->tex_cache.push_back(std::move(e));
  c->tex_created++;
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

int private_input_if_aliased(const void* in, const void* out, size_t bytes, bool identical_is_unsafe,
                             cudaStream_t stream, const void** src, PrivateInput* tmp) {
  *src = in;
  const uintptr_t a = reinterpret_cast<uintptr_t>(in), b = reinterpret_cast<uintptr_t>(out);
  const bool overlap = a < b + bytes && b < a + bytes;
  // a misaligned input is copied too: the kernels load whole 16-byte blocks
  if (aligned16(in) && (!overlap || (a == b && !identical_is_unsafe && aligned16(out)))) return GAES_OK;
  GAES_CK(cudaMallocAsync(&tmp->ptr, bytes, stream));
  tmp->stream = stream;
  GAES_CK(cudaMemcpyAsync(tmp->ptr, in, bytes, cudaMemcpyDeviceToDevice, stream));
  *src = tmp->ptr;
  return GAES_OK;
}



int aligned_input(const void* p, size_t bytes, cudaStream_t stream, const void** src, PrivateInput* tmp) {
  *src = p;
  if (!p || aligned16(p) || bytes == 0) return GAES_OK;
  GAES_CK(cudaMallocAsync(&tmp->ptr, bytes, stream));
  tmp->stream = stream;
  GAES_CK(cudaMemcpyAsync(tmp->ptr, p, bytes, cudaMemcpyDeviceToDevice, stream));
  *src = tmp->ptr;
  return GAES_OK;
}

int aligned_output(void* out, size_t bytes, cudaStream_t stream, void** dst, PrivateOutput* tmp) {
  *dst = out;
  if (!out || aligned16(out) || bytes == 0) return GAES_OK;
  GAES_CK(cudaMallocAsync(&tmp->ptr, bytes, stream));
  tmp->stream = stream;
  tmp->dst = out;
  tmp->bytes = bytes;
  *dst = tmp->ptr;
  return GAES_OK;
}

std::vector<int> device_local_cpus(int dev) {
  std::vector<int> cpus;
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) {
    cudaGetLastError();
    return cpus;
  }
  std::string id(bus);
  for (auto& ch : id) ch = (char)std::tolower((unsigned char)ch);
  FILE* f = std::fopen(("/sys/bus/pci/devices/" + id + "/local_cpulist").c_str(), "r");
  if (!f) return cpus;
  char buf[4096] = {0};
  const size_t got = std::fread(buf, 1, sizeof(buf) - 1, f);
  std::fclose(f);
  buf[got] = 0;
  cpu_set_t allowed;
  const bool have_mask = sched_getaffinity(0, sizeof(allowed), &allowed) == 0;
  for (char* p = buf; *p && *p != '\n';) {  // "0-31,64-95"
    char* end = nullptr;
    const long lo = std::strtol(p, &end, 10);
    if (end == p) break;
    long hi = lo;
    p = end;
    if (*p == '-') {
      hi = std::strtol(p + 1, &end, 10);
      p = end;
    }
    for (long c = lo; c <= hi && c < CPU_SETSIZE; c++)
      if (!have_mask || CPU_ISSET((int)c, &allowed)) cpus.push_back((int)c);
    if (*p == ',') p++;
  }
  return cpus;
}

host::HostPool* device_pool(DevCtx* c) {
  std::call_once(c->pool_once, [c] {
    // this device's share of the process's copy threads (logical devices
    // on one node split its CPUs), pinned to the CPUs local to the GPU
    const int n = std::max(1, host::host_threads() / std::max(1, device_count()));
    c->pool = new host::HostPool(n - 1, device_local_cpus(c->dev));  // leaked with the context
  });
  return c->pool;
}

int ilp_default() {
  // ILP 1 measured ~1% faster than 2 at configs 2 and 3 (finer tail, 40 regs)
  static int ilp = std::max(1, std::min(2, tune_int("ILP", 1)));
  return ilp;
}

cudaError_t launch_enc_folded(DevCtx* c, const void* in, void* out, uint64_t n, const uint32_t* compact,
                              const RoundKeys& k, int ilp, cudaStream_t s, cudaTextureObject_t tin, bool host_job) {
  if (g_variant.load() == 2) {
    static thread_local BitsliceKeys bk;
    bs_make_keys(k.w, bk);
    note_kernel("k_bs_blocks");
    return launch_bs_blocks(in, out, n, bk, c->sms, s);
  }
  return launch_folded(c, false, in, out, n, compact, k, s, tin, host_job);
}

cudaError_t launch_folded(DevCtx* c, bool dec, const void* in, void* out, uint64_t n, const uint32_t* compact,
                          const RoundKeys& k, cudaStream_t s, cudaTextureObject_t tin, bool host_job) {
  const cudaTextureObject_t tsb = sbox_tex(c, compact);  // nonzero only for the GF layer's tables
  if (tsb && n <= small_blocks_max(c->sms) && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
    note_kernel(dec ? "k_blocks_small_dec" : "k_blocks_small_enc");
    return launch_blocks_small(dec, in, out, n, dec ? c->std_td : c->std_te, k, c->sms, s, tsb, host_job);
  }
  note_kernel(dec ? "k_blocks_dec_folded" : (tsb ? "k_blocks_enc_folded+texsbox" : "k_blocks_enc_folded"));
  return launch_blocks(dec, kIvFolded, ilp_default(), in, out, n, compact, k, nullptr, 1, c->sms, s, tin, 0, tsb);
}

}  // namespace rt
}  // namespace gaes
