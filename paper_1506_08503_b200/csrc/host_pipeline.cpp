// host_pipeline.cpp -- see host_pipeline.h.
//
// Reference boundary replaced: pkg/src/gaes/backend.py:56-61 forwards
// cbc_encrypt / cbc_decrypt (7 arguments) to the active kernel module;
// _kernel.pyx:12-101 is the kernel.  parallel.py:37-50 (plan) and :66-75
// (thread fan-out over contiguous row ranges) become the GPU shard plan.
#include "host_pipeline.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <thread>

#include "host_pool.h"
#include "round_keys.h"

namespace gaes {
namespace rt {

using namespace gaes::host;

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
  static size_t b = (size_t)std::max(0, tune_int("ZEROCOPY_MB", 64)) << 20;
  return b;
}

// Pageable jobs up to this size run as one kernel on the pinned staging
// buffers (see run_job).
size_t small_zero_copy_bytes() {
  static size_t b = (size_t)std::max(0, tune_int("SMALL_ZEROCOPY_KB", 1024)) << 10;
  return b;
}

size_t chunk_bytes() {
  static size_t b = (size_t)std::max(1, tune_int("CHUNK_MB", 32)) << 20;
  return b;
}

// Device address of pinned staging memory (nullptr if it has none).
static uint8_t* dev_view(uint8_t* h) {
  void* d = nullptr;
  if (!h || cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return static_cast<uint8_t*>(d);
}

int ensure_slot(Slot& s, size_t bytes, size_t iv_bytes, bool staged_in, bool staged_out) {
  if (s.cap < bytes) {
    if (s.d_in) cudaFree(s.d_in);
    if (s.d_out) cudaFree(s.d_out);
    if (s.h_in) cudaFreeHost(s.h_in);
    if (s.h_out) cudaFreeHost(s.h_out);
    s.d_in = s.d_out = s.h_in = s.h_out = s.dv_in = s.dv_out = nullptr;
    s.cap = 0;
    GAES_CK(cudaMalloc(&s.d_in, bytes));
    GAES_CK(cudaMalloc(&s.d_out, bytes));
    s.cap = bytes;
  }
  if (staged_in && !s.h_in) {
    GAES_CK(cudaMallocHost(&s.h_in, s.cap));
    s.dv_in = dev_view(s.h_in);
  }
  if (staged_out && !s.h_out) {
    GAES_CK(cudaMallocHost(&s.h_out, s.cap));
    s.dv_out = dev_view(s.h_out);
  }
  if (iv_bytes && s.iv_cap < iv_bytes) {
    if (s.d_iv) cudaFree(s.d_iv);
    if (s.h_iv) cudaFreeHost(s.h_iv);
    s.d_iv = s.h_iv = s.dv_iv = nullptr;
    s.iv_cap = 0;
    GAES_CK(cudaMalloc(&s.d_iv, iv_bytes));
    GAES_CK(cudaMallocHost(&s.h_iv, iv_bytes));
    s.dv_iv = dev_view(s.h_iv);
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
  const cudaTextureObject_t tsb = sbox_tex(c, compact);
  switch (j.mode) {
    case Mode::kFolded:
      if (j.dec) {
        GAES_CK(launch_folded(c, true, in, out, nblk, compact, j.rk, stream, tin, /*host_job=*/true));
      } else if (j.standard || g_variant.load() < 2) {
        GAES_CK(launch_enc_folded(c, in, out, nblk, compact, j.rk, ilp_default(), stream, tin,
                                  /*host_job=*/true));
      } else {  // bitsliced kernel has the standard S-box built in; caller tables -> T-table
        GAES_CK(launch_blocks(false, kIvFolded, ilp_default(), in, out, nblk, compact, j.rk, nullptr, 1,
                              c->sms, stream, 0, 0, tsb));
        note_kernel("k_blocks_enc_folded");
      }
      break;
    case Mode::kChain:
      GAES_CK(launch_blocks(j.dec, kIvChain, ilp_default(), in, out, nblk, compact, j.rk,
                            j.ivs ? ivs : nullptr, bpr, c->sms, stream, tin, j.ivs ? tiv : 0, tsb));
      note_kernel(j.dec ? "k_blocks_dec_chain" : "k_blocks_enc_chain");
      break;
    case Mode::kEncRows:
      GAES_CK(launch_cbc_enc_rows(in, out, rows, bpr, compact, j.rk, j.ivs ? ivs : nullptr, c->sms,
                                  stream, tin, tsb));
      note_kernel(last_rows_kernel());
      break;
    case Mode::kManyKey: {
      const size_t kb = j.n_keys * 16, rkb = j.n_keys * 176;
      GAES_CK(launch_many_key(j.dec, in, out, nblk, j.first + r0, j.bpk, compact,
                              lane->d_mk + kb + (j.dec ? rkb : 0), j.mk_ivs ? lane->d_mk + kb + 2 * rkb : nullptr, c->sms,
                              stream, tin, tsb));
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
  parallel_ranges(rows, std::max<size_t>(1, copy_grain() / m), [&](size_t lo, size_t hi) {
    stage_copy(dst + lo * m, src + lo * m, (hi - lo) * m);
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

// Locks the first free lane of c (lane 0 for a lone caller, so its staging
// buffers -- allocated on first use, cudaMallocHost costs milliseconds -- are
// reused call after call; lanes 1.. only for concurrent callers); if all
// are busy, waits on one chosen by thread.
std::unique_lock<std::mutex> lock_lane(DevCtx* c, Lane** out) {
  static const int lanes = std::max(1, std::min(kLanes, tune_int("LANES", kLanes)));
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

// Optional pipeline timeline (GAES_TRACE=<csv path>, measurement only): per
// staged chunk, device events before the H2D and after the H2D, the kernel
// and the D2H, appended to the file as ms relative to the first chunk.
struct Trace {
  const char* path = nullptr;
  std::vector<cudaEvent_t> ev;  // 4 per chunk
  std::vector<size_t> bytes;
  std::vector<double> host;  // 3 per chunk: slot wait begins, slot free, chunk issued (ms)
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit Trace(size_t nchunks) {
    path = std::getenv("GAES_TRACE");
    if (!path || !*path) {
      path = nullptr;
      return;
    }
    ev.resize(4 * nchunks);
    for (auto& e : ev) cudaEventCreate(&e);
    bytes.resize(nchunks);
    host.resize(3 * nchunks);
  }
  void host_mark(size_t ci, int k) {
    if (path)
      host[3 * ci + k] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  void mark(size_t ci, int k, cudaStream_t s) {
    if (path) cudaEventRecord(ev[4 * ci + k], s);
  }
  ~Trace() {
    if (!path) return;
    cudaDeviceSynchronize();
    if (FILE* f = std::fopen(path, "a")) {
      std::fprintf(f, "chunk,bytes,h2d_start,h2d_end,kernel_end,d2h_end,host_wait,host_free,host_issued\n");
      for (size_t ci = 0; ci < bytes.size(); ci++) {
        float t[4] = {0, 0, 0, 0};
        for (int k = 0; k < 4; k++) cudaEventElapsedTime(&t[k], ev[0], ev[4 * ci + k]);
        std::fprintf(f, "%zu,%zu,%.4f,%.4f,%.4f,%.4f,%.4f,%.4f,%.4f\n", ci, bytes[ci], t[0], t[1], t[2], t[3],
                     host[3 * ci] - host[0], host[3 * ci + 1] - host[0], host[3 * ci + 2] - host[0]);
      }
      std::fclose(f);
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
};

// Runs rows [0, j.n) of `j` on device context c (one shard).
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
    // byte-level tables for k_generic_cbc, on the lane's own stream and
    // complete before any slot stream launches (the slot streams are
    // non-blocking: a legacy-stream cudaMemcpy from pageable memory would
    // not order them)
    uint8_t* sc = lane->d_scratch;
    cudaStream_t s0 = lane->slots[0].stream;
    GAES_CK(cudaMemcpyAsync(sc, j.box, 256, cudaMemcpyHostToDevice, s0));
    GAES_CK(cudaMemcpyAsync(sc + 256, j.lut, 4096, cudaMemcpyHostToDevice, s0));
    GAES_CK(cudaMemcpyAsync(sc + 256 + 4096, j.perm, 16, cudaMemcpyHostToDevice, s0));
    GAES_CK(cudaMemcpyAsync(sc + 256 + 4096 + 16, j.raw_rk, 176, cudaMemcpyHostToDevice, s0));
    GAES_CK(cudaStreamSynchronize(s0));
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
    g_keys_expanded.fetch_add((int64_t)j.n_keys, std::memory_order_relaxed);
    GAES_CK(cudaStreamSynchronize(s0));
  }

  const bool in_pinned = is_pinned(j.data);
  const bool out_pinned = is_pinned(j.out);
  if (!(in_pinned && out_pinned) && j.n * j.m >= ((size_t)256 << 10)) current_pool().warm();
  const bool need_iv = j.ivs != nullptr;
  const bool iv_pinned = need_iv && is_pinned(j.ivs);

  // Pinned caller buffers and a job small enough that the staged pipeline's
  // ramp dominates: one zero-copy launch -- the kernel reads and writes the
  // caller's host memory over PCIe itself, no staging copies
  // (scripts/exp/zerocopy_probe.py: 21 vs 15 GB/s at 1 MiB, 34 vs 32 at
  // 16 MiB, 38.6 vs 37.9 at 64 MiB; the staged pipeline leads from 256 MiB).
  // Not for byte-level generic tables (byte loads over PCIe), overlapping
  // in/out (the kernels assume distinct buffers) or buffers that are not
  // 16-byte aligned (the kernels move whole 16-byte blocks; a misaligned
  // vector access would fault the context) -- those take the staged
  // pipeline, whose DMA copies accept any alignment.
  const size_t total = j.n * j.m;
  const uintptr_t ia = reinterpret_cast<uintptr_t>(j.data), oa = reinterpret_cast<uintptr_t>(j.out);
  const bool aligned = aligned16(j.data) && aligned16(j.out) && (!need_iv || aligned16(j.ivs));
  if (in_pinned && out_pinned && (!need_iv || iv_pinned) && aligned && j.mode != Mode::kGeneric &&
      total <= zero_copy_bytes() && !(ia < oa + total && oa < ia + total)) {
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
  // Small jobs on pageable caller buffers: stage into the lane's pinned
  // buffer and let ONE kernel read it and write the pinned output staging
  // over PCIe, instead of an H2D copy, a kernel and a D2H copy -- below
  // ~1 MiB the two DMA round trips' fixed latency is most of the call.
  // (Byte-level generic tables excluded, as for caller zero-copy.)
  if (!in_pinned && !out_pinned && j.mode != Mode::kGeneric && total <= small_zero_copy_bytes()) {
    Slot& s = lane->slots[0];
    int rc = ensure_slot(s, std::max(total, (size_t)1 << 20), need_iv ? std::max(j.n * 16, (size_t)1 << 16) : 0,
                         true, true);
    if (rc) return rc;
    if (s.dv_in && s.dv_out && (!need_iv || s.dv_iv)) {
      bool shared = false;
      if (j.auto_iv)
        shared = stage_and_check_iv(s.h_in, j.data, j.m, j.ivs, j.n, j.iv0);
      else
        par_memcpy(s.h_in, j.data, total);
      Job view;
      const Job* jc = &j;
      if (shared) {
        view = j;
        view.mode = j.mode_shared;
        view.rk = j.rk_shared;
        view.ivs = nullptr;
        jc = &view;
      }
      if (jc->ivs) std::memcpy(s.h_iv, j.ivs, j.n * 16);
      rc = launch_chunk(c, lane, *jc, s.stream, s.dv_in, s.dv_out, s.dv_iv, 0, j.n, compact, 0);
      if (rc) return rc;
      GAES_CK(cudaStreamSynchronize(s.stream));
      par_memcpy(j.out, s.h_out, total);
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
  static const size_t pageable_chunk = (size_t)std::max(1, tune_int("PAGEABLE_CHUNK_MB", 16)) << 20;
  const size_t base_bytes = (in_pinned && out_pinned) ? chunk_bytes() : std::min<size_t>(chunk_bytes(), pageable_chunk);
  const size_t base_rows = std::max<size_t>(1, base_bytes / j.m);
  // (splitting small staged jobs further was measured slower: per-chunk
  // fixed costs outweigh the copy/transfer overlap below ~2 MiB)
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
  Trace trace(nchunks);
  for (size_t ci = 0; ci < nchunks; ci++) {
    Slot& s = lane->slots[ci % kSlots];
    trace.host_mark(ci, 0);
    if (ci >= (size_t)kSlots) {
      int rc = finish_slot(s);
      if (rc) return rc;
    }
    trace.host_mark(ci, 1);
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
    if (trace.path) trace.bytes[ci] = bytes;
    trace.mark(ci, 0, s.stream);
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
    trace.mark(ci, 1, s.stream);
    const bool iv_tex = jc->ivs && jc->mode == Mode::kChain && j.m == 16;
    int rc = launch_chunk(c, lane, *jc, s.stream, s.d_in, s.d_out, s.d_iv, r0, rows, compact,
                          tex_for(c, s.d_in, s.cap, s.stream),
                          iv_tex ? tex_for(c, s.d_iv, s.iv_cap, s.stream) : TexLease());
    if (rc) return rc;
    trace.mark(ci, 2, s.stream);
    if (out_pinned) {
      GAES_CK(cudaMemcpyAsync(j.out + off, s.d_out, bytes, cudaMemcpyDeviceToHost, s.stream));
    } else {
      GAES_CK(cudaMemcpyAsync(s.h_out, s.d_out, bytes, cudaMemcpyDeviceToHost, s.stream));
      s.pending_dst = j.out + off;
      s.pending_bytes = bytes;
    }
    trace.mark(ci, 3, s.stream);
    GAES_CK(cudaEventRecord(s.done, s.stream));
    trace.host_mark(ci, 2);
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

// Shard rows across devices.  One device: the caller's thread and the
// process pool.  Several: shard 0 on the caller's thread, the others on
// their device's persistent runner threads; each shard stages through its
// device's own NUMA-local copy pool, so the shards' host copies run in
// parallel instead of queueing for one pool.  A many-key shard uploads and
// expands only the keys its rows use.
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
    if (j.mode == Mode::kManyKey) {  // this shard's keys only (rows are blocks here)
      const size_t k_lo = s.first / j.bpk, k_hi = (s.first + s.n + j.bpk - 1) / j.bpk;
      s.mk_keys = j.mk_keys + k_lo * 16;
      if (j.mk_ivs) s.mk_ivs = j.mk_ivs + k_lo * 16;
      s.n_keys = k_hi - k_lo;
      s.first -= k_lo * j.bpk;
    }
    return s;
  };
  if (chunks.size() == 1) return run_job(ctxs[0], shard_job(0));
  std::vector<int> rcs(chunks.size(), GAES_OK);
  std::vector<std::string> errs(chunks.size());
  std::mutex mu;
  std::condition_variable cv;
  size_t left = chunks.size() - 1;
  auto run_one = [&](size_t i) {
    host::PoolScope scope(device_pool(ctxs[i]));
    rcs[i] = run_job(ctxs[i], shard_job(i));
    if (rcs[i]) errs[i] = t_err;
  };
  for (size_t i = 1; i < chunks.size(); i++)
    ctxs[i]->runner.post([&, i] {
      run_one(i);
      std::lock_guard<std::mutex> lk(mu);
      if (--left == 0) cv.notify_all();
    });
  run_one(0);
  {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return left == 0; });
  }
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

int many_key_host(bool dec, const uint8_t* data, size_t bpk, size_t k, const uint8_t* keys,
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

}  // namespace rt
}  // namespace gaes
