// abi.cpp -- the C ABI of libgaes_b200.so (include/gaes_b200.h): argument
// checks, device-resident entry points and measurement support; host-buffer
// entries forward to host_pipeline.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gaes_b200.h"
#include "device_ctx.h"
#include "gf.cuh"
#include "host_pipeline.h"
#include "kernels.h"
#include "round_keys.h"

using namespace gaes;
using namespace gaes::host;
using namespace gaes::rt;

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

GAES_API int gaes_debug_counters(int64_t* out, int n) {
  if (!out || n < 0) return fail(GAES_EINVAL, "null counter buffer");
  host::PoolStats& st = host::pool_stats();
  int64_t tex_created = 0, tex_cached = 0, runners = 0;
  DevCtx* c = nullptr;
  if (device_count() > 0 && current_ctx(&c) == GAES_OK) {
    std::lock_guard<std::mutex> lk(c->tex_mu);
    tex_created = (int64_t)c->tex_created;
    tex_cached = (int64_t)c->tex_cache.size();
  }
  for (int d = 0; d < std::max(0, device_count()); d++) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (g_ctx[d]) runners += g_ctx[d]->runner.threads();
  }
  const int64_t v[] = {st.pools.load(), st.regions.load(), st.max_active.load(), st.busy_fallbacks.load(),
                       tex_created, tex_cached, g_keys_expanded.load(), runners};
  const int k = std::min<int>(n, (int)(sizeof(v) / sizeof(v[0])));
  for (int i = 0; i < k; i++) out[i] = v[i];
  return k;
}

GAES_API int64_t gaes_host_pool_selftest(int regions, int parts, int workers) {
  if (regions < 0 || parts <= 0 || workers < 0) return fail(GAES_EINVAL, "bad self-test arguments");
  // A private pool hammered with back-to-back regions of `parts` parts; every
  // part of every region must run exactly once (a part claimed twice, or
  // never, is an error).  Returns the number of violations.
  host::HostPool pool(workers);
  std::vector<std::atomic<int>> hits((size_t)parts);
  int64_t bad = 0;
  for (int r = 0; r < regions; r++) {
    for (auto& h : hits) h.store(0, std::memory_order_relaxed);
    const std::function<void(size_t)> fn = [&](size_t i) {
      hits[i].fetch_add(1, std::memory_order_relaxed);
      if ((i & 7) == 0) std::this_thread::yield();  // widen the windows a stale claimant could use
    };
    while (!pool.try_run((size_t)parts, fn)) {
    }
    for (auto& h : hits) bad += h.load() != 1;
  }
  return bad;
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
  GAES_CK(launch_round_probe(c->d_std_enc, k, 16, r.sink, c->sms, 0, c->tex_s_enc));  // warm-up
  GAES_CK(cudaEventRecord(r.a, 0));
  GAES_CK(launch_round_probe(c->d_std_enc, k, iters, r.sink, c->sms, 0, c->tex_s_enc));
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

GAES_API int gaes_uses_sbox_texture(int device) {
  DevCtx* c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  return c->tex_s_enc && c->tex_s_dec ? 1 : 0;
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
  void* dst = nullptr;
  PrivateInput tmp;
  PrivateOutput tmpo;
  rc = private_input_if_aliased(in, out, n_blocks * 16, false, (cudaStream_t)stream, &src, &tmp);
  if (!rc) rc = aligned_output(out, n_blocks * 16, (cudaStream_t)stream, &dst, &tmpo);
  if (rc) return rc;
  rc = for_segments(c, n_blocks, [&](size_t off, size_t cnt) {
    const uint4* i = static_cast<const uint4*>(src) + off;
    GAES_CK(launch_enc_folded(c, i, static_cast<uint4*>(dst) + off, cnt, c->d_std_enc, k, ilp_default(),
                              (cudaStream_t)stream, tex_for(c, i, cnt * 16, (cudaStream_t)stream)));
    return GAES_OK;
  });
  return rc ? rc : tmpo.finish();
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
  void* dst = nullptr;
  PrivateInput tmp;
  PrivateOutput tmpo;
  rc = private_input_if_aliased(in, out, n_blocks * 16, false, (cudaStream_t)stream, &src, &tmp);
  if (!rc) rc = aligned_output(out, n_blocks * 16, (cudaStream_t)stream, &dst, &tmpo);
  if (rc) return rc;
  rc = for_segments(c, n_blocks, [&](size_t off, size_t cnt) {
    const uint4* i = static_cast<const uint4*>(src) + off;
    GAES_CK(launch_folded(c, true, i, static_cast<uint4*>(dst) + off, cnt, c->d_std_dec, k, (cudaStream_t)stream,
                          tex_for(c, i, cnt * 16, (cudaStream_t)stream)));
    return GAES_OK;
  });
  return rc ? rc : tmpo.finish();
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
  void* out_w = nullptr;
  PrivateInput tmp, tmpiv;
  PrivateOutput tmpo;
  rc = private_input_if_aliased(in, out, n * m, false, (cudaStream_t)stream, &src, &tmp);
  if (!rc) rc = aligned_output(out, n * m, (cudaStream_t)stream, &out_w, &tmpo);
  if (!rc) rc = aligned_input(ivs_dev, n * 16, (cudaStream_t)stream, &ivs_dev, &tmpiv);
  if (rc) return rc;
  if (bpr == 1) {
    GAES_CK(launch_blocks(false, kIvChain, ilp_default(), src, out_w, n, c->d_std_enc, k, ivs_dev, 1, c->sms,
                          (cudaStream_t)stream, tex_for(c, src, n * 16, (cudaStream_t)stream),
                          tex_for(c, ivs_dev, n * 16, (cudaStream_t)stream), sbox_tex(c, c->d_std_enc)));
    note_kernel("k_blocks_enc_chain");
  } else {
    // segments of whole rows, each inside one texture
    const size_t seg_blocks = tex_segment_blocks(c);
    const size_t seg_rows = seg_blocks >= bpr ? seg_blocks / bpr : n;
    const uint8_t* i8 = static_cast<const uint8_t*>(src);
    uint8_t* o8 = static_cast<uint8_t*>(out_w);
    const uint8_t* v8 = static_cast<const uint8_t*>(ivs_dev);
    for (size_t r = 0; r < n; r += seg_rows) {
      const size_t cnt = std::min(seg_rows, n - r);
      GAES_CK(launch_cbc_enc_rows(i8 + r * m, o8 + r * m, cnt, bpr, c->d_std_enc, k, v8 ? v8 + r * 16 : nullptr,
                                  c->sms, (cudaStream_t)stream, tex_for(c, i8 + r * m, cnt * m, (cudaStream_t)stream),
                                  sbox_tex(c, c->d_std_enc)));
    }
    note_kernel(last_rows_kernel());
  }
  return tmpo.finish();
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
  void* out_w = nullptr;
  PrivateInput tmp, tmpiv;
  PrivateOutput tmpo;
  rc = private_input_if_aliased(in, out, n * m, bpr > 1, (cudaStream_t)stream, &src, &tmp);
  if (!rc) rc = aligned_output(out, n * m, (cudaStream_t)stream, &out_w, &tmpo);
  if (!rc) rc = aligned_input(ivs_dev, n * 16, (cudaStream_t)stream, &ivs_dev, &tmpiv);
  if (rc) return rc;
  GAES_CK(launch_blocks(true, kIvChain, ilp_default(), src, out_w, n * bpr, c->d_std_dec, k, ivs_dev, bpr, c->sms,
                        (cudaStream_t)stream, tex_for(c, src, n * bpr * 16, (cudaStream_t)stream),
                        bpr == 1 && ivs_dev ? tex_for(c, ivs_dev, n * 16, (cudaStream_t)stream) : TexLease(),
                        sbox_tex(c, c->d_std_dec)));
  note_kernel("k_blocks_dec_chain");
  return tmpo.finish();
}

GAES_API int gaes_expand_keys_dev(const void* keys, size_t k, void* rk_enc, void* rk_dec, void* stream) {
  if (k == 0) return GAES_OK;
  if (!keys || !rk_enc) return fail(GAES_EINVAL, "null pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  // the schedules are written as 32-bit words: misaligned outputs go through
  // private buffers
  void *enc = nullptr, *dec = nullptr;
  PrivateOutput tenc, tdec;
  rc = aligned_output(rk_enc, k * 176, (cudaStream_t)stream, &enc, &tenc);
  if (!rc) rc = aligned_output(rk_dec, k * 176, (cudaStream_t)stream, &dec, &tdec);
  if (rc) return rc;
  GAES_CK(launch_expand_keys((const uint8_t*)keys, k, c->d_std_enc, (uint8_t*)enc, (uint8_t*)dec,
                             (cudaStream_t)stream));
  note_kernel("k_expand_keys");
  rc = tenc.finish();
  return rc ? rc : tdec.finish();
}

GAES_API int gaes_many_key_encrypt_dev(const void* in, void* out, size_t blocks_per_key, size_t k,
                                       const void* rk_enc, const void* ivs_dev, void* stream) {
  if (k == 0 || blocks_per_key == 0) return GAES_OK;
  if (!in || !out || !rk_enc) return fail(GAES_EINVAL, "null pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  const void *src = nullptr, *rks = nullptr, *kivs = nullptr;
  void* dst = nullptr;
  PrivateInput tmp, trk, tiv;
  PrivateOutput tmpo;
  rc = private_input_if_aliased(in, out, blocks_per_key * k * 16, false, (cudaStream_t)stream, &src, &tmp);
  if (!rc) rc = aligned_output(out, blocks_per_key * k * 16, (cudaStream_t)stream, &dst, &tmpo);
  if (!rc) rc = aligned_input(rk_enc, k * 176, (cudaStream_t)stream, &rks, &trk);
  if (!rc) rc = aligned_input(ivs_dev, k * 16, (cudaStream_t)stream, &kivs, &tiv);
  if (rc) return rc;
  rc = for_segments(c, blocks_per_key * k, [&](size_t off, size_t cnt) {
    const uint4* i = static_cast<const uint4*>(src) + off;
    GAES_CK(launch_many_key(false, i, static_cast<uint4*>(dst) + off, cnt, off, blocks_per_key, c->d_std_enc, rks,
                            kivs, c->sms, (cudaStream_t)stream, tex_for(c, i, cnt * 16, (cudaStream_t)stream),
                            sbox_tex(c, c->d_std_enc)));
    note_kernel("k_many_key_enc");
    return GAES_OK;
  });
  return rc ? rc : tmpo.finish();
}

GAES_API int gaes_many_key_decrypt_dev(const void* in, void* out, size_t blocks_per_key, size_t k,
                                       const void* rk_dec, const void* ivs_dev, void* stream) {
  if (k == 0 || blocks_per_key == 0) return GAES_OK;
  if (!in || !out || !rk_dec) return fail(GAES_EINVAL, "null pointer");
  DevCtx* c = nullptr;
  int rc = current_ctx(&c);
  if (rc) return rc;
  const void *src = nullptr, *rks = nullptr, *kivs = nullptr;
  void* dst = nullptr;
  PrivateInput tmp, trk, tiv;
  PrivateOutput tmpo;
  rc = private_input_if_aliased(in, out, blocks_per_key * k * 16, false, (cudaStream_t)stream, &src, &tmp);
  if (!rc) rc = aligned_output(out, blocks_per_key * k * 16, (cudaStream_t)stream, &dst, &tmpo);
  if (!rc) rc = aligned_input(rk_dec, k * 176, (cudaStream_t)stream, &rks, &trk);
  if (!rc) rc = aligned_input(ivs_dev, k * 16, (cudaStream_t)stream, &kivs, &tiv);
  if (rc) return rc;
  rc = for_segments(c, blocks_per_key * k, [&](size_t off, size_t cnt) {
    const uint4* i = static_cast<const uint4*>(src) + off;
    GAES_CK(launch_many_key(true, i, static_cast<uint4*>(dst) + off, cnt, off, blocks_per_key, c->d_std_dec, rks,
                            kivs, c->sms, (cudaStream_t)stream, tex_for(c, i, cnt * 16, (cudaStream_t)stream),
                            sbox_tex(c, c->d_std_dec)));
    note_kernel("k_many_key_dec");
    return GAES_OK;
  });
  return rc ? rc : tmpo.finish();
}

}  // extern "C"
