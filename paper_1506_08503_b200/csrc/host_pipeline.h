// host_pipeline.h -- host-buffer jobs of libgaes_b200.so (internal): the
// 7-argument backend contract and the shared-IV / many-key host entries run
// as Jobs -- one zero-copy launch for small pinned jobs, else a chunked
// H2D -> kernel -> D2H pipeline on a lane -- sharded over GPUs with the
// reference's plan semantics (parallel.py:37-50).
#pragma once
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "device_ctx.h"

namespace gaes {
namespace rt {

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

// Runs rows [0, j.n) of `j` on device context c (one shard).
int run_job(DevCtx* c, const Job& j);
// Shards j over the GPUs in use (gaes_set_num_gpus); one host thread each.
int run_sharded(const Job& j);
std::vector<std::pair<size_t, size_t>> plan_rows(size_t n, int workers);
int gpus_in_use();
int check_grid(const void* data, const void* out, size_t n, size_t m);
// gaes_cbc_encrypt / gaes_cbc_decrypt (the reference backend contract).
int cbc_host(bool dec, const uint8_t* data, const uint8_t* ivs, size_t n, size_t m, const uint8_t* rk,
             const uint8_t* box, const uint8_t* lut, const uint8_t* perm, uint8_t* out);
// gaes_encrypt_shared_iv / gaes_decrypt_shared_iv.
int shared_iv_host(bool dec, const uint8_t* data, size_t n, size_t m, const uint8_t* iv, const uint8_t* rk,
                   uint8_t* out);
// gaes_many_key_encrypt / gaes_many_key_decrypt.
int many_key_host(bool dec, const uint8_t* data, size_t bpk, size_t k, const uint8_t* keys, const uint8_t* ivs,
                  uint8_t* out);

}  // namespace rt
}  // namespace gaes
