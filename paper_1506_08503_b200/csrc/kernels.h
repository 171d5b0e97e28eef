// kernels.h -- internal (C++) launch interface between the kernels and the
// host dispatcher.  Not part of the C ABI (see include/gaes_b200.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "types.h"

namespace gaes {

static constexpr int kBlockThreads = 1024;     // k_blocks / k_cbc_enc_rows: 1 CTA per SM
static constexpr int kManyKeyThreads = 768;    // k_many_key: 44 round-key registers per thread (<= 85 regs)
static constexpr int kSmallThreads = 512;      // k_blocks_small: up to 3 CTAs per SM (PDL co-residence)
static constexpr int kSmallSmemBytes = 65536;  // region 0 (T0 | T1)
static constexpr int kBsThreads = 128;         // k_bs_blocks: ~170 registers per thread
static constexpr int kBsCtasPerSm = 3;
static constexpr int kIvFolded = 0;
static constexpr int kIvChain = 1;
static constexpr int kIvRows = 2;  // internal: kIvChain with bpr == 1 and per-row IVs

cudaError_t launch_gf_build(uint32_t* enc, uint32_t* dec, uint8_t* sbox, uint8_t* inv, int* err, cudaStream_t s);
cudaError_t launch_build_tables(const uint8_t* box, const uint8_t* lut, uint32_t* out, cudaStream_t s);
// tin: optional linear texture over `in` (uint4 texels); tiv: optional
// texture over `ivs` (per-row IVs with one block per row); 0 = plain LDG.
// tsb: optional u8 texture of the S-box matching `compact` (round 10 then
// reads it through the TEX pipe and the S table is not replicated in smem).
cudaError_t launch_blocks(bool dec, int ivmode, int ilp, const void* in, void* out, uint64_t n_blocks,
                          const uint32_t* compact, const RoundKeys& rk, const void* ivs, uint64_t bpr, int sms,
                          cudaStream_t s, cudaTextureObject_t tin = 0, cudaTextureObject_t tiv = 0,
                          cudaTextureObject_t tsb = 0);
// Small batches (n <= small_blocks_max(sms)), shared IV folded into the key,
// standard tables (t0 = Te0 / Td0 of the GF layer, tsb its S-box texture):
// k_blocks_small -- 64 KiB of tables filled from the kernel parameters, up
// to 3 CTAs per SM so the next launch fills while this one computes.
uint64_t small_blocks_max(int sms);
// early: the caller's stream has nothing in flight to overlap the fill with
// (synchronous host-buffer jobs): load the input first, then fill.
cudaError_t launch_blocks_small(bool dec, const void* in, void* out, uint64_t n_blocks, const uint32_t* t0,
                                const RoundKeys& rk, int sms, cudaStream_t s, cudaTextureObject_t tsb,
                                bool early = false);
// Row CBC encrypt: the TMA-staged kernel when it applies (texture S-box,
// >= 8 even blocks per row, enough rows), four lanes per row when there are
// too few rows to fill the GPU, else the LDG/STG kernel.
const char* last_rows_kernel();  // which row-CBC encrypt kernel the last launch on this thread used
cudaError_t launch_cbc_enc_rows(const void* in, void* out, uint64_t n_rows, uint64_t bpr, const uint32_t* compact,
                                const RoundKeys& rk, const void* ivs, int sms, cudaStream_t s,
                                cudaTextureObject_t tin = 0, cudaTextureObject_t tsb = 0);
cudaError_t launch_generic(bool dec, const uint8_t* data, const uint8_t* ivs, uint64_t n, uint64_t m,
                           const uint8_t* rk, const uint8_t* box, const uint8_t* lut, const uint8_t* perm,
                           uint8_t* out, int sms, cudaStream_t s);
struct BitsliceKeys;
cudaError_t launch_bs_blocks(const void* in, void* out, uint64_t n_blocks, const BitsliceKeys& keys, int sms,
                             cudaStream_t s);
cudaError_t launch_round_probe(const uint32_t* compact, const RoundKeys& rk, uint32_t iters, uint32_t* sink,
                               int sms, cudaStream_t s,
                               cudaTextureObject_t tsb = 0);
// Shared-memory lookup peak: 16 conflict-free LDS.32 per thread per iteration.
cudaError_t launch_lds_peak(uint32_t iters, uint32_t* sink, int sms, cudaStream_t s);
cudaError_t launch_expand_keys(const uint8_t* keys, uint64_t k, const uint32_t* compact_enc, uint8_t* rk_enc,
                               uint8_t* rk_dec, cudaStream_t s);
cudaError_t launch_many_key(bool dec, const void* in, void* out, uint64_t n_blocks, uint64_t first, uint64_t bpk,
                            const uint32_t* compact, const void* rks, const void* ivs, int sms, cudaStream_t s,
                            cudaTextureObject_t tin = 0, cudaTextureObject_t tsb = 0);

}  // namespace gaes
