// aes_ttable.cuh -- T-table round function with the tables in shared memory.
//
// Formulation (the reference's round, _kernel.pyx:36-51, regrouped): for
// rounds 1..9 one output column is
//     t_c = XOR_j T_j[ s[(c + j) mod 4].byte j ]  ^  rk_r[c]
// where T_j[x] = pack_r mix_lut[r][j][S[x]] fuses SubBytes, the ShiftRows
// gather (shift_src[4c+j] = 4((c+j) mod 4) + j) and the MixColumns LUT
// sum (_kernel.pyx:44-47).  Round 10 is S[...] gathered into bytes.
// Decryption uses the equivalent inverse cipher: InvShift and InvSub
// commute, and InvMix is GF(2)-linear, so ARK(r) followed by InvMix equals
// InvMix followed by ARK with InvMix(rk_r) (checked on the host for the
// tables passed in), giving the same shape with T_j built from S^-1 and the
// inverse mix rows, and source word (c - j) mod 4.
//
// Shared-memory layout (bank-conflict free by construction): every table
// is replicated 32x so lane l always reads bank l.  Entry x of a region
// starts at byte x*256; words [0,32) hold table A[x] (one copy per lane),
// words [32,64) hold table B[x].  With lanebase = 4*lane the byte address
// of A[byte] for lane l is (byte << 8) | 4l -- a single PRMT builds it from
// the state word (no shift, no mask), and LDS [addr + UR + imm] adds the
// region/table offset for free.
//     region 0: T0 | T1      region 1: T2 | T3      region 2: S | (unused)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "types.h"

namespace gaes {

__device__ __forceinline__ uint32_t lds_u32(const char* smem, uint32_t addr, int off) {
  return *reinterpret_cast<const uint32_t*>(smem + addr + off);
}

// (byte k of s) << 8 | lanebase  -- one PRMT.
template <int K>
__device__ __forceinline__ uint32_t taddr(uint32_t s, uint32_t lanebase) {
  return __byte_perm(s, lanebase, 0x5504 | (K << 4));
}

// Word i of the compact tables, staged in the unused upper half of region 2
// (the S region only uses words 0..31 of each 256-byte entry).
__device__ __forceinline__ uint32_t* stage_word(char* smem, int i) {
  return reinterpret_cast<uint32_t*>(smem + kOffS + (i >> 5) * 256 + 128 + (i & 31) * 4);
}

// Replicate the compact tables into the CTA's shared memory.  Two phases:
// one coalesced pass brings the 5 KiB compact set from L2 into smem (a
// single L2 round trip per thread), then smem-to-smem replication.  Reading
// L2 inside the replication loop made every thread wait ~10 dependent L2
// round trips (~8 us per launch).
__device__ __forceinline__ void fill_tables(char* smem, const uint32_t* __restrict__ compact, bool with_s = true) {
  for (int i = threadIdx.x; i < kCompactWords; i += blockDim.x) *stage_word(smem, i) = __ldg(compact + i);
  __syncthreads();
  // 5 tables x 256 entries x 8 uint4 (32 lane copies) per entry; the S table
  // (the 5th) only when round 10 reads it from shared memory
  const int words = (with_s ? 5 : 4) * 256 * 8;
  for (int q = threadIdx.x; q < words; q += blockDim.x) {
    const int quad = q & 7;
    const int x = (q >> 3) & 255;
    const int tbl = q >> 11;
    const uint32_t v = *stage_word(smem, tbl * 256 + x);
    *reinterpret_cast<uint4*>(smem + (tbl >> 1) * kRegionBytes + x * 256 + (tbl & 1) * 128 + quad * 16) =
        make_uint4(v, v, v, v);
  }
  __syncthreads();
}

// S-box byte through the texture path (a 256-byte u8 linear texture: the
// last round's 16 lookups ride the TEX pipe instead of the saturated L1 /
// shared data pipe -- profiles/r1_formulation_choice.md).
__device__ __forceinline__ uint32_t tex_sbox(cudaTextureObject_t t, uint32_t x) {
  return (uint32_t)tex1Dfetch<unsigned char>(t, (int)x);
}

// One full AES-128 encryption of a state already XORed with rk0.  tsb: S-box
// texture for round 10, or 0 to read the replicated S table in smem.
__device__ __forceinline__ void encrypt_rounds(const char* smem, uint32_t lb, uint32_t& s0, uint32_t& s1,
                                               uint32_t& s2, uint32_t& s3, const RoundKeys& rk,
                                               cudaTextureObject_t tsb = 0) {
#pragma unroll
  for (int r = 1; r < 10; r++) {
    const uint32_t t0 = lds_u32(smem, taddr<0>(s0, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s1, lb), kOffT1) ^
                        lds_u32(smem, taddr<2>(s2, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s3, lb), kOffT3) ^
                        rk.w[4 * r + 0];
    const uint32_t t1 = lds_u32(smem, taddr<0>(s1, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s2, lb), kOffT1) ^
                        lds_u32(smem, taddr<2>(s3, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s0, lb), kOffT3) ^
                        rk.w[4 * r + 1];
    const uint32_t t2 = lds_u32(smem, taddr<0>(s2, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s3, lb), kOffT1) ^
                        lds_u32(smem, taddr<2>(s0, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s1, lb), kOffT3) ^
                        rk.w[4 * r + 2];
    const uint32_t t3 = lds_u32(smem, taddr<0>(s3, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s0, lb), kOffT1) ^
                        lds_u32(smem, taddr<2>(s1, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s2, lb), kOffT3) ^
                        rk.w[4 * r + 3];
    s0 = t0; s1 = t1; s2 = t2; s3 = t3;
  }
  // round 10: SubBytes + ShiftRows gather, no MixColumns (_kernel.pyx:41)
  // bytes assembled with integer multiply-adds (FMA pipe) to keep the ALU
  // pipe free for the address PRMTs and XORs.
#define GAES_LAST(a, b, c, d)                                                        \
  ((lds_u32(smem, taddr<3>(d, lb), kOffS) * 256u + lds_u32(smem, taddr<2>(c, lb), kOffS)) * 65536u + \
   (lds_u32(smem, taddr<1>(b, lb), kOffS) * 256u + lds_u32(smem, taddr<0>(a, lb), kOffS)))
#define GAES_LAST_T(a, b, c, d)                                                                     \
  ((tex_sbox(tsb, (d) >> 24) * 256u + tex_sbox(tsb, ((c) >> 16) & 0xFF)) * 65536u +                 \
   (tex_sbox(tsb, ((b) >> 8) & 0xFF) * 256u + tex_sbox(tsb, (a) & 0xFF)))
  uint32_t o0, o1, o2, o3;
  if (tsb) {
    o0 = GAES_LAST_T(s0, s1, s2, s3) ^ rk.w[40];
    o1 = GAES_LAST_T(s1, s2, s3, s0) ^ rk.w[41];
    o2 = GAES_LAST_T(s2, s3, s0, s1) ^ rk.w[42];
    o3 = GAES_LAST_T(s3, s0, s1, s2) ^ rk.w[43];
  } else {
    o0 = GAES_LAST(s0, s1, s2, s3) ^ rk.w[40];
    o1 = GAES_LAST(s1, s2, s3, s0) ^ rk.w[41];
    o2 = GAES_LAST(s2, s3, s0, s1) ^ rk.w[42];
    o3 = GAES_LAST(s3, s0, s1, s2) ^ rk.w[43];
  }
  s0 = o0; s1 = o1; s2 = o2; s3 = o3;
}

// Equivalent inverse cipher; input state already XORed with rk10; output
// is InvSub(InvShift(...)) of round 1, NOT yet XORed with rk0.
__device__ __forceinline__ void decrypt_rounds(const char* smem, uint32_t lb, uint32_t& s0, uint32_t& s1,
                                               uint32_t& s2, uint32_t& s3, const RoundKeys& rk,
                                               cudaTextureObject_t tsb = 0) {
#pragma unroll
  for (int r = 9; r >= 1; r--) {
    const uint32_t t0 = lds_u32(smem, taddr<0>(s0, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s3, lb), kOffT1) ^
                        lds_u32(smem, taddr<2>(s2, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s1, lb), kOffT3) ^
                        rk.w[4 * r + 0];
    const uint32_t t1 = lds_u32(smem, taddr<0>(s1, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s0, lb), kOffT1) ^
                        lds_u32(smem, taddr<2>(s3, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s2, lb), kOffT3) ^
                        rk.w[4 * r + 1];
    const uint32_t t2 = lds_u32(smem, taddr<0>(s2, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s1, lb), kOffT1) ^
                        lds_u32(smem, taddr<2>(s0, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s3, lb), kOffT3) ^
                        rk.w[4 * r + 2];
    const uint32_t t3 = lds_u32(smem, taddr<0>(s3, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s2, lb), kOffT1) ^
                        lds_u32(smem, taddr<2>(s1, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s0, lb), kOffT3) ^
                        rk.w[4 * r + 3];
    s0 = t0; s1 = t1; s2 = t2; s3 = t3;
  }
  uint32_t o0, o1, o2, o3;
  if (tsb) {
    o0 = GAES_LAST_T(s0, s3, s2, s1);
    o1 = GAES_LAST_T(s1, s0, s3, s2);
    o2 = GAES_LAST_T(s2, s1, s0, s3);
    o3 = GAES_LAST_T(s3, s2, s1, s0);
  } else {
    o0 = GAES_LAST(s0, s3, s2, s1);
    o1 = GAES_LAST(s1, s0, s3, s2);
    o2 = GAES_LAST(s2, s1, s0, s3);
    o3 = GAES_LAST(s3, s2, s1, s0);
  }
#undef GAES_LAST
#undef GAES_LAST_T
  s0 = o0; s1 = o1; s2 = o2; s3 = o3;
}

// ---------------------------------------------------------------------------
// Small-batch formulation (k_blocks_small): only region 0 (T0 | T1, 64 KiB)
// is filled.  MixColumns' matrices are circulant (aes_cbc.py:118-132:
// circ(2,3,1,1) and circ(14,11,13,9)), so T_j = rotl(T0, 8j): T2 = rot16(T0)
// and T3 = rot16(T1), and since rotation is XOR-linear one PRMT per output
// column covers both: t_c = T0[.] ^ T1[.] ^ rot16(T0[.] ^ T1[.]) ^ rk.  The
// same 144 conflict-free lookups per block, half the table fill, and the
// fill comes from the kernel parameters (no global round trip).  Standard
// tables only (the round-10 S-box is the GF layer's texture).
__device__ __forceinline__ uint32_t rot16(uint32_t x) { return __byte_perm(x, 0, 0x1032); }

__device__ __forceinline__ void encrypt_rounds_rot(const char* smem, uint32_t lb, uint32_t& s0, uint32_t& s1,
                                                   uint32_t& s2, uint32_t& s3, const RoundKeys& rk,
                                                   cudaTextureObject_t tsb) {
#pragma unroll
  for (int r = 1; r < 10; r++) {
    const uint32_t t0 = lds_u32(smem, taddr<0>(s0, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s1, lb), kOffT1) ^
                        rot16(lds_u32(smem, taddr<2>(s2, lb), kOffT0) ^ lds_u32(smem, taddr<3>(s3, lb), kOffT1)) ^
                        rk.w[4 * r + 0];
    const uint32_t t1 = lds_u32(smem, taddr<0>(s1, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s2, lb), kOffT1) ^
                        rot16(lds_u32(smem, taddr<2>(s3, lb), kOffT0) ^ lds_u32(smem, taddr<3>(s0, lb), kOffT1)) ^
                        rk.w[4 * r + 1];
    const uint32_t t2 = lds_u32(smem, taddr<0>(s2, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s3, lb), kOffT1) ^
                        rot16(lds_u32(smem, taddr<2>(s0, lb), kOffT0) ^ lds_u32(smem, taddr<3>(s1, lb), kOffT1)) ^
                        rk.w[4 * r + 2];
    const uint32_t t3 = lds_u32(smem, taddr<0>(s3, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s0, lb), kOffT1) ^
                        rot16(lds_u32(smem, taddr<2>(s1, lb), kOffT0) ^ lds_u32(smem, taddr<3>(s2, lb), kOffT1)) ^
                        rk.w[4 * r + 3];
    s0 = t0; s1 = t1; s2 = t2; s3 = t3;
  }
#define GAES_LAST_T(a, b, c, d)                                                                     \
  ((tex_sbox(tsb, (d) >> 24) * 256u + tex_sbox(tsb, ((c) >> 16) & 0xFF)) * 65536u +                 \
   (tex_sbox(tsb, ((b) >> 8) & 0xFF) * 256u + tex_sbox(tsb, (a) & 0xFF)))
  const uint32_t o0 = GAES_LAST_T(s0, s1, s2, s3) ^ rk.w[40];
  const uint32_t o1 = GAES_LAST_T(s1, s2, s3, s0) ^ rk.w[41];
  const uint32_t o2 = GAES_LAST_T(s2, s3, s0, s1) ^ rk.w[42];
  const uint32_t o3 = GAES_LAST_T(s3, s0, s1, s2) ^ rk.w[43];
  s0 = o0; s1 = o1; s2 = o2; s3 = o3;
}

// Equivalent inverse cipher with Td_j = rotl(Td0, 8j); source word (c - j) mod 4.
__device__ __forceinline__ void decrypt_rounds_rot(const char* smem, uint32_t lb, uint32_t& s0, uint32_t& s1,
                                                   uint32_t& s2, uint32_t& s3, const RoundKeys& rk,
                                                   cudaTextureObject_t tsb) {
#pragma unroll
  for (int r = 9; r >= 1; r--) {
    const uint32_t t0 = lds_u32(smem, taddr<0>(s0, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s3, lb), kOffT1) ^
                        rot16(lds_u32(smem, taddr<2>(s2, lb), kOffT0) ^ lds_u32(smem, taddr<3>(s1, lb), kOffT1)) ^
                        rk.w[4 * r + 0];
    const uint32_t t1 = lds_u32(smem, taddr<0>(s1, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s0, lb), kOffT1) ^
                        rot16(lds_u32(smem, taddr<2>(s3, lb), kOffT0) ^ lds_u32(smem, taddr<3>(s2, lb), kOffT1)) ^
                        rk.w[4 * r + 1];
    const uint32_t t2 = lds_u32(smem, taddr<0>(s2, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s1, lb), kOffT1) ^
                        rot16(lds_u32(smem, taddr<2>(s0, lb), kOffT0) ^ lds_u32(smem, taddr<3>(s3, lb), kOffT1)) ^
                        rk.w[4 * r + 2];
    const uint32_t t3 = lds_u32(smem, taddr<0>(s3, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s2, lb), kOffT1) ^
                        rot16(lds_u32(smem, taddr<2>(s1, lb), kOffT0) ^ lds_u32(smem, taddr<3>(s0, lb), kOffT1)) ^
                        rk.w[4 * r + 3];
    s0 = t0; s1 = t1; s2 = t2; s3 = t3;
  }
  const uint32_t o0 = GAES_LAST_T(s0, s3, s2, s1);
  const uint32_t o1 = GAES_LAST_T(s1, s0, s3, s2);
  const uint32_t o2 = GAES_LAST_T(s2, s1, s0, s3);
  const uint32_t o3 = GAES_LAST_T(s3, s2, s1, s0);
#undef GAES_LAST_T
  s0 = o0; s1 = o1; s2 = o2; s3 = o3;
}

}  // namespace gaes
