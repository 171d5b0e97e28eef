// aes_bitslice.cuh -- bitsliced AES-128 encryption (LOP3 formulation).
//
// 32 blocks per thread.  After a 32x32 bit transpose of each of the four
// column words, register st[32c + 8r + b] holds bit b of state byte 4c + r
// (row r, column c) for all 32 blocks (bit k = block k).  Then
//   SubBytes    = 16 evaluations of the Boyar-Peralta S-box circuit
//                 (113 gates: 32 AND + 81 XOR/XNOR; Boyar & Peralta, "A new
//                 combinational logic minimization technique with
//                 applications to cryptology", eprint 2009/191), which ptxas
//                 packs into 3-input LOP3s;
//   ShiftRows   = register renaming (free);
//   MixColumns  = out_r = xtime(a_r ^ a_{r+1}) ^ (a_0^a_1^a_2^a_3) ^ a_r per
//                 plane (the reference's circulant (2,3,1,1), aes_cbc.py:35);
//   AddRoundKey = XOR with key masks (0 or ~0 per plane, from the constant
//                 bank), folded into the MixColumns XOR trees.
// No shared memory and no table lookups: the formulation is bound by the
// ALU pipe (LOP3/SHF/PRMT), which makes it the complement of the T-table
// kernel (bound by the LSU/shared-memory pipe) -- see DESIGN.md.
//
// All functions are __host__ __device__ so tests can check them on the CPU.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define BS_HD __host__ __device__ __forceinline__
#else
#define BS_HD inline
#endif

namespace gaes {

BS_HD uint32_t bs_prmt(uint32_t a, uint32_t b, uint32_t sel) {
#if defined(__CUDA_ARCH__)
  return __byte_perm(a, b, sel);
#else
  const uint64_t x = ((uint64_t)b << 32) | a;
  uint32_t r = 0;
  for (int i = 0; i < 4; i++) r |= (uint32_t)((x >> (8 * ((sel >> (4 * i)) & 7))) & 0xFF) << (8 * i);
  return r;
#endif
}

// In-place 32x32 bit transpose: afterwards bit i of A[j] == old bit j of A[i].
BS_HD void transpose32(uint32_t* A) {
  // j = 16 and j = 8 swap whole bytes: two PRMTs per register pair.
#pragma unroll
  for (int k = 0; k < 16; k++) {
    const uint32_t a = A[k], b = A[k + 16];
    A[k] = bs_prmt(a, b, 0x5410);       // low halves: a.lo | b.lo << 16
    A[k + 16] = bs_prmt(a, b, 0x7632);  // high halves: a.hi | b.hi << 16
  }
#pragma unroll
  for (int g = 0; g < 32; g += 16)
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const uint32_t a = A[g + k], b = A[g + k + 8];
      A[g + k] = bs_prmt(a, b, 0x6240);      // a.b0 b.b0 a.b2 b.b2
      A[g + k + 8] = bs_prmt(a, b, 0x7351);  // a.b1 b.b1 a.b3 b.b3
    }
  // j = 4, 2, 1: mask-and-shift swaps (2 SHF + 2 LOP3 per pair).
#define GAES_TSTEP(J, M)                                                   \
  _Pragma("unroll") for (int g = 0; g < 32; g += 2 * J)                    \
  _Pragma("unroll") for (int k = 0; k < J; k++) {                          \
    const uint32_t a = A[g + k], b = A[g + k + J];                         \
    A[g + k] = (a & (M)) | ((b << J) & ~(M));                              \
    A[g + k + J] = ((a >> J) & (M)) | (b & ~(M));                          \
  }
  GAES_TSTEP(4, 0x0F0F0F0Fu)
  GAES_TSTEP(2, 0x33333333u)
  GAES_TSTEP(1, 0x55555555u)
#undef GAES_TSTEP
}

// Boyar-Peralta S-box.  Planes q0 (LSB) .. q7 (MSB) in and out.
BS_HD void bs_sbox(uint32_t& q0, uint32_t& q1, uint32_t& q2, uint32_t& q3, uint32_t& q4, uint32_t& q5,
                   uint32_t& q6, uint32_t& q7) {
  const uint32_t x0 = q7, x1 = q6, x2 = q5, x3 = q4, x4 = q3, x5 = q2, x6 = q1, x7 = q0;
  // top linear layer
  const uint32_t y14 = x3 ^ x5, y13 = x0 ^ x6, y9 = x0 ^ x3, y8 = x0 ^ x5;
  const uint32_t t0 = x1 ^ x2;
  const uint32_t y1 = t0 ^ x7;
  const uint32_t y4 = y1 ^ x3, y12 = y13 ^ y14, y2 = y1 ^ x0, y5 = y1 ^ x6;
  const uint32_t y3 = y5 ^ y8;
  const uint32_t t1 = x4 ^ y12;
  const uint32_t y15 = t1 ^ x5, y20 = t1 ^ x1;
  const uint32_t y6 = y15 ^ x7, y10 = y15 ^ t0, y11 = y20 ^ y9;
  const uint32_t y7 = x7 ^ y11, y17 = y10 ^ y11, y19 = y10 ^ y8, y16 = t0 ^ y11;
  const uint32_t y21 = y13 ^ y16, y18 = x0 ^ y16;
  // non-linear middle
  const uint32_t t2 = y12 & y15, t3 = y3 & y6, t4 = t3 ^ t2, t5 = y4 & x7, t6 = t5 ^ t2;
  const uint32_t t7 = y13 & y16, t8 = y5 & y1, t9 = t8 ^ t7, t10 = y2 & y7, t11 = t10 ^ t7;
  const uint32_t t12 = y9 & y11, t13 = y14 & y17, t14 = t13 ^ t12, t15 = y8 & y10, t16 = t15 ^ t12;
  const uint32_t t17 = t4 ^ t14, t18 = t6 ^ t16, t19 = t9 ^ t14, t20 = t11 ^ t16;
  const uint32_t t21 = t17 ^ y20, t22 = t18 ^ y19, t23 = t19 ^ y21, t24 = t20 ^ y18;
  const uint32_t t25 = t21 ^ t22, t26 = t21 & t23, t27 = t24 ^ t26, t28 = t25 & t27, t29 = t28 ^ t22;
  const uint32_t t30 = t23 ^ t24, t31 = t22 ^ t26, t32 = t31 & t30, t33 = t32 ^ t24, t34 = t23 ^ t33;
  const uint32_t t35 = t27 ^ t33, t36 = t24 & t35, t37 = t36 ^ t34, t38 = t27 ^ t36, t39 = t29 & t38;
  const uint32_t t40 = t25 ^ t39;
  const uint32_t t41 = t40 ^ t37, t42 = t29 ^ t33, t43 = t29 ^ t40, t44 = t33 ^ t37, t45 = t42 ^ t41;
  const uint32_t z0 = t44 & y15, z1 = t37 & y6, z2 = t33 & x7, z3 = t43 & y16, z4 = t40 & y1, z5 = t29 & y7;
  const uint32_t z6 = t42 & y11, z7 = t45 & y17, z8 = t41 & y10, z9 = t44 & y12, z10 = t37 & y3;
  const uint32_t z11 = t33 & y4, z12 = t43 & y13, z13 = t40 & y5, z14 = t29 & y2, z15 = t42 & y9;
  const uint32_t z16 = t45 & y14, z17 = t41 & y8;
  // bottom linear layer
  const uint32_t t46 = z15 ^ z16, t47 = z10 ^ z11, t48 = z5 ^ z13, t49 = z9 ^ z10, t50 = z2 ^ z12;
  const uint32_t t51 = z2 ^ z5, t52 = z7 ^ z8, t53 = z0 ^ z3, t54 = z6 ^ z7, t55 = z16 ^ z17;
  const uint32_t t56 = z12 ^ t48, t57 = t50 ^ t53, t58 = z4 ^ t46, t59 = z3 ^ t54, t60 = t46 ^ t57;
  const uint32_t t61 = z14 ^ t57, t62 = t52 ^ t58, t63 = t49 ^ t58, t64 = z4 ^ t59, t65 = t61 ^ t62;
  const uint32_t t66 = z1 ^ t63;
  const uint32_t s0 = t59 ^ t63, s6 = t56 ^ ~t62, s7 = t48 ^ ~t60, t67 = t64 ^ t65;
  const uint32_t s3 = t53 ^ t66, s4 = t51 ^ t66, s5 = t47 ^ t65, s1 = t64 ^ ~s3, s2 = t55 ^ ~t67;
  q7 = s0; q6 = s1; q5 = s2; q4 = s3; q3 = s4; q2 = s5; q1 = s6; q0 = s7;
}

BS_HD void bs_sub_bytes(uint32_t* st) {
#pragma unroll
  for (int i = 0; i < 16; i++) {
    uint32_t* q = st + 8 * i;  // byte 4c + r lives at 32c + 8r = 8 * (4c + r)
    bs_sbox(q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7]);
  }
}

// Plane index of state byte (column c, row r), bit b.
#define GAES_BS(c, r, b) (32 * ((c) & 3) + 8 * (r) + (b))

// ShiftRows + MixColumns + AddRoundKey: in -> out (distinct arrays).
// kp: 128 key masks for this round (kp[GAES_BS(c, r, b)]).
BS_HD void bs_shift_mix_ark(const uint32_t* in, uint32_t* out, const uint32_t* kp) {
#pragma unroll
  for (int c = 0; c < 4; c++) {
    // logical a_r = physical byte (c + r, r) after ShiftRows (aes_cbc.py:41)
    uint32_t t[4][8], S[8];
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int b = 0; b < 8; b++) t[r][b] = in[GAES_BS(c + r, r, b)] ^ in[GAES_BS(c + r + 1, (r + 1) & 3, b)];
#pragma unroll
    for (int b = 0; b < 8; b++) S[b] = t[0][b] ^ t[2][b];
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const uint32_t* tr = t[r];
      const uint32_t x[8] = {tr[7], tr[0] ^ tr[7], tr[1], tr[2] ^ tr[7], tr[3] ^ tr[7], tr[4], tr[5], tr[6]};
#pragma unroll
      for (int b = 0; b < 8; b++)
        out[GAES_BS(c, r, b)] = x[b] ^ S[b] ^ in[GAES_BS(c + r, r, b)] ^ kp[GAES_BS(c, r, b)];
    }
  }
}

// Last round: ShiftRows + AddRoundKey.
BS_HD void bs_shift_ark(const uint32_t* in, uint32_t* out, const uint32_t* kp) {
#pragma unroll
  for (int c = 0; c < 4; c++)
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int b = 0; b < 8; b++) out[GAES_BS(c, r, b)] = in[GAES_BS(c + r, r, b)] ^ kp[GAES_BS(c, r, b)];
}

// Key masks: kp[r][32c + q] = bit q of round-key word c of round r, as 0 / ~0.
struct BitsliceKeys {
  uint32_t kp[11][128];
};

BS_HD void bs_make_keys(const uint32_t* w /*44 words*/, BitsliceKeys& k) {
  for (int r = 0; r < 11; r++)
    for (int c = 0; c < 4; c++)
      for (int q = 0; q < 32; q++) k.kp[r][32 * c + q] = ((w[4 * r + c] >> q) & 1u) ? 0xFFFFFFFFu : 0u;
}

// Encrypt 32 blocks held as w[k][c] (block k, column word c) in st[4k + c]
// layout on input; output in the same layout.  st: 128 words.
BS_HD void bs_encrypt32(uint32_t* st, const BitsliceKeys& keys) {
  // gather columns: tmp[32c + k] = word c of block k, then transpose each 32
  uint32_t a[128];
#pragma unroll
  for (int k = 0; k < 32; k++)
#pragma unroll
    for (int c = 0; c < 4; c++) a[32 * c + k] = st[4 * k + c];
#pragma unroll
  for (int c = 0; c < 4; c++) transpose32(a + 32 * c);
#pragma unroll
  for (int i = 0; i < 128; i++) a[i] ^= keys.kp[0][i];
  // Rounds 1..9 stay a loop: one unrolled round body is ~2K instructions,
  // ten of them overflow the instruction cache (ncu: stalled_no_instructions).
#pragma unroll 1
  for (int r = 1; r < 10; r++) {
    bs_sub_bytes(a);
    uint32_t b[128];
    bs_shift_mix_ark(a, b, keys.kp[r]);
#pragma unroll
    for (int i = 0; i < 128; i++) a[i] = b[i];
  }
  bs_sub_bytes(a);
  {
    uint32_t b[128];
    bs_shift_ark(a, b, keys.kp[10]);
#pragma unroll
    for (int i = 0; i < 128; i++) a[i] = b[i];
  }
#pragma unroll
  for (int c = 0; c < 4; c++) transpose32(a + 32 * c);
#pragma unroll
  for (int k = 0; k < 32; k++)
#pragma unroll
    for (int c = 0; c < 4; c++) st[4 * k + c] = a[32 * c + k];
}

#undef GAES_BS

}  // namespace gaes
