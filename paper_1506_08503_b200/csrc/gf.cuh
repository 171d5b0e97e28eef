// gf.cuh -- GF(2^8) layer for the device (north_star subsystem (1)).
//
// Field: polynomials over GF(2) modulo x^8 + x^4 + x^3 + x + 1 (0x11B,
// gf256.py:21).  The substitution tables are *generated* from field
// arithmetic exactly as the reference does (sbox_gen.py:22-55):
//   S[v]    = A  . inv(v)  + 0x63,  A  = circulant(1,1,1,1,1,0,0,0) MSB-first
//   S^-1[v] = inv(A' . v + 0x05),   A' = circulant(0,1,0,1,0,0,1,0) MSB-first
// with the MSB-first bit-vector / right-shift circulant conventions of
// gf256.py:78-115.  The inverse is a^254 (gf256.py:66-75), computed here
// by square-and-multiply (same value, 13 multiplies instead of 254).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define GF_HD __host__ __device__ __forceinline__
#else
#define GF_HD inline
#endif

namespace gaes {

static constexpr unsigned kReductionPoly = 0x11B;  // gf256.py:21

// gf256.py:38-50: shift-and-XOR multiply with interleaved reduction.
GF_HD uint8_t gf_mul(uint8_t a_in, uint8_t b_in) {
  unsigned a = a_in, b = b_in, acc = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    if (b & 1) acc ^= a;
    a <<= 1;
    if (a & 0x100) a ^= kReductionPoly;
    b >>= 1;
  }
  return (uint8_t)acc;
}

// gf256.py:66-75: inverse = a^254 (a^(2^8-2)), inv(0) = 0.
GF_HD uint8_t gf_inv(uint8_t a) {
  if (a == 0) return 0;
  // 254 = 0b11111110: a^254 = prod_{i=1..7} a^(2^i)
  uint8_t sq = gf_mul(a, a);  // a^2
  uint8_t acc = sq;
#pragma unroll
  for (int i = 2; i <= 7; i++) {
    sq = gf_mul(sq, sq);  // a^(2^i)
    acc = gf_mul(acc, sq);
  }
  return acc;
}

// gf256.py:96-115 (bit_circulant + gf2_affine) on MSB-first bit vectors:
// row r of the circulant is `row` cyclically shifted right by r; output bit
// i (MSB-first) = XOR_j A[i][j] & y[j]  ^  b[i].
GF_HD uint8_t gf2_affine_msb(uint8_t row_bits_msb_first, uint8_t y, uint8_t b) {
  // row_bits_msb_first: bit (7-j) holds A[0][j].
  unsigned out = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    // row i = row 0 shifted right by i (MSB-first) == rotate right by i of
    // the byte encoding.
    unsigned ri = ((row_bits_msb_first >> i) | (row_bits_msb_first << (8 - i))) & 0xFF;
#if defined(__CUDA_ARCH__)
    unsigned bit = __popc(ri & y) & 1;
#else
    unsigned bit = __builtin_popcount(ri & y) & 1;
#endif
    out = (out << 1) | bit;
  }
  return (uint8_t)(out ^ b);
}

static constexpr uint8_t kForwardAffineRow = 0xF8;  // (1,1,1,1,1,0,0,0) sbox_gen.py:16
static constexpr uint8_t kForwardAffineConst = 0x63;
static constexpr uint8_t kInverseAffineRow = 0x52;  // (0,1,0,1,0,0,1,0) sbox_gen.py:18
static constexpr uint8_t kInverseAffineConst = 0x05;

GF_HD uint8_t sbox_forward(uint8_t v) {  // sbox_gen.py:22-34
  return gf2_affine_msb(kForwardAffineRow, gf_inv(v), kForwardAffineConst);
}
GF_HD uint8_t sbox_inverse(uint8_t v) {  // sbox_gen.py:37-55
  return gf_inv(gf2_affine_msb(kInverseAffineRow, v, kInverseAffineConst));
}

// aes_cbc.py:34-36 mix rows; circulant() (gf256.py:158-165): row r = row 0
// shifted right by r, so M[r][j] = row0[(j - r) & 3].
GF_HD uint8_t mix_row0(bool inverse, int k) {
  const uint32_t fwd = 0x01010302u;  // bytes (2, 3, 1, 1)
  const uint32_t inv = 0x090D0B0Eu;  // bytes (14, 11, 13, 9)
  return (uint8_t)(((inverse ? inv : fwd) >> (8 * (k & 3))) & 0xFF);
}
GF_HD uint8_t mix_coef(bool inverse, int r, int j) { return mix_row0(inverse, (j - r) & 3); }

}  // namespace gaes
