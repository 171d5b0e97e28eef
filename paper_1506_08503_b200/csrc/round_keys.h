// round_keys.h -- host-side round-key preparation for the kernels' RoundKeys
// parameter (little-endian column words, IV folding, equivalent-inverse-
// cipher keys).  Internal to libgaes_b200.so.
#pragma once
#include <cstdint>

#include "gf.cuh"
#include "types.h"

namespace gaes {
namespace host {

// --------------------------------------------------------------------------
// Round keys.
inline uint32_t le32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// out byte r of column = XOR_j lut[r][j][b_j]  (_kernel.pyx:44-47 applied to a key column)
inline uint32_t mix_word_lut(uint32_t w, const uint8_t* lut) {
  uint32_t o = 0;
  for (int r = 0; r < 4; r++) {
    uint8_t acc = 0;
    for (int j = 0; j < 4; j++) acc ^= lut[(r * 4 + j) * 256 + ((w >> (8 * j)) & 0xFF)];
    o |= (uint32_t)acc << (8 * r);
  }
  return o;
}

inline uint32_t inv_mix_word_std(uint32_t w) {
  uint32_t o = 0;
  for (int r = 0; r < 4; r++) {
    uint8_t acc = 0;
    for (int j = 0; j < 4; j++) acc ^= gf_mul(mix_coef(true, r, j), (uint8_t)(w >> (8 * j)));
    o |= (uint32_t)acc << (8 * r);
  }
  return o;
}

// fold: XOR the shared IV into the first (encrypt) / last (decrypt) key.
inline RoundKeys make_enc_keys(const uint8_t* rk, const uint8_t* iv, bool fold) {
  RoundKeys k;
  for (int i = 0; i < 44; i++) k.w[i] = le32(rk + 4 * i);
  for (int c = 0; c < 4; c++) {
    k.iv[c] = iv ? le32(iv + 4 * c) : 0u;
    if (fold) k.w[c] ^= k.iv[c];
  }
  return k;
}

inline RoundKeys make_dec_keys(const uint8_t* rk, const uint8_t* iv, bool fold, const uint8_t* inv_lut) {
  RoundKeys k;
  for (int i = 0; i < 44; i++) {
    const uint32_t w = le32(rk + 4 * i);
    if (i >= 4 && i < 40)
      k.w[i] = inv_lut ? mix_word_lut(w, inv_lut) : inv_mix_word_std(w);
    else
      k.w[i] = w;
  }
  for (int c = 0; c < 4; c++) {
    k.iv[c] = iv ? le32(iv + 4 * c) : 0u;
    if (fold) k.w[c] ^= k.iv[c];
  }
  return k;
}

// Each lut[r][j] row must be GF(2)-linear for the equivalent inverse cipher.
inline bool lut_is_linear(const uint8_t* lut) {
  for (int t = 0; t < 16; t++) {
    const uint8_t* row = lut + t * 256;
    if (row[0] != 0) return false;
    for (int x = 1; x < 256; x++) {
      uint8_t acc = 0;
      for (int b = 0; b < 8; b++)
        if (x & (1 << b)) acc ^= row[1 << b];
      if (row[x] != acc) return false;
    }
  }
  return true;
}

}  // namespace host
}  // namespace gaes
