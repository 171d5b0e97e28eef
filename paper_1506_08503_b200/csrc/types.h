// types.h -- host/device shared constants and parameter structs.
#pragma once
#include <stdint.h>

namespace gaes {

// Shared-memory T-table layout (see aes_ttable.cuh).
static constexpr int kRegionBytes = 65536;
static constexpr int kSmemBytes = 3 * kRegionBytes;  // 192 KiB, 1 CTA / SM
static constexpr int kOffT0 = 0;
static constexpr int kOffT1 = 128;
static constexpr int kOffT2 = kRegionBytes;
static constexpr int kOffT3 = kRegionBytes + 128;
static constexpr int kOffS = 2 * kRegionBytes;

// Compact (unreplicated) device table set, 5 x 256 words:
//   t[0..3][x] = T0..T3, t[4][x] = S[x] (low byte).
static constexpr int kCompactWords = 5 * 256;

// T0 (encrypt Te0 or decrypt Td0) for the small-batch kernel's fill, passed
// as a kernel parameter (constant bank).
struct SmallTables {
  uint32_t t0[256];
};

struct RoundKeys {
  // encrypt: w[4r+c] = LE word of rk[r][4c..4c+3]   (r = 0..10)
  // decrypt: w[0..3] = rk0, w[4r+c] = InvMix(rk_r) for r = 1..9, w[40..43] = rk10
  uint32_t w[44];
  uint32_t iv[4];  // shared IV for the CHAIN modes (not folded)
};

}  // namespace gaes
