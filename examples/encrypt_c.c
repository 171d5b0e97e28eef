/*
 * encrypt_c.c -- the C ABI used directly from C (no Python, no torch).
 *
 *   gcc -O2 -I include examples/encrypt_c.c -L paper_1506_08503_b200 \
 *       -lgaes_b200 -Wl,-rpath,$PWD/paper_1506_08503_b200 -o encrypt_c
 *   ./encrypt_c
 *
 * Expands the key on the host (key_schedule.py:50-70 restated in a few
 * lines), then checks the FIPS-197 C.1 block through the shared-IV entry
 * point and the SP 800-38A F.2.1 4-block CBC vector (encrypt + decrypt)
 * through the per-row-IV entry points.  Exit 0 = bit-exact.
 */
#include <stdio.h>
#include <stdint.h>
#include <string.h>

#include "gaes_b200.h"

/* key_schedule.py:50-70 restated in a few lines (host side of the example) */
static uint8_t xtime(uint8_t a) { return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1B : 0)); }
static uint8_t gmul(uint8_t a, uint8_t b) {
  uint8_t r = 0;
  while (b) { if (b & 1) r ^= a; a = xtime(a); b >>= 1; }
  return r;
}
static uint8_t sbox(uint8_t v) { /* inverse (a^254) then the AES affine map */
  uint8_t inv = 1, x = v;
  if (!v) inv = 0;
  else for (int e = 254; e; e >>= 1) { if (e & 1) inv = gmul(inv, x); x = gmul(x, x); }
  uint8_t s = inv;
  for (int i = 1; i < 5; i++) s ^= (uint8_t)((inv << i) | (inv >> (8 - i)));
  return s ^ 0x63;
}
static void expand(const uint8_t key[16], uint8_t rk[176]) {
  uint8_t rcon = 1;
  memcpy(rk, key, 16);
  for (int r = 1; r <= 10; r++) {
    const uint8_t *p = rk + 16 * (r - 1);
    uint8_t *c = rk + 16 * r;
    uint8_t t[4] = {sbox(p[13]), sbox(p[14]), sbox(p[15]), sbox(p[12])};
    t[0] ^= rcon;
    rcon = xtime(rcon);
    for (int i = 0; i < 4; i++) c[i] = p[i] ^ t[i];
    for (int i = 4; i < 16; i++) c[i] = p[i] ^ c[i - 4];
  }
}

static int hex_eq(const uint8_t *b, const char *hex, size_t n) {
  for (size_t i = 0; i < n; i++) {
    unsigned v;
    sscanf(hex + 2 * i, "%2x", &v);
    if (b[i] != v) return 0;
  }
  return 1;
}

int main(void) {
  if (gaes_device_count() < 1) { printf("no CUDA device\n"); return 2; }
  uint8_t key[16], rk[176], iv[16] = {0}, pt[16], ct[16];
  for (int i = 0; i < 16; i++) { key[i] = (uint8_t)i; pt[i] = (uint8_t)(0x11 * i); }
  expand(key, rk);
  if (gaes_encrypt_shared_iv(pt, 1, 16, iv, rk, ct)) { printf("error: %s\n", gaes_last_error()); return 1; }
  int ok = hex_eq(ct, "69c4e0d86a7b0430d8cdb78070b4c55a", 16);
  /* SP 800-38A F.2.1: one 4-block CBC row */
  static const char *K = "2b7e151628aed2a6abf7158809cf4f3c", *IV = "000102030405060708090a0b0c0d0e0f";
  static const char *P = "6bc1bee22e409f96e93d7e117393172aae2d8a571e03ac9c9eb76fac45af8e51"
                         "30c81c46a35ce411e5fbc1191a0a52eff69f2445df4f9b17ad2b417be66c3710";
  uint8_t k2[16], iv2[16], p2[64], c2[64], back[64];
  for (int i = 0; i < 16; i++) { unsigned v; sscanf(K + 2 * i, "%2x", &v); k2[i] = (uint8_t)v;
                                 sscanf(IV + 2 * i, "%2x", &v); iv2[i] = (uint8_t)v; }
  for (int i = 0; i < 64; i++) { unsigned v; sscanf(P + 2 * i, "%2x", &v); p2[i] = (uint8_t)v; }
  expand(k2, rk);
  if (gaes_cbc_encrypt_std(p2, iv2, 1, 64, rk, c2) || gaes_cbc_decrypt_std(c2, iv2, 1, 64, rk, back)) {
    printf("error: %s\n", gaes_last_error());
    return 1;
  }
  ok &= hex_eq(c2, "7649abac8119b246cee98e9b12e9197d5086cb9b507219ee95db113a917678b2", 32);
  ok &= memcmp(back, p2, 64) == 0;
  printf("%s (abi %d, %d device(s), %llu launches)\n", ok ? "ok" : "MISMATCH", gaes_version(),
         gaes_device_count(), (unsigned long long)gaes_launch_count());
  return ok ? 0 : 1;
}
