"""CPU check of the bitsliced round function (csrc/aes_bitslice.cuh, host build).

The header is __host__ __device__; compiled here with g++ against the C
oracle it must reproduce the oracle's ciphertexts, and the Boyar-Peralta
circuit must equal the GF-layer S-box on all 256 inputs.
"""

import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROGRAM = r'''
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cstdint>
#include "aes_bitslice.cuh"
#include "gf.cuh"
extern "C" {
void oracle_gen_sbox(uint8_t out[256]);
void oracle_gen_keys(const uint8_t key[16], const uint8_t sbox[256], uint8_t rk[176]);
void oracle_mix_lut(const uint8_t first_row[4], uint8_t lut[4096]);
int oracle_cbc_encrypt(const uint8_t*, const uint8_t*, size_t, size_t, const uint8_t*, const uint8_t*,
                       const uint8_t*, const uint8_t*, uint8_t*, int);
}
int main() {
  uint8_t sbox[256], lut[4096], key[16], rk[176], row[4] = {2, 3, 1, 1};
  const uint8_t shift[16] = {0, 5, 10, 15, 4, 9, 14, 3, 8, 13, 2, 7, 12, 1, 6, 11};
  oracle_gen_sbox(sbox);
  oracle_mix_lut(row, lut);
  // S-box circuit vs field arithmetic, all inputs (8 lanes of 32 values)
  for (int base = 0; base < 256; base += 32) {
    uint32_t q[8] = {0};
    for (int k = 0; k < 32; k++)
      for (int b = 0; b < 8; b++) q[b] |= (uint32_t)(((base + k) >> b) & 1) << k;
    gaes::bs_sbox(q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7]);
    for (int k = 0; k < 32; k++) {
      int v = 0;
      for (int b = 0; b < 8; b++) v |= ((q[b] >> k) & 1) << b;
      if (v != sbox[base + k] || v != gaes::sbox_forward((uint8_t)(base + k))) { printf("sbox %d\n", base + k); return 2; }
    }
  }
  uint32_t A[32], B[32];
  srand(3);
  for (int i = 0; i < 32; i++) A[i] = B[i] = (uint32_t)rand() * 2654435761u ^ (uint32_t)rand();
  gaes::transpose32(A);
  for (int i = 0; i < 32; i++)
    for (int j = 0; j < 32; j++)
      if (((A[j] >> i) & 1) != ((B[i] >> j) & 1)) { printf("transpose %d %d\n", i, j); return 3; }
  for (int trial = 0; trial < 64; trial++) {
    for (int i = 0; i < 16; i++) key[i] = (uint8_t)rand();
    oracle_gen_keys(key, sbox, rk);
    uint32_t w[44];
    memcpy(w, rk, 176);
    static gaes::BitsliceKeys K;
    gaes::bs_make_keys(w, K);
    uint8_t pt[512], ct[512], iv[512] = {0};
    for (int i = 0; i < 512; i++) pt[i] = (uint8_t)rand();
    uint32_t st[128];
    memcpy(st, pt, 512);
    gaes::bs_encrypt32(st, K);
    oracle_cbc_encrypt(pt, iv, 32, 16, rk, sbox, lut, shift, ct, 1);
    if (memcmp(st, ct, 512)) { printf("encrypt trial %d\n", trial); return 4; }
  }
  printf("ok\n");
  return 0;
}
'''


def test_bitsliced_round_function_on_cpu(tmp_path):
    if not shutil.which("g++") or not shutil.which("gcc"):
        pytest.skip("no host compiler")
    src = tmp_path / "t.cpp"
    src.write_text(PROGRAM)
    obj = tmp_path / "oracle.o"
    subprocess.check_call(["gcc", "-O2", "-c", os.path.join(REPO, "oracle", "gaes_oracle.c"), "-o", str(obj)])
    exe = tmp_path / "t"
    subprocess.check_call(["g++", "-O1", "-w", "-I", os.path.join(REPO, "paper_1506_08503_b200", "csrc"),
                           str(src), str(obj), "-lpthread", "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout + out.stderr
