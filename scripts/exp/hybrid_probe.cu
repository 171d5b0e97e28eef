// Experiment: T-table kernel (1024 threads, 40 regs, 192 KiB smem, LSU-bound)
// co-resident with a 64-thread bitsliced CTA per SM (2 warps, <= 232 regs,
// ALU-bound) on a second stream; static split of 2^24 blocks.  Reports the
// combined GB/s for several bitsliced fractions.
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "aes_bitslice.cuh"
#include "aes_ttable.cuh"
#include "gf.cuh"
using namespace gaes;

__global__ void build(uint32_t* out) {
  const int v = threadIdx.x;
  const uint8_t S = sbox_forward((uint8_t)v);
  for (int j = 0; j < 4; j++) {
    uint32_t te = 0;
    for (int r = 0; r < 4; r++) te |= (uint32_t)gf_mul(mix_coef(false, r, j), S) << (8 * r);
    out[j * 256 + v] = te;
  }
  out[1024 + v] = S;
}

__global__ void __launch_bounds__(1024, 1) tt(const uint4* in, uint4* out, uint64_t n, const uint32_t* compact,
                                              const __grid_constant__ RoundKeys rk) {
  extern __shared__ __align__(1024) char smem[];
  fill_tables(smem, compact);
  const uint32_t lb = (threadIdx.x & 31) * 4;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n; b += T) {
    uint4 v = __ldcs(in + b);
    uint32_t s0 = v.x ^ rk.w[0], s1 = v.y ^ rk.w[1], s2 = v.z ^ rk.w[2], s3 = v.w ^ rk.w[3];
    encrypt_rounds(smem, lb, s0, s1, s2, s3, rk);
    __stcs(out + b, make_uint4(s0, s1, s2, s3));
  }
}

__global__ void __maxnreg__(232)
    bs(const uint4* in, uint4* out, uint64_t n, const __grid_constant__ BitsliceKeys keys) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t ch = warp; ch < (n + 1023) / 1024; ch += n_warps) {
    uint32_t st[128];
    for (int k = 0; k < 32; k++) {
      const uint64_t b = ch * 1024 + lane + 32 * k;
      const uint4 v = b < n ? __ldcs(in + b) : make_uint4(0, 0, 0, 0);
      st[4 * k] = v.x; st[4 * k + 1] = v.y; st[4 * k + 2] = v.z; st[4 * k + 3] = v.w;
    }
    bs_encrypt32(st, keys);
    for (int k = 0; k < 32; k++) {
      const uint64_t b = ch * 1024 + lane + 32 * k;
      if (b < n) __stcs(out + b, make_uint4(st[4 * k], st[4 * k + 1], st[4 * k + 2], st[4 * k + 3]));
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t n = 1ull << 24;
  uint4 *in, *out, *ref;
  uint32_t* tab;
  cudaMalloc(&in, n * 16);
  cudaMalloc(&out, n * 16);
  cudaMalloc(&ref, n * 16);
  cudaMalloc(&tab, 1280 * 4);
  cudaMemset(in, 0x5a, n * 16);
  build<<<1, 256>>>(tab);
  RoundKeys rk;
  for (int i = 0; i < 44; i++) rk.w[i] = 0x01020304u * (i + 1);
  static BitsliceKeys bk;
  bs_make_keys(rk.w, bk);
  cudaFuncSetAttribute(tt, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  tt<<<sms, 1024, kSmemBytes, a>>>(in, ref, n, tab, rk);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double fr[] = {0.0, 0.01, 0.02, 0.03, 0.05, 0.08};
  for (double f : fr) {
    const uint64_t nbs = ((uint64_t)(f * n)) & ~1023ull, ntt = n - nbs;
    float best = 1e9;
    for (int rep = 0; rep < 6; rep++) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, a);
      cudaStreamWaitEvent(b, e0, 0);
      tt<<<sms, 1024, kSmemBytes, a>>>(in, out, ntt, tab, rk);
      if (nbs) bs<<<sms, 64, 0, b>>>(in + ntt, out + ntt, nbs, bk);
      cudaEvent_t j;
      cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
      cudaEventRecord(j, b);
      cudaStreamWaitEvent(a, j, 0);
      cudaEventRecord(e1, a);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
      cudaEventDestroy(j);
    }
    std::vector<uint4> h1(n), h2(n);
    cudaMemcpy(h1.data(), out, n * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), ref, n * 16, cudaMemcpyDeviceToHost);
    const bool same = memcmp(h1.data(), h2.data(), n * 16) == 0;
    printf("bitsliced share %.2f: %.1f GB/s (%s)\n", f, n * 16 / (best / 1e3) / 1e9, same ? "bit-exact" : "MISMATCH");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
