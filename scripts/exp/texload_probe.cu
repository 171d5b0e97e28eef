// Experiment: stream the input through the texture path (tex1Dfetch<uint4>
// on a linear texture) instead of LDG, to take the 16-byte global loads off
// the LSU data pipe that the T-table lookups saturate.
#include <cstdio>
#include <cuda_runtime.h>
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

template <bool TEX>
__global__ void __launch_bounds__(1024, 1) enc(const uint4* in, cudaTextureObject_t tin, uint4* out, uint64_t n,
                                               const uint32_t* compact, const __grid_constant__ RoundKeys rk) {
  extern __shared__ __align__(1024) char smem[];
  fill_tables(smem, compact);
  const uint32_t lb = (threadIdx.x & 31) * 4;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto ld = [&](uint64_t i) { return TEX ? tex1Dfetch<uint4>(tin, (int)i) : __ldcs(in + i); };
  uint4 cur = b < n ? ld(b) : make_uint4(0, 0, 0, 0);
  while (b < n) {
    const uint64_t nb = b + T;
    const uint4 nxt = nb < n ? ld(nb) : cur;
    uint32_t s0 = cur.x ^ rk.w[0], s1 = cur.y ^ rk.w[1], s2 = cur.z ^ rk.w[2], s3 = cur.w ^ rk.w[3];
    encrypt_rounds(smem, lb, s0, s1, s2, s3, rk);
    __stcs(out + b, make_uint4(s0, s1, s2, s3));
    cur = nxt;
    b = nb;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t n = 1ull << 24;
  uint4 *in, *out;
  uint32_t* tab;
  cudaMalloc(&in, n * 16);
  cudaMalloc(&out, n * 16);
  cudaMalloc(&tab, 1280 * 4);
  cudaMemset(in, 0x3c, n * 16);
  build<<<1, 256>>>(tab);
  RoundKeys rk;
  for (int i = 0; i < 44; i++) rk.w[i] = 0x9e3779b9u * (i + 1);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = in;
  rd.res.linear.desc = cudaCreateChannelDesc<uint4>();
  rd.res.linear.sizeInBytes = n * 16;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  cudaError_t e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  printf("texture: %s\n", cudaGetErrorString(e));
  cudaFuncSetAttribute(enc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  cudaFuncSetAttribute(enc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; mode++) {
    for (int w = 0; w < 3; w++) {
      if (mode) enc<true><<<sms, 1024, kSmemBytes>>>(in, tex, out, n, tab, rk);
      else enc<false><<<sms, 1024, kSmemBytes>>>(in, tex, out, n, tab, rk);
    }
    cudaEventRecord(a);
    for (int r = 0; r < 20; r++) {
      if (mode) enc<true><<<sms, 1024, kSmemBytes>>>(in, tex, out, n, tab, rk);
      else enc<false><<<sms, 1024, kSmemBytes>>>(in, tex, out, n, tab, rk);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s loads: %.1f GB/s\n", mode ? "texture" : "LDG    ", n * 16 / (ms / 20 / 1e3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
