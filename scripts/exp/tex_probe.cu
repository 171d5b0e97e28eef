// Experiment: does the texture path add table-lookup bandwidth beside LDS?
// Runs the encrypt round function on register-resident states (no HBM) with
// a fraction of the T-table lookups served by tex1Dfetch from a 5 KiB linear
// texture instead of the lane-replicated shared-memory tables, and reports
// lookups/s.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_1506_08503_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "aes_ttable.cuh"
#include "gf.cuh"
using namespace gaes;

// MODE 0: all LDS.  MODE 1: T3 lookups via texture.  MODE 2: T2+T3 via texture.
template <int MODE>
__global__ void __launch_bounds__(1024, 1) probe(const uint32_t* compact, cudaTextureObject_t tex, uint32_t iters,
                                                  uint32_t* sink) {
  extern __shared__ __align__(1024) char smem[];
  fill_tables(smem, compact);
  const uint32_t lb = (threadIdx.x & 31) * 4;
  uint32_t s0 = threadIdx.x, s1 = blockIdx.x, s2 = threadIdx.x * 7, s3 = ~threadIdx.x;
  for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 1; r < 10; r++) {
#define L0(x) lds_u32(smem, taddr<0>(x, lb), kOffT0)
#define L1(x) lds_u32(smem, taddr<1>(x, lb), kOffT1)
#define L2(x) (MODE >= 2 ? (uint32_t)tex1Dfetch<unsigned int>(tex, 512 + ((x >> 16) & 0xFF)) : lds_u32(smem, taddr<2>(x, lb), kOffT2))
#define L3(x) (MODE >= 1 ? (uint32_t)tex1Dfetch<unsigned int>(tex, 768 + (x >> 24)) : lds_u32(smem, taddr<3>(x, lb), kOffT3))
      const uint32_t t0 = L0(s0) ^ L1(s1) ^ L2(s2) ^ L3(s3) ^ r;
      const uint32_t t1 = L0(s1) ^ L1(s2) ^ L2(s3) ^ L3(s0) ^ r;
      const uint32_t t2 = L0(s2) ^ L1(s3) ^ L2(s0) ^ L3(s1) ^ r;
      const uint32_t t3 = L0(s3) ^ L1(s0) ^ L2(s1) ^ L3(s2) ^ r;
      s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
  }
  if ((s0 ^ s1 ^ s2 ^ s3) == 0x12345678u) sink[0] = s0;
}

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

template <int MODE>
double run(const uint32_t* d, cudaTextureObject_t tex, uint32_t* sink, int sms, uint32_t iters) {
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  probe<MODE><<<sms, 1024, kSmemBytes>>>(d, tex, 4, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<MODE><<<sms, 1024, kSmemBytes>>>(d, tex, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double lookups = (double)sms * 1024 * iters * 144.0;
  return lookups / (ms / 1e3) / 1e9;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *d, *sink;
  cudaMalloc(&d, 1280 * 4);
  cudaMalloc(&sink, 4);
  build<<<1, 256>>>(d);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = d;
  rd.res.linear.desc = cudaCreateChannelDesc<unsigned int>();
  rd.res.linear.sizeInBytes = 1280 * 4;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  const uint32_t iters = 256;
  printf("mode0 all-LDS      %.1f G lookups/s\n", run<0>(d, tex, sink, sms, iters));
  printf("mode1 T3 via TEX   %.1f G lookups/s\n", run<1>(d, tex, sink, sms, iters));
  printf("mode2 T2,T3 via TEX %.1f G lookups/s\n", run<2>(d, tex, sink, sms, iters));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
