// Experiment: serve (part of) the last round's 16 S-box lookups from the
// texture path (a 256-byte u8 linear texture: 8 sectors) instead of the
// lane-replicated S table in shared memory, so the TEX pipe carries some of
// the lookup work beside the saturated L1/shared data pipe.  Full encrypt
// (rounds 1-9 T-table LDS + round 10) on register-resident states, no HBM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_1506_08503_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "aes_ttable.cuh"
#include "gf.cuh"
using namespace gaes;

__device__ __forceinline__ uint32_t sx(cudaTextureObject_t t, uint32_t x) {
  return (uint32_t)tex1Dfetch<unsigned char>(t, (int)x);
}

// NT = number of the 16 last-round lookups served by the texture.
template <int NT>
__global__ void __launch_bounds__(1024, 1) probe(const uint32_t* compact, cudaTextureObject_t tex, uint32_t iters,
                                                  uint32_t* sink) {
  extern __shared__ __align__(1024) char smem[];
  fill_tables(smem, compact);
  const uint32_t lb = (threadIdx.x & 31) * 4;
  uint32_t s0 = threadIdx.x, s1 = blockIdx.x, s2 = threadIdx.x * 7, s3 = ~threadIdx.x;
  for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 1; r < 10; r++) {
      const uint32_t t0 = lds_u32(smem, taddr<0>(s0, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s1, lb), kOffT1) ^
                          lds_u32(smem, taddr<2>(s2, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s3, lb), kOffT3) ^ r;
      const uint32_t t1 = lds_u32(smem, taddr<0>(s1, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s2, lb), kOffT1) ^
                          lds_u32(smem, taddr<2>(s3, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s0, lb), kOffT3) ^ r;
      const uint32_t t2 = lds_u32(smem, taddr<0>(s2, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s3, lb), kOffT1) ^
                          lds_u32(smem, taddr<2>(s0, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s1, lb), kOffT3) ^ r;
      const uint32_t t3 = lds_u32(smem, taddr<0>(s3, lb), kOffT0) ^ lds_u32(smem, taddr<1>(s0, lb), kOffT1) ^
                          lds_u32(smem, taddr<2>(s1, lb), kOffT2) ^ lds_u32(smem, taddr<3>(s2, lb), kOffT3) ^ r;
      s0 = t0; s1 = t1; s2 = t2; s3 = t3;
    }
    // round 10: lookup k (0..15) of word c = k/4, byte b = k%4 from s[(c+b)%4]
    uint32_t w[4] = {s0, s1, s2, s3};
    uint32_t o[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
      uint32_t acc = 0;
#pragma unroll
      for (int b = 3; b >= 0; b--) {
        const int k = c * 4 + b;
        const uint32_t src = w[(c + b) & 3];
        uint32_t v;
        if (k < NT) v = sx(tex, (src >> (8 * b)) & 0xFF);
        else {
          uint32_t a;
          if (b == 0) a = taddr<0>(src, lb);
          else if (b == 1) a = taddr<1>(src, lb);
          else if (b == 2) a = taddr<2>(src, lb);
          else a = taddr<3>(src, lb);
          v = lds_u32(smem, a, kOffS);
        }
        acc = acc * 256u + v;
      }
      o[c] = acc ^ (uint32_t)c;
    }
    s0 = o[0]; s1 = o[1]; s2 = o[2]; s3 = o[3];
  }
  if ((s0 ^ s1 ^ s2 ^ s3) == 0x12345678u) sink[0] = s0;
}

__global__ void build(uint32_t* out, unsigned char* sbox) {
  const int v = threadIdx.x;
  const uint8_t S = sbox_forward((uint8_t)v);
  for (int j = 0; j < 4; j++) {
    uint32_t te = 0;
    for (int r = 0; r < 4; r++) te |= (uint32_t)gf_mul(mix_coef(false, r, j), S) << (8 * r);
    out[j * 256 + v] = te;
  }
  out[1024 + v] = S;
  sbox[v] = S;
}

template <int NT>
double run(const uint32_t* d, cudaTextureObject_t tex, uint32_t* sink, int sms, uint32_t iters) {
  cudaFuncSetAttribute(probe<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  probe<NT><<<sms, 1024, kSmemBytes>>>(d, tex, 4, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<NT><<<sms, 1024, kSmemBytes>>>(d, tex, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double blocks = (double)sms * 1024 * iters;
  return blocks * 16 / (ms / 1e3) / 1e9;  // plaintext-equivalent GB/s
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *d, *sink;
  unsigned char* sb;
  cudaMalloc(&d, 1280 * 4);
  cudaMalloc(&sb, 256);
  cudaMalloc(&sink, 4);
  build<<<1, 256>>>(d, sb);
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = sb;
  rd.res.linear.desc = cudaCreateChannelDesc<unsigned char>();
  rd.res.linear.sizeInBytes = 256;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  const uint32_t iters = 256;
  for (int rep = 0; rep < 2; rep++) {
    printf("S via TEX  0/16: %.1f GB/s-equivalent\n", run<0>(d, tex, sink, sms, iters));
    printf("S via TEX  2/16: %.1f\n", run<2>(d, tex, sink, sms, iters));
    printf("S via TEX  4/16: %.1f\n", run<4>(d, tex, sink, sms, iters));
    printf("S via TEX  8/16: %.1f\n", run<8>(d, tex, sink, sms, iters));
    printf("S via TEX 16/16: %.1f\n", run<16>(d, tex, sink, sms, iters));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
