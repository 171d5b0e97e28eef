// Small-batch (config 1, 2^16 blocks) cost decomposition on the GPU box.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1506_08503_b200/csrc \
//        scripts/r2/small_probe.cu -o /tmp/small_probe -L paper_1506_08503_b200 -lgaes_b200 \
//        -Xlinker -rpath=$PWD/paper_1506_08503_b200 && /tmp/small_probe
//
// Per variant: CUDA events around one launch after a 512 MiB L2 flush (the
// bench discipline), the same in a CUDA graph (flush+step graph minus
// flush-only graph), and back to back without a flush.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <functional>
#include <vector>

#include "aes_ttable.cuh"
#include "gaes_b200.h"

using namespace gaes;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void k_flush(uint4* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, v, v, v);
}
__global__ void k_empty() {}
__global__ void __launch_bounds__(1024, 1) k_empty_smem() {
  extern __shared__ char smem[];
  if (threadIdx.x == 1025) smem[0] = 1;
}
__global__ void __launch_bounds__(1024, 1) k_fill_only(const uint32_t* compact, uint32_t* sink) {
  extern __shared__ __align__(1024) char smem[];
  fill_tables(smem, compact, false);
  if (threadIdx.x == 0 && smem[5] == 123) sink[0] = 1;
}

// Fill variants: T tables built from T0 passed in the kernel parameters
// (constant bank; no global round trip), T_j = rotl(T0, 8j).
struct FillParams {
  uint32_t t0[256];
};
__device__ __forceinline__ void fill_from_params(char* smem, const FillParams& fp) {
  const int words = 4 * 256 * 8;
  for (int q = threadIdx.x; q < words; q += blockDim.x) {
    const int quad = q & 7, x = (q >> 3) & 255, tbl = q >> 11;
    const uint32_t t = fp.t0[x];
    const uint32_t v = __funnelshift_l(t, t, 8 * tbl);
    *reinterpret_cast<uint4*>(smem + (tbl >> 1) * kRegionBytes + x * 256 + (tbl & 1) * 128 + quad * 16) =
        make_uint4(v, v, v, v);
  }
  __syncthreads();
}
__global__ void __launch_bounds__(1024, 1) k_fill_params(const __grid_constant__ FillParams fp, uint32_t* sink) {
  extern __shared__ __align__(1024) char smem[];
  fill_from_params(smem, fp);
  if (threadIdx.x == 0 && smem[5] == 123) sink[0] = 1;
}
__global__ void __launch_bounds__(1024, 1) k_fill_const(uint32_t* sink) {
  extern __shared__ __align__(1024) char smem[];
  for (int q = threadIdx.x; q < 4 * 256 * 8; q += blockDim.x)
    *reinterpret_cast<uint4*>(smem + (q >> 11 >> 1) * kRegionBytes + ((q >> 3) & 255) * 256 + ((q >> 11) & 1) * 128 +
                              (q & 7) * 16) = make_uint4(q, q, q, q);
  __syncthreads();
  if (threadIdx.x == 0 && smem[5] == 123) sink[0] = 1;
}
// k_blocks' single-pass path with the parameter fill
__global__ void __launch_bounds__(1024, 1) k_enc_pfill(const uint4* __restrict__ in, uint4* __restrict__ out,
                                                       uint64_t n, const __grid_constant__ FillParams fp,
                                                       const __grid_constant__ RoundKeys rk, cudaTextureObject_t tsb) {
  extern __shared__ __align__(1024) char smem[];
  if ((uint64_t)blockIdx.x * 32 >= n) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  uint64_t b = ((uint64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + lane;
  uint4 cur = make_uint4(0, 0, 0, 0);
  if (b < n) cur = __ldcs(in + b);
  fill_from_params(smem, fp);
  for (; b < n; b += T) {
    uint32_t s0 = cur.x ^ rk.w[0], s1 = cur.y ^ rk.w[1], s2 = cur.z ^ rk.w[2], s3 = cur.w ^ rk.w[3];
    const uint64_t nb = b + T;
    if (nb < n) cur = __ldcs(in + nb);
    encrypt_rounds(smem, lane * 4, s0, s1, s2, s3, rk, tsb);
    __stcs(out + b, make_uint4(s0, s1, s2, s3));
  }
}

// T0 only, filled from the kernel parameters (32 KiB of STS)
__global__ void __launch_bounds__(1024, 1) k_t0p(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                                                 const __grid_constant__ FillParams fp,
                                                 const __grid_constant__ RoundKeys rk, cudaTextureObject_t tsb) {
  extern __shared__ __align__(1024) char smem[];
  if ((uint64_t)blockIdx.x * 32 >= n) return;
  const uint32_t lane = threadIdx.x & 31;
  uint64_t b = ((uint64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + lane;
  uint4 cur = make_uint4(0, 0, 0, 0);
  if (b < n) cur = __ldcs(in + b);
  for (int q = threadIdx.x; q < 256 * 8; q += blockDim.x) {
    const uint32_t v = fp.t0[q >> 3];
    *reinterpret_cast<uint4*>(smem + (q >> 3) * 128 + (q & 7) * 16) = make_uint4(v, v, v, v);
  }
  __syncthreads();
  if (b >= n) return;
  const uint32_t lb = lane * 4;
  uint32_t s0 = cur.x ^ rk.w[0], s1 = cur.y ^ rk.w[1], s2 = cur.z ^ rk.w[2], s3 = cur.w ^ rk.w[3];
  auto T = [&](uint32_t s, int k) {
    const uint32_t a = __byte_perm(s, 0, 0x4440 | k) * 128 + lb;
    return *reinterpret_cast<const uint32_t*>(smem + a);
  };
#pragma unroll
  for (int r = 1; r < 10; r++) {
    const uint32_t t0 = T(s0, 0) ^ __funnelshift_l(T(s1, 1), T(s1, 1), 8) ^ __funnelshift_l(T(s2, 2), T(s2, 2), 16) ^
                        __funnelshift_l(T(s3, 3), T(s3, 3), 24) ^ rk.w[4 * r + 0];
    const uint32_t t1 = T(s1, 0) ^ __funnelshift_l(T(s2, 1), T(s2, 1), 8) ^ __funnelshift_l(T(s3, 2), T(s3, 2), 16) ^
                        __funnelshift_l(T(s0, 3), T(s0, 3), 24) ^ rk.w[4 * r + 1];
    const uint32_t t2 = T(s2, 0) ^ __funnelshift_l(T(s3, 1), T(s3, 1), 8) ^ __funnelshift_l(T(s0, 2), T(s0, 2), 16) ^
                        __funnelshift_l(T(s1, 3), T(s1, 3), 24) ^ rk.w[4 * r + 2];
    const uint32_t t3 = T(s3, 0) ^ __funnelshift_l(T(s0, 1), T(s0, 1), 8) ^ __funnelshift_l(T(s1, 2), T(s1, 2), 16) ^
                        __funnelshift_l(T(s2, 3), T(s2, 3), 24) ^ rk.w[4 * r + 3];
    s0 = t0; s1 = t1; s2 = t2; s3 = t3;
  }
  auto S = [&](uint32_t x) { return (uint32_t)tex1Dfetch<unsigned char>(tsb, (int)x); };
  auto last = [&](uint32_t a, uint32_t bb, uint32_t c, uint32_t d) {
    return S(a & 0xFF) | (S((bb >> 8) & 0xFF) << 8) | (S((c >> 16) & 0xFF) << 16) | (S(d >> 24) << 24);
  };
  const uint32_t o0 = last(s0, s1, s2, s3) ^ rk.w[40], o1 = last(s1, s2, s3, s0) ^ rk.w[41];
  const uint32_t o2 = last(s2, s3, s0, s1) ^ rk.w[42], o3 = last(s3, s0, s1, s2) ^ rk.w[43];
  __stcs(out + b, make_uint4(o0, o1, o2, o3));
}

// T0 only (32 KiB, 32 copies), T_j = rotl(T0, 8j); round 10 from the S-box texture.
__global__ void __launch_bounds__(1024, 1) k_t0(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n,
                                                const uint32_t* __restrict__ compact,
                                                const __grid_constant__ RoundKeys rk, cudaTextureObject_t tsb) {
  extern __shared__ __align__(1024) char smem[];
  if ((uint64_t)blockIdx.x * 32 >= n) return;
  const uint32_t lane = threadIdx.x & 31;
  uint64_t b = ((uint64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + lane;
  uint4 cur = make_uint4(0, 0, 0, 0);
  if (b < n) cur = __ldcs(in + b);
  // fill: entry x at 128 x, 32 copies
  for (int q = threadIdx.x; q < 256 * 8; q += blockDim.x) {
    const uint32_t v = __ldg(compact + (q >> 3));
    *reinterpret_cast<uint4*>(smem + (q >> 3) * 128 + (q & 7) * 16) = make_uint4(v, v, v, v);
  }
  __syncthreads();
  if (b >= n) return;
  const uint32_t lb = lane * 4;
  uint32_t s0 = cur.x ^ rk.w[0], s1 = cur.y ^ rk.w[1], s2 = cur.z ^ rk.w[2], s3 = cur.w ^ rk.w[3];
  auto T = [&](uint32_t s, int k) {
    const uint32_t byte = (s >> (8 * k)) & 0xFF;
    return *reinterpret_cast<const uint32_t*>(smem + byte * 128 + lb);
  };
#pragma unroll
  for (int r = 1; r < 10; r++) {
    const uint32_t t0 = T(s0, 0) ^ __funnelshift_l(T(s1, 1), T(s1, 1), 8) ^ __funnelshift_l(T(s2, 2), T(s2, 2), 16) ^
                        __funnelshift_l(T(s3, 3), T(s3, 3), 24) ^ rk.w[4 * r + 0];
    const uint32_t t1 = T(s1, 0) ^ __funnelshift_l(T(s2, 1), T(s2, 1), 8) ^ __funnelshift_l(T(s3, 2), T(s3, 2), 16) ^
                        __funnelshift_l(T(s0, 3), T(s0, 3), 24) ^ rk.w[4 * r + 1];
    const uint32_t t2 = T(s2, 0) ^ __funnelshift_l(T(s3, 1), T(s3, 1), 8) ^ __funnelshift_l(T(s0, 2), T(s0, 2), 16) ^
                        __funnelshift_l(T(s1, 3), T(s1, 3), 24) ^ rk.w[4 * r + 2];
    const uint32_t t3 = T(s3, 0) ^ __funnelshift_l(T(s0, 1), T(s0, 1), 8) ^ __funnelshift_l(T(s1, 2), T(s1, 2), 16) ^
                        __funnelshift_l(T(s2, 3), T(s2, 3), 24) ^ rk.w[4 * r + 3];
    s0 = t0; s1 = t1; s2 = t2; s3 = t3;
  }
  auto S = [&](uint32_t x) { return (uint32_t)tex1Dfetch<unsigned char>(tsb, (int)x); };
  auto last = [&](uint32_t a, uint32_t bb, uint32_t c, uint32_t d) {
    return S(a & 0xFF) | (S((bb >> 8) & 0xFF) << 8) | (S((c >> 16) & 0xFF) << 16) | (S(d >> 24) << 24);
  };
  const uint32_t o0 = last(s0, s1, s2, s3) ^ rk.w[40], o1 = last(s1, s2, s3, s0) ^ rk.w[41];
  const uint32_t o2 = last(s2, s3, s0, s1) ^ rk.w[42], o3 = last(s3, s0, s1, s2) ^ rk.w[43];
  __stcs(out + b, make_uint4(o0, o1, o2, o3));
}

int main() {
  const size_t n = 1 << 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint4 *flush, *in, *out, *out2;
  const size_t fl = (512u << 20) / 16;
  CK(cudaMalloc(&flush, fl * 16));
  CK(cudaMalloc(&in, n * 16));
  CK(cudaMalloc(&out, n * 16));
  CK(cudaMalloc(&out2, n * 16));
  CK(cudaMemset(in, 7, n * 16));
  uint8_t rk[176], iv[16] = {0}, sbox[256], inv[256];
  uint32_t te[1024], td[1024];
  for (int i = 0; i < 176; i++) rk[i] = (uint8_t)(i * 7);
  if (gaes_gf_tables(0, sbox, inv, te, td) != 0) {
    printf("gf tables: %s\n", gaes_last_error());
    return 1;
  }
  uint32_t* compact;
  uint32_t* sink;
  uint8_t* d_s;
  CK(cudaMalloc(&compact, 5 * 1024));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&d_s, 256));
  std::vector<uint32_t> comp(1280);
  for (int i = 0; i < 1024; i++) comp[i] = te[i];
  for (int i = 0; i < 256; i++) comp[1024 + i] = sbox[i];
  CK(cudaMemcpy(compact, comp.data(), 5 * 1024, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_s, sbox, 256, cudaMemcpyHostToDevice));
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = d_s;
  rd.res.linear.desc = cudaCreateChannelDesc<unsigned char>();
  rd.res.linear.sizeInBytes = 256;
  cudaTextureDesc td_ = {};
  td_.readMode = cudaReadModeElementType;
  cudaTextureObject_t tsb;
  CK(cudaCreateTextureObject(&tsb, &rd, &td_, nullptr));
  CK(cudaFuncSetAttribute(k_empty_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  CK(cudaFuncSetAttribute(k_fill_only, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  CK(cudaFuncSetAttribute(k_t0, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
  CK(cudaFuncSetAttribute(k_t0p, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
  CK(cudaFuncSetAttribute(k_fill_params, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  CK(cudaFuncSetAttribute(k_fill_const, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  CK(cudaFuncSetAttribute(k_enc_pfill, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
  FillParams fp;
  for (int i = 0; i < 256; i++) fp.t0[i] = te[i];
  uint4* out3;
  CK(cudaMalloc(&out3, n * 16));
  RoundKeys k = {};
  for (int i = 0; i < 44; i++) k.w[i] = rk[4 * i] | (rk[4 * i + 1] << 8) | (rk[4 * i + 2] << 16) | ((uint32_t)rk[4 * i + 3] << 24);

  auto do_flush = [&](int i) { k_flush<<<sms * 4, 1024, 0, s>>>(flush, fl, i); };
  const int grid = (int)std::min<size_t>(sms, (n + 31) / 32);
  std::vector<std::pair<const char*, std::function<void()>>> variants = {
      {"empty kernel 148x1024, no smem", [&] { k_empty<<<sms, 1024, 0, s>>>(); }},
      {"empty kernel 148x1024, 192 KiB dyn smem", [&] { k_empty_smem<<<sms, 1024, kSmemBytes, s>>>(); }},
      {"table fill only (128 KiB)", [&] { k_fill_only<<<sms, 1024, kSmemBytes, s>>>(compact, sink); }},
      {"library gaes_encrypt_blocks_dev 2^16",
       [&] {
         if (gaes_encrypt_blocks_dev(in, out, n, rk, iv, s)) printf("err %s\n", gaes_last_error());
       }},
      {"T0-only 32 KiB kernel 2^16", [&] { k_t0<<<grid, 1024, 32768, s>>>(in, out2, n, compact, k, tsb); }},
      {"fill from kernel params (128 KiB)", [&] { k_fill_params<<<sms, 1024, kSmemBytes, s>>>(fp, sink); }},
      {"fill constants only (128 KiB)", [&] { k_fill_const<<<sms, 1024, kSmemBytes, s>>>(sink); }},
      {"encrypt 2^16, param fill", [&] { k_enc_pfill<<<grid, 1024, kSmemBytes, s>>>(in, out3, n, fp, k, tsb); }},
      {"T0-only, param fill, 2^16", [&] { k_t0p<<<grid, 1024, 32768, s>>>(in, out2, n, fp, k, tsb); }},
  };
  const int R = 50;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  std::vector<cudaEvent_t> ea(R), eb(R);
  for (int i = 0; i < R; i++) {
    CK(cudaEventCreate(&ea[i]));
    CK(cudaEventCreate(&eb[i]));
  }
  for (auto& v : variants) {
    for (int w = 0; w < 5; w++) v.second();
    CK(cudaStreamSynchronize(s));
    // 1. events per step after flush
    for (int i = 0; i < R; i++) {
      do_flush(i);
      CK(cudaEventRecord(ea[i], s));
      v.second();
      CK(cudaEventRecord(eb[i], s));
    }
    CK(cudaStreamSynchronize(s));
    float tot = 0, mn = 1e9;
    for (int i = 0; i < R; i++) {
      float t;
      CK(cudaEventElapsedTime(&t, ea[i], eb[i]));
      tot += t;
      mn = std::min(mn, t);
    }
    // 2. graphs
    auto graph_us = [&](bool with_step, bool with_flush) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < R; i++) {
        if (with_flush) do_flush(i);
        if (with_step) v.second();
      }
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaStreamSynchronize(s));
      CK(cudaEventRecord(a, s));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(b, s));
      CK(cudaStreamSynchronize(s));
      float t;
      CK(cudaEventElapsedTime(&t, a, b));
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
      return t * 1e3f / R;
    };
    const float g_both = graph_us(true, true), g_fl = graph_us(false, true), g_b2b = graph_us(true, false);
    // 3. back to back, stream launches
    CK(cudaEventRecord(a, s));
    for (int i = 0; i < R; i++) v.second();
    CK(cudaEventRecord(b, s));
    CK(cudaStreamSynchronize(s));
    float tb;
    CK(cudaEventElapsedTime(&tb, a, b));
    printf("%-44s events after flush: mean %6.2f us min %6.2f | graph after flush %6.2f | graph b2b %6.2f | stream b2b %6.2f\n",
           v.first, tot * 1e3f / R, mn * 1e3f, g_both - g_fl, g_b2b, tb * 1e3f / R);
  }
  // ring of 256 cold 1 MiB batches (inputs + outputs 512 MiB > L2), steps
  // back to back in one graph: the bench's "inputs larger than L2" discipline
  {
    const int RING = 256;
    uint4 *rin, *rout;
    CK(cudaMalloc(&rin, RING * n * 16));
    CK(cudaMalloc(&rout, RING * n * 16));
    CK(cudaMemset(rin, 3, RING * n * 16));
    std::vector<std::pair<const char*, std::function<void(int)>>> rv = {
        {"library (k_blocks, PDL)", [&](int i) { gaes_encrypt_blocks_dev(rin + (size_t)i * n, rout + (size_t)i * n, n, rk, iv, s); }},
        {"param fill, full tables", [&](int i) { k_enc_pfill<<<grid, 1024, kSmemBytes, s>>>(rin + (size_t)i * n, rout + (size_t)i * n, n, fp, k, tsb); }},
        {"T0-only param fill", [&](int i) { k_t0p<<<grid, 1024, 32768, s>>>(rin + (size_t)i * n, rout + (size_t)i * n, n, fp, k, tsb); }},
    };
    for (auto& v : rv) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < RING; i++) v.second(i);
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaStreamSynchronize(s));
      CK(cudaEventRecord(a, s));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(b, s));
      CK(cudaStreamSynchronize(s));
      float tg;
      CK(cudaEventElapsedTime(&tg, a, b));
      // the same steps as stream launches
      CK(cudaEventRecord(a, s));
      for (int i = 0; i < RING; i++) v.second(i);
      CK(cudaEventRecord(b, s));
      CK(cudaStreamSynchronize(s));
      float ts;
      CK(cudaEventElapsedTime(&ts, a, b));
      printf("ring of %d cold batches, %-28s graph %6.2f us/step (%5.0f GB/s) | stream %6.2f us/step\n", RING, v.first,
             tg * 1e3f / RING, n * 16 / (tg * 1e3f / RING) / 1e3, ts * 1e3f / RING);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  // correctness of the T0 kernel vs the library
  std::vector<uint8_t> h1(n * 16), h2(n * 16);
  CK(cudaMemcpy(h1.data(), out, n * 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), out2, n * 16, cudaMemcpyDeviceToHost));
  printf("T0-only kernel == library: %s\n", h1 == h2 ? "yes" : "NO");
  CK(cudaMemcpy(h2.data(), out3, n * 16, cudaMemcpyDeviceToHost));
  printf("param-fill kernel == library: %s\n", h1 == h2 ? "yes" : "NO");
  k_t0p<<<grid, 1024, 32768, s>>>(in, out2, n, fp, k, tsb);
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(h2.data(), out2, n * 16, cudaMemcpyDeviceToHost));
  printf("T0 param-fill kernel == library: %s\n", h1 == h2 ? "yes" : "NO");
  return 0;
}
