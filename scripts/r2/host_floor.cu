// Host-call floor of the drop-in path, from C (no Python): what one
// gaes_cbc_encrypt_std / gaes_encrypt_shared_iv call on pageable buffers
// costs end to end for N = 1 .. 65536 blocks, beside the floors of any GPU
// round trip (an empty kernel + stream sync, a small H2D + sync) and of the
// runtime queries the call makes.
//
//   nvcc -O3 -std=c++17 -I include scripts/r2/host_floor.cu -o /tmp/host_floor \
//        -L paper_1506_08503_b200 -l:libgaes_b200.so -Xlinker -rpath=$PWD/paper_1506_08503_b200
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <vector>

#include "gaes_b200.h"

__global__ void k_nop() {}

// data arriving inside the launch (large kernel parameters, <= 32764 bytes)
struct Big {
  uint32_t n;
  uint4 d[1000];
};
__global__ void k_param_copy(const __grid_constant__ Big p, uint4* out) {
  for (uint32_t i = threadIdx.x + blockIdx.x * blockDim.x; i < p.n; i += gridDim.x * blockDim.x) out[i] = p.d[i];
}
__global__ void k_host_copy(const uint4* in, uint4* out, uint32_t n) {
  for (uint32_t i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i];
}

static double time_us(const std::function<void()>& f, int reps = 2000) {
  for (int i = 0; i < 200; i++) f();
  std::vector<double> ts;
  for (int r = 0; r < 5; r++) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps / 5; i++) f();
    ts.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / (reps / 5));
  }
  std::sort(ts.begin(), ts.end());
  return ts[2];
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  void* d;
  cudaMalloc(&d, 1 << 20);
  std::vector<uint8_t> h(1 << 20, 1), o(1 << 20);
  printf("empty kernel launch + cudaStreamSynchronize: %.2f us\n", time_us([&] {
           k_nop<<<1, 32, 0, s>>>();
           cudaStreamSynchronize(s);
         }));
  uint8_t* hp;
  cudaMallocHost(&hp, 1 << 20);
  printf("16 KiB H2D from pinned + sync: %.2f us\n", time_us([&] {
           cudaMemcpyAsync(d, hp, 16384, cudaMemcpyHostToDevice, s);
           cudaStreamSynchronize(s);
         }));
  printf("16 KiB H2D + D2H pinned + sync: %.2f us\n", time_us([&] {
           cudaMemcpyAsync(d, hp, 16384, cudaMemcpyHostToDevice, s);
           cudaMemcpyAsync(hp, d, 16384, cudaMemcpyDeviceToHost, s);
           cudaStreamSynchronize(s);
         }));
  {
    static Big big;
    big.n = 1000;
    uint8_t *hin, *hout;
    cudaMallocHost(&hin, 16000);
    cudaMallocHost(&hout, 16000);
    uint4 *din, *dout;
    cudaHostGetDevicePointer((void**)&din, hin, 0);
    cudaHostGetDevicePointer((void**)&dout, hout, 0);
    printf("kernel copies 16 KB pinned->pinned (zero-copy) + sync: %.2f us\n", time_us([&] {
             k_host_copy<<<8, 128, 0, s>>>(din, dout, 1000);
             cudaStreamSynchronize(s);
           }));
    printf("kernel copies 16 KB from its parameters -> pinned + sync: %.2f us\n", time_us([&] {
             k_param_copy<<<8, 128, 0, s>>>(big, dout);
             cudaStreamSynchronize(s);
           }));
    printf("memcpy 16 KB into the param struct + the same: %.2f us\n", time_us([&] {
             memcpy(big.d, h.data(), 16000);
             k_param_copy<<<8, 128, 0, s>>>(big, dout);
             cudaStreamSynchronize(s);
           }));
    printf("kernel writes 16 KB to pinned from device + sync: %.2f us\n", time_us([&] {
             k_host_copy<<<8, 128, 0, s>>>((const uint4*)d, dout, 1000);
             cudaStreamSynchronize(s);
           }));
    printf("kernel reads 16 KB pinned -> device + sync: %.2f us\n", time_us([&] {
             k_host_copy<<<8, 128, 0, s>>>(din, (uint4*)d, 1000);
             cudaStreamSynchronize(s);
           }));
  }
  cudaPointerAttributes a;
  printf("cudaPointerGetAttributes (pageable): %.3f us\n",
         time_us([&] { cudaPointerGetAttributes(&a, h.data()); }, 20000));
  int dev;
  printf("cudaGetDevice: %.3f us\n", time_us([&] { cudaGetDevice(&dev); }, 20000));
  uint8_t rk[176] = {0}, iv[16] = {0};
  std::vector<uint8_t> ivs((size_t)16 << 16, 7);
  for (size_t n : {1, 10, 100, 1000, 10000, 65536}) {
    const double t = time_us([&] {
      int rc = gaes_cbc_encrypt_std(h.data(), ivs.data(), n, 16, rk, o.data());
      if (rc) {
        printf("error %s\n", gaes_last_error());
        exit(1);
      }
    }, n > 10000 ? 500 : 2000);
    const double t2 = time_us([&] { gaes_encrypt_shared_iv(h.data(), n, 16, iv, rk, o.data()); },
                              n > 10000 ? 500 : 2000);
    printf("N=%6zu pageable: gaes_cbc_encrypt_std %.2f us (%s), gaes_encrypt_shared_iv %.2f us\n", n, t,
           gaes_last_kernel(), t2);
  }
  return 0;
}
