// Launch overhead vs table fill: back-to-back launches of 148 x 1024-thread
// CTAs with 192 KiB dynamic smem, (a) empty, (b) with the table fill.
#include <cstdio>
#include <cuda_runtime.h>
#include "aes_ttable.cuh"
using namespace gaes;
__global__ void __launch_bounds__(1024, 1) empty_k(int* sink) {
  extern __shared__ __align__(1024) char smem[];
  if (threadIdx.x == 9999) sink[0] = smem[0];
}
__global__ void __launch_bounds__(1024, 1) fill_k(const uint32_t* compact, int* sink) {
  extern __shared__ __align__(1024) char smem[];
  fill_tables(smem, compact);
  if (threadIdx.x == 9999) sink[0] = smem[0];
}
__global__ void small_k(int* sink) { if (threadIdx.x == 9999) sink[0] = 1; }
__global__ void __launch_bounds__(256, 1) fill256_k(const uint32_t* compact, int* sink) {
  extern __shared__ __align__(1024) char smem[];
  fill_tables(smem, compact);
  if (threadIdx.x == 9999) sink[0] = smem[0];
}
// GPU-side cost per launch: 200 launches captured in a CUDA graph, replayed
// (host enqueue rate out of the picture).
template <typename F>
float timeit_graph(F f) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 200; i++) f(s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 200 * 1e3;
}
template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < 200; i++) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 200 * 1e3;
}
int main() {
  int *sink; uint32_t* tab;
  cudaMalloc(&sink, 4); cudaMalloc(&tab, 1280 * 4); cudaMemset(tab, 1, 1280 * 4);
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  cudaFuncSetAttribute(fill_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  printf("small kernel (1 CTA x 32):           %.2f us\n", timeit([&] { small_k<<<1, 32>>>(sink); }));
  printf("148 x 1024 thr, no smem:              %.2f us\n", timeit([&] { empty_k<<<148, 1024, 0>>>(sink); }));
  printf("148 x 1024 thr, 192 KiB smem, empty:  %.2f us\n", timeit([&] { empty_k<<<148, 1024, kSmemBytes>>>(sink); }));
  printf("148 x 1024 thr, 192 KiB smem, fill:   %.2f us\n", timeit([&] { fill_k<<<148, 1024, kSmemBytes>>>(tab, sink); }));
  printf("64 x 1024 thr, 192 KiB smem, fill:    %.2f us\n", timeit([&] { fill_k<<<64, 1024, kSmemBytes>>>(tab, sink); }));
  cudaFuncSetAttribute(fill256_k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  printf("148 x 256 thr, 192 KiB smem, fill:    %.2f us\n", timeit([&] { fill256_k<<<148, 256, kSmemBytes>>>(tab, sink); }));
  printf("148 x 256 thr, no smem, empty:        %.2f us\n", timeit([&] { empty_k<<<148, 256, 0>>>(sink); }));
  printf("graph: small kernel (1 CTA x 32):           %.2f us\n", timeit_graph([&](cudaStream_t s) { small_k<<<1, 32, 0, s>>>(sink); }));
  printf("graph: 148 x 1024 thr, 192 KiB smem, empty:  %.2f us\n", timeit_graph([&](cudaStream_t s) { empty_k<<<148, 1024, kSmemBytes, s>>>(sink); }));
  printf("graph: 148 x 1024 thr, 192 KiB smem, fill:   %.2f us\n", timeit_graph([&](cudaStream_t s) { fill_k<<<148, 1024, kSmemBytes, s>>>(tab, sink); }));
  printf("graph: 148 x 256 thr, 192 KiB smem, fill:    %.2f us\n", timeit_graph([&](cudaStream_t s) { fill256_k<<<148, 256, kSmemBytes, s>>>(tab, sink); }));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
