// api_cost.cu — host-side cost of the CUDA runtime calls the loader makes
// (diagnostics: gt_open on small grammars is bound by host enqueue time).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/api tools/api_cost.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <thread>

__global__ void k_empty(int* p) {
  if (p && threadIdx.x == 1234567) *p = 0;
}

template <class F>
static double per_call_us(int n, F f) {
  auto a = std::chrono::steady_clock::now();
  for (int i = 0; i < n; i++) f(i);
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count() / n;
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  k_empty<<<1, 32, 0, st>>>(nullptr);
  cudaStreamSynchronize(st);
  const int N = 2000;
  printf("launch (1 block):            %.2f us\n", per_call_us(N, [&](int) { k_empty<<<1, 32, 0, st>>>(nullptr); }));
  cudaStreamSynchronize(st);
  printf("launch (2368x256):           %.2f us\n",
         per_call_us(N, [&](int) { k_empty<<<2368, 256, 0, st>>>(nullptr); }));
  cudaStreamSynchronize(st);
  printf("mallocAsync+freeAsync 1MB:   %.2f us\n", per_call_us(N, [&](int) {
           void* p;
           cudaMallocAsync(&p, 1 << 20, st);
           cudaFreeAsync(p, st);
         }));
  cudaStreamSynchronize(st);
  void* d;
  cudaMalloc(&d, 1 << 20);
  printf("memsetAsync 1MB:             %.2f us\n", per_call_us(N, [&](int) { cudaMemsetAsync(d, 0, 1 << 20, st); }));
  cudaStreamSynchronize(st);
  printf("memcpyAsync D2D 4B:          %.2f us\n", per_call_us(N, [&](int) { cudaMemcpyAsync(d, (char*)d + 64, 4, cudaMemcpyDeviceToDevice, st); }));
  cudaStreamSynchronize(st);
  int* h;
  cudaMallocHost(&h, 64);
  printf("d2h 8B + streamSync:         %.2f us\n", per_call_us(500, [&](int) {
           cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, st);
           cudaStreamSynchronize(st);
         }));
  printf("launch + streamSync:         %.2f us\n", per_call_us(500, [&](int) {
           k_empty<<<1, 32, 0, st>>>(nullptr);
           cudaStreamSynchronize(st);
         }));
  printf("streamCreate+Destroy:        %.2f us\n", per_call_us(200, [&](int) {
           cudaStream_t s;
           cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
           cudaStreamDestroy(s);
         }));
  printf("eventCreate+Record+Destroy:  %.2f us\n", per_call_us(N, [&](int) {
           cudaEvent_t e;
           cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
           cudaEventRecord(e, st);
           cudaEventDestroy(e);
         }));
  printf("std::thread create+join:     %.2f us\n", per_call_us(200, [&](int) {
           std::thread t([] {});
           t.join();
         }));
  printf("cudaGetDevice+Attribute:     %.2f us\n", per_call_us(N, [&](int) {
           int dev, v;
           cudaGetDevice(&dev);
           cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
         }));
  printf("cudaMemGetInfo:              %.2f us\n", per_call_us(200, [&](int) {
           size_t a, b;
           cudaMemGetInfo(&a, &b);
         }));
  return 0;
}
