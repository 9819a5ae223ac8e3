// barrier_probe.cu — per-level cost floor of a persistent level loop on B200.
//
// Measures, for L levels in one launch: (a) cooperative-groups grid.sync
// alone, (b) a monotonic-counter barrier (one red.release per block, acquire
// spin), (c) either barrier plus the dependent chain a level carries in the
// top-down pass (item load -> row gather through L2 -> RED), to separate the
// barrier from the work latency.  Diagnostics only (not part of the library).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bp tools/barrier_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;
typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ void bar_mono(u32* ctr, u32 target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    u32 v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// mode 0: cg barrier only; 1: mono barrier only; 2: cg + chain; 3: mono + chain
template <int MODE>
__global__ void k_levels(int L, u32* ctr, const u32* items, const u64* rows, u64* out, u32 n_per_level) {
  cg::grid_group grid = cg::this_grid();
  const u32 gtid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int l = 0; l < L; l++) {
    if (MODE >= 2 && gtid < n_per_level) {
      const u32 it = items[(u64)l * n_per_level + gtid];
      u64 v;
      asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(rows + it));
      atomicAdd(out + (it ^ 1), v + 1);
    }
    if (MODE == 0 || MODE == 2) grid.sync();
    else bar_mono(ctr, (u32)gridDim.x * (l + 1));
  }
}

template <int MODE>
float run(int blocks, int threads, int L, u32 npl, u32* ctr, const u32* items, const u64* rows, u64* out) {
  auto kern = k_levels<MODE>;
  void* args[] = {&L, &ctr, &items, &rows, &out, &npl};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 50;
  float best = 1e30f;
  for (int w = 0; w < 3; w++) {
    cudaEventRecord(a);
    for (int r = 0; r < reps; r++) {
      cudaMemsetAsync(ctr, 0, 4);
      cudaLaunchCooperativeKernel((const void*)kern, blocks, threads, args, 0, 0);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return best * 1000.f / reps;  // us per launch
}

int main() {
  const int L = 24;
  const u32 npl = 46000;  // ~C2 edges per level
  const u64 nrows = 1u << 20;
  u32 *ctr, *items;
  u64 *rows, *out;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&items, (u64)L * npl * 4);
  cudaMalloc(&rows, nrows * 8);
  cudaMalloc(&out, nrows * 8);
  std::vector<u32> h((u64)L * npl);
  srand(1);
  for (auto& x : h) x = (u32)(((u64)rand() * 2654435761ull) % nrows);
  cudaMemcpy(items, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(rows, 1, nrows * 8);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int cfgs[][2] = {{1, 1024}, {1, 512}, {2, 512}, {1, 256}, {4, 256}};
  printf("L=%d levels, items/level %u (chain modes)\n", L, npl);
  for (auto& c : cfgs) {
    const int blocks = nsm * c[0], threads = c[1];
    const float empty = run<0>(blocks, threads, 0, npl, ctr, items, rows, out);
    const float t0 = run<0>(blocks, threads, L, npl, ctr, items, rows, out);
    const float t1 = run<1>(blocks, threads, L, npl, ctr, items, rows, out);
    const float t2 = run<2>(blocks, threads, L, npl, ctr, items, rows, out);
    const float t3 = run<3>(blocks, threads, L, npl, ctr, items, rows, out);
    printf("grid %4d x %4d: launch %.2f us | per level: cg %.2f us, mono %.2f us, cg+chain %.2f us, mono+chain %.2f us\n",
           blocks, threads, empty, (t0 - empty) / L, (t1 - empty) / L, (t2 - empty) / L, (t3 - empty) / L);
  }
  return 0;
}
