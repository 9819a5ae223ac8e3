// cluster_probe.cu — can a cooperative (grid-sync) launch carry 16-CTA
// clusters, how many are co-resident, and what do a cluster barrier and a
// DSMEM gather + RED cost per step?  Diagnostics for the cluster-resident
// top-down pass (csrc/cluster_pass.cu).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cp tools/cluster_probe.cu && /tmp/cp
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;
typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ u32 mapa(u32 a, u32 rank) {
  u32 r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void red_add(u32 a, u64 v) {
  asm volatile("red.relaxed.cluster.shared::cluster.add.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void red_or(u32 a, u64 v) {
  asm volatile("red.relaxed.cluster.shared::cluster.or.b64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void ld2(u32 a, u64& x, u64& y) {
  asm volatile("ld.shared::cluster.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void cluster_bar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ u64 gtimer() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

extern __shared__ __align__(16) u64 rows[];

__global__ void k_probe(int steps, int mode, u32 nrows, u32 cs, u64* out, u64* t) {
  cg::grid_group grid = cg::this_grid();
  cg::cluster_group cl = cg::this_cluster();
  const u32 rank = cl.block_rank();
  for (u32 i = threadIdx.x; i < 2 * nrows; i += blockDim.x) rows[i] = 0;
  cl.sync();
  grid.sync();
  const u64 t0 = gtimer();
  const u32 base = (u32)__cvta_generic_to_shared(rows);
  u32 h = threadIdx.x * 2654435761u + rank * 40503u;
  u64 acc = 0;
  for (int s = 0; s < steps; s++) {
    if (mode >= 1) {  // DSMEM gather and / or REDs per thread per step
      h = h * 1664525u + 1013904223u;
      const u32 r = (h >> 8) % (nrows * cs);
      u64 x = 0, y = 0;
      if (mode != 4 && mode != 5 && mode != 7) ld2(mapa(base + (r / cs) * 16, r % cs), x, y);
      acc += x | y;
      const u32 d = (h >> 3) % (nrows * cs);
      const u32 a = mapa(base + (d / cs) * 16, d % cs);
      if (mode <= 2 || mode == 4) red_add(a, 1 + (acc & 1));
      if (mode <= 2 || mode == 5) red_or(a + 8, 1ull << (s & 63));
      if (mode == 6 || mode == 7)
        asm volatile("red.relaxed.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(a), "r"((u32)(1 + (acc & 1))) : "memory");
    }
    if (mode == 2) grid.sync();
    else cluster_bar();
  }
  const u64 t1 = gtimer();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    t[0] = t1 - t0;
  }
  if (acc == 0x1234567) out[0] = acc;
}

int main() {
  int dev = 0;
  cudaSetDevice(dev);
  const int block = 1024;
  const u32 nrows = 5300;  // ~84k heads / 16 CTAs
  const size_t smem = (size_t)nrows * 16;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  u64 *out, *t;
  cudaMalloc(&out, 64);
  cudaMalloc(&t, 64);
  for (int cs : {16, 8, 4}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cfg.gridDim = dim3(cs);
    int nclus = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclus, k_probe, &cfg);
    printf("cluster %d: max active clusters %d (%s)\n", cs, nclus, cudaGetErrorString(e));
    if (nclus < 1) continue;
    cfg.gridDim = dim3(cs * nclus);
    for (int mode : {0, 1, 2, 3, 4, 5, 6, 7}) {
      const int steps = 200;
      e = cudaLaunchKernelEx(&cfg, k_probe, steps, mode, nrows, (u32)cs, out, t);
      cudaError_t e2 = cudaDeviceSynchronize();
      u64 ht = 0;
      cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
      printf("  grid %d CTAs, mode %d (%s): %s / %s  %.3f us per step\n", cs * nclus, mode,
             mode == 0 ? "cluster barrier" : mode == 1 ? "gather + 2 RED + cluster barrier" : mode == 2 ? "gather + 2 RED + grid.sync" : mode == 3 ? "gather only" : mode == 4 ? "RED add.u64 only" : mode == 5 ? "RED or.b64 only" : mode == 6 ? "gather + RED add.u32" : "RED add.u32 only",
             cudaGetErrorString(e), cudaGetErrorString(e2), ht / 1e3 / steps);
    }
  }
  return 0;
}
