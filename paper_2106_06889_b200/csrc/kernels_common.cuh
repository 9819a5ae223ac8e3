// kernels_common.cuh — device helpers shared by the loader and the task kernels.
#pragma once

#include "gt_internal.cuh"

namespace gt {

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// off[r] = lower_bound(sorted_key, r) for r in [0, R]; sorted_key ascending.
__global__ void k_csr_offsets(const u32* sorted_key, u64 n, u64 R, u64* off);

__global__ void k_iota_u32(u32* out, u64 n);

// loader.cu kernels reused by the lazily built lists (contract.cu)
// out[i] = map[in[i]]; rank[order[i]] = i; cur = incl - degt
__global__ void k_map_u32(const u32* __restrict__ in, u64 n, const u32* __restrict__ map, u32* out);
__global__ void k_rank_of(const u32* __restrict__ order, u64 n, u32* rank);
__global__ void k_cursor(const u32* __restrict__ degt, const u32* __restrict__ incl, u64 n, u32* cur);
__global__ void k_unpack3_n(const U3* __restrict__ in, const u32* __restrict__ n_dev, u32* a, u32* b, u32* c);
__global__ void k_te_level_off(const u64* __restrict__ ls, const u32* __restrict__ incl,
                               const u32* __restrict__ degt, u64 R, u64 nl, u64* off);

// out[key[i]] += val(i) for keys sorted ascending, warp-aggregated atomics
// (at most one atomic per key run per warp).
template <class ValF>
__global__ void k_seg_sum_sorted(const u32* key, u64 n, ValF val, u64* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < n; base += stride) {
    u64 i = base + threadIdx.x;
    bool ok = i < n;
    u32 k = ok ? key[i] : 0xFFFFFFFFu;
    u64 v = ok ? val(i) : 0;
    unsigned lane = lane_id();
    // segmented inclusive scan (run = equal consecutive keys)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      u64 ov = __shfl_up_sync(0xFFFFFFFFu, v, d);
      u32 ok2 = __shfl_up_sync(0xFFFFFFFFu, k, d);
      if (lane >= (unsigned)d && ok2 == k) v += ov;
    }
    u32 nk = __shfl_down_sync(0xFFFFFFFFu, k, 1);
    bool last = (lane == 31) || nk != k;
    if (ok && last && v) atomicAdd((unsigned long long*)&out[k], (unsigned long long)v);
  }
}

}  // namespace gt
