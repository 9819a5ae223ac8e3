// cub_ops.cu — device-wide sort/scan/select plumbing (CUB, CUDA 12.9 toolkit
// headers, instantiated into this library).  Used by the DAG loader and by
// the result-assembly steps; the analytics kernels themselves are ours.
#include <algorithm>

#include <cub/cub.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/tabulate_output_iterator.h>

#include "gt_internal.cuh"

namespace gt {

// CUB temporary storage: a per-thread, per-stream buffer reused across calls
// (stream order makes the reuse safe) for requests up to kTempCache bytes —
// an allocation + free per CUB call is ~4 us of host time, and a small
// grammar's gt_open makes a dozen CUB calls.  Never freed (process lifetime;
// freeing from a thread_local destructor would run after the CUDA teardown).
constexpr size_t kTempCache = 64ull << 20;
struct TempSlot {
  cudaStream_t s = nullptr;
  void* p = nullptr;
  size_t bytes = 0;
};
static void* temp_for(cudaStream_t s, size_t bytes) {
  static thread_local TempSlot slots[4];
  TempSlot* t = nullptr;
  for (auto& x : slots)
    if (x.s == s) t = &x;
  if (!t)
    for (auto& x : slots)
      if (!x.s) {
        t = &x;
        t->s = s;
        break;
      }
  if (!t) return nullptr;
  if (t->bytes < bytes) {
    if (t->p) cudaFreeAsync(t->p, s);
    t->p = nullptr;
    t->bytes = 0;
    GT_CUDA(cudaMallocAsync(&t->p, bytes, s));
    t->bytes = bytes;
  }
  return t->p;
}

template <class F>
static void with_temp(const char* name, F f, cudaStream_t s) {
  size_t bytes = 0;
  f(nullptr, bytes);
  void* cached = bytes && bytes <= kTempCache ? temp_for(s, std::max<size_t>(bytes, 4096)) : nullptr;
  DBuf tmp;
  if (!cached) tmp.alloc(bytes ? bytes : 16, s);
  ProfScope ps(name, s);
  f(cached ? cached : tmp.p, bytes);
  g_launches += 4;  // CUB device-wide primitives launch a small fixed set of kernels
}

void sort_pairs_u64_u32(u64* ki, u64* ko, u32* vi, u32* vo, u64 n, int end_bit, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::SortPairs64", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, (int64_t)n, 0, end_bit, s));
  }, s);
}

void sort_pairs_u32_u32(u32* ki, u32* ko, u32* vi, u32* vo, u64 n, int end_bit, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::SortPairs32", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, (int64_t)n, 0, end_bit, s));
  }, s);
}

void sort_pairs_u32_u64(u32* ki, u32* ko, u64* vi, u64* vo, u64 n, int end_bit, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::SortPairs32x64", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, (int64_t)n, 0, end_bit, s));
  }, s);
}

void sort_pairs_u32_u3(u32* ki, u32* ko, U3* vi, U3* vo, u64 n, int end_bit, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::SortPairs32x96", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, (int64_t)n, 0, end_bit, s));
  }, s);
}

void sort_keys_u32(const u32* ki, u32* ko, u64 n, int end_bit, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::SortKeys32", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceRadixSort::SortKeys(t, b, ki, ko, (int64_t)n, 0, end_bit, s));
  }, s);
}

void sort_keys_u64(u64* ki, u64* ko, u64 n, int end_bit, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::SortKeys64", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceRadixSort::SortKeys(t, b, ki, ko, (int64_t)n, 0, end_bit, s));
  }, s);
}

void exclusive_scan_u64(const u64* in, u64* out, u64 n, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::ExclusiveSum", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceScan::ExclusiveSum(t, b, in, out, (int64_t)n, s));
  }, s);
}

void inclusive_scan_u32(const u32* in, u32* out, u64 n, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::InclusiveSum", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceScan::InclusiveSum(t, b, in, out, (int64_t)n, s));
  }, s);
}

void select_flagged_index(const uint8_t* flags, u32* out_idx, u64* d_count, u64 n,
                          cudaStream_t s) {
  if (!n) {
    GT_CUDA(cudaMemsetAsync(d_count, 0, sizeof(u64), s));
    return;
  }
  thrust::counting_iterator<u32> it(0);
  with_temp("cub::SelectFlagged", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceSelect::Flagged(t, b, it, flags, out_idx, d_count, (int64_t)n, s));
  }, s);
}

template <class T>
struct NonzeroAt {
  const T* v;
  __device__ __forceinline__ bool operator()(const u32& i) const { return v[i] != 0; }
};

// indices i < n with v[i] != 0, ascending (one select pass, no flag array)
void select_nonzero_index(const void* v, bool v32, u32* out_idx, u64* d_count, u64 n, cudaStream_t s) {
  if (!n) {
    GT_CUDA(cudaMemsetAsync(d_count, 0, sizeof(u64), s));
    return;
  }
  thrust::counting_iterator<u32> it(0);
  with_temp("cub::SelectIf", [&](void* t, size_t& b) {
    if (v32)
      GT_CUDA(cub::DeviceSelect::If(t, b, it, out_idx, d_count, (int64_t)n, NonzeroAt<u32>{(const u32*)v}, s));
    else
      GT_CUDA(cub::DeviceSelect::If(t, b, it, out_idx, d_count, (int64_t)n, NonzeroAt<u64>{(const u64*)v}, s));
  }, s);
}

// the k-th selected index i becomes record k: (i % V, v[i], i / V)
template <class T>
struct RecordWriter {
  const T* v;
  u64 V;
  u32* id;
  u64* cnt;
  u32* file;
  __device__ __forceinline__ void operator()(int64_t k, u32 i) const {
    id[k] = (u32)(i % V);
    cnt[k] = v[i];
    if (file) file[k] = (u32)(i / V);
  }
};

void select_nonzero_records(const void* v, bool v32, u64 V, u64 n, u32* id, u64* cnt, u32* file, u64* d_count,
                            cudaStream_t s) {
  if (!n) {
    GT_CUDA(cudaMemsetAsync(d_count, 0, sizeof(u64), s));
    return;
  }
  thrust::counting_iterator<u32> it(0);
  with_temp("cub::SelectIf", [&](void* t, size_t& b) {
    if (v32) {
      const u32* p = (const u32*)v;
      auto out = thrust::make_tabulate_output_iterator(RecordWriter<u32>{p, V, id, cnt, file});
      GT_CUDA(cub::DeviceSelect::If(t, b, it, out, d_count, (int64_t)n, NonzeroAt<u32>{p}, s));
    } else {
      const u64* p = (const u64*)v;
      auto out = thrust::make_tabulate_output_iterator(RecordWriter<u64>{p, V, id, cnt, file});
      GT_CUDA(cub::DeviceSelect::If(t, b, it, out, d_count, (int64_t)n, NonzeroAt<u64>{p}, s));
    }
  }, s);
}

void sort_pairs_u64_u64(u64* ki, u64* ko, u64* vi, u64* vo, u64 n, int end_bit, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::SortPairs64x64", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceRadixSort::SortPairs(t, b, ki, ko, vi, vo, (int64_t)n, 0, end_bit, s));
  }, s);
}

void reduce_by_key_u64(const u64* keys, const u64* vals, u64* ukeys, u64* sums, u64* d_nruns, u64 n,
                       cudaStream_t s) {
  if (!n) {
    GT_CUDA(cudaMemsetAsync(d_nruns, 0, sizeof(u64), s));
    return;
  }
  with_temp("cub::ReduceByKey", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceReduce::ReduceByKey(t, b, keys, ukeys, vals, sums, d_nruns, ::cuda::std::plus<u64>(),
                                           (int64_t)n, s));
  }, s);
}

void sort_segments_u32(const u32* ki, u32* ko, u64 n, u64 nseg, const u64* off, cudaStream_t s) {
  if (!n) return;
  with_temp("cub::SegmentedSort32", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceSegmentedSort::SortKeys(t, b, ki, ko, (int)n, (int)nseg, off, off + 1, s));
  }, s);
}

// sort the listed segments [beg[i], end[i]) of ki into ko (other positions of
// ko are left undefined)
void sort_segments_listed_u32(const u32* ki, u32* ko, u64 n, u64 nseg, const int* beg, const int* end,
                              cudaStream_t s) {
  if (!n || !nseg) return;
  with_temp("cub::SegmentedSort32", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceSegmentedSort::SortKeys(t, b, ki, ko, (int)n, (int)nseg, beg, end, s));
  }, s);
}

void reduce_max_u64(const u64* in, u64* out, u64 n, cudaStream_t s) {
  if (!n) {
    GT_CUDA(cudaMemsetAsync(out, 0, sizeof(u64), s));
    return;
  }
  with_temp("cub::ReduceMax", [&](void* t, size_t& b) {
    GT_CUDA(cub::DeviceReduce::Max(t, b, in, out, (int64_t)n, s));
  }, s);
}

}  // namespace gt
