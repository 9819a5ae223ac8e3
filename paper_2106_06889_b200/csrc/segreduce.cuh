// segreduce.cuh — the load-balanced segmented gather-reduce every traversal
// step of the library is built from.
//
//   out[dst[i], col] (+)= combine(freq[i], in(src[i], col))   for i in [0, n)
//
// over an item list sorted by dst.  It is the B200 form of the reference's
// work partitioning (engine.py:74-106 partition_work: rules longer than
// chunk_factor x average are split into contiguous ranges
// "fine-grained thread-level partitioning"): items, not rules, are dealt out
// in fixed-size chunks, so a rule with 10^6 parents costs 10^6/chunk chunks
// spread over the whole GPU instead of one serial warp.  Runs of equal dst
// are combined in registers (warp shuffle segmented scan, or a team's
// sequential walk) and each run is flushed with ONE fire-and-forget u64
// reduction (atomicAdd / atomicOr without return -> RED at L2): no
// read-modify-write round trip on the critical path, and a hot destination
// costs one reduction per chunk, not one per item (the warp aggregation of
// north_star).  Outputs may be pre-seeded; everything is an integer sum or
// bitwise OR, so the result is order-independent and bit-exact.
//
// Uses:  top-down level propagation (dst = child, src = parent; items = the
//        level's non-root parent edges), bottom-up sums (dst = rule, src =
//        child), reduce-by-word (dst = word, src = rule), gram-run rows
//        (dst = run, src = rule or root segment).
#pragma once

#include <cooperative_groups.h>

#include <algorithm>
#include <type_traits>

#include "kernels_common.cuh"

namespace cg = cooperative_groups;

namespace gt {

// Values are combined in u64 registers; rows / outputs are u64, or u32 for
// per-file counts when every file has < 2^32 words (DeviceDag::cnt32: a
// per-file cell never exceeds its file's word count), halving the row bytes
// of the 64-column passes.
struct SumMode {
  using V = u64;
  __device__ static __forceinline__ V zero() { return 0; }
  __device__ static __forceinline__ u64 combine(u32 f, u64 x) { return (u64)f * x; }
  __device__ static __forceinline__ u64 merge(u64 a, u64 b) { return a + b; }
  __device__ static __forceinline__ void atomic(u64* p, u64 v) {
    if (v) atomicAdd((unsigned long long*)p, (unsigned long long)v);
  }
  __device__ static __forceinline__ void atomic(u32* p, u64 v) {
    if (v) atomicAdd((unsigned*)p, (unsigned)v);
  }
};

struct OrMode {
  using V = u64;
  __device__ static __forceinline__ V zero() { return 0; }
  __device__ static __forceinline__ u64 combine(u32, u64 x) { return x; }
  __device__ static __forceinline__ u64 merge(u64 a, u64 b) { return a | b; }
  __device__ static __forceinline__ void atomic(u64* p, u64 v) {
    if (v) atomicOr((unsigned long long*)p, (unsigned long long)v);
  }
  __device__ static __forceinline__ void atomic(u32* p, u64 v) {
    if (v) atomicOr((unsigned*)p, (unsigned)v);
  }
};

// height pass (bottom-up levels without Kahn): height(r) = max(height(r),
// 1 + height(child)), combined with u64 atomicMax
struct HeightMode {
  using V = u64;
  __device__ static __forceinline__ V zero() { return 0; }
  __device__ static __forceinline__ u64 combine(u32, u64 x) { return x + 1; }
  __device__ static __forceinline__ u64 merge(u64 a, u64 b) { return a > b ? a : b; }
  __device__ static __forceinline__ void atomic(u64* p, u64 v) {
    atomicMax((unsigned long long*)p, (unsigned long long)v);
  }
};

// Word count and inverted index in ONE pass (gt_run_many): every rule row is
// a 16-byte pair {corpus weight (sum), file-presence bitset (or)} — the two
// tasks share the same edges, levels and barriers, so the step pays one
// latency-bound level chain instead of two.  A pair is gathered with one
// 16-byte load (one sector) and flushed with one RED.ADD + one RED.OR.
struct u64x2 {
  u64 a, b;
};
struct PairPtr {  // where a pair is reduced into: the weight and presence words
  u64* a;
  u64* b;
};
struct WcPresMode {
  using V = u64x2;
  __device__ static __forceinline__ V zero() { return {0, 0}; }
  __device__ static __forceinline__ V combine(u32 f, V x) { return {(u64)f * x.a, x.b}; }
  __device__ static __forceinline__ V merge(V x, V y) { return {x.a + y.a, x.b | y.b}; }
  __device__ static __forceinline__ void atomic(PairPtr p, V v) {
    if (v.a) atomicAdd((unsigned long long*)p.a, (unsigned long long)v.a);
    if (v.b) atomicOr((unsigned long long*)p.b, (unsigned long long)v.b);
  }
};

// warp shuffles of a mode's value (u64 or a pair)
__device__ __forceinline__ u64 shfl_up(u64 v, int s) { return __shfl_up_sync(0xFFFFFFFFu, v, s); }
__device__ __forceinline__ u64 shfl_idx(u64 v, int l) { return __shfl_sync(0xFFFFFFFFu, v, l); }
__device__ __forceinline__ u64x2 shfl_up(u64x2 v, int s) {
  return {__shfl_up_sync(0xFFFFFFFFu, v.a, s), __shfl_up_sync(0xFFFFFFFFu, v.b, s)};
}
__device__ __forceinline__ u64x2 shfl_idx(u64x2 v, int l) {
  return {__shfl_sync(0xFFFFFFFFu, v.a, l), __shfl_sync(0xFFFFFFFFu, v.b, l)};
}

// ---- source row functors ----------------------------------------------------
// Row and output reads go through L2 (ld.global.cg): the level loops of a
// persistent launch read rows other SMs wrote before the grid barrier, and a
// line cached in a non-coherent L1 earlier could be stale.
__device__ __forceinline__ u64 ldcg(const u64* p) {
  return (u64)__ldcg(reinterpret_cast<const unsigned long long*>(p));
}

__device__ __forceinline__ u64 ldcg(const u32* p) { return (u64)__ldcg(reinterpret_cast<const unsigned*>(p)); }

template <class T>
struct RowSrcT {  // in[src*C + col]
  const T* in;
  u32 C;
  __device__ __forceinline__ u64 operator()(u32 s, u32 col) const { return ldcg(in + (u64)s * C + col); }
};
using RowSrc = RowSrcT<u64>;

// two adjacent columns of a source row (col even): one 16-byte (u64 rows) or
// 8-byte (u32 rows) load for RowSrcT, two scalar reads otherwise
template <class Src>
__device__ __forceinline__ void load_pair(const Src& in, u32 s, u32 col, u64* a, u64* b) {
  *a = in(s, col);
  *b = in(s, col + 1);
}
__device__ __forceinline__ void load_pair(const RowSrcT<u64>& in, u32 s, u32 col, u64* a, u64* b) {
  const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(in.in + (u64)s * in.C + col));
  *a = v.x;
  *b = v.y;
}
__device__ __forceinline__ void load_pair(const RowSrcT<u32>& in, u32 s, u32 col, u64* a, u64* b) {
  const uint2 v = __ldcg(reinterpret_cast<const uint2*>(in.in + (u64)s * in.C + col));
  *a = v.x;
  *b = v.y;
}

// row sources whose paired path loads the items' metadata one per lane
template <class Src>
struct LaneMeta {
  static constexpr bool value = false;
};
template <class T>
struct LaneMeta<RowSrcT<T>> {
  static constexpr bool value = true;
};

// ---- output address functors --------------------------------------------------
template <class T>
struct OutRowMajorT {  // out[dst*C + col]
  T* out;
  u32 C;
  __device__ __forceinline__ T* operator()(u32 d, u32 col) const { return out + (u64)d * C + col; }
};
using OutRowMajor = OutRowMajorT<u64>;
template <class T>
struct TdRowsT {  // out[dst*C + col] for the top-down pass (a distinct kernel name in ncu)
  T* out;
  u32 C;
  __device__ __forceinline__ T* operator()(u32 d, u32 col) const { return out + (u64)d * C + col; }
};
using TdRows = TdRowsT<u64>;
template <class T>
struct OutColMajorT {  // out[col*V + dst]
  T* out;
  u64 V;
  __device__ __forceinline__ T* operator()(u32 d, u32 col) const { return out + (u64)col * V + d; }
};
using OutColMajor = OutColMajorT<u64>;

// the fused word count + presence pass: interleaved 16-byte rule rows
struct RowSrcPair {
  const u64* in;
  __device__ __forceinline__ u64x2 operator()(u32 s, u32) const {
    const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(in + 2ull * s));
    return {v.x, v.y};
  }
};
struct TdRowsPair {
  u64* out;
  __device__ __forceinline__ PairPtr operator()(u32 d, u32) const { return {out + 2ull * d, out + 2ull * d + 1}; }
};
// per word: the count vector u64[V] and the presence vector u64[V]
struct OutPair {
  u64* cnt;
  u64* pres;
  __device__ __forceinline__ PairPtr operator()(u32 d, u32) const { return {cnt + d, pres + d}; }
};

__device__ __forceinline__ u32 item_freq(const u32* freq, u64 i) { return freq ? freq[i] : 1u; }
// item lists are read once per pass: streamed (evict-first), so they do not
// push the gathered rows out of L2
__device__ __forceinline__ u32 item_freq_cs(const u32* freq, u64 i) { return freq ? __ldcs(freq + i) : 1u; }

// ---------------------------------------------------------------------------
// one column: a warp owns tiles of 32*K consecutive items; runs are combined
// with a shuffle segmented scan and carried across the K steps of the tile.
// ---------------------------------------------------------------------------
template <class Mode, class Src, class Out>
__device__ __forceinline__ void segred1_body(const u32* __restrict__ dst, const u32* __restrict__ src,
                                             const u32* __restrict__ freq, u64 n, int K, Src in,
                                             Out out, u64 warp, u64 nwarps) {
  // K 32-item steps per tile; the (up to) U steps of a group are
  // loaded together (U independent row gathers in flight per lane), then
  // reduced one after the other with the carried run
  using V = typename Mode::V;
  constexpr int U = 4;
  const unsigned lane = threadIdx.x & 31u;
  const u64 TILE = 32ull * K;
  for (u64 t0 = warp * TILE; t0 < n; t0 += nwarps * TILE) {
    const u64 tend = t0 + TILE < n ? t0 + TILE : n;
    u32 carry_d = 0xFFFFFFFFu;
    V carry_v = Mode::zero();
#pragma unroll 1
    for (int k0 = 0; k0 < K; k0 += U) {
      u32 dd[U];
      V vv[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const u64 i = t0 + (u64)(k0 + u) * 32 + lane;
        const bool in_tile = k0 + u < K && i < tend;
        dd[u] = in_tile ? __ldcs(dst + i) : 0xFFFFFFFFu;
        vv[u] = in_tile ? Mode::combine(item_freq_cs(freq, i), in(__ldcs(src + i), 0)) : Mode::zero();
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (k0 + u >= K) break;  // warp-uniform
        const u32 d = dd[u];
        V v = vv[u];
        const bool ok = d != 0xFFFFFFFFu;
        const u32 d0 = __shfl_sync(0xFFFFFFFFu, d, 0);
        if (carry_d != 0xFFFFFFFFu && d0 != carry_d) {  // the carried run ended at the last step
          if (lane == 0) Mode::atomic(out(carry_d, 0), carry_v);
          carry_d = 0xFFFFFFFFu;
          carry_v = Mode::zero();
        }
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
          const V ov = shfl_up(v, s);
          const u32 od = __shfl_up_sync(0xFFFFFFFFu, d, s);
          if (lane >= (unsigned)s && od == d) v = Mode::merge(v, ov);
        }
        if (d == carry_d) v = Mode::merge(v, carry_v);
        const u32 dn = __shfl_down_sync(0xFFFFFFFFu, d, 1);
        if (ok && lane != 31 && dn != d) Mode::atomic(out(d, 0), v);  // run ends inside this step
        carry_d = __shfl_sync(0xFFFFFFFFu, d, 31);
        carry_v = shfl_idx(v, 31);
      }
    }
    if (lane == 0 && carry_d != 0xFFFFFFFFu) Mode::atomic(out(carry_d, 0), carry_v);
  }
}

template <class Mode, class Src, class Out>
__global__ void __launch_bounds__(256) k_segred1(const u32* __restrict__ dst,
                                                 const u32* __restrict__ src,
                                                 const u32* __restrict__ freq, u64 n, int K,
                                                 Src in, Out out) {
  segred1_body<Mode>(dst, src, freq, n, K, in, out, ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5,
                     ((u64)gridDim.x * blockDim.x) >> 5);
}

// ---------------------------------------------------------------------------
// C columns: a team of G lanes owns chunks of K consecutive items and walks
// them with the lanes spread over the columns (coalesced row gathers); item
// values are fetched B at a time ahead of the run bookkeeping.
// ---------------------------------------------------------------------------
template <int G, class Mode, bool MULTI, class Src, class Out>
__device__ __forceinline__ void segredG_body(const u32* __restrict__ dst, const u32* __restrict__ src,
                                             const u32* __restrict__ freq, u64 n, u32 K, u32 C, Src in,
                                             Out out, u64 gtid, u64 nthreads) {
  constexpr int B = 8;
  const u64 teams = nthreads / G;
  const u32 tl = threadIdx.x % G;
  if (C == 2u * G && !LaneMeta<Src>::value) {
    // (gram-run rows: the per-item metadata loads are broadcast; measured
    // faster there than the lane-loaded form below)
    constexpr int BB = 8;
    const u32 c0 = 2 * tl;
    for (u64 t = gtid / G; t * K < n; t += teams) {
      const u64 a = t * K, b = a + K < n ? a + K : n;
      u32 cd = dst[a];
      u64 acc0 = 0, acc1 = 0;
      for (u64 i0 = a; i0 < b; i0 += BB) {
        u32 dd[BB];
        u64 v0[BB], v1[BB];
#pragma unroll
        for (int j = 0; j < BB; j++) {
          const u64 i = i0 + j;
          const bool ok = i < b;
          dd[j] = ok ? dst[i] : 0xFFFFFFFFu;
          u64 x = 0, y = 0;
          if (ok) {
            load_pair(in, src[i], c0, &x, &y);
            const u32 f = item_freq(freq, i);
            x = Mode::combine(f, x);
            y = Mode::combine(f, y);
          }
          v0[j] = x;
          v1[j] = y;
        }
#pragma unroll
        for (int j = 0; j < BB; j++) {
          if (dd[j] == 0xFFFFFFFFu) break;
          if (dd[j] != cd) {
            Mode::atomic(out(cd, c0), acc0);
            Mode::atomic(out(cd, c0 + 1), acc1);
            acc0 = acc1 = 0;
            cd = dd[j];
          }
          acc0 = Mode::merge(acc0, v0[j]);
          acc1 = Mode::merge(acc1, v1[j]);
        }
      }
      Mode::atomic(out(cd, c0), acc0);
      Mode::atomic(out(cd, c0 + 1), acc1);
    }
    return;
  }
  if (C == 2u * G) {
    // two ADJACENT columns per lane: the team reads a whole row with one
    // vector load per lane (C = 64: one 512 / 256-byte access per item).  The
    // items' (dst, src, freq) are loaded G at a time, one per lane, and
    // broadcast by shuffles, so only the row gathers (BB in flight) remain
    // on each group's dependent path.
    constexpr int BB = 8;
    const u32 c0 = 2 * tl;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned tmask = (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u)) << (lane & ~(unsigned)(G - 1));
    for (u64 t = gtid / G; t * K < n; t += teams) {
      const u64 a = t * K, b = a + K < n ? a + K : n;
      u32 cd = dst[a];
      u64 acc0 = 0, acc1 = 0;
      for (u64 i0 = a; i0 < b; i0 += G) {
        const u64 im = i0 + tl;
        const bool okm = im < b;
        const u32 md = okm ? dst[im] : 0xFFFFFFFFu;
        const u32 ms = okm ? src[im] : 0u;
        const u32 mf = okm ? item_freq(freq, im) : 0u;
#pragma unroll 1
        for (int g = 0; g < G; g += BB) {
          u32 dd[BB];
          u64 v0[BB], v1[BB];
#pragma unroll
          for (int j = 0; j < BB; j++) {
            dd[j] = __shfl_sync(tmask, md, g + j, G);
            const u32 sj = __shfl_sync(tmask, ms, g + j, G);
            const u32 fj = __shfl_sync(tmask, mf, g + j, G);
            u64 x = 0, y = 0;
            if (dd[j] != 0xFFFFFFFFu) {
              load_pair(in, sj, c0, &x, &y);
              x = Mode::combine(fj, x);
              y = Mode::combine(fj, y);
            }
            v0[j] = x;
            v1[j] = y;
          }
#pragma unroll
          for (int j = 0; j < BB; j++) {
            if (dd[j] == 0xFFFFFFFFu) break;
            if (dd[j] != cd) {
              Mode::atomic(out(cd, c0), acc0);
              Mode::atomic(out(cd, c0 + 1), acc1);
              acc0 = acc1 = 0;
              cd = dd[j];
            }
            acc0 = Mode::merge(acc0, v0[j]);
            acc1 = Mode::merge(acc1, v1[j]);
          }
          if (dd[BB - 1] == 0xFFFFFFFFu) break;  // past the chunk end (team-uniform)
        }
      }
      Mode::atomic(out(cd, c0), acc0);
      Mode::atomic(out(cd, c0 + 1), acc1);
    }
    return;
  }
  if (MULTI && C <= 4u * G) {
    // (persistent level loops only: measured faster there — C4 64-file
    // top-down pass 7.5 -> 3.9 ms — and slower for the flat launches)
    // up to 4 columns per lane in registers: the item list is walked once and
    // B x NC row gathers are in flight per lane
    constexpr int NC = 4, BB = 4;
    const u32 nc = (C + G - 1) / G;
    for (u64 t = gtid / G; t * K < n; t += teams) {
      const u64 a = t * K, b = a + K < n ? a + K : n;
      u32 cd = dst[a];
      u64 acc[NC] = {0, 0, 0, 0};
      for (u64 i0 = a; i0 < b; i0 += BB) {
        u32 dd[BB];
        u64 v[BB][NC];
#pragma unroll
        for (int j = 0; j < BB; j++) {
          const u64 i = i0 + j;
          const bool ok = i < b;
          dd[j] = ok ? dst[i] : 0xFFFFFFFFu;
          const u32 sj = ok ? src[i] : 0u;
          const u32 fj = ok ? item_freq(freq, i) : 0u;
#pragma unroll
          for (int k = 0; k < NC; k++) {
            const u32 col = tl + (u32)k * G;
            v[j][k] = (ok && (u32)k < nc && col < C) ? Mode::combine(fj, in(sj, col)) : 0;
          }
        }
#pragma unroll
        for (int j = 0; j < BB; j++) {
          if (dd[j] == 0xFFFFFFFFu) break;
          if (dd[j] != cd) {
#pragma unroll
            for (int k = 0; k < NC; k++) {
              const u32 col = tl + (u32)k * G;
              if ((u32)k < nc && col < C) Mode::atomic(out(cd, col), acc[k]);
              acc[k] = 0;
            }
            cd = dd[j];
          }
#pragma unroll
          for (int k = 0; k < NC; k++) acc[k] = Mode::merge(acc[k], v[j][k]);
        }
      }
#pragma unroll
      for (int k = 0; k < NC; k++) {
        const u32 col = tl + (u32)k * G;
        if ((u32)k < nc && col < C) Mode::atomic(out(cd, col), acc[k]);
      }
    }
    return;
  }
  for (u64 t = gtid / G; t * K < n; t += teams) {
    const u64 a = t * K, b = a + K < n ? a + K : n;  // K: items per team (runtime)
    const u32 dfirst = dst[a];
    for (u32 col = tl; col < C; col += G) {
      u32 cd = dfirst;
      u64 acc = 0;
      for (u64 i0 = a; i0 < b; i0 += B) {
        u64 v[B];
        u32 dd[B];
#pragma unroll
        for (int j = 0; j < B; j++) {
          const u64 i = i0 + j;
          dd[j] = i < b ? dst[i] : 0xFFFFFFFFu;
          v[j] = i < b ? Mode::combine(item_freq(freq, i), in(src[i], col)) : 0;
        }
#pragma unroll
        for (int j = 0; j < B; j++) {
          if (dd[j] == 0xFFFFFFFFu) break;
          if (dd[j] != cd) {
            auto* p = out(cd, col);
            Mode::atomic(p, acc);
            cd = dd[j];
            acc = 0;
          }
          acc = Mode::merge(acc, v[j]);
        }
      }
      auto* p = out(cd, col);
      Mode::atomic(p, acc);
    }
  }
}

template <int G, class Mode, class Src, class Out>
__global__ void __launch_bounds__(256) k_segredG(const u32* __restrict__ dst,
                                                 const u32* __restrict__ src,
                                                 const u32* __restrict__ freq, u64 n, u32 K, u32 C,
                                                 Src in, Out out) {
  segredG_body<G, Mode, false>(dst, src, freq, n, K, C, in, out, (u64)blockIdx.x * blockDim.x + threadIdx.x,
                               (u64)gridDim.x * blockDim.x);
}

// ---------------------------------------------------------------------------
// Top-down seeds (init_top_down_masks, engine.py:178-193): the root's direct
// references per owned segment (rs lists sorted by (rule, segment)).  Global
// mode adds every owned segment's count into row[rule]; per-file mode into
// row[rule*C + segment]; presence (OrMode) sets bit segment%64 of
// row[rule*C + segment/64].  Lanes of a warp hitting the same cell are
// combined with a segmented shuffle scan (keys ascend along the list), one
// reduction per run.  zero_n: rows to clear first (persistent phase 0 only).
// ---------------------------------------------------------------------------
struct SeedArgs {
  const u32* rule;
  const u32* seg;
  const u32* cnt;
  u64 n;
  u32 file_lo, nseg;
  int per_file;
  u32 C;
  void* row;  // u64 rows, or u32 (per-file counts under DeviceDag::cnt32)
  u64 zero_n;
};

// Reduce-by-word folded into the same launch after the last level (C = 1):
// out[w] (+)= f * row[r] over the word-major own pairs, then the root's plain
// words of the owned segments (reduce_words_round + root_words_round,
// _kernels.py:154-188); out is cleared in phase 0.
struct PostArgs {
  const u32* dst;  // ow_word
  const u32* src;  // ow_rule (tid)
  const u32* freq;
  u64 n;
  u64* out;  // nullptr: no post phase
  u64 out_n;
  u64* out2;  // WcPresMode: the presence vector u64[V] beside the counts in out
  const u32* rw_word;
  const u32* rw_seg;
  const u32* rw_cnt;
  u64 n_rw;
  u32 file_lo, nseg;
  int per_file;
  // compaction of out (after one more barrier) into render-order records:
  // 1 = nonzero counts -> (word, count) records (word count); 2 = presence
  // words -> (word groups, ascending files) (inverted index, <= 64 files);
  // 3 = both from the fused pair (WcPresMode): word-count records (wid,
  // rcnt) and the inverted-index groups / files (gid, goff, rid) share the
  // word order, so one scan gives both.  Outputs sized for the worst case;
  // tot = {records, groups}; bsum = 2 * gridDim scratch.
  int compact;
  u32* wid;
  u32* rid;
  u64* rcnt;
  u32* gid;
  u64* goff;
  u64* tot;
  u64* bsum;
  // diagnostics (GT_TRACE=2): %globaltimer of block 0 at the phase
  // boundaries — [0] entry, [1] seeds done, [2 + it] level it done, then the
  // word reduce and the compaction
  u64* stamps;
  // compaction: u32 copies of the counts (saturating; tot[2] != 0 when one
  // needed 64 bits) and of the group offsets, written beside the u64 ones
  u32* rcnt32;
  u32* goff32;
  // compact 2 / 3: the file ids written rid_bytes (1 / 2) wide into rid_n
  // instead of rid (4: rid)
  void* rid_n;
  int rid_bytes;
  // rows cleared again after the word reduce has read them (while the
  // compaction runs): the next step's phase 0 then seeds them without a
  // clearing pass and its grid barrier
  u64* zero_tail;
  u64 zero_tail_n;
};

__device__ __forceinline__ void seg_stamp(u64* stamps, int k) {
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0 && k < 64) {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[k] = t;
  }
}

// block-wide exclusive scan of two counters (1024 threads); returns the
// block totals through *ta / *tb
__device__ __forceinline__ void block_scan2(u32 a, u32 b, u32* ea, u32* eb, u32* ta, u32* tb) {
  __shared__ u32 wa[32], wb[32];
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  u32 ia = a, ib = b;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 xa = __shfl_up_sync(0xFFFFFFFFu, ia, d), xb = __shfl_up_sync(0xFFFFFFFFu, ib, d);
    if (lane >= (unsigned)d) {
      ia += xa;
      ib += xb;
    }
  }
  if (lane == 31) {
    wa[wid] = ia;
    wb[wid] = ib;
  }
  __syncthreads();
  if (wid == 0) {
    const unsigned nw = blockDim.x >> 5;
    u32 va = lane < nw ? wa[lane] : 0u, vb = lane < nw ? wb[lane] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 xa = __shfl_up_sync(0xFFFFFFFFu, va, d), xb = __shfl_up_sync(0xFFFFFFFFu, vb, d);
      if (lane >= (unsigned)d) {
        va += xa;
        vb += xb;
      }
    }
    if (lane < nw) {
      wa[lane] = va;
      wb[lane] = vb;
    }
  }
  __syncthreads();
  const u32 pa = wid ? wa[wid - 1] : 0u, pb = wid ? wb[wid - 1] : 0u;
  *ea = pa + ia - a;
  *eb = pb + ib - b;
  *ta = wa[(blockDim.x >> 5) - 1];
  *tb = wb[(blockDim.x >> 5) - 1];
  __syncthreads();
}

// the compaction of the post phase: blocks own contiguous word ranges, count
// them, learn their offsets after a grid barrier, and write in order.  Per
// word: a = records (1 per nonzero count, or the popcount of the presence
// word), b = groups (1 per nonempty word; compact 2 and 3 only).
__device__ __forceinline__ void post_word(const PostArgs& p, u64 w, u64* v, u64* pr) {
  *v = __ldcg(reinterpret_cast<const unsigned long long*>(p.out + w));
  *pr = p.compact == 3 ? __ldcg(reinterpret_cast<const unsigned long long*>(p.out2 + w))
                       : (p.compact == 2 ? *v : 0ull);
}

__device__ __forceinline__ void post_compact(const PostArgs& p, cg::grid_group& grid) {
  const u64 V = p.out_n, nb = gridDim.x;
  const u64 CH = (V + nb - 1) / nb, lo = blockIdx.x * CH, hi = lo + CH < V ? lo + CH : V;
  const bool groups = p.compact >= 2;
  __shared__ unsigned long long sa, sb;
  if (threadIdx.x == 0) sa = sb = 0;
  __syncthreads();
  unsigned long long la = 0, lb = 0;
  for (u64 w = lo + threadIdx.x; w < hi; w += blockDim.x) {
    u64 v, pr;
    post_word(p, w, &v, &pr);
    if (v || pr) {
      la += groups ? (unsigned long long)__popcll(pr) : 1ull;
      lb += 1;
    }
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) {
    la += __shfl_xor_sync(0xFFFFFFFFu, la, d);
    lb += __shfl_xor_sync(0xFFFFFFFFu, lb, d);
  }
  if ((threadIdx.x & 31u) == 0 && (la || lb)) {  // one shared atomic per warp
    atomicAdd(&sa, la);
    if (groups) atomicAdd(&sb, lb);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    p.bsum[blockIdx.x] = sa;
    p.bsum[nb + blockIdx.x] = sb;
  }
  grid.sync();
  // this block's offsets: sums over the blocks before it (one warp)
  __shared__ unsigned long long oa, ob;
  if (threadIdx.x < 32) {
    unsigned long long xa = 0, xb = 0;
    for (u64 j = threadIdx.x; j < blockIdx.x; j += 32) {
      xa += __ldcg(reinterpret_cast<const unsigned long long*>(p.bsum + j));
      xb += __ldcg(reinterpret_cast<const unsigned long long*>(p.bsum + nb + j));
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      xa += __shfl_xor_sync(0xFFFFFFFFu, xa, d);
      xb += __shfl_xor_sync(0xFFFFFFFFu, xb, d);
    }
    if (threadIdx.x == 0) {
      oa = xa;
      ob = xb;
      if (blockIdx.x == nb - 1) {
        p.tot[0] = xa + __ldcg(reinterpret_cast<const unsigned long long*>(p.bsum + blockIdx.x));
        p.tot[1] = xb + __ldcg(reinterpret_cast<const unsigned long long*>(p.bsum + nb + blockIdx.x));
        if (groups) p.goff[p.tot[1]] = p.tot[0];
        if (groups && p.goff32) p.goff32[p.tot[1]] = (u32)p.tot[0];
      }
    }
  }
  __syncthreads();
  u64 ba = oa, bb = ob;
  bool big = false;
  for (u64 t0 = lo; t0 < hi; t0 += blockDim.x) {  // block-uniform trip count
    const u64 w = t0 + threadIdx.x;
    u64 v = 0, pr = 0;
    if (w < hi) post_word(p, w, &v, &pr);
    const bool nz = v || pr;
    const u32 a = nz ? (groups ? (u32)__popcll(pr) : 1u) : 0u, b = (groups && nz) ? 1u : 0u;
    u32 ea, eb, ta, tb;
    block_scan2(a, b, &ea, &eb, &ta, &tb);
    if (nz) {
      const u32 v32 = v > 0xFFFFFFFFull ? 0xFFFFFFFFu : (u32)v;
      big |= v > 0xFFFFFFFFull;
      if (!groups) {
        p.rid[ba + ea] = (u32)w;
        p.rcnt[ba + ea] = v;
        if (p.rcnt32) p.rcnt32[ba + ea] = v32;
      } else {
        if (p.compact == 3) {  // the word-count record of this word
          p.wid[bb + eb] = (u32)w;
          p.rcnt[bb + eb] = v;
          if (p.rcnt32) p.rcnt32[bb + eb] = v32;
        }
        p.gid[bb + eb] = (u32)w;
        p.goff[bb + eb] = ba + ea;
        if (p.goff32) p.goff32[bb + eb] = (u32)(ba + ea);
        // (each lane writes its own word's files; a warp-cooperative
        // coalesced emission measured slower: C5 0.27 -> 0.32 ms)
        u64 q = ba + ea, x = pr;
        if (p.rid_bytes == 1) {
          uint8_t* o = static_cast<uint8_t*>(p.rid_n);
          while (x) {
            o[q++] = (uint8_t)(p.file_lo + (u32)(__ffsll((long long)x) - 1));
            x &= x - 1;
          }
        } else if (p.rid_bytes == 2) {
          unsigned short* o = static_cast<unsigned short*>(p.rid_n);
          while (x) {
            o[q++] = (unsigned short)(p.file_lo + (u32)(__ffsll((long long)x) - 1));
            x &= x - 1;
          }
        } else {
          while (x) {
            p.rid[q++] = p.file_lo + (u32)(__ffsll((long long)x) - 1);
            x &= x - 1;
          }
        }
      }
    }
    ba += ta;
    bb += tb;
  }
  if (big && p.rcnt32) atomicOr(reinterpret_cast<unsigned long long*>(p.tot + 2), 1ull);
}

// The root's plain words arrive sorted by (word, segment): a word of a
// many-file corpus has one entry per file (C3: up to 10^5), and one atomic
// per entry serialised them in one L2 slice (the C3 word count spent most of
// its 0.25 ms there).  A warp combines each run of equal keys first (sum of
// a, OR of b) and its last lane issues the run's atomics.  Every lane of the
// warp must call it (key ~0: no entry).
__device__ __forceinline__ void key_run_atomics(u64 key, u64 a, u64 b, u64* outA, u64* outB) {
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u64 oa = __shfl_up_sync(0xFFFFFFFFu, a, d), ob = __shfl_up_sync(0xFFFFFFFFu, b, d);
    const u64 ok = __shfl_up_sync(0xFFFFFFFFu, key, d);
    if (lane >= (unsigned)d && ok == key) {
      a += oa;
      b |= ob;
    }
  }
  const u64 nk = __shfl_down_sync(0xFFFFFFFFu, key, 1);
  if (key != ~0ull && (lane == 31 || nk != key)) {
    if (a && outA) atomicAdd((unsigned long long*)(outA + key), (unsigned long long)a);
    if (b && outB) atomicOr((unsigned long long*)(outB + key), (unsigned long long)b);
  }
}

template <class Mode, class T = u64>
__device__ __forceinline__ void seed_rows_body(const SeedArgs& a) {
  using V = typename Mode::V;
  constexpr bool pair = std::is_same<Mode, WcPresMode>::value;
  T* row = reinterpret_cast<T*>(a.row);
  const unsigned lane = threadIdx.x & 31u;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const bool is_or = std::is_same<Mode, OrMode>::value;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < a.n; base += stride) {
    const u64 i = base + threadIdx.x;
    u64 key = ~0ull;
    V v = Mode::zero();
    if (i < a.n) {
      const u32 sg = a.seg[i] - a.file_lo;
      if (sg < a.nseg) {
        const u64 r = a.rule[i];
        if constexpr (pair) {  // corpus weight + presence bit of the segment
          key = r;
          v = V{(u64)a.cnt[i], 1ull << (sg & 63u)};
        } else if (!a.per_file) {
          key = r;
          v = a.cnt[i];
        } else if (is_or) {
          key = r * a.C + (sg >> 6);
          v = 1ull << (sg & 63u);
        } else {
          key = r * a.C + sg;
          v = a.cnt[i];
        }
      }
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const V ov = shfl_up(v, d);
      const u64 ok = __shfl_up_sync(0xFFFFFFFFu, key, d);
      if (lane >= (unsigned)d && ok == key) v = Mode::merge(v, ov);
    }
    const u64 nk = __shfl_down_sync(0xFFFFFFFFu, key, 1);
    if (key != ~0ull && (lane == 31 || nk != key)) {
      if constexpr (pair) Mode::atomic(PairPtr{(u64*)row + 2 * key, (u64*)row + 2 * key + 1}, v);
      else Mode::atomic(&row[key], v);
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent level loop: ONE cooperative launch runs levels [L0, L1] of a
// level-ordered item list (lvl_off on the device), the whole grid resident
// and separated by grid-wide barriers instead of kernel boundaries.  Level
// sizes follow the DAG (a handful to 10^6 items), so the per-level work is
// re-dealt over all resident warps/teams each time.
// ---------------------------------------------------------------------------
constexpr int kLevelBlock = 1024;  // one block per SM: the grid barrier spans 148 arrivals

template <int G, class Mode, class Src, class Out>
__global__ void __launch_bounds__(kLevelBlock) k_segred_levels(const u32* __restrict__ dst,
                                                       const u32* __restrict__ src,
                                                       const u32* __restrict__ freq,
                                                       const u64* __restrict__ lvl_off, int L0, int L1,
                                                       int reverse, u32 C, Src in, Out out) {
  cg::grid_group grid = cg::this_grid();
  // teams numbered round-robin over the blocks (small levels reach every SM)
  const u64 gtid = ((u64)(threadIdx.x / G) * gridDim.x + blockIdx.x) * G + threadIdx.x % G;
  const u64 nthreads = (u64)gridDim.x * blockDim.x;
  for (int it = 0; it <= L1 - L0; it++) {
    const int L = reverse ? L1 - it : L0 + it;
    const u64 a = lvl_off[L], n = lvl_off[L + 1] - a;
    if (n) {
      if (G == 1) {
        const u64 nwarps = nthreads >> 5;
        int K = (int)((n + 32 * nwarps - 1) / (32 * nwarps));
        K = K < 1 ? 1 : (K > 16 ? 16 : K);
        segred1_body<Mode>(dst + a, src + a, freq ? freq + a : nullptr, n, K, in, out, gtid >> 5, nwarps);
      } else {
        const u64 teams = nthreads / G;
        u32 K = (u32)((n + teams - 1) / teams);
        K = K < 2 ? 2 : (K > 64 ? 64 : K);
        segredG_body<G, Mode, true>(dst + a, src + a, freq ? freq + a : nullptr, n, K, C, in, out, gtid, nthreads);
      }
    }
    if (it < L1 - L0) grid.sync();
  }
}

// C == 1 persistent level loop with the items of short levels (at most
// kPre 32-item steps per warp) prefetched into registers before the grid
// barrier that precedes them: item lists are static, so after the barrier
// only the row gathers, the warp scans and one reduction per run remain on
// the level's critical path.  Larger levels run the tiled body.  BLOCK
// threads per block, one block per SM: a smaller block shortens the
// block-wide part of every barrier (the C2 pass is 24 barrier-separated
// levels of ~5*10^4 items), a larger one keeps more gathers in flight on
// levels of 10^5-10^6 items.
template <int BLOCK, int kPre, class Mode, class Src, class Out>
__global__ void __launch_bounds__(BLOCK, 1) k_segred1_levels(const u32* __restrict__ dst,
                                                          const u32* __restrict__ src,
                                                          const u32* __restrict__ freq,
                                                          const u64* __restrict__ lvl_off, int L0, int L1,
                                                          int reverse, int prefetch, SeedArgs seed, PostArgs post,
                                                          Src in, Out out) {
  using V = typename Mode::V;
  constexpr bool pair = std::is_same<Mode, WcPresMode>::value;
  cg::grid_group grid = cg::this_grid();
  seg_stamp(post.stamps, 0);
  if (post.rcnt32 && blockIdx.x == 0 && threadIdx.x == 0) post.tot[2] = 0;  // read after the compaction
  if (seed.row) {  // phase 0: clear the rows (and the reduce output), then the root seeds
    u64* zr = reinterpret_cast<u64*>(seed.row);
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < seed.zero_n; i += (u64)gridDim.x * blockDim.x)
      zr[i] = 0;
    // (the reduce output is only written after many level barriers)
    if (post.out)
      for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < post.out_n; i += (u64)gridDim.x * blockDim.x) {
        post.out[i] = 0;
        if (pair) post.out2[i] = 0;
      }
    if (seed.zero_n) grid.sync();  // (zero_n == 0: the rows were cleared by the last step)
    seed_rows_body<Mode>(seed);
    grid.sync();
  }
  seg_stamp(post.stamps, 1);
  const u64 nthreads = (u64)gridDim.x * blockDim.x;
  // warps numbered round-robin over the blocks: a level smaller than the
  // grid is spread over every SM instead of filling the first blocks
  const u64 nwarps = nthreads >> 5, warp = (u64)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const unsigned lane = threadIdx.x & 31u;
  const int nit = L1 - L0 + 1;
  // this lane's items of a short level: steps p < pk of the warp's tile
  u32 pd[kPre], ps[kPre], pf[kPre];
  int pk = 0;
  auto fetch = [&](int it) {
    pk = 0;
    if (!prefetch || it >= nit) return;
    const int L = reverse ? L1 - it : L0 + it;
    const u64 a = lvl_off[L], n = lvl_off[L + 1] - a;
    const u64 K = (n + 32 * nwarps - 1) / (32 * nwarps);
    if (K > (u64)kPre) return;
    pk = K < 1 ? 1 : (int)K;
    const u64 t0 = a + warp * 32ull * pk + lane;
#pragma unroll
    for (int p = 0; p < kPre; p++) {
      const u64 i = t0 + 32ull * p;
      const bool ok = p < pk && i < a + n;
      pd[p] = ok ? dst[i] : 0xFFFFFFFFu;
      ps[p] = ok ? src[i] : 0u;
      pf[p] = ok ? (freq ? freq[i] : 1u) : 0u;
    }
  };
  fetch(0);
  for (int it = 0; it < nit; it++) {
    if (pk) {
      u32 dd[kPre];
      V vv[kPre];
      const int K = pk;
#pragma unroll
      for (int p = 0; p < kPre; p++) {
        dd[p] = pd[p];
        vv[p] = dd[p] != 0xFFFFFFFFu ? Mode::combine(pf[p], in(ps[p], 0)) : Mode::zero();
      }
      fetch(it + 1);  // the next level's items load while these gathers are in flight
      if (__any_sync(0xFFFFFFFFu, dd[0] != 0xFFFFFFFFu)) {
        u32 carry_d = 0xFFFFFFFFu;
        V carry_v = Mode::zero();
#pragma unroll
        for (int p = 0; p < kPre; p++) {
          if (p >= K) break;  // warp-uniform
          const u32 d = dd[p];
          V v = vv[p];
          const u32 d0 = __shfl_sync(0xFFFFFFFFu, d, 0);
          if (carry_d != 0xFFFFFFFFu && d0 != carry_d) {
            if (lane == 0) Mode::atomic(out(carry_d, 0), carry_v);
            carry_d = 0xFFFFFFFFu;
            carry_v = Mode::zero();
          }
#pragma unroll
          for (int s = 1; s < 32; s <<= 1) {
            const V ov = shfl_up(v, s);
            const u32 od = __shfl_up_sync(0xFFFFFFFFu, d, s);
            if (lane >= (unsigned)s && od == d) v = Mode::merge(v, ov);
          }
          if (d == carry_d) v = Mode::merge(v, carry_v);
          const u32 dn = __shfl_down_sync(0xFFFFFFFFu, d, 1);
          if (d != 0xFFFFFFFFu && lane != 31 && dn != d) Mode::atomic(out(d, 0), v);
          carry_d = __shfl_sync(0xFFFFFFFFu, d, 31);
          carry_v = shfl_idx(v, 31);
        }
        if (lane == 0 && carry_d != 0xFFFFFFFFu) Mode::atomic(out(carry_d, 0), carry_v);
      }
    } else {
      const int L = reverse ? L1 - it : L0 + it;
      const u64 a = lvl_off[L], n = lvl_off[L + 1] - a;
      if (n) {
        int K = (int)((n + 32 * nwarps - 1) / (32 * nwarps));
        K = K < 1 ? 1 : (K > 16 ? 16 : K);
        segred1_body<Mode>(dst + a, src + a, freq ? freq + a : nullptr, n, K, in, out, warp, nwarps);
      }
      fetch(it + 1);
    }
    if (it + 1 < nit) grid.sync();
    seg_stamp(post.stamps, 2 + it);
  }
  if (post.out) {  // the word reduce over the finished rows
    grid.sync();
    seg_stamp(post.stamps, 2 + nit);
    if (post.n) {
      int K = (int)((post.n + 32 * nwarps - 1) / (32 * nwarps));
      K = K < 1 ? 1 : (K > 16 ? 16 : K);
      if constexpr (pair)
        segred1_body<Mode>(post.dst, post.src, post.freq, post.n, K, in, OutPair{post.out, post.out2}, warp, nwarps);
      else
        segred1_body<Mode>(post.dst, post.src, post.freq, post.n, K, in, OutColMajorT<u64>{post.out, post.out_n},
                           warp, nwarps);
    }
    const bool is_or = std::is_same<Mode, OrMode>::value;
    // (one atomic per run of a word within a warp: key_run_atomics)
    for (u64 b0 = ((u64)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull; b0 < post.n_rw; b0 += nthreads) {
      const u64 i = b0 + (threadIdx.x & 31u);
      u64 key = ~0ull, a = 0, bits = 0;
      if (i < post.n_rw) {
        const u32 sg = post.rw_seg[i] - post.file_lo;
        if (sg < post.nseg) {
          key = post.rw_word[i];
          if (pair) a = post.rw_cnt[i], bits = 1ull << (sg & 63u);
          else if (is_or) bits = post.per_file ? 1ull << (sg & 63u) : 1ull;
          else a = post.rw_cnt[i];
        }
      }
      key_run_atomics(key, a, bits, is_or ? nullptr : post.out, pair ? post.out2 : (is_or ? post.out : nullptr));
    }
    if (post.compact) {
      grid.sync();
      seg_stamp(post.stamps, 3 + nit);
      // the rows are read by no one after the reduce: clear them for the
      // next step (the compaction only reads the outputs)
      for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < post.zero_tail_n; i += nthreads)
        post.zero_tail[i] = 0;
      post_compact(post, grid);
      seg_stamp(post.stamps, 4 + nit);
    }
  }
}

// Items per warp tile / team chunk: as large as possible (fewer boundary
// atomics, longer carried runs) while still giving every SM a full load of
// resident threads; small levels therefore run one step per warp instead of
// a handful of warps walking long tiles serially.
constexpr u64 kResidentThreads = 148ull * 2048ull;

inline u64 pow2_floor(u64 x) {
  u64 p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

// host launcher: picks the variant for C columns; n == 0 is a no-op.
template <class Mode, class Src, class Out>
void seg_reduce(const char* name, const u32* dst, const u32* src, const u32* freq, u64 n, u32 C,
                Src in, Out out, cudaStream_t st) {
  if (!n || !C) return;
  if (C == 1) {
    const int K = (int)std::min<u64>(16, std::max<u64>(1, pow2_floor(n / kResidentThreads)));
    const u64 tiles = (n + 32ull * K - 1) / (32ull * K);
    GT_KLAUNCH(name, (k_segred1<Mode, Src, Out>), grid_for(tiles * 32, 256, 148u * 32u), 256, st,
               dst, src, freq, n, K, in, out);
    return;
  }
#define GT_SEGRED_G(GG)                                                                           \
  do {                                                                                            \
    const u32 K = (u32)std::min<u64>(64, std::max<u64>(8, pow2_floor(n * GG / kResidentThreads))); \
    const u64 chunks = (n + K - 1) / K;                                                           \
    GT_KLAUNCH(name, (k_segredG<GG, Mode, Src, Out>), grid_for(chunks * GG, 256, 148u * 64u), 256, \
               st, dst, src, freq, n, K, C, in, out);                                             \
  } while (0)
  if (C <= 2) GT_SEGRED_G(2);
  else if (C <= 4) GT_SEGRED_G(4);
  else if (C <= 8) GT_SEGRED_G(8);
  else if (C <= 16) GT_SEGRED_G(16);
  else GT_SEGRED_G(32);
#undef GT_SEGRED_G
}

// Host launcher of the persistent level loop: levels [L0, L1] of the item
// list (dst/src/freq base pointers; lvl_off_dev = device copy of the level
// offsets).  One cooperative launch with every block resident.
template <int G, class Mode, class Src, class Out>
void seg_reduce_levels_G(const char* name, const u32* dst, const u32* src, const u32* freq,
                         const u64* lvl_off_dev, int L0, int L1, int reverse, u32 C, Src in, Out out,
                         cudaStream_t st) {
  auto kern = k_segred_levels<G, Mode, Src, Out>;
  static int per_sm = -1;  // per instantiation
  if (per_sm < 0) {
    GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLevelBlock, 0));
    if (per_sm < 1) per_sm = 1;
  }
  int dev = 0, nsm = 148;
  GT_CUDA(cudaGetDevice(&dev));
  GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  dim3 grid((unsigned)(nsm * per_sm)), block(kLevelBlock);
  void* args[] = {(void*)&dst, (void*)&src, (void*)&freq, (void*)&lvl_off_dev, (void*)&L0, (void*)&L1,
                  (void*)&reverse, (void*)&C, (void*)&in, (void*)&out};
  ProfScope ps(name, st);
  GT_CUDA(cudaLaunchCooperativeKernel((const void*)kern, grid, block, args, 0, st));
  g_launches++;
}


// ---------------------------------------------------------------------------
// Persistent level loop with TMA-staged items (C == 1).  Each block owns an
// even slice of every level; its slices are cut into chunks of at most kTmaCh
// items whose (dst, src, freq) arrays are brought into shared memory by 1-D
// bulk copies (cp.async.bulk ... mbarrier::complete_tx) double-buffered one
// chunk ahead — including ACROSS the grid barrier, since the item lists are
// static: after a barrier the block's first chunk of the next level is
// already in shared memory and only the row gathers remain on the critical
// path.  Runs are combined per 32-item warp step (shuffle segmented scan) and
// flushed with one reduction each.
// ---------------------------------------------------------------------------
constexpr int kTmaBlock = 1024;
constexpr u32 kTmaCh = 4096;             // items per staged chunk
constexpr u32 kTmaPad = kTmaCh + 8;      // + alignment slack (16-byte aligned copies)

__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct TmaUnit {
  int it;  // level iteration index (0-based), -1 = none
  u64 s, e;
};

template <class Mode, class Src, class Out>
__global__ void __launch_bounds__(kTmaBlock) k_levels_tma(const u32* __restrict__ dst, const u32* __restrict__ src,
                                                          const u32* __restrict__ freq,
                                                          const u64* __restrict__ lvl_off, int L0, int L1,
                                                          int reverse, Src in, Out out) {
  extern __shared__ __align__(128) u32 tma_smem[];
  __shared__ __align__(8) u64 bars[2];
  cg::grid_group grid = cg::this_grid();
  const int narr = freq ? 3 : 2;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int nlev = L1 - L0 + 1;
  auto level_of = [&](int it) { return reverse ? L1 - it : L0 + it; };
  // the block's slice of level iteration `it`
  auto slice = [&](int it, u64* s0, u64* s1) {
    const int L = level_of(it);
    const u64 a = lvl_off[L], n = lvl_off[L + 1] - a;
    const u64 S = (n + gridDim.x - 1) / gridDim.x;
    *s0 = a + min(n, (u64)blockIdx.x * S);
    *s1 = a + min(n, (u64)(blockIdx.x + 1) * S);
  };
  // the unit after (it, end e) in this block's sequence
  auto next_unit = [&](int it, u64 e) {
    TmaUnit u{-1, 0, 0};
    u64 s0, s1;
    slice(it, &s0, &s1);
    if (e < s1) return TmaUnit{it, e, min(s1, e + kTmaCh)};
    for (int j = it + 1; j < nlev; j++) {
      slice(j, &s0, &s1);
      if (s1 > s0) return TmaUnit{j, s0, min(s1, s0 + kTmaCh)};
    }
    return u;
  };
  auto first_unit = [&]() {
    for (int j = 0; j < nlev; j++) {
      u64 s0, s1;
      slice(j, &s0, &s1);
      if (s1 > s0) return TmaUnit{j, s0, min(s1, s0 + kTmaCh)};
    }
    return TmaUnit{-1, 0, 0};
  };
  auto buf = [&](int b, int arr) { return tma_smem + ((u64)b * 3 + arr) * kTmaPad; };
  // one elected thread arms the buffer's barrier and issues the bulk copies
  auto issue = [&](const TmaUnit& u, int b) {
    if (threadIdx.x != 0 || u.it < 0) return;
    // the buffer was last read through the generic proxy (ordered by the
    // block barrier); order those reads before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const u64 a4 = u.s & ~3ull, e4 = (u.e + 3) & ~3ull;
    const u32 bytes = (u32)((e4 - a4) * 4);
    mbar_expect_tx(&bars[b], bytes * narr);
    bulk_g2s(buf(b, 0), dst + a4, bytes, &bars[b]);
    bulk_g2s(buf(b, 1), src + a4, bytes, &bars[b]);
    if (freq) bulk_g2s(buf(b, 2), freq + a4, bytes, &bars[b]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  TmaUnit cur = first_unit();
  issue(cur, 0);
  u32 q = 0;  // sequence number of `cur`: buffer q & 1, parity (q >> 1) & 1
  for (int it = 0; it < nlev; it++) {
    while (cur.it == it) {
      const TmaUnit nxt = next_unit(cur.it, cur.e);
      issue(nxt, (q + 1) & 1);  // the other buffer was released at the end of the last unit
      const int b = q & 1;
      mbar_wait(&bars[b], (q >> 1) & 1);
      const u64 a4 = cur.s & ~3ull;
      const u32* sd = buf(b, 0);
      const u32* ss = buf(b, 1);
      const u32* sf = freq ? buf(b, 2) : nullptr;
      for (u64 base = cur.s + (u64)warp * 32; base < cur.e; base += (u64)nwarp * 32) {
        const u64 i = base + lane;
        const bool ok = i < cur.e;
        const u32 d = ok ? sd[i - a4] : 0xFFFFFFFFu;
        u64 v = ok ? Mode::combine(sf ? sf[i - a4] : 1u, in(ss[i - a4], 0)) : 0;
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
          const u64 ov = __shfl_up_sync(0xFFFFFFFFu, v, k);
          const u32 od = __shfl_up_sync(0xFFFFFFFFu, d, k);
          if (lane >= (unsigned)k && od == d) v = Mode::merge(v, ov);
        }
        const u32 dn = __shfl_down_sync(0xFFFFFFFFu, d, 1);
        if (ok && (lane == 31 || dn != d)) Mode::atomic(out(d, 0), v);
      }
      __syncthreads();  // buffer b is free again
      cur = nxt;
      q++;
    }
    if (it + 1 < nlev) grid.sync();
  }
}

// host launcher of the TMA-staged loop (C == 1)
template <class Mode, class Src, class Out>
void seg_reduce_levels_tma(const char* name, const u32* dst, const u32* src, const u32* freq,
                           const u64* lvl_off_dev, int L0, int L1, Src in, Out out, cudaStream_t st,
                           bool reverse) {
  auto kern = k_levels_tma<Mode, Src, Out>;
  const size_t smem = (size_t)2 * 3 * kTmaPad * 4;
  static int per_sm = -1;  // per instantiation
  if (per_sm < 0) {
    GT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTmaBlock, smem));
    if (per_sm < 1) per_sm = 1;
  }
  int dev = 0, nsm = 148;
  GT_CUDA(cudaGetDevice(&dev));
  GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  int rv = reverse ? 1 : 0;
  void* args[] = {(void*)&dst, (void*)&src, (void*)&freq, (void*)&lvl_off_dev, (void*)&L0, (void*)&L1,
                  (void*)&rv, (void*)&in, (void*)&out};
  ProfScope ps(name, st);
  GT_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)(nsm * per_sm)), dim3(kTmaBlock), args,
                                      smem, st));
  g_launches++;
}

template <int BLOCK, int PRE, class Mode, class Src, class Out>
void seg_reduce_levels1_b(const char* name, const u32* dst, const u32* src, const u32* freq,
                          const u64* lvl_off_dev, int L0, int L1, int reverse, int prefetch, const SeedArgs* seed,
                          const PostArgs* post, Src in, Out out, cudaStream_t st) {
  auto kern = k_segred1_levels<BLOCK, PRE, Mode, Src, Out>;
  int dev = 0, nsm = 148;
  GT_CUDA(cudaGetDevice(&dev));
  GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  SeedArgs sa = seed ? *seed : SeedArgs{};
  PostArgs pa = post ? *post : PostArgs{};
  void* args[] = {(void*)&dst, (void*)&src, (void*)&freq, (void*)&lvl_off_dev, (void*)&L0, (void*)&L1,
                  (void*)&reverse, (void*)&prefetch, (void*)&sa, (void*)&pa, (void*)&in, (void*)&out};
  ProfScope ps(name, st);
  GT_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)nsm), dim3(BLOCK), args, 0, st));
  g_launches++;
}

// avg_items: mean items per level (host-side hint).  Levels of at most one
// 32-item step per warp are the common case on shallow-fan-out DAGs (C2:
// ~5*10^4 items over 24 levels) and prefetch one step; DAGs whose levels
// run several steps per warp (C4/C5: 10^5-10^6) prefetch up to four.
// Measured per pass: C2 94 -> 70 us, C4 0.39 -> 0.36 ms, C5 0.70 -> 0.68 ms.
template <class Mode, class Src, class Out>
void seg_reduce_levels1(const char* name, const u32* dst, const u32* src, const u32* freq,
                        const u64* lvl_off_dev, int L0, int L1, int reverse, u64 avg_items, const SeedArgs* seed,
                        const PostArgs* post, Src in, Out out, cudaStream_t st) {
  static const int prefetch = getenv("GT_LEVEL_PREFETCH") ? atoi(getenv("GT_LEVEL_PREFETCH")) : 1;
  static const int force_pre = getenv("GT_LEVEL_PRE") ? atoi(getenv("GT_LEVEL_PRE")) : 0;
  const int pre = force_pre ? force_pre : (avg_items > 148ull * kLevelBlock ? 4 : 1);
  if (pre == 4)
    seg_reduce_levels1_b<kLevelBlock, 4, Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, reverse, prefetch, seed,
                                               post, in, out, st);
  else
    seg_reduce_levels1_b<kLevelBlock, 1, Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, reverse, prefetch, seed,
                                               post, in, out, st);
}

// levels [L0, L1] in increasing order, or decreasing with reverse = true
template <class Mode, class Src, class Out>
void seg_reduce_levels(const char* name, const u32* dst, const u32* src, const u32* freq,
                       const u64* lvl_off_dev, int L0, int L1, u32 C, Src in, Out out, cudaStream_t st,
                       bool reverse = false, u64 avg_items = 0, const SeedArgs* seed = nullptr,
                       const PostArgs* post = nullptr) {
  // seed (C == 1 only): zero + seed the rows as phase 0 of the same launch
  if (!C) return;
  if (L1 < L0 && !seed) return;
  const int rv = reverse ? 1 : 0;
  // the TMA-staged variant is opt-in: measured slower on every config (C2 top-
  // down pass 0.223 vs 0.188 ms per step, C5 0.73 vs 0.68 ms) — the item
  // loads it hides are not on the critical path; the row gathers and the
  // grid barrier are
  static const bool use_tma = getenv("GT_LEVELS_TMA") != nullptr;
  if (C == 1 && use_tma && !seed && !post)
    seg_reduce_levels_tma<Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, in, out, st, reverse);
  else if (C == 1) seg_reduce_levels1<Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, rv, avg_items, seed, post, in, out, st);
  else if (C <= 2) seg_reduce_levels_G<2, Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, rv, C, in, out, st);
  else if (C <= 4) seg_reduce_levels_G<4, Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, rv, C, in, out, st);
  else if (C <= 8) seg_reduce_levels_G<8, Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, rv, C, in, out, st);
  else if (C <= 16) seg_reduce_levels_G<16, Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, rv, C, in, out, st);
  else seg_reduce_levels_G<32, Mode>(name, dst, src, freq, lvl_off_dev, L0, L1, rv, C, in, out, st);
}

}  // namespace gt
