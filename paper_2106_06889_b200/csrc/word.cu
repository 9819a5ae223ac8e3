// word.cu — word-level analytics on the device DAG (top-down strategy).
//
// Reference algorithm (engine.py:178-302, _kernels.py:129-188): Alg. 1
// top-down weight propagation in mask rounds, then Σ own_freq·weight into
// hash tables plus a scan of the root's plain words.  B200 formulation:
//   * rounds become precomputed levels (loader.cu); each level is ONE pull
//     launch: a rule reads its parents' finished rows (par CSR, parents
//     ascending) — no atomics, no masks, no host round trip.  Light rules
//     get a team of G lanes (one lane per weight column), heavy rules
//     (>16 parents) a whole warp whose stripes split the parent list and
//     are combined with shuffles (the paper's split of high-fan-out work).
//   * root occurrences seed the rows from the (rule, segment) list, so the
//     same kernel serves corpus-global weights (1 column = all owned files),
//     per-file weights (F columns) and per-file presence bitsets (OR mode,
//     ceil(F/64) 64-bit columns; exact for inverted index, which only needs
//     presence: 8 B per rule instead of 8·F B).
//   * the reduce is a pull over the word-major transpose of the own pairs:
//     a reduce-by-key over (word, rule, freq) entries sorted by word, with
//     plain stores for runs interior to a tile and atomics only for runs
//     crossing a tile boundary (hot Zipf words cost one atomic per tile, not
//     one per occurrence).  Root words come from the (word, segment) list.
#include <algorithm>
#include <type_traits>

#include "kernels_common.cuh"
#include "word.cuh"

namespace gt {

struct SumMode {
  __device__ static __forceinline__ u64 combine(u64 acc, u32 f, u64 x) { return acc + (u64)f * x; }
  __device__ static __forceinline__ u64 merge(u64 a, u64 b) { return a + b; }
  __device__ static __forceinline__ void seed(u64& acc, u32 col, u32 seg_rel, u32 cnt) {
    if (seg_rel == col) acc += cnt;
  }
  __device__ static __forceinline__ void atomic(u64* p, u64 v) {
    if (v) atomicAdd((unsigned long long*)p, (unsigned long long)v);
  }
};

struct OrMode {
  __device__ static __forceinline__ u64 combine(u64 acc, u32, u64 x) { return acc | x; }
  __device__ static __forceinline__ u64 merge(u64 a, u64 b) { return a | b; }
  __device__ static __forceinline__ void seed(u64& acc, u32 col, u32 seg_rel, u32) {
    if ((seg_rel >> 6) == col) acc |= 1ull << (seg_rel & 63u);
  }
  __device__ static __forceinline__ void atomic(u64* p, u64 v) {
    if (v) atomicOr((unsigned long long*)p, (unsigned long long)v);
  }
};

template <class Mode>
__device__ __forceinline__ u64 seed1(u64 acc, u32 col, u32 sg, u32 cnt) {
  Mode::seed(acc, col, sg, cnt);
  return acc;
}

// ---------------------------------------------------------------------------
// level pull: rows out[c*C .. c*C+C) for the rules of one top-down level
//   row(c) = seed(c) (+|) Σ_{p in parents(c), p != 0} f(p,c) · row(p)
// ---------------------------------------------------------------------------
template <int G, class Mode>
__global__ void __launch_bounds__(256) k_td_level(const u32* __restrict__ order, u64 lo, u64 mid,
                                                  u64 hi, const u64* __restrict__ par_off,
                                                  const u32* __restrict__ par_ids,
                                                  const u32* __restrict__ par_freqs,
                                                  const u64* __restrict__ rs_off,
                                                  const u32* __restrict__ rs_seg,
                                                  const u32* __restrict__ rs_cnt, u32 file_lo,
                                                  u32 nseg, u32 C, u32 per_file,
                                                  u64* __restrict__ row) {
  const u64 gtid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 nthreads = (u64)gridDim.x * blockDim.x;
  const unsigned lane = threadIdx.x & 31u;
  const u64 nlight = mid - lo;
  // light rules: one team of G lanes per rule
  {
    const u64 teams = nthreads / G;
    const u32 tl = lane % G;
    for (u64 t = gtid / G; t < nlight; t += teams) {
      const u32 c = order[lo + t];
      const u64 e0 = par_off[c], e1 = par_off[c + 1];
      const u64 s0 = rs_off[c], s1 = rs_off[c + 1];
      for (u32 col = tl; col < C; col += G) {
        u64 acc = 0;
        for (u64 s = s0; s < s1; s++) {
          u32 sg = rs_seg[s] - file_lo;
          if (sg < nseg) acc = per_file ? seed1<Mode>(acc, col, sg, rs_cnt[s]) : Mode::merge(acc, (u64)rs_cnt[s]);
        }
        for (u64 e = e0; e < e1; e++) {
          const u32 p = par_ids[e];
          if (p) acc = Mode::combine(acc, par_freqs[e], row[(u64)p * C + col]);
        }
        row[(u64)c * C + col] = acc;
      }
    }
  }
  // heavy rules: one warp per rule; 32/G stripes split the parent list
  {
    constexpr u32 S = 32 / G;
    const u64 nheavy = hi - mid;
    const u64 nw = nthreads >> 5;
    const u32 col0 = lane % G, stripe = lane / G;
    for (u64 w = gtid >> 5; w < nheavy; w += nw) {
      const u32 c = order[mid + w];
      const u64 e0 = par_off[c], e1 = par_off[c + 1];
      const u64 s0 = rs_off[c], s1 = rs_off[c + 1];
      for (u32 cb = 0; cb < C; cb += G) {
        const u32 col = cb + col0;
        const bool ok = col < C;
        u64 acc = 0;
        if (ok) {
          for (u64 e = e0 + stripe; e < e1; e += S) {
            const u32 p = par_ids[e];
            if (p) acc = Mode::combine(acc, par_freqs[e], row[(u64)p * C + col]);
          }
        }
#pragma unroll
        for (u32 d = G; d < 32; d <<= 1) acc = Mode::merge(acc, __shfl_xor_sync(0xFFFFFFFFu, acc, d));
        if (ok && stripe == 0) {
          for (u64 s = s0; s < s1; s++) {
            u32 sg = rs_seg[s] - file_lo;
            if (sg < nseg) acc = per_file ? seed1<Mode>(acc, col, sg, rs_cnt[s]) : Mode::merge(acc, (u64)rs_cnt[s]);
          }
          row[(u64)c * C + col] = acc;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// reduce-by-word, one column (global word count / F<=64 presence):
//   out[v] = Σ_{(v,r,f) in ow, r != 0} f · row[r]   (Mode combine)
// warp tiles of 32*K entries; runs interior to a tile are stored, runs that
// touch a tile boundary are combined atomically.
// ---------------------------------------------------------------------------
template <int K, class Mode>
__global__ void __launch_bounds__(256) k_reduce_words_1(const u32* __restrict__ ow_word,
                                                        const u32* __restrict__ ow_rule,
                                                        const u32* __restrict__ ow_freq, u64 n,
                                                        const u64* __restrict__ row,
                                                        u64* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31u;
  const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  constexpr u64 TILE = 32ull * K;
  for (u64 t0 = warp * TILE; t0 < n; t0 += nwarps * TILE) {
    const u32 first_word = ow_word[t0];
    u32 carry_w = 0xFFFFFFFFu;
    u64 carry_v = 0;
#pragma unroll 4
    for (int k = 0; k < K; k++) {
      const u64 i = t0 + (u64)k * 32 + lane;
      const bool ok = i < n;
      const u32 wd = ok ? ow_word[i] : 0xFFFFFFFFu;
      const u32 w0 = __shfl_sync(0xFFFFFFFFu, wd, 0);
      if (carry_w != 0xFFFFFFFFu && w0 != carry_w) {  // carried run ended at the previous step
        if (lane == 0) {
          if (carry_w == first_word) Mode::atomic(&out[carry_w], carry_v);
          else out[carry_w] = carry_v;
        }
        carry_w = 0xFFFFFFFFu;
        carry_v = 0;
      }
      u64 v = 0;
      if (ok) {
        const u32 r = ow_rule[i];
        if (r) v = Mode::combine(0, ow_freq[i], row[r]);
      }
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        u64 ov = __shfl_up_sync(0xFFFFFFFFu, v, d);
        u32 ow = __shfl_up_sync(0xFFFFFFFFu, wd, d);
        if (lane >= (unsigned)d && ow == wd) v = Mode::merge(v, ov);
      }
      if (wd == carry_w) v = Mode::merge(v, carry_v);
      const u32 nxt = __shfl_down_sync(0xFFFFFFFFu, wd, 1);
      const bool last = lane == 31 || nxt != wd;
      if (ok && last && lane != 31) {
        if (wd == first_word) Mode::atomic(&out[wd], v);
        else out[wd] = v;
      }
      carry_w = __shfl_sync(0xFFFFFFFFu, wd, 31);
      carry_v = __shfl_sync(0xFFFFFFFFu, v, 31);
    }
    if (lane == 0 && carry_w != 0xFFFFFFFFu) Mode::atomic(&out[carry_w], carry_v);
  }
}

// reduce-by-word, C columns: team of G lanes walks a chunk of K entries
//   out[col*V + v] = Σ f · row[r*C + col]
template <int G, int K, class Mode>
__global__ void __launch_bounds__(256) k_reduce_words_cols(const u32* __restrict__ ow_word,
                                                           const u32* __restrict__ ow_rule,
                                                           const u32* __restrict__ ow_freq,
                                                           u64 n, const u64* __restrict__ row,
                                                           u32 C, u64 V, u64* __restrict__ out) {
  const u64 gtid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 teams = ((u64)gridDim.x * blockDim.x) / G;
  const u32 tl = threadIdx.x % G;
  for (u64 t = gtid / G; t * K < n; t += teams) {
    const u64 a = t * K, b = min(n, a + K);
    const u32 wfirst = ow_word[a];
    const u32 wlast = ow_word[b - 1];
    const bool shared_first = a > 0 && ow_word[a - 1] == wfirst;
    const bool shared_last = b < n && ow_word[b] == wlast;
    for (u32 col = tl; col < C; col += G) {
      u32 cw = wfirst;
      u64 acc = 0;
      for (u64 i = a; i < b; i++) {
        const u32 wd = ow_word[i];
        if (wd != cw) {
          u64* dst = &out[(u64)col * V + cw];
          if (cw == wfirst && shared_first) Mode::atomic(dst, acc);
          else *dst = acc;
          cw = wd;
          acc = 0;
        }
        const u32 r = ow_rule[i];
        if (r) acc = Mode::combine(acc, ow_freq[i], row[(u64)r * C + col]);
      }
      u64* dst = &out[(u64)col * V + cw];
      if ((cw == wfirst && shared_first) || shared_last) Mode::atomic(dst, acc);
      else *dst = acc;
    }
  }
}

// root words of owned segments: (word, seg, cnt) sorted by word
template <class Mode>
__global__ void k_root_words(const u32* __restrict__ rw_word, const u32* __restrict__ rw_seg,
                             const u32* __restrict__ rw_cnt, u64 n, u32 file_lo, u32 nseg,
                             int per_file, u32 C, u64 V, u64* __restrict__ out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 sg = rw_seg[i] - file_lo;
    if (sg >= nseg) continue;
    u32 w = rw_word[i];
    if (!per_file) {
      Mode::atomic(&out[w], Mode::combine(0, rw_cnt[i], 1ull));
    } else {
      u64 acc = 0;
      u32 col = std::is_same<Mode, OrMode>::value ? (sg >> 6) : sg;
      Mode::seed(acc, col, sg, rw_cnt[i]);
      Mode::atomic(&out[(u64)col * V + w], acc);
    }
  }
}

// ---------------------------------------------------------------------------
// assembly
// ---------------------------------------------------------------------------
__global__ void k_nonzero_flags(const u64* v, u64 n, uint8_t* f) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) f[i] = v[i] != 0;
}

// records from selected indices: id = idx % V (word), count, file = idx / V
__global__ void k_records(const u32* sel, const u64* nsel, const u64* vals, u64 V, u32* id,
                          u64* cnt, u32* file) {
  u64 n = *nsel;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 j = sel[i];
    id[i] = (u32)(j % V);
    cnt[i] = vals[j];
    if (file) file[i] = (u32)(j / V);
  }
}

// sort keys: (file << CB) | (W - count)  -> (file asc, count desc), stable on word
__global__ void k_sort_keys(const u64* cnt, const u32* file, u64 n, u64 W, int CB, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = ((file ? (u64)file[i] : 0ull) << CB) | (W - cnt[i]);
}

__global__ void k_unkey(const u64* key, u64 n, u64 W, int CB, u64* cnt) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  u64 m = (CB >= 64) ? ~0ull : ((1ull << CB) - 1);
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    cnt[i] = W - (key[i] & m);
}

// presence bitsets -> per-word file counts
__global__ void k_popc(const u64* pres, u64 V, u32 FW, u64* pc, uint8_t* nz) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 v = (u64)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride) {
    u64 c = 0;
    for (u32 j = 0; j < FW; j++) c += __popcll(pres[(u64)j * V + v]);
    pc[v] = c;
    nz[v] = c != 0;
  }
}

__global__ void k_ii_write(const u32* words, const u64* ngroups, const u64* pres, const u64* pc_off,
                           u64 V, u32 FW, u32 file_lo, u32* gid, u64* goff, u32* files) {
  u64 n = *ngroups;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += stride) {
    u32 v = words[g];
    gid[g] = v;
    u64 o = pc_off[v];
    goff[g] = o;
    for (u32 j = 0; j < FW; j++) {
      u64 b = pres[(u64)j * V + v];
      while (b) {
        int t = __ffsll((long long)b) - 1;
        files[o++] = file_lo + j * 64 + (u32)t;
        b &= b - 1;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------

#define KL(k, grid, ...) GT_KLAUNCH(#k, k, grid, 256, st, __VA_ARGS__)

template <int G, class Mode>
static void td_levels_G(const DeviceDag* d, u32 C, u32 per_file, u64* row) {
  cudaStream_t st = d->stream;
  const u32 nseg = (u32)(d->file_hi - d->file_lo);
  for (int L = 1; L <= d->td.nl; L++) {
    u64 lo = d->td.off[L], mid = d->td.heavy_off[L], hi = d->td.off[L + 1];
    if (hi == lo) continue;
    u64 work = (mid - lo) * G + (hi - mid) * 32;
    KL((k_td_level<G, Mode>), grid_for(work, 256, 148u * 64u), d->td.order.as<u32>(), lo, mid, hi,
       d->par_off.as<u64>(), d->par_ids.as<u32>(), d->par_freqs.as<u32>(), d->rs_off.as<u64>(),
       d->rs_seg.as<u32>(), d->rs_cnt.as<u32>(), (u32)d->file_lo, nseg, C, per_file, row);
  }
}

template <class Mode>
static void td_levels(const DeviceDag* d, u32 C, u64* row, u32 per_file = 1) {
  // root row stays zero: its own words are counted per segment (rw lists)
  GT_CUDA(cudaMemsetAsync(row, 0, sizeof(u64) * C, d->stream));
  if (C <= 1) td_levels_G<1, Mode>(d, C, per_file, row);
  else if (C <= 2) td_levels_G<2, Mode>(d, C, per_file, row);
  else if (C <= 4) td_levels_G<4, Mode>(d, C, per_file, row);
  else if (C <= 8) td_levels_G<8, Mode>(d, C, per_file, row);
  else if (C <= 16) td_levels_G<16, Mode>(d, C, per_file, row);
  else td_levels_G<32, Mode>(d, C, per_file, row);
}

template <class Mode>
static void reduce_words(const DeviceDag* d, u32 C, const u64* row, u64* out, bool per_file) {
  cudaStream_t st = d->stream;
  const u64 V = d->nw, n = d->E_own;
  GT_CUDA(cudaMemsetAsync(out, 0, sizeof(u64) * V * C, st));
  if (n) {
    if (C == 1) {
      constexpr int K = 16;
      u64 tiles = (n + 32 * K - 1) / (32 * K);
      KL((k_reduce_words_1<K, Mode>), grid_for(tiles * 32, 256, 148u * 16u), d->ow_word.as<u32>(),
         d->ow_rule.as<u32>(), d->ow_freq.as<u32>(), n, row, out);
    } else {
      constexpr int K = 64;
      u64 chunks = (n + K - 1) / K;
      if (C <= 8) KL((k_reduce_words_cols<8, K, Mode>), grid_for(chunks * 8, 256, 148u * 32u), d->ow_word.as<u32>(), d->ow_rule.as<u32>(), d->ow_freq.as<u32>(), n, row, C, V, out);
      else if (C <= 16) KL((k_reduce_words_cols<16, K, Mode>), grid_for(chunks * 16, 256, 148u * 32u), d->ow_word.as<u32>(), d->ow_rule.as<u32>(), d->ow_freq.as<u32>(), n, row, C, V, out);
      else KL((k_reduce_words_cols<32, K, Mode>), grid_for(chunks * 32, 256, 148u * 32u), d->ow_word.as<u32>(), d->ow_rule.as<u32>(), d->ow_freq.as<u32>(), n, row, C, V, out);
    }
  }
  if (d->n_rw)
    KL(k_root_words<Mode>, grid_for(d->n_rw, 256), d->rw_word.as<u32>(), d->rw_seg.as<u32>(),
       d->rw_cnt.as<u32>(), d->n_rw, (u32)d->file_lo, (u32)(d->file_hi - d->file_lo),
       per_file ? 1 : 0, C, V, out);
}

// global word counts (corpus or owned shard) -> dense u64[V]
void td_word_counts(DeviceDag* d, DBuf& counts) {
  cudaStream_t st = d->stream;
  DBuf w(d->R * 8, st);
  td_levels<SumMode>(d, 1, w.as<u64>(), 0);
  counts.alloc(d->nw * 8 + 8, st);
  reduce_words<SumMode>(d, 1, w.as<u64>(), counts.as<u64>(), false);
}

// per-file counts -> dense u64[Fo][V]
void td_file_counts(DeviceDag* d, DBuf& counts) {
  cudaStream_t st = d->stream;
  const u32 C = (u32)(d->file_hi - d->file_lo);
  DBuf w(d->R * 8 * (u64)std::max<u32>(C, 1), st);
  td_levels<SumMode>(d, C, w.as<u64>());
  counts.alloc(d->nw * 8 * (u64)std::max<u32>(C, 1) + 8, st);
  reduce_words<SumMode>(d, C, w.as<u64>(), counts.as<u64>(), true);
}

// per-file weights only -> u64[R][Fo]
void td_file_weights(DeviceDag* d, DBuf& w, u32* C_out) {
  const u32 C = std::max<u32>(1, (u32)(d->file_hi - d->file_lo));
  w.alloc(d->R * 8 * (u64)C, d->stream);
  td_levels<SumMode>(d, C, w.as<u64>());
  *C_out = C;
}

// per-file presence bitsets -> dense u64[FW][V]
void td_file_presence(DeviceDag* d, DBuf& pres, u32* FW_out) {
  cudaStream_t st = d->stream;
  const u32 Fo = (u32)(d->file_hi - d->file_lo);
  const u32 FW = std::max<u32>(1, (Fo + 63) / 64);
  DBuf m(d->R * 8 * (u64)FW, st);
  td_levels<OrMode>(d, FW, m.as<u64>());
  pres.alloc(d->nw * 8 * (u64)FW + 8, st);
  reduce_words<OrMode>(d, FW, m.as<u64>(), pres.as<u64>(), true);
  *FW_out = FW;
}

// ---- assembly -------------------------------------------------------------

void assemble_counts(DeviceDag* d, const u64* dense, u64 V, u32 ncols, bool by_count, DevRecords* R) {
  // ncols == 0: one global table; ncols >= 1: per-file tables (file-major)
  cudaStream_t st = d->stream;
  const bool pf = ncols > 0;
  const u64 N = V * (u64)(pf ? ncols : 1);
  if (N >= (1ull << 32)) fail(GT_E_RESOURCE, "dense per-file table of %lu entries exceeds 2^32; use the bottom-up strategy", (unsigned long)N);
  DBuf flags(N + 1, st), sel(N * 4 + 4, st), cnt(8, st);
  KL(k_nonzero_flags, grid_for(N, 256), dense, N, flags.as<uint8_t>());
  select_flagged_index(flags.as<uint8_t>(), sel.as<u32>(), cnt.as<u64>(), N, st);
  u64 n;
  GT_CUDA(cudaMemcpyAsync(&n, cnt.p, 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  R->n = n;
  R->id.alloc(n * 4 + 4, st);
  R->count.alloc(n * 8 + 8, st);
  DBuf file;
  if (pf) file.alloc(n * 4 + 4, st);
  KL(k_records, grid_for(n, 256), sel.as<u32>(), cnt.as<u64>(), dense, V, R->id.as<u32>(),
     R->count.as<u64>(), pf ? file.as<u32>() : nullptr);
  if (pf) {
    R->group_off.alloc((ncols + 1) * 8, st);
    KL(k_csr_offsets, grid_for(ncols + 1, 256), file.as<u32>(), n, (u64)ncols, R->group_off.as<u64>());
    R->n_groups = ncols;
  }
  if (by_count && n) {
    const u64 W = d->W;
    const int CB = std::max(1, bitlen(W));
    const int FB = pf ? bitlen(ncols - 1) : 0;
    DBuf k1(n * 8, st), k2(n * 8, st), id2(n * 4, st);
    KL(k_sort_keys, grid_for(n, 256), R->count.as<u64>(), pf ? file.as<u32>() : nullptr, n, W, CB, k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), R->id.as<u32>(), id2.as<u32>(), n, CB + FB, st);
    KL(k_unkey, grid_for(n, 256), k2.as<u64>(), n, W, CB, R->count.as<u64>());
    R->id = std::move(id2);
  }
}

void assemble_presence(DeviceDag* d, const u64* pres, u32 FW, DevRecords* R) {
  cudaStream_t st = d->stream;
  const u64 V = d->nw;
  DBuf pc(V * 8 + 8, st), pco(V * 8 + 8, st), nz(V + 1, st), words(V * 4 + 4, st), cnt(8, st);
  KL(k_popc, grid_for(V, 256), pres, V, FW, pc.as<u64>(), nz.as<uint8_t>());
  exclusive_scan_u64(pc.as<u64>(), pco.as<u64>(), V, st);
  select_flagged_index(nz.as<uint8_t>(), words.as<u32>(), cnt.as<u64>(), V, st);
  u64 ng = 0, last_off = 0, last_pc = 0;
  GT_CUDA(cudaMemcpyAsync(&ng, cnt.p, 8, cudaMemcpyDeviceToHost, st));
  if (V) {
    GT_CUDA(cudaMemcpyAsync(&last_off, pco.as<u64>() + V - 1, 8, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaMemcpyAsync(&last_pc, pc.as<u64>() + V - 1, 8, cudaMemcpyDeviceToHost, st));
  }
  GT_CUDA(cudaStreamSynchronize(st));
  const u64 n = last_off + last_pc;
  R->n = n;
  R->n_groups = ng;
  R->group_id.alloc(ng * 4 + 4, st);
  R->group_off.alloc((ng + 1) * 8, st);
  R->id.alloc(n * 4 + 4, st);
  KL(k_ii_write, grid_for(ng, 256), words.as<u32>(), cnt.as<u64>(), pres, pco.as<u64>(), V, FW,
     (u32)d->file_lo, R->group_id.as<u32>(), R->group_off.as<u64>(), R->id.as<u32>());
  GT_CUDA(cudaMemcpyAsync(R->group_off.as<u64>() + ng, &n, 8, cudaMemcpyHostToDevice, st));
  GT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gt
