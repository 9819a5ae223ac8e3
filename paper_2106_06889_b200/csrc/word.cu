// word.cu — word-level analytics on the device DAG (top-down strategy).
//
// Reference algorithm (engine.py:178-302, _kernels.py:129-188): Alg. 1
// top-down weight propagation in mask rounds, then Σ own_freq·weight into
// hash tables plus a scan of the root's plain words.  B200 formulation:
//   * rounds become precomputed levels (loader.cu); all levels run in ONE
//     persistent cooperative launch (segreduce.cuh k_segred_levels): the
//     level's (child, parent) edges are dealt to lanes in equal chunks, runs
//     of one child are combined by warp scans and flushed with one RED per
//     run — no masks, no host round trip, and heavy rules cost the same per
//     edge as light ones (the paper's split of high-fan-out work, by edges).
//   * root occurrences seed the rows from the (rule, segment) list, so the
//     same pass serves corpus-global weights (1 column = all owned files),
//     per-file weights (F columns) and per-file presence bitsets (OR mode,
//     ceil(F/64) 64-bit columns; exact for inverted index, which only needs
//     presence: 8 B per rule instead of 8*F B).
//   * the reduce is the same segmented gather-reduce over the word-major
//     transpose of the own pairs (word, rule, freq): one RED per word run
//     per chunk (hot Zipf words cost one atomic per chunk, not one per
//     occurrence).  Root words come from the (word, segment) list.
#include <algorithm>
#include <type_traits>

#include "kernels_common.cuh"
#include "segreduce.cuh"
#include "sparse.cuh"
#include "bottomup.cuh"
#include "word.cuh"

namespace gt {

// Seeds of the top-down pass (segreduce.cuh seed_rows_body): the root's
// direct references per owned segment; also run as phase 0 of the C = 1
// persistent level loop.
template <class Mode, class T = u64>
__global__ void __launch_bounds__(256) k_seed(SeedArgs a) {
  seed_rows_body<Mode, T>(a);
}

// root words of owned segments: (word, seg, cnt) sorted by word
template <class Mode, class T = u64>
__global__ void k_root_words(const u32* __restrict__ rw_word, const u32* __restrict__ rw_seg,
                             const u32* __restrict__ rw_cnt, u64 n, u32 file_lo, u32 nseg,
                             int per_file, u32 C, u64 V, int row_major, T* __restrict__ out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  const bool is_or = std::is_same<Mode, OrMode>::value;
  if (sizeof(T) == 8 && (!per_file || is_or)) {
    // corpus counts and presence: a word's entries (one per file) combined
    // per warp run first (key_run_atomics)
    for (u64 b0 = ((u64)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull; b0 < n; b0 += stride) {
      const u64 i = b0 + (threadIdx.x & 31u);
      u64 key = ~0ull, a = 0, bits = 0;
      if (i < n) {
        const u32 sg = rw_seg[i] - file_lo;
        if (sg < nseg) {
          const u64 w = rw_word[i];
          if (!per_file) {
            key = w;
            if (is_or) bits = 1ull;
            else a = rw_cnt[i];
          } else {  // presence bitsets: cell (word, segment / 64)
            const u64 col = sg >> 6;
            key = row_major ? w * C + col : col * V + w;
            bits = 1ull << (sg & 63u);
          }
        }
      }
      u64* o = reinterpret_cast<u64*>(out);
      key_run_atomics(key, a, bits, is_or ? nullptr : o, is_or ? o : nullptr);
    }
    return;
  }
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 sg = rw_seg[i] - file_lo;
    if (sg >= nseg) continue;
    u32 w = rw_word[i];
    if (!per_file) {
      Mode::atomic(&out[w], Mode::combine(rw_cnt[i], 1ull));
    } else {
      const u32 col = is_or ? (sg >> 6) : sg;
      const u64 v = is_or ? (1ull << (sg & 63u)) : (u64)rw_cnt[i];
      Mode::atomic(&out[row_major ? (u64)w * C + col : (u64)col * V + w], v);
    }
  }
}

// the compaction alone (large grammars: the level pass and the word reduce run
// as their own full-occupancy launches before it); cooperative, one block per SM
__global__ void __launch_bounds__(512) k_post_compact(PostArgs p) {
  cg::grid_group grid = cg::this_grid();
  post_compact(p, grid);
}

// the root's plain words into the {count, presence} pair outputs
__global__ void k_root_words_pair(const u32* __restrict__ rw_word, const u32* __restrict__ rw_seg,
                                  const u32* __restrict__ rw_cnt, u64 n, u32 file_lo, u32 nseg, u64* cnt,
                                  u64* pres) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 b0 = ((u64)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull; b0 < n; b0 += stride) {
    const u64 i = b0 + (threadIdx.x & 31u);
    u64 key = ~0ull, a = 0, bits = 0;
    if (i < n) {
      const u32 sg = rw_seg[i] - file_lo;
      if (sg < nseg) key = rw_word[i], a = rw_cnt[i], bits = 1ull << (sg & 63u);
    }
    key_run_atomics(key, a, bits, cnt, pres);
  }
}

// ---------------------------------------------------------------------------
// assembly
// ---------------------------------------------------------------------------
// records from selected indices: id = idx % V (word), count, file = idx / V
template <class T>
__global__ void k_records(const u32* sel, const u64* nsel, const T* vals, u64 V, u32* id,
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
// sort keys (file << CB) | (W - count): K = u32 when they fit 32 bits
template <class K>
__global__ void k_sort_keys(const u64* cnt, const u32* file, u64 n, u64 W, int CB, K* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = (K)(((file ? (u64)file[i] : 0ull) << CB) | (W - cnt[i]));
}

template <class K>
__global__ void k_unkey(const K* key, u64 n, u64 W, int CB, u64* cnt) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  u64 m = (CB >= 64) ? ~0ull : ((1ull << CB) - 1);
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    cnt[i] = W - ((u64)key[i] & m);
}

__global__ void k_nz_u64(const u64* v, u64 n, uint8_t* f) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) f[i] = v[i] != 0;
}

// inverted-index groups: the words with at least one file
__global__ void k_ii_groups(const u32* words, const u64* ngroups, const u64* off, u64 n, u32* gid,
                            u64* goff) {
  const u64 ng = *ngroups;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g <= ng; g += stride) {
    if (g == ng) {
      goff[g] = n;
    } else {
      gid[g] = words[g];
      goff[g] = off[words[g]];
    }
  }
}

// inverted index with at most 64 owned files (one presence word per vocab
// word): ONE scan over packed (has-files << 32 | popcount) gives both the
// group index and the record offset of every word, so groups and records
// come out of one emit pass (no select, no second scan)
__global__ void k_ii_keys(const u64* __restrict__ pres, u64 V, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w <= V; w += stride) {
    const u64 pc = w < V ? (u64)__popcll(pres[w]) : 0;
    key[w] = (pc ? (1ull << 32) : 0ull) | pc;
  }
}

__global__ void k_ii_emit(const u64* __restrict__ pres, u64 V, const u64* __restrict__ pref, u32 file_lo,
                          u32* files, u32* gid, u64* goff) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w <= V; w += stride) {
    const u64 k = pref[w];
    const u64 g = k >> 32, o = k & 0xFFFFFFFFull;
    if (w == V) {
      goff[g] = o;
      continue;
    }
    u64 b = pres[w];
    if (!b) continue;
    gid[g] = (u32)w;
    goff[g] = o;
    u64 q = o;
    while (b) {
      files[q++] = file_lo + (u32)(__ffsll((long long)b) - 1);
      b &= b - 1;
    }
  }
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------

#define KL(k, grid, ...) GT_KLAUNCH(#k, k, grid, 256, st, __VA_ARGS__)

// Level 1 holds the rules (heads) whose every parent is the root: no
// non-root edge enters it (a non-root parent sits at level >= 1), so the
// passes start at level 2 — one grid barrier fewer per pass.
constexpr int kFirstEdgeLevel = 2;

// Top-down weights (Alg. 1, engine.py:196-227): rows of C columns per rule,
// seeded from the root references, then one segmented gather-reduce launch
// per top-down level over that level's non-root parent edges.
template <class Mode, class T = u64>
static void td_levels(const DeviceDag* d, const TdLists& tl, u32 C, T* row, u32 per_file = 1,
                      const PostArgs* post = nullptr) {
  cudaStream_t st = d->stream;
  // rows indexed by tid (DeviceDag::tid) or tid' (heads): seeds and edges carry them
  const SeedArgs seed{tl.rs_rule_t, d->rs_seg.as<u32>(), d->rs_cnt.as<u32>(), d->n_rs, (u32)d->file_lo,
                      (u32)(d->file_hi - d->file_lo), per_file ? 1 : 0, C, row, (u64)C * tl.rows};
  // C = 1 with u64 rows: the zeroing and the seeds run as phase 0 of the
  // persistent launch
  const bool fused_seed = C == 1 && sizeof(T) == 8;
  if (!fused_seed) {
    GT_CUDA(cudaMemsetAsync(row, 0, sizeof(T) * C * tl.rows, st));
    if (d->n_rs) KL((k_seed<Mode, T>), grid_for(d->n_rs, 256), seed);
  }
  // all levels in one persistent launch, grid barriers between levels
  const std::vector<u64>& to = *tl.te_off;
  seg_reduce_levels<Mode>("k_td_levels", tl.te_child, tl.te_par, tl.te_freq, tl.te_off_dev, kFirstEdgeLevel, tl.nl, C,
                          RowSrcT<T>{row, C}, TdRowsT<T>{row, C}, st, false,
                          tl.nl ? (to[tl.nl + 1] - to[1]) / tl.nl : 0,
                          fused_seed ? &seed : nullptr, fused_seed ? post : nullptr);
}


// u64 rows -> u32 (saturating; *ovf set when a weight needs more than 32 bits)
__global__ void k_narrow_rows(const u64* __restrict__ row, u64 n, u32* out, u32* ovf) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  bool big = false;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 v = row[i];
    big |= v > 0xFFFFFFFFull;
    out[i] = v > 0xFFFFFFFFull ? 0xFFFFFFFFu : (u32)v;
  }
  if (__any_sync(0xFFFFFFFFu, big) && (threadIdx.x & 31u) == 0) *ovf = 1;
}

// Σ_r own_freq(r,w)·row[r] per word (reduce_words_round, _kernels.py:154-172)
// as a gather-reduce over the word-major own pairs, then the root's plain
// words per owned segment (root_words_round, _kernels.py:175-188).
// out: [C][V] (file-major: the per-file count tables in render order), or
// [V][C] with row_major (presence bitsets: a word's FW words contiguous, so
// the team's reductions and the later bit expansion are coalesced)
template <class Mode, class T = u64>
static void reduce_words(const DeviceDag* d, const TdLists& tl, u32 C, const T* row, T* out, bool per_file,
                         bool row_major = false) {
  cudaStream_t st = d->stream;
  const u64 V = d->nw;
  GT_CUDA(cudaMemsetAsync(out, 0, sizeof(T) * V * C, st));
  // C = 1 on a grammar whose u64 rows outgrow L2 (C5: 18M rules, 144 MB):
  // the word-major gathers fetch one random row per own pair, so the rows
  // are narrowed to u32 first (72 MB: they stay in L2 across the reduce);
  // a weight of 2^32 or more (flagged) reruns the reduce on the u64 rows
  static const bool wide = getenv("GT_REDUCE_U64") != nullptr;  // diagnostics: always gather u64 rows
  if constexpr (sizeof(T) == 8) {
    if (std::is_same<Mode, SumMode>::value && C == 1 && !wide && tl.rows * 8 > (64ull << 20)) {
      const Carve cv(st, {tl.rows * 4 + 4, 4});
      GT_CUDA(cudaMemsetAsync(cv.at<u32>(1), 0, 4, st));
      KL(k_narrow_rows, grid_for(tl.rows, 256), reinterpret_cast<const u64*>(row), tl.rows, cv.at<u32>(0),
         cv.at<u32>(1));
      if (row_major)
        seg_reduce<Mode>("k_reduce_words", tl.ow_word, tl.ow_src, tl.ow_freq, tl.n_own, C, RowSrcT<u32>{cv.at<u32>(0), C}, OutRowMajorT<T>{out, C}, st);
      else
        seg_reduce<Mode>("k_reduce_words", tl.ow_word, tl.ow_src, tl.ow_freq, tl.n_own, C, RowSrcT<u32>{cv.at<u32>(0), C}, OutColMajorT<T>{out, V}, st);
      u32 ovf = 0;
      GT_CUDA(cudaMemcpyAsync(&ovf, cv.at<u32>(1), 4, cudaMemcpyDeviceToHost, st));
      GT_CUDA(cudaStreamSynchronize(st));
      if (!ovf) {
        if (d->n_rw)
          KL((k_root_words<Mode, T>), grid_for(d->n_rw, 256), d->rw_word.as<u32>(), d->rw_seg.as<u32>(),
             d->rw_cnt.as<u32>(), d->n_rw, (u32)d->file_lo, (u32)(d->file_hi - d->file_lo), per_file ? 1 : 0, C, V,
             row_major ? 1 : 0, out);
        return;
      }
      GT_CUDA(cudaMemsetAsync(out, 0, sizeof(T) * V * C, st));  // a weight >= 2^32: the u64 rows
    }
  }
  if (row_major)
    seg_reduce<Mode>("k_reduce_words", tl.ow_word, tl.ow_src, tl.ow_freq, tl.n_own, C, RowSrcT<T>{row, C}, OutRowMajorT<T>{out, C}, st);
  else
    seg_reduce<Mode>("k_reduce_words", tl.ow_word, tl.ow_src, tl.ow_freq, tl.n_own, C, RowSrcT<T>{row, C}, OutColMajorT<T>{out, V}, st);
  if (d->n_rw)
    KL((k_root_words<Mode, T>), grid_for(d->n_rw, 256), d->rw_word.as<u32>(), d->rw_seg.as<u32>(),
       d->rw_cnt.as<u32>(), d->n_rw, (u32)d->file_lo, (u32)(d->file_hi - d->file_lo),
       per_file ? 1 : 0, C, V, row_major ? 1 : 0, out);
}

// C = 1 top-down pass with the word reduce and the root words folded into
// the same cooperative launch (phase 0 clears rows and output) — for small
// grammars, where the separate launches cost more than the reduce itself
// (C2: word count 0.133 -> 0.120 ms).  A large reduce is bandwidth-bound and
// needs the full-occupancy flat launch (C5: fused 1.77 ms vs 0.92 ms).
constexpr u64 kFusedReduceMax = 4ull << 20;

template <class Mode>
static void td_words_fused(DeviceDag* d, u64* row, u64* out, bool per_file, PostArgs* compact = nullptr) {
  const TdLists tl = td_lists(d, true);
  if (d->E_own > kFusedReduceMax) {
    td_levels<Mode>(d, tl, 1, row, per_file ? 1 : 0);
    reduce_words<Mode>(d, tl, 1, row, out, per_file);
    return;
  }
  PostArgs post{tl.ow_word, tl.ow_src, tl.ow_freq, tl.n_own, out, d->nw, nullptr,
                d->rw_word.as<u32>(), d->rw_seg.as<u32>(), d->rw_cnt.as<u32>(), d->n_rw, (u32)d->file_lo,
                (u32)(d->file_hi - d->file_lo), per_file ? 1 : 0};
  if (compact) {
    post.compact = compact->compact;
    post.rid = compact->rid;
    post.rcnt = compact->rcnt;
    post.gid = compact->gid;
    post.goff = compact->goff;
    post.tot = compact->tot;
    post.bsum = compact->bsum;
  }
  td_levels<Mode>(d, tl, 1, row, per_file ? 1 : 0, &post);
}

// small grammars, one launch per task: top-down pass + word reduce + root
// words + the render-order compaction (word count records / inverted-index
// groups); false when the grammar takes the multi-launch path
// (the fused compaction's block scans count records in u32 and its packed
// offsets must stay below 2^32: V * 64 records at most)
static bool small_task(const DeviceDag* d) { return d->E_own <= kFusedReduceMax && d->nw * 64 < (1ull << 32); }

bool td_word_records(DeviceDag* d, DevRecords* R) {
  if (!small_task(d)) return false;
  cudaStream_t st = d->stream;
  const u64 V = d->nw;
  const Carve cv(st, {d->R * 8, 2 * 1024 * 8, 16});  // rows, block sums, totals
  d->word_counts.alloc(V * 8 + 8, st);
  R->id.alloc(V * 4 + 4, st);
  R->count.alloc(V * 8 + 8, st);
  PostArgs c{};
  c.compact = 1;
  c.rid = R->id.as<u32>();
  c.rcnt = R->count.as<u64>();
  c.tot = cv.at<u64>(2);
  c.bsum = cv.at<u64>(1);
  td_words_fused<SumMode>(d, cv.at<u64>(0), d->word_counts.as<u64>(), false, &c);
  u64 h[2];
  GT_CUDA(cudaMemcpyAsync(h, c.tot, 16, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  R->n = h[0];
  return true;
}

bool td_presence_records(DeviceDag* d, DevRecords* R) {
  const u32 Fo = (u32)(d->file_hi - d->file_lo);
  if (!small_task(d) || Fo > 64) return false;
  cudaStream_t st = d->stream;
  const u64 V = d->nw;
  const Carve cv(st, {d->R * 8, V * 8 + 8, 2 * 1024 * 8, 16});  // rows, presence, block sums, totals
  R->id.alloc(V * (u64)std::max<u32>(Fo, 1) * 4 + 4, st);
  R->group_id.alloc(V * 4 + 4, st);
  R->group_off.alloc((V + 1) * 8, st);
  PostArgs c{};
  c.compact = 2;
  c.rid = R->id.as<u32>();
  c.gid = R->group_id.as<u32>();
  c.goff = R->group_off.as<u64>();
  c.tot = cv.at<u64>(3);
  c.bsum = cv.at<u64>(2);
  td_words_fused<OrMode>(d, cv.at<u64>(0), cv.at<u64>(1), true, &c);
  u64 h[2];
  GT_CUDA(cudaMemcpyAsync(h, c.tot, 16, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  R->n = h[0];
  R->n_groups = h[1];
  return true;
}

// Word count AND inverted index (<= 64 owned files) in ONE launch: the
// rows are {corpus weight, presence bitset} pairs (segreduce.cuh WcPresMode),
// so both tasks share the top-down level chain — the latency-bound part of a
// small grammar's pass — and the word reduce, the root words and the
// compaction (compact 3: the word-count records and the inverted-index
// groups have the same words in the same order).  Leaves the dense u64[V]
// counts in d->word_counts like td_word_records.
bool td_wc_ii_records(DeviceDag* d, DevRecords* wc, DevRecords* ii, cudaEvent_t done) {
  const u32 Fo = (u32)(d->file_hi - d->file_lo);
  if (Fo > 64 || d->nw * 64 >= (1ull << 32)) return false;
  // large grammars (> 4·10^6 own pairs) share the pass only over the
  // contraction's heads, whose 16-byte pair rows stay in L2 for the word
  // reduce's gathers (C5: 20 MB instead of 288 MB); then the level pass, the
  // full-occupancy word reduce and the compaction are separate launches
  const bool small = small_task(d);
  const TdLists tl = td_lists(d, true);
  if (!small && !tl.contracted) return false;
  cudaStream_t st = d->stream;
  const u64 V = d->nw;
  // every buffer of the step is carved from one grow-only block kept on the
  // DAG (repeated steps allocate nothing; the records are views that the
  // stream-ordered D2H reads before the next step on the stream rewrites
  // them): rows (pairs), presence, block sums, totals (+ the u32 overflow
  // flag), the dense counts, then the records
  const size_t sz[] = {d->R * 16, V * 8 + 8, 2 * 1024 * 8, 24, V * 8 + 8, V * 4 + 4, V * 8 + 8, V * 4 + 4,
                       V * (u64)std::max<u32>(Fo, 1) * 4 + 4, V * 4 + 4, (V + 1) * 8,
                       (V + 1) * 4};  // (offsets < V * 64 < 2^32: small_task)
  constexpr int NB = sizeof(sz) / sizeof(sz[0]);
  size_t off[NB + 1] = {0};
  for (int i = 0; i < NB; i++) off[i + 1] = off[i] + ((sz[i] + 255) & ~(size_t)255);
  if (d->step_cache.bytes < off[NB]) d->step_cache.alloc(off[NB], st);
  char* base = d->step_cache.as<char>();
  auto at = [&](int i) { return base + off[i]; };
  d->word_counts = DBuf::view(at(4), sz[4]);
  // the inverted index's file ids narrow when every owned file id fits
  const int rid_bytes = d->file_hi <= 256 ? 1 : d->file_hi <= 65536 ? 2 : 4;
  wc->id = DBuf::view(at(5), sz[5]);
  wc->count = DBuf::view(at(6), sz[6]);
  wc->count32 = DBuf::view(at(7), sz[7]);
  if (rid_bytes < 4) {
    ii->id_narrow = DBuf::view(at(8), sz[8]);
    ii->id_bytes = rid_bytes;
  } else {
    ii->id = DBuf::view(at(8), sz[8]);
  }
  ii->group_id = DBuf::view(at(9), sz[9]);
  ii->group_off = DBuf::view(at(10), sz[10]);
  ii->group_off32 = DBuf::view(at(11), sz[11]);
  u64* row = reinterpret_cast<u64*>(at(0));
  // rows left zeroed by the last small step on this block need no clearing
  const u64 rows_n = 2 * tl.rows;
  const bool clean = small && d->rows_clean_at == (const void*)row && d->rows_clean >= rows_n;
  const SeedArgs seed{tl.rs_rule_t, d->rs_seg.as<u32>(), d->rs_cnt.as<u32>(), d->n_rs, (u32)d->file_lo,
                      Fo, 1, 1u, row, clean ? 0 : rows_n};
  PostArgs post{tl.ow_word, tl.ow_src, tl.ow_freq, tl.n_own,
                d->word_counts.as<u64>(), V, reinterpret_cast<u64*>(at(1)), d->rw_word.as<u32>(), d->rw_seg.as<u32>(),
                d->rw_cnt.as<u32>(), d->n_rw, (u32)d->file_lo, Fo, 1};
  post.compact = 3;
  post.wid = wc->id.as<u32>();
  post.rcnt = wc->count.as<u64>();
  post.rid = ii->id.as<u32>();
  post.rid_n = ii->id_narrow.p;
  post.rid_bytes = rid_bytes;
  post.gid = ii->group_id.as<u32>();
  post.goff = ii->group_off.as<u64>();
  post.tot = reinterpret_cast<u64*>(at(3));
  post.bsum = reinterpret_cast<u64*>(at(2));
  post.rcnt32 = wc->count32.as<u32>();
  post.goff32 = ii->group_off32.as<u32>();
  static const bool tr = getenv("GT_TRACE") && atoi(getenv("GT_TRACE")) == 2;
  DBuf stamps;
  if (tr) {
    stamps.alloc(64 * 8, st);
    GT_CUDA(cudaMemsetAsync(stamps.p, 0, 64 * 8, st));
    post.stamps = stamps.as<u64>();
  }
  const std::vector<u64>& to = *tl.te_off;
  const u64 avg = tl.nl ? (to[tl.nl + 1] - to[1]) / tl.nl : 0;
  if (small) {
    post.zero_tail = row;
    post.zero_tail_n = rows_n;
    seg_reduce_levels1<WcPresMode>("k_td_levels", tl.te_child, tl.te_par, tl.te_freq, tl.te_off_dev, kFirstEdgeLevel, tl.nl, 0, avg,
                                   &seed, &post, RowSrcPair{row}, TdRowsPair{row}, st);
    d->rows_clean = rows_n;
    d->rows_clean_at = row;
  } else {
    d->rows_clean = 0;
    GT_CUDA(cudaMemsetAsync(post.out, 0, V * 8, st));
    GT_CUDA(cudaMemsetAsync(post.out2, 0, V * 8, st));
    GT_CUDA(cudaMemsetAsync(post.tot, 0, 24, st));
    seg_reduce_levels1<WcPresMode>("k_td_levels", tl.te_child, tl.te_par, tl.te_freq, tl.te_off_dev, kFirstEdgeLevel, tl.nl, 0, avg,
                                   &seed, nullptr, RowSrcPair{row}, TdRowsPair{row}, st);
    {  // (seg_reduce's C = 1 launch; its multi-column forms have no pair mode)
      const u64 n = tl.n_own;
      const int K = (int)std::min<u64>(16, std::max<u64>(1, pow2_floor(n / kResidentThreads)));
      const u64 tiles = (n + 32ull * K - 1) / (32ull * K);
      if (n)
        GT_KLAUNCH("k_reduce_words", (k_segred1<WcPresMode, RowSrcPair, OutPair>), grid_for(tiles * 32, 256, 148u * 32u),
                   256, st, tl.ow_word, tl.ow_src, tl.ow_freq, n, K, RowSrcPair{row}, OutPair{post.out, post.out2});
    }
    if (d->n_rw)
      KL(k_root_words_pair, grid_for(d->n_rw, 256), d->rw_word.as<u32>(), d->rw_seg.as<u32>(), d->rw_cnt.as<u32>(),
         d->n_rw, (u32)d->file_lo, Fo, post.out, post.out2);
    // the records: one cooperative compaction, or on a large vocabulary the
    // full-occupancy select / scan / emit kernels (the compaction walks each
    // block's word range in barrier-separated steps: C5, 10^6 words, 0.26 vs
    // 0.17 ms; C4, 10^5 words, 0.04 vs 0.09 ms).  GT_LARGE_ASSEMBLE=0/1 forces
    static const int force = getenv("GT_LARGE_ASSEMBLE") ? atoi(getenv("GT_LARGE_ASSEMBLE")) : -1;
    if (force == 1 || (force < 0 && V >= (1ull << 19))) {
      assemble_counts(d, post.out, V, 0, false, wc);
      assemble_presence(d, post.out2, 1, ii);
      wc->count32_ok = ii->group_off32_ok = false;
      ii->id_narrow.release();
      ii->id_bytes = 4;
      if (done) GT_CUDA(cudaEventRecord(done, st));
      return true;
    }
    int nsm = 148;
    GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, d->device));
    static int per_sm = -1;  // every resident block (bsum holds 2 * 1024 block counts)
    if (per_sm < 0) {
      GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_post_compact, 512, 0));
      per_sm = std::max(1, std::min(per_sm, 4));
    }
    void* args[] = {(void*)&post};
    ProfScope ps("k_post_compact", st);
    GT_CUDA(cudaLaunchCooperativeKernel((const void*)k_post_compact, dim3((unsigned)(nsm * per_sm)), dim3(512), args,
                                        0, st));
    g_launches++;
  }
  u64 h[3];
  GT_CUDA(cudaMemcpyAsync(h, post.tot, 24, cudaMemcpyDeviceToHost, st));
  if (done) GT_CUDA(cudaEventRecord(done, st));
  GT_CUDA(cudaStreamSynchronize(st));
  wc->count32_ok = h[2] == 0;
  ii->group_off32_ok = true;
  if (tr) {
    u64 t[64];
    GT_CUDA(cudaMemcpy(t, stamps.p, 64 * 8, cudaMemcpyDeviceToHost));
    const int nit = std::max(0, tl.nl - kFirstEdgeLevel + 1);  // (levels run by the pass)
    fprintf(stderr, "[wc+ii] seeds %.1f us | levels:", (t[1] - t[0]) / 1e3);
    for (int i = 0; i < nit && 2 + i < 64; i++) fprintf(stderr, " %.1f", (t[2 + i] - (i ? t[1 + i] : t[1])) / 1e3);
    if (4 + nit < 64)
      fprintf(stderr, " | barrier %.1f | reduce+root %.1f | compact %.1f us\n", (t[2 + nit] - t[1 + nit]) / 1e3,
              (t[3 + nit] - t[2 + nit]) / 1e3, (t[4 + nit] - t[3 + nit]) / 1e3);
  }
  ii->n = h[0];
  ii->n_groups = h[1];
  wc->n = h[1];
  return true;
}

void bu_root_words_dense(DeviceDag* d, u64* out) {
  cudaStream_t st = d->stream;
  if (d->n_rw)
    KL(k_root_words<SumMode>, grid_for(d->n_rw, 256), d->rw_word.as<u32>(), d->rw_seg.as<u32>(),
       d->rw_cnt.as<u32>(), d->n_rw, (u32)d->file_lo, (u32)(d->file_hi - d->file_lo), 0, 1u, d->nw, 0, out);
}

void td_root_seeds(DeviceDag* d, u64* row) {
  cudaStream_t st = d->stream;
  GT_CUDA(cudaMemsetAsync(row, 0, sizeof(u64) * d->R, st));
  if (d->n_rs)
    KL(k_seed<SumMode>, grid_for(d->n_rs, 256),
       SeedArgs{d->rs_rule.as<u32>(), d->rs_seg.as<u32>(), d->rs_cnt.as<u32>(), d->n_rs, (u32)d->file_lo,
                (u32)(d->file_hi - d->file_lo), 0, 1u, row, 0});
}

u64 scratch_budget(const DeviceDag* d) {
  size_t free_b = 0, total_b = 0;
  GT_CUDA(cudaMemGetInfo(&free_b, &total_b));
  cudaMemPool_t pool;
  GT_CUDA(cudaDeviceGetDefaultMemPool(&pool, d->device));
  u64 res = 0, used = 0;
  GT_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res));
  GT_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  return (u64)((double)(free_b + (res > used ? res - used : 0)) * 0.8);
}

// global word counts (corpus or owned shard) -> dense u64[V]
void td_word_counts(DeviceDag* d, DBuf& counts) {
  cudaStream_t st = d->stream;
  DBuf w(d->R * 8, st);
  counts.alloc(d->nw * 8 + 8, st);
  td_words_fused<SumMode>(d, w.as<u64>(), counts.as<u64>(), false);
}

// per-file cells fit u32 when every owned file has < 2^32 words (a weight or
// count of one file never exceeds its word count); C = 1 keeps u64 rows (the
// fused phase-0 seed of the C = 1 level loop writes u64)
static bool rows32(const DeviceDag* d, u32 C) { return d->cnt32 && C >= 2; }

// per-file counts -> dense [Fo][V] of u64, or u32 (*is32)
void td_file_counts(DeviceDag* d, DBuf& counts, bool* is32) {
  cudaStream_t st = d->stream;
  const u32 C = (u32)(d->file_hi - d->file_lo);
  const u64 Cm = std::max<u32>(C, 1);
  *is32 = rows32(d, C);
  const TdLists tl = td_lists(d, true);
  if (*is32) {
    DBuf w(tl.rows * 4 * Cm, st);
    td_levels<SumMode, u32>(d, tl, C, w.as<u32>());
    counts.alloc(d->nw * 4 * Cm + 8, st);
    reduce_words<SumMode, u32>(d, tl, C, w.as<u32>(), counts.as<u32>(), true);
    return;
  }
  DBuf w(tl.rows * 8 * Cm, st);
  td_levels<SumMode>(d, tl, C, w.as<u64>());
  counts.alloc(d->nw * 8 * Cm + 8, st);
  reduce_words<SumMode>(d, tl, C, w.as<u64>(), counts.as<u64>(), true);
}

// per-file weights only -> [R][Fo] of u64, or u32 (*is32)
void td_file_weights(DeviceDag* d, DBuf& w, u32* C_out, bool* is32, bool heads, bool* contracted) {
  const u32 C = std::max<u32>(1, (u32)(d->file_hi - d->file_lo));
  *is32 = rows32(d, C);
  const TdLists tl = td_lists(d, heads);  // every rule's row (callers index by tid), or the heads'
  if (contracted) *contracted = tl.contracted;
  if (*is32) {
    w.alloc(tl.rows * 4 * (u64)C, d->stream);
    td_levels<SumMode, u32>(d, tl, C, w.as<u32>());
  } else {
    w.alloc(tl.rows * 8 * (u64)C, d->stream);
    td_levels<SumMode>(d, tl, C, w.as<u64>());
  }
  *C_out = C;
}

// per-file presence bitsets -> dense u64[V][FW] (row-major); the rule rows
// (u64[R][FW]) are handed back in *rows_out when requested (sparse path)
void td_file_presence(DeviceDag* d, DBuf& pres, u32* FW_out, DBuf* rows_out) {
  cudaStream_t st = d->stream;
  const u32 Fo = (u32)(d->file_hi - d->file_lo);
  const u32 FW = std::max<u32>(1, (Fo + 63) / 64);
  DBuf m(d->R * 8 * (u64)FW, st);
  pres.alloc(d->nw * 8 * (u64)FW + 8, st);
  if (FW == 1 && !rows_out) {
    td_words_fused<OrMode>(d, m.as<u64>(), pres.as<u64>(), true);
  } else {
    const TdLists tl = td_lists(d, rows_out == nullptr);  // rows handed back: every rule's
    td_levels<OrMode>(d, tl, FW, m.as<u64>());
    reduce_words<OrMode>(d, tl, FW, m.as<u64>(), pres.as<u64>(), true, true);
  }
  *FW_out = FW;
  if (rows_out) *rows_out = std::move(m);
}

// ---- assembly -------------------------------------------------------------

// records in (file, -count, id) order (sort / term vector, tasks.py:122-168):
// one stable radix sort on (file << CB) | (W - count) carrying the id
void order_by_count(DeviceDag* d, DevRecords* R, u32 ncols, const u32* file) {
  cudaStream_t st = d->stream;
  R->count32_ok = false;  // (reordered below: the u32 copy no longer matches)
  const u64 n = R->n;
  const bool pf = ncols > 0;
  if (!n) return;
  // a per-file count never exceeds its file's words; when that bound still
  // needs a u64 key, the count field spans the largest count instead (one
  // reduction + read-back) — often a u32 key
  u64 W = pf && d->max_file_tokens ? d->max_file_tokens : d->W;
  if (bitlen(W) + (pf ? bitlen(ncols - 1) : 0) > 32) {
    DBuf mx(8, st);
    reduce_max_u64(R->count.as<u64>(), mx.as<u64>(), n, st);
    GT_CUDA(cudaMemcpyAsync(&W, mx.p, 8, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaStreamSynchronize(st));
    W = std::max<u64>(W, 1);
  }
  const int CB = std::max(1, bitlen(W));
  const int FB = pf ? bitlen(ncols - 1) : 0;
  DBuf k1(n * 8, st), k2(n * 8, st), id2(n * 4, st);
  if (CB + FB <= 32) {  // u32 keys: half the radix key traffic
    KL(k_sort_keys<u32>, grid_for(n, 256), R->count.as<u64>(), file, n, W, CB, k1.as<u32>());
    sort_pairs_u32_u32(k1.as<u32>(), k2.as<u32>(), R->id.as<u32>(), id2.as<u32>(), n, CB + FB, st);
    KL(k_unkey<u32>, grid_for(n, 256), k2.as<u32>(), n, W, CB, R->count.as<u64>());
  } else {
    KL(k_sort_keys<u64>, grid_for(n, 256), R->count.as<u64>(), file, n, W, CB, k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), R->id.as<u32>(), id2.as<u32>(), n, CB + FB, st);
    KL(k_unkey<u64>, grid_for(n, 256), k2.as<u64>(), n, W, CB, R->count.as<u64>());
  }
  R->id = std::move(id2);
}

void assemble_counts(DeviceDag* d, const void* dense, u64 V, u32 ncols, bool by_count, DevRecords* R, bool dense32) {
  // ncols == 0: one global table; ncols >= 1: per-file tables (file-major)
  cudaStream_t st = d->stream;
  const bool pf = ncols > 0;
  const u64 N = V * (u64)(pf ? ncols : 1);
  if (N >= (1ull << 32)) fail(GT_E_RESOURCE, "dense per-file table of %lu entries exceeds 2^32; use the bottom-up strategy", (unsigned long)N);
  DBuf cnt(8, st), file;
  u64 n;
  if (N <= (1ull << 26)) {
    // the select writes the records itself (worst-case sized outputs, no
    // index list and no second pass)
    R->id.alloc(N * 4 + 4, st);
    R->count.alloc(N * 8 + 8, st);
    if (pf) file.alloc(N * 4 + 4, st);
    select_nonzero_records(dense, dense32, V, N, R->id.as<u32>(), R->count.as<u64>(),
                           pf ? file.as<u32>() : nullptr, cnt.as<u64>(), st);
    GT_CUDA(cudaMemcpyAsync(&n, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaStreamSynchronize(st));
  } else {
    DBuf sel(N * 4 + 4, st);
    select_nonzero_index(dense, dense32, sel.as<u32>(), cnt.as<u64>(), N, st);
    GT_CUDA(cudaMemcpyAsync(&n, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaStreamSynchronize(st));
    R->id.alloc(n * 4 + 4, st);
    R->count.alloc(n * 8 + 8, st);
    if (pf) file.alloc(n * 4 + 4, st);
    if (dense32)
      KL(k_records<u32>, grid_for(n, 256), sel.as<u32>(), cnt.as<u64>(), (const u32*)dense, V, R->id.as<u32>(),
         R->count.as<u64>(), pf ? file.as<u32>() : nullptr);
    else
      KL(k_records<u64>, grid_for(n, 256), sel.as<u32>(), cnt.as<u64>(), (const u64*)dense, V, R->id.as<u32>(),
         R->count.as<u64>(), pf ? file.as<u32>() : nullptr);
  }
  R->n = n;
  if (pf) {
    R->group_off.alloc((ncols + 1) * 8, st);
    KL(k_csr_offsets, grid_for(ncols + 1, 256), file.as<u32>(), n, (u64)ncols, R->group_off.as<u64>());
    R->n_groups = ncols;
  }
  if (by_count && n) order_by_count(d, R, ncols, pf ? file.as<u32>() : nullptr);
}

// inverted index from the word presence bitsets u64[FW][V]: per word, the
// ascending global file ids of its set bits (warp-cooperative expansion,
// sparse.cu bits_to_csr), grouped by word in ascending word order
void assemble_presence(DeviceDag* d, const u64* pres, u32 FW, DevRecords* R) {
  cudaStream_t st = d->stream;
  const u64 V = d->nw;
  // the packed (has-files << 32 | popcount) scan needs every record offset
  // below 2^32: at most min(Fo, 64) records per word
  const u64 Fo = d->file_hi - d->file_lo;
  if (FW == 1 && V * std::min<u64>(std::max<u64>(Fo, 1), 64) < (1ull << 32)) {
    DBuf key((V + 1) * 8, st), pref((V + 1) * 8, st);
    KL(k_ii_keys, grid_for(V + 1, 256), pres, V, key.as<u64>());
    exclusive_scan_u64(key.as<u64>(), pref.as<u64>(), V + 1, st);
    u64 h;
    GT_CUDA(cudaMemcpyAsync(&h, pref.as<u64>() + V, 8, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaStreamSynchronize(st));
    const u64 ng = h >> 32, n = h & 0xFFFFFFFFull;
    R->n = n;
    R->n_groups = ng;
    R->id.alloc(n * 4 + 4, st);
    R->group_id.alloc(ng * 4 + 4, st);
    R->group_off.alloc((ng + 1) * 8, st);
    KL(k_ii_emit, grid_for(V + 1, 256), pres, V, pref.as<u64>(), (u32)d->file_lo, R->id.as<u32>(),
       R->group_id.as<u32>(), R->group_off.as<u64>());
    return;
  }
  if (V < (1ull << 24)) {
    // one packed scan for the group indices and record offsets
    DBuf files, gid, goff;
    u64 n = 0, ng = 0;
    bits_groups(pres, V, FW, (u32)d->file_lo, files, gid, goff, &n, &ng, st);
    R->n = n;
    R->n_groups = ng;
    R->id = std::move(files);
    R->group_id = std::move(gid);
    R->group_off = std::move(goff);
    return;
  }
  DBuf off, files, pc;
  bits_count(pres, V, FW, FW, 1, off, pc, st);
  DBuf nz(V + 1, st), words(V * 4 + 4, st), cnt(16, st);
  KL(k_nz_u64, grid_for(V, 256), pc.as<u64>(), V, nz.as<uint8_t>());
  select_flagged_index(nz.as<uint8_t>(), words.as<u32>(), cnt.as<u64>(), V, st);
  // one host round trip for both sizes: records n and groups ng
  GT_CUDA(cudaMemcpyAsync(cnt.as<u64>() + 1, off.as<u64>() + V, 8, cudaMemcpyDeviceToDevice, st));
  u64 h[2] = {0, 0};
  GT_CUDA(cudaMemcpyAsync(h, cnt.p, 16, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  const u64 ng = h[0], n = h[1];
  bits_expand(pres, V, FW, FW, 1, off, n, files, nullptr, st, (u32)d->file_lo);
  R->n = n;
  R->n_groups = ng;
  R->group_id.alloc(ng * 4 + 4, st);
  R->group_off.alloc((ng + 1) * 8, st);
  KL(k_ii_groups, grid_for(ng + 1, 256), words.as<u32>(), cnt.as<u64>(), off.as<u64>(), n,
     R->group_id.as<u32>(), R->group_off.as<u64>());
  R->id = std::move(files);
}

}  // namespace gt
