// sparse.cu — presence-guided sparse per-file weights, for corpora with many
// files (F > file_set_width; config C3: 10^5 files).
//
// The reference switches to its bottom-up strategy for F > 64
// (engine.py:63-71): dense R x F weight matrices (dag.py:79, engine.py:164)
// do not fit, and it rebuilds per-rule local word tables bottom-up and merges
// them into per-file tables (engine.py:338-518).  At 10^5 files that merge is
// the bulk of the work (Σ over root references of the child table size,
// ~10^9 inserts at C3).  The B200 formulation keeps the top-down direction
// but makes it sparse, guided by a cheap dense structure:
//
//   1. presence bitsets, 1 bit per (rule, file): the top-down pass in OrMode
//      (word.cu), 8·⌈F/64⌉ B per rule;
//   2. the (rule, file) pairs with a set bit, as a CSR sorted by file within
//      each rule (popcount + scan + warp-cooperative bit expansion);
//   3. u64 weights on exactly those pairs: root seeds, then per top-down level
//      every non-root parent edge (c, p, f) adds f·w(p, file) into
//      w(c, file) for every file of p (edge-balanced expansion; the target
//      slot found by binary search in c's file list, which contains p's);
//   4. outputs: term-vector cells (word, file) are exactly the inverted-index
//      presence cells, so they are allocated from the word presence bitsets
//      and filled with Σ own_freq·w(rule, file) + root words; sequence tasks
//      expand gram occurrences over their rule's files and reduce by
//      (gram run, file).
// Work is proportional to the nonzero (rule, file) and (word, file) pairs,
// not to R·F or to Σ local-table sizes.  All sums are integer: bit-exact.
#include <algorithm>

#include "kernels_common.cuh"
#include "sparse.cuh"

namespace gt {

namespace {

__device__ __forceinline__ u64 lower_bound_u32(const u32* a, u64 n, u32 x) {
  u64 lo = 0, hi = n;
  while (lo < hi) {
    const u64 m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// last g with pos[g] <= i (pos = exclusive scan of the group sizes)
__device__ __forceinline__ u64 find_group(const u64* pos, u64 G, u64 i) {
  u64 lo = 0, hi = G;
  while (hi - lo > 1) {
    const u64 m = (lo + hi) >> 1;
    if (pos[m] <= i) lo = m;
    else hi = m;
  }
  return lo;
}

// popcount of each bitset row (warp per row): row r has FW words at stride
// `rs` words, word j at r*rs_row + j*rs_col
__global__ void k_popc_rows(const u64* __restrict__ bits, u64 nrows, u32 FW, u64 rs_row, u64 rs_col,
                            u64* __restrict__ cnt, int packed) {
  const unsigned lane = threadIdx.x & 31u;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 r = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows; r += nw) {
    u64 c = 0;
    for (u32 j = lane; j < FW; j += 32) c += __popcll(bits[r * rs_row + (u64)j * rs_col]);
#pragma unroll
    for (int d = 16; d; d >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, d);
    if (lane == 0) cnt[r] = packed ? ((c ? (1ull << 40) : 0ull) | c) : c;
  }
}

constexpr int kExpU = 4;

// set bits of each row -> ascending column indices at off[r] (warp per row,
// 32 words per step, ballot-free: popcount prefix by shuffle scan)
// (packed: off[r] = (nonempty rows before r) << 40 | (bits before r), the
// group index and record offset from ONE scan; the nonempty rows' ids and
// record offsets are written to gid / goff — the inverted-index groups)
__global__ void k_expand_rows(const u64* __restrict__ bits, u64 nrows, u32 FW, u64 rs_row, u64 rs_col,
                              const u64* __restrict__ off, u32 col_base, u32* __restrict__ col,
                              u32* __restrict__ row_of, int packed, u32* __restrict__ gid,
                              u64* __restrict__ goff) {
  const unsigned lane = threadIdx.x & 31u;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 M = (1ull << 40) - 1;
  for (u64 r = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nrows; r += nw) {
    u64 o = packed ? (off[r] & M) : off[r];
    if ((packed ? (off[r + 1] & M) : off[r + 1]) == o) continue;
    if (packed && lane == 0) {
      const u64 g = off[r] >> 40;
      gid[g] = (u32)r;
      goff[g] = o;
    }
    // four 32-word steps' loads in flight per lane (a row of a many-file
    // corpus is thousands of words: one dependent load per step was the
    // bound — C3 inverted index 0.62 ms)
    for (u32 jj = 0; jj < FW; jj += 32 * kExpU) {
      u64 bb[kExpU];
#pragma unroll
      for (int u = 0; u < kExpU; u++) {
        const u32 j = jj + 32u * u + lane;
        bb[u] = j < FW ? bits[r * rs_row + (u64)j * rs_col] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kExpU; u++) {
      if (jj + 32u * u >= FW) break;  // warp-uniform
      const u32 j0 = jj + 32u * u;
      const u32 j = j0 + lane;
      u64 b = bb[u];
      const u32 c = (u32)__popcll(b);
      u32 inc = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= (unsigned)d) inc += t;
      }
      const u32 tot = __shfl_sync(0xFFFFFFFFu, inc, 31);
      if (tot >= 256) {
        // dense step: the warp writes one word's set bits at a time, lane l
        // owning bits l and l + 32, so consecutive outputs come from
        // consecutive lanes (a lane walking its own dense word would spread
        // each store instruction over 32 sectors)
        const u32 ex = inc - c;
        for (int w = 0; w < 32; w++) {
          const u64 bw = __shfl_sync(0xFFFFFFFFu, b, w);
          if (!bw) continue;
          const u64 ow = o + __shfl_sync(0xFFFFFFFFu, ex, w);
          const u32 jw = j0 + (u32)w;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const u32 t = lane + 32u * h;
            if ((bw >> t) & 1ull) {
              const u64 q = ow + (u64)__popcll(bw & ((1ull << t) - 1ull));
              col[q] = col_base + jw * 64u + t;
              if (row_of) row_of[q] = (u32)r;
            }
          }
        }
      } else {
        u64 q = o + inc - c;
        while (b) {
          const int t = __ffsll((long long)b) - 1;
          col[q] = col_base + j * 64u + (u32)t;
          if (row_of) row_of[q] = (u32)r;
          q++;
          b &= b - 1;
        }
      }
      o += tot;
      }
    }
  }
}

// FW == 1 (at most 64 files): one thread per row
__global__ void k_popc_rows1(const u64* __restrict__ bits, u64 nrows, u64 rs_row, u64* __restrict__ cnt) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += stride)
    cnt[r] = __popcll(bits[r * rs_row]);
}

__global__ void k_expand_rows1(const u64* __restrict__ bits, u64 nrows, u64 rs_row, const u64* __restrict__ off,
                               u32 col_base, u32* __restrict__ col, u32* __restrict__ row_of) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += stride) {
    u64 b = bits[r * rs_row], q = off[r];
    while (b) {
      const int t = __ffsll((long long)b) - 1;
      col[q] = col_base + (u32)t;
      if (row_of) row_of[q] = (u32)r;
      q++;
      b &= b - 1;
    }
  }
}

// root seeds: w(rule, seg) += cnt for owned segments
__global__ void k_sparse_seed(const u32* __restrict__ rs_rule, const u32* __restrict__ rs_seg,
                              const u32* __restrict__ rs_cnt, u64 n, u32 file_lo, u32 nseg,
                              const u64* __restrict__ off, const u32* __restrict__ file,
                              u64* __restrict__ wt) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 sg = rs_seg[i] - file_lo;
    if (sg >= nseg) continue;
    const u32 r = rs_rule[i];
    const u64 a = off[r];
    const u64 q = a + lower_bound_u32(file + a, off[r + 1] - a, sg);
    atomicAdd((unsigned long long*)&wt[q], (unsigned long long)rs_cnt[i]);
  }
}

// group sizes: |files(key[i])|
__global__ void k_list_len(const u32* __restrict__ key, u64 n, const u64* __restrict__ off,
                           u64* __restrict__ deg) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    deg[i] = off[key[i] + 1] - off[key[i]];
}

// Expansion of a group list (group e = one edge or own pair, owning the
// files of its source rule, pos = exclusive scan of the group sizes): each
// thread takes kExp consecutive items, locates its first group once (binary
// search over pos) and then walks: within a group the source files ascend,
// so the target slot advances by a linear merge through the target's
// (ascending, superset) file list instead of a binary search per item.
constexpr u64 kExp = 16;

// first index in [lo, hi) with a[idx] >= x (a ascending), galloping from lo:
// O(log distance), so a sparse source list walking a dense target list
// costs no more than the binary searches it replaces
__device__ __forceinline__ u64 gallop_u32(const u32* a, u64 lo, u64 hi, u32 x) {
  if (lo >= hi || a[lo] >= x) return lo;
  u64 step = 1, prev = lo;
  while (lo + step < hi && a[lo + step] < x) {
    prev = lo + step;
    step <<= 1;
  }
  u64 l = prev + 1, h = lo + step < hi ? lo + step : hi;
  while (l < h) {
    const u64 m = (l + h) >> 1;
    if (a[m] < x) l = m + 1;
    else h = m;
  }
  return l;
}

// one top-down level: for every edge (c, p, f) and every file of p:
//   w(c, file) += f · w(p, file)
__global__ void k_sparse_level(const u32* __restrict__ child, const u32* __restrict__ par,
                               const u32* __restrict__ freq, u64 n, const u64* __restrict__ pos,
                               const u64* __restrict__ deg, const u64* __restrict__ off,
                               const u32* __restrict__ file, u64* __restrict__ wt) {
  if (!n) return;
  const u64 T = pos[n - 1] + deg[n - 1];
  const u64 stride = (u64)gridDim.x * blockDim.x * kExp;
  for (u64 i0 = ((u64)blockIdx.x * blockDim.x + threadIdx.x) * kExp; i0 < T; i0 += stride) {
    const u64 i1 = i0 + kExp < T ? i0 + kExp : T;
    u64 e = find_group(pos, n, i0);
    u64 gend = pos[e] + deg[e];
    u32 p = par[e], c = child[e];
    u64 f = freq[e];
    u64 k = off[p] + (i0 - pos[e]);
    u64 q = off[c] + lower_bound_u32(file + off[c], off[c + 1] - off[c], file[k]);
    for (u64 i = i0; i < i1; i++) {
      if (i == gend) {  // next non-empty group
        do e++;
        while (deg[e] == 0);
        gend = pos[e] + deg[e];
        p = par[e];
        c = child[e];
        f = freq[e];
        k = off[p];
        q = off[c] + lower_bound_u32(file + off[c], off[c + 1] - off[c], file[k]);
      } else if (i != i0) {
        k++;
        q = gallop_u32(file, q, off[c + 1], file[k]);
      }
      atomicAdd((unsigned long long*)&wt[q], (unsigned long long)(f * wt[k]));
    }
  }
}

// term-vector cells: every own pair (w, r, f) adds f · w(r, file) to cell
// (w, file) for every file of r (chunked walk as k_sparse_level; the word's
// file list is a superset of the rule's)
__global__ void k_tv_own(const u32* __restrict__ ow_word, const u32* __restrict__ ow_rule,
                         const u32* __restrict__ ow_freq, u64 n, const u64* __restrict__ pos,
                         const u64* __restrict__ deg, const u64* __restrict__ off,
                         const u32* __restrict__ file, const u64* __restrict__ wt,
                         const u64* __restrict__ woff, const u32* __restrict__ wfile,
                         u64* __restrict__ cnt) {
  if (!n) return;
  const u64 T = pos[n - 1] + deg[n - 1];
  const u64 stride = (u64)gridDim.x * blockDim.x * kExp;
  for (u64 i0 = ((u64)blockIdx.x * blockDim.x + threadIdx.x) * kExp; i0 < T; i0 += stride) {
    const u64 i1 = i0 + kExp < T ? i0 + kExp : T;
    u64 e = find_group(pos, n, i0);
    u64 gend = pos[e] + deg[e];
    u32 r = ow_rule[e], w = ow_word[e];
    u64 f = ow_freq[e];
    u64 k = off[r] + (i0 - pos[e]);
    u64 q = woff[w] + lower_bound_u32(wfile + woff[w], woff[w + 1] - woff[w], file[k]);
    for (u64 i = i0; i < i1; i++) {
      if (i == gend) {
        do e++;
        while (deg[e] == 0);
        gend = pos[e] + deg[e];
        r = ow_rule[e];
        w = ow_word[e];
        f = ow_freq[e];
        k = off[r];
        q = woff[w] + lower_bound_u32(wfile + woff[w], woff[w + 1] - woff[w], file[k]);
      } else if (i != i0) {
        k++;
        q = gallop_u32(wfile, q, woff[w + 1], file[k]);
      }
      atomicAdd((unsigned long long*)&cnt[q], (unsigned long long)(f * wt[k]));
    }
  }
}

__global__ void k_tv_root(const u32* __restrict__ rw_word, const u32* __restrict__ rw_seg,
                          const u32* __restrict__ rw_cnt, u64 n, u32 file_lo, u32 nseg,
                          const u64* __restrict__ woff, const u32* __restrict__ wfile,
                          u64* __restrict__ cnt) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 sg = rw_seg[i] - file_lo;
    if (sg >= nseg) continue;
    const u32 w = rw_word[i];
    const u64 a = woff[w];
    const u64 q = a + lower_bound_u32(wfile + a, woff[w + 1] - a, sg);
    atomicAdd((unsigned long long*)&cnt[q], (unsigned long long)rw_cnt[i]);
  }
}

// (file, W - count) sort keys of the word-major cells
template <class K>
__global__ void k_tv_keys(const u32* __restrict__ wfile, const u64* __restrict__ cnt, u64 n, u64 W,
                          int CB, K* __restrict__ key) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = (K)(((u64)wfile[i] << CB) | (W - cnt[i]));
}

template <class K>
__global__ void k_tv_unkey(const K* __restrict__ key, u64 n, u64 W, int CB, u64* __restrict__ cnt,
                           u32* __restrict__ file) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 m = (1ull << CB) - 1;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 k = key[i];
    cnt[i] = W - (k & m);
    file[i] = (u32)(k >> CB);
  }
}

// gram occurrences -> (run << FB | file, weight) items: an occurrence from
// rule s < R expands over the files of s; one from root segment s - R is a
// single item of weight 1
__global__ void k_occ_deg(const u32* __restrict__ src, u64 N, u32 R, const u64* __restrict__ off,
                          u64* __restrict__ deg) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    const u32 s = src[i];
    deg[i] = s < R ? off[s + 1] - off[s] : 1ull;
  }
}

__global__ void k_occ_items(const u32* __restrict__ rid, const u32* __restrict__ src, u64 N, u32 R,
                            const u64* __restrict__ pos, const u64* __restrict__ deg,
                            const u64* __restrict__ off, const u32* __restrict__ file,
                            const u64* __restrict__ wt, int FB, u64* __restrict__ key,
                            u64* __restrict__ val) {
  if (!N) return;
  const u64 T = pos[N - 1] + deg[N - 1];
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < T; i += stride) {
    const u64 o = find_group(pos, N, i);
    const u32 s = src[o];
    u32 f;
    u64 v;
    if (s < R) {
      const u64 k = off[s] + (i - pos[o]);
      f = file[k];
      v = wt[k];
    } else {
      f = s - R;
      v = 1;
    }
    key[i] = ((u64)rid[o] << FB) | f;
    val[i] = v;
  }
}

}  // namespace

#define SK(k, n, ...) GT_KLAUNCH(#k, k, grid_for((n), 256), 256, st, __VA_ARGS__)
#define SKW(k, nwarps, ...) GT_KLAUNCH(#k, k, grid_for((u64)(nwarps) * 32, 256, 148u * 64u), 256, st, __VA_ARGS__)
#define SKE(k, ...) GT_KLAUNCH(#k, k, 148u * 16u, 256, st, __VA_ARGS__)

namespace {
template <class T>
T d2h1(const void* p, cudaStream_t st) {
  T v;
  GT_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  return v;
}

}  // namespace

// rows of bitsets -> CSR (off, col[, row_of]); returns the pair count
void bits_count(const u64* bits, u64 nrows, u32 FW, u64 rs_row, u64 rs_col, DBuf& off, DBuf& cnt,
                cudaStream_t st) {
  cnt.alloc(nrows * 8 + 8, st);
  off.alloc((nrows + 1) * 8, st);
  if (FW == 1) SK(k_popc_rows1, nrows, bits, nrows, rs_row, cnt.as<u64>());
  else SKW(k_popc_rows, nrows, bits, nrows, FW, rs_row, rs_col, cnt.as<u64>(), 0);
  GT_CUDA(cudaMemsetAsync(cnt.as<u64>() + nrows, 0, 8, st));
  exclusive_scan_u64(cnt.as<u64>(), off.as<u64>(), nrows + 1, st);
}

void bits_expand(const u64* bits, u64 nrows, u32 FW, u64 rs_row, u64 rs_col, const DBuf& off, u64 P,
                 DBuf& col, DBuf* row_of, cudaStream_t st, u32 col_base) {
  col.alloc(P * 4 + 4, st);
  if (row_of) row_of->alloc(P * 4 + 4, st);
  if (FW == 1)
    SK(k_expand_rows1, nrows, bits, nrows, rs_row, off.as<u64>(), col_base, col.as<u32>(),
       row_of ? row_of->as<u32>() : (u32*)nullptr);
  else
    SKW(k_expand_rows, nrows, bits, nrows, FW, rs_row, rs_col, off.as<u64>(), col_base, col.as<u32>(),
        row_of ? row_of->as<u32>() : (u32*)nullptr, 0, (u32*)nullptr, (u64*)nullptr);
}

__global__ void k_set_u64(u64* p, u64 v) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *p = v;
}

// inverted-index groups from word-major bitsets (FW words per row): one
// packed scan (group index << 40 | record offset; rows < 2^24) gives each
// row's group index and record offset; returns
// (records, groups) and fills files / gid / goff (goff[groups] = records)
void bits_groups(const u64* bits, u64 nrows, u32 FW, u32 col_base, DBuf& files, DBuf& gid, DBuf& goff, u64* n_out,
                 u64* ng_out, cudaStream_t st) {
  DBuf key((nrows + 1) * 8, st), pref((nrows + 1) * 8, st);
  GT_CUDA(cudaMemsetAsync(key.as<u64>() + nrows, 0, 8, st));
  SKW(k_popc_rows, nrows, bits, nrows, FW, (u64)FW, 1ull, key.as<u64>(), 1);
  exclusive_scan_u64(key.as<u64>(), pref.as<u64>(), nrows + 1, st);
  const u64 h = d2h1<u64>(pref.as<u64>() + nrows, st);
  const u64 ng = h >> 40, n = h & ((1ull << 40) - 1);
  files.alloc(n * 4 + 4, st);
  gid.alloc(ng * 4 + 4, st);
  goff.alloc((ng + 1) * 8, st);
  SK(k_set_u64, 1, goff.as<u64>() + ng, n);
  SKW(k_expand_rows, nrows, bits, nrows, FW, (u64)FW, 1ull, pref.as<u64>(), col_base, files.as<u32>(),
      (u32*)nullptr, 1, gid.as<u32>(), goff.as<u64>());
  *n_out = n;
  *ng_out = ng;
}

u64 bits_to_csr(const u64* bits, u64 nrows, u32 FW, u64 rs_row, u64 rs_col, DBuf& off, DBuf& col,
                DBuf* row_of, cudaStream_t st, u32 col_base, DBuf* row_cnt) {
  DBuf cnt;
  bits_count(bits, nrows, FW, rs_row, rs_col, off, cnt, st);
  const u64 P = d2h1<u64>(off.as<u64>() + nrows, st);
  bits_expand(bits, nrows, FW, rs_row, rs_col, off, P, col, row_of, st, col_base);
  if (row_cnt) *row_cnt = std::move(cnt);
  return P;
}

void sparse_file_weights(DeviceDag* d, SparseW* s, DBuf* word_pres, u32* FW_out) {
  cudaStream_t st = d->stream;
  Phases ph("sparse-w", st);
  const u64 R = d->R;
  DBuf pres, rows;
  u32 FW;
  td_file_presence(d, pres, &FW, &rows);
  if (word_pres) *word_pres = std::move(pres);
  *FW_out = FW;
  ph.mark("presence");
  s->P = bits_to_csr(rows.as<u64>(), R, FW, FW, 1, s->off, s->file, nullptr, st);
  rows.release();
  s->wt.alloc(s->P * 8 + 8, st);
  GT_CUDA(cudaMemsetAsync(s->wt.p, 0, s->P * 8 + 8, st));
  const u32 nseg = (u32)(d->file_hi - d->file_lo);
  if (d->n_rs)
    SK(k_sparse_seed, d->n_rs, d->rs_rule_t.as<u32>(), d->rs_seg.as<u32>(), d->rs_cnt.as<u32>(), d->n_rs,
       (u32)d->file_lo, nseg, s->off.as<u64>(), s->file.as<u32>(), s->wt.as<u64>());
  ph.mark("pairs+seeds");
  const u64 Etd = d->te_off.empty() ? 0 : d->te_off.back();
  DBuf deg(Etd * 8 + 8, st), pos(Etd * 8 + 8, st);
  for (int L = 1; L <= d->td.nl; L++) {
    const u64 a = d->te_off[L], n = d->te_off[L + 1] - a;
    if (!n) continue;
    SK(k_list_len, n, d->te_par.as<u32>() + a, n, s->off.as<u64>(), deg.as<u64>());
    exclusive_scan_u64(deg.as<u64>(), pos.as<u64>(), n, st);
    SKE(k_sparse_level, d->te_child.as<u32>() + a, d->te_par.as<u32>() + a, d->te_freq.as<u32>() + a, n,
        pos.as<u64>(), deg.as<u64>(), s->off.as<u64>(), s->file.as<u32>(), s->wt.as<u64>());
  }
  ph.mark("levels");
}

void sparse_term_vector(DeviceDag* d, DevRecords* Rr) {
  cudaStream_t st = d->stream;
  Phases ph("tv-sparse", st);
  const u64 V = d->nw;
  const u32 Fo = (u32)(d->file_hi - d->file_lo);
  SparseW s;
  DBuf pres;
  u32 FW;
  sparse_file_weights(d, &s, &pres, &FW);
  ph.mark("weights");
  // (word, file) cells = word presence bits; word-major, files ascending
  DBuf woff, wfile, wword;
  const u64 O = bits_to_csr(pres.as<u64>(), V, FW, FW, 1, woff, wfile, &wword, st);
  pres.release();
  DBuf cnt(O * 8 + 8, st);
  GT_CUDA(cudaMemsetAsync(cnt.p, 0, O * 8 + 8, st));
  const u64 Eo = d->E_own;
  if (Eo) {
    DBuf deg(Eo * 8 + 8, st), pos(Eo * 8 + 8, st);
    SK(k_list_len, Eo, d->ow_rule_t.as<u32>(), Eo, s.off.as<u64>(), deg.as<u64>());
    exclusive_scan_u64(deg.as<u64>(), pos.as<u64>(), Eo, st);
    SKE(k_tv_own, d->ow_word.as<u32>(), d->ow_rule_t.as<u32>(), d->ow_freq.as<u32>(), Eo, pos.as<u64>(),
        deg.as<u64>(), s.off.as<u64>(), s.file.as<u32>(), s.wt.as<u64>(), woff.as<u64>(),
        wfile.as<u32>(), cnt.as<u64>());
  }
  if (d->n_rw)
    SK(k_tv_root, d->n_rw, d->rw_word.as<u32>(), d->rw_seg.as<u32>(), d->rw_cnt.as<u32>(), d->n_rw,
       (u32)d->file_lo, Fo, woff.as<u64>(), wfile.as<u32>(), cnt.as<u64>());
  ph.mark("cells");
  s = SparseW();
  // file-major, (-count, word) within a file: one stable radix sort of the
  // word-major cells on (file, W - count); W = the longest file's words, or
  // the largest cell count when that bound needs a u64 key
  u64 W = d->max_file_tokens ? d->max_file_tokens : d->W;
  if (O && bitlen(W) + std::max(1, bitlen(Fo ? Fo - 1 : 0)) > 32) {
    DBuf mx(8, st);
    reduce_max_u64(cnt.as<u64>(), mx.as<u64>(), O, st);
    W = std::max<u64>(1, d2h1<u64>(mx.p, st));
  }
  const int CB = std::max(1, bitlen(W));
  const int FB = std::max(1, bitlen(Fo ? Fo - 1 : 0));
  DBuf k1(O * 8 + 8, st), k2(O * 8 + 8, st);
  Rr->n = O;
  Rr->id.alloc(O * 4 + 4, st);
  if (CB + FB <= 32) {  // u32 keys (C3: 13 + 17 bits)
    SK(k_tv_keys<u32>, O, wfile.as<u32>(), cnt.as<u64>(), O, W, CB, k1.as<u32>());
    sort_pairs_u32_u32(k1.as<u32>(), k2.as<u32>(), wword.as<u32>(), Rr->id.as<u32>(), O, CB + FB, st);
    Rr->count = std::move(cnt);
    SK(k_tv_unkey<u32>, O, k2.as<u32>(), O, W, CB, Rr->count.as<u64>(), wfile.as<u32>());
  } else {
    SK(k_tv_keys<u64>, O, wfile.as<u32>(), cnt.as<u64>(), O, W, CB, k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), wword.as<u32>(), Rr->id.as<u32>(), O, CB + FB, st);
    Rr->count = std::move(cnt);
    SK(k_tv_unkey<u64>, O, k2.as<u64>(), O, W, CB, Rr->count.as<u64>(), wfile.as<u32>());
  }
  Rr->n_groups = Fo;
  Rr->group_off.alloc(((u64)Fo + 1) * 8, st);
  SK(k_csr_offsets, (u64)Fo + 1, wfile.as<u32>(), O, (u64)Fo, Rr->group_off.as<u64>());
  ph.mark("sort");
}

u64 sparse_run_cells(DeviceDag* d, const SparseW& s, const u32* rid, const u32* src, u64 N, int FB,
                     DBuf& cell_key, DBuf& cell_cnt) {
  cudaStream_t st = d->stream;
  if (!N) return 0;
  DBuf deg(N * 8 + 8, st), pos(N * 8 + 8, st);
  SK(k_occ_deg, N, src, N, (u32)d->R, s.off.as<u64>(), deg.as<u64>());
  exclusive_scan_u64(deg.as<u64>(), pos.as<u64>(), N, st);
  const u64 T = d2h1<u64>(pos.as<u64>() + N - 1, st) + d2h1<u64>(deg.as<u64>() + N - 1, st);
  DBuf key(T * 8 + 8, st), val(T * 8 + 8, st);
  SKE(k_occ_items, rid, src, N, (u32)d->R, pos.as<u64>(), deg.as<u64>(), s.off.as<u64>(),
      s.file.as<u32>(), s.wt.as<u64>(), FB, key.as<u64>(), val.as<u64>());
  deg.release();
  pos.release();
  DBuf k2(T * 8 + 8, st), v2(T * 8 + 8, st);
  u32 nruns_bits = 1;
  {
    u32 last_rid = d2h1<u32>(rid + N - 1, st);
    nruns_bits = (u32)std::max(1, bitlen(last_rid));
  }
  sort_pairs_u64_u64(key.as<u64>(), k2.as<u64>(), val.as<u64>(), v2.as<u64>(), T, FB + (int)nruns_bits, st);
  key.release();
  val.release();
  cell_key.alloc(T * 8 + 8, st);
  cell_cnt.alloc(T * 8 + 8, st);
  DBuf nc(8, st);
  reduce_by_key_u64(k2.as<u64>(), v2.as<u64>(), cell_key.as<u64>(), cell_cnt.as<u64>(), nc.as<u64>(), T, st);
  return d2h1<u64>(nc.p, st);
}

}  // namespace gt
