// bottomup.cu — the reference's bottom-up strategy (Alg. 2) on the device:
// per-rule local word tables in one pooled arena of open-addressing hash
// tables, built children-first, then the level-2 merge into per-file (or one
// global) result.
//
// Reference: local_table_bounds engine.py:338-367 (+ bounds_round
// _kernels.py:191-202), plan_pool engine.py:370-377 / CountTableSet
// table.py:69-237 (a memory pool of per-entry-locked chained tables, Fig. 4),
// bottom_up_traverse engine.py:409-446 (own_insert_round _kernels.py:219-233,
// merge_round :236-250), reduce_bottom_up engine.py:478-518
// (root_words_round :175-188, merge_try_round :253-276 with the stop-flag
// retry protocol of Fig. 7).
//
// B200 formulation:
//   * bounds: bound[r] = min(own_distinct + Σ_children bound, min(exp_len, V)),
//     one persistent pass over the child edges in decreasing top-down level
//     order (children before parents; the cap is applied when a bound is read);
//   * arena: table r = [toff[r], toff[r] + cap[r]) of (u32 key, u64 count)
//     slots, cap = next pow2 >= 2·bound (load <= 1/2, as table.py sizes its
//     entry ranges), linear probing; insert = CAS on the key slot + u64
//     atomicAdd on the count; lanes of a warp inserting the same (table, key)
//     combine first (__match_any_sync) — the warp-aggregated tables of
//     north_star, lock-free, no retry rounds;
//   * merges: one launch per top-down level; every (rule, child, freq) edge
//     expands into the child's slots (edge-balanced: exclusive scan of the
//     child capacities, binary search per slot), occupied slots insert
//     f·count into the parent's table;
//   * level 2: root words + Σ cnt·table(child) over the owned segments into
//     a dense u64[V] (global) or into per-file tables in the same kind of
//     arena, then compaction and render-order sorts.
// Output equals the top-down paths' bit for bit (integer sums).
#include <algorithm>

#include "bottomup.cuh"
#include "segreduce.cuh"
#include "sparse.cuh"

namespace gt {

namespace {

constexpr u32 kEmpty = 0xFFFFFFFFu;

__device__ __forceinline__ u32 hash32(u32 x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ u64 find_grp(const u64* pos, u64 G, u64 i) {
  u64 lo = 0, hi = G;
  while (hi - lo > 1) {
    const u64 m = (lo + hi) >> 1;
    if (pos[m] <= i) lo = m;
    else hi = m;
  }
  return lo;
}

// open-addressing insert-or-add into table [base, base + cap); false = full
__device__ __forceinline__ bool ht_add(u32* keys, u64* vals, u64 base, u32 cap, u32 w, u64 v) {
  const u32 mask = cap - 1;
  u32 h = hash32(w) & mask;
  for (u32 probe = 0; probe < cap; probe++) {
    u32* kp = keys + base + h;
    u32 k = *(volatile u32*)kp;
    if (k == kEmpty) {
      const u32 prev = atomicCAS(kp, kEmpty, w);
      k = prev == kEmpty ? w : prev;
    }
    if (k == w) {
      atomicAdd((unsigned long long*)(vals + base + h), (unsigned long long)v);
      return true;
    }
    h = (h + 1) & mask;
  }
  return false;
}

// warp-aggregated insert: lanes with the same (table, key) sum their deltas
// first (one probe sequence per distinct key per warp).  All lanes call it.
__device__ __forceinline__ void ht_add_warp(u32* keys, u64* vals, const u64* toff, const u32* tcap, u32 t,
                                            u32 w, u64 v, bool active, u32* full) {
  const unsigned act = __ballot_sync(0xFFFFFFFFu, active);
  if (!active) return;
  const u64 key = ((u64)t << 32) | w;
  const unsigned peers = __match_any_sync(act, key);
  const unsigned lane = threadIdx.x & 31u;
  u64 sum = 0;
  for (unsigned m = peers; m; m &= m - 1) sum += __shfl_sync(peers, v, __ffs(m) - 1);
  if ((int)lane != __ffs(peers) - 1 || sum == 0) return;
  if (!ht_add(keys, vals, toff[t], tcap[t], w, sum)) *full = 1;
}

// bounds: own distinct words; the cap is applied where a bound is read
__global__ void k_own_distinct(const u64* own_off, u64 R, u64* bound) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride)
    bound[r] = own_off[r + 1] - own_off[r];
}

// the table-size cap of a rule: min(exp_len, V) for words (local_table_bounds
// caps, engine.py:338-367), max(exp_len - (l-1), 0) for l-grams (exp_windows,
// sequence.py:319-321; V = ~0 there)
__device__ __forceinline__ u64 table_cap(u64 exp_len, u64 sub, u64 V) {
  const u64 e = exp_len > sub ? exp_len - sub : 0;
  return e < V ? e : V;
}

struct CappedBound {  // min(bound[c], cap(c))
  const u64* bound;
  const u64* exp_len;
  u64 V, sub;
  __device__ __forceinline__ u64 operator()(u32 c, u32) const {
    const u64 b = ldcg(bound + c), cap = table_cap(exp_len[c], sub, V);
    return b < cap ? b : cap;
  }
};

__global__ void k_table_caps(const u64* bound, const u64* exp_len, u64 V, u64 sub, u64 R, u32* tcap, u64* tcap64) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride) {
    u64 b = bound[r];
    const u64 cap = table_cap(exp_len[r], sub, V);
    if (b > cap) b = cap;
    u32 c = 0;
    if (b) {
      c = 2;
      while ((u64)c < 2 * b) c <<= 1;
    }
    tcap[r] = c;
    tcap64[r] = c;
  }
}

// own items of every non-root rule: (key, rule, freq) — the own words
// (ow_word, ow_rule, ow_freq) or the attributed gram windows (run id, rule,
// 1); rules >= rule_limit (root segments of the gram windows) are skipped
__global__ void k_own_insert(const u32* ow_word, const u32* ow_rule, const u32* ow_freq, u64 n, u32 rule_limit,
                             u32* keys, u64* vals, const u64* toff, const u32* tcap, u32* full) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const u64 i = base + threadIdx.x;
    const u32 r = i < n ? ow_rule[i] : 0u;
    const bool a = r != 0 && r < rule_limit;
    ht_add_warp(keys, vals, toff, tcap, a ? r : 0, a ? ow_word[i] : 0, a ? (ow_freq ? ow_freq[i] : 1u) : 0, a,
                full);
  }
}

__global__ void k_child_slots(const u32* child, u64 n, const u32* tcap, u64* deg) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) deg[i] = tcap[child[i]];
}

// child -> parent merge of one level: every slot of every (rule, child, f)
// item; occupied slots add f·count into the rule's table
__global__ void k_merge_level(const u32* rule, const u32* child, const u32* freq, u64 n, const u64* pos,
                              const u64* deg, u32* keys, u64* vals, const u64* toff, const u32* tcap,
                              u32* full) {
  if (!n) return;
  const u64 T = pos[n - 1] + deg[n - 1];
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < T; base += stride) {
    const u64 i = base + threadIdx.x;
    bool a = false;
    u32 r = 0, w = 0;
    u64 v = 0;
    if (i < T) {
      const u64 e = find_grp(pos, n, i);
      const u32 c = child[e];
      const u64 s = toff[c] + (i - pos[e]);
      w = keys[s];
      if (w != kEmpty) {
        a = true;
        r = rule[e];
        v = (u64)freq[e] * vals[s];
      }
    }
    ht_add_warp(keys, vals, toff, tcap, r, w, v, a, full);
  }
}

// level 2, global: root references of the owned segments (root_freq over the
// owned range, k_seed) times each child table, into the dense counts
__global__ void k_root_slots(const u64* seedw, u64 R, const u32* tcap, u64* deg) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride)
    deg[r] = (r && seedw[r]) ? tcap[r] : 0;
}

__global__ void k_level2_global(const u64* seedw, u64 R, const u64* pos, const u64* deg, const u32* keys,
                                const u64* vals, const u64* toff, u64* out) {
  const u64 T = pos[R - 1] + deg[R - 1];
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < T; i += stride) {
    const u64 r = find_grp(pos, R, i);
    const u64 s = toff[r] + (i - pos[r]);
    const u32 w = keys[s];
    if (w != kEmpty) atomicAdd((unsigned long long*)&out[w], (unsigned long long)(seedw[r] * vals[s]));
  }
}

// level 2, per file: file table bounds, then root words and root references
__global__ void k_file_bounds(const u32* rs_rule, const u32* rs_seg, u64 nrs, const u32* rw_seg, u64 nrw,
                              u32 file_lo, u32 nseg, const u64* bound, u64* fb) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < nrs + nrw; i += stride) {
    if (i < nrs) {
      const u32 sg = rs_seg[i] - file_lo;
      if (sg < nseg) atomicAdd((unsigned long long*)&fb[sg], (unsigned long long)bound[rs_rule[i]]);
    } else {
      const u32 sg = rw_seg[i - nrs] - file_lo;
      if (sg < nseg) atomicAdd((unsigned long long*)&fb[sg], 1ull);
    }
  }
}

// per-file table caps: min(bound, tokens_f - sub, V)
__global__ void k_file_caps(const u64* fb, const u64* seg_tokens, u32 file_lo, u64 V, u64 sub, u32 nseg, u32* fcap,
                            u64* fcap64) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 f = (u64)blockIdx.x * blockDim.x + threadIdx.x; f < nseg; f += stride) {
    u64 b = fb[f];
    const u64 cap = table_cap(seg_tokens[file_lo + f], sub, V);
    if (b > cap) b = cap;
    u32 c = 0;
    if (b) {
      c = 2;
      while ((u64)c < 2 * b) c <<= 1;
    }
    fcap[f] = c;
    fcap64[f] = c;
  }
}

__global__ void k_file_root_words(const u32* rw_word, const u32* rw_seg, const u32* rw_cnt, u64 n, u32 file_lo,
                                  u32 nseg, u32* keys, u64* vals, const u64* foff, const u32* fcap, u32* full) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const u64 i = base + threadIdx.x;
    const u32 sg = i < n ? rw_seg[i] - file_lo : 0xFFFFFFFFu;
    const bool a = i < n && sg < nseg;
    ht_add_warp(keys, vals, foff, fcap, a ? sg : 0, a ? rw_word[i] : 0, a ? rw_cnt[i] : 0, a, full);
  }
}

__global__ void k_rs_slots(const u32* rs_rule, const u32* rs_seg, u64 n, u32 file_lo, u32 nseg, const u32* tcap,
                           u64* deg) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    deg[i] = (rs_seg[i] - file_lo < nseg) ? tcap[rs_rule[i]] : 0;
}

__global__ void k_level2_files(const u32* rs_rule, const u32* rs_seg, const u32* rs_cnt, u64 n, u32 file_lo,
                               const u64* pos, const u64* deg, const u32* keys, const u64* vals,
                               const u64* toff, u32* fkeys, u64* fvals, const u64* foff, const u32* fcap,
                               u32* full) {
  if (!n) return;
  const u64 T = pos[n - 1] + deg[n - 1];
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < T; base += stride) {
    const u64 i = base + threadIdx.x;
    bool a = false;
    u32 f = 0, w = 0;
    u64 v = 0;
    if (i < T) {
      const u64 e = find_grp(pos, n, i);
      const u64 s = toff[rs_rule[e]] + (i - pos[e]);
      w = keys[s];
      if (w != kEmpty) {
        a = true;
        f = rs_seg[e] - file_lo;
        v = (u64)rs_cnt[e] * vals[s];
      }
    }
    ht_add_warp(fkeys, fvals, foff, fcap, f, w, v, a, full);
  }
}

// l-gram windows (bottom-up gram strategy): own window count per rule
// (own_candidates, sequence.py:319-321), root-segment windows per file (the
// file-table bounds) and their inserts into the per-file tables
__global__ void k_gram_counts(const u32* src, u64 n, u32 R, u64* own_c, u64* fb) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 s = src[i];
    atomicAdd((unsigned long long*)(s < R ? own_c + s : fb + (s - R)), 1ull);
  }
}

__global__ void k_file_root_grams(const u32* run, const u32* src, u64 n, u32 R, u32* keys, u64* vals,
                                  const u64* foff, const u32* fcap, u32* full) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const u64 i = base + threadIdx.x;
    const u32 s = i < n ? src[i] : 0u;
    const bool a = i < n && s >= R;
    ht_add_warp(keys, vals, foff, fcap, a ? s - R : 0, a ? run[i] : 0, 1ull, a, full);
  }
}

// (run << FB | file) keys of the occupied per-file slots
__global__ void k_key_rf(const u32* file, const u32* run, u64 n, int FB, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = ((u64)run[i] << FB) | file[i];
}

__global__ void k_split_rf(const u64* key, const u32* idx, const u64* cnt, u64 n, int FB, u32* crun, u32* ccol,
                           u64* ccnt) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    crun[i] = (u32)(key[i] >> FB);
    ccol[i] = (u32)(key[i] & ((1ull << FB) - 1));
    ccnt[i] = cnt[idx[i]];
  }
}

__global__ void k_occupied(const u32* keys, u64 n, uint8_t* f) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) f[i] = keys[i] != kEmpty;
}

// file of each compacted slot (binary search in the file table offsets)
__global__ void k_slot_records(const u32* sel, const u64* nsel, const u32* keys, const u64* vals, const u64* foff,
                               u32 nseg, u32* file, u32* word, u64* cnt) {
  const u64 n = *nsel;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 s = sel[i];
    u64 lo = 0, hi = nseg;
    while (hi - lo > 1) {
      const u64 m = (lo + hi) >> 1;
      if (foff[m] <= s) lo = m;
      else hi = m;
    }
    file[i] = (u32)lo;
    word[i] = keys[s];
    cnt[i] = vals[s];
  }
}

__global__ void k_key_fw(const u32* file, const u32* word, u64 n, int WB, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = ((u64)file[i] << WB) | word[i];
}

__global__ void k_key_wf(const u32* file, const u32* word, u64 n, int FB, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = ((u64)word[i] << FB) | file[i];
}

__global__ void k_gather_u32(const u32* idx, u64 n, const u32* src, u32* dst) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[idx[i]];
}

__global__ void k_gather_u64b(const u32* idx, u64 n, const u64* src, u64* dst) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[idx[i]];
}

__global__ void k_tv_key(const u32* file, const u64* cnt, u64 n, u64 W, int CB, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = ((u64)file[i] << CB) | (W - cnt[i]);
}

__global__ void k_add_u32(u32* a, u64 n, u32 v) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] += v;
}

__global__ void k_word_of_key(const u64* key, u64 n, int FB, u32* word, uint8_t* head) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    word[i] = (u32)(key[i] >> FB);
    head[i] = i == 0 || (key[i] >> FB) != (key[i - 1] >> FB);
  }
}

__global__ void k_groups_from_heads(const u32* sel, const u64* ng, const u32* word, u64 n, u32* gid, u64* goff) {
  const u64 G = *ng;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g <= G; g += stride) {
    if (g == G) {
      goff[g] = n;
    } else {
      gid[g] = word[sel[g]];
      goff[g] = sel[g];
    }
  }
}

#define BK(k, n, ...) GT_KLAUNCH(#k, k, grid_for((n), 256), 256, st, __VA_ARGS__)
#define BKE(k, ...) GT_KLAUNCH(#k, k, 148u * 16u, 256, st, __VA_ARGS__)

template <class T>
T rd1(const void* p, cudaStream_t st) {
  T v;
  GT_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  return v;
}

// the arena of per-rule tables
struct RuleTables {
  DBuf bound, tcap, toff, keys, vals;
  u64 S = 0;
};

// the own items of a table arena (see k_own_insert)
struct OwnItems {
  const u32* key;
  const u32* rule;
  const u32* freq;  // nullable: 1 per item
  u64 n;
  u32 rule_limit;
};

// Per-rule tables built children-first (bottom_up_traverse, engine.py:409-446).
// own_bound: u64[R] own table sizes (consumed as the bound array); V / sub:
// the table caps (table_cap).  false = the arena would exceed `budget`.
bool build_rule_tables(DeviceDag* d, RuleTables* T, u64 budget, const OwnItems& own, DBuf&& own_bound, u64 V,
                       u64 sub) {
  cudaStream_t st = d->stream;
  const u64 R = d->R;
  // bounds (local_table_bounds, engine.py:338-367)
  T->bound = std::move(own_bound);
  seg_reduce_levels<SumMode>("k_bu_bounds", d->be_rule.as<u32>(), d->be_child.as<u32>(), nullptr,
                             d->be_off_dev.as<u64>(), 0, d->td.nl, 1,
                             CappedBound{T->bound.as<u64>(), d->exp_len.as<u64>(), V, sub},
                             OutRowMajor{T->bound.as<u64>(), 1}, st, true);
  // arena (plan_pool, engine.py:370-377)
  DBuf cap64(R * 8 + 8, st);
  T->tcap.alloc(R * 4, st);
  BK(k_table_caps, R, T->bound.as<u64>(), d->exp_len.as<u64>(), V, sub, R, T->tcap.as<u32>(), cap64.as<u64>());
  GT_CUDA(cudaMemsetAsync(cap64.as<u64>() + R, 0, 8, st));
  T->toff.alloc((R + 1) * 8, st);
  exclusive_scan_u64(cap64.as<u64>(), T->toff.as<u64>(), R + 1, st);
  T->S = rd1<u64>(T->toff.as<u64>() + R, st);
  if (T->S * 12 > budget) return false;
  T->keys.alloc(T->S * 4 + 4, st);
  T->vals.alloc(T->S * 8 + 8, st);
  GT_CUDA(cudaMemsetAsync(T->keys.p, 0xFF, T->S * 4 + 4, st));
  GT_CUDA(cudaMemsetAsync(T->vals.p, 0, T->S * 8 + 8, st));
  DBuf full(4, st);
  GT_CUDA(cudaMemsetAsync(full.p, 0, 4, st));
  // own items (own_insert_round _kernels.py:219-233 / window_count_round :279-309)
  if (own.n)
    BK(k_own_insert, own.n, own.key, own.rule, own.freq, own.n, own.rule_limit, T->keys.as<u32>(),
       T->vals.as<u64>(), T->toff.as<u64>(), T->tcap.as<u32>(), full.as<u32>());
  // children first: decreasing top-down level, root (level 0) excluded
  // (merge_round, _kernels.py:236-250)
  const u64 Eb = d->be_off.empty() ? 0 : d->be_off.back();
  DBuf deg(Eb * 8 + 8, st), pos(Eb * 8 + 8, st);
  for (int L = d->td.nl; L >= 1; L--) {
    const u64 a = d->be_off[L], n = d->be_off[L + 1] - a;
    if (!n) continue;
    BK(k_child_slots, n, d->be_child.as<u32>() + a, n, T->tcap.as<u32>(), deg.as<u64>());
    exclusive_scan_u64(deg.as<u64>(), pos.as<u64>(), n, st);
    BKE(k_merge_level, d->be_rule.as<u32>() + a, d->be_child.as<u32>() + a, d->be_freq.as<u32>() + a, n,
        pos.as<u64>(), deg.as<u64>(), T->keys.as<u32>(), T->vals.as<u64>(), T->toff.as<u64>(),
        T->tcap.as<u32>(), full.as<u32>());
  }
  if (rd1<u32>(full.p, st)) fail(GT_E_RESOURCE, "local table full (bound violated)");
  return true;
}

// the word tables: own distinct words, caps min(exp_len, V)
bool build_word_tables(DeviceDag* d, RuleTables* T, u64 budget) {
  cudaStream_t st = d->stream;
  DBuf own(d->R * 8, st);
  BK(k_own_distinct, d->R, d->own_off.as<u64>(), d->R, own.as<u64>());
  return build_rule_tables(d, T, budget, OwnItems{d->ow_word.as<u32>(), d->ow_rule.as<u32>(), d->ow_freq.as<u32>(),
                                                  d->E_own, (u32)d->R},
                           std::move(own), d->nw, 0);
}

__global__ void k_table_batch(const u32* keys_in, const u64* deltas, u64 n, u32* keys, u64* vals, const u64* toff,
                              const u32* tcap, u32* full) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 base = (u64)blockIdx.x * blockDim.x; base < n; base += stride) {
    const u64 i = base + threadIdx.x;
    const bool a = i < n;
    ht_add_warp(keys, vals, toff, tcap, 0, a ? keys_in[i] : 0, a ? deltas[i] : 0, a, full);
  }
}

}  // namespace

// add_batch (_kernels.py:117-126, the reference's table stress kernel): n
// (key, delta) inserts from all warps concurrently into one table of `cap`
// slots; returns the occupied (key, count) slots.  Test hook for the pooled
// tables' insert path.
int table_add_batch(int device, const u32* h_keys, const u64* h_deltas, u64 n, u32 cap, u32* h_out_keys,
                    u64* h_out_vals) {
  if (cap == 0 || (cap & (cap - 1))) fail(GT_E_USAGE, "table capacity must be a power of two");
  GT_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  GT_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  u32 full_h = 0;
  {
    DBuf k(n * 4 + 4, st), dl(n * 8 + 8, st), keys((u64)cap * 4, st), vals((u64)cap * 8, st), toff(16, st),
        tcap(8, st), full(4, st);
    if (n) {
      GT_CUDA(cudaMemcpyAsync(k.p, h_keys, n * 4, cudaMemcpyHostToDevice, st));
      GT_CUDA(cudaMemcpyAsync(dl.p, h_deltas, n * 8, cudaMemcpyHostToDevice, st));
    }
    const u64 toff_h[2] = {0, cap};
    GT_CUDA(cudaMemcpyAsync(toff.p, toff_h, 16, cudaMemcpyHostToDevice, st));
    GT_CUDA(cudaMemcpyAsync(tcap.p, &cap, 4, cudaMemcpyHostToDevice, st));
    GT_CUDA(cudaMemsetAsync(keys.p, 0xFF, (u64)cap * 4, st));
    GT_CUDA(cudaMemsetAsync(vals.p, 0, (u64)cap * 8, st));
    GT_CUDA(cudaMemsetAsync(full.p, 0, 4, st));
    if (n)
      GT_KLAUNCH("k_table_batch", k_table_batch, grid_for(n, 256), 256, st, k.as<u32>(), dl.as<u64>(), n,
                 keys.as<u32>(), vals.as<u64>(), toff.as<u64>(), tcap.as<u32>(), full.as<u32>());
    GT_CUDA(cudaMemcpyAsync(h_out_keys, keys.p, (u64)cap * 4, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaMemcpyAsync(h_out_vals, vals.p, (u64)cap * 8, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaMemcpyAsync(&full_h, full.p, 4, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaStreamSynchronize(st));
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return full_h ? GT_E_RESOURCE : GT_OK;
}

bool bu_word_counts(DeviceDag* d, DBuf& counts, u64 budget) {
  cudaStream_t st = d->stream;
  const u64 R = d->R, V = d->nw;
  RuleTables T;
  if (!build_word_tables(d, &T, budget)) return false;
  counts.alloc(V * 8 + 8, st);
  GT_CUDA(cudaMemsetAsync(counts.p, 0, V * 8 + 8, st));
  // root words of the owned segments (root_words_round) ...
  if (d->n_rw) bu_root_words_dense(d, counts.as<u64>());
  // ... and the root's references times their tables (reduce_bottom_up)
  DBuf seedw(R * 8, st), deg(R * 8, st), pos(R * 8, st);
  td_root_seeds(d, seedw.as<u64>());
  BK(k_root_slots, R, seedw.as<u64>(), R, T.tcap.as<u32>(), deg.as<u64>());
  exclusive_scan_u64(deg.as<u64>(), pos.as<u64>(), R, st);
  BKE(k_level2_global, seedw.as<u64>(), R, pos.as<u64>(), deg.as<u64>(), T.keys.as<u32>(), T.vals.as<u64>(),
      T.toff.as<u64>(), counts.as<u64>());
  return true;
}

bool bu_file_tables(DeviceDag* d, int task, DevRecords* Rr, u64 budget) {
  cudaStream_t st = d->stream;
  const u64 V = d->nw;
  const u32 file_lo = (u32)d->file_lo, nseg = (u32)(d->file_hi - d->file_lo);
  RuleTables T;
  if (!build_word_tables(d, &T, budget)) return false;
  // per-file output tables appended to the plan (extra_bounds of plan_pool)
  DBuf fb((u64)nseg * 8 + 8, st), fcap((u64)nseg * 4 + 4, st), fcap64((u64)nseg * 8 + 8, st),
      foff((u64)nseg * 8 + 8, st);
  GT_CUDA(cudaMemsetAsync(fb.p, 0, (u64)nseg * 8 + 8, st));
  if (d->n_rs + d->n_rw)
    BK(k_file_bounds, d->n_rs + d->n_rw, d->rs_rule.as<u32>(), d->rs_seg.as<u32>(), d->n_rs, d->rw_seg.as<u32>(),
       d->n_rw, file_lo, nseg, T.bound.as<u64>(), fb.as<u64>());
  BK(k_file_caps, nseg, fb.as<u64>(), d->seg_tokens.as<u64>(), file_lo, V, 0ull, nseg, fcap.as<u32>(),
     fcap64.as<u64>());
  GT_CUDA(cudaMemsetAsync(fcap64.as<u64>() + nseg, 0, 8, st));
  exclusive_scan_u64(fcap64.as<u64>(), foff.as<u64>(), (u64)nseg + 1, st);
  const u64 FS = rd1<u64>(foff.as<u64>() + nseg, st);
  if ((T.S + FS) * 12 > budget) return false;
  DBuf fkeys(FS * 4 + 4, st), fvals(FS * 8 + 8, st), full(4, st);
  GT_CUDA(cudaMemsetAsync(fkeys.p, 0xFF, FS * 4 + 4, st));
  GT_CUDA(cudaMemsetAsync(fvals.p, 0, FS * 8 + 8, st));
  GT_CUDA(cudaMemsetAsync(full.p, 0, 4, st));
  if (d->n_rw)
    BK(k_file_root_words, d->n_rw, d->rw_word.as<u32>(), d->rw_seg.as<u32>(), d->rw_cnt.as<u32>(), d->n_rw,
       file_lo, nseg, fkeys.as<u32>(), fvals.as<u64>(), foff.as<u64>(), fcap.as<u32>(), full.as<u32>());
  if (d->n_rs) {
    DBuf deg(d->n_rs * 8 + 8, st), pos(d->n_rs * 8 + 8, st);
    BK(k_rs_slots, d->n_rs, d->rs_rule.as<u32>(), d->rs_seg.as<u32>(), d->n_rs, file_lo, nseg,
       T.tcap.as<u32>(), deg.as<u64>());
    exclusive_scan_u64(deg.as<u64>(), pos.as<u64>(), d->n_rs, st);
    BKE(k_level2_files, d->rs_rule.as<u32>(), d->rs_seg.as<u32>(), d->rs_cnt.as<u32>(), d->n_rs, file_lo,
        pos.as<u64>(), deg.as<u64>(), T.keys.as<u32>(), T.vals.as<u64>(), T.toff.as<u64>(), fkeys.as<u32>(),
        fvals.as<u64>(), foff.as<u64>(), fcap.as<u32>(), full.as<u32>());
  }
  if (rd1<u32>(full.p, st)) fail(GT_E_RESOURCE, "per-file word table full (bound violated)");
  T = RuleTables();
  // compaction: (file, word, count) of the occupied slots
  DBuf occ(FS + 1, st), sel(FS * 4 + 4, st), nsel(8, st);
  BK(k_occupied, FS, fkeys.as<u32>(), FS, occ.as<uint8_t>());
  select_flagged_index(occ.as<uint8_t>(), sel.as<u32>(), nsel.as<u64>(), FS, st);
  const u64 n = rd1<u64>(nsel.p, st);
  DBuf file(n * 4 + 4, st), word(n * 4 + 4, st), cnt(n * 8 + 8, st);
  BK(k_slot_records, n, sel.as<u32>(), nsel.as<u64>(), fkeys.as<u32>(), fvals.as<u64>(), foff.as<u64>(), nseg,
     file.as<u32>(), word.as<u32>(), cnt.as<u64>());
  fkeys.release();
  fvals.release();
  const int WB = std::max(1, bitlen(V ? V - 1 : 0));
  const int FB = std::max(1, bitlen(nseg ? nseg - 1 : 0));
  DBuf k1(n * 8 + 8, st), k2(n * 8 + 8, st), idx(n * 4 + 4, st), idx2(n * 4 + 4, st);
  BK(k_iota_u32, n, idx.as<u32>(), n);
  if (task == GT_TERMVECTOR) {
    // (file, word) order, then stable (file, -count): render order
    BK(k_key_fw, n, file.as<u32>(), word.as<u32>(), n, WB, k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), idx.as<u32>(), idx2.as<u32>(), n, WB + FB, st);
    DBuf f2(n * 4 + 4, st), c2(n * 8 + 8, st);
    BK(k_gather_u32, n, idx2.as<u32>(), n, file.as<u32>(), f2.as<u32>());
    BK(k_gather_u64b, n, idx2.as<u32>(), n, cnt.as<u64>(), c2.as<u64>());
    // count field sized by the largest file (a per-file count never exceeds
    // its file's words), as sparse.cu; the key must hold file and count bits
    const u64 W = d->max_file_tokens ? d->max_file_tokens : d->W;
    const int CB = std::max(1, bitlen(W));
    if (CB + FB > 64) fail(GT_E_RESOURCE, "term-vector sort key of %d bits exceeds 64", CB + FB);
    BK(k_tv_key, n, f2.as<u32>(), c2.as<u64>(), n, W, CB, k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), idx2.as<u32>(), idx.as<u32>(), n, CB + FB, st);
    Rr->n = n;
    Rr->id.alloc(n * 4 + 4, st);
    Rr->count.alloc(n * 8 + 8, st);
    BK(k_gather_u32, n, idx.as<u32>(), n, word.as<u32>(), Rr->id.as<u32>());
    BK(k_gather_u64b, n, idx.as<u32>(), n, cnt.as<u64>(), Rr->count.as<u64>());
    BK(k_gather_u32, n, idx.as<u32>(), n, file.as<u32>(), f2.as<u32>());
    Rr->n_groups = nseg;
    Rr->group_off.alloc(((u64)nseg + 1) * 8, st);
    BK(k_csr_offsets, (u64)nseg + 1, f2.as<u32>(), n, (u64)nseg, Rr->group_off.as<u64>());
  } else {
    // inverted index: (word, file) order, grouped by word, files global
    BK(k_key_wf, n, file.as<u32>(), word.as<u32>(), n, FB, k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), idx.as<u32>(), idx2.as<u32>(), n, WB + FB, st);
    Rr->n = n;
    Rr->id.alloc(n * 4 + 4, st);
    BK(k_gather_u32, n, idx2.as<u32>(), n, file.as<u32>(), Rr->id.as<u32>());
    BK(k_add_u32, n, Rr->id.as<u32>(), n, file_lo);
    DBuf wd(n * 4 + 4, st), head(n + 1, st), gsel(n * 4 + 4, st), ng(8, st);
    BK(k_word_of_key, n, k2.as<u64>(), n, FB, wd.as<u32>(), head.as<uint8_t>());
    select_flagged_index(head.as<uint8_t>(), gsel.as<u32>(), ng.as<u64>(), n, st);
    const u64 G = rd1<u64>(ng.p, st);
    Rr->n_groups = G;
    Rr->group_id.alloc(G * 4 + 4, st);
    Rr->group_off.alloc((G + 1) * 8, st);
    BK(k_groups_from_heads, G + 1, gsel.as<u32>(), ng.as<u64>(), wd.as<u32>(), n, Rr->group_id.as<u32>(),
       Rr->group_off.as<u64>());
  }
  GT_CUDA(cudaStreamSynchronize(st));
  return true;
}

// Bottom-up l-gram counting (count_sequences strategy="bottomup",
// sequence.py:369-415): per-rule window tables sized by local_table_bounds
// over the own window counts capped by exp_windows, filled with each rule's
// attributed windows (keys = gram run ids of the sorted windows: packed or
// gram-mode grams share one u32 key space) and merged children-first scaled
// by body frequency; then the root: every file's segment windows plus
// seg_count(c, f) x table(c) for the root's children (level 2) into per-file
// tables.  Out: nonzero (run, file, count) cells in (run, file) order —
// the input of seq.cu's render-order record assembly.  src: rule id (< R)
// or R + owned segment per window occurrence; false = over budget.
bool bu_seq_cells(DeviceDag* d, u32 l, const u32* run, const u32* src, u64 N, u64 nruns, DBuf& crun, DBuf& ccol,
                  DBuf& ccnt, u64* n_out, u64 budget) {
  cudaStream_t st = d->stream;
  const u64 R = d->R, m = l - 1;
  const u32 file_lo = (u32)d->file_lo, nseg = (u32)(d->file_hi - d->file_lo);
  DBuf own(R * 8, st), fb((u64)nseg * 8 + 8, st);
  GT_CUDA(cudaMemsetAsync(own.p, 0, R * 8, st));
  GT_CUDA(cudaMemsetAsync(fb.p, 0, (u64)nseg * 8 + 8, st));
  if (N) BK(k_gram_counts, N, src, N, (u32)R, own.as<u64>(), fb.as<u64>());
  RuleTables T;
  if (!build_rule_tables(d, &T, budget, OwnItems{run, src, nullptr, N, (u32)R}, std::move(own), ~0ull, m))
    return false;
  // per-file tables: bound = segment windows + the root references' bounds,
  // cap = min(tokens_f - (l-1), distinct grams)
  DBuf fcap((u64)nseg * 4 + 4, st), fcap64((u64)nseg * 8 + 8, st), foff((u64)nseg * 8 + 8, st);
  if (d->n_rs)
    BK(k_file_bounds, d->n_rs, d->rs_rule.as<u32>(), d->rs_seg.as<u32>(), d->n_rs, (const u32*)nullptr, 0ull,
       file_lo, nseg, T.bound.as<u64>(), fb.as<u64>());
  BK(k_file_caps, nseg, fb.as<u64>(), d->seg_tokens.as<u64>(), file_lo, nruns, m, nseg, fcap.as<u32>(),
     fcap64.as<u64>());
  GT_CUDA(cudaMemsetAsync(fcap64.as<u64>() + nseg, 0, 8, st));
  exclusive_scan_u64(fcap64.as<u64>(), foff.as<u64>(), (u64)nseg + 1, st);
  const u64 FS = rd1<u64>(foff.as<u64>() + nseg, st);
  if ((T.S + FS) * 12 > budget) return false;
  DBuf fkeys(FS * 4 + 4, st), fvals(FS * 8 + 8, st), full(4, st);
  GT_CUDA(cudaMemsetAsync(fkeys.p, 0xFF, FS * 4 + 4, st));
  GT_CUDA(cudaMemsetAsync(fvals.p, 0, FS * 8 + 8, st));
  GT_CUDA(cudaMemsetAsync(full.p, 0, 4, st));
  if (N)  // _count_segments: the root segments' own windows
    BK(k_file_root_grams, N, run, src, N, (u32)R, fkeys.as<u32>(), fvals.as<u64>(), foff.as<u64>(),
       fcap.as<u32>(), full.as<u32>());
  if (d->n_rs) {  // level 2: seg_count(c, f) x table(c) (merge_with_retries over the root's children)
    DBuf deg(d->n_rs * 8 + 8, st), pos(d->n_rs * 8 + 8, st);
    BK(k_rs_slots, d->n_rs, d->rs_rule.as<u32>(), d->rs_seg.as<u32>(), d->n_rs, file_lo, nseg,
       T.tcap.as<u32>(), deg.as<u64>());
    exclusive_scan_u64(deg.as<u64>(), pos.as<u64>(), d->n_rs, st);
    BKE(k_level2_files, d->rs_rule.as<u32>(), d->rs_seg.as<u32>(), d->rs_cnt.as<u32>(), d->n_rs, file_lo,
        pos.as<u64>(), deg.as<u64>(), T.keys.as<u32>(), T.vals.as<u64>(), T.toff.as<u64>(), fkeys.as<u32>(),
        fvals.as<u64>(), foff.as<u64>(), fcap.as<u32>(), full.as<u32>());
  }
  if (rd1<u32>(full.p, st)) fail(GT_E_RESOURCE, "per-file gram table full (bound violated)");
  T = RuleTables();
  // occupied slots -> (file, run, count) -> (run, file) order
  DBuf occ(FS + 1, st), sel(FS * 4 + 4, st), nsel(8, st);
  BK(k_occupied, FS, fkeys.as<u32>(), FS, occ.as<uint8_t>());
  select_flagged_index(occ.as<uint8_t>(), sel.as<u32>(), nsel.as<u64>(), FS, st);
  const u64 n = rd1<u64>(nsel.p, st);
  DBuf file(n * 4 + 4, st), key(n * 4 + 4, st), cnt(n * 8 + 8, st);
  BK(k_slot_records, n, sel.as<u32>(), nsel.as<u64>(), fkeys.as<u32>(), fvals.as<u64>(), foff.as<u64>(), nseg,
     file.as<u32>(), key.as<u32>(), cnt.as<u64>());
  fkeys.release();
  fvals.release();
  const int FB = std::max(1, bitlen(nseg ? nseg - 1 : 0));
  const int KB = std::max(1, bitlen(nruns ? nruns - 1 : 0));
  if (KB + FB > 64) fail(GT_E_RESOURCE, "gram x file key of %d bits exceeds 64", KB + FB);
  DBuf k1(n * 8 + 8, st), k2(n * 8 + 8, st), idx(n * 4 + 4, st), idx2(n * 4 + 4, st);
  BK(k_iota_u32, n, idx.as<u32>(), n);
  BK(k_key_rf, n, file.as<u32>(), key.as<u32>(), n, FB, k1.as<u64>());
  sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), idx.as<u32>(), idx2.as<u32>(), n, KB + FB, st);
  crun.alloc(n * 4 + 4, st);
  ccol.alloc(n * 4 + 4, st);
  ccnt.alloc(n * 8 + 8, st);
  BK(k_split_rf, n, k2.as<u64>(), idx2.as<u32>(), cnt.as<u64>(), n, FB, crun.as<u32>(), ccol.as<u32>(),
     ccnt.as<u64>());
  *n_out = n;
  return true;
}

}  // namespace gt
