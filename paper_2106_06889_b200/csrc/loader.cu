// loader.cu — GTDC -> device DAG (CSR arrays) + topological level scheduler.
//
// Replaces deserialize_grammar (grammar.py:193-228), build_dag
// (dag.py:131-230) and the round discovery the reference's engine performs
// every traversal (engine.py:196-227 top-down mask rounds, engine.py:313-335
// bottom-up readiness rounds).  The host only walks the u32 length words (a
// sequential chain) and validates the dictionary; everything proportional to
// E runs on the device:
//   unpack -> (rule,symbol) radix sort -> run-length encode -> own/sub CSR
//   -> parent CSR (stable sort by child) -> per-rule sums
//   -> bottom-up layering (Kahn from the leaves; = reference bottom-up rounds,
//      doubles as the cycle check) -> top-down layering (Kahn over non-root
//      in-edges; = reference top-down rounds; carries reachability)
//   -> exp_len by bottom-up level -> root segments, segment tokens, root
//      occurrence lists -> word-major transpose of the own pairs.
// Error checks are reported in the reference's order and with its messages;
// the exact rule named in a cycle message needs the reference's DFS order,
// so only on that error path the host replays _topo_order (grammar.py:127).
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <initializer_list>
#include <memory>
#include <mutex>
#include <thread>

#include "kernels_common.cuh"
#include "segreduce.cuh"

namespace cg = cooperative_groups;

namespace gt {

thread_local u64 g_launches = 0;

void DBuf::alloc(size_t n, cudaStream_t st) {
  release();
  s = st;
  bytes = n;
  if (n) GT_CUDA(cudaMallocAsync(&p, n, st));
}

void DBuf::release() {
  if (p) cudaFreeAsync(p, s);
  p = nullptr;
  bytes = 0;
}

__global__ void k_csr_offsets(const u32* key, u64 n, u64 R, u64* off) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r <= R; r += stride) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
      u64 m = (lo + hi) >> 1;
      if (key[m] < r) lo = m + 1;
      else hi = m;
    }
    off[r] = lo;
  }
}

__global__ void k_iota_u32(u32* out, u64 n) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = (u32)i;
}

namespace {

// ---------------------------------------------------------------------------
// host parse (grammar.py:193-228 checks, same order and messages)
// ---------------------------------------------------------------------------

struct Parse {
  u64 nw = 0, ns = 0, R = 0;
  size_t rules_pos = 0;       // byte offset of the rules section
  u32* rstart = nullptr;      // u32 index (within the section) of rule i's first symbol (pinned)
  // body offset of rule i = rstart[i] - (i + 1) (one length word per rule)
  u64 Rp = 0;                 // rules fully parsed (R unless truncated)
  u64 boff(u64 i) const { return i < Rp ? (u64)rstart[i] - (i + 1) : E; }
  u64 blen(u64 i) const { return boff(i + 1) - boff(i); }
  u64 E = 0;
  long trunc_rule = -1;       // first incomplete rule (error pending range checks)
  std::string trunc_what;
  u64 trailing = 0;
};

static u32 rd32(const uint8_t* p) {
  u32 v;
  memcpy(&v, p, 4);
  return v;
}

static bool utf8_ok(const uint8_t* s, size_t n) {
  size_t i = 0;
  while (i < n) {
    uint8_t c = s[i];
    if (c < 0x80) {
      i++;
      continue;
    }
    int k;
    uint8_t lo = 0x80, hi = 0xBF;
    if (c >= 0xC2 && c <= 0xDF) k = 1;
    else if (c == 0xE0) { k = 2; lo = 0xA0; }
    else if (c >= 0xE1 && c <= 0xEC) k = 2;
    else if (c == 0xED) { k = 2; hi = 0x9F; }
    else if (c >= 0xEE && c <= 0xEF) k = 2;
    else if (c == 0xF0) { k = 3; lo = 0x90; }
    else if (c >= 0xF1 && c <= 0xF3) k = 3;
    else if (c == 0xF4) { k = 3; hi = 0x8F; }
    else return false;
    if (i + (size_t)k >= n) return false;
    if (s[i + 1] < lo || s[i + 1] > hi) return false;
    for (int j = 2; j <= k; j++)
      if (s[i + j] < 0x80 || s[i + j] > 0xBF) return false;
    i += (size_t)k + 1;
  }
  return true;
}

static void parse_dict(const uint8_t* d, size_t n, Parse* P) {
  if (n < 4 || memcmp(d, "GTDC", 4) != 0) fail(GT_E_FORMAT, "bad magic: not a GTDC file");
  size_t pos = 4;
  auto need = [&](u64 k, const char* what, long idx) {
    if ((u64)pos + k > (u64)n) {
      char buf[96];
      if (idx >= 0) snprintf(buf, sizeof buf, what, idx);
      else snprintf(buf, sizeof buf, "%s", what);
      fail(GT_E_FORMAT, "truncated input while reading %s", buf);
    }
  };
  need(1, "version", -1);
  uint8_t ver = d[pos++];
  if (ver != 1) fail(GT_E_FORMAT, "unsupported version %d", (int)ver);
  need(4, "word count", -1);
  P->nw = rd32(d + pos), pos += 4;
  need(4, "splitter count", -1);
  P->ns = rd32(d + pos), pos += 4;
  need(4, "rule count", -1);
  P->R = rd32(d + pos), pos += 4;
  if (P->R < 1) fail(GT_E_FORMAT, "grammar must contain a root rule");
  for (u64 i = 0; i < P->nw; i++) {
    need(4, "word %ld length", (long)i);
    u32 ln = rd32(d + pos);
    pos += 4;
    need(ln, "word %ld", (long)i);
    // ASCII fast path (8 bytes at a time), full UTF-8 validation otherwise
    const uint8_t* w = d + pos;
    u64 hi = 0;
    u32 k = 0;
    for (; k + 8 <= ln; k += 8) {
      u64 x;
      memcpy(&x, w + k, 8);
      hi |= x;
    }
    for (; k < ln; k++) hi |= w[k];
    if ((hi & 0x8080808080808080ull) && !utf8_ok(w, ln))
      fail(GT_E_FORMAT, "word %ld is not valid UTF-8", (long)i);
    pos += ln;
  }
  P->rules_pos = pos;
}

// The rules section is a chain of (length, body) records: walking it is the
// one inherently sequential step of the load, so it runs on the host while
// the section itself is already streaming to the device.
static void parse_rules(const uint8_t* d, size_t n, Parse* P) {
  size_t pos = P->rules_pos;
  u32* rs = P->rstart;
  u64 E = 0, i = 0;
  for (; i < P->R; i++) {
    if ((u64)pos + 4 > (u64)n) {
      P->trunc_rule = (long)i;
      P->trunc_what = "rule %ld body length";
      break;
    }
    u32 ln = rd32(d + pos);
    if ((u64)pos + 4 + 4ull * ln > (u64)n) {
      P->trunc_rule = (long)i;
      P->trunc_what = "rule %ld body";
      break;
    }
    rs[i] = (u32)((pos + 4 - P->rules_pos) / 4);
    E += ln;
    pos += 4 + 4ull * ln;
  }
  P->Rp = i;
  if (P->trunc_rule < 0) P->trailing = (u64)n - (u64)pos;
  P->E = E;
}

// range check of rules [0, upto) on the host: only used on error paths
static void host_range_check(const uint8_t* d, const Parse& P, u64 upto) {
  u64 limit = P.nw + P.ns + P.R;
  const uint8_t* sec = d + P.rules_pos;
  for (u64 i = 0; i < upto; i++) {
    u64 lo = P.rstart[i], ln = P.blen(i);
    u32 mx = 0;
    for (u64 j = 0; j < ln; j++) mx = std::max(mx, rd32(sec + 4 * (lo + j)));
    if (ln && mx >= limit)
      fail(GT_E_FORMAT, "rule %lu contains symbol %u out of range", (unsigned long)i, mx);
  }
}

// _topo_order (grammar.py:127-161) replay for the cycle message only
[[noreturn]] static void cycle_message(const uint8_t* d, const Parse& P) {
  u64 R = P.R, base = P.nw + P.ns;
  const uint8_t* sec = d + P.rules_pos;
  std::vector<int8_t> state(R, 0);
  std::vector<std::pair<u64, u64>> st;
  for (u64 start = 0; start < R; start++) {
    if (state[start]) continue;
    st.clear();
    st.push_back({start, 0});
    state[start] = 1;
    while (!st.empty()) {
      auto [r, pos] = st.back();
      st.pop_back();
      u64 len = P.blen(r);
      bool adv = false;
      while (pos < len) {
        u64 s = rd32(sec + 4 * (P.rstart[r] + pos));
        pos++;
        if (s >= base) {
          u64 c = s - base;
          if (state[c] == 1) fail(GT_E_CORRUPTION, "rule reference cycle through rule %lu", (unsigned long)c);
          if (state[c] == 0) {
            st.push_back({r, pos});
            st.push_back({c, 0});
            state[c] = 1;
            adv = true;
            break;
          }
        }
      }
      if (!adv) state[r] = 2;
    }
  }
  fail(GT_E_CORRUPTION, "rule reference cycle (not located)");
}

// ---------------------------------------------------------------------------
// device kernels of the build
// ---------------------------------------------------------------------------

__global__ void k_mark_len(const u32* rstart, u64 R, u32* mark) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += stride)
    mark[rstart[i] - 1] = 1;
}

// ---- rule-chain parse on the device (pointer doubling) ----------------------
// The rules section is a chain of (length, body) records: record i starts at
// p_i, p_{i+1} = p_i + 1 + len(p_i).  With J_0(j) = j + 1 + raw[j] (clamped
// to the end n) for EVERY word j and J_{k+1} = J_k o J_k, the start of rule i
// is J applied along the binary digits of i to p_0 = 0: log2(R) doubling
// passes over the section plus log2(R) passes over the rules, all parallel.
__global__ void k_jump0(const u32* raw, u64 n, u32* J) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j <= n; j += stride) {
    const u64 nx = j < n ? j + 1 + (u64)raw[j] : n;
    J[j] = (u32)(nx < n ? nx : n);
  }
}

__global__ void k_jump_double(const u32* __restrict__ Jk, u64 n, u32* __restrict__ Jk1) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j <= n; j += stride) Jk1[j] = Jk[Jk[j]];
}

// start of rule i = J applied along the binary digits of i to p_0 = 0 (one
// thread per rule, K dependent table lookups)
__global__ void k_chain_pos(const u32* __restrict__ J, u64 n, int K, u64 R, u32* pos) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += stride) {
    u32 p = 0;
    for (int k = K - 1; k >= 0; k--)
      if ((i >> k) & 1) p = J[(u64)k * (n + 1) + p];
    pos[i] = p;
  }
}

// every rule start inside the section, the last record ending exactly at the
// end; rstart = first symbol of each rule
__global__ void k_chain_check(const u32* pos, const u32* raw, u64 R, u64 n, u32* bad, u32* rstart) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += stride) {
    const u64 p = pos[i];
    if (p >= n) {
      *bad = 1;
      continue;
    }
    rstart[i] = (u32)(p + 1);
    if (i + 1 == R && p + 1 + (u64)raw[p] != n) *bad = 1;
  }
}

__global__ void k_boff(const u32* rstart, u64 R, u64 E, u64* boff) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= R; i += stride)
    boff[i] = i < R ? (u64)rstart[i] - (i + 1) : E;
}

__global__ void k_unpack(const u32* raw, const u32* mark, const u32* incl, u64 n, u32* body,
                         u32* owner, u64 limit, u32* bad_rule) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    if (mark[p]) continue;
    u32 r = incl[p] - 1;
    u64 i = p - ((u64)r + 1);
    u32 s = raw[p];
    body[i] = s;
    owner[i] = r;
    if ((u64)s >= limit) atomicMin(bad_rule, r);
  }
}

__global__ void k_make_keys(const u32* body, const u32* owner, u64 E, int SB, u64* keys) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += stride)
    keys[i] = ((u64)owner[i] << SB) | body[i];
}

__global__ void k_heads(const u64* k, u64 n, uint8_t* head) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    head[i] = (i == 0 || k[i] != k[i - 1]);
}

__global__ void k_heads_seg(const u32* sym, const u32* owner, u64 n, uint8_t* head) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    head[i] = (i == 0 || sym[i] != sym[i - 1] || owner[i] != owner[i - 1]);
}

__global__ void k_rle_seg(const u32* sym_sorted, const u32* owner, const u32* hidx, const u64* Ud, u64 n, u64 nw,
                          u64 base, u32* pr_rule, u32* pr_sym, u32* pr_cnt, uint8_t* is_own, uint8_t* is_sub) {
  const u64 U = *Ud;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += stride) {
    const u64 a = hidx[u], b = (u + 1 < U) ? hidx[u + 1] : n;
    const u64 sym = sym_sorted[a];
    pr_rule[u] = owner[a];
    pr_cnt[u] = (u32)(b - a);
    is_own[u] = sym < nw;
    is_sub[u] = sym >= base;
    pr_sym[u] = (u32)(sym >= base ? sym - base : sym);
  }
}

// unique (rule, sym) runs -> pair arrays + class flags
__global__ void k_rle(const u64* sk, const u32* hidx, const u64* Ud, u64 n, int SB, u64 nw, u64 base,
                      u32* pr_rule, u32* pr_sym, u32* pr_cnt, uint8_t* is_own, uint8_t* is_sub) {
  const u64 U = *Ud;
  u64 stride = (u64)gridDim.x * blockDim.x;
  u64 mask = (1ull << SB) - 1;
  for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += stride) {
    u64 a = hidx[u], b = (u + 1 < U) ? hidx[u + 1] : n;
    u64 key = sk[a];
    u64 sym = key & mask;
    pr_rule[u] = (u32)(key >> SB);
    pr_cnt[u] = (u32)(b - a);
    is_own[u] = sym < nw;
    is_sub[u] = sym >= base;
    pr_sym[u] = (u32)(sym >= base ? sym - base : sym);
  }
}

__global__ void k_gather3(const u32* idx, u64 n, const u32* a, const u32* b, const u32* c, u32* oa,
                          u32* ob, u32* oc) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 j = idx[i];
    oa[i] = a[j];
    ob[i] = b[j];
    if (c) oc[i] = c[j];
  }
}

// distinct children / non-root parents counters; root-parent flag
__global__ void k_degrees(const u64* sub_off, const u64* par_off, const u32* par_ids, u64 R,
                          u32* rem_bu, u32* rem_td, uint8_t* root_parent) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride) {
    rem_bu[r] = (u32)(sub_off[r + 1] - sub_off[r]);
    u64 np = par_off[r + 1] - par_off[r];
    bool rp = np && par_ids[par_off[r]] == 0;
    root_parent[r] = rp;
    rem_td[r] = (u32)(np - (rp ? 1 : 0));
  }
}

__global__ void k_flag_zero(const u32* rem, u64 R, u64 first, uint8_t* flag) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride)
    flag[r] = (r >= first) && rem[r] == 0;
}

// Warp-aggregated "decrement and detect completion": lanes hitting the same
// counter subtract together (one atomic per distinct counter per warp, so a
// rule with 10^5 parents finishing in one layer does not serialise 10^5
// same-address atomics); exactly one lane reports the counter reaching zero.
// Must be called by every lane of the warp.
__device__ __forceinline__ bool dec_to_zero(u32* rem, u32 key, bool active) {
  const unsigned act = __ballot_sync(0xFFFFFFFFu, active);
  if (!active) return false;
  const unsigned peers = __match_any_sync(act, key);
  const unsigned lane = threadIdx.x & 31u;
  if ((int)lane != __ffs(peers) - 1) return false;
  const u32 k = (u32)__popc(peers);
  return atomicSub(&rem[key], k) == k;
}

// ---------------------------------------------------------------------------
// Persistent Kahn layering: ONE cooperative launch runs every layer, frontier
// counts live on the device, layers are separated by grid barriers (no host
// round trip per layer).  Bottom-up (TD = false): frontier = rules whose
// children all finished, edges = parents (par CSR).  Top-down (TD = true):
// frontier = rules whose non-root parents all finished, edges = children
// (sub CSR), reachability from the root carried along.  A rule with more
// than kLight edges is split into chunk tasks of kChunk edges that every
// warp of the grid shares after a second barrier (a rule with 10^6 parents
// is never one warp's serial loop).
// ---------------------------------------------------------------------------
constexpr u32 kLight = 8, kChunk = 256;

// warp-aggregated append of the lanes with `take` set (one atomic per warp
// on the shared frontier counter instead of one per completed rule; must be
// called by every lane of the warp)
__device__ __forceinline__ void warp_append(bool take, u32 v, u32* q, u64* cnt) {
  const unsigned m = __ballot_sync(0xFFFFFFFFu, take);
  if (!m) return;
  const unsigned lane = threadIdx.x & 31u;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if ((int)lane == leader) base = atomicAdd((unsigned long long*)cnt, (unsigned long long)__popc(m));
  base = __shfl_sync(0xFFFFFFFFu, base, leader);
  if (take) q[base + __popc(m & ((1u << lane) - 1u))] = v;
}

struct KahnCtl {
  u64 cnt[3];    // rotating frontier counts: layer L reads cnt[L%3], appends to cnt[(L+1)%3]
  u64 ntask[2];  // heavy-task counts, layer L uses ntask[L&1]
  u64 processed;
  u64 layers;
};

__device__ __forceinline__ u64 ld_cg64(const u64* p) {
  return (u64)__ldcg(reinterpret_cast<const unsigned long long*>(p));
}

constexpr int kKahnBlock = 1024;  // few, large blocks: cheaper grid barriers

template <bool TD>
__global__ void __launch_bounds__(kKahnBlock) k_kahn(KahnCtl* ctl, u32* q0, u32* q1, const u64* __restrict__ off,
                                              const u32* __restrict__ ids, u32* rem, u32* lvl,
                                              const u64* __restrict__ par_off,
                                              const u32* __restrict__ par_ids,
                                              const uint8_t* __restrict__ root_parent, uint8_t* reach,
                                              uint2* tasks, u64 max_layers) {
  cg::grid_group grid = cg::this_grid();
  const u64 gtid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 nthreads = (u64)gridDim.x * blockDim.x;
  const unsigned lane = threadIdx.x & 31u;
  u64 total = 0, L = 1;
  for (;; L++) {
    const u64 n = ld_cg64(&ctl->cnt[L % 3]);
    if (n == 0 || L > max_layers) break;
    total += n;
    if (gtid == 0) {
      ctl->cnt[(L + 2) % 3] = 0;
      ctl->ntask[(L + 1) & 1] = 0;
    }
    const u32* cur = (L & 1) ? q1 : q0;
    u32* nxt = (L & 1) ? q0 : q1;
    u64* ncnt = &ctl->cnt[(L + 1) % 3];
    u64* ntask = &ctl->ntask[L & 1];
    // phase A: light rules inline, heavy rules -> chunk tasks
    for (u64 base = (u64)blockIdx.x * blockDim.x; base < n; base += nthreads) {
      const u64 i = base + threadIdx.x;
      const bool active = i < n;
      u32 r = 0;
      u64 e0 = 0, len = 0;
      if (active) {
        r = __ldcg(cur + i);
        lvl[r] = (u32)L;
        if (TD) {
          bool rc = root_parent[r];
          const volatile uint8_t* rv = reach;
          for (u64 e = par_off[r]; e < par_off[r + 1] && !rc; e++) {
            const u32 p = par_ids[e];
            if (p != 0 && rv[p]) rc = true;
          }
          reach[r] = rc;
        }
        e0 = off[r];
        len = off[r + 1] - e0;
        if (len > kLight) {
          const u64 nch = (len + kChunk - 1) / kChunk;
          const u64 t0 = atomicAdd((unsigned long long*)ntask, (unsigned long long)nch);
          for (u64 k = 0; k < nch; k++) tasks[t0 + k] = make_uint2(r, (u32)(k * kChunk));
          len = 0;
        }
      }
      // the warp's light edges dealt round-robin over its lanes: exclusive
      // scan of the per-lane counts, then lane j takes edge k*32 + j and finds
      // its owning lane by a shuffle binary search (no lane walks a long list)
      u32 inc = (u32)len;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= (unsigned)d) inc += t;
      }
      const u32 excl = inc - (u32)len;
      const u32 tot = __shfl_sync(0xFFFFFFFFu, inc, 31);
      for (u32 k0 = 0; k0 < tot; k0 += 32) {
        const u32 q = k0 + lane;
        // owner = last lane whose exclusive start <= q
        int lo = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
          const u32 st_ex = __shfl_sync(0xFFFFFFFFu, excl, lo + step);
          if (st_ex <= q) lo += step;
        }
        const u32 own_start = __shfl_sync(0xFFFFFFFFu, excl, lo);
        const u64 own_e0 = __shfl_sync(0xFFFFFFFFu, e0, lo);
        const bool a = q < tot;
        const u32 c = a ? ids[own_e0 + (q - own_start)] : 0u;
        warp_append(dec_to_zero(rem, c, a), c, nxt, ncnt);
      }
    }
    grid.sync();
    // phase B: chunk tasks, one warp per task (most top-down layers have none:
    // then the second barrier is skipped, uniformly across the grid)
    const u64 nt = ld_cg64(ntask);
    if (nt == 0) continue;
    for (u64 t = gtid >> 5; t < nt; t += nthreads >> 5) {
      const uint2 tk = __ldcg(tasks + t);
      const u64 a = off[tk.x] + tk.y, b = min(off[tk.x + 1], a + kChunk);
      for (u64 e = a; e < b; e += 32) {
        const bool act = e + lane < b;
        const u32 c = act ? ids[e + lane] : 0u;
        warp_append(dec_to_zero(rem, c, act), c, nxt, ncnt);
      }
    }
    grid.sync();
  }
  if (gtid == 0) {
    ctl->processed = total;
    ctl->layers = L - 1;
  }
}

// Bottom-up sums in ONE persistent reverse-level pass over the child edges
// (children before parents): height(r) = max(1, 1 + height(child)) (the
// reference's bottom-up round, engine.py:313-335) and exp_len(r) = own tokens
// + Σ f · exp_len(child) (grammar.py:109-124).  Per 32-item warp step both
// values are combined by dst with shuffle scans and flushed with one atomicMax
// and one atomicAdd per run.
__global__ void __launch_bounds__(1024) k_bu_pair(const u32* __restrict__ rule, const u32* __restrict__ child,
                                                  const u32* __restrict__ freq, const u64* __restrict__ lvl_off,
                                                  int L1, u64* hgt, u64* elen) {
  cg::grid_group grid = cg::this_grid();
  const unsigned lane = threadIdx.x & 31u;
  const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (int L = L1; L >= 0; L--) {
    const u64 a = lvl_off[L], n = lvl_off[L + 1] - a;
    for (u64 base = a + warp * 32; base < a + n; base += nwarps * 32) {
      const u64 i = base + lane;
      const bool ok = i < a + n;
      const u32 d = ok ? rule[i] : 0xFFFFFFFFu;
      u64 hv = 0, ev = 0;
      if (ok) {
        const u32 c = child[i];
        hv = ld_cg64(hgt + c) + 1;
        ev = (u64)freq[i] * ld_cg64(elen + c);
      }
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const u64 oh = __shfl_up_sync(0xFFFFFFFFu, hv, k);
        const u64 oe = __shfl_up_sync(0xFFFFFFFFu, ev, k);
        const u32 od = __shfl_up_sync(0xFFFFFFFFu, d, k);
        if (lane >= (unsigned)k && od == d) {
          hv = hv > oh ? hv : oh;
          ev += oe;
        }
      }
      const u32 dn = __shfl_down_sync(0xFFFFFFFFu, d, 1);
      if (ok && (lane == 31 || dn != d)) {
        atomicMax((unsigned long long*)&hgt[d], (unsigned long long)hv);
        if (ev) atomicAdd((unsigned long long*)&elen[d], (unsigned long long)ev);
      }
    }
    if (L > 0) grid.sync();
  }
}


// level key of every edge; edges not kept (root parents) sort after all levels
__global__ void k_edge_level_keys2(const u32* group_of, const uint8_t* keep, const u32* lvl, u32 drop_key, u64 n,
                                   u32* key) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = (keep && !keep[i]) ? drop_key : lvl[group_of[i]];
}

__global__ void k_flag_nonzero_u32(const u32* v, u64 n, uint8_t* f) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) f[i] = v[i] != 0;
}

__global__ void k_root_cycle(const u64* par_off, const u32* par_ids, const uint8_t* reach, u32* bad) {
  for (u64 e = par_off[0] + threadIdx.x; e < par_off[1]; e += blockDim.x) {
    const u32 p = par_ids[e];
    if (p == 0 || reach[p]) *bad = 1;
  }
}

__global__ void k_fill_u64(u64* a, u64 n, u64 v) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = v;
}

__global__ void k_u64_to_u32(const u64* a, u64 n, u32* b) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = (u32)a[i];
}

__global__ void k_first_unreached(const uint8_t* reach, u64 R, u32* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = 1 + (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride)
    if (!reach[r]) atomicMin(out, (u32)r);
}

// level sort key: level*2 + heavy (heavy = more than `th` CSR entries)
__global__ void k_level_key(const u32* lvl, const u64* off, u64 R, u64 th, u32* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride)
    key[r] = lvl[r] * 2u + ((off[r + 1] - off[r]) > th ? 1u : 0u);
}

// root body: splitter flags, per-position segment (inclusive scan later)
__global__ void k_root_flags(const u32* body, u64 L0, u64 nw, u64 base, uint8_t* spl, u32* splu) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < L0; p += stride) {
    u32 s = body[p];
    bool f = s >= nw && s < base;
    spl[p] = f;
    splu[p] = f;
  }
}

__global__ void k_check_splitters(const u32* body, const u32* spos, const u64* nspl, u64 nw,
                                  u32* first_bad) {
  u64 n = *nspl;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
    if ((u64)body[spos[k]] - nw != k) atomicMin(first_bad, (u32)k);
}

__global__ void k_segments(const u32* spos, u64 F, u64 L0, bool headless, u64* lo, u64* hi) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 f = (u64)blockIdx.x * blockDim.x + threadIdx.x; f < F; f += stride) {
    if (headless) {
      lo[f] = 0;
      hi[f] = L0;
    } else {
      lo[f] = f ? (u64)spos[f - 1] + 1 : 0;
      hi[f] = spos[f];
    }
  }
}

// root positions -> (rule|word, segment) keys; class flags
__global__ void k_root_keys(const u32* body, const u32* seg_incl, u64 L0, u64 nw, u64 base,
                            int SBF, bool headless, u64* rkey, uint8_t* isr, u64* wkey,
                            uint8_t* isw, u32* seg_of) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < L0; p += stride) {
    u32 s = body[p];
    u32 seg = headless ? 0u : seg_incl[p];  // splitters before p (p itself not a splitter)
    seg_of[p] = seg;
    bool rr = s >= base, ww = s < nw;
    isr[p] = rr;
    isw[p] = ww;
    rkey[p] = rr ? (((u64)(s - base) << SBF) | seg) : 0;
    wkey[p] = ww ? (((u64)s << SBF) | seg) : 0;
  }
}

// compacted sorted keys -> RLE (id, seg, cnt)
__global__ void k_rle_keys(const u64* sk, const u32* hidx, u64 U, u64 n, int SBF, u32* id,
                           u32* seg, u32* cnt) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += stride) {
    u64 a = hidx[u], b = (u + 1 < U) ? hidx[u + 1] : n;
    u64 k = sk[a];
    id[u] = (u32)(k >> SBF);
    seg[u] = (u32)(k & ((1ull << SBF) - 1));
    cnt[u] = (u32)(b - a);
  }
}

__global__ void k_gather_u64(const u32* idx, u64 n, const u64* src, u64* dst) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[idx[i]];
}

struct ValU32 {
  const u32* a;
  __device__ u64 operator()(u64 i) const { return a[i]; }
};
struct ValU32NonRoot {
  const u32* a;
  const u32* who;
  __device__ u64 operator()(u64 i) const { return who[i] ? (u64)a[i] : 0ull; }
};
struct ValRootLen {
  const u32* body;
  const u64* exp_len;
  u64 nw, base;
  __device__ u64 operator()(u64 p) const {
    u32 s = body[p];
    return s < nw ? 1ull : (s >= base ? exp_len[s - base] : 0ull);
  }
};

template <class T>
static void d2h(T* dst, const void* src, size_t n, cudaStream_t s) {
  GT_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  GT_CUDA(cudaStreamSynchronize(s));
}

#define LAUNCH(k, n, ...) GT_KLAUNCH(#k, k, grid_for((n), 256), 256, st, __VA_ARGS__)

static void build_levels(DeviceDag* d, const DBuf& lvl, const DBuf& off, u64 th, int nl, Levels* out) {
  cudaStream_t st = d->stream;
  u64 R = d->R;
  DBuf key(R * 4, st), key2(R * 4, st), ids(R * 4, st);
  out->order.alloc(R * 4, st);
  LAUNCH(k_level_key, R, lvl.as<u32>(), off.as<u64>(), R, th, key.as<u32>());
  LAUNCH(k_iota_u32, R, ids.as<u32>(), R);
  sort_pairs_u32_u32(key.as<u32>(), key2.as<u32>(), ids.as<u32>(), out->order.as<u32>(), R,
                     bitlen((u64)nl * 2 + 1), st);
  // boundaries for keys 0..2*nl+1
  u64 nk = (u64)nl * 2 + 2;
  DBuf koff((nk + 1) * 8, st);
  LAUNCH(k_csr_offsets, nk + 1, key2.as<u32>(), R, nk, koff.as<u64>());
  std::vector<u64> h(nk + 1);
  d2h(h.data(), koff.p, nk + 1, st);
  out->nl = nl;
  out->off.assign(nl + 2, 0);
  out->heavy_off.assign(nl + 2, 0);
  for (int L = 0; L <= nl; L++) {
    out->off[L] = h[2 * L];
    out->heavy_off[L] = h[2 * L + 1];
  }
  out->off[nl + 1] = R;
}

// The stream-ordered pool keeps freed memory (release threshold = inf) and,
// once per device, is grown to GT_POOL_RESERVE_FRAC (default 0.4) of the HBM
// in one allocation: the task paths allocate and free multi-GB scratch whose
// sizes vary run to run, and growing the pool on demand (mapping physical
// pages inside a run) costs 10^2 ms per GB-scale step and fragments it.
static void reserve_pool(int device, cudaStream_t st) {
  static std::mutex mu;  // contexts may be opened from several threads (one per device)
  std::lock_guard<std::mutex> lock(mu);
  static bool done[64] = {};
  cudaMemPool_t pool;
  GT_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  u64 thr = UINT64_MAX;
  GT_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  if (done[device & 63]) return;
  done[device & 63] = true;
  double frac = 0.4;
  if (const char* e = getenv("GT_POOL_RESERVE_FRAC")) frac = atof(e);
  size_t free_b = 0, total_b = 0;
  GT_CUDA(cudaMemGetInfo(&free_b, &total_b));
  size_t want = (size_t)(frac * (double)total_b);
  if (want > free_b / 10 * 9) want = free_b / 10 * 9;
  u64 cur = 0;
  GT_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &cur));
  if (want <= cur || want < (64ull << 20)) return;
  void* p = nullptr;
  if (cudaMallocAsync(&p, want, st) == cudaSuccess) {
    GT_CUDA(cudaFreeAsync(p, st));
    GT_CUDA(cudaStreamSynchronize(st));
  } else {
    cudaGetLastError();  // best effort: the pool then grows on demand
  }
}

// buffers allocated on a helper stream are released on the context stream
static void rebind_stream(cudaStream_t st, std::initializer_list<DBuf*> bufs) {
  for (DBuf* b : bufs) b->s = st;
}

struct PinnedU64 {  // grow-only pinned host buffer (deferred read-backs)
  u64* p = nullptr;
  u64 cap = 0;
  u64* get(u64 n) {
    if (n > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = std::max<u64>(n, 1u << 12);
      GT_CUDA(cudaMallocHost(&p, cap * 8));
    }
    return p;
  }
};

// grow-only pinned host buffer (the rule-start table of the chain walk)
struct PinnedU32 {
  u32* p = nullptr;
  u64 cap = 0;
  u32* get(u64 n) {
    if (n > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = std::max<u64>(n, 1u << 16);
      GT_CUDA(cudaMallocHost(&p, cap * 4));
    }
    return p;
  }
};

}  // namespace

void ensure_bu_levels(DeviceDag* d) {
  if (d->bu.order.p || d->R == 0) return;
  GT_CUDA(cudaSetDevice(d->device));
  const int nl = d->bu.nl;
  build_levels(d, d->bu_level, d->sub_off, 16, nl, &d->bu);
}

void build_device_dag(const uint8_t* blob, size_t nbytes, int device, u64 file_lo, u64 file_hi,
                      DeviceDag* d) {
  auto t0 = std::chrono::steady_clock::now();
  Phases ph("gt_open");
  Parse P;
  if (nbytes < 4 || memcmp(blob, "GTDC", 4) != 0) fail(GT_E_FORMAT, "bad magic: not a GTDC file");
  GT_CUDA(cudaSetDevice(device));
  d->device = device;
  if (!d->stream) GT_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
  cudaStream_t st = d->stream;
  ph.st = st;
  reserve_pool(device, st);
  ph.mark("stream");
  // the whole blob streams to the device while the host validates the
  // header and dictionary (overlaps when `blob` is pinned); the rules section
  // is then re-aligned on the device (the dictionary has byte lengths)
  DBuf dblob(nbytes + 4, st);
  GT_CUDA(cudaMemcpyAsync(dblob.p, blob, nbytes, cudaMemcpyHostToDevice, st));
  parse_dict(blob, nbytes, &P);
  ph.mark("host parse: dictionary");
  const u64 nsec = (nbytes - P.rules_pos) / 4;
  DBuf raw(nsec * 4 + 4, st);
  if (nsec) GT_CUDA(cudaMemcpyAsync(raw.p, dblob.as<uint8_t>() + P.rules_pos, nsec * 4, cudaMemcpyDeviceToDevice, st));
  dblob.release();
  // the rule-start table: on the device by pointer doubling; the host walk
  // (parse_rules, the reference's sequential reader) runs only to produce the
  // exact error of a malformed section, or when an error path needs it
  static thread_local PinnedU32 rstart_host;
  bool host_chain = false;
  auto need_host_chain = [&]() {
    if (host_chain) return;
    GT_CUDA(cudaStreamSynchronize(st));
    P.rstart = rstart_host.get(P.R);
    parse_rules(blob, nbytes, &P);
    host_chain = true;
  };
  DBuf rstart(P.R * 4 + 4, st);
  {
    const u64 n = nsec;
    const int K = bitlen(P.R - 1);  // J_0 .. J_{K-1}
    bool ok = n >= 1 && n < 0xFFFFFFFFull && (nbytes - P.rules_pos) % 4 == 0;
    if (ok) {
      DBuf J((u64)std::max(K, 1) * (n + 1) * 4, st), pos(P.R * 4, st), bad(4, st);
      u32* Jb = J.as<u32>();
      LAUNCH(k_jump0, n + 1, raw.as<u32>(), n, Jb);
      for (int k = 1; k < K; k++)
        LAUNCH(k_jump_double, n + 1, Jb + (u64)(k - 1) * (n + 1), n, Jb + (u64)k * (n + 1));
      LAUNCH(k_chain_pos, P.R, Jb, n, K, P.R, pos.as<u32>());
      GT_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
      LAUNCH(k_chain_check, P.R, pos.as<u32>(), raw.as<u32>(), P.R, n, bad.as<u32>(), rstart.as<u32>());
      u32 b = 0;
      d2h(&b, bad.p, 1, st);
      ok = b == 0;
    }
    if (ok) {
      P.E = n - P.R;
      P.Rp = P.R;
      P.trailing = 0;
    } else {
      need_host_chain();  // malformed: reproduce the reference's error
      if (P.trunc_rule >= 0) {
        host_range_check(blob, P, (u64)P.trunc_rule);
        char buf[96];
        snprintf(buf, sizeof buf, P.trunc_what.c_str(), P.trunc_rule);
        fail(GT_E_FORMAT, "truncated input while reading %s", buf);
      }
      if (P.trailing) {
        host_range_check(blob, P, P.R);
        fail(GT_E_FORMAT, "%lu trailing bytes after rules section", (unsigned long)P.trailing);
      }
    }
  }
  ph.mark("rule chain (device)");
  const u64 R = P.R, E = P.E, nw = P.nw, ns = P.ns, base = nw + ns, limit = nw + ns + R;
  d->nw = nw;
  d->ns = ns;
  d->R = R;
  d->E = E;
  const u64 nraw = E + R;

  // ---- unpack --------------------------------------------------------------
  DBuf mark(nraw * 4 + 4, st), incl(nraw * 4 + 4, st);
  DBuf& owner = d->pos_owner;
  owner.alloc(E * 4 + 4, st);
  DBuf bad(4, st);
  d->body.alloc(E * 4 + 4, st);
  d->boff.alloc((R + 1) * 8, st);
  if (host_chain) GT_CUDA(cudaMemcpyAsync(rstart.p, P.rstart, R * 4, cudaMemcpyHostToDevice, st));
  LAUNCH(k_boff, R + 1, rstart.as<u32>(), R, E, d->boff.as<u64>());
  GT_CUDA(cudaMemsetAsync(mark.p, 0, nraw * 4, st));
  GT_CUDA(cudaMemsetAsync(bad.p, 0xFF, 4, st));
  LAUNCH(k_mark_len, R, rstart.as<u32>(), R, mark.as<u32>());
  inclusive_scan_u32(mark.as<u32>(), incl.as<u32>(), nraw, st);
  LAUNCH(k_unpack, nraw, raw.as<u32>(), mark.as<u32>(), incl.as<u32>(), nraw, d->body.as<u32>(),
         owner.as<u32>(), limit, bad.as<u32>());
  raw.release();
  mark.release();
  incl.release();
  rstart.release();
  u32 bad_rule;
  d2h(&bad_rule, bad.p, 1, st);
  if (bad_rule != 0xFFFFFFFFu) {
    need_host_chain();
    host_range_check(blob, P, bad_rule + 1);
  }
  ph.mark("upload+unpack");

  // ---- root side (splitters, segments, root occurrence lists): only needs
  // the root body, so it runs on its own stream and host thread while the
  // main pipeline builds the CSR, the layering and the level lists; its
  // errors are raised after the main pipeline's, in the reference's order
  // (dag.py:131-230: cycle, unreachable, then _segments_of_root)
  const u64 L0 = R ? rd32(blob + P.rules_pos) : 0;  // the root's body length
  d->L0 = L0;
  cudaEvent_t ev_body;
  GT_CUDA(cudaEventCreateWithFlags(&ev_body, cudaEventDisableTiming));
  GT_CUDA(cudaEventRecord(ev_body, st));
  Error root_err{GT_OK, ""};
  cudaStream_t s_root = nullptr;
  GT_CUDA(cudaStreamCreateWithFlags(&s_root, cudaStreamNonBlocking));
  auto root_side = [&]() {
    try {
      GT_CUDA(cudaSetDevice(device));
      cudaStream_t st = s_root;
      GT_CUDA(cudaStreamWaitEvent(st, ev_body, 0));
      DBuf cnt(16, st);
  // ---- root segments (dag.py:107-128) -------------------------------------
    const bool headless = ns == 0;
    DBuf spl(L0 + 1, st), splu(L0 * 4 + 4, st), sincl(L0 * 4 + 4, st), spos(L0 * 4 + 4, st);
    LAUNCH(k_root_flags, L0, d->body.as<u32>(), L0, nw, base, spl.as<uint8_t>(), splu.as<u32>());
    select_flagged_index(spl.as<uint8_t>(), spos.as<u32>(), cnt.as<u64>(), L0, st);
    inclusive_scan_u32(splu.as<u32>(), sincl.as<u32>(), L0, st);
    u64 nspl;
    d2h(&nspl, cnt.p, 1, st);
    if (!headless) {
      DBuf fb(4, st);
      GT_CUDA(cudaMemsetAsync(fb.p, 0xFF, 4, st));
      LAUNCH(k_check_splitters, nspl ? nspl : 1, d->body.as<u32>(), spos.as<u32>(), cnt.as<u64>(), nw,
             fb.as<u32>());
      u32 k;
      d2h(&k, fb.p, 1, st);
      if (k != 0xFFFFFFFFu) {
        u32 pos, sym;
        d2h(&pos, spos.as<u32>() + k, 1, st);
        d2h(&sym, d->body.as<u32>() + pos, 1, st);
        fail(GT_E_CORRUPTION, "splitter %u out of order at root position %u", sym, pos);
      }
      if (nspl != ns) fail(GT_E_CORRUPTION, "root body is missing file splitters");
      u32 last = 0;
      if (nspl) d2h(&last, spos.as<u32>() + nspl - 1, 1, st);
      if (!nspl || (u64)last + 1 != L0) fail(GT_E_CORRUPTION, "root body has content after the last splitter");
    }
    const u64 F = headless ? 1 : ns;
    d->F = F;
    d->file_lo = std::min(file_lo, F);
    d->file_hi = std::min(file_hi, F);
    if (d->file_hi < d->file_lo) d->file_hi = d->file_lo;
    d->seg_lo.alloc(F * 8, st);
    d->seg_hi.alloc(F * 8, st);
    LAUNCH(k_segments, F, spos.as<u32>(), F, L0, headless, d->seg_lo.as<u64>(), d->seg_hi.as<u64>());
  // ---- segment tokens + root occurrence lists ------------------------------
    const int SBF = std::max(1, bitlen(F - 1));
    DBuf rkey(L0 * 8 + 8, st), wkey(L0 * 8 + 8, st), isr(L0 + 1, st), isw(L0 + 1, st);
    DBuf& segof = d->root_seg;
    segof.alloc(L0 * 4 + 4, st);
    LAUNCH(k_root_keys, L0, d->body.as<u32>(), sincl.as<u32>(), L0, nw, base, SBF, headless,
           rkey.as<u64>(), isr.as<uint8_t>(), wkey.as<u64>(), isw.as<uint8_t>(), segof.as<u32>());
    auto occ_list = [&](DBuf& key, DBuf& is, int idbits, DBuf& oid, DBuf& oseg, DBuf& ocnt, u64* nout) {
      DBuf sidx2(L0 * 4 + 4, st), k2(L0 * 8 + 8, st), k3(L0 * 8 + 8, st), h2(L0 + 1, st), hi2(L0 * 4 + 4, st);
      select_flagged_index(is.as<uint8_t>(), sidx2.as<u32>(), cnt.as<u64>(), L0, st);
      u64 m;
      d2h(&m, cnt.p, 1, st);
      LAUNCH(k_gather_u64, m, sidx2.as<u32>(), m, key.as<u64>(), k2.as<u64>());
      sort_keys_u64(k2.as<u64>(), k3.as<u64>(), m, idbits + SBF, st);
      LAUNCH(k_heads, m, k3.as<u64>(), m, h2.as<uint8_t>());
      select_flagged_index(h2.as<uint8_t>(), hi2.as<u32>(), cnt.as<u64>(), m, st);
      u64 u;
      d2h(&u, cnt.p, 1, st);
      oid.alloc(u * 4 + 4, st);
      oseg.alloc(u * 4 + 4, st);
      ocnt.alloc(u * 4 + 4, st);
      LAUNCH(k_rle_keys, u, k3.as<u64>(), hi2.as<u32>(), u, m, SBF, oid.as<u32>(), oseg.as<u32>(),
             ocnt.as<u32>());
      *nout = u;
    };
    occ_list(rkey, isr, std::max(1, bitlen(R - 1)), d->rs_rule, d->rs_seg, d->rs_cnt, &d->n_rs);
    occ_list(wkey, isw, std::max(1, bitlen(nw ? nw - 1 : 0)), d->rw_word, d->rw_seg, d->rw_cnt, &d->n_rw);
    d->rs_off.alloc((R + 1) * 8, st);
    LAUNCH(k_csr_offsets, R + 1, d->rs_rule.as<u32>(), d->n_rs, R, d->rs_off.as<u64>());
      GT_CUDA(cudaStreamSynchronize(st));
    } catch (const Error& e) {
      root_err = e;
    } catch (const std::bad_alloc&) {
      root_err = Error{GT_E_RESOURCE, "out of host memory"};
    }
  };
  std::thread root_thread(root_side);
  bool root_joined = false;
  auto join_root = [&]() {
    if (root_joined) return;
    root_thread.join();
    root_joined = true;
    cudaEventDestroy(ev_body);
    rebind_stream(st, {&d->seg_lo, &d->seg_hi, &d->root_seg, &d->rs_rule, &d->rs_seg, &d->rs_cnt, &d->rs_off,
                       &d->rw_word, &d->rw_seg, &d->rw_cnt});
    cudaStreamDestroy(s_root);
    if (root_err.code != GT_OK) throw root_err;
  };
  struct JoinGuard {
    std::function<void()> f;
    ~JoinGuard() {
      try {
        f();
      } catch (...) {
      }
    }
  } join_guard{[&] {
    if (!root_joined) {  // error path of the main pipeline
      root_thread.join();
      root_joined = true;
      cudaStreamSynchronize(s_root);
      cudaEventDestroy(ev_body);
      rebind_stream(st, {&d->seg_lo, &d->seg_hi, &d->root_seg, &d->rs_rule, &d->rs_seg, &d->rs_cnt,
                         &d->rs_off, &d->rw_word, &d->rw_seg, &d->rw_cnt});
      cudaStreamDestroy(s_root);
    }
  }};


  // ---- (rule, symbol) sort + RLE -> own / sub CSR ----------------------
  // bodies are contiguous per rule, so the (rule, symbol) order is a
  // segmented sort of the body by symbol (one pass for the short bodies);
  // a 64-bit global radix sort of (rule << SB | symbol) beyond 2^31 symbols
  const int SB = std::max(1, bitlen(limit - 1));
  DBuf head(E + 1, st), hidx(E * 4 + 4, st), cnt(16, st);
  DBuf sbody, skeys;
  // (measured: the global sort wins on C2-sized grammars, the segmented one from ~10^7 symbols)
  const bool segmented = E >= (8ull << 20) && E < (1ull << 31) && R < (1ull << 31);
  if (segmented) {
    sbody.alloc(E * 4 + 4, st);
    sort_segments_u32(d->body.as<u32>(), sbody.as<u32>(), E, R, d->boff.as<u64>(), st);
    LAUNCH(k_heads_seg, E, sbody.as<u32>(), owner.as<u32>(), E, head.as<uint8_t>());
  } else {
    const int KB = SB + std::max(1, bitlen(R - 1));
    DBuf keys(E * 8 + 8, st);
    skeys.alloc(E * 8 + 8, st);
    LAUNCH(k_make_keys, E, d->body.as<u32>(), owner.as<u32>(), E, SB, keys.as<u64>());
    sort_keys_u64(keys.as<u64>(), skeys.as<u64>(), E, KB, st);
    LAUNCH(k_heads, E, skeys.as<u64>(), E, head.as<uint8_t>());
  }
  // runs of equal (rule, symbol), sized by the worst case E so the only host
  // round trip of this phase is the one for the own / sub pair counts
  DBuf cnt3(32, st);
  select_flagged_index(head.as<uint8_t>(), hidx.as<u32>(), cnt3.as<u64>(), E, st);
  DBuf pr_rule(E * 4 + 4, st), pr_sym(E * 4 + 4, st), pr_cnt(E * 4 + 4, st);
  DBuf is_own(E + 1, st), is_sub(E + 1, st);
  GT_CUDA(cudaMemsetAsync(is_own.p, 0, E + 1, st));
  GT_CUDA(cudaMemsetAsync(is_sub.p, 0, E + 1, st));
  if (segmented)
    LAUNCH(k_rle_seg, E, sbody.as<u32>(), owner.as<u32>(), hidx.as<u32>(), cnt3.as<u64>(), E, nw, base,
           pr_rule.as<u32>(), pr_sym.as<u32>(), pr_cnt.as<u32>(), is_own.as<uint8_t>(), is_sub.as<uint8_t>());
  else
    LAUNCH(k_rle, E, skeys.as<u64>(), hidx.as<u32>(), cnt3.as<u64>(), E, SB, nw, base, pr_rule.as<u32>(),
           pr_sym.as<u32>(), pr_cnt.as<u32>(), is_own.as<uint8_t>(), is_sub.as<uint8_t>());
  sbody.release();
  skeys.release();
  head.release();
  DBuf selO(E * 4 + 4, st), selS(E * 4 + 4, st);
  select_flagged_index(is_own.as<uint8_t>(), selO.as<u32>(), cnt3.as<u64>() + 1, E, st);
  select_flagged_index(is_sub.as<uint8_t>(), selS.as<u32>(), cnt3.as<u64>() + 2, E, st);
  {
    u64 h[2];
    d2h(h, cnt3.as<u64>() + 1, 2, st);
    d->E_own = h[0];
    d->E_sub = h[1];
  }
  const u64 Eo = d->E_own, Es = d->E_sub;
  DBuf own_rule(Eo * 4 + 4, st);
  d->own_ids.alloc(Eo * 4 + 4, st);
  d->own_freqs.alloc(Eo * 4 + 4, st);
  LAUNCH(k_gather3, Eo, selO.as<u32>(), Eo, pr_rule.as<u32>(), pr_sym.as<u32>(), pr_cnt.as<u32>(),
         own_rule.as<u32>(), d->own_ids.as<u32>(), d->own_freqs.as<u32>());
  DBuf sub_rule(Es * 4 + 4, st);
  d->sub_ids.alloc(Es * 4 + 4, st);
  d->sub_freqs.alloc(Es * 4 + 4, st);
  LAUNCH(k_gather3, Es, selS.as<u32>(), Es, pr_rule.as<u32>(), pr_sym.as<u32>(), pr_cnt.as<u32>(),
         sub_rule.as<u32>(), d->sub_ids.as<u32>(), d->sub_freqs.as<u32>());
  selO.release();
  selS.release();
  pr_rule.release();
  pr_sym.release();
  pr_cnt.release();
  is_own.release();
  is_sub.release();
  hidx.release();
  d->own_off.alloc((R + 1) * 8, st);
  d->sub_off.alloc((R + 1) * 8, st);
  LAUNCH(k_csr_offsets, R + 1, own_rule.as<u32>(), Eo, R, d->own_off.as<u64>());
  LAUNCH(k_csr_offsets, R + 1, sub_rule.as<u32>(), Es, R, d->sub_off.as<u64>());
  ph.mark("own/sub CSR");

  // ---- word-major transpose of the own pairs (no host sync: side stream) ----
  cudaStream_t s_own = nullptr;
  GT_CUDA(cudaStreamCreateWithFlags(&s_own, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s, main;
    DeviceDag* d;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      rebind_stream(main, {&d->ow_word, &d->ow_rule, &d->ow_freq, &d->ow_off});
      cudaStreamDestroy(s);
    }
  } own_guard{s_own, st, d};
  {
    cudaEvent_t ev;
    GT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    GT_CUDA(cudaEventRecord(ev, st));
    GT_CUDA(cudaStreamWaitEvent(s_own, ev, 0));
    cudaEventDestroy(ev);
  }
    {
    cudaStream_t st = s_own;
    DBuf id2(Eo * 4 + 4, st), sid(Eo * 4 + 4, st);
    d->ow_word.alloc(Eo * 4 + 4, st);
    d->ow_rule.alloc(Eo * 4 + 4, st);
    d->ow_freq.alloc(Eo * 4 + 4, st);
    d->ow_off.alloc((nw + 1) * 8, st);
    LAUNCH(k_iota_u32, Eo, id2.as<u32>(), Eo);
    sort_pairs_u32_u32(d->own_ids.as<u32>(), d->ow_word.as<u32>(), id2.as<u32>(), sid.as<u32>(), Eo,
                       std::max(1, bitlen(nw ? nw - 1 : 0)), st);
    LAUNCH(k_gather3, Eo, sid.as<u32>(), Eo, own_rule.as<u32>(), d->own_freqs.as<u32>(),
           (const u32*)nullptr, d->ow_rule.as<u32>(), d->ow_freq.as<u32>(), (u32*)nullptr);
    LAUNCH(k_csr_offsets, nw + 1, d->ow_word.as<u32>(), Eo, nw, d->ow_off.as<u64>());
  }

  // ---- parents: stable sort of sub pairs by child -------------------------
  DBuf idx(Es * 4 + 4, st), sidx(Es * 4 + 4, st), child_sorted(Es * 4 + 4, st);
  LAUNCH(k_iota_u32, Es, idx.as<u32>(), Es);
  sort_pairs_u32_u32(d->sub_ids.as<u32>(), child_sorted.as<u32>(), idx.as<u32>(), sidx.as<u32>(), Es,
                     std::max(1, bitlen(R - 1)), st);
  d->par_ids.alloc(Es * 4 + 4, st);
  d->par_freqs.alloc(Es * 4 + 4, st);
  d->par_off.alloc((R + 1) * 8, st);
  LAUNCH(k_gather3, Es, sidx.as<u32>(), Es, sub_rule.as<u32>(), d->sub_freqs.as<u32>(),
         (const u32*)nullptr, d->par_ids.as<u32>(), d->par_freqs.as<u32>(), (u32*)nullptr);
  LAUNCH(k_csr_offsets, R + 1, child_sorted.as<u32>(), Es, R, d->par_off.as<u64>());
  idx.release();
  sidx.release();
  ph.mark("parent CSR");

  // ---- per-rule sums -------------------------------------------------------
  d->own_tok.alloc(R * 8, st);
  d->num_out.alloc(R * 8, st);
  d->num_in.alloc(R * 8, st);
  GT_CUDA(cudaMemsetAsync(d->own_tok.p, 0, R * 8, st));
  GT_CUDA(cudaMemsetAsync(d->num_out.p, 0, R * 8, st));
  GT_CUDA(cudaMemsetAsync(d->num_in.p, 0, R * 8, st));
  LAUNCH(k_seg_sum_sorted, Eo, own_rule.as<u32>(), Eo, ValU32{d->own_freqs.as<u32>()}, d->own_tok.as<u64>());
  LAUNCH(k_seg_sum_sorted, Es, sub_rule.as<u32>(), Es, ValU32{d->sub_freqs.as<u32>()}, d->num_out.as<u64>());
  LAUNCH(k_seg_sum_sorted, Es, child_sorted.as<u32>(), Es,
         (ValU32NonRoot{d->par_freqs.as<u32>(), d->par_ids.as<u32>()}), d->num_in.as<u64>());

  // ---- bottom-up layering (cycle check) then top-down layering -----------
  DBuf rem_bu(R * 4, st), rem_td(R * 4, st), rootp(R, st), flag(R, st);
  DBuf fr(R * 4 + 4, st), nx(R * 4 + 4, st), fcnt(16, st);
  d->bu_level.alloc(R * 4, st);
  d->td_level.alloc(R * 4, st);
  GT_CUDA(cudaMemsetAsync(d->bu_level.p, 0, R * 4, st));
  GT_CUDA(cudaMemsetAsync(d->td_level.p, 0, R * 4, st));
  LAUNCH(k_degrees, R, d->sub_off.as<u64>(), d->par_off.as<u64>(), d->par_ids.as<u32>(), R,
         rem_bu.as<u32>(), rem_td.as<u32>(), rootp.as<uint8_t>());
  // persistent Kahn layering, bottom-up (doubles as the cycle check), then
  // top-down (carries reachability): one cooperative launch each
  const u64 ntask_max = Es / kChunk + R + 1;
  DBuf tasks(ntask_max * 8, st), ctl_b(sizeof(KahnCtl), st);
  KahnCtl* ctl = ctl_b.as<KahnCtl>();
  DBuf reach(R, st), firstu(4, st);
  GT_CUDA(cudaMemsetAsync(reach.p, 0, R, st));
  auto kahn = [&](bool td, DBuf& rem, const DBuf& off, const DBuf& ids, DBuf& lvl) {
    GT_CUDA(cudaMemsetAsync(ctl, 0, sizeof(KahnCtl), st));
    LAUNCH(k_flag_zero, R, rem.as<u32>(), R, td ? 1 : 0, flag.as<uint8_t>());
    // first frontier -> q1 (layer 1 reads q1), its count -> cnt[1]
    select_flagged_index(flag.as<uint8_t>(), nx.as<u32>(), &ctl->cnt[1], R, st);
    const void* kern = td ? (const void*)k_kahn<true> : (const void*)k_kahn<false>;
    static int per_sm[2] = {-1, -1};
    int& ps = per_sm[td ? 1 : 0];
    if (ps < 0) {
      GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, kKahnBlock, 0));
      ps = std::max(ps, 1);
    }
    int nsm = 148;
    GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    u32* q0 = fr.as<u32>();
    u32* q1 = nx.as<u32>();
    const u64* po = d->par_off.as<u64>();
    const u32* pi = d->par_ids.as<u32>();
    const uint8_t* rp = rootp.as<uint8_t>();
    uint8_t* rc = reach.as<uint8_t>();
    uint2* tk = tasks.as<uint2>();
    const u64* o = off.as<u64>();
    const u32* ii = ids.as<u32>();
    u32* rm = rem.as<u32>();
    u32* lv = lvl.as<u32>();
    u64 maxl = R + 2;
    void* args[] = {(void*)&ctl, (void*)&q0, (void*)&q1, (void*)&o, (void*)&ii, (void*)&rm, (void*)&lv,
                    (void*)&po, (void*)&pi, (void*)&rp, (void*)&rc, (void*)&tk, (void*)&maxl};
    {
      ProfScope ps_(td ? "k_kahn<td>" : "k_kahn<bu>", st);
      GT_CUDA(cudaLaunchCooperativeKernel(kern, dim3((unsigned)(nsm * ps)), dim3(kKahnBlock), args, 0, st));
      g_launches++;
    }
  };
  // top-down Kahn layering: the frontier never reaches a rule on (or below)
  // a reference cycle, so an incomplete layering is the cycle check
  // (grammar.py:127-161 order: cycles before unreachable rules, dag.py:173-184)
  u64 processed = 0;
  kahn(true, rem_td, d->sub_off, d->sub_ids, d->td_level);
  // every rule but the root must be layered, and no reachable rule (nor the
  // root itself) may reference the root: either way there is a cycle; then
  // the first unreachable rule.  One host round trip for all three checks.
  KahnCtl h;
  u32 chk[2];
  {
    DBuf cd(8, st);
    GT_CUDA(cudaMemsetAsync(cd.p, 0, 4, st));
    GT_CUDA(cudaMemsetAsync(cd.as<u32>() + 1, 0xFF, 4, st));
    LAUNCH(k_root_cycle, 1, d->par_off.as<u64>(), d->par_ids.as<u32>(), reach.as<uint8_t>(), cd.as<u32>());
    LAUNCH(k_first_unreached, R, reach.as<uint8_t>(), R, cd.as<u32>() + 1);
    GT_CUDA(cudaMemcpyAsync(&h, ctl, sizeof h, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaMemcpyAsync(chk, cd.p, 8, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaStreamSynchronize(st));
  }
  processed = h.processed;
  const int ntd = (int)h.layers;
  if (processed + 1 < R || chk[0]) {
    need_host_chain();
    cycle_message(blob, P);
  }
  if (chk[1] != 0xFFFFFFFFu) fail(GT_E_CORRUPTION, "rule %u is not reachable from the root", chk[1]);
  ph.mark("top-down layering");
  rem_bu.release();
  rem_td.release();
  fr.release();
  nx.release();

  // ---- level-ordered edge lists (radix sort is stable: within a level the
  // edges keep (child, parent) resp. (rule, child) order) -------------------
  // host values read back once at the end of gt_open (one pinned staging
  // buffer: te and be level offsets, root height, W)
  static thread_local PinnedU64 stage_host;
  u64* stage = stage_host.get(2 * ((u64)ntd + 3) + 2);
  auto level_edges = [&](const u32* group_of, const uint8_t* keep, const u32* lvl, int nl,
                         const u32* a_src, const u32* b_src, const u32* f_src, DBuf& oa, DBuf& ob,
                         DBuf& of, u64* off_stage, DBuf& off_dev) {
    // every edge is sorted (dropped ones under key nl + 1, after all levels),
    // so no count has to come back to the host first
    DBuf idx(Es * 4 + 4, st), key(Es * 4 + 4, st), key2(Es * 4 + 4, st), idx2(Es * 4 + 4, st);
    LAUNCH(k_iota_u32, Es, idx.as<u32>(), Es);
    LAUNCH(k_edge_level_keys2, Es, group_of, keep, lvl, (u32)nl + 1, Es, key.as<u32>());
    sort_pairs_u32_u32(key.as<u32>(), key2.as<u32>(), idx.as<u32>(), idx2.as<u32>(), Es,
                       std::max(1, bitlen((u64)nl + 1)), st);
    oa.alloc(Es * 4 + 16, st);  // + 16: the TMA-staged level loop copies whole 16-byte words
    ob.alloc(Es * 4 + 16, st);
    of.alloc(Es * 4 + 16, st);
    LAUNCH(k_gather3, Es, idx2.as<u32>(), Es, a_src, b_src, f_src, oa.as<u32>(), ob.as<u32>(), of.as<u32>());
    DBuf koff(((u64)nl + 3) * 8, st);
    LAUNCH(k_csr_offsets, (u64)nl + 3, key2.as<u32>(), Es, (u64)nl + 2, koff.as<u64>());
    GT_CUDA(cudaMemcpyAsync(off_stage, koff.p, ((u64)nl + 3) * 8, cudaMemcpyDeviceToHost, st));
    off_dev = std::move(koff);
  };
  {
    // td: par entries (grouped by child) whose parent is not the root
    DBuf keep(Es + 1, st);
    LAUNCH(k_flag_nonzero_u32, Es, d->par_ids.as<u32>(), Es, keep.as<uint8_t>());
    level_edges(child_sorted.as<u32>(), keep.as<uint8_t>(), d->td_level.as<u32>(), ntd,
                child_sorted.as<u32>(), d->par_ids.as<u32>(), d->par_freqs.as<u32>(), d->te_child,
                d->te_par, d->te_freq, stage, d->te_off_dev);
    // be: sub entries (grouped by rule) by the rule's TOP-DOWN level; walked
    // in decreasing level order every child is finished before its parents
    // (a child's td level exceeds each parent's), which is all the bottom-up
    // sums need.  The root (td level 0) comes last.
    level_edges(sub_rule.as<u32>(), nullptr, d->td_level.as<u32>(), ntd, sub_rule.as<u32>(),
                d->sub_ids.as<u32>(), d->sub_freqs.as<u32>(), d->be_rule, d->be_child, d->be_freq,
                stage + (ntd + 3), d->be_off_dev);
  }
  sub_rule.release();
  child_sorted.release();
  // bottom-up levels = heights (leaf = 1; the reference's bottom-up rounds,
  // engine.py:313-335), one persistent max pass in decreasing td level order
  // heights (bottom-up levels) and exp_len in one persistent reverse pass
  int nbu = 0;
  d->exp_len.alloc(R * 8, st);
  {
    DBuf hgt(R * 8, st);
    LAUNCH(k_fill_u64, R, hgt.as<u64>(), R, 1ull);
    GT_CUDA(cudaMemcpyAsync(d->exp_len.p, d->own_tok.p, R * 8, cudaMemcpyDeviceToDevice, st));
    {
      static int per_sm = -1;
      if (per_sm < 0) {
        GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bu_pair, 1024, 0));
        per_sm = std::max(per_sm, 1);
      }
      int nsm = 148;
      GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
      const u32* br = d->be_rule.as<u32>();
      const u32* bc = d->be_child.as<u32>();
      const u32* bf = d->be_freq.as<u32>();
      const u64* bo = d->be_off_dev.as<u64>();
      int L1 = ntd;
      u64* hg = hgt.as<u64>();
      u64* el = d->exp_len.as<u64>();
      void* args[] = {(void*)&br, (void*)&bc, (void*)&bf, (void*)&bo, (void*)&L1, (void*)&hg, (void*)&el};
      ProfScope ps_("k_bu_pair", st);
      GT_CUDA(cudaLaunchCooperativeKernel((const void*)k_bu_pair, dim3((unsigned)(nsm * per_sm)), dim3(1024), args,
                                          0, st));
      g_launches++;
    }
    LAUNCH(k_u64_to_u32, R, hgt.as<u64>(), R, d->bu_level.as<u32>());
    // height of the root (the highest rule) and W, read back at the end
    u64* hw = stage + 2 * ((u64)ntd + 3);
    GT_CUDA(cudaMemcpyAsync(&hw[0], hgt.p, 8, cudaMemcpyDeviceToHost, st));
    GT_CUDA(cudaMemcpyAsync(&hw[1], d->exp_len.p, 8, cudaMemcpyDeviceToHost, st));
  }
  // level counts (bu.nl set from the root height at the end); the bottom-up
  // rule lists (sequence tasks' head/tail pass) are built on first use
  // (ensure_bu_levels), the top-down pass runs over the te edge lists
  d->td.nl = ntd;
  // the reference's bottom-up rounds exclude the root (engine.py:305-310)
  GT_CUDA(cudaMemsetAsync(d->bu_level.p, 0, 4, st));
  ph.mark("level lists");

  // ---- exp_len by bottom-up level (grammar.py:109-124) --------------------
  // (exp_len computed with the heights above)
  ph.mark("segments+exp_len");

  // ---- join the root side; segment tokens need exp_len ----------------------
  join_root();
  {
    DBuf& segof = d->root_seg;
    d->seg_tokens.alloc(d->F * 8, st);
    GT_CUDA(cudaMemsetAsync(d->seg_tokens.p, 0, d->F * 8, st));
    LAUNCH(k_seg_sum_sorted, d->L0, segof.as<u32>(), d->L0,
           (ValRootLen{d->body.as<u32>(), d->exp_len.as<u64>(), nw, base}), d->seg_tokens.as<u64>());
  }
  ph.mark("root side joined");

  GT_CUDA(cudaStreamSynchronize(st));
  GT_CUDA(cudaStreamSynchronize(s_own));
  own_rule.release();
  {
    d->te_off.assign(stage, stage + ntd + 3);
    d->be_off.assign(stage + ntd + 3, stage + 2 * (ntd + 3));
    const u64* hw = stage + 2 * ((u64)ntd + 3);
    nbu = (int)hw[0];
    d->depth = (i64)hw[0] - 1;
    d->W = hw[1];
    d->bu.nl = nbu;
  }
  ph.mark("finish");
  d->init_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace gt
