// loader.cu — GTDC -> device DAG (CSR arrays) + topological level scheduler.
//
// Replaces deserialize_grammar (grammar.py:193-228), build_dag
// (dag.py:131-230) and the round discovery the reference's engine performs
// every traversal (engine.py:196-227 top-down mask rounds, engine.py:313-335
// bottom-up readiness rounds).  The host validates the header and the
// dictionary while the blob uploads; everything proportional to E runs on
// the device:
//   rule-chain parse (chunk tables + doubling over chunk states; word-level
//   doubling / host walk only as fallbacks) -> unpack (body, owner)
//   -> own/sub CSR (csr_build.cu: per-rule register sorts, the root sorted
//      in place) -> parent CSR and the word-major own transpose (payload
//      radix sorts; side stream) -> per-rule sums
//   -> top-down layering (persistent Kahn over non-root in-edges with a
//      bitmap frontier; = reference top-down rounds; carries reachability;
//      an incomplete layering is the cycle check)
//   -> tid numbering + top-down edge lists, bottom-up edge lists (side
//      stream) -> heights (= reference bottom-up rounds) and exp_len in one
//      reverse pass -> root segments, segment tokens, root occurrence lists
//      (helper thread + stream).
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

static bool trace2() {
  static const bool v = getenv("GT_TRACE") && atoi(getenv("GT_TRACE")) == 2;
  return v;
}

void DBuf::alloc(size_t n, cudaStream_t st) {
  release();
  s = st;
  bytes = n;
  if (!n) return;
  if (!trace2()) {
    GT_CUDA(cudaMallocAsync(&p, n, st));
    return;
  }
  auto a = std::chrono::steady_clock::now();
  GT_CUDA(cudaMallocAsync(&p, n, st));
  sync_stats().alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  sync_stats().nalloc++;
}

void DBuf::release() {
  if (p && !own) {
    p = nullptr;
    bytes = 0;
    own = true;
    return;
  }
  if (p) {
    if (!trace2()) {
      cudaFreeAsync(p, s);
    } else {
      auto a = std::chrono::steady_clock::now();
      cudaFreeAsync(p, s);
      sync_stats().alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
      sync_stats().nfree++;
    }
  }
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

// CSR row offsets of a sorted key list in one coalesced pass: element i
// writes the offsets of the rows (key[i-1], key[i]] (O(n + R), for keys
// dense in [0, R): a gap is filled by one thread; sparse keys use the
// per-row binary search above)
__global__ void k_csr_offsets_lin(const u32* __restrict__ key, u64 n, u64 R, u64* off) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += stride) {
    const u64 lo = i == 0 ? 0 : (u64)key[i - 1] + 1;
    const u64 hi = i == n ? R : (u64)key[i];
    for (u64 r = lo; r <= hi; r++) off[r] = i;
  }
}

__global__ void k_pack2(const u32* __restrict__ a, const u32* __restrict__ b, u64 n, u64* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = ((u64)a[i] << 32) | b[i];
}

__global__ void k_unpack2(const u64* __restrict__ in, u64 n, u32* a, u32* b) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 v = in[i];
    a[i] = (u32)(v >> 32);
    b[i] = (u32)v;
  }
}

__global__ void k_pack3(const u32* __restrict__ a, const u32* __restrict__ b, const u32* __restrict__ c, u64 n,
                        U3* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = U3{a[i], b[i], c[i]};
}

// (map[a], map[b], c) triples (map = the tid numbering; nullptr: identity)
__global__ void k_pack3_map(const u32* __restrict__ a, const u32* __restrict__ b, const u32* __restrict__ c, u64 n,
                            const u32* __restrict__ map, U3* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = U3{map[a[i]], map[b[i]], c[i]};
}

__global__ void k_map_u32(const u32* __restrict__ in, u64 n, const u32* __restrict__ map, u32* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = map[in[i]];
}

__global__ void k_rank_of(const u32* __restrict__ order, u64 n, u32* rank) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) rank[order[i]] = (u32)i;
}

__global__ void k_unpack3(const U3* __restrict__ in, u64 n, u32* a, u32* b, u32* c) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const U3 v = in[i];
    a[i] = v.a;
    b[i] = v.b;
    c[i] = v.c;
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

// ---- rule-chain parse, chunked form (the common case) ----------------------
// After the root record the section is cut into chunks of kChunkB words.
// If every non-root record is shorter than kWin words, the chain enters
// chunk c at one of its first kWin words, so each chunk is summarised by a
// kWin-entry table: entry offset -> (entry offset into chunk c+1, records
// started in c) — one warp per chunk, one lane per candidate entry, walking
// the chunk through L1.  The chunk tables are then composed by groups of 32
// (k_chain_up / k_chain_top / k_chain_down below) instead of pointer
// doubling over every word of the section (log2(R) passes over n words), and
// a final walk per chunk writes the rule starts.  A table entry that would need a wider
// window is INVALID; if the true chain meets one (a record of >= kWin words
// other than the root) or the section is malformed, the word-level doubling
// above runs instead, and after it the host walk for the exact error.
constexpr u32 kChunkB = 1024, kWin = 32, kStInvalid = 0xFFFFFFFFu;
constexpr u32 kMaskW = kChunkB / 32;  // 32-bit words of one candidate's start mask

// one warp per chunk: lane o walks the chain from entry offset o, records its
// exit state and record count, and marks the record starts it visits in a
// 1024-bit mask (shared memory, then stored so that the final pass only reads
// the mask of the true entry)
constexpr int kTabWarps = 8;
__global__ void __launch_bounds__(kTabWarps * 32) k_chunk_tables(const u32* __restrict__ raw, u64 n, u64 p1,
                                                                  u64 nch, u64 c0, u64 c1, u32* nxt, u32* cnt,
                                                                  u32* mask) {
  __shared__ u32 sm[kTabWarps][kWin][kMaskW + 1];
  const u32 wib = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const u64 warp = (u64)blockIdx.x * kTabWarps + wib;
  const u64 nwarps = (u64)gridDim.x * kTabWarps;
  const u32 END = (u32)(nch * kWin);
  u32(*m)[kMaskW + 1] = sm[wib];
  for (u64 c = c0 + warp; c < c1; c += nwarps) {
    for (u32 w = 0; w < kMaskW; w++) m[lane][w] = 0;
    const u64 cs = p1 + c * kChunkB, ce = cs + kChunkB < n ? cs + kChunkB : n;
    u64 p = cs + lane;
    u32 k = 0, state;
    if (p >= ce) {
      state = kStInvalid;  // an entry past the end of a short last chunk
    } else {
      while (p < ce) {
        const u32 o = (u32)(p - cs);
        m[lane][o >> 5] |= 1u << (o & 31u);
        k++;
        p += 1 + (u64)raw[p];
      }
      if (p >= n) state = p == n ? END : kStInvalid;
      else state = p - ce < kWin ? (u32)((c + 1) * kWin + (p - ce)) : kStInvalid;
    }
    nxt[c * kWin + lane] = state;
    cnt[c * kWin + lane] = k;
    __syncwarp();
    u32* mg = mask + c * (u64)(kWin * kMaskW);
    for (u32 r = 0; r < kWin; r++) mg[r * kMaskW + lane] = m[r][lane];  // row r = candidate r, coalesced
    __syncwarp();
  }
  if (warp == 0 && lane == 0 && c1 == nch) {
    nxt[END] = END;
    cnt[END] = 0;
  }
}

// ---- chunk-chain composition by groups of 32 (replaces the doubling) -----
// Level k has n_k "chunks", each a 32-entry table (state c*32 + o: entry
// offset o into chunk c; END = n_k*32).  One warp per group of 32 chunks
// stages the group's tables in shared memory and walks them from each of the
// 32 entries of its first chunk (lane o), recording the entry state and the
// records before each chunk of the path (path tables, for the way down) and
// the group's exit as a level-(k+1) state.  ceil(log32(chunks)) levels up,
// one warp-walk at the top, one expansion per level down: C2 2 levels (3.3k
// chunks), C5 4 (70k), instead of log2(chunks) grid-synchronised doubling
// passes over every state.
constexpr int kChainWarps = 4;
__global__ void __launch_bounds__(kChainWarps * 32) k_chain_up(const u32* __restrict__ nx, const u32* __restrict__ ct,
                                                              u64 nck, u32* nx_up, u32* ct_up, u32* path_s,
                                                              u32* path_c) {
  __shared__ u32 snx[kChainWarps][32][33], sct[kChainWarps][32][33];
  const u32 wib = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  const u64 ng = (nck + 31) / 32;
  const u64 g = (u64)blockIdx.x * kChainWarps + wib;
  if (g >= ng) return;
  const u64 c0 = g * 32, nc = nck - c0 < 32 ? nck - c0 : 32;
  const u32 END = (u32)(nck * 32), END_UP = (u32)(ng * 32);
#pragma unroll 4
  for (u32 j = 0; j < (u32)nc; j++) {  // coalesced: chunk j's 32 entries
    snx[wib][j][lane] = nx[(c0 + j) * 32 + lane];
    sct[wib][j][lane] = ct[(c0 + j) * 32 + lane];
  }
  __syncwarp();
  u32 s = (u32)(c0 * 32 + lane), cum = 0;
  u32* ps = path_s + (g * 32 + lane) * 32;
  u32* pc = path_c + (g * 32 + lane) * 32;
  for (u32 j = 0; j < (u32)nc; j++) {
    ps[j] = s;
    pc[j] = cum;
    if (s == END || s == kStInvalid) continue;
    if (s / 32 != c0 + j) {  // (cannot happen on a well-formed table)
      s = kStInvalid;
      continue;
    }
    const u32 x = s & 31u;
    cum += sct[wib][j][x];
    s = snx[wib][j][x];
  }
  u32 up;
  if (s == END) up = END_UP;
  else if (s == kStInvalid || s / 32 != c0 + 32 || (s / 32) % 32 != 0) up = kStInvalid;
  else up = (u32)((g + 1) * 32 + (s & 31u));
  nx_up[g * 32 + lane] = up;
  ct_up[g * 32 + lane] = cum;
}

// the top level (<= 32 chunks): one warp stages the tables, lane 0 walks the
// chain from state 0; the walk must end at END having started R - 1 records
__global__ void k_chain_top(const u32* __restrict__ nx, const u32* __restrict__ ct, u64 nck, u64 R, u32* entry,
                            u32* base, u32* bad) {
  __shared__ u32 snx[32][33], sct[32][33];
  const u32 lane = threadIdx.x & 31u;
  for (u32 j = 0; j < (u32)nck; j++) {
    snx[j][lane] = nx[j * 32 + lane];
    sct[j][lane] = ct[j * 32 + lane];
  }
  __syncwarp();
  if (lane) return;
  const u32 END = (u32)(nck * 32);
  u32 s = 0;
  u64 cum = 0;
  for (u32 j = 0; j < (u32)nck; j++) {
    entry[j] = s;
    base[j] = (u32)cum;
    if (s == END) continue;
    if (s == kStInvalid || s / 32 != j) {
      *bad = 1;
      return;
    }
    cum += sct[j][s & 31u];
    s = snx[j][s & 31u];
  }
  if (s != END || cum != R - 1) *bad = 1;
}

// one level down: chunk c of level k enters at the path state of its group's
// true entry (thread per chunk)
__global__ void k_chain_down(const u32* __restrict__ path_s, const u32* __restrict__ path_c,
                             const u32* __restrict__ entry_up, const u32* __restrict__ base_up, u64 nck, u32* entry,
                             u32* base, u32* bad) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 ng = (nck + 31) / 32;
  const u32 END = (u32)(nck * 32), END_UP = (u32)(ng * 32);
  for (u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x; c < nck; c += stride) {
    const u64 g = c / 32, j = c % 32;
    const u32 e = entry_up[g];
    if (e == END_UP) {
      entry[c] = END;
      base[c] = base_up[g];
      continue;
    }
    if (e == kStInvalid || e / 32 != g) {
      *bad = 1;
      entry[c] = END;
      continue;
    }
    const u64 k = (g * 32 + (e & 31u)) * 32 + j;
    const u32 st = path_s[k];
    if (st == kStInvalid || (st != END && st / 32 != c)) {
      *bad = 1;
      entry[c] = END;
      continue;
    }
    entry[c] = st;
    base[c] = base_up[g] + path_c[k];
  }
}

// rule starts from the true entry's mask: one warp per chunk, lane w expands
// mask word w at its popcount prefix.  Runs before the host sees the check:
// indices are bounded by R so that a failed parse only leaves rstart to be
// overwritten by the fallback.
__global__ void k_chunk_starts(u64 p1, u64 nch, u64 R, const u32* entry, const u32* base, const u32* mask,
                               u32* rstart) {
  const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const u32 lane = threadIdx.x & 31u;
  const u32 END = (u32)(nch * kWin);
  for (u64 c = warp; c < nch; c += nwarps) {
    const u32 st = entry[c];
    if (st == END) continue;
    u32 bits = mask[c * (u64)(kWin * kMaskW) + (u64)(st % kWin) * kMaskW + lane];
    const u32 pc = __popc(bits);
    u32 pre = pc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 o = __shfl_up_sync(0xFFFFFFFFu, pre, d);
      if (lane >= (u32)d) pre += o;
    }
    u64 i = 1 + (u64)base[c] + pre - pc;
    const u64 pos0 = p1 + c * kChunkB + lane * 32u;
    while (bits) {
      const u32 b = __ffs(bits) - 1;
      bits &= bits - 1;
      if (i < R) rstart[i] = (u32)(pos0 + b + 1);
      i++;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) rstart[0] = 1;
}

__global__ void k_boff(const u32* rstart, u64 R, u64 E, u64* boff) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= R; i += stride)
    boff[i] = i < R ? (u64)rstart[i] - (i + 1) : E;
}

// Rule bodies unpacked straight from the records (rstart[r] = first body
// word of rule r; the body runs to the next record's length word): a thread
// per rule of at most 32 symbols; longer bodies (the root) are queued for
// k_unpack_long, which spreads them over the grid.  Replaces a mark array
// over every raw word, its scan and a pass over every raw word.
constexpr u32 kUnpackShort = 32;
__global__ void k_unpack_rules(const u32* __restrict__ raw, const u32* __restrict__ rstart, u64 R, u64 nraw,
                               u32* body, u32* owner, u64 limit, u32* bad_rule, u32* longq, u32* nlong) {
  // a warp takes 32 consecutive rules and writes their (contiguous) bodies
  // together: output q of the warp goes to lane q % 32 (coalesced), its rule
  // found by a shuffle search over the lanes' body offsets
  const unsigned lane = threadIdx.x & 31u;
  const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 r0 = warp * 32; r0 < R; r0 += nwarps * 32) {
    const u64 r = r0 + lane;
    u32 len = 0, s = 0;
    if (r < R) {
      s = rstart[r];
      const u64 e = r + 1 < R ? (u64)rstart[r + 1] - 1 : nraw;
      // (a speculative chain parse that failed leaves rule starts that are
      // not a chain: nothing outside the section is touched, the run is redone)
      if (e < s || e > nraw || s < r + 1 || e - (r + 1) > nraw - R) atomicMin(bad_rule, (u32)r);
      else if (e - s > kUnpackShort) longq[atomicAdd(nlong, 1u)] = (u32)r;  // the long body: k_unpack_long
      else len = (u32)(e - s);
    }
    u32 x = len;  // inclusive prefix of the short lengths
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, d);
      if (lane >= (unsigned)d) x += y;
    }
    const u32 pre = x - len, tot = __shfl_sync(0xFFFFFFFFu, x, 31);
    for (u32 q0 = 0; q0 < tot; q0 += 32) {
      const u32 q = q0 + lane;
      int o = 0;  // the last lane whose short body starts at or before q
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const u32 pv = __shfl_sync(0xFFFFFFFFu, pre, (o + step) & 31);
        if (o + step < 32 && pv <= q) o += step;
      }
      const u32 so = __shfl_sync(0xFFFFFFFFu, s, o), po = __shfl_sync(0xFFFFFFFFu, pre, o);
      if (q < tot) {
        const u64 ro = r0 + (u64)o, p = (u64)so + (q - po);
        const u32 v = raw[p];
        body[p - (ro + 1)] = v;
        owner[p - (ro + 1)] = (u32)ro;
        if ((u64)v >= limit) atomicMin(bad_rule, (u32)ro);
      }
    }
  }
}

__global__ void k_unpack_long(const u32* __restrict__ raw, const u32* __restrict__ rstart, u64 R, u64 nraw,
                              const u32* __restrict__ longq, const u32* __restrict__ nlong, u32* body, u32* owner,
                              u64 limit, u32* bad_rule) {
  const u32 n = *nlong;
  // few long bodies (the root): each over the whole grid; many: a block each
  const bool spread = n <= 64;
  const u64 stride = spread ? (u64)gridDim.x * blockDim.x : blockDim.x;
  const u64 t0 = spread ? (u64)blockIdx.x * blockDim.x + threadIdx.x : threadIdx.x;
  for (u32 q = spread ? 0 : blockIdx.x; q < n; q += spread ? 1 : gridDim.x) {
    const u64 r = longq[q];
    const u64 s = rstart[r], e = r + 1 < R ? (u64)rstart[r + 1] - 1 : nraw, b = s - (r + 1);
    bool bad = false;
    for (u64 p = s + t0; p < e; p += stride) {
      const u32 v = raw[p];
      body[b + (p - s)] = v;
      owner[b + (p - s)] = (u32)r;
      bad |= (u64)v >= limit;
    }
    if (bad) atomicMin(bad_rule, (u32)r);
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
// Persistent top-down Kahn layering: ONE cooperative launch runs every layer,
// layers separated by grid barriers (no host round trip per layer).  The
// frontier of layer L is a BITMAP of rules (bit set by the edge that took a
// rule's counter of non-root parents to zero during layer L-1, with a
// fire-and-forget atomicOr): warps scan it 1024 rules per step and deal the
// set bits to lanes, so no frontier queue, no counter atomic with return on
// the append path.  Reachability from the root is pushed along the edges
// (reach[child] = 1 from a reached parent, a plain byte store) and is final
// when the child's counter reaches zero.  A rule with more than kLight
// children is split into chunk tasks of kChunk edges that every warp of the
// grid shares after a second barrier (a rule with 10^6 children is never
// one warp's serial loop).
// ---------------------------------------------------------------------------
constexpr u32 kLight = 8, kChunk = 256;

struct KahnCtl {
  u32 any[3];    // layer L is non-empty: any[L % 3] (set by the layer that fills it)
  u32 pad;
  u64 ntask[2];  // heavy-task counts, layer L uses ntask[L & 1]
  u64 processed;
  u64 layers;
  u64 t[64];     // %globaltimer at the start of layers 1..63 (GT_TRACE=2 prints them)
  u64 bar;       // k_kahn3's layer barrier: arrivals (bits 0-31), active blocks of even / odd layers (32-47 / 48-63)
  u32 root_cycle;       // k_kahn3's fused checks: a reachable rule (or the root) references the root
  u32 first_unreached;  // smallest rule >= 1 not reachable from the root (0xFFFFFFFF: none)
  u32 checked;          // the fused checks ran
};

__device__ __forceinline__ u64 globaltimer() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Sum of a per-thread count into *dst with ONE atomic per block (every
// thread of a full grid adding to one address serialises ~10^5 atomics in
// one L2 slice: ~65 us at 148 x 1024 threads).  Called by every thread.
__device__ __forceinline__ void block_add_u64(u64 v, u64* dst) {
  __shared__ unsigned long long s_sum;
#pragma unroll
  for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
  if (threadIdx.x == 0) s_sum = 0;
  __syncthreads();
  if ((threadIdx.x & 31u) == 0 && v) atomicAdd(&s_sum, (unsigned long long)v);
  __syncthreads();
  if (threadIdx.x == 0 && s_sum) atomicAdd((unsigned long long*)dst, s_sum);
}

__device__ __forceinline__ u64 ld_cg64(const u64* p) {
  return (u64)__ldcg(reinterpret_cast<const unsigned long long*>(p));
}

constexpr int kKahnBlock = 1024;  // few, large blocks: cheaper grid barriers

// first frontier: rules (not the root) without non-root parents
__global__ void k_kahn_first(const u32* rem, u64 R, u32* bm, KahnCtl* ctl) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = 1 + (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride)
    if (rem[r] == 0) {
      atomicOr(&bm[r >> 5], 1u << (r & 31u));
      ctl->any[1] = 1;
    }
}

// one edge of a frontier rule: push reachability, take the child's counter
// down (warp-aggregated) and put it into the next frontier at zero
__device__ __forceinline__ void kahn_edge(u32 c, bool act, bool reached, u32* rem, uint8_t* reach, u32* nxt,
                                          u32* any_next) {
  if (act && reached) reach[c] = 1;
  if (dec_to_zero(rem, c, act)) {
    atomicOr(&nxt[c >> 5], 1u << (c & 31u));
    *any_next = 1;
  }
}

__global__ void __launch_bounds__(kKahnBlock) k_kahn(KahnCtl* ctl, u32* bm0, u32* bm1, u64 nwords,
                                                     const u64* __restrict__ off, const u32* __restrict__ ids,
                                                     u32* rem, u32* lvl, uint8_t* reach, uint2* tasks,
                                                     u64 max_layers) {
  cg::grid_group grid = cg::this_grid();
  const u64 gtid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 nthreads = (u64)gridDim.x * blockDim.x;
  const u64 warp = gtid >> 5, nwarps = nthreads >> 5;
  const unsigned lane = threadIdx.x & 31u;
  const volatile uint8_t* rv = reach;
  // words per warp step: the smallest power of two that covers the bitmap in
  // one step per warp (a second step doubles a layer's dependent chain)
  u32 WS = 1;
  while (WS < 32 && (u64)WS * nwarps < nwords) WS *= 2;
  u64 found = 0, L = 1;
  for (;; L++) {
    if (__ldcg(&ctl->any[L % 3]) == 0 || L > max_layers) break;
    if (gtid == 0) {
      ctl->any[(L + 2) % 3] = 0;
      ctl->ntask[(L + 1) & 1] = 0;
    }
    u32* cur = (L & 1) ? bm1 : bm0;
    u32* nxt = (L & 1) ? bm0 : bm1;
    u32* any_next = &ctl->any[(L + 1) % 3];
    u64* ntask = &ctl->ntask[L & 1];
    // phase A: WS bitmap words (32 * WS rules) per warp step, WS <= 32 sized
    // so that a small grammar still spreads over every warp
    for (u64 w0 = warp * WS; w0 < nwords; w0 += nwarps * WS) {
      const u64 wi = w0 + lane;
      const u32 bits = lane < WS && wi < nwords ? __ldcg(cur + wi) : 0u;
      if (bits) cur[wi] = 0;  // cleared for layer L + 2
      const u32 pc = __popc(bits);
      u32 incl = pc;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= (unsigned)d) incl += t;
      }
      const u32 excl_b = incl - pc;
      const u32 T = __shfl_sync(0xFFFFFFFFu, incl, 31);
      for (u32 q0 = 0; q0 < T; q0 += 32) {
        // rule q0 + lane of the step: owning lane by a shuffle binary search,
        // then the matching set bit of that lane's word
        const u32 q = q0 + lane;
        int lo = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1) {
          const u32 se = __shfl_sync(0xFFFFFFFFu, excl_b, lo + step);
          if (se <= q) lo += step;
        }
        const u32 ow_bits = __shfl_sync(0xFFFFFFFFu, bits, lo);
        const u32 ow_ex = __shfl_sync(0xFFFFFFFFu, excl_b, lo);
        const bool active = q < T;
        u32 r = 0;
        u64 e0 = 0, len = 0;
        bool rc = false;
        if (active) {
          const u32 bp = __fns(ow_bits, 0, (int)(q - ow_ex) + 1);
          r = (u32)((w0 + (u64)lo) * 32 + bp);
          lvl[r] = (u32)L;
          found++;
          rc = rv[r] != 0;
          e0 = off[r];
          len = off[r + 1] - e0;
          if (len > kLight) {
            const u64 nch = (len + kChunk - 1) / kChunk;
            const u64 t0 = atomicAdd((unsigned long long*)ntask, (unsigned long long)nch);
            for (u64 k = 0; k < nch; k++) tasks[t0 + k] = make_uint2(r, (u32)(k * kChunk));
            len = 0;
          }
        }
        // the light edges of the step's rules dealt round-robin over the lanes
        u32 inc = (u32)len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const u32 t = __shfl_up_sync(0xFFFFFFFFu, inc, d);
          if (lane >= (unsigned)d) inc += t;
        }
        const u32 excl = inc - (u32)len;
        const u32 tot = __shfl_sync(0xFFFFFFFFu, inc, 31);
        for (u32 k0 = 0; k0 < tot; k0 += 32) {
          const u32 qe = k0 + lane;
          int le = 0;
#pragma unroll
          for (int step = 16; step; step >>= 1) {
            const u32 st_ex = __shfl_sync(0xFFFFFFFFu, excl, le + step);
            if (st_ex <= qe) le += step;
          }
          const u32 own_start = __shfl_sync(0xFFFFFFFFu, excl, le);
          const u64 own_e0 = __shfl_sync(0xFFFFFFFFu, e0, le);
          const bool own_rc = __shfl_sync(0xFFFFFFFFu, rc, le);
          const bool a = qe < tot;
          const u32 c = a ? ids[own_e0 + (qe - own_start)] : 0u;
          kahn_edge(c, a, own_rc, rem, reach, nxt, any_next);
        }
      }
    }
    grid.sync();
    // phase B: chunk tasks, one warp per task (most layers have none: then
    // the second barrier is skipped, uniformly across the grid)
    const u64 nt = ld_cg64(ntask);
    if (nt == 0) continue;
    for (u64 t = warp; t < nt; t += nwarps) {
      const uint2 tk = __ldcg(tasks + t);
      const bool trc = rv[tk.x] != 0;
      const u64 a = off[tk.x] + tk.y, b = min(off[tk.x + 1], a + kChunk);
      for (u64 e = a; e < b; e += 32) {
        const bool act = e + lane < b;
        const u32 c = act ? ids[e + lane] : 0u;
        kahn_edge(c, act, trc, rem, reach, nxt, any_next);
      }
    }
    grid.sync();
  }
  block_add_u64(found, &ctl->processed);
  if (gtid == 0) ctl->layers = L - 1;
}

// ---------------------------------------------------------------------------
// Batched Kahn layering (the default): same layers, reachability and heavy-
// rule chunk tasks as k_kahn, but every warp owns ONE contiguous range of
// bitmap words for all layers and runs each layer as four memory waves with
// every load of a wave in flight at once:
//   bitmap words (4 per lane) -> the frontier rules' CSR bounds and reach
//   (8 rules per lane, staged in shared memory) -> the child ids (4 edges per
//   lane, owner found by a binary search over the staged edge prefix) -> the
//   warp-aggregated counter decrements (4 atomics per lane in flight).
// k_kahn issues the same accesses as dependent chains (one rule / one edge
// per lane per round trip): ncu on C5 showed 33 % of its stall samples on
// the atomic results and 21 % on the offset and id loads.
// ---------------------------------------------------------------------------
constexpr int kK2Words = 4;            // bitmap words per lane per batch
constexpr u32 kK2Cap = 128;            // frontier rules staged per warp per round
constexpr int kK2PerLane = kK2Cap / 32;
constexpr int kK2Edges = 4;            // child edges per lane in flight
constexpr size_t kK2SmemPerWarp = kK2Cap * 8 + (kK2Cap + 1) * 4 + kK2Cap * 4 + kK2Cap;
constexpr size_t kK2Smem = 32 * ((kK2SmemPerWarp + 15) / 16 * 16);

__global__ void __launch_bounds__(kKahnBlock) k_kahn2(KahnCtl* ctl, u32* bm0, u32* bm1, u64 nwords,
                                                      const u64* __restrict__ off, const u32* __restrict__ ids,
                                                      u32* rem, u32* lvl, uint8_t* reach, uint2* tasks,
                                                      u64 max_layers) {
  extern __shared__ __align__(16) unsigned char k2_smem[];
  cg::grid_group grid = cg::this_grid();
  const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  unsigned char* base = k2_smem + (size_t)wib * ((kK2SmemPerWarp + 15) / 16 * 16);
  u64* s_e0 = reinterpret_cast<u64*>(base);
  u32* s_pre = reinterpret_cast<u32*>(base + kK2Cap * 8);
  u32* s_rule = reinterpret_cast<u32*>(base + kK2Cap * 8 + (kK2Cap + 1) * 4);
  uint8_t* s_rc = base + kK2Cap * 8 + (kK2Cap + 1) * 4 + kK2Cap * 4;
  const u64 gtid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 warp = gtid >> 5, nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 M = (nwords + nwarps - 1) / nwarps;
  const u64 wlo = min(warp * M, nwords), whi = min(wlo + M, nwords);
  const volatile uint8_t* rv = reach;
  u64 found = 0, L = 1;
  for (;; L++) {
    if (__ldcg(&ctl->any[L % 3]) == 0 || L > max_layers) break;
    if (gtid == 0) {
      ctl->any[(L + 2) % 3] = 0;
      ctl->ntask[(L + 1) & 1] = 0;
      if (L < 64) ctl->t[L] = globaltimer();
    }
    u32* cur = (L & 1) ? bm1 : bm0;
    u32* nxt = (L & 1) ? bm0 : bm1;
    u64* ntask = &ctl->ntask[L & 1];
    bool set_any = false;
    for (u64 b0 = wlo; b0 < whi; b0 += 32 * kK2Words) {
      u32 bits[kK2Words];
      u32 cnt = 0;
#pragma unroll
      for (int k = 0; k < kK2Words; k++) {
        const u64 wi = b0 + (u64)k * 32 + lane;
        bits[k] = wi < whi ? __ldcg(cur + wi) : 0u;
      }
#pragma unroll
      for (int k = 0; k < kK2Words; k++) {
        if (bits[k]) cur[b0 + (u64)k * 32 + lane] = 0;  // cleared for layer L + 2
        cnt += __popc(bits[k]);
      }
      u32 incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= (unsigned)d) incl += t;
      }
      const u32 T = __shfl_sync(0xFFFFFFFFu, incl, 31);
      const u32 excl = incl - cnt;
      found += cnt;
      for (u32 q0 = 0; q0 < T; q0 += kK2Cap) {
        const u32 n = min(T - q0, kK2Cap);
        // stage this round's frontier rules (ascending rule order)
        __syncwarp();
        if (excl < q0 + kK2Cap && excl + cnt > q0) {
          u32 q = excl;
#pragma unroll
          for (int k = 0; k < kK2Words; k++) {
            u32 b = bits[k];
            while (b && q < q0 + kK2Cap) {
              const u32 bp = __ffs(b) - 1;
              b &= b - 1;
              if (q >= q0) s_rule[q - q0] = (u32)((b0 + (u64)k * 32 + lane) * 32 + bp);
              q++;
            }
          }
        }
        __syncwarp();
        // wave 2: CSR bounds and reach of the staged rules (contiguous 8 per lane)
        u64 e0v[kK2PerLane], e1v[kK2PerLane];
        uint8_t rcv[kK2PerLane];
#pragma unroll
        for (int j = 0; j < kK2PerLane; j++) {
          const u32 i = lane * kK2PerLane + j;
          e0v[j] = e1v[j] = 0;
          rcv[j] = 0;
          if (i < n) {
            const u32 r = s_rule[i];
            e0v[j] = off[r];
            e1v[j] = off[r + 1];
            rcv[j] = rv[r];
            lvl[r] = (u32)L;
          }
        }
        u32 lsum = 0;
#pragma unroll
        for (int j = 0; j < kK2PerLane; j++) {
          const u32 i = lane * kK2PerLane + j;
          u64 len = e1v[j] - e0v[j];
          if (i < n && len > kLight) {  // heavy rule: chunk tasks for phase B
            const u32 r = s_rule[i];
            const u64 nch = (len + kChunk - 1) / kChunk;
            const u64 t0 = atomicAdd((unsigned long long*)ntask, (unsigned long long)nch);
            for (u64 k = 0; k < nch; k++) tasks[t0 + k] = make_uint2(r, (u32)(k * kChunk));
            len = 0;
          }
          if (i < n) {
            s_e0[i] = e0v[j];
            s_rc[i] = rcv[j];
            s_pre[i] = lsum;  // in-lane prefix, the lane's base added below
          }
          lsum += (u32)len;
        }
        u32 linc = lsum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const u32 t = __shfl_up_sync(0xFFFFFFFFu, linc, d);
          if (lane >= (unsigned)d) linc += t;
        }
        const u32 NE = __shfl_sync(0xFFFFFFFFu, linc, 31);
        const u32 lbase = linc - lsum;
#pragma unroll
        for (int j = 0; j < kK2PerLane; j++) {
          const u32 i = lane * kK2PerLane + j;
          if (i < n) s_pre[i] += lbase;
        }
        if (lane == 0) s_pre[n] = NE;
        __syncwarp();
        // waves 3 + 4: child ids, then the decrements, kK2Edges per lane in flight
        for (u32 k0 = 0; k0 < NE; k0 += 32 * kK2Edges) {
          u32 c[kK2Edges];
          bool act[kK2Edges], rch[kK2Edges];
#pragma unroll
          for (int j = 0; j < kK2Edges; j++) {
            const u32 qe = k0 + (u32)j * 32 + lane;
            act[j] = qe < NE;
            c[j] = 0;
            rch[j] = false;
            if (act[j]) {
              u32 lo = 0, hi = n;  // s_pre[lo] <= qe < s_pre[hi]
              while (hi - lo > 1) {
                const u32 mid = (lo + hi) >> 1;
                if (s_pre[mid] <= qe) lo = mid;
                else hi = mid;
              }
              c[j] = ids[s_e0[lo] + (qe - s_pre[lo])];
              rch[j] = s_rc[lo] != 0;
            }
          }
          u32 old[kK2Edges], kk[kK2Edges];
#pragma unroll
          for (int j = 0; j < kK2Edges; j++) {
            if (act[j] && rch[j]) reach[c[j]] = 1;
            const unsigned am = __ballot_sync(0xFFFFFFFFu, act[j]);
            kk[j] = 0;
            old[j] = 1;
            if (act[j]) {
              const unsigned peers = __match_any_sync(am, c[j]);
              if ((int)lane == __ffs(peers) - 1) {
                kk[j] = (u32)__popc(peers);
                old[j] = atomicSub(&rem[c[j]], kk[j]);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < kK2Edges; j++)
            if (kk[j] && old[j] == kk[j]) {
              atomicOr(&nxt[c[j] >> 5], 1u << (c[j] & 31u));
              set_any = true;
            }
        }
      }
    }
    if (__any_sync(0xFFFFFFFFu, set_any) && lane == 0) ctl->any[(L + 1) % 3] = 1;
    grid.sync();
    // phase B: heavy-rule chunk tasks, one warp per task
    const u64 nt = ld_cg64(ntask);
    if (nt == 0) continue;
    u32* any_next = &ctl->any[(L + 1) % 3];
    for (u64 t = warp; t < nt; t += nwarps) {
      const uint2 tk = __ldcg(tasks + t);
      const bool trc = rv[tk.x] != 0;
      const u64 a = off[tk.x] + tk.y, b = min(off[tk.x + 1], a + kChunk);
      for (u64 e = a; e < b; e += 32) {
        const bool act = e + lane < b;
        const u32 c = act ? ids[e + lane] : 0u;
        kahn_edge(c, act, trc, rem, reach, nxt, any_next);
      }
    }
    grid.sync();
  }
  block_add_u64(found, &ctl->processed);
  if (gtid == 0) {
    ctl->layers = L - 1;
    if (L < 64) ctl->t[L] = globaltimer();
  }
}

// ---------------------------------------------------------------------------
// Owner-scan Kahn layering for grammars whose sub CSR fits in shared memory
// (C1-C3): every warp owns a fixed range of rules for all layers and keeps
// that range's child lists AND its rules' remaining-parent counts in shared
// memory.  Decrements never touch those counts directly: a parent processed
// in layer L adds (fire-and-forget, warp-aggregated RED) to delta[L & 1] of
// the child; at the start of layer L + 1 the owner reads delta[L & 1] for
// its range (one coalesced wave, together with the reach bytes and the
// previous layer's activity flag), subtracts, clears it for layer L + 2 and
// finds its ready rules (count zero).  So a layer is: one load wave, the
// ready rules' REDs and reach pushes straight from shared memory, one grid
// barrier — no frontier bitmap, no atomic with return (k_kahn/k_kahn2 wait on
// atomic results, and same-address atomics on Zipf-popular children
// serialise).  Decrements of layer L are invisible to layer L's readiness by
// construction (they land in the other delta array).  The layering ends one
// (empty) layer after the last non-empty one.  Same layers, reachability and
// processed count as k_kahn / k_kahn2.
// ---------------------------------------------------------------------------
constexpr u32 kK3WarpWords = 1536;  // per-warp shared memory (u32 words)
constexpr int kK3Batch = 8;         // delta words loaded per lane per wave
constexpr u32 kK3List = 32 * kK3Batch;
constexpr u32 kK3Done = 0xFFFFFFFFu;

__global__ void __launch_bounds__(kKahnBlock) k_kahn3(KahnCtl* ctl, const u64* __restrict__ off,
                                                      const u32* __restrict__ ids, u64 R, u32* rem, u32* delta1,
                                                      u32* gdelta0, u32* lvl, uint8_t* reach, u64 max_layers) {
  extern __shared__ __align__(16) u32 k3_smem[];
  __shared__ u32 s_go, s_prev[2];
  cg::grid_group grid = cg::this_grid();
  const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  u32* sw = k3_smem + (size_t)wib * kK3WarpWords;
  const u64 gtid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  const u64 warp = gtid >> 5, nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 nwords = (R + 31) / 32;
  const u64 M = (nwords + nwarps - 1) / nwarps;
  const u64 wlo = min(warp * M, nwords), whi = min(wlo + M, nwords);
  const u64 m = whi - wlo, r0 = wlo * 32, r1 = min(whi * 32, R);
  const u64 nr = r1 > r0 ? r1 - r0 : 0;
  const u64 eb = nr ? off[r0] : 0, ee = nr ? off[r1] : 0;
  u32* s_list = sw;                 // this batch's ready rules: slot | reach << 31
  u32* s_cnt = sw + kK3List;        // nr remaining-parent counts (kK3Done once layered)
  u32* s_off = s_cnt + nr;          // nr + 1 offsets relative to eb
  u32* s_ids = s_off + nr + 1;
  // global-count mode (gdelta0 given: the grammar is too large for shared
  // memory): the counts stay in rem, both delta arrays come zeroed
  const bool gmode = gdelta0 != nullptr;
  const bool resident = !gmode && kK3List + 2 * nr + 1 + (ee - eb) <= kK3WarpWords;
  u32* cnt = gmode ? rem + r0 : s_cnt;
  u32* delta[2] = {gmode ? gdelta0 : rem, delta1};  // smem mode: rem doubles as delta[0]
  if (gtid == 0) {
    ctl->t[0] = globaltimer();
    ctl->first_unreached = 0xFFFFFFFFu;
    ctl->checked = 1;
  }
  // prologue: 8 loads per lane in flight per step (the copies are tiny but
  // each dependent load -> store step costs a full L2 round trip)
  const u32 nr32 = (u32)nr, ne32 = (u32)(ee - eb);
  if (gmode && gtid == 0) rem[0] = kK3Done;  // the root is layer 0
  for (u32 i0 = 0; !gmode && i0 < nr32; i0 += 256) {
    u32 t[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const u32 i = i0 + k * 32 + lane;
      t[k] = i < nr32 ? __ldcg(rem + r0 + i) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const u32 i = i0 + k * 32 + lane;
      if (i < nr32) {
        s_cnt[i] = r0 + i == 0 ? kK3Done : t[k];  // the root is layer 0
        rem[r0 + i] = 0;
        delta1[r0 + i] = 0;
      }
    }
  }
  if (resident && nr32) {  // (a warp past the last rule has no range: off[r0] may not exist)
    for (u32 i0 = 0; i0 <= nr32; i0 += 256) {
      u64 t[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const u32 i = i0 + k * 32 + lane;
        t[k] = i <= nr32 ? off[r0 + i] : 0;
      }
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const u32 i = i0 + k * 32 + lane;
        if (i <= nr32) s_off[i] = (u32)(t[k] - eb);
      }
    }
    for (u32 i0 = 0; i0 < ne32; i0 += 256) {
      u32 t[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const u32 i = i0 + k * 32 + lane;
        t[k] = i < ne32 ? ids[eb + i] : 0u;
      }
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const u32 i = i0 + k * 32 + lane;
        if (i < ne32) s_ids[i] = t[k];
      }
    }
  }
  if (threadIdx.x == 0) s_prev[0] = s_prev[1] = 0;
  grid.sync();
  const volatile uint8_t* rv = reach;
  u64 found = 0, L = 1;
  for (;; L++) {
    u32* din = delta[(L - 1) & 1];  // decrements made in layer L - 1
    u32* dout = delta[L & 1];
    const volatile uint8_t* rvw = rv + r0;
    u32 v[kK3Batch], rcb = 0;
#pragma unroll
    for (int k = 0; k < kK3Batch; k++) {
      const u32 slot = k * 32 + lane;
      const bool ok = slot < nr32;
      v[k] = ok && L > 1 ? __ldcg(din + r0 + slot) : 0u;
      rcb |= (ok && rvw[slot]) ? 1u << k : 0u;
    }
    if (L > 1 && s_go == 0) break;  // layer L - 1 was empty (s_go set by the barrier below)
    if (L > max_layers) break;
    if (gtid == 0 && L < 64) ctl->t[L] = globaltimer();
    bool active = false;
    for (u64 i0 = 0; i0 < m; i0 += kK3Batch) {
      if (i0) {
        rcb = 0;
#pragma unroll
        for (int k = 0; k < kK3Batch; k++) {
          const u32 slot = (u32)i0 * 32 + k * 32 + lane;
          const bool ok = slot < nr32;
          v[k] = ok && L > 1 ? __ldcg(din + r0 + slot) : 0u;
          rcb |= (ok && rvw[slot]) ? 1u << k : 0u;
        }
      }
      // counters -> ready rules, compacted into the warp's list
      u32 nready = 0;
      u32* dinw = din + r0;
#pragma unroll
      for (int k = 0; k < kK3Batch; k++) {
        if ((u32)i0 + k >= (u32)m) break;
        const u32 slot = (u32)i0 * 32 + k * 32 + lane;
        bool ready = false;
        if (slot < nr32 && (!gmode || L == 1 || v[k])) {
          u32 c = gmode ? __ldcg(cnt + slot) : cnt[slot];
          if (v[k]) {
            dinw[slot] = 0;  // cleared for layer L + 1's decrements
            c -= v[k];
          }
          ready = c == 0;
          if (ready) c = kK3Done;
          if (v[k] || ready) cnt[slot] = c;
        }
        const unsigned mask = __ballot_sync(0xFFFFFFFFu, ready);
        if (ready) s_list[nready + __popc(mask & lt_mask)] = slot | (((rcb >> k) & 1u) << 31);
        nready += __popc(mask);
      }
      if (!nready) continue;
      active = true;
      __syncwarp();
      // the ready rules, one per lane: each walks its own children (fire-
      // and-forget REDs; most rules have < 8 children)
      for (u32 q0 = 0; q0 < nready; q0 += 32) {
        const bool act = q0 + lane < nready;
        u32 slot = 0, rc = 0, e0 = 0, deg = 0;
        u64 g0 = 0;
        if (act) {
          const u32 e = s_list[q0 + lane];
          slot = e & 0x7FFFFFFFu;
          rc = e >> 31;
          const u64 r = r0 + slot;
          lvl[r] = (u32)L;
          found++;
          if (resident) {
            e0 = s_off[slot];
            deg = s_off[slot + 1] - e0;
          } else {
            g0 = off[r];
            deg = (u32)(off[r + 1] - g0);
          }
        }
        const bool light = act && deg <= 32;
        for (u32 j = 0;; j++) {
          const bool go = light && j < deg;
          if (!__any_sync(0xFFFFFFFFu, go)) break;
          if (go) {
            const u32 c = resident ? s_ids[e0 + j] : ids[g0 + j];
            if (rc) reach[c] = 1;
            atomicAdd(&dout[c], 1u);
          }
        }
        // heavy rules (> 32 children): the whole warp walks each one
        unsigned hm = __ballot_sync(0xFFFFFFFFu, act && deg > 32);
        while (hm) {
          const int src = __ffs(hm) - 1;
          hm &= hm - 1;
          const u32 he0 = __shfl_sync(0xFFFFFFFFu, e0, src), hdeg = __shfl_sync(0xFFFFFFFFu, deg, src);
          const u64 hg0 = __shfl_sync(0xFFFFFFFFu, g0, src);
          const u32 hrc = __shfl_sync(0xFFFFFFFFu, rc, src);
          for (u32 q = lane; q < hdeg; q += 32) {
            const u32 c = resident ? s_ids[he0 + q] : ids[hg0 + q];
            if (hrc) reach[c] = 1;
            atomicAdd(&dout[c], 1u);
          }
        }
      }
      __syncwarp();
    }
    // layer barrier carrying the layer's activity: one release-add per
    // block of (1 arrival + the block's activity in this layer's parity
    // field), thread 0 spins until every block arrived, and the field's
    // growth since the same-parity layer before tells whether ANY block was
    // active (a fast block's next-layer add can only touch the other field)
    const int blk_active = __syncthreads_or(active);
    if (threadIdx.x == 0) {
      const int sh = 32 + 16 * (int)(L & 1);
      const u64 add = 1ull + (blk_active ? (1ull << sh) : 0ull);
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&ctl->bar), "l"(add) : "memory");
      const u64 target = (u64)gridDim.x * L;
      u64 v;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&ctl->bar) : "memory");
      } while ((v & 0xFFFFFFFFull) < target);
      const u32 f = (u32)(v >> sh) & 0xFFFFu;
      s_go = (f - s_prev[L & 1]) & 0xFFFFu;
      s_prev[L & 1] = f;
    }
    __syncthreads();
  }
  // fused checks (every reach byte is final after the last barrier): the
  // first unreachable rule, and a reachable rule (or the root) referencing
  // the root — replaces two launches and their host round trip
  {
    u32 minr = 0xFFFFFFFFu;
    bool cyc = false;
    for (u32 s0 = 0; s0 < nr32; s0 += 32) {  // warp-uniform trip count
      const u32 slot = s0 + lane;
      const u64 r = r0 + slot;
      const bool ok = slot < nr32;
      const bool rr = ok && (r == 0 || rv[r] != 0);
      if (ok && !rr) minr = min(minr, (u32)r);
      // child lists ascend, so only a rule's first child can be the root
      if (rr) {
        if (resident) cyc |= s_off[slot + 1] > s_off[slot] && s_ids[s_off[slot]] == 0;
        else cyc |= off[r + 1] > off[r] && ids[off[r]] == 0;
      }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) minr = min(minr, __shfl_xor_sync(0xFFFFFFFFu, minr, d));
    cyc = __any_sync(0xFFFFFFFFu, cyc);
    if (lane == 0) {
      if (minr != 0xFFFFFFFFu) atomicMin(&ctl->first_unreached, minr);
      if (cyc) ctl->root_cycle = 1;
    }
  }
  block_add_u64(found, &ctl->processed);
  if (gtid == 0) ctl->layers = L - 2;  // L - 1 was the first empty layer
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
  const u64 warp = (u64)(threadIdx.x >> 5) * gridDim.x + blockIdx.x;  // round-robin over the SMs
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


// in-degrees straight from the (parent-major) sub pairs, no parent sort:
// rem[c] = distinct non-root parents of c (the top-down Kahn counters),
// rootp[c] = c is referenced by the root
__global__ void k_in_degrees(const u32* __restrict__ prule, const u32* __restrict__ child, u64 n, u32* rem,
                             uint8_t* rootp) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 p = prule[i], c = child[i];
    if (p == 0) rootp[c] = 1;
    else atomicAdd(&rem[c], 1u);
  }
}

// a reachable rule (or the root itself) referencing the root is a cycle
__global__ void k_root_cycle2(const u32* __restrict__ prule, const u32* __restrict__ child, u64 n,
                              const uint8_t* __restrict__ reach, u32* bad) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (child[i] == 0) {
      const u32 p = prule[i];
      if (p == 0 || reach[p]) *bad = 1;
    }
}

}  // namespace (the list kernels below are shared with contract.cu)

// top-down edge lists by scatter: every child's non-root parent edges get a
// contiguous slot range in (td level, child) = tid order (exclusive scan of
// the in-degrees in tid order); within a child the slot order is the order
// the atomics land in — the segmented reduce only needs each child's items
// contiguous, and its sums are exact integers
__global__ void k_cursor(const u32* __restrict__ degt, const u32* __restrict__ incl, u64 n, u32* cur) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) cur[t] = incl[t] - degt[t];
}

// (one 12-byte record per edge: a random slot costs one write sector, not
// three — the separate arrays come from one coalesced unpack afterwards;
// C5: 3.2 ms with three scattered 4-byte stores per edge)
__global__ void k_te_scatter(const u32* __restrict__ prule, const u32* __restrict__ child,
                             const u32* __restrict__ freq, u64 n, const u32* __restrict__ tid, u32* cur,
                             U3* te) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 p = prule[i];
    if (p == 0) continue;
    const u32 tc = tid[child[i]];
    const u32 slot = atomicAdd(&cur[tc], 1u);
    te[slot] = U3{tc, tid[p], freq[i]};
  }
}

// level offsets of the td edge lists: off[L] = first edge whose child is in
// level >= L (ls[L] = first tid of level >= L, L = 0..nl+1), off[nl+2] = all
// ---- stable counting sort by a small key (the level numberings) -----------
// n keys in [0, nb) with nb <= kLoBins: ord[i] = the i-th element in (key,
// index) order, rank[e] = its position, starts[k] = the first position of
// key k (k = 0..nb; starts[nb] = n).  Three launches (per-block counts, one
// single-block scan, a stable block-ordered scatter) instead of a radix sort,
// a rank pass and a binary search per key.
constexpr int kLoBins = 64, kLoBlock = 1024;
__global__ void __launch_bounds__(kLoBlock) k_lo_count(const u32* __restrict__ key, u64 n, u64 chunk, u32 nb,
                                                     u32* cnt) {
  __shared__ u32 h[kLoBins];
  for (u32 i = threadIdx.x; i < kLoBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const u64 lo = (u64)blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  for (u64 b = lo; b < hi; b += blockDim.x) {
    const u64 i = b + threadIdx.x;
    const u32 k = i < hi ? key[i] : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, k);
    if (k != 0xFFFFFFFFu && (threadIdx.x & 31u) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&h[k], (u32)__popc(peers));
  }
  __syncthreads();
  for (u32 k = threadIdx.x; k < nb; k += blockDim.x) cnt[(u64)k * gridDim.x + blockIdx.x] = h[k];
}

// exclusive scan of the (key-major) block counts in place; starts[k] = the
// offset of key k in block 0
__global__ void __launch_bounds__(kLoBlock) k_lo_scan(u32* cnt, u32 nblk, u32 nb, u64 n, u64* starts) {
  __shared__ u32 wsum[32];
  __shared__ u32 carry;
  const u32 m = nblk * nb, lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u32 t0 = 0; t0 < m; t0 += blockDim.x) {
    const u32 i = t0 + threadIdx.x;
    const u32 v = i < m ? cnt[i] : 0u;
    u32 x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, d);
      if (lane >= (u32)d) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      u32 z = lane < blockDim.x / 32 ? wsum[lane] : 0u;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u32 y = __shfl_up_sync(0xFFFFFFFFu, z, d);
        if (lane >= (u32)d) z += y;
      }
      wsum[lane] = z;  // inclusive over warps
    }
    __syncthreads();
    const u32 c0 = carry;
    const u32 ex = c0 + (w ? wsum[w - 1] : 0u) + x - v;
    if (i < m) {
      cnt[i] = ex;
      if (i % nblk == 0) starts[i / nblk] = ex;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + wsum[blockDim.x / 32 - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) starts[nb] = n;
}

__global__ void __launch_bounds__(kLoBlock) k_lo_scatter(const u32* __restrict__ key, u64 n, u64 chunk, u32 nb,
                                                       const u32* __restrict__ off, u32* ord, u32* rank) {
  __shared__ u32 run[kLoBins], tt[kLoBins];
  __shared__ u32 wc[kLoBlock / 32][kLoBins];
  const u32 lane = threadIdx.x & 31u, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (u32 k = threadIdx.x; k < nb; k += blockDim.x) run[k] = off[(u64)k * gridDim.x + blockIdx.x];
  const u64 lo = (u64)blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  for (u64 b = lo; b < hi; b += blockDim.x) {
    for (u32 k = lane; k < kLoBins; k += 32) wc[w][k] = 0;
    __syncthreads();
    const u64 i = b + threadIdx.x;
    const bool ok = i < hi;
    const u32 k = ok ? key[i] : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, k);
    const u32 r = __popc(peers & ((1u << lane) - 1u));
    if (ok && r == 0) wc[w][k] = (u32)__popc(peers);
    __syncthreads();
    if (threadIdx.x < nb) {  // exclusive prefix over the warps, per key
      u32 a = 0;
      for (u32 q = 0; q < nw; q++) {
        const u32 c = wc[q][threadIdx.x];
        wc[q][threadIdx.x] = a;
        a += c;
      }
      tt[threadIdx.x] = a;
    }
    __syncthreads();
    if (ok) {
      const u32 pos = run[k] + wc[w][k] + r;
      ord[pos] = (u32)i;
      rank[i] = pos;
    }
    __syncthreads();
    if (threadIdx.x < nb) run[threadIdx.x] += tt[threadIdx.x];
  }
}

// k_unpack3 over the first *n_dev records (the count stays on the device)
__global__ void k_unpack3_n(const U3* __restrict__ in, const u32* __restrict__ n_dev, u32* a, u32* b, u32* c) {
  const u64 n = *n_dev;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const U3 v = in[i];
    a[i] = v.a;
    b[i] = v.b;
    c[i] = v.c;
  }
}

__global__ void k_te_level_off(const u64* __restrict__ ls, const u32* __restrict__ incl,
                               const u32* __restrict__ degt, u64 R, u64 nl, u64* off) {
  const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nl + 2) return;
  const u64 tot = R ? incl[R - 1] : 0;
  const u64 t = k <= nl + 1 ? ls[k] : R;
  off[k] = t < R ? incl[t] - degt[t] : tot;
}

namespace {

// rule id of every sub pair (expanding sub_off), for the lazily built parent CSR
__global__ void k_expand_owner(const u64* __restrict__ off, u64 R, u32* owner) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride)
    for (u64 e = off[r]; e < off[r + 1]; e++) owner[e] = (u32)r;
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
__global__ void k_root_keys(const u32* body, const u32* seg_incl, u64 L0, u64 nw, u64 base, u64 limit,
                            int SBF, bool headless, u64* rkey, uint8_t* isr, u64* wkey,
                            uint8_t* isw, u32* seg_of) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < L0; p += stride) {
    u32 s = body[p];
    u32 seg = headless ? 0u : seg_incl[p];  // splitters before p (p itself not a splitter)
    seg_of[p] = seg;
    // (a symbol past the rules is reported by the unpack; here it is no occurrence)
    bool rr = s >= base && s < limit, ww = s < nw;
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
  stream_sync(s);
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
  out->off_dev.alloc((nl + 2) * 8, st);
  GT_CUDA(cudaMemcpyAsync(out->off_dev.p, out->off.data(), (nl + 2) * 8, cudaMemcpyHostToDevice, st));
  stream_sync(st);  // the host vector is the copy's source
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
    stream_sync(st);
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

// Host -> device copy of the GTDC bytes.  Pinned sources go straight to the
// copy engine.  A large pageable source (Python bytes, a file read) would go
// through the driver's own staging at ~10 GB/s; instead it is copied into two
// pinned 64 MB staging buffers by several host threads while the copy engine
// drains the other buffer (C4, 227 MB: pageable gt_open 31 -> 20 ms).
static void h2d_blob(void* dst, const uint8_t* src, size_t n, cudaStream_t st) {
  constexpr size_t kCh = 64ull << 20;
  bool direct = n < (32ull << 20);
  if (!direct) {
    cudaPointerAttributes at{};
    direct = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
    if (!direct) cudaGetLastError();
  }
  if (direct) {
    GT_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
    return;
  }
  struct Stage {
    uint8_t* p[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    Stage() {
      for (int i = 0; i < 2; i++) {
        GT_CUDA(cudaMallocHost(&p[i], kCh));
        GT_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
      }
    }
  };
  static thread_local Stage stg;  // process lifetime (pinned pages are never returned)
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  for (size_t off = 0, i = 0; off < n; off += kCh, i++) {
    const int b = (int)(i & 1);
    if (i >= 2) GT_CUDA(cudaEventSynchronize(stg.ev[b]));  // its previous copy has left the buffer
    const size_t len = std::min(kCh, n - off);
    const size_t part = (len + hw - 1) / hw;
    // (the workers get plain pointers: `stg` is thread_local, a worker would
    // see its own instance)
    uint8_t* sp = stg.p[b];
    const uint8_t* from = src + off;
    std::vector<std::thread> th;
    for (unsigned t = 1; t < hw && t * part < len; t++)
      th.emplace_back([sp, from, part, len, t] { memcpy(sp + t * part, from + t * part, std::min(part, len - t * part)); });
    memcpy(sp, from, std::min(part, len));
    for (auto& x : th) x.join();
    GT_CUDA(cudaMemcpyAsync((uint8_t*)dst + off, stg.p[b], len, cudaMemcpyHostToDevice, st));
    GT_CUDA(cudaEventRecord(stg.ev[b], st));
  }
}

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

// dag.py's parent CSR (par_ids / par_freqs / par_off, parents ascending per
// child) and num_in_edge: no task reads them (the top-down edge lists are
// scattered from the sub pairs at load), so they are built on first request
// (gt_dag_array) with one stable sort of the sub pairs by child
void ensure_parents(DeviceDag* d) {
  if (d->par_off.p || d->R == 0) return;
  GT_CUDA(cudaSetDevice(d->device));
  cudaStream_t st = d->stream;
  const u64 R = d->R, Es = d->E_sub;
  DBuf prule(Es * 4 + 4, st), child_sorted(Es * 4 + 4, st), v1(Es * 8 + 8, st), v2(Es * 8 + 8, st);
  LAUNCH(k_expand_owner, R, d->sub_off.as<u64>(), R, prule.as<u32>());
  LAUNCH(k_pack2, Es, prule.as<u32>(), d->sub_freqs.as<u32>(), Es, v1.as<u64>());
  sort_pairs_u32_u64(d->sub_ids.as<u32>(), child_sorted.as<u32>(), v1.as<u64>(), v2.as<u64>(), Es,
                     std::max(1, bitlen(R - 1)), st);
  d->par_ids.alloc(Es * 4 + 4, st);
  d->par_freqs.alloc(Es * 4 + 4, st);
  d->par_off.alloc((R + 1) * 8, st);
  LAUNCH(k_unpack2, Es, v2.as<u64>(), Es, d->par_ids.as<u32>(), d->par_freqs.as<u32>());
  LAUNCH(k_csr_offsets_lin, Es + 1, child_sorted.as<u32>(), Es, R, d->par_off.as<u64>());
  d->num_in.alloc(R * 8, st);
  GT_CUDA(cudaMemsetAsync(d->num_in.p, 0, R * 8, st));
  LAUNCH(k_seg_sum_sorted, Es, child_sorted.as<u32>(), Es,
         (ValU32NonRoot{d->par_freqs.as<u32>(), d->par_ids.as<u32>()}), d->num_in.as<u64>());
  GT_CUDA(cudaStreamSynchronize(st));
}

// The derived arrays (DeviceDag::derived), on first use:
//   be lists — sub entries (grouped by rule) by the rule's TOP-DOWN level;
//     walked in decreasing level order every child is finished before its
//     parents (a child's td level exceeds each parent's), which is all the
//     bottom-up sums need; the root (td level 0) comes last;
//   heights (= the reference's bottom-up rounds, engine.py:313-335; leaf = 1)
//     and exp_len (grammar.py:109-124) in ONE persistent reverse pass;
//   segment_token_counts (dag.py:88-104), the longest file, W, depth.
void ensure_derived(DeviceDag* d) {
  if (d->derived) return;
  GT_CUDA(cudaSetDevice(d->device));
  cudaStream_t st = d->stream;
  const u64 R = d->R, Es = d->E_sub, nw = d->nw, base = d->nw + d->ns;
  const int ntd = d->td.nl;
  static thread_local PinnedU64 stage_host;
  u64* stage = stage_host.get((u64)ntd + 3 + 3);
  {
    const Carve cv(st, {Es * 4 + 4, Es * 4 + 4, Es * 12 + 12, Es * 12 + 12});
    const DPtr key{cv.at<void>(0)}, key2{cv.at<void>(1)}, v1{cv.at<void>(2)}, v2{cv.at<void>(3)};
    const u32* sr = d->sub_rule.as<u32>();
    LAUNCH(k_edge_level_keys2, Es, sr, nullptr, d->td_level.as<u32>(), (u32)ntd + 1, Es, key.as<u32>());
    LAUNCH(k_pack3, Es, sr, d->sub_ids.as<u32>(), d->sub_freqs.as<u32>(), Es, v1.as<U3>());
    sort_pairs_u32_u3(key.as<u32>(), key2.as<u32>(), v1.as<U3>(), v2.as<U3>(), Es,
                      std::max(1, bitlen((u64)ntd + 1)), st);
    d->be_rule.alloc(Es * 4 + 16, st);
    d->be_child.alloc(Es * 4 + 16, st);
    d->be_freq.alloc(Es * 4 + 16, st);
    LAUNCH(k_unpack3, Es, v2.as<U3>(), Es, d->be_rule.as<u32>(), d->be_child.as<u32>(), d->be_freq.as<u32>());
    d->be_off_dev.alloc(((u64)ntd + 3) * 8, st);
    LAUNCH(k_csr_offsets, (u64)ntd + 3, key2.as<u32>(), Es, (u64)ntd + 2, d->be_off_dev.as<u64>());
    GT_CUDA(cudaMemcpyAsync(stage, d->be_off_dev.p, ((u64)ntd + 3) * 8, cudaMemcpyDeviceToHost, st));
  }
  d->exp_len.alloc(R * 8, st);
  {
    DBuf hgt(R * 8, st);
    LAUNCH(k_fill_u64, R, hgt.as<u64>(), R, 1ull);
    GT_CUDA(cudaMemcpyAsync(d->exp_len.p, d->own_tok.p, R * 8, cudaMemcpyDeviceToDevice, st));
    static int per_sm = -1;
    if (per_sm < 0) {
      GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bu_pair, 1024, 0));
      per_sm = std::max(per_sm, 1);
    }
    int nsm = 148;
    GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, d->device));
    const u32* br = d->be_rule.as<u32>();
    const u32* bc = d->be_child.as<u32>();
    const u32* bf = d->be_freq.as<u32>();
    const u64* bo = d->be_off_dev.as<u64>();
    int L1 = ntd;
    u64* hg = hgt.as<u64>();
    u64* el = d->exp_len.as<u64>();
    void* args[] = {(void*)&br, (void*)&bc, (void*)&bf, (void*)&bo, (void*)&L1, (void*)&hg, (void*)&el};
    {
      ProfScope ps_("k_bu_pair", st);
      GT_CUDA(cudaLaunchCooperativeKernel((const void*)k_bu_pair, dim3((unsigned)(nsm * per_sm)), dim3(1024), args,
                                          0, st));
      g_launches++;
    }
    LAUNCH(k_u64_to_u32, R, hgt.as<u64>(), R, d->bu_level.as<u32>());
    // the reference's bottom-up rounds exclude the root (engine.py:305-310)
    GT_CUDA(cudaMemsetAsync(d->bu_level.p, 0, 4, st));
    u64* hw = stage + (ntd + 3);
    GT_CUDA(cudaMemcpyAsync(&hw[0], hgt.p, 8, cudaMemcpyDeviceToHost, st));          // root height
    GT_CUDA(cudaMemcpyAsync(&hw[1], d->exp_len.p, 8, cudaMemcpyDeviceToHost, st));  // W
  }
  {
    d->seg_tokens.alloc(d->F * 8, st);
    GT_CUDA(cudaMemsetAsync(d->seg_tokens.p, 0, d->F * 8, st));
    LAUNCH(k_seg_sum_sorted, d->L0, d->root_seg.as<u32>(), d->L0,
           (ValRootLen{d->body.as<u32>(), d->exp_len.as<u64>(), nw, base}), d->seg_tokens.as<u64>());
    DBuf mx(8, st);
    reduce_max_u64(d->seg_tokens.as<u64>(), mx.as<u64>(), d->F, st);
    GT_CUDA(cudaMemcpyAsync(stage + (ntd + 3) + 2, mx.p, 8, cudaMemcpyDeviceToHost, st));  // longest file
  }
  stream_sync(st);
  d->be_off.assign(stage, stage + ntd + 3);
  const u64* hw = stage + (ntd + 3);
  d->bu.nl = (int)hw[0];
  d->depth = (i64)hw[0] - 1;
  d->W = hw[1];
  d->max_file_tokens = hw[2];
  static const bool rows64 = getenv("GT_ROWS64") != nullptr;
  d->cnt32 = !rows64 && hw[2] < (1ull << 32);
  if (d->cnt32) d->load_flags |= 2;
  d->derived = true;
}

void build_device_dag(const uint8_t* blob, size_t nbytes, int device, u64 file_lo, u64 file_hi,
                      DeviceDag* d) {
  auto t0 = std::chrono::steady_clock::now();
  Phases ph("gt_open");
  Parse P;
  if (nbytes < 4 || memcmp(blob, "GTDC", 4) != 0) fail(GT_E_FORMAT, "bad magic: not a GTDC file");
  GT_CUDA(cudaSetDevice(device));
  d->device = device;
  if (!d->stream) d->stream = stream_acquire(device);
  cudaStream_t st = d->stream;
  ph.bind(st);
  reserve_pool(device, st);
  ph.mark("stream");
  // the whole blob streams to the device while the host validates the
  // header and dictionary (overlaps when `blob` is pinned); the rules section
  // is then re-aligned on the device (the dictionary has byte lengths)
  DBuf dblob(nbytes + 4, st);
  // a pinned (or small) blob streams in pieces on a copy stream, one event
  // each: the rules section is re-aligned piece by piece and the rule-chain
  // tables start on the chunks that have arrived while the rest streams
  std::vector<std::pair<size_t, cudaEvent_t>> pieces;  // (end byte, arrival)
  cudaStream_t s_cp = nullptr;
  {
    bool direct = nbytes < (32ull << 20);
    if (!direct) {
      cudaPointerAttributes at{};
      direct = cudaPointerGetAttributes(&at, blob) == cudaSuccess && at.type == cudaMemoryTypeHost;
      if (!direct) cudaGetLastError();
    }
    // (a small blob arrives about when the host has parsed its dictionary:
    // pieces only add waits and launches there — C2, 18 MB: 1.15 vs 1.44 ms)
    static const bool one_copy = getenv("GT_H2D_ONE") != nullptr;  // diagnostics: one copy on the main stream
    if (direct && !one_copy && nbytes >= (64ull << 20)) {
      s_cp = stream_acquire(device);
      cudaEvent_t alloc_ev;
      GT_CUDA(cudaEventCreateWithFlags(&alloc_ev, cudaEventDisableTiming));
      GT_CUDA(cudaEventRecord(alloc_ev, st));  // (dblob is a stream-ordered allocation on st)
      GT_CUDA(cudaStreamWaitEvent(s_cp, alloc_ev, 0));
      cudaEventDestroy(alloc_ev);
      const size_t piece = std::max<size_t>(16ull << 20, (nbytes + 7) / 8);
      for (size_t o = 0; o < nbytes; o += piece) {
        const size_t len = std::min(piece, nbytes - o);
        GT_CUDA(cudaMemcpyAsync(dblob.as<uint8_t>() + o, blob + o, len, cudaMemcpyHostToDevice, s_cp));
        cudaEvent_t ev;
        GT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        GT_CUDA(cudaEventRecord(ev, s_cp));
        pieces.push_back({o + len, ev});
      }
    } else {
      h2d_blob(dblob.p, blob, nbytes, st);
    }
  }
  struct PieceGuard {  // error paths: the copy stream and events go back
    std::vector<std::pair<size_t, cudaEvent_t>>* pc;
    cudaStream_t* s;
    int device;
    ~PieceGuard() {
      for (auto& x : *pc)
        if (x.second) cudaEventDestroy(x.second);
      if (*s) {
        cudaStreamSynchronize(*s);
        stream_release(device, *s);
      }
    }
  } piece_guard{&pieces, &s_cp, device};
  parse_dict(blob, nbytes, &P);
  ph.mark("host parse: dictionary");
  const u64 nsec = (nbytes - P.rules_pos) / 4;
  // device ids and body offsets of the rule-chain parse and the CSR build are
  // u32: a rules section of 2^32 - 1 or more words cannot be represented
  // (fail loudly instead of truncating rule starts)
  if (nsec >= 0xFFFFFFFFull)
    fail(GT_E_RESOURCE, "grammar too large: rules section of %lu words exceeds the 2^32 - 2 word limit",
         (unsigned long)nsec);
  DBuf raw(nsec * 4 + 4, st);
  u64 w_done = 0;       // raw words re-aligned (queued on st)
  size_t piece_at = 0;  // next piece to wait for
  auto realign_to = [&](u64 w_hi) {
    if (w_hi > w_done)
      GT_CUDA(cudaMemcpyAsync(raw.as<uint8_t>() + w_done * 4, dblob.as<uint8_t>() + P.rules_pos + w_done * 4,
                              (w_hi - w_done) * 4, cudaMemcpyDeviceToDevice, st));
    w_done = std::max(w_done, w_hi);
  };
  // the next piece: st waits for its arrival and re-aligns the words it completes
  auto arrive_piece = [&]() {
    if (piece_at >= pieces.size()) return false;
    auto& pc = pieces[piece_at++];
    GT_CUDA(cudaStreamWaitEvent(st, pc.second, 0));
    cudaEventDestroy(pc.second);
    pc.second = nullptr;
    const size_t end = pc.first;
    realign_to(end >= nbytes ? nsec : std::min<u64>(nsec, end > P.rules_pos ? (end - P.rules_pos) / 4 : 0));
    return true;
  };
  auto arrive_all = [&]() {
    while (arrive_piece()) {
    }
    realign_to(nsec);
    if (s_cp) {
      stream_release(device, s_cp);  // (every later use of the blob waits on st, which waited on each piece)
      s_cp = nullptr;
    }
    dblob.release();
  };
  // the root record first (the root side below reads it)
  {
    const u64 root_words = nsec ? std::min<u64>(nsec, 1 + (u64)rd32(blob + P.rules_pos)) : 0;
    if (pieces.empty()) arrive_all();
    while (w_done < root_words && arrive_piece()) {
    }
  }
  // ---- root side (splitters, segments, root occurrence lists): only needs
  // the root body, so it runs on its own stream and host thread while the
  // main pipeline builds the CSR, the layering and the level lists; its
  // errors are raised after the main pipeline's, in the reference's order
  // (dag.py:131-230: cycle, unreachable, then _segments_of_root)
  // (the root is the first record of the section: its body is raw[1, 1 + L0)
  // whatever the rest of the chain holds; a length past the section fails
  // the chain parse below, the root side then reads a clamped range)
  const u64 rR = P.R, rnw = P.nw, rns = P.ns, rbase = rnw + rns, rlimit = rbase + rR;
  const u64 L0 = rR && nsec ? std::min<u64>(rd32(blob + P.rules_pos), nsec - 1) : 0;  // the root's body length
  const u32* rbody = raw.as<u32>() + 1;
  d->L0 = L0;
  cudaEvent_t ev_body;
  GT_CUDA(cudaEventCreateWithFlags(&ev_body, cudaEventDisableTiming));
  GT_CUDA(cudaEventRecord(ev_body, st));
  Error root_err{GT_OK, ""};
  cudaStream_t s_root = stream_acquire(device);
  auto root_side = [&]() {
    try {
      GT_CUDA(cudaSetDevice(device));
      cudaStream_t st = s_root;
      GT_CUDA(cudaStreamWaitEvent(st, ev_body, 0));
      DBuf cnt(16, st);
  // ---- root segments (dag.py:107-128) -------------------------------------
    const bool headless = rns == 0;
    DBuf spl(L0 + 1, st), splu(L0 * 4 + 4, st), sincl(L0 * 4 + 4, st), spos(L0 * 4 + 4, st);
    LAUNCH(k_root_flags, L0, rbody, L0, rnw, rbase, spl.as<uint8_t>(), splu.as<u32>());
    select_flagged_index(spl.as<uint8_t>(), spos.as<u32>(), cnt.as<u64>(), L0, st);
    inclusive_scan_u32(splu.as<u32>(), sincl.as<u32>(), L0, st);
    u64 nspl;
    d2h(&nspl, cnt.p, 1, st);
    if (!headless) {
      DBuf fb(4, st);
      GT_CUDA(cudaMemsetAsync(fb.p, 0xFF, 4, st));
      LAUNCH(k_check_splitters, nspl ? nspl : 1, rbody, spos.as<u32>(), cnt.as<u64>(), rnw,
             fb.as<u32>());
      u32 k;
      d2h(&k, fb.p, 1, st);
      if (k != 0xFFFFFFFFu) {
        u32 pos, sym;
        d2h(&pos, spos.as<u32>() + k, 1, st);
        d2h(&sym, rbody + pos, 1, st);
        fail(GT_E_CORRUPTION, "splitter %u out of order at root position %u", sym, pos);
      }
      if (nspl != rns) fail(GT_E_CORRUPTION, "root body is missing file splitters");
      u32 last = 0;
      if (nspl) d2h(&last, spos.as<u32>() + nspl - 1, 1, st);
      if (!nspl || (u64)last + 1 != L0) fail(GT_E_CORRUPTION, "root body has content after the last splitter");
    }
    const u64 F = headless ? 1 : rns;
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
    LAUNCH(k_root_keys, L0, rbody, sincl.as<u32>(), L0, rnw, rbase, rlimit, SBF, headless,
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
    occ_list(rkey, isr, std::max(1, bitlen(rR - 1)), d->rs_rule, d->rs_seg, d->rs_cnt, &d->n_rs);
    occ_list(wkey, isw, std::max(1, bitlen(rnw ? rnw - 1 : 0)), d->rw_word, d->rw_seg, d->rw_cnt, &d->n_rw);
    d->rs_off.alloc((rR + 1) * 8, st);
    if (d->n_rs * 4 >= rR)  // dense keys: one coalesced pass; sparse: a search per row
      LAUNCH(k_csr_offsets_lin, d->n_rs + 1, d->rs_rule.as<u32>(), d->n_rs, rR, d->rs_off.as<u64>());
    else
      LAUNCH(k_csr_offsets, rR + 1, d->rs_rule.as<u32>(), d->n_rs, rR, d->rs_off.as<u64>());
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
    stream_release(device, s_root);
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
      stream_release(device, s_root);
    }
  }};


  // the rule-start table: on the device by pointer doubling; the host walk
  // (parse_rules, the reference's sequential reader) runs only to produce the
  // exact error of a malformed section, or when an error path needs it
  static thread_local PinnedU32 rstart_host;
  bool host_chain = false;
  auto need_host_chain = [&]() {
    if (host_chain) return;
    stream_sync(st);
    P.rstart = rstart_host.get(P.R);
    parse_rules(blob, nbytes, &P);
    host_chain = true;
  };
  DBuf rstart(P.R * 4 + 4, st);
  // flags read back once after the unpack: [0] first rule with a symbol past
  // the rules, [1] long bodies queued, [2] the chunked chain parse failed
  DBuf uflags(16, st);
  GT_CUDA(cudaMemsetAsync(uflags.p, 0, 16, st));
  bool chain_speculative = false;  // the chunked parse's check is read with the unpack's
  auto word_chain = [&](u64 n, int K) {  // the word-level doubling (and its check)
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
    return b == 0;
  };
  auto chain_error = [&]() {  // malformed: reproduce the reference's error
    need_host_chain();
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
  };
  {
    const u64 n = nsec;
    const int K = bitlen(P.R - 1);  // J_0 .. J_{K-1}
    bool ok = n >= 1 && n < 0xFFFFFFFFull && (nbytes - P.rules_pos) % 4 == 0;
    bool done = false;
    static const bool words_only = getenv("GT_CHAIN_WORDS") != nullptr;  // diagnostics: skip the chunked form
    const u64 p1 = ok ? 1 + (u64)rd32(blob + P.rules_pos) : 0;  // the first record after the root
    if (ok && !words_only && P.R >= 2 && p1 < n && n >= P.R) {
      const u64 nch = (n - p1 + kChunkB - 1) / kChunkB, S = nch * kWin + 1;
      // level tables: level 0 from the chunk walks, then one per 32x fewer
      // chunks up to <= 32 (sizes summed into one carve)
      std::vector<u64> nk{nch};
      while (nk.back() > 32) nk.push_back((nk.back() + 31) / 32);
      const int NL = (int)nk.size();  // levels 0 .. NL-1; NL-1 is the top
      std::vector<size_t> sz;
      for (int k = 0; k < NL; k++) {
        const u64 st_k = (k ? nk[k] * 32 : S) * 4;
        sz.push_back(st_k);  // nx_k
        sz.push_back(st_k);  // ct_k
        sz.push_back(nk[k] * 4 + 4);  // entry_k
        sz.push_back(nk[k] * 4 + 4);  // base_k
        if (k + 1 < NL) {
          sz.push_back(nk[k + 1] * 32 * 32 * 4);  // path_s_k
          sz.push_back(nk[k + 1] * 32 * 32 * 4);  // path_c_k
        }
      }
      sz.push_back(4);                                 // bad
      sz.push_back(nch * kWin * kMaskW * 4);           // masks
      std::vector<size_t> off(sz.size());
      size_t tot = 0;
      for (size_t i = 0; i < sz.size(); i++) {
        off[i] = tot;
        tot += (sz[i] + 255) & ~(size_t)255;
      }
      DBuf blk(tot, st);
      int ix = 0;
      auto take = [&]() { return reinterpret_cast<u32*>(blk.as<char>() + off[ix++]); };
      std::vector<u32*> nxk(NL), ctk(NL), enk(NL), bak(NL), psk(NL, nullptr), pck(NL, nullptr);
      for (int k = 0; k < NL; k++) {
        nxk[k] = take();
        ctk[k] = take();
        enk[k] = take();
        bak[k] = take();
        if (k + 1 < NL) {
          psk[k] = take();
          pck[k] = take();
        }
      }
      u32* badp = take();
      u32* maskp = take();
      const DPtr entry{enk[0]}, base{bak[0]}, bad{badp}, mask{maskp};
      u64 c_done = 0;
      auto tables_to_here = [&]() {  // the chunks complete in the re-aligned words
        const u64 c_new = w_done >= n ? nch : (w_done > p1 ? (w_done - p1) / kChunkB : 0);
        if (c_new > c_done)
          GT_KLAUNCH("k_chunk_tables", k_chunk_tables, grid_for((c_new - c_done) * 32, kTabWarps * 32),
                     kTabWarps * 32, st, raw.as<u32>(), n, p1, nch, c_done, c_new, nxk[0], ctk[0], mask.as<u32>());
        c_done = std::max(c_done, c_new);
      };
      tables_to_here();
      while (arrive_piece()) tables_to_here();
      arrive_all();
      tables_to_here();
      GT_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
      for (int k = 0; k + 1 < NL; k++) {
        const u64 ng = nk[k + 1];
        GT_KLAUNCH("k_chain_up", k_chain_up, (unsigned)((ng + kChainWarps - 1) / kChainWarps), kChainWarps * 32, st,
                   nxk[k], ctk[k], nk[k], nxk[k + 1], ctk[k + 1], psk[k], pck[k]);
      }
      GT_KLAUNCH("k_chain_top", k_chain_top, 1, 32, st, nxk[NL - 1], ctk[NL - 1], nk[NL - 1], P.R, enk[NL - 1],
                 bak[NL - 1], badp);
      for (int k = NL - 2; k >= 0; k--)
        LAUNCH(k_chain_down, nk[k], psk[k], pck[k], enk[k + 1], bak[k + 1], nk[k], enk[k], bak[k], badp);
      LAUNCH(k_chunk_starts, nch * 32, p1, nch, P.R, entry.as<u32>(), base.as<u32>(), mask.as<u32>(),
             rstart.as<u32>());
      // the check travels with the unpack's flags (no host round trip here):
      // the unpack runs on these starts and is redone if they were no chain
      GT_CUDA(cudaMemcpyAsync(uflags.as<u32>() + 2, badp, 4, cudaMemcpyDeviceToDevice, st));
      done = chain_speculative = true;
    }
    arrive_all();  // (a no-op after the chunked path)
    if (ok && !done) ok = word_chain(n, K);
    if (ok) {
      P.E = n - P.R;
      P.Rp = P.R;
      P.trailing = 0;
    } else {
      chain_error();
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
  DBuf& owner = d->pos_owner;
  owner.alloc(E * 4 + 4, st);
  DBuf longq(R * 4 + 4, st);
  d->body.alloc(E * 4 + 4, st);
  d->boff.alloc((R + 1) * 8, st);
  u32 uf[3] = {0, 0, 0};
  auto unpack = [&]() {
    if (host_chain) GT_CUDA(cudaMemcpyAsync(rstart.p, P.rstart, R * 4, cudaMemcpyHostToDevice, st));
    LAUNCH(k_boff, R + 1, rstart.as<u32>(), R, E, d->boff.as<u64>());
    GT_CUDA(cudaMemsetAsync(uflags.p, 0xFF, 4, st));
    GT_CUDA(cudaMemsetAsync(uflags.as<u32>() + 1, 0, 4, st));
    LAUNCH(k_unpack_rules, R, raw.as<u32>(), rstart.as<u32>(), R, nraw, d->body.as<u32>(), owner.as<u32>(),
           limit, uflags.as<u32>(), longq.as<u32>(), uflags.as<u32>() + 1);
    GT_KLAUNCH("k_unpack_long", k_unpack_long, grid_for(nraw, 256), 256, st, raw.as<u32>(), rstart.as<u32>(), R,
               nraw, longq.as<u32>(), uflags.as<u32>() + 1, d->body.as<u32>(), owner.as<u32>(), limit,
               uflags.as<u32>());
    d2h(uf, uflags.p, 3, st);
  };
  unpack();
  if (chain_speculative) {
    if (uf[2]) {  // the chunked parse met a record of 32+ words (or a malformed section)
      GT_CUDA(cudaMemsetAsync(uflags.as<u32>() + 2, 0, 4, st));
      if (!word_chain(nsec, bitlen(P.R - 1))) chain_error();
      unpack();
    } else {
      d->load_flags |= 1;
    }
  }
  longq.release();
  rstart.release();
  const u32 bad_rule = uf[0];
  if (bad_rule != 0xFFFFFFFFu) {
    need_host_chain();
    host_range_check(blob, P, bad_rule + 1);
  }
  ph.mark("upload+unpack");

  // ---- own / sub CSR: per-rule sort + RLE (csr_build.cu); the global
  // (rule, symbol) sort below remains for sections beyond 2^31 symbols
  const int SB = std::max(1, bitlen(limit - 1));
  DBuf own_rule, sub_rule;
  static const bool csr_sort = getenv("GT_CSR_SORT") != nullptr;  // diagnostics: the global-sort form
  const bool fused = !csr_sort && E < (1ull << 31) && SB + std::max(1, bitlen(R - 1)) <= 64;
  if (fused) {
    build_rule_pairs(d, owner.as<u32>(), own_rule, sub_rule, st);
  } else {
    // ---- (rule, symbol) sort + RLE -> own / sub CSR ----------------------
    // bodies are contiguous per rule, so the (rule, symbol) order is a
    // segmented sort of the body by symbol (one pass for the short bodies);
    // a 64-bit global radix sort of (rule << SB | symbol) beyond 2^31 symbols
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
    own_rule.alloc(Eo * 4 + 4, st);
    d->own_ids.alloc(Eo * 4 + 4, st);
    d->own_freqs.alloc(Eo * 4 + 4, st);
    LAUNCH(k_gather3, Eo, selO.as<u32>(), Eo, pr_rule.as<u32>(), pr_sym.as<u32>(), pr_cnt.as<u32>(),
           own_rule.as<u32>(), d->own_ids.as<u32>(), d->own_freqs.as<u32>());
    sub_rule.alloc(Es * 4 + 4, st);
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
  }
  const u64 Eo = d->E_own, Es = d->E_sub;
  ph.mark("own/sub CSR");

  // ---- word-major transpose of the own pairs (no host sync: side stream) ----
  cudaStream_t s_own = stream_acquire(device);
  struct StreamGuard {
    cudaStream_t s, main;
    DeviceDag* d;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      rebind_stream(main, {&d->ow_word, &d->ow_rule, &d->ow_freq, &d->ow_off});
      stream_release(d->device, s);
    }
  } own_guard{s_own, st, d};
  // ---- in-degrees straight from the sub pairs ------------------------------
  // (no parent sort on the critical path: the top-down edge lists are
  // scattered from the sub pairs below, and dag.py's parent CSR and
  // num_in_edge are built on first use, ensure_parents)
  if (!fused) {  // (the per-rule pass produced them)
    d->own_tok.alloc(R * 8, st);
    d->num_out.alloc(R * 8, st);
    GT_CUDA(cudaMemsetAsync(d->own_tok.p, 0, R * 8, st));
    GT_CUDA(cudaMemsetAsync(d->num_out.p, 0, R * 8, st));
    LAUNCH(k_seg_sum_sorted, Eo, own_rule.as<u32>(), Eo, ValU32{d->own_freqs.as<u32>()}, d->own_tok.as<u64>());
    LAUNCH(k_seg_sum_sorted, Es, sub_rule.as<u32>(), Es, ValU32{d->sub_freqs.as<u32>()}, d->num_out.as<u64>());
  }
  DBuf rem_td(R * 4 + 4, st), rootp(R + 1, st), indeg(R * 4 + 4, st);
  GT_CUDA(cudaMemsetAsync(rem_td.p, 0, R * 4, st));
  GT_CUDA(cudaMemsetAsync(rootp.p, 0, R, st));
  LAUNCH(k_in_degrees, Es, sub_rule.as<u32>(), d->sub_ids.as<u32>(), Es, rem_td.as<u32>(), rootp.as<uint8_t>());
  GT_CUDA(cudaMemcpyAsync(indeg.p, rem_td.p, R * 4, cudaMemcpyDeviceToDevice, st));  // the layering consumes rem_td
  ph.mark("in-degrees");

  // ---- top-down layering ---------------------------------------------------
  DBuf bm(std::max<u64>(((R + 31) / 32) * 8 + 8, R * 4 + 4), st);  // two frontier bitmaps, or delta[1] of k_kahn3
  DBuf kdelta;  // k_kahn3's delta arrays in the global-count mode
  d->bu_level.alloc(R * 4, st);
  d->td_level.alloc(R * 4, st);
  GT_CUDA(cudaMemsetAsync(d->bu_level.p, 0, R * 4, st));
  GT_CUDA(cudaMemsetAsync(d->td_level.p, 0, R * 4, st));
  // persistent top-down Kahn layering (doubles as the cycle check, carries
  // reachability): one cooperative launch
  const u64 ntask_max = Es / kChunk + R + 1;
  DBuf tasks(ntask_max * 8, st), ctl_b(sizeof(KahnCtl), st);
  KahnCtl* ctl = ctl_b.as<KahnCtl>();
  DBuf reach(R, st);
  bool kahn_checks_fused = false;  // k_kahn3 computes the reachability / root-cycle checks itself
  auto kahn = [&](DBuf& rem, const DBuf& off, const DBuf& ids, DBuf& lvl) {
    const u64 nwords = (R + 31) / 32;
    int nsm = 148;
    GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    // GT_KAHN=1|2|3 (diagnostics) forces the dependent-chain, batched-bitmap
    // or owner-scan kernel; by default owner-scan when a warp's share of the
    // sub CSR fits its shared memory, else batched-bitmap
    static const int forced = getenv("GT_KAHN") ? atoi(getenv("GT_KAHN")) : 0;
    const u64 nwarps3 = (u64)nsm * (kKahnBlock / 32), M3 = (nwords + nwarps3 - 1) / nwarps3;
    const bool fits3 = kK3List + 64 * M3 + 1 + 2 * ((Es + nwarps3 - 1) / nwarps3) <= kK3WarpWords;
    // mode 4 (diagnostics): owner-scan with the counts in global memory —
    // measured slower than the batched bitmap on C5 (235 vs 138 us per
    // layer: each warp scans ~120 counter words per layer in dependent waves)
    const int mode = forced >= 1 && forced <= 4 ? forced : (fits3 ? 3 : 2);
    GT_CUDA(cudaMemsetAsync(ctl, 0, sizeof(KahnCtl), st));
    // reachability starts at the rules the root references
    GT_CUDA(cudaMemcpyAsync(reach.p, rootp.p, R, cudaMemcpyDeviceToDevice, st));
    uint8_t* rc = reach.as<uint8_t>();
    const u64* o = off.as<u64>();
    const u32* ii = ids.as<u32>();
    u32* rm = rem.as<u32>();
    u32* lv = lvl.as<u32>();
    u64 maxl = R + 2;
    if (mode >= 3) {
      kahn_checks_fused = true;
      static bool attr = false;
      const size_t smem = (size_t)32 * kK3WarpWords * 4;
      u32* gd0 = nullptr;
      if (mode == 4 || !fits3) {
        kdelta.alloc(R * 8 + 8, st);
        GT_CUDA(cudaMemsetAsync(kdelta.p, 0, R * 8 + 8, st));
        gd0 = kdelta.as<u32>();
      }
      if (!attr) {
        GT_CUDA(cudaFuncSetAttribute(k_kahn3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
      }
      u64 Rv = R;
      // delta[1]: the frontier bitmaps' space (R words, see bm) or, in the
      // global-count mode, the second half of kdelta
      u32* d1 = gd0 ? gd0 + R + 1 : bm.as<u32>();
      void* args[] = {(void*)&ctl, (void*)&o,  (void*)&ii, (void*)&Rv,  (void*)&rm,
                      (void*)&d1,  (void*)&gd0, (void*)&lv, (void*)&rc, (void*)&maxl};
      ProfScope ps_("k_kahn<td>", st);
      GT_CUDA(cudaLaunchCooperativeKernel((const void*)k_kahn3, dim3((unsigned)nsm), dim3(kKahnBlock), args, smem, st));
      g_launches++;
      return;
    }
    GT_CUDA(cudaMemsetAsync(bm.p, 0, 2 * nwords * 4, st));
    u32* b0 = bm.as<u32>();
    u32* b1 = b0 + nwords;
    LAUNCH(k_kahn_first, R, rem.as<u32>(), R, b1, ctl);  // layer 1 reads b1
    const bool v1 = mode == 1;
    const void* kfn = v1 ? (const void*)k_kahn : (const void*)k_kahn2;
    const size_t smem = v1 ? 0 : kK2Smem;
    static int per_sm[2] = {-1, -1};
    if (per_sm[v1] < 0) {
      if (!v1) GT_CUDA(cudaFuncSetAttribute(k_kahn2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kK2Smem));
      GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[v1], kfn, kKahnBlock, smem));
      per_sm[v1] = std::max(per_sm[v1], 1);
    }
    uint2* tk = tasks.as<uint2>();
    u64 nw_ = nwords;
    void* args[] = {(void*)&ctl, (void*)&b0, (void*)&b1, (void*)&nw_, (void*)&o, (void*)&ii, (void*)&rm,
                    (void*)&lv, (void*)&rc, (void*)&tk, (void*)&maxl};
    ProfScope ps_("k_kahn<td>", st);
    GT_CUDA(cudaLaunchCooperativeKernel(kfn, dim3((unsigned)(nsm * per_sm[v1])), dim3(kKahnBlock), args, smem, st));
    g_launches++;
  };
  // top-down Kahn layering: the frontier never reaches a rule on (or below)
  // a reference cycle, so an incomplete layering is the cycle check
  // (grammar.py:127-161 order: cycles before unreachable rules, dag.py:173-184)
  u64 processed = 0;
  ph.mark("layering setup");
  kahn(rem_td, d->sub_off, d->sub_ids, d->td_level);
  ph.mark("layering kernel");
  // the word-major own transpose on the side stream, queued behind the
  // layering (which fills every SM: side kernels queued before it only
  // delay its start) so it overlaps the host check and the edge lists below
  {
    cudaEvent_t ev;
    GT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    GT_CUDA(cudaEventRecord(ev, st));
    GT_CUDA(cudaStreamWaitEvent(s_own, ev, 0));
    cudaEventDestroy(ev);
  }
    {
    cudaStream_t st = s_own;
    // (rule, freq) travel with the word keys through the radix sort: no
    // permutation gather afterwards
    DBuf v1(Eo * 8 + 8, st), v2(Eo * 8 + 8, st);
    d->ow_word.alloc(Eo * 4 + 4, st);
    d->ow_rule.alloc(Eo * 4 + 4, st);
    d->ow_freq.alloc(Eo * 4 + 4, st);
    d->ow_off.alloc((nw + 1) * 8, st);
    LAUNCH(k_pack2, Eo, own_rule.as<u32>(), d->own_freqs.as<u32>(), Eo, v1.as<u64>());
    sort_pairs_u32_u64(d->own_ids.as<u32>(), d->ow_word.as<u32>(), v1.as<u64>(), v2.as<u64>(), Eo,
                       std::max(1, bitlen(nw ? nw - 1 : 0)), st);
    LAUNCH(k_unpack2, Eo, v2.as<u64>(), Eo, d->ow_rule.as<u32>(), d->ow_freq.as<u32>());
    if (Eo * 4 >= nw)  // dense keys: one coalesced pass; sparse: a search per row
      LAUNCH(k_csr_offsets_lin, Eo + 1, d->ow_word.as<u32>(), Eo, nw, d->ow_off.as<u64>());
    else
      LAUNCH(k_csr_offsets, nw + 1, d->ow_word.as<u32>(), Eo, nw, d->ow_off.as<u64>());
  }

  // every rule but the root must be layered, and no reachable rule (nor the
  // root itself) may reference the root: either way there is a cycle; then
  // the first unreachable rule.  One host round trip for all three checks.
  static thread_local KahnCtl* hp = nullptr;  // pinned: a pageable read-back is staged by the driver
  if (!hp) GT_CUDA(cudaMallocHost(&hp, sizeof(KahnCtl)));
  KahnCtl& h = *hp;
  u32 chk[2];
  {
    DBuf cd(8, st);
    if (!kahn_checks_fused) {
      GT_CUDA(cudaMemsetAsync(cd.p, 0, 4, st));
      GT_CUDA(cudaMemsetAsync(cd.as<u32>() + 1, 0xFF, 4, st));
      LAUNCH(k_root_cycle2, Es, sub_rule.as<u32>(), d->sub_ids.as<u32>(), Es, reach.as<uint8_t>(), cd.as<u32>());
      LAUNCH(k_first_unreached, R, reach.as<uint8_t>(), R, cd.as<u32>() + 1);
      GT_CUDA(cudaMemcpyAsync(chk, cd.p, 8, cudaMemcpyDeviceToHost, st));
    }
    GT_CUDA(cudaMemcpyAsync(&h, ctl, sizeof h, cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    if (kahn_checks_fused) {
      chk[0] = h.root_cycle;
      chk[1] = h.first_unreached;
    }
  }
  processed = h.processed;
  const int ntd = (int)h.layers;
  if (trace2() && ntd > 0 && h.t[1]) {
    if (h.t[0]) fprintf(stderr, "[gt_open] kahn prologue %.1f us\n", (h.t[1] - h.t[0]) / 1e3);
    fprintf(stderr, "[gt_open] kahn layers (us):");
    for (int L = 1; L <= ntd && L + 1 < 64; L++) fprintf(stderr, " %.1f", (h.t[L + 1] - h.t[L]) / 1e3);
    fprintf(stderr, "\n");
  }
  if (processed + 1 < R || chk[0]) {
    need_host_chain();
    cycle_message(blob, P);
  }
  if (chk[1] != 0xFFFFFFFFu) fail(GT_E_CORRUPTION, "rule %u is not reachable from the root", chk[1]);
  ph.mark("top-down layering");
  rem_td.release();
  bm.release();
  kdelta.release();

  // ---- level-ordered edge lists (radix sort is stable: within a level the
  // edges keep (child, parent) resp. (rule, child) order) -------------------
  // host values read back once at the end of gt_open (one pinned staging
  // buffer: the te level offsets)
  static thread_local PinnedU64 stage_host;
  u64* stage = stage_host.get((u64)ntd + 3);
  // tid: rules numbered by top-down level (stable: ascending rule id within
  // a level, so a level's rows are contiguous and ordered like the reference)
  {
    const Carve cv(st, {R * 4, R * 4, R * 4, R * 4 + 4, R * 4 + 4, R * 4 + 4, ((u64)ntd + 3) * 8});
    u32 *iota = cv.at<u32>(0), *slev = cv.at<u32>(1), *ord = cv.at<u32>(2), *degt = cv.at<u32>(3),
        *incl = cv.at<u32>(4), *cur = cv.at<u32>(5);
    u64* ls = cv.at<u64>(6);
    d->tid.alloc(R * 4, st);
    if ((u64)ntd + 1 <= (u64)kLoBins && R < (1ull << 32)) {
      // levels 0..ntd: the stable counting sort gives ord, tid and the level starts
      const u64 nblk = std::min<u64>(1024, std::max<u64>(1, (R + 4095) / 4096));
      const u64 chunk = (R + nblk - 1) / nblk;
      const u32 nb = (u32)ntd + 1;
      DBuf lcb(nblk * nb * 4 + 4, st);
      u32* lcnt = lcb.as<u32>();
      GT_KLAUNCH("k_lo_count", k_lo_count, (unsigned)nblk, kLoBlock, st, d->td_level.as<u32>(), R, chunk, nb, lcnt);
      GT_KLAUNCH("k_lo_scan", k_lo_scan, 1, kLoBlock, st, lcnt, (u32)nblk, nb, R, ls);
      GT_KLAUNCH("k_lo_scatter", k_lo_scatter, (unsigned)nblk, kLoBlock, st, d->td_level.as<u32>(), R, chunk, nb,
                 (const u32*)lcnt, ord, d->tid.as<u32>());
    } else {
      LAUNCH(k_iota_u32, R, iota, R);
      sort_pairs_u32_u32(d->td_level.as<u32>(), slev, iota, ord, R, std::max(1, bitlen((u64)ntd)), st);
      LAUNCH(k_rank_of, R, ord, R, d->tid.as<u32>());
      // td: the non-root parent edges of every child, children in tid order
      LAUNCH(k_csr_offsets, (u64)ntd + 2, slev, R, (u64)ntd + 1, ls);
    }
    LAUNCH(k_map_u32, R, ord, R, indeg.as<u32>(), degt);
    inclusive_scan_u32(degt, incl, R, st);
    LAUNCH(k_cursor, R, degt, incl, R, cur);
    d->te_child.alloc(Es * 4 + 16, st);  // + 16: the TMA-staged level loop copies whole 16-byte words
    d->te_par.alloc(Es * 4 + 16, st);
    d->te_freq.alloc(Es * 4 + 16, st);
    {
      DBuf te(Es * 12 + 12, st);
      LAUNCH(k_te_scatter, Es, sub_rule.as<u32>(), d->sub_ids.as<u32>(), d->sub_freqs.as<u32>(), Es,
             d->tid.as<u32>(), cur, te.as<U3>());
      // (slots past the non-root edges stay unwritten: unpack only E_td)
      LAUNCH(k_unpack3_n, Es, te.as<U3>(), incl + (R - 1), d->te_child.as<u32>(), d->te_par.as<u32>(),
             d->te_freq.as<u32>());
    }
    d->te_off_dev.alloc(((u64)ntd + 3) * 8, st);
    LAUNCH(k_te_level_off, (u64)ntd + 3, ls, incl, degt, R, (u64)ntd, d->te_off_dev.as<u64>());
    GT_CUDA(cudaMemcpyAsync(stage, d->te_off_dev.p, ((u64)ntd + 3) * 8, cudaMemcpyDeviceToHost, st));
  }
  indeg.release();
  d->sub_rule = std::move(sub_rule);  // kept for the lazy builds (ensure_derived, ensure_parents)
  d->td.nl = ntd;
  ph.mark("level lists");

  join_root();
  raw.release();  // (the root side read the root body from it)
  ph.mark("root side joined");

  // the seeds' and the reduce's rule ids in tid numbering (after the own
  // transpose on the side stream)
  {
    cudaEvent_t ev;
    GT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    GT_CUDA(cudaEventRecord(ev, s_own));
    GT_CUDA(cudaStreamWaitEvent(st, ev, 0));
    cudaEventDestroy(ev);
    d->rs_rule_t.alloc(d->n_rs * 4 + 4, st);
    d->ow_rule_t.alloc(Eo * 4 + 4, st);
    if (d->n_rs) LAUNCH(k_map_u32, d->n_rs, d->rs_rule.as<u32>(), d->n_rs, d->tid.as<u32>(), d->rs_rule_t.as<u32>());
    if (Eo) LAUNCH(k_map_u32, Eo, d->ow_rule.as<u32>(), Eo, d->tid.as<u32>(), d->ow_rule_t.as<u32>());
  }

  stream_sync(st);
  stream_sync(s_own);
  own_rule.release();
  d->te_off.assign(stage, stage + ntd + 3);
  static const bool eager = getenv("GT_EAGER_DERIVED") != nullptr;  // diagnostics: derive at open
  if (eager) ensure_derived(d);
  ph.mark("finish");
  d->init_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// entries of (seg) lists inside [lo, lo + n)
__global__ void k_flag_seg_range(const u32* __restrict__ seg, u64 m, u32 lo, u32 n, uint8_t* f) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) f[i] = seg[i] - lo < n;
}

__global__ void k_gather4(const u32* __restrict__ idx, const u64* __restrict__ n_dev, const u32* a, const u32* b,
                          const u32* c, const u32* e, u32* oa, u32* ob, u32* oc, u32* oe) {
  const u64 n = *n_dev;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 j = idx[i];
    oa[i] = a[j];
    ob[i] = b[j];
    oc[i] = c[j];
    if (e) oe[i] = e[j];
  }
}

// gt_set_files: the owned file range, and the root occurrence lists cut to
// it (the whole-corpus lists are kept aside in d->full and restored when
// the range covers every file again)
void set_file_range(DeviceDag* d, u64 lo, u64 hi) {
  lo = std::min(lo, d->F);
  hi = std::min(hi, d->F);
  if (hi < lo) hi = lo;
  d->file_lo = lo;
  d->file_hi = hi;
  GT_CUDA(cudaSetDevice(d->device));
  cudaStream_t st = d->stream;
  auto& f = d->full;
  const bool whole = lo == 0 && hi == d->F;
  if (whole) {
    if (f.saved) {
      d->rs_rule = std::move(f.rs_rule), d->rs_rule_t = std::move(f.rs_rule_t), d->rs_seg = std::move(f.rs_seg);
      d->rs_cnt = std::move(f.rs_cnt), d->rs_off = std::move(f.rs_off);
      d->rw_word = std::move(f.rw_word), d->rw_seg = std::move(f.rw_seg), d->rw_cnt = std::move(f.rw_cnt);
      d->n_rs = f.n_rs, d->n_rw = f.n_rw;
      f.saved = false;
      refresh_contracted_seeds(d);
    }
    return;
  }
  if (!f.saved) {
    f.rs_rule = std::move(d->rs_rule), f.rs_rule_t = std::move(d->rs_rule_t), f.rs_seg = std::move(d->rs_seg);
    f.rs_cnt = std::move(d->rs_cnt), f.rs_off = std::move(d->rs_off);
    f.rw_word = std::move(d->rw_word), f.rw_seg = std::move(d->rw_seg), f.rw_cnt = std::move(d->rw_cnt);
    f.n_rs = d->n_rs, f.n_rw = d->n_rw;
    f.saved = true;
  }
  const u32 l32 = (u32)lo, n32 = (u32)(hi - lo);
  const u64 m = std::max(f.n_rs, f.n_rw);
  DBuf flag(m + 1, st), idx(m * 4 + 4, st), cnt(16, st);
  u64 h[2] = {0, 0};
  if (f.n_rs) {
    LAUNCH(k_flag_seg_range, f.n_rs, f.rs_seg.as<u32>(), f.n_rs, l32, n32, flag.as<uint8_t>());
    select_flagged_index(flag.as<uint8_t>(), idx.as<u32>(), cnt.as<u64>(), f.n_rs, st);
    GT_CUDA(cudaMemcpyAsync(&h[0], cnt.p, 8, cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    const u64 n = h[0];
    d->rs_rule.alloc(n * 4 + 4, st), d->rs_rule_t.alloc(n * 4 + 4, st), d->rs_seg.alloc(n * 4 + 4, st);
    d->rs_cnt.alloc(n * 4 + 4, st);
    LAUNCH(k_gather4, n, idx.as<u32>(), cnt.as<u64>(), f.rs_rule.as<u32>(), f.rs_seg.as<u32>(), f.rs_cnt.as<u32>(),
           f.rs_rule_t.as<u32>(), d->rs_rule.as<u32>(), d->rs_seg.as<u32>(), d->rs_cnt.as<u32>(),
           d->rs_rule_t.as<u32>());
    d->rs_off.alloc((d->R + 1) * 8, st);
    LAUNCH(k_csr_offsets, d->R + 1, d->rs_rule.as<u32>(), n, d->R, d->rs_off.as<u64>());
    d->n_rs = n;
  }
  if (f.n_rw) {
    LAUNCH(k_flag_seg_range, f.n_rw, f.rw_seg.as<u32>(), f.n_rw, l32, n32, flag.as<uint8_t>());
    select_flagged_index(flag.as<uint8_t>(), idx.as<u32>(), cnt.as<u64>() + 1, f.n_rw, st);
    GT_CUDA(cudaMemcpyAsync(&h[1], cnt.as<u64>() + 1, 8, cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    const u64 n = h[1];
    d->rw_word.alloc(n * 4 + 4, st), d->rw_seg.alloc(n * 4 + 4, st), d->rw_cnt.alloc(n * 4 + 4, st);
    LAUNCH(k_gather4, n, idx.as<u32>(), cnt.as<u64>() + 1, f.rw_word.as<u32>(), f.rw_seg.as<u32>(),
           f.rw_cnt.as<u32>(), (const u32*)nullptr, d->rw_word.as<u32>(), d->rw_seg.as<u32>(), d->rw_cnt.as<u32>(),
           (u32*)nullptr);
    d->n_rw = n;
  }
  refresh_contracted_seeds(d);
  stream_sync(st);
}

// ---------------------------------------------------------------------------
// Replication of a loaded DAG onto another device (the DAG is
// built once and broadcast to the other GPUs over NVLink instead of N host
// uploads and N device builds): every device array is copied peer-to-peer,
// the host-side level tables and scalars by value.  The copy keeps the
// source's file range; lazily built arrays travel if they exist.
// ---------------------------------------------------------------------------
void enable_peer(int a, int b) {
  if (a == b) return;
  static std::mutex mu;
  static bool done[64][64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (done[a & 63][b & 63]) return;
  done[a & 63][b & 63] = true;
  int ok = 0;
  GT_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
  if (!ok) return;
  int cur = 0;
  GT_CUDA(cudaGetDevice(&cur));
  GT_CUDA(cudaSetDevice(a));
  const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
  if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) GT_CUDA(e);
  cudaGetLastError();
  GT_CUDA(cudaSetDevice(cur));
}

void clone_device_dag(const DeviceDag& s, int device, DeviceDag* d) {
  auto t0 = std::chrono::steady_clock::now();
  GT_CUDA(cudaSetDevice(s.device));
  GT_CUDA(cudaStreamSynchronize(s.stream));  // the source is complete
  GT_CUDA(cudaSetDevice(device));
  d->device = device;
  if (!d->stream) d->stream = stream_acquire(device);
  cudaStream_t st = d->stream;
  reserve_pool(device, st);
  enable_peer(device, s.device);
  auto cp = [&](const DBuf& a, DBuf& b) {
    if (!a.p) return;
    b.alloc(a.bytes, st);
    GT_CUDA(cudaMemcpyPeerAsync(b.p, device, a.p, s.device, a.bytes, st));
  };
  const DBuf* src[] = {&s.body, &s.boff, &s.pos_owner, &s.root_seg, &s.own_ids, &s.own_freqs, &s.own_off,
                       &s.own_tok, &s.sub_ids, &s.sub_freqs, &s.sub_off, &s.par_ids, &s.par_freqs, &s.par_off,
                       &s.num_in, &s.num_out, &s.exp_len, &s.td_level, &s.bu_level, &s.seg_lo, &s.seg_hi,
                       &s.seg_tokens, &s.ow_word, &s.ow_rule, &s.ow_freq, &s.ow_off, &s.rs_rule, &s.rs_seg,
                       &s.rs_cnt, &s.rs_off, &s.rw_word, &s.rw_seg, &s.rw_cnt, &s.td.order, &s.td.off_dev,
                       &s.bu.order, &s.bu.off_dev, &s.tid, &s.rs_rule_t, &s.ow_rule_t, &s.te_child, &s.te_par,
                       &s.te_freq, &s.te_off_dev, &s.be_rule, &s.be_child, &s.be_freq, &s.be_off_dev, &s.sub_rule};
  DBuf* dst[] = {&d->body, &d->boff, &d->pos_owner, &d->root_seg, &d->own_ids, &d->own_freqs, &d->own_off,
                 &d->own_tok, &d->sub_ids, &d->sub_freqs, &d->sub_off, &d->par_ids, &d->par_freqs, &d->par_off,
                 &d->num_in, &d->num_out, &d->exp_len, &d->td_level, &d->bu_level, &d->seg_lo, &d->seg_hi,
                 &d->seg_tokens, &d->ow_word, &d->ow_rule, &d->ow_freq, &d->ow_off, &d->rs_rule, &d->rs_seg,
                 &d->rs_cnt, &d->rs_off, &d->rw_word, &d->rw_seg, &d->rw_cnt, &d->td.order, &d->td.off_dev,
                 &d->bu.order, &d->bu.off_dev, &d->tid, &d->rs_rule_t, &d->ow_rule_t, &d->te_child, &d->te_par,
                 &d->te_freq, &d->te_off_dev, &d->be_rule, &d->be_child, &d->be_freq, &d->be_off_dev, &d->sub_rule};
  static_assert(sizeof(src) / sizeof(src[0]) == sizeof(dst) / sizeof(dst[0]), "clone lists");
  for (size_t i = 0; i < sizeof(src) / sizeof(src[0]); i++) cp(*src[i], *dst[i]);
  if (s.full.saved) {  // the source is a shard: the whole-corpus lists travel too
    cp(s.full.rs_rule, d->full.rs_rule), cp(s.full.rs_rule_t, d->full.rs_rule_t), cp(s.full.rs_seg, d->full.rs_seg);
    cp(s.full.rs_cnt, d->full.rs_cnt), cp(s.full.rs_off, d->full.rs_off), cp(s.full.rw_word, d->full.rw_word);
    cp(s.full.rw_seg, d->full.rw_seg), cp(s.full.rw_cnt, d->full.rw_cnt);
    d->full.n_rs = s.full.n_rs, d->full.n_rw = s.full.n_rw, d->full.saved = true;
  }
  d->nw = s.nw, d->ns = s.ns, d->R = s.R, d->E = s.E, d->F = s.F, d->L0 = s.L0, d->W = s.W;
  d->file_lo = s.file_lo, d->file_hi = s.file_hi, d->depth = s.depth;
  d->E_own = s.E_own, d->E_sub = s.E_sub, d->n_rs = s.n_rs, d->n_rw = s.n_rw;
  d->td.off = s.td.off, d->td.heavy_off = s.td.heavy_off, d->td.nl = s.td.nl;
  d->bu.off = s.bu.off, d->bu.heavy_off = s.bu.heavy_off, d->bu.nl = s.bu.nl;
  d->te_off = s.te_off, d->be_off = s.be_off;
  d->derived = s.derived, d->load_flags = s.load_flags, d->max_file_tokens = s.max_file_tokens, d->cnt32 = s.cnt32;
  GT_CUDA(cudaStreamSynchronize(st));
  d->init_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

static std::mutex g_stream_mu;
static std::vector<cudaStream_t> g_stream_pool[64];

cudaStream_t stream_acquire(int device) {
  {
    std::lock_guard<std::mutex> lock(g_stream_mu);
    auto& v = g_stream_pool[device & 63];
    if (!v.empty()) {
      cudaStream_t s = v.back();
      v.pop_back();
      return s;
    }
  }
  cudaStream_t s = nullptr;
  GT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

void stream_release(int device, cudaStream_t s) {
  if (!s) return;
  std::lock_guard<std::mutex> lock(g_stream_mu);
  g_stream_pool[device & 63].push_back(s);
}

}  // namespace gt
