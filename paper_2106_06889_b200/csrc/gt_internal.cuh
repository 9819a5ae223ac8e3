// gt_internal.cuh — shared definitions of libgtadoc_b200 (host + device).
//
// Device data layout (all device arrays are 4-byte ids/freqs and 8-byte
// weights/counts; SURVEY.md §8(d) widths):
//   body      u32[E]      rule bodies, root first (grammar.py bodies)
//   boff      u64[R+1]    body offsets
//   own_*     CSR by rule of distinct (word, freq)      (dag.py own_ids/own_freqs)
//   sub_*     CSR by rule of distinct (child, freq)     (dag.py sub_ids/sub_freqs)
//   par_*     CSR by rule of (parent asc, freq)         (dag.py par_ids/par_freqs)
//   ow_*      own pairs transposed: sorted by (word, rule)  -> pull reduce
//   rs_*      root occurrences per (rule, segment) sorted by rule -> per-file seeds
//   rw_*      root word occurrences per (word, segment) sorted by word
//   te_*      (child, parent, freq) edges grouped by top-down level (engine.py round)
//   be_*      (rule, child, freq) edges grouped by bottom-up level (height) -> seq windows
//   bu_order  rules grouped by bottom-up level (height+1), built lazily
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <chrono>

#include <initializer_list>
#include <string>
#include <vector>

#include "../../include/gtadoc_b200.h"

typedef uint32_t u32;
typedef uint64_t u64;
typedef int64_t i64;

namespace gt {

// ---- errors ---------------------------------------------------------------

struct Error {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...);
void set_last_error(const std::string& s);

#define GT_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      ::gt::fail(GT_E_DEVICE, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_),  \
                 __FILE__, __LINE__, cudaGetErrorString(e_));                      \
  } while (0)

// ---- device buffers ---------------------------------------------------------

// Stream-ordered device allocation (cudaMallocAsync from the device mempool).
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  bool own = true;  // false: a view into memory held elsewhere (never freed here)
  DBuf() = default;
  static DBuf view(void* q, size_t n) {
    DBuf b;
    b.p = q;
    b.bytes = n;
    b.own = false;
    return b;
  }
  DBuf(size_t n, cudaStream_t st) { alloc(n, st); }
  void alloc(size_t n, cudaStream_t st);
  void release();
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      s = o.s;
      own = o.own;
      o.p = nullptr;
      o.bytes = 0;
      o.own = true;
    }
    return *this;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// One stream-ordered allocation carved into 256-byte aligned pieces: a
// scope's temporaries cost one cudaMallocAsync / cudaFreeAsync pair instead
// of one per buffer (each ~1.8 us of host time; small grammars are
// host-bound in gt_open).
struct Carve {
  DBuf buf;
  size_t off[24];
  int n = 0;
  Carve(cudaStream_t st, std::initializer_list<size_t> sizes) {
    size_t tot = 0;
    for (size_t sz : sizes) {
      off[n++] = tot;
      tot += (sz + 255) & ~(size_t)255;
    }
    buf.alloc(tot ? tot : 256, st);
  }
  template <class T>
  T* at(int i) const {
    return reinterpret_cast<T*>(static_cast<char*>(buf.p) + off[i]);
  }
};

// a non-owning view with DBuf's accessor (a carved piece used where a DBuf was)
struct DPtr {
  void* p;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// ---- the device DAG ---------------------------------------------------------

struct Levels {
  // rules grouped by level; within a level: light rules first, then heavy
  DBuf order;                  // u32[n]
  std::vector<u64> off;        // host: level L occupies [off[L], off[L+1]) (L=0..nl-1)
  std::vector<u64> heavy_off;  // host: first heavy rule of level L
  DBuf off_dev;                // device copy of off (persistent level loops)
  int nl = 0;
};

struct DeviceDag {
  int device = 0;
  cudaStream_t stream = nullptr;
  u64 nw = 0, ns = 0, R = 0, E = 0, F = 0, L0 = 0, W = 0;
  u64 file_lo = 0, file_hi = 0;  // owned file range (sharding)
  i64 depth = 0;
  DBuf body, boff;                     // u32[E], u64[R+1]
  DBuf pos_owner;                      // u32[E] rule of each body position
  DBuf root_seg;                       // u32[L0] segment of each root position
  DBuf own_ids, own_freqs, own_off;    // u32, u32, u64[R+1]
  DBuf own_tok;                        // u64[R]
  DBuf sub_ids, sub_freqs, sub_off;    // u32, u32, u64[R+1]
  DBuf par_ids, par_freqs, par_off;    // u32, u32, u64[R+1]
  DBuf num_in, num_out, exp_len;       // u64[R]
  DBuf td_level, bu_level;             // u32[R]
  DBuf seg_lo, seg_hi, seg_tokens;     // u64[F]
  DBuf ow_word, ow_rule, ow_freq;      // u32[E_own] sorted by (word, rule)
  DBuf ow_off;                         // u64[V+1]
  DBuf rs_rule, rs_seg, rs_cnt;        // root rule occurrences by (rule, seg)
  DBuf rs_off;                         // u64[R+1]
  DBuf rw_word, rw_seg, rw_cnt;        // root word occurrences by (word, seg)
  u64 E_own = 0, E_sub = 0, n_rs = 0, n_rw = 0;
  Levels td, bu;
  // level-ordered edge lists for the segmented gather-reduce (segreduce.cuh)
  //   te_*: non-root parent edges (child, parent, freq) by (td level, child, parent)
  //   be_*: child edges (rule, child, freq) by (bu level, rule, child)
  // top-down rows are indexed by `tid` (rules numbered by top-down level,
  // ascending rule id within a level: a level's rows are contiguous, so the
  // reductions of a level and the parent gathers of the next stay in L2);
  // te_child / te_par, rs_rule_t and ow_rule_t hold tids
  DBuf tid;                 // u32[R]: rule -> tid
  DBuf rs_rule_t, ow_rule_t;
  DBuf te_child, te_par, te_freq;
  std::vector<u64> te_off;  // host: td level L items [te_off[L], te_off[L+1])
  DBuf te_off_dev;          // device copy (persistent level loops)
  DBuf be_rule, be_child, be_freq;
  std::vector<u64> be_off;  // host: bu level L items [be_off[L], be_off[L+1])
  DBuf be_off_dev;
  // root occurrence lists of the whole corpus while a file-range shard is
  // set (gt_set_files keeps only the shard's entries in rs_* / rw_*, so its
  // seeds and root words cost O(shard), not O(corpus))
  struct RootLists {
    DBuf rs_rule, rs_rule_t, rs_seg, rs_cnt, rs_off, rw_word, rw_seg, rw_cnt;
    u64 n_rs = 0, n_rw = 0;
    bool saved = false;
  } full;
  DBuf sub_rule;       // u32[E_sub]: the rule of every sub pair (lazy builds)
  // the single-parent contraction of the top-down pass (contract.cu, built
  // lazily once the DAG serves repeated top-down runs): a rule with exactly
  // one non-root parent edge (p, f) and no root reference has w(r) = f·w(p),
  // so w(r) = M(r)·w(H(r)) for its nearest multi-parent ancestor H ("head").
  // Tid space: c_hd / c_ml / c_lvp = H (a tid), M and the contracted level
  // L' of every tid; c_tid maps tid -> tid' (heads by (L', tid), singles
  // last).  The pass then runs over the heads only: edges H(p) -> c with
  // frequency f·M(p), own pairs (word, tid'(H(r)), Σ f·M(r)) word-major.
  DBuf c_hd, c_ml, c_lvp;
  bool contracted = false;
  bool c_tried = false;  // built (or given up: a multiplier outgrew 32 bits)
  u32 runs = 0;          // public run calls served (gt_run / gt_run_many): the build policy
  u32 c_levels = 0;
  u64 c_R = 0;           // heads
  u64 c_n_own = 0;       // merged own pairs
  DBuf c_tid, c_te_child, c_te_par, c_te_freq, c_te_off_dev, c_ow_word, c_ow_src, c_ow_freq, c_rs_rule_t;
  std::vector<u64> c_te_off;
  // derived arrays (ensure_derived): no top-down word count / inverted
  // index reads them, so gt_open leaves them to the first task that does
  // (be lists, heights = bu_level, depth, exp_len, W, seg_tokens,
  // max_file_tokens, cnt32)
  bool derived = false;
  u64 load_flags = 0;  // gt_info.load_flags
  u64 max_file_tokens = 0;
  bool cnt32 = false;  // every file < 2^32 words: per-file rows / counts in u32 (GT_ROWS64=1: never)
  double init_ms = 0;
  // scratch kept across runs
  DBuf word_counts;  // u64[V] of the last global run
  DBuf step_cache;   // the fused word count + inverted index step's buffers (grow-only)
  u64 rows_clean = 0;             // leading u64 words of the step's rows left zeroed by the last step
  const void* rows_clean_at = nullptr;  // (at this step_cache block)

  u64 bytes_held() const {
    const DBuf* all[] = {&body, &boff, &pos_owner, &root_seg, &own_ids, &own_freqs, &own_off,
                         &own_tok, &sub_ids, &sub_freqs, &sub_off, &par_ids, &par_freqs, &par_off,
                         &num_in, &num_out, &exp_len, &td_level, &bu_level, &seg_lo, &seg_hi,
                         &seg_tokens, &ow_word, &ow_rule, &ow_freq, &ow_off, &rs_rule, &rs_seg,
                         &rs_cnt, &rs_off, &rw_word, &rw_seg, &rw_cnt, &td.order, &bu.order,
                         &tid, &rs_rule_t, &ow_rule_t, &te_child, &te_par, &te_freq, &be_rule, &be_child, &be_freq, &word_counts,
                         &te_off_dev, &be_off_dev, &sub_rule, &step_cache, &c_hd, &c_ml, &c_lvp, &c_tid, &c_te_child, &c_te_par, &c_te_freq, &c_te_off_dev, &c_ow_word, &c_ow_src, &c_ow_freq,
                         &c_rs_rule_t};
    u64 t = 0;
    for (const DBuf* b : all) t += b->own ? b->bytes : 0;  // (views into step_cache count once)
    return t;
  }
};

// The top-down pass's inputs: the whole DAG, or its single-parent
// contraction (heads only) when the loader built it and the caller can use
// head rows (word count / inverted index: every rule's own words are folded
// into its head's list with the multiplier)
struct TdLists {
  u64 rows = 0;  // rows of the pass (rules or heads)
  const u32* te_child = nullptr;
  const u32* te_par = nullptr;
  const u32* te_freq = nullptr;
  const u64* te_off_dev = nullptr;
  const std::vector<u64>* te_off = nullptr;
  int nl = 0;
  const u32* ow_word = nullptr;
  const u32* ow_src = nullptr;
  const u32* ow_freq = nullptr;
  u64 n_own = 0;
  const u32* rs_rule_t = nullptr;
  bool contracted = false;
};
// contract.cu: the pass's lists; `contract` asks for the heads-only lists,
// which are built during the DAG's second public run call (GT_CONTRACT=0:
// never, 2: on the first request)
TdLists td_lists(DeviceDag* d, bool contract);
void ensure_contracted(DeviceDag* d);
void refresh_contracted_seeds(DeviceDag* d);  // after the owned file range changed

// loader.cu
void build_device_dag(const uint8_t* blob, size_t n, int device, u64 file_lo, u64 file_hi,
                      DeviceDag* d);

// bottom-up rule lists by level (built on first use)
void ensure_bu_levels(DeviceDag* d);
void ensure_parents(DeviceDag* d);  // par_* and num_in (built on first request)
void ensure_derived(DeviceDag* d);  // see DeviceDag::derived
void set_file_range(DeviceDag* d, u64 lo, u64 hi);  // gt_set_files
// replicate a loaded DAG onto `device` (peer copies over NVLink)
void clone_device_dag(const DeviceDag& src, int device, DeviceDag* d);
void enable_peer(int a, int b);  // device a may read device b's memory (when supported)

// cub_ops.cu (plumbing around CUB device-wide primitives)
void sort_pairs_u64_u32(u64* keys_in, u64* keys_out, u32* vals_in, u32* vals_out, u64 n,
                        int end_bit, cudaStream_t s);
void sort_pairs_u32_u32(u32* keys_in, u32* keys_out, u32* vals_in, u32* vals_out, u64 n,
                        int end_bit, cudaStream_t s);
void sort_keys_u64(u64* keys_in, u64* keys_out, u64 n, int end_bit, cudaStream_t s);
void sort_keys_u32(const u32* keys_in, u32* keys_out, u64 n, int end_bit, cudaStream_t s);
void exclusive_scan_u64(const u64* in, u64* out, u64 n, cudaStream_t s);
void inclusive_scan_u32(const u32* in, u32* out, u64 n, cudaStream_t s);
// ordered compaction of indices i in [0,n) with flags[i] != 0; count -> d_count
void select_flagged_index(const uint8_t* flags, u32* out_idx, u64* d_count, u64 n, cudaStream_t s);
void select_nonzero_index(const void* v, bool v32, u32* out_idx, u64* d_count, u64 n, cudaStream_t s);
void select_nonzero_records(const void* v, bool v32, u64 V, u64 n, u32* id, u64* cnt, u32* file, u64* d_count,
                            cudaStream_t s);
void reduce_max_u64(const u64* in, u64* out, u64 n, cudaStream_t s);
// sort the keys of each segment [off[i], off[i+1]) independently (n < 2^31)
void sort_segments_u32(const u32* keys_in, u32* keys_out, u64 n, u64 nseg, const u64* off, cudaStream_t s);
struct U3 {
  u32 a, b, c;
};
void sort_pairs_u32_u64(u32* ki, u32* ko, u64* vi, u64* vo, u64 n, int end_bit, cudaStream_t s);
void sort_pairs_u32_u3(u32* ki, u32* ko, U3* vi, U3* vo, u64 n, int end_bit, cudaStream_t s);
void sort_segments_listed_u32(const u32* ki, u32* ko, u64 n, u64 nseg, const int* beg, const int* end,
                              cudaStream_t s);
struct DeviceDag;
void build_rule_pairs(DeviceDag* d, const u32* owner, DBuf& own_rule, DBuf& sub_rule, cudaStream_t st);
void sort_pairs_u64_u64(u64* keys_in, u64* keys_out, u64* vals_in, u64* vals_out, u64 n, int end_bit,
                        cudaStream_t s);
// runs of equal keys (sorted input) -> unique keys, sums, run count (device)
void reduce_by_key_u64(const u64* keys, const u64* vals, u64* ukeys, u64* sums, u64* d_nruns, u64 n,
                       cudaStream_t s);

// launch bookkeeping
extern thread_local u64 g_launches;

// Optional per-kernel timing (gt_profile): CUDA events around every launch on
// the launching stream; aggregated by kernel name in gt_profile_report.
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
struct Profiler {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get();
};
extern thread_local Profiler g_prof;
struct ProfScope {
  ProfRec rec{};
  cudaStream_t s = nullptr;
  bool on = false;
  ProfScope(const char* name, cudaStream_t st);
  ~ProfScope();
};

#define GT_KLAUNCH(name, kernel, grid, block, st, ...) \
  do {                                                 \
    ::gt::ProfScope ps_(name, st);                     \
    kernel<<<(grid), (block), 0, (st)>>>(__VA_ARGS__); \
    ::gt::g_launches++;                                \
  } while (0)

// Per-device pool of non-blocking streams: creating and destroying a stream
// costs ~100 us of host time (tools/api_cost.cu), more than a small grammar's
// whole traversal, so contexts and the loader's helper streams reuse them.
// A stream is released idle (synchronised) and may serve any later context.
cudaStream_t stream_acquire(int device);
void stream_release(int device, cudaStream_t s);

// host-side stream sync; under GT_TRACE=2 the time the calling thread spent
// waiting is accumulated (Phases prints it: wall - wait = host work)
struct SyncStats {
  double wait_ms = 0, alloc_ms = 0;
  int n = 0, nalloc = 0, nfree = 0;
  u64 launches0 = 0;
};
inline SyncStats& sync_stats() {
  static thread_local SyncStats s;
  return s;
}
inline void stream_sync(cudaStream_t s) {
  static const bool tr = getenv("GT_TRACE") && atoi(getenv("GT_TRACE")) == 2;
  if (!tr) {
    GT_CUDA(cudaStreamSynchronize(s));
    return;
  }
  auto a = std::chrono::steady_clock::now();
  GT_CUDA(cudaStreamSynchronize(s));
  sync_stats().wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  sync_stats().n++;
}

// GT_TRACE=1: synchronising phase timer on stderr (diagnostics only).
// GT_TRACE=2: non-intrusive timeline: at each mark the host time and a
// stream event are recorded without a sync; printed at destruction as
// (host ms, device ms) since construction — device > host means the GPU
// was the bottleneck up to that point, host >> device means it sat idle.
struct Phases {
  int mode;
  const char* tag;
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point t, t0;
  cudaEvent_t e0 = nullptr;
  struct Mark {
    const char* what;
    double host_ms;
    cudaEvent_t ev;
  };
  std::vector<Mark> marks;
  explicit Phases(const char* tg, cudaStream_t s = nullptr)
      : mode(getenv("GT_TRACE") ? atoi(getenv("GT_TRACE")) : 0), tag(tg), st(s),
        t(std::chrono::steady_clock::now()), t0(t) {
    if (mode == 2 && st) {
      cudaEventCreate(&e0);
      cudaEventRecord(e0, st);
    }
  }
  void bind(cudaStream_t s) {
    st = s;
    t0 = t = std::chrono::steady_clock::now();
    if (mode == 2 && !e0) {
      cudaEventCreate(&e0);
      cudaEventRecord(e0, st);
      sync_stats() = SyncStats{};
      sync_stats().launches0 = g_launches;
    }
  }
  void mark(const char* what) {
    if (!mode) return;
    auto n = std::chrono::steady_clock::now();
    if (mode == 2) {
      if (!st) return;
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      cudaEventRecord(ev, st);
      marks.push_back({what, std::chrono::duration<double, std::milli>(n - t0).count(), ev});
      return;
    }
    if (st) cudaStreamSynchronize(st);
    n = std::chrono::steady_clock::now();
    fprintf(stderr, "[%s] %-28s %9.3f ms\n", tag, what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
  ~Phases() {
    if (mode != 2 || !e0) return;
    cudaEventSynchronize(marks.empty() ? e0 : marks.back().ev);
    for (auto& m : marks) {
      float dm = 0;
      cudaEventElapsedTime(&dm, e0, m.ev);
      fprintf(stderr, "[%s] %-28s host %8.3f ms  device %8.3f ms\n", tag, m.what, m.host_ms, dm);
      cudaEventDestroy(m.ev);
    }
    fprintf(stderr, "[%s] host waited %.3f ms in %d syncs; %d allocs + %d frees took %.3f ms; %llu launches\n", tag,
            sync_stats().wait_ms, sync_stats().n, sync_stats().nalloc, sync_stats().nfree, sync_stats().alloc_ms,
            (unsigned long long)(g_launches - sync_stats().launches0));
    cudaEventDestroy(e0);
  }
};

inline int bitlen(u64 v) {
  int b = 0;
  while (v) {
    b++;
    v >>= 1;
  }
  return b;
}

inline unsigned grid_for(u64 n, unsigned block, unsigned max_blocks = 148u * 16u) {
  u64 g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (unsigned)g;
}

}  // namespace gt
