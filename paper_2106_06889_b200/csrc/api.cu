// api.cu — the C-ABI (include/gtadoc_b200.h) over the device DAG and kernels.
//
// gt_run mirrors tasks.py:171-185 run_task: strategy selection
// (engine.py:63-71, tasks.py:47-56 hooks), the traversal + reduce on the
// device, device-side result assembly in render order (tasks.py:122-168
// sorting rules), and one D2H copy of the compact arrays into pinned host
// memory owned by the gt_result.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "gt_internal.cuh"
#include "seq.cuh"
#include "sparse.cuh"
#include "bottomup.cuh"
#include "naive.cuh"
#include "word.cuh"

namespace gt {

static thread_local std::string t_err;

void set_last_error(const std::string& s) { t_err = s; }

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Error{code, buf};
}

// ---- per-kernel profiler -----------------------------------------------------
thread_local Profiler g_prof;

cudaEvent_t Profiler::get() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  GT_CUDA(cudaEventCreate(&e));
  return e;
}

ProfScope::ProfScope(const char* name, cudaStream_t st) : s(st), on(g_prof.on) {
  if (!on) return;
  rec.name = name;
  rec.a = g_prof.get();
  rec.b = g_prof.get();
  cudaEventRecord(rec.a, s);
}

ProfScope::~ProfScope() {
  if (!on) return;
  cudaEventRecord(rec.b, s);
  g_prof.recs.push_back(rec);
}

// ---- pinned host memory pool (results own blocks until gt_result_free) ----
namespace {
std::mutex g_pool_mu;
std::multimap<size_t, void*> g_pool;  // capacity -> block

size_t size_class(size_t n) {
  size_t c = 4096;
  while (c < n) c <<= 1;
  return c;
}

void* pinned_get(size_t n, size_t* cap) {
  size_t c = size_class(n);
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    auto it = g_pool.find(c);
    if (it != g_pool.end()) {
      void* p = it->second;
      g_pool.erase(it);
      *cap = c;
      return p;
    }
  }
  void* p = nullptr;
  GT_CUDA(cudaMallocHost(&p, c));
  *cap = c;
  return p;
}

void pinned_put(void* p, size_t cap) {
  std::lock_guard<std::mutex> g(g_pool_mu);
  g_pool.emplace(cap, p);
}
}  // namespace

}  // namespace gt

using namespace gt;

namespace gt {
// the shards' dense word counts summed on one device, every shard's vector
// read in place through peer memory (NVLink) when the devices differ
__global__ void k_sum_shards(const u64* const* __restrict__ srcs, int n, u64 V, u64* out) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < V; i += stride) {
    u64 t = 0;
    for (int k = 0; k < n; k++) t += __ldcg(reinterpret_cast<const unsigned long long*>(srcs[k]) + i);
    out[i] = t;
  }
}
}  // namespace gt

struct gt_ctx {
  DeviceDag d;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

struct gt_result {
  gt_view v{};
  std::vector<std::pair<void*, size_t>> blocks;
  ~gt_result() {
    for (auto& b : blocks) pinned_put(b.first, b.second);
  }
};

template <class F>
static int guard(F f) {
  try {
    f();
    return GT_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return GT_E_RESOURCE;
  }
}

extern "C" {

int gt_abi_version(void) { return GT_ABI_VERSION; }

const char* gt_last_error(void) { return t_err.c_str(); }

int gt_open(const uint8_t* gtdc, size_t nbytes, int device, uint64_t file_lo, uint64_t file_hi,
            gt_ctx** out) {
  *out = nullptr;
  gt_ctx* c = new gt_ctx();
  int st = guard([&] {
    build_device_dag(gtdc, nbytes, device, file_lo, file_hi, &c->d);
    for (auto& e : c->ev) GT_CUDA(cudaEventCreate(&e));
  });
  if (st != GT_OK) {
    gt_close(c);
    return st;
  }
  *out = c;
  return GT_OK;
}

int gt_info_get(const gt_ctx* c, gt_info* o) {
  memset(o, 0, sizeof *o);
  const int st = guard([&] { ensure_derived(const_cast<DeviceDag*>(&c->d)); });
  if (st != GT_OK) return st;
  const DeviceDag& d = c->d;
  o->num_words = d.nw;
  o->num_splitters = d.ns;
  o->num_rules = d.R;
  o->num_files = d.F;
  o->total_elements = d.E;
  o->root_len = d.L0;
  o->sub_pairs = d.E_sub;
  o->own_pairs = d.E_own;
  o->words = d.W;
  o->depth = d.depth;
  o->td_levels = d.td.nl;
  o->bu_levels = d.bu.nl > 0 ? d.bu.nl - 1 : 0;
  o->device_bytes = d.bytes_held();
  o->init_ms = d.init_ms;
  o->td_edges = d.te_off.empty() ? 0 : d.te_off.back();
  o->load_flags = d.load_flags;
  return GT_OK;
}

void gt_close(gt_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->d.device);
  // no host synchronisation: every device array is freed stream-ordered on
  // the context's stream (after any work still queued there), events may be
  // destroyed while pending, and the stream goes back to the pool for the
  // next gt_open, whose work queues behind those frees
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  cudaStream_t s = c->d.stream;
  const int dev = c->d.device;
  delete c;  // DBuf destructors free on the stream
  if (s) stream_release(dev, s);
}

}  // extern "C"

// GT_FORCE_SPARSE=1: per-file tasks take the sparse path at any F (diagnostics)
static bool force_sparse() {
  static const bool v = getenv("GT_FORCE_SPARSE") != nullptr;
  return v;
}

static int select_strategy(const DeviceDag& d, int task, int requested, int fsw) {
  if (requested == GT_TOPDOWN || requested == GT_BOTTOMUP) return requested;
  bool needs_file_info = task >= GT_INVERTEDINDEX;
  if (needs_file_info) return (i64)d.F > (i64)fsw ? GT_BOTTOMUP : GT_TOPDOWN;
  return GT_TOPDOWN;
}

template <class T>
static const T* pull(gt_result* r, const DBuf& b, u64 n, cudaStream_t st, u64* bytes) {
  if (!b.p) return nullptr;
  size_t cap;
  size_t nb = n * sizeof(T);
  void* h = pinned_get(nb ? nb : 8, &cap);
  r->blocks.push_back({h, cap});
  if (nb) GT_CUDA(cudaMemcpyAsync(h, b.p, nb, cudaMemcpyDeviceToHost, st));
  *bytes += nb;
  return (const T*)h;
}

// u64 -> u32 (the caller guarantees every value fits)
__global__ void k_narrow_u64(const u64* __restrict__ in, u64 n, u32* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = (u32)in[i];
}

// a u64 device array copied to the host as u32 (narrowed on the device; the
// temporary is freed stream-ordered after the copy)
static const uint32_t* pull_narrow(gt_result* r, const DBuf& b, u64 n, cudaStream_t st, u64* bytes) {
  if (!b.p) return nullptr;
  DBuf t(n * 4 + 4, st);
  if (n) GT_KLAUNCH("k_narrow_u64", k_narrow_u64, grid_for(n, 256), 256, st, b.as<u64>(), n, t.as<u32>());
  return pull<uint32_t>(r, t, n, st, bytes);
}

// u32 ids -> 1 / 2 bytes (the caller guarantees every id fits)
__global__ void k_narrow_ids(const u32* __restrict__ in, u64 n, int bytes, void* out) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (bytes == 1) static_cast<uint8_t*>(out)[i] = (uint8_t)in[i];
    else static_cast<unsigned short*>(out)[i] = (unsigned short)in[i];
  }
}

// enqueue the D2H copies of a result's compact arrays into pinned blocks the
// gt_result owns; returns the bytes.  count_bound: an upper bound of every
// count (0: unknown) — below 2^32 the counts travel as u32; id_bound: one
// past the largest record id (0: unknown) — ids below 2^8 / 2^16 travel 1 / 2
// bytes wide (ABI 3)
static u64 pull_records(gt_result* r, DevRecords& R, int task, int seq_len, int wbits, int strat, cudaStream_t st,
                        u64 count_bound = 0, u64 id_bound = 0) {
  u64 bytes = 0;
  gt_view& v = r->v;
  v.task = task;
  v.seq_len = seq_len;
  v.wbits = wbits;
  v.strategy = strat;
  v.n = R.n;
  v.n_groups = R.n_groups;
  const u64 l = (u64)seq_len;
  static const bool wide = getenv("GT_D2H_U64") != nullptr;  // diagnostics: always u64 counts / offsets
  if (!wide && R.group_off32_ok) v.group_off32 = pull<uint32_t>(r, R.group_off32, R.n_groups + 1, st, &bytes);
  else if (!wide && R.n < (1ull << 32)) v.group_off32 = pull_narrow(r, R.group_off, R.n_groups + 1, st, &bytes);
  else v.group_off = pull<uint64_t>(r, R.group_off, R.n_groups + 1, st, &bytes);
  v.group_id = pull<uint32_t>(r, R.group_id, R.n_groups, st, &bytes);
  v.group_key = pull<uint64_t>(r, R.group_key, R.n_groups, st, &bytes);
  v.group_gram = pull<uint32_t>(r, R.group_gram, R.n_groups * l, st, &bytes);
  v.id_bytes = 4;
  if (!wide && R.id_bytes < 4 && R.id_narrow.p) {  // written narrow by the producing kernel
    v.id_bytes = R.id_bytes;
    v.id_narrow = R.id_bytes == 1 ? (const void*)pull<uint8_t>(r, R.id_narrow, R.n, st, &bytes)
                                   : (const void*)pull<uint16_t>(r, R.id_narrow, R.n, st, &bytes);
  } else if (!wide && R.id.p && id_bound && id_bound <= 65536) {
    const int nb = id_bound <= 256 ? 1 : 2;
    DBuf t(R.n * nb + 8, st);
    if (R.n) GT_KLAUNCH("k_narrow_ids", k_narrow_ids, grid_for(R.n, 256), 256, st, R.id.as<u32>(), R.n, nb, t.p);
    v.id_bytes = nb;
    v.id_narrow = nb == 1 ? (const void*)pull<uint8_t>(r, t, R.n, st, &bytes)
                          : (const void*)pull<uint16_t>(r, t, R.n, st, &bytes);
  } else {
    v.id = pull<uint32_t>(r, R.id, R.n, st, &bytes);
  }
  v.key = pull<uint64_t>(r, R.key, R.n, st, &bytes);
  v.gram = pull<uint32_t>(r, R.gram, R.n * l, st, &bytes);
  if (!wide && R.count32_ok) v.count32 = pull<uint32_t>(r, R.count32, R.n, st, &bytes);
  else if (!wide && count_bound && count_bound < (1ull << 32)) v.count32 = pull_narrow(r, R.count, R.n, st, &bytes);
  else v.count = pull<uint64_t>(r, R.count, R.n, st, &bytes);
  v.d2h_bytes = bytes;
  return bytes;
}

// one past the largest record id of a task: files for the inverted indexes,
// words for the word-id records
static u64 id_bound(const DeviceDag& d, int task) {
  if (task == GT_INVERTEDINDEX || task == GT_RANKEDINVERTEDINDEX) return std::max<u64>(d.file_hi, 1);
  if (task == GT_WORDCOUNT || task == GT_SORT || task == GT_TERMVECTOR) return std::max<u64>(d.nw, 1);
  return 0;
}

// every count of a task's records is at most the longest owned file's words
// (per-file tasks) or W (corpus tasks); 0 = not known without the derived
// arrays
static u64 count_bound(const DeviceDag& d, int task) {
  if (!d.derived) return 0;
  if (task == GT_WORDCOUNT || task == GT_SORT) return std::max<u64>(d.W, 1);
  return std::max<u64>(d.max_file_tokens, 1);
}

static void finish(gt_ctx* c, gt_result* r, DevRecords& R, int task, int seq_len, int wbits,
                   int strat, std::chrono::steady_clock::time_point t0, u64 launches0) {
  cudaStream_t st = c->d.stream;
  pull_records(r, R, task, seq_len, wbits, strat, st, count_bound(c->d, task), id_bound(c->d, task));
  gt_view& v = r->v;
  GT_CUDA(cudaEventRecord(c->ev[2], st));
  GT_CUDA(cudaStreamSynchronize(st));
  float ms = 0, ms2 = 0;
  GT_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  GT_CUDA(cudaEventElapsedTime(&ms2, c->ev[1], c->ev[2]));
  v.device_ms = ms;
  v.d2h_ms = ms2;
  v.kernel_launches = g_launches - launches0;
  v.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

extern "C" {

// one count per public run call (gt_run, gt_run_many; a gt_run inside
// gt_run_many is the same call): the contraction is built on a DAG's second
static thread_local int g_run_depth = 0;
struct RunCount {
  RunCount(gt_ctx* c) {
    if (g_run_depth++ == 0 && c) c->d.runs++;
  }
  ~RunCount() { g_run_depth--; }
};

int gt_run(gt_ctx* c, int task, int seq_len, int strategy, int file_set_width, gt_result** out) {
  RunCount rc_(c);
  *out = nullptr;
  gt_result* r = new gt_result();
  int status = guard([&] {
    if (task < GT_WORDCOUNT || task > GT_RANKEDINVERTEDINDEX) fail(GT_E_USAGE, "unknown task %d", task);
    if (strategy < GT_AUTO || strategy > GT_BOTTOMUP) fail(GT_E_USAGE, "unknown strategy %d", strategy);
    if (task >= GT_SEQCOUNT && seq_len < 1) fail(GT_E_USAGE, "sequence length must be >= 1");
    DeviceDag& d = c->d;
    GT_CUDA(cudaSetDevice(d.device));
    cudaStream_t st = d.stream;
    // a top-down word count / inverted index reads no derived array
    if (!((task == GT_WORDCOUNT || task == GT_INVERTEDINDEX) && strategy != GT_BOTTOMUP)) ensure_derived(&d);
    auto t0 = std::chrono::steady_clock::now();
    u64 launches0 = g_launches;
    int strat = select_strategy(d, task, strategy, file_set_width);
    GT_CUDA(cudaEventRecord(c->ev[0], st));
    DevRecords R;
    int wbits = 0;
    const u32 Fo = (u32)(d.file_hi - d.file_lo);
    // an empty shard has no per-file output (word counts stay a zero vector)
    const bool empty_shard = Fo == 0 && task != GT_WORDCOUNT && task != GT_SORT;
    switch (empty_shard ? -1 : task) {
      case -1: {
        if (task == GT_TERMVECTOR || task == GT_SEQCOUNT || task == GT_RANKEDINVERTEDINDEX ||
            task == GT_INVERTEDINDEX) {
          R.group_off.alloc(8, st);
          GT_CUDA(cudaMemsetAsync(R.group_off.p, 0, 8, st));
        }
        if (task >= GT_SEQCOUNT) wbits = (u64)seq_len * std::max(1, bitlen(d.nw ? d.nw - 1 : 1)) <= 63 ? std::max(1, bitlen(d.nw ? d.nw - 1 : 1)) : 0;
        break;
      }
      case GT_WORDCOUNT:
      case GT_SORT: {
        // a forced bottom-up runs Alg. 2 with the pooled hash tables; auto
        // and top-down run Alg. 1 (engine.py:63-71 picks top-down here)
        if (strat == GT_BOTTOMUP && strategy == GT_BOTTOMUP && bu_word_counts(&d, d.word_counts, scratch_budget(&d))) {
          strat = GT_BOTTOMUP;
          assemble_counts(&d, d.word_counts.as<u64>(), d.nw, 0, task == GT_SORT, &R);
        } else if (td_word_records(&d, &R)) {  // small grammar: one launch
          strat = GT_TOPDOWN;
          if (task == GT_SORT) order_by_count(&d, &R, 0, nullptr);
        } else {
          td_word_counts(&d, d.word_counts);
          strat = GT_TOPDOWN;
          assemble_counts(&d, d.word_counts.as<u64>(), d.nw, 0, task == GT_SORT, &R);
        }
        break;
      }
      case GT_TERMVECTOR: {
        // the reference goes bottom-up for F > file_set_width; the device
        // equivalent is the presence-guided sparse per-file pass (sparse.cu)
        if (strategy == GT_BOTTOMUP && bu_file_tables(&d, GT_TERMVECTOR, &R, scratch_budget(&d))) {
          strat = GT_BOTTOMUP;
        } else if (strat == GT_BOTTOMUP || (u64)Fo * d.nw >= (1ull << 32) || force_sparse()) {
          sparse_term_vector(&d, &R);
          strat = GT_TOPDOWN_SPARSE;
        } else {
          DBuf cnt;
          bool c32 = false;
          td_file_counts(&d, cnt, &c32);
          assemble_counts(&d, cnt.p, d.nw, Fo, true, &R, c32);
          strat = GT_TOPDOWN;
        }
        break;
      }
      case GT_INVERTEDINDEX: {
        if (strategy == GT_BOTTOMUP && bu_file_tables(&d, GT_INVERTEDINDEX, &R, scratch_budget(&d))) {
          strat = GT_BOTTOMUP;
        } else if (td_presence_records(&d, &R)) {  // small grammar, <= 64 files: one launch
          strat = GT_TOPDOWN;
        } else {
          DBuf pres;
          u32 FW;
          td_file_presence(&d, pres, &FW);
          assemble_presence(&d, pres.as<u64>(), FW, &R);
          strat = GT_TOPDOWN;
        }
        break;
      }
      default: {
        // a forced bottom-up runs Alg. 2 for grams (pooled window tables);
        // auto for F > file_set_width takes the sparse top-down path
        const int mode = strategy == GT_BOTTOMUP ? GT_BOTTOMUP
                         : (strat == GT_BOTTOMUP || force_sparse()) ? GT_TOPDOWN_SPARSE : GT_TOPDOWN;
        strat = run_sequences(&d, task, seq_len, mode, &R, &wbits);
        break;
      }
    }
    GT_CUDA(cudaEventRecord(c->ev[1], st));
    finish(c, r, R, task, seq_len, wbits, strat, t0, launches0);
  });
  if (status != GT_OK) {
    delete r;
    return status;
  }
  *out = r;
  return GT_OK;
}

int gt_run_many(gt_ctx* c, const int* tasks, int ntasks, int seq_len, int strategy, int file_set_width,
                gt_result** outs) {
  RunCount rc_(c);
  for (int i = 0; i < ntasks; i++) outs[i] = nullptr;
  if (ntasks < 0) {
    set_last_error("gt_run_many: negative task count");
    return GT_E_USAGE;
  }
  // the fusable group: the first word count / sort with the first inverted
  // index (one top-down pass of {weight, presence} pairs, word.cu
  // td_wc_ii_records) when both would run top-down on one launch
  int iw = -1, ii = -1;
  for (int i = 0; i < ntasks; i++) {
    if (iw < 0 && (tasks[i] == GT_WORDCOUNT || tasks[i] == GT_SORT)) iw = i;
    if (ii < 0 && tasks[i] == GT_INVERTEDINDEX) ii = i;
  }
  const int fsw = file_set_width;
  for (int i = 0; i < ntasks; i++) {
    if (iw >= 0 && ii >= 0 && (i == iw || i == ii) && strategy != GT_BOTTOMUP &&
        select_strategy(c->d, GT_INVERTEDINDEX, strategy, fsw) == GT_TOPDOWN) {
      if (i != std::min(iw, ii)) continue;  // produced with its partner
      gt_result* rw = new gt_result();
      gt_result* ri = new gt_result();
      bool fused = false;
      int status = guard([&] {
        DeviceDag& d = c->d;
        GT_CUDA(cudaSetDevice(d.device));
        cudaStream_t st = d.stream;
        auto t0 = std::chrono::steady_clock::now();
        u64 launches0 = g_launches;
        GT_CUDA(cudaEventRecord(c->ev[0], st));
        DevRecords W, I;
        const bool sort = tasks[iw] == GT_SORT;
        if (!td_wc_ii_records(&d, &W, &I, sort ? nullptr : c->ev[1])) return;
        fused = true;
        if (sort) {
          ensure_derived(&d);
          order_by_count(&d, &W, 0, nullptr);
          GT_CUDA(cudaEventRecord(c->ev[1], st));
        }
        pull_records(rw, W, tasks[iw], seq_len, 0, GT_TOPDOWN, st, count_bound(d, tasks[iw]), id_bound(d, tasks[iw]));
        pull_records(ri, I, GT_INVERTEDINDEX, seq_len, 0, GT_TOPDOWN, st, 0, id_bound(d, GT_INVERTEDINDEX));
        GT_CUDA(cudaEventRecord(c->ev[2], st));
        GT_CUDA(cudaStreamSynchronize(st));
        float ms = 0, ms2 = 0;
        GT_CUDA(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
        GT_CUDA(cudaEventElapsedTime(&ms2, c->ev[1], c->ev[2]));
        const double tot = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        // the shared pass is charged to the word-count result
        rw->v.device_ms = ms;
        ri->v.device_ms = 0.0;
        rw->v.d2h_ms = ri->v.d2h_ms = ms2;
        rw->v.total_ms = ri->v.total_ms = tot;
        rw->v.kernel_launches = g_launches - launches0;
        ri->v.kernel_launches = 0;
      });
      if (status != GT_OK) {
        delete rw;
        delete ri;
        for (int j = 0; j < ntasks; j++) gt_result_free(outs[j]), outs[j] = nullptr;
        return status;
      }
      if (fused) {
        outs[iw] = rw;
        outs[ii] = ri;
        continue;
      }
      delete rw;
      delete ri;
      iw = ii = -1;  // not fusable on this grammar: run them one by one
    }
    if (outs[i]) continue;
    const int st = gt_run(c, tasks[i], seq_len, strategy, file_set_width, &outs[i]);
    if (st != GT_OK) {
      for (int j = 0; j < ntasks; j++) gt_result_free(outs[j]), outs[j] = nullptr;
      return st;
    }
  }
  return GT_OK;
}

int gt_run_naive(gt_ctx* c, int task, int seq_len, gt_result** out) {
  *out = nullptr;
  gt_result* r = new gt_result();
  int status = guard([&] {
    if (task < GT_WORDCOUNT || task > GT_RANKEDINVERTEDINDEX) fail(GT_E_USAGE, "unknown task %d", task);
    if (task >= GT_SEQCOUNT && seq_len < 1) fail(GT_E_USAGE, "sequence length must be >= 1");
    DeviceDag& d = c->d;
    GT_CUDA(cudaSetDevice(d.device));
    ensure_derived(&d);
    auto t0 = std::chrono::steady_clock::now();
    u64 launches0 = g_launches;
    GT_CUDA(cudaEventRecord(c->ev[0], d.stream));
    DevRecords R;
    int wbits = 0;
    naive_run(&d, task, seq_len, &R, &wbits);
    GT_CUDA(cudaEventRecord(c->ev[1], d.stream));
    finish(c, r, R, task, seq_len, wbits, GT_AUTO, t0, launches0);
  });
  if (status != GT_OK) {
    delete r;
    return status;
  }
  *out = r;
  return GT_OK;
}

int gt_count_tokens(gt_ctx* c, int task, int seq_len, const uint32_t* tokens, const uint64_t* file_off,
                    uint64_t nfiles, gt_result** out) {
  *out = nullptr;
  gt_result* r = new gt_result();
  int status = guard([&] {
    if (task < GT_WORDCOUNT || task > GT_RANKEDINVERTEDINDEX) fail(GT_E_USAGE, "unknown task %d", task);
    if (task >= GT_SEQCOUNT && seq_len < 1) fail(GT_E_USAGE, "sequence length must be >= 1");
    DeviceDag& d = c->d;
    if (nfiles != d.F) fail(GT_E_USAGE, "gt_count_tokens: %lu token streams for %lu files",
                            (unsigned long)nfiles, (unsigned long)d.F);
    for (u64 i = 0; i < file_off[nfiles]; i++)
      if (tokens[i] >= d.nw) fail(GT_E_USAGE, "gt_count_tokens: token %lu is word id %u >= %lu", (unsigned long)i,
                                  tokens[i], (unsigned long)d.nw);
    GT_CUDA(cudaSetDevice(d.device));
    ensure_derived(&d);
    auto t0 = std::chrono::steady_clock::now();
    u64 launches0 = g_launches;
    GT_CUDA(cudaEventRecord(c->ev[0], d.stream));
    DevRecords R;
    int wbits = 0;
    naive_run(&d, task, seq_len, &R, &wbits, tokens, file_off);
    GT_CUDA(cudaEventRecord(c->ev[1], d.stream));
    finish(c, r, R, task, seq_len, wbits, GT_AUTO, t0, launches0);
  });
  if (status != GT_OK) {
    delete r;
    return status;
  }
  *out = r;
  return GT_OK;
}

int gt_set_files(gt_ctx* c, uint64_t file_lo, uint64_t file_hi) {
  return guard([&] {
    DeviceDag& d = c->d;
    if (file_lo > file_hi) fail(GT_E_USAGE, "file range [%lu, %lu) is empty-reversed", (unsigned long)file_lo, (unsigned long)file_hi);
    set_file_range(&d, file_lo, file_hi);
  });
}

int gt_clone(const gt_ctx* src, int device, gt_ctx** out) {
  *out = nullptr;
  gt_ctx* c = new gt_ctx();
  int st = guard([&] {
    int ndev = 0;
    GT_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) fail(GT_E_USAGE, "gt_clone: no device %d (%d visible)", device, ndev);
    clone_device_dag(src->d, device, &c->d);
    for (auto& e : c->ev) GT_CUDA(cudaEventCreate(&e));
  });
  if (st != GT_OK) {
    gt_close(c);
    return st;
  }
  *out = c;
  return GT_OK;
}

int gt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int gt_sum_word_counts(gt_ctx* dst, gt_ctx* const* srcs, int n) {
  return guard([&] {
    if (n < 1) fail(GT_E_USAGE, "gt_sum_word_counts: no shards");
    DeviceDag& d = dst->d;
    const u64 V = d.nw;
    for (int k = 0; k < n; k++) {
      const DeviceDag& s = srcs[k]->d;
      if (s.nw != V) fail(GT_E_USAGE, "gt_sum_word_counts: shard %d has %lu words, not %lu", k,
                          (unsigned long)s.nw, (unsigned long)V);
      if (!s.word_counts.p) fail(GT_E_USAGE, "gt_sum_word_counts: shard %d has no word counts (run WORDCOUNT first)", k);
      GT_CUDA(cudaSetDevice(s.device));
      GT_CUDA(cudaStreamSynchronize(s.stream));
    }
    GT_CUDA(cudaSetDevice(d.device));
    cudaStream_t st = d.stream;
    std::vector<const u64*> ptrs(n);
    std::vector<DBuf> staged;  // shards whose memory dst's device cannot read
    staged.reserve(n);
    for (int k = 0; k < n; k++) {
      const DeviceDag& s = srcs[k]->d;
      int ok = s.device == d.device;
      if (!ok) {
        enable_peer(d.device, s.device);
        GT_CUDA(cudaDeviceCanAccessPeer(&ok, d.device, s.device));
      }
      if (ok) {
        ptrs[k] = s.word_counts.as<u64>();
      } else {
        staged.emplace_back(V * 8 + 8, st);
        GT_CUDA(cudaMemcpyPeerAsync(staged.back().p, d.device, s.word_counts.p, s.device, V * 8, st));
        ptrs[k] = staged.back().as<u64>();
      }
    }
    DBuf dp((u64)n * 8, st), total(V * 8 + 8, st);
    GT_CUDA(cudaMemcpyAsync(dp.p, ptrs.data(), (u64)n * 8, cudaMemcpyHostToDevice, st));
    GT_KLAUNCH("k_sum_shards", k_sum_shards, grid_for(V, 256), 256, st, dp.as<const u64*>(), n, V, total.as<u64>());
    GT_CUDA(cudaStreamSynchronize(st));
    d.word_counts = std::move(total);
  });
}

int gt_assemble_counts(gt_ctx* c, int task, const uint64_t* dev_counts, gt_result** out) {
  *out = nullptr;
  gt_result* r = new gt_result();
  int status = guard([&] {
    if (task != GT_WORDCOUNT && task != GT_SORT) fail(GT_E_USAGE, "gt_assemble_counts: task %d is not wordcount/sort", task);
    DeviceDag& d = c->d;
    GT_CUDA(cudaSetDevice(d.device));
    if (task == GT_SORT) ensure_derived(&d);
    auto t0 = std::chrono::steady_clock::now();
    u64 launches0 = g_launches;
    GT_CUDA(cudaEventRecord(c->ev[0], d.stream));
    DevRecords R;
    assemble_counts(&d, dev_counts, d.nw, 0, task == GT_SORT, &R);
    GT_CUDA(cudaEventRecord(c->ev[1], d.stream));
    finish(c, r, R, task, 3, 0, GT_TOPDOWN, t0, launches0);
  });
  if (status != GT_OK) {
    delete r;
    return status;
  }
  *out = r;
  return GT_OK;
}

int gt_table_add_batch(int device, const uint32_t* keys, const uint64_t* deltas, uint64_t n, uint32_t capacity,
                       uint32_t* out_keys, uint64_t* out_counts) {
  int rc = GT_OK;
  int st = guard([&] { rc = table_add_batch(device, keys, deltas, n, capacity, out_keys, out_counts); });
  if (st == GT_OK && rc != GT_OK) set_last_error("table full");
  return st != GT_OK ? st : rc;
}

int gt_result_view(const gt_result* r, gt_view* out) {
  *out = r->v;
  return GT_OK;
}

void gt_result_free(gt_result* r) { delete r; }

uint64_t* gt_device_word_counts(gt_ctx* c) { return c->d.word_counts.as<uint64_t>(); }

int gt_flush_l2(gt_ctx* c) {
  return guard([&] {
    // one 256 MiB (> 126 MB L2) scratch per device, deliberately never freed:
    // a static destructor calling into CUDA after context teardown at exit
    // would crash the process
    static void* bufs[64] = {};
    const size_t n = 256ull << 20;
    void*& buf = bufs[c->d.device & 63];
    if (!buf) GT_CUDA(cudaMalloc(&buf, n));
    GT_CUDA(cudaMemsetAsync(buf, (int)(g_launches & 0xFF), n, c->d.stream));
  });
}

int gt_profile(gt_ctx* c, int enable) {
  return guard([&] {
    if (c) GT_CUDA(cudaStreamSynchronize(c->d.stream));
    g_prof.on = enable != 0;
  });
}

int64_t gt_profile_report(gt_ctx* c, char* buf, size_t cap) {
  // records are drained into a per-thread aggregate; the aggregate is only
  // cleared when it is actually copied out (buf != NULL), so the usual
  // size-query-then-read call pair sees the same report
  static thread_local std::vector<std::pair<std::string, std::pair<u64, double>>> agg;
  std::string text;
  int st = guard([&] {
    if (c) GT_CUDA(cudaStreamSynchronize(c->d.stream));
    else GT_CUDA(cudaDeviceSynchronize());
    for (auto& r : g_prof.recs) {
      float ms = 0;
      GT_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      auto it = std::find_if(agg.begin(), agg.end(), [&](auto& x) { return x.first == r.name; });
      if (it == agg.end()) agg.push_back({r.name, {1, ms}});
      else it->second.first++, it->second.second += ms;
      g_prof.pool.push_back(r.a);
      g_prof.pool.push_back(r.b);
    }
    g_prof.recs.clear();
    char line[256];
    for (auto& x : agg) {
      snprintf(line, sizeof line, "%s\t%lu\t%.6f\n", x.first.c_str(), (unsigned long)x.second.first,
               x.second.second);
      text += line;
    }
  });
  if (st != GT_OK) return -1;
  if (buf && cap) {
    size_t n = std::min(cap - 1, text.size());
    memcpy(buf, text.data(), n);
    buf[n] = 0;
    agg.clear();
  }
  return (int64_t)text.size() + 1;
}

int gt_sync(gt_ctx* c) {
  return guard([&] { GT_CUDA(cudaStreamSynchronize(c->d.stream)); });
}

int64_t gt_dag_array(gt_ctx* c, const char* name, int64_t* out, int64_t cap) {
  DeviceDag& d = c->d;
  int64_t result = -1;
  int st = guard([&] {
    GT_CUDA(cudaSetDevice(d.device));
    cudaStream_t s = d.stream;
    std::string nm(name);
    auto fetch32 = [&](const DBuf& b, u64 n) {
      std::vector<int64_t> v(n);
      std::vector<u32> t(n);
      if (n) GT_CUDA(cudaMemcpyAsync(t.data(), b.p, n * 4, cudaMemcpyDeviceToHost, s));
      GT_CUDA(cudaStreamSynchronize(s));
      for (u64 i = 0; i < n; i++) v[i] = t[i];
      return v;
    };
    auto fetch64 = [&](const DBuf& b, u64 n) {
      std::vector<int64_t> v(n);
      if (n) GT_CUDA(cudaMemcpyAsync(v.data(), b.p, n * 8, cudaMemcpyDeviceToHost, s));
      GT_CUDA(cudaStreamSynchronize(s));
      return v;
    };
    std::vector<int64_t> v;
    ensure_derived(&c->d);
    if (nm == "par_ids" || nm == "par_freqs" || nm == "par_off" || nm == "num_in_edge") ensure_parents(&c->d);
    if (nm == "own_ids") v = fetch32(d.own_ids, d.E_own);
    else if (nm == "own_freqs") v = fetch32(d.own_freqs, d.E_own);
    else if (nm == "own_off") v = fetch64(d.own_off, d.R + 1);
    else if (nm == "own_token_count") v = fetch64(d.own_tok, d.R);
    else if (nm == "sub_ids") v = fetch32(d.sub_ids, d.E_sub);
    else if (nm == "sub_freqs") v = fetch32(d.sub_freqs, d.E_sub);
    else if (nm == "sub_off") v = fetch64(d.sub_off, d.R + 1);
    else if (nm == "par_ids") v = fetch32(d.par_ids, d.E_sub);
    else if (nm == "par_freqs") v = fetch32(d.par_freqs, d.E_sub);
    else if (nm == "par_off") v = fetch64(d.par_off, d.R + 1);
    else if (nm == "num_in_edge") v = fetch64(d.num_in, d.R);
    else if (nm == "num_out_edge") v = fetch64(d.num_out, d.R);
    else if (nm == "exp_len") v = fetch64(d.exp_len, d.R);
    else if (nm == "td_level") v = fetch32(d.td_level, d.R);
    else if (nm == "tid") v = fetch32(d.tid, d.R);  // top-down row of every rule
    // the single-parent contraction in tid space (contract.cu; diagnostics:
    // builds it on request; empty when a multiplier outgrew 32 bits)
    else if (nm == "cont_sizes") {  // [heads, edges, levels] of the built contraction (empty: none)
      if (d.contracted) v = {(int64_t)d.c_R, (int64_t)d.c_te_off.back(), (int64_t)d.c_levels};
    }
    else if (nm == "cont_head" || nm == "cont_mult" || nm == "cont_level" || nm == "cont_row") {
      ensure_contracted(&d);
      if (d.contracted) {
        const DBuf& b = nm == "cont_head" ? d.c_hd : nm == "cont_mult" ? d.c_ml : nm == "cont_level" ? d.c_lvp : d.c_tid;
        v = fetch32(b, d.R);
      }
    }
    else if (nm == "bu_level") v = fetch32(d.bu_level, d.R);
    else if (nm == "segment_token_counts") v = fetch64(d.seg_tokens, d.F);
    else if (nm == "root_freq") {
      auto so = fetch64(d.sub_off, 2);
      auto ids = fetch32(d.sub_ids, d.E_sub);
      auto fr = fetch32(d.sub_freqs, d.E_sub);
      v.assign(d.R, 0);
      for (int64_t j = so[0]; j < so[1]; j++) v[ids[j]] = fr[j];
    } else if (nm == "segments") {
      auto lo = fetch64(d.seg_lo, d.F), hi = fetch64(d.seg_hi, d.F);
      for (u64 f = 0; f < d.F; f++) {
        v.push_back(lo[f]);
        v.push_back(hi[f]);
      }
    } else {
      fail(GT_E_USAGE, "unknown DAG array %s", name);
    }
    result = (int64_t)v.size();
    if (out) {
      if (cap < result) fail(GT_E_USAGE, "buffer too small");
      memcpy(out, v.data(), v.size() * 8);
    }
  });
  return st == GT_OK ? result : -1;
}

}  // extern "C"
