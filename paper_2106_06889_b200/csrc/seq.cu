// seq.cu — l-gram counting per file on the device DAG (sequence_count /
// ranked_inverted_index).
//
// Reference (sequence.py:50-417, _kernels.py:279-309): per-rule head/tail
// buffers of l-1 words (Fig. 6), local streams that inline children as
// absorbed / owned span / head|GAP|tail (Fig. 7), windows counted once per
// rule into hash tables, then scaled merges into per-file tables.
//
// B200 formulation, same exactly-once attribution: a window of rule r's
// expansion belongs to r iff it is not inside one child's expansion, i.e.
// it starts at a word symbol of r's body or inside the last min(l-1, |c|)
// words (the tail) of a child c, and completes within r's body before a
// splitter.  One thread per body position enumerates those windows directly
// from the tail of its own symbol and the heads of the following symbols —
// no local streams are materialised.  Counting is sort-based instead of
// hashing: window keys (packed big-endian, l*wbits <= 63, else l word ids)
// are radix-sorted with their source (rule, or root segment), each key run
// is reduced against the per-file weight rows (F columns, from the same
// top-down level pull as term vectors), and the nonzero (gram, file, count)
// records are ordered for render with two stable radix sorts.
#include <cooperative_groups.h>

#include <algorithm>

#include "kernels_common.cuh"
#include "segreduce.cuh"
#include "bottomup.cuh"
#include "seq.cuh"
#include "sparse.cuh"

namespace gt {

namespace {

// heads/tails (sequence.py:110-140): the first / last min(l-1, exp_len)
// words of a rule's expansion, from its body and its children's (finished:
// lower bottom-up level).  Children's buffers are read through L2 (ld.cg):
// they were written by other SMs before the last grid barrier.
__device__ __forceinline__ void head_tail_rule(u32 r, const u32* __restrict__ body, const u64* __restrict__ boff,
                                               u64 nw, u64 base, const u64* __restrict__ exp_len, u32 m, u32* H,
                                               u32* T, u32* hl, u32* tl) {
  const u64 el = exp_len[r];
  const u32 target = (u32)(el < m ? el : m);
  const u64 b0 = boff[r], b1 = boff[r + 1];
  u32 n = 0;
  for (u64 q = b0; q < b1 && n < target; q++) {
    const u32 s = body[q];
    if (s < nw) {
      H[(u64)r * m + n++] = s;
    } else if (s >= base) {
      const u32 c = s - (u32)base;
      const u32 hc = __ldcg(hl + c);
      for (u32 j = 0; j < hc && n < target; j++) H[(u64)r * m + n++] = __ldcg(H + (u64)c * m + j);
    }
  }
  hl[r] = target;
  n = 0;
  for (u64 q = b1; q > b0 && n < target; q--) {
    const u32 s = body[q - 1];
    if (s < nw) {
      T[(u64)r * m + (target - 1 - n++)] = s;
    } else if (s >= base) {
      const u32 c = s - (u32)base;
      for (u32 j = __ldcg(tl + c); j > 0 && n < target; j--)
        T[(u64)r * m + (target - 1 - n++)] = __ldcg(T + (u64)c * m + j - 1);
    }
  }
  tl[r] = target;
}

// every bottom-up level in ONE cooperative launch (grid barrier between
// levels instead of a launch per level)
__global__ void __launch_bounds__(1024) k_head_tail_levels(const u32* __restrict__ order, const u64* __restrict__ off,
                                                           int nl, const u32* __restrict__ body,
                                                           const u64* __restrict__ boff, u64 nw, u64 base,
                                                           const u64* __restrict__ exp_len, u32 m, u32* H, u32* T,
                                                           u32* hl, u32* tl) {
  cg::grid_group grid = cg::this_grid();
  const u64 stride = (u64)gridDim.x * blockDim.x;
  // 32 consecutive rules per warp, warps round-robin over the SMs (a small
  // level reaches every SM instead of the first blocks)
  const u64 t0 = ((u64)(threadIdx.x >> 5) * gridDim.x + blockIdx.x) * 32 + (threadIdx.x & 31u);
  for (int L = 1; L <= nl; L++) {
    const u64 lo = off[L], hi = off[L + 1];
    for (u64 i = lo + t0; i < hi; i += stride) {
      const u32 r = order[i];
      if (r != 0) head_tail_rule(r, body, boff, nw, base, exp_len, m, H, T, hl, tl);
    }
    if (L < nl) grid.sync();
  }
}

struct WinCtx {
  const u32* body;
  const u32* owner;
  const u32* tid;  // rule -> tid (the weight rows' numbering); nullptr: rule ids
  const u64* boff;
  const u32* root_seg;
  const u32 *H, *T, *hl, *tl;
  u64 nw, base;
  u32 l, m, wbits, R, file_lo, nseg;
};

// number of windows attributed at body position p, plus its source id
__device__ __forceinline__ u32 windows_at(const WinCtx& c, u64 p, u32* src, u32* tail_len,
                                          u32* start_sym) {
  const u32 r = c.owner[p];
  if (r == 0) {
    u32 sg = c.root_seg[p] - c.file_lo;
    if (sg >= c.nseg) return 0;
    *src = c.R + sg;
  } else {
    *src = c.tid ? c.tid[r] : r;  // weight-row numbering (top-down) or rule id (bottom-up tables)
  }
  const u32 s = c.body[p];
  u32 tlen;
  if (s < c.nw) tlen = 1;
  else if (s >= c.base) tlen = c.tl[s - (u32)c.base];
  else return 0;  // splitter
  *tail_len = tlen;
  *start_sym = s;
  if (tlen == 0) return 0;
  // words available after p within the body (up to l-1, stop at a splitter)
  u32 avail = 0;
  const u64 end = c.boff[r + 1];
  for (u64 q = p + 1; q < end && avail < c.m; q++) {
    u32 t = c.body[q];
    if (t < c.nw) avail++;
    else if (t >= c.base) avail += c.hl[t - (u32)c.base];
    else break;
  }
  if (avail > c.m) avail = c.m;
  // start t in [0, tlen) succeeds iff (tlen - t) + avail >= l
  i64 hi = (i64)tlen + (i64)avail - (i64)c.l;  // last successful t
  if (hi < 0) return 0;
  return (u32)std::min<i64>(tlen, hi + 1);
}

// word j of window starting at tail index t of the symbol at p
template <class Put>
__device__ __forceinline__ void window_words(const WinCtx& c, u64 p, u32 s, u32 tlen, u32 t, Put put) {
  u32 j = 0;
  if (s < c.nw) put(j++, s);
  else {
    const u32* T = c.T + (u64)(s - (u32)c.base) * c.m;
    for (u32 k = t; k < tlen; k++) put(j++, T[k]);
  }
  for (u64 q = p + 1; j < c.l; q++) {
    u32 x = c.body[q];
    if (x < c.nw) put(j++, x);
    else if (x >= c.base) {
      const u32 cc = x - (u32)c.base;
      const u32* H = c.H + (u64)cc * c.m;
      for (u32 k = 0; k < c.hl[cc] && j < c.l; k++) put(j++, H[k]);
    }
  }
}

__global__ void k_count_windows(WinCtx c, u64 E, u64* cnt) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += stride) {
    u32 src, tlen, s;
    cnt[p] = windows_at(c, p, &src, &tlen, &s);
  }
}

__global__ void k_write_windows(WinCtx c, u64 E, const u64* off, int packed, u64* key, u32* gram,
                                u32* srcs) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += stride) {
    u32 src, tlen, s;
    u32 n = windows_at(c, p, &src, &tlen, &s);
    u64 o = off[p];
    for (u32 t = 0; t < n; t++) {
      srcs[o + t] = src;
      if (packed) {
        u64 k = 0;
        window_words(c, p, s, tlen, t, [&](u32, u32 w) { k = (k << c.wbits) | w; });
        key[o + t] = k;
      } else {
        u32* g = gram + (o + t) * c.l;
        window_words(c, p, s, tlen, t, [&](u32 j, u32 w) { g[j] = w; });
      }
    }
  }
}

__global__ void k_gather_col(const u32* gram, const u32* idx, u64 n, u32 l, u32 j, u32* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = gram[(u64)idx[i] * l + j];
}

__global__ void k_permute_gram(const u32* gram, const u32* src, const u32* idx, u64 n, u32 l,
                               u32* gram2, u32* src2) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 k = idx[i];
    src2[i] = src[k];
    for (u32 j = 0; j < l; j++) gram2[i * l + j] = gram[(u64)k * l + j];
  }
}

__global__ void k_run_heads(const u64* key, const u32* gram, u64 n, u32 l, int packed, uint8_t* h) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    bool head = i == 0;
    if (!head) {
      if (packed) head = key[i] != key[i - 1];
      else
        for (u32 j = 0; j < l && !head; j++) head = gram[i * l + j] != gram[(i - 1) * l + j];
    }
    h[i] = head;
  }
}

// gram-run rows: an occurrence from rule s < R adds that rule's per-file
// weight row; an occurrence counted directly in root segment s-R adds 1 to
// that file's column
template <class T>
struct SeqSrc {
  const T* w;
  u32 R, C;
  __device__ __forceinline__ u64 operator()(u32 s, u32 col) const {
    return s < R ? w[(u64)s * C + col] : (s - R == col ? 1ull : 0ull);
  }
};

// two adjacent columns in one vector load (segreduce.cuh paired path)
__device__ __forceinline__ void load_pair(const SeqSrc<u32>& in, u32 s, u32 col, u64* a, u64* b) {
  if (s < in.R) {
    const uint2 v = *reinterpret_cast<const uint2*>(in.w + (u64)s * in.C + col);
    *a = v.x;
    *b = v.y;
  } else {
    *a = s - in.R == col ? 1ull : 0ull;
    *b = s - in.R == col + 1 ? 1ull : 0ull;
  }
}
__device__ __forceinline__ void load_pair(const SeqSrc<u64>& in, u32 s, u32 col, u64* a, u64* b) {
  if (s < in.R) {
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(in.w + (u64)s * in.C + col);
    *a = v.x;
    *b = v.y;
  } else {
    *a = s - in.R == col ? 1ull : 0ull;
    *b = s - in.R == col + 1 ? 1ull : 0ull;
  }
}

__global__ void k_heads_u32(const uint8_t* h, u64 n, u32* o) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) o[i] = h[i];
}

__global__ void k_dec_u32(u32* v, u64 n) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) v[i] -= 1;
}

// dense rows -> cells: selected index j = run*C + col
template <class T>
__global__ void k_cells_dense(const u32* sel, const u64* nsel, const T* rows, u32 C, u32* crun,
                              u32* ccol, u64* ccnt) {
  u64 n = *nsel;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 j = sel[i];
    crun[i] = j / C;
    ccol[i] = j % C;
    ccnt[i] = rows[j];
  }
}

// sparse cells: key = run << FB | col
__global__ void k_cells_keys(const u64* key, u64 n, int FB, u32* crun, u32* ccol) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    crun[i] = (u32)(key[i] >> FB);
    ccol[i] = (u32)(key[i] & ((1ull << FB) - 1));
  }
}

// cells (run, col, count) -> sort key (major << CB) | (W - count)
__global__ void k_rec_keys(const u32* crun, const u32* ccol, const u64* ccnt, u64 n, u64 W, int CB,
                           int by_file, u64* skey, u32* rec) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    skey[i] = ((u64)(by_file ? ccol[i] : crun[i]) << CB) | (W - ccnt[i]);
    rec[i] = (u32)i;
  }
}

// payload-carrying record sort (packed grams)
// record sort keys (major << CB | W - count); K = u32 when CB + MB <= 32
// (C2: 28 + 4 bits — a quarter less radix traffic than u64 keys)
template <class K>
__global__ void k_rec_keys2(const u32* crun, const u32* ccol, const u64* ccnt, u64 n, u64 W, int CB, int by_file,
                            K* skey) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    skey[i] = (K)(((u64)(by_file ? ccol[i] : crun[i]) << CB) | (W - ccnt[i]));
}

__global__ void k_cell_grams(const u32* crun, u64 n, const u32* run_start, const u64* skey_sorted, u64* gk) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) gk[i] = skey_sorted[run_start[crun[i]]];
}

// sorted (major << CB | W - count) -> count, major
template <class K>
__global__ void k_unkey2(const K* key, u64 n, u64 W, int CB, u64* cnt, u32* major, u32) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 m = (1ull << CB) - 1;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 k = key[i];
    cnt[i] = W - (k & m);
    major[i] = (u32)(k >> CB);
  }
}

__global__ void k_add_u32_base(u32* a, u64 n, u32 v) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] += v;
}

__global__ void k_heads_u32v(const u32* g, u64 n, uint8_t* h) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) h[i] = i == 0 || g[i] != g[i - 1];
}

// RANKEDINVERTEDINDEX on <= 16 owned files: the cells of one gram run
// (files ascending, at most 16, ~3 on C2) ordered by (-count, file) in place
// of a corpus-wide radix sort of (run | W - count) keys — a thread per cell
// finds its run's bounds and its rank (cells of the run with a larger count,
// or an equal count and a smaller file: files are distinct within a run)
__global__ void k_rii_rank(const u32* __restrict__ run, u64 n, const u32* __restrict__ col,
                           const u64* __restrict__ cnt, u32 file_lo, u32* __restrict__ out_id,
                           u64* __restrict__ out_cnt) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 r = run[i], f = col[i];
    const u64 c = cnt[i];
    u64 a = i, b = i + 1;
    while (a > 0 && run[a - 1] == r) a--;
    while (b < n && run[b] == r) b++;
    u64 rank = 0;
    for (u64 j = a; j < b; j++) {
      const u64 cj = cnt[j];
      rank += cj > c || (cj == c && col[j] < f);
    }
    out_id[a + rank] = f + file_lo;
    out_cnt[a + rank] = c;
  }
}

__global__ void k_group_out2(const u32* gsel, const u64* ng_p, u64 n, const u32* run, const u32* run_start,
                             const u64* skey_sorted, u64* goff, u64* gkey) {
  const u64 ng = *ng_p;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g <= ng; g += stride) {
    if (g == ng) {
      goff[g] = n;
      continue;
    }
    const u32 i = gsel[g];
    goff[g] = i;
    gkey[g] = skey_sorted[run_start[run[i]]];
  }
}

__global__ void k_rec_out(const u32* rec, u64 n, const u32* crun, const u32* ccol, const u64* ccnt,
                          const u32* run_start, const u64* skey_sorted, const u32* gram, u32 l,
                          int packed, u32 file_lo, int write_gram, u64* key_out, u32* gram_out,
                          u64* cnt_out, u32* id_out, u32* major_out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 j = rec[i];
    const u32 run = crun[j], col = ccol[j];
    cnt_out[i] = ccnt[j];
    if (id_out) id_out[i] = file_lo + col;
    if (major_out) major_out[i] = col;
    const u32 rs = run_start[run];
    if (write_gram) {
      if (packed) key_out[i] = skey_sorted[rs];
      else
        for (u32 k = 0; k < l; k++) gram_out[(u64)i * l + k] = gram[(u64)rs * l + k];
    }
  }
}

__global__ void k_group_heads(const u32* rec, u64 n, const u32* crun, uint8_t* h) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    h[i] = i == 0 || crun[rec[i]] != crun[rec[i - 1]];
}

__global__ void k_group_out(const u32* gsel, const u64* ng_p, const u32* rec, const u32* crun,
                            const u32* run_start, const u64* keys, const u32* gram, u32 l,
                            int packed, u64* goff, u64* gkey, u32* ggram) {
  u64 ng = *ng_p;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += stride) {
    u32 i = gsel[g];
    goff[g] = i;
    u32 rs = run_start[crun[rec[i]]];
    if (packed) gkey[g] = keys[rs];
    else
      for (u32 k = 0; k < l; k++) ggram[(u64)g * l + k] = gram[(u64)rs * l + k];
  }
}

// window sources from rule ids to weight-row ids (tid) after a bottom-up
// attempt fell back to the top-down path
// window sources in tid numbering -> the contraction's head rows, with the
// rule's multiplier (root windows, src >= R, keep their file column, x1)
__global__ void k_src_head(u32* src, u64 n, u32 R, const u32* __restrict__ ctid, const u32* __restrict__ hd,
                           const u32* __restrict__ ml, u32* mult) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 s = src[i];
    if (s < R) {
      src[i] = ctid[hd[s]];
      mult[i] = ml[s];
    } else {
      mult[i] = 1u;
    }
  }
}

__global__ void k_src_tid(u32* src, u64 n, const u32* tid, u32 R) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (src[i] < R) src[i] = tid[src[i]];
}

#define SL(k, n, ...) GT_KLAUNCH(#k, k, grid_for((n), 256), 256, st, __VA_ARGS__)

template <class T>
static T d2h1(const void* p, cudaStream_t st) {
  T v;
  GT_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  return v;
}

}  // namespace

int run_sequences(DeviceDag* d, int task, int l_, int mode, DevRecords* Rr, int* wbits_out) {
  cudaStream_t st = d->stream;
  Phases ph("seq", st);
  const u32 l = (u32)l_, m = l - 1;
  const u64 R = d->R, E = d->E, nw = d->nw, base = d->nw + d->ns;
  // pack_width, sequence.py:229-231
  const int wbits = std::max(1, bitlen(nw ? nw - 1 : 1));
  const int packed = (u64)l * wbits <= 63;
  *wbits_out = packed ? wbits : 0;
  const u32 Fo = (u32)(d->file_hi - d->file_lo);
  const u32 C = std::max<u32>(1, Fo);

  // phase 1: head/tail buffers by bottom-up level (sequence.py:110-140)
  const u32 mm = std::max<u32>(m, 1);
  DBuf H(R * mm * 4, st), T(R * mm * 4, st), hl(R * 4, st), tl(R * 4, st);
  GT_CUDA(cudaMemsetAsync(hl.p, 0, R * 4, st));
  GT_CUDA(cudaMemsetAsync(tl.p, 0, R * 4, st));
  if (m) {
    ensure_bu_levels(d);
    if (d->bu.nl >= 1) {
      int dev = 0, nsm = 148;
      GT_CUDA(cudaGetDevice(&dev));
      GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      const u32* ord = d->bu.order.as<u32>();
      const u64* lo = d->bu.off_dev.as<u64>();
      int nl = d->bu.nl;
      const u32* bd = d->body.as<u32>();
      const u64* bo = d->boff.as<u64>();
      const u64* el = d->exp_len.as<u64>();
      u32 *Hp = H.as<u32>(), *Tp = T.as<u32>(), *hlp = hl.as<u32>(), *tlp = tl.as<u32>();
      u64 nw_ = nw, base_ = base;
      u32 m_ = m;
      void* args[] = {(void*)&ord, (void*)&lo, (void*)&nl, (void*)&bd, (void*)&bo, (void*)&nw_, (void*)&base_,
                      (void*)&el, (void*)&m_, (void*)&Hp, (void*)&Tp, (void*)&hlp, (void*)&tlp};
      ProfScope ps("k_head_tail_levels", st);
      GT_CUDA(cudaLaunchCooperativeKernel((const void*)k_head_tail_levels, dim3((unsigned)nsm), dim3(1024), args,
                                          0, st));
      g_launches++;
    }
  }
  ph.mark("heads/tails");
  // per-file rule weights: dense top-down rows (F columns) or, for many
  // files, the presence-guided sparse (rule, file) weights (sparse.cu);
  // none for the bottom-up tables
  bool bottomup = mode == GT_BOTTOMUP;
  bool sparse = mode == GT_TOPDOWN_SPARSE;
  DBuf w;
  bool w32 = false, wheads = false;
  SparseW sw;
  auto weights = [&] {
    if (sparse) {
      u32 FW;
      sparse_file_weights(d, &sw, nullptr, &FW);
    } else {
      u32 Cw;
      // the dense rows of the contraction's heads when it is in use (a
      // window's weight is its rule's multiplier times its head's row) on
      // up to 16 owned files (C2 sequence count 1.54 -> 1.50 ms); on 64 the
      // scaled gathers of the window pass cost more than the shorter level
      // pass saves (C4 ranked inverted index 19.5 vs 21.0 ms)
      td_file_weights(d, w, &Cw, &w32, C <= 16, &wheads);
    }
  };
  if (!bottomup) weights();
  ph.mark("weights");
  // phase 2: windows attributed per body position (two passes + scan)
  WinCtx c{d->body.as<u32>(), d->pos_owner.as<u32>(), bottomup ? nullptr : d->tid.as<u32>(), d->boff.as<u64>(),
           d->root_seg.as<u32>(),
           H.as<u32>(), T.as<u32>(), hl.as<u32>(), tl.as<u32>(), nw, base, l, m, (u32)wbits,
           (u32)R, (u32)d->file_lo, Fo};
  DBuf cnt(E * 8 + 8, st), off(E * 8 + 8, st);
  SL(k_count_windows, E, c, E, cnt.as<u64>());
  exclusive_scan_u64(cnt.as<u64>(), off.as<u64>(), E, st);
  u64 N = 0;
  if (E) N = d2h1<u64>(off.as<u64>() + E - 1, st) + d2h1<u64>(cnt.as<u64>() + E - 1, st);
  cnt.release();
  if (N >= (1ull << 32)) fail(GT_E_RESOURCE, "%lu windows exceed the 2^32 record limit", (unsigned long)N);
  DBuf key(packed ? N * 8 + 8 : 8, st), gram(packed ? 8 : N * l * 4 + 4, st), src(N * 4 + 4, st);
  SL(k_write_windows, E, c, E, off.as<u64>(), packed, key.as<u64>(), gram.as<u32>(), src.as<u32>());
  off.release();

  ph.mark("windows");
  // sort by gram
  DBuf skey, sgram, ssrc(N * 4 + 4, st);
  if (packed) {
    skey.alloc(N * 8 + 8, st);
    sort_pairs_u64_u32(key.as<u64>(), skey.as<u64>(), src.as<u32>(), ssrc.as<u32>(), N,
                       std::max(1, (int)(l * wbits)), st);
  } else {
    DBuf idx(N * 4 + 4, st), idx2(N * 4 + 4, st), col(N * 4 + 4, st), col2(N * 4 + 4, st);
    SL(k_iota_u32, N, idx.as<u32>(), N);
    for (int j = (int)l - 1; j >= 0; j--) {
      SL(k_gather_col, N, gram.as<u32>(), idx.as<u32>(), N, l, (u32)j, col.as<u32>());
      sort_pairs_u32_u32(col.as<u32>(), col2.as<u32>(), idx.as<u32>(), idx2.as<u32>(), N, wbits, st);
      std::swap(idx, idx2);
    }
    sgram.alloc(N * l * 4 + 4, st);
    SL(k_permute_gram, N, gram.as<u32>(), src.as<u32>(), idx.as<u32>(), N, l, sgram.as<u32>(), ssrc.as<u32>());
  }
  ph.mark("gram sort");
  key.release();
  gram.release();
  src.release();

  // key runs -> per-run file counts
  DBuf heads(N + 1, st), runs(N * 4 + 4, st), dcnt(16, st);
  SL(k_run_heads, N, skey.as<u64>(), sgram.as<u32>(), N, l, packed, heads.as<uint8_t>());
  select_flagged_index(heads.as<uint8_t>(), runs.as<u32>(), dcnt.as<u64>(), N, st);
  const u64 nruns = d2h1<u64>(dcnt.p, st);
  // run id of every occurrence = inclusive scan of the run heads - 1
  DBuf rid(N * 4 + 4, st);
  if (nruns) {
    DBuf h32(N * 4 + 4, st);
    SL(k_heads_u32, N, heads.as<uint8_t>(), N, h32.as<u32>());
    inclusive_scan_u32(h32.as<u32>(), rid.as<u32>(), N, st);
    SL(k_dec_u32, N, rid.as<u32>(), N);
  }
  heads.release();
  ph.mark("runs");
  // nonzero (run, file) cells in (gram asc, file asc) order
  DBuf crun, ccol, ccnt;
  u64 n = 0;
  if (bottomup && !bu_seq_cells(d, l, rid.as<u32>(), ssrc.as<u32>(), nruns ? N : 0, nruns, crun, ccol, ccnt, &n,
                                scratch_budget(d))) {
    // the table arena exceeds the memory budget: the top-down sparse path
    bottomup = false;
    sparse = true;
    SL(k_src_tid, N, ssrc.as<u32>(), N, d->tid.as<u32>(), (u32)R);
    weights();
  }
  if (bottomup) {
    // cells come from the tables
  } else if (sparse) {
    const int FB = std::max(1, bitlen(C - 1));
    DBuf ckey;
    n = sparse_run_cells(d, sw, rid.as<u32>(), ssrc.as<u32>(), nruns ? N : 0, FB, ckey, ccnt);
    crun.alloc(n * 4 + 4, st);
    ccol.alloc(n * 4 + 4, st);
    SL(k_cells_keys, n, ckey.as<u64>(), n, FB, crun.as<u32>(), ccol.as<u32>());
    sw = SparseW();
  } else {
    const u64 NR = nruns * C;
    if (NR >= (1ull << 32)) fail(GT_E_RESOURCE, "%lu gram x file cells exceed the 2^32 limit", (unsigned long)NR);
    // per-file weights fit u32 (w32) -> so do the (gram, file) cells
    // (GT_SEQ_ROWS=64: u64 cell rows over u32 weights, diagnostics)
    static const bool rows64_env = getenv("GT_SEQ_ROWS") && atoi(getenv("GT_SEQ_ROWS")) == 64;
    const bool r32 = w32 && !rows64_env;
    const u64 eb = r32 ? 4 : 8;
    DBuf rows(NR * eb + 8, st);
    GT_CUDA(cudaMemsetAsync(rows.p, 0, NR * eb, st));
    DBuf mult;
    const u32* wf = nullptr;  // per-window multiplier (contraction), or none
    if (wheads && N) {
      mult.alloc(N * 4 + 4, st);
      SL(k_src_head, N, ssrc.as<u32>(), N, (u32)R, d->c_tid.as<u32>(), d->c_hd.as<u32>(), d->c_ml.as<u32>(),
         mult.as<u32>());
      wf = mult.as<u32>();
    }
    if (nruns) {
      if (w32 && r32)
        seg_reduce<SumMode>("k_run_rows", rid.as<u32>(), ssrc.as<u32>(), wf, N, C,
                            SeqSrc<u32>{w.as<u32>(), (u32)R, C}, OutRowMajorT<u32>{rows.as<u32>(), C}, st);
      else if (w32)
        seg_reduce<SumMode>("k_run_rows", rid.as<u32>(), ssrc.as<u32>(), wf, N, C,
                            SeqSrc<u32>{w.as<u32>(), (u32)R, C}, OutRowMajor{rows.as<u64>(), C}, st);
      else
        seg_reduce<SumMode>("k_run_rows", rid.as<u32>(), ssrc.as<u32>(), wf, N, C,
                            SeqSrc<u64>{w.as<u64>(), (u32)R, C}, OutRowMajor{rows.as<u64>(), C}, st);
    }
    w.release();
    DBuf sel(NR * 4 + 4, st);
    select_nonzero_index(rows.p, r32, sel.as<u32>(), dcnt.as<u64>(), NR, st);
    n = d2h1<u64>(dcnt.p, st);
    crun.alloc(n * 4 + 4, st);
    ccol.alloc(n * 4 + 4, st);
    ccnt.alloc(n * 8 + 8, st);
    if (r32)
      SL(k_cells_dense<u32>, n, sel.as<u32>(), dcnt.as<u64>(), rows.as<u32>(), C, crun.as<u32>(),
         ccol.as<u32>(), ccnt.as<u64>());
    else
      SL(k_cells_dense<u64>, n, sel.as<u32>(), dcnt.as<u64>(), rows.as<u64>(), C, crun.as<u32>(),
         ccol.as<u32>(), ccnt.as<u64>());
  }
  ssrc.release();
  rid.release();
  ph.mark("cells");
  // the count field of the record sort key spans the largest cell count (one
  // reduction + read-back): C4 39 -> 32-bit keys, one radix pass fewer
  u64 Wt = d->max_file_tokens ? d->max_file_tokens : d->W;
  // RII on <= 16 owned files ranks each run's cells in place (k_rii_rank): no
  // record keys, no count bound (C2: 0.29 ms of sort -> 0.15 ms; at 64 files
  // the O(cells^2) ranks cost more than the radix sort: C4 4.2 vs ~2 ms)
  const bool rii_rank = packed && task != GT_SEQCOUNT && C <= 16;
  if (!rii_rank && n &&
      bitlen(Wt) + (task == GT_SEQCOUNT ? std::max(1, bitlen(C - 1)) : std::max(1, bitlen(nruns))) > 32) {
    DBuf mx(8, st);
    reduce_max_u64(ccnt.as<u64>(), mx.as<u64>(), n, st);
    Wt = std::max<u64>(1, d2h1<u64>(mx.p, st));
  }
  const int CB = std::max(1, bitlen(Wt));
  const bool by_file = task == GT_SEQCOUNT;
  const int MB = by_file ? std::max(1, bitlen(C - 1)) : std::max(1, bitlen(nruns));
  if (!rii_rank && CB + MB > 64) fail(GT_E_RESOURCE, "sort key of %d bits exceeds 64", CB + MB);
  if (packed) {
    // the sort carries its payload: SEQCOUNT sorts (file | W - count) with the
    // packed gram as the value, RII (run | W - count) with the file — every
    // output field comes out of the sorted arrays, no permutation gathers
    const bool k32 = CB + MB <= 32;
    DBuf sk, sk2;
    if (!rii_rank) {
      sk.alloc(n * 8 + 8, st);
      sk2.alloc(n * 8 + 8, st);
      if (k32)
        SL(k_rec_keys2<u32>, n, crun.as<u32>(), ccol.as<u32>(), ccnt.as<u64>(), n, Wt, CB, by_file ? 1 : 0,
           sk.as<u32>());
      else
        SL(k_rec_keys2<u64>, n, crun.as<u32>(), ccol.as<u32>(), ccnt.as<u64>(), n, Wt, CB, by_file ? 1 : 0,
           sk.as<u64>());
    }
    Rr->n = n;
    Rr->count.alloc(n * 8 + 8, st);
    if (by_file) {
      DBuf gk(n * 8 + 8, st);
      Rr->key.alloc(n * 8 + 8, st);
      SL(k_cell_grams, n, crun.as<u32>(), n, runs.as<u32>(), skey.as<u64>(), gk.as<u64>());
      DBuf major(n * 4 + 4, st);
      if (k32) {
        sort_pairs_u32_u64(sk.as<u32>(), sk2.as<u32>(), gk.as<u64>(), Rr->key.as<u64>(), n, CB + MB, st);
        SL(k_unkey2<u32>, n, sk2.as<u32>(), n, Wt, CB, Rr->count.as<u64>(), major.as<u32>(), 0u);
      } else {
        sort_pairs_u64_u64(sk.as<u64>(), sk2.as<u64>(), gk.as<u64>(), Rr->key.as<u64>(), n, CB + MB, st);
        SL(k_unkey2<u64>, n, sk2.as<u64>(), n, Wt, CB, Rr->count.as<u64>(), major.as<u32>(), 0u);
      }
      Rr->n_groups = Fo;
      Rr->group_off.alloc((Fo + 1) * 8, st);
      SL(k_csr_offsets, Fo + 1, major.as<u32>(), n, (u64)Fo, Rr->group_off.as<u64>());
    } else if (rii_rank) {
      // runs of at most 64 cells: ranked in place, no record sort
      Rr->id.alloc(n * 4 + 4, st);
      DBuf gh(n + 1, st), gsel(n * 4 + 4, st);
      SL(k_heads_u32v, n, crun.as<u32>(), n, gh.as<uint8_t>());
      select_flagged_index(gh.as<uint8_t>(), gsel.as<u32>(), dcnt.as<u64>(), n, st);
      const u64 ng = d2h1<u64>(dcnt.p, st);
      SL(k_rii_rank, n, crun.as<u32>(), n, ccol.as<u32>(), ccnt.as<u64>(), (u32)d->file_lo, Rr->id.as<u32>(),
         Rr->count.as<u64>());
      Rr->n_groups = ng;
      Rr->group_off.alloc((ng + 1) * 8, st);
      Rr->group_key.alloc(ng * 8 + 8, st);
      SL(k_group_out2, ng + 1, gsel.as<u32>(), dcnt.as<u64>(), n, crun.as<u32>(), runs.as<u32>(),
         skey.as<u64>(), Rr->group_off.as<u64>(), Rr->group_key.as<u64>());
    } else {
      Rr->id.alloc(n * 4 + 4, st);
      DBuf rn(n * 4 + 4, st), gh(n + 1, st), gsel(n * 4 + 4, st);
      if (k32) {
        sort_pairs_u32_u32(sk.as<u32>(), sk2.as<u32>(), ccol.as<u32>(), Rr->id.as<u32>(), n, CB + MB, st);
        SL(k_unkey2<u32>, n, sk2.as<u32>(), n, Wt, CB, Rr->count.as<u64>(), rn.as<u32>(), (u32)d->file_lo);
      } else {
        sort_pairs_u64_u32(sk.as<u64>(), sk2.as<u64>(), ccol.as<u32>(), Rr->id.as<u32>(), n, CB + MB, st);
        SL(k_unkey2<u64>, n, sk2.as<u64>(), n, Wt, CB, Rr->count.as<u64>(), rn.as<u32>(), (u32)d->file_lo);
      }
      SL(k_add_u32_base, n, Rr->id.as<u32>(), n, (u32)d->file_lo);
      SL(k_heads_u32v, n, rn.as<u32>(), n, gh.as<uint8_t>());
      select_flagged_index(gh.as<uint8_t>(), gsel.as<u32>(), dcnt.as<u64>(), n, st);
      const u64 ng = d2h1<u64>(dcnt.p, st);
      Rr->n_groups = ng;
      Rr->group_off.alloc((ng + 1) * 8, st);
      Rr->group_key.alloc(ng * 8 + 8, st);
      SL(k_group_out2, ng + 1, gsel.as<u32>(), dcnt.as<u64>(), n, rn.as<u32>(), runs.as<u32>(), skey.as<u64>(),
         Rr->group_off.as<u64>(), Rr->group_key.as<u64>());
    }
    ph.mark("record sort");
  } else {
  DBuf sk(n * 8 + 8, st), sk2(n * 8 + 8, st), rec(n * 4 + 4, st), rec2(n * 4 + 4, st);
  SL(k_rec_keys, n, crun.as<u32>(), ccol.as<u32>(), ccnt.as<u64>(), n, Wt, CB, by_file ? 1 : 0,
     sk.as<u64>(), rec.as<u32>());
  sort_pairs_u64_u32(sk.as<u64>(), sk2.as<u64>(), rec.as<u32>(), rec2.as<u32>(), n, CB + MB, st);
  sk.release();
  sk2.release();
  ph.mark("record sort");
  Rr->n = n;
  Rr->count.alloc(n * 8 + 8, st);
  if (by_file) {
    // SEQCOUNT: per file, (-count, gram) order
    if (packed) Rr->key.alloc(n * 8 + 8, st);
    else Rr->gram.alloc(n * l * 4 + 4, st);
    DBuf major(n * 4 + 4, st);
    SL(k_rec_out, n, rec2.as<u32>(), n, crun.as<u32>(), ccol.as<u32>(), ccnt.as<u64>(), runs.as<u32>(),
       skey.as<u64>(), sgram.as<u32>(), l, packed, (u32)d->file_lo, 1, Rr->key.as<u64>(),
       Rr->gram.as<u32>(), Rr->count.as<u64>(), (u32*)nullptr, major.as<u32>());
    Rr->n_groups = Fo;
    Rr->group_off.alloc((Fo + 1) * 8, st);
    SL(k_csr_offsets, Fo + 1, major.as<u32>(), n, (u64)Fo, Rr->group_off.as<u64>());
  } else {
    // RANKEDINVERTEDINDEX: grams ascending, per gram (-count, file)
    Rr->id.alloc(n * 4 + 4, st);
    SL(k_rec_out, n, rec2.as<u32>(), n, crun.as<u32>(), ccol.as<u32>(), ccnt.as<u64>(), runs.as<u32>(),
       skey.as<u64>(), sgram.as<u32>(), l, packed, (u32)d->file_lo, 0, (u64*)nullptr, (u32*)nullptr,
       Rr->count.as<u64>(), Rr->id.as<u32>(), (u32*)nullptr);
    DBuf gh(n + 1, st), gsel(n * 4 + 4, st);
    SL(k_group_heads, n, rec2.as<u32>(), n, crun.as<u32>(), gh.as<uint8_t>());
    select_flagged_index(gh.as<uint8_t>(), gsel.as<u32>(), dcnt.as<u64>(), n, st);
    const u64 ng = d2h1<u64>(dcnt.p, st);
    Rr->n_groups = ng;
    Rr->group_off.alloc((ng + 1) * 8, st);
    if (packed) Rr->group_key.alloc(ng * 8 + 8, st);
    else Rr->group_gram.alloc(ng * l * 4 + 4, st);
    SL(k_group_out, ng, gsel.as<u32>(), dcnt.as<u64>(), rec2.as<u32>(), crun.as<u32>(), runs.as<u32>(),
       skey.as<u64>(), sgram.as<u32>(), l, packed, Rr->group_off.as<u64>(), Rr->group_key.as<u64>(),
       Rr->group_gram.as<u32>());
    GT_CUDA(cudaMemcpyAsync(Rr->group_off.as<u64>() + ng, &n, 8, cudaMemcpyHostToDevice, st));
  }
  }
  GT_CUDA(cudaStreamSynchronize(st));
  ph.mark("records");
  return bottomup ? GT_BOTTOMUP : (sparse ? GT_TOPDOWN_SPARSE : GT_TOPDOWN);
}

}  // namespace gt
