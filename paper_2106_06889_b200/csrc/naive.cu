// naive.cu — decompress-then-count on the device: the reference's naive
// counterparts (oracle_task, tasks.py:191-227; oracle.py:19-60) as an
// independent ground truth at the corpus sizes the CPU oracles cannot hold
// (SURVEY.md §8f rank 2).  It never touches the compressed-domain engine:
// the grammar is expanded into the token stream (chunked by files), tokens
// and windows are counted by radix sort + run-length encoding, and the
// results are ordered for render exactly like the compressed path's, so the
// two can be compared array for array.  Verification only: gt_run never
// calls into this file.
//
// Expansion: every root position gets its token offset (exclusive scan of
// word = 1 / rule = exp_len / splitter = 0); rule occurrences longer than a
// threshold are split one body level at a time (offsets from a per-body
// prefix of symbol lengths), shorter ones are expanded by one thread each
// with an explicit stack.
#include <algorithm>
#include <vector>

#include "kernels_common.cuh"
#include "naive.cuh"

namespace gt {

namespace {

constexpr u64 kSmall = 512;  // rule occurrences at most this long: one thread

__global__ void k_sym_len(const u32* body, u64 n, u64 nw, u64 base, const u64* exp_len, u64* len) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 s = body[i];
    len[i] = s < nw ? 1ull : (s >= base ? exp_len[s - base] : 0ull);
  }
}

// per-body exclusive prefix: pre[q] = S[q] - S[boff[owner[q]]]
__global__ void k_body_prefix(const u64* S, const u32* owner, const u64* boff, u64 n, u64* pre) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) pre[q] = S[q] - S[boff[owner[q]]];
}

// root positions [a, b): words are written, rule occurrences become items
__global__ void k_root_items(const u32* body, u64 a, u64 b, const u64* pre, u64 base_off, u64 nw, u64 base,
                             u32* tok, u32* it_rule, u64* it_off, u64* nit) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = a + (u64)blockIdx.x * blockDim.x + threadIdx.x; p < b; p += stride) {
    const u32 s = body[p];
    const u64 o = pre[p] - base_off;
    if (s < nw) tok[o] = s;
    else if (s >= base) {
      const u64 k = atomicAdd((unsigned long long*)nit, 1ull);
      it_rule[k] = s - (u32)base;
      it_off[k] = o;
    }
  }
}

// one level of splitting: body symbols of the big items (edge-balanced over
// the bodies); small rule occurrences go to the final list
__global__ void k_split(const u32* it_rule, const u64* it_off, u64 nit, const u64* pos, const u64* blen,
                        const u32* body, const u64* boff, const u64* pre, const u64* exp_len, u64 nw, u64 base,
                        u32* tok, u32* big_rule, u64* big_off, u64* nbig, u32* sm_rule, u64* sm_off, u64* nsm) {
  if (!nit) return;
  const u64 T = pos[nit - 1] + blen[nit - 1];
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < T; i += stride) {
    u64 lo = 0, hi = nit;
    while (hi - lo > 1) {
      const u64 m = (lo + hi) >> 1;
      if (pos[m] <= i) lo = m;
      else hi = m;
    }
    const u32 r = it_rule[lo];
    const u64 q = boff[r] + (i - pos[lo]);
    const u32 s = body[q];
    const u64 o = it_off[lo] + pre[q];
    if (s < nw) {
      tok[o] = s;
    } else if (s >= base) {
      const u32 c = s - (u32)base;
      if (exp_len[c] > kSmall) {
        const u64 k = atomicAdd((unsigned long long*)nbig, 1ull);
        big_rule[k] = c;
        big_off[k] = o;
      } else {
        const u64 k = atomicAdd((unsigned long long*)nsm, 1ull);
        sm_rule[k] = c;
        sm_off[k] = o;
      }
    }
  }
}

__global__ void k_classify(const u32* it_rule, const u64* it_off, u64 n, const u64* exp_len, u32* big_rule,
                           u64* big_off, u64* nbig, u32* sm_rule, u64* sm_off, u64* nsm) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 r = it_rule[i];
    if (exp_len[r] > kSmall) {
      const u64 k = atomicAdd((unsigned long long*)nbig, 1ull);
      big_rule[k] = r;
      big_off[k] = it_off[i];
    } else {
      const u64 k = atomicAdd((unsigned long long*)nsm, 1ull);
      sm_rule[k] = r;
      sm_off[k] = it_off[i];
    }
  }
}

__global__ void k_item_blen(const u32* rule, u64 n, const u64* boff, u64* blen) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    blen[i] = boff[rule[i] + 1] - boff[rule[i]];
}

// a short occurrence expanded by one thread (explicit stack; depth <= 64)
__global__ void k_expand_small(const u32* rule, const u64* off, u64 n, const u32* body, const u64* boff, u64 nw,
                               u64 base, u32* tok) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u64 sq[64];
    u64 se[64];
    int sp = 0;
    sq[0] = boff[rule[i]];
    se[0] = boff[rule[i] + 1];
    u64 o = off[i];
    while (sp >= 0) {
      if (sq[sp] == se[sp]) {
        sp--;
        continue;
      }
      const u32 s = body[sq[sp]++];
      if (s < nw) tok[o++] = s;
      else if (s >= base) {
        const u32 c = s - (u32)base;
        sp++;
        sq[sp] = boff[c];
        se[sp] = boff[c + 1];
      }
    }
  }
}

// per token: (file << WB) | word; per window: (file << GB) | packed gram
__global__ void k_token_keys(const u32* tok, u64 n, const u64* fstart, u32 nf, int WB, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 lo = 0, hi = nf;
    while (hi - lo > 1) {
      const u32 m = (lo + hi) >> 1;
      if (fstart[m] <= i) lo = m;
      else hi = m;
    }
    key[i] = ((u64)lo << WB) | tok[i];
  }
}

__global__ void k_window_keys(const u32* tok, u64 n, const u64* fstart, const u64* fend, u32 nf, u32 l, int wbits,
                              int GB, u64* key, uint8_t* valid) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 lo = 0, hi = nf;
    while (hi - lo > 1) {
      const u32 m = (lo + hi) >> 1;
      if (fstart[m] <= i) lo = m;
      else hi = m;
    }
    const bool ok = i + l <= fend[lo];
    u64 g = 0;
    if (ok)
      for (u32 j = 0; j < l; j++) g = (g << wbits) | tok[i + j];
    key[i] = ((u64)lo << GB) | g;
    valid[i] = ok;
  }
}

// ---- wide grams (64 < l * wbits <= 128): (hi, lo) keys, file sorted apart --
__device__ __forceinline__ void shl128(u64& hi, u64& lo, int s, u64 v) {  // (hi:lo) = (hi:lo) << s | v
  hi = s >= 64 ? (lo << (s - 64)) : ((hi << s) | (s ? (lo >> (64 - s)) : 0ull));
  lo = s >= 64 ? 0ull : (lo << s);
  lo |= v;
}

__global__ void k_window_keys_wide(const u32* tok, u64 n, const u64* fstart, const u64* fend, u32 nf, u32 l,
                                   int wbits, u64* khi, u64* klo, u32* kfile, uint8_t* valid) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 lo = 0, hi = nf;
    while (hi - lo > 1) {
      const u32 m = (lo + hi) >> 1;
      if (fstart[m] <= i) lo = m;
      else hi = m;
    }
    const bool ok = i + l <= fend[lo];
    u64 gh = 0, gl = 0;
    if (ok)
      for (u32 j = 0; j < l; j++) shl128(gh, gl, wbits, tok[i + j]);
    khi[i] = gh;
    klo[i] = gl;
    kfile[i] = lo;
    valid[i] = ok;
  }
}

__global__ void k_heads_wide(const u32* f, const u64* hi, const u64* lo, u64 n, uint8_t* h) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    h[i] = i == 0 || f[i] != f[i - 1] || hi[i] != hi[i - 1] || lo[i] != lo[i - 1];
}

__global__ void k_heads_wide2(const u64* hi, const u64* lo, u64 n, uint8_t* h) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    h[i] = i == 0 || hi[i] != hi[i - 1] || lo[i] != lo[i - 1];
}

__global__ void k_runs_wide(const u32* f, const u64* hi, const u64* lo, const u32* hidx, u64 U, u64 n, u32 add_file,
                            u32* ofile, u64* ohi, u64* olo, u64* ocnt) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += stride) {
    const u64 a = hidx[u], b = u + 1 < U ? hidx[u + 1] : n;
    ofile[u] = f[a] + add_file;
    ohi[u] = hi[a];
    olo[u] = lo[a];
    ocnt[u] = b - a;
  }
}

// (hi:lo) of record idx[i] -> its l word ids (big-endian by position)
__global__ void k_decode_wide(const u32* idx, u64 n, const u64* hi, const u64* lo, u32 l, int wbits, u32* gram) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 m = (1ull << wbits) - 1;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 k = idx ? idx[i] : (u32)i;
    const u64 h = hi[k], o = lo[k];
    for (u32 j = 0; j < l; j++) {
      const int sh = (int)(l - 1 - j) * wbits;
      u64 w;
      if (sh >= 64) w = h >> (sh - 64);
      else if (sh + wbits <= 64) w = o >> sh;
      else w = (o >> sh) | (h << (64 - sh));
      gram[i * l + j] = (u32)(w & m);
    }
  }
}

__global__ void k_heads64(const u64* k, u64 n, uint8_t* h) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) h[i] = i == 0 || k[i] != k[i - 1];
}

// runs of the sorted keys -> (file relative to file_lo, low key, count)
__global__ void k_runs(const u64* sk, const u32* hidx, u64 U, u64 n, u32 add_file, int SH, u32* ofile, u64* olow,
                       u64* ocnt) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 m = SH >= 64 ? ~0ull : ((1ull << SH) - 1);
  for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += stride) {
    const u64 a = hidx[u], b = u + 1 < U ? hidx[u + 1] : n;
    const u64 k = sk[a];
    ofile[u] = (u32)(k >> SH) + add_file;
    olow[u] = k & m;
    ocnt[u] = b - a;
  }
}

__global__ void k_files_counts_key(const u32* file, const u64* inv_cnt, u64 n, int CB, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    key[i] = ((u64)file[i] << CB) | inv_cnt[i];
}

__global__ void k_add_dense(const u64* word, const u64* cnt, u64 n, u64* dense) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd((unsigned long long*)&dense[word[i]], (unsigned long long)cnt[i]);
}

__global__ void k_inv_count_key(const u64* cnt, u64 n, u64 W, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) key[i] = W - cnt[i];
}

__global__ void k_gather64(const u32* idx, u64 n, const u64* a, u64* b) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[idx[i]];
}

__global__ void k_gather32(const u32* idx, u64 n, const u32* a, u32* b) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[idx[i]];
}

__global__ void k_iota32(u32* a, u64 n) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = (u32)i;
}

__global__ void k_lo32(const u64* a, u64 n, u32* b) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = (u32)a[i];
}

__global__ void k_add32(u32* a, u64 n, u32 v) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] += v;
}

__global__ void k_group_heads_u32(const u32* g, u64 n, uint8_t* h) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) h[i] = i == 0 || g[i] != g[i - 1];
}

__global__ void k_group_heads_u64(const u64* g, u64 n, uint8_t* h) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) h[i] = i == 0 || g[i] != g[i - 1];
}

__global__ void k_groups_out(const u32* sel, const u64* ng, u64 n, const u32* gid32, const u64* gid64, u32* o32,
                             u64* o64, u64* goff) {
  const u64 G = *ng;
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g <= G; g += stride) {
    if (g == G) {
      goff[g] = n;
      continue;
    }
    goff[g] = sel[g];
    if (o32) o32[g] = gid32[sel[g]];
    if (o64) o64[g] = gid64[sel[g]];
  }
}

#define NK(k, n, ...) GT_KLAUNCH(#k, k, grid_for((n), 256), 256, st, __VA_ARGS__)

template <class T>
T rd(const void* p, cudaStream_t st) {
  T v;
  GT_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  return v;
}

}  // namespace

void naive_run(DeviceDag* d, int task, int l_, DevRecords* Rr, int* wbits_out, const uint32_t* htok,
               const uint64_t* hoff) {
  cudaStream_t st = d->stream;
  const u64 E = d->E, nw = d->nw, base = d->nw + d->ns, V = d->nw;
  const u32 nseg = (u32)(d->file_hi - d->file_lo);
  const u32 l = (u32)l_;
  const int WB = std::max(1, bitlen(nw ? nw - 1 : 0));
  const bool gram_task = task == GT_SEQCOUNT || task == GT_RANKEDINVERTEDINDEX;
  const int wbits = std::max(1, bitlen(nw ? nw - 1 : 1));
  // grams wider than 63 bits (the compressed path's gram mode) are counted on
  // 128-bit (hi, lo) keys with the file sorted apart
  const bool wide = gram_task && (u64)l * wbits > 63;
  if (gram_task && (u64)l * wbits > 128)
    fail(GT_E_USAGE, "naive sequence counting supports grams of at most 128 bits (%u words of %d bits)", l, wbits);
  *wbits_out = gram_task && !wide ? wbits : 0;
  const bool text = htok != nullptr;  // count given token streams, no expansion
  std::vector<u64> seg_lo, seg_hi;
  // per-body symbol-length prefixes and root token offsets
  DBuf len, S, pre;
  std::vector<u64> ftok(nseg + 1), fend(nseg);
  if (text) {
    for (u32 f = 0; f < nseg; f++) {
      ftok[f] = hoff[d->file_lo + f];
      fend[f] = hoff[d->file_lo + f + 1];
    }
  } else {
  len.alloc(E * 8 + 8, st);
  S.alloc(E * 8 + 8, st);
  pre.alloc(E * 8 + 8, st);
  NK(k_sym_len, E, d->body.as<u32>(), E, nw, base, d->exp_len.as<u64>(), len.as<u64>());
  GT_CUDA(cudaMemsetAsync(len.as<u64>() + E, 0, 8, st));
  exclusive_scan_u64(len.as<u64>(), S.as<u64>(), E + 1, st);
  NK(k_body_prefix, E, S.as<u64>(), d->pos_owner.as<u32>(), d->boff.as<u64>(), E, pre.as<u64>());
  len.release();
  S.release();
  seg_lo.resize(d->F);
  seg_hi.resize(d->F);
  GT_CUDA(cudaMemcpyAsync(seg_lo.data(), d->seg_lo.p, d->F * 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(seg_hi.data(), d->seg_hi.p, d->F * 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  // token offset of root position p = pre[p] (the root is rule 0); a file
  // ends where its splitter (length 0) starts
  std::vector<u64> root_pre(d->L0 + 1);
  if (d->L0) GT_CUDA(cudaMemcpyAsync(root_pre.data(), pre.p, d->L0 * 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaStreamSynchronize(st));
  root_pre[d->L0] = d->W;
  for (u32 f = 0; f < nseg; f++) {
    ftok[f] = root_pre[seg_lo[d->file_lo + f]];
    fend[f] = root_pre[std::min<u64>(seg_hi[d->file_lo + f], d->L0)];
  }
  }
  const u64 kChunk = 1ull << 29;  // tokens per chunk (4 bytes each)
  DBuf dense;
  if (task == GT_WORDCOUNT || task == GT_SORT) {
    dense.alloc(V * 8 + 8, st);
    GT_CUDA(cudaMemsetAsync(dense.p, 0, V * 8 + 8, st));
  }
  std::vector<DBuf> rf, rk, rc, rh;  // per-chunk (file, low key, count[, high key]) records
  std::vector<u64> rn;
  const int FB = std::max(1, bitlen(nseg ? nseg - 1 : 0));
  u32 f0 = 0;
  while (f0 < nseg) {
    // files per chunk: bounded by tokens and, for windows, by the key bits
    // left above the packed gram (file bits + l*wbits <= 64)
    u64 max_files = ~0ull;
    if (gram_task && !wide && (u64)l * wbits < 64) {
      const int free_bits = 64 - (int)(l * wbits);
      max_files = free_bits >= 32 ? ~0ull : (1ull << free_bits);
    } else if (gram_task && !wide) {
      max_files = 1;
    }
    u32 f1 = f0 + 1;
    while (f1 < nseg && fend[f1] - ftok[f0] <= kChunk && (u64)(f1 + 1 - f0) <= max_files) f1++;
    const u64 t0 = ftok[f0], ntok = fend[f1 - 1] - t0;
    const u32 nf = f1 - f0;
    DBuf tok(ntok * 4 + 4, st), fstart(nf * 8 + 8, st), fendd(nf * 8 + 8, st);
    {
      std::vector<u64> a(nf), b(nf);
      for (u32 k = 0; k < nf; k++) a[k] = ftok[f0 + k] - t0, b[k] = fend[f0 + k] - t0;
      GT_CUDA(cudaMemcpyAsync(fstart.p, a.data(), nf * 8, cudaMemcpyHostToDevice, st));
      GT_CUDA(cudaMemcpyAsync(fendd.p, b.data(), nf * 8, cudaMemcpyHostToDevice, st));
      GT_CUDA(cudaStreamSynchronize(st));
    }
    DBuf cnt(32, st);
    if (text) {
      GT_CUDA(cudaMemcpyAsync(tok.p, htok + t0, ntok * 4, cudaMemcpyHostToDevice, st));
    } else {
    // expansion of root positions [seg_lo[f0], seg_hi[f1-1])
    const u64 pa = seg_lo[d->file_lo + f0], pb = seg_hi[d->file_lo + f1 - 1];
    const u64 cap = std::max<u64>(pb - pa, 1);
    DBuf ir(cap * 4, st), io(cap * 8, st);
    GT_CUDA(cudaMemsetAsync(cnt.p, 0, 32, st));
    if (pb > pa)
      NK(k_root_items, pb - pa, d->body.as<u32>(), pa, pb, pre.as<u64>(), t0, nw, base, tok.as<u32>(),
         ir.as<u32>(), io.as<u64>(), cnt.as<u64>());
    u64 nit = rd<u64>(cnt.p, st);
    // classify the root items, then split big ones level by level
    std::vector<std::pair<DBuf, DBuf>> smalls;
    std::vector<u64> nsmalls;
    {
      DBuf br(nit * 4 + 4, st), bo(nit * 8 + 8, st), sr(nit * 4 + 4, st), so(nit * 8 + 8, st);
      GT_CUDA(cudaMemsetAsync(cnt.p, 0, 32, st));
      if (nit)
        NK(k_classify, nit, ir.as<u32>(), io.as<u64>(), nit, d->exp_len.as<u64>(), br.as<u32>(), bo.as<u64>(),
           cnt.as<u64>(), sr.as<u32>(), so.as<u64>(), cnt.as<u64>() + 1);
      u64 h[2];
      GT_CUDA(cudaMemcpyAsync(h, cnt.p, 16, cudaMemcpyDeviceToHost, st));
      GT_CUDA(cudaStreamSynchronize(st));
      nit = h[0];
      smalls.emplace_back(std::move(sr), std::move(so));
      nsmalls.push_back(h[1]);
      ir = std::move(br);
      io = std::move(bo);
    }
    while (nit) {
      DBuf bl(nit * 8 + 8, st), ps(nit * 8 + 8, st);
      NK(k_item_blen, nit, ir.as<u32>(), nit, d->boff.as<u64>(), bl.as<u64>());
      exclusive_scan_u64(bl.as<u64>(), ps.as<u64>(), nit, st);
      const u64 T = rd<u64>(ps.as<u64>() + nit - 1, st) + rd<u64>(bl.as<u64>() + nit - 1, st);
      DBuf br(T * 4 + 4, st), bo(T * 8 + 8, st), sr(T * 4 + 4, st), so(T * 8 + 8, st);
      GT_CUDA(cudaMemsetAsync(cnt.p, 0, 32, st));
      GT_KLAUNCH("k_split", k_split, 148u * 16u, 256, st, ir.as<u32>(), io.as<u64>(), nit, ps.as<u64>(),
                 bl.as<u64>(), d->body.as<u32>(), d->boff.as<u64>(), pre.as<u64>(), d->exp_len.as<u64>(), nw,
                 base, tok.as<u32>(), br.as<u32>(), bo.as<u64>(), cnt.as<u64>(), sr.as<u32>(), so.as<u64>(),
                 cnt.as<u64>() + 1);
      u64 h[2];
      GT_CUDA(cudaMemcpyAsync(h, cnt.p, 16, cudaMemcpyDeviceToHost, st));
      GT_CUDA(cudaStreamSynchronize(st));
      smalls.emplace_back(std::move(sr), std::move(so));
      nsmalls.push_back(h[1]);
      ir = std::move(br);
      io = std::move(bo);
      nit = h[0];
    }
    for (size_t k = 0; k < smalls.size(); k++)
      if (nsmalls[k])
        NK(k_expand_small, nsmalls[k], smalls[k].first.as<u32>(), smalls[k].second.as<u64>(), nsmalls[k],
           d->body.as<u32>(), d->boff.as<u64>(), nw, base, tok.as<u32>());
    smalls.clear();
    }
    // counting
    if (wide) {
      // valid windows -> (file, hi, lo) sorted LSD: lo, hi, file (stable radix
      // passes carrying the window index), then runs
      const int GB = (int)(l * wbits), FB = std::max(1, bitlen(nf ? nf - 1 : 0));
      DBuf khi(ntok * 8 + 8, st), klo(ntok * 8 + 8, st), kf(ntok * 4 + 4, st), val(ntok + 1, st);
      NK(k_window_keys_wide, ntok, tok.as<u32>(), ntok, fstart.as<u64>(), fendd.as<u64>(), nf, l, wbits,
         khi.as<u64>(), klo.as<u64>(), kf.as<u32>(), val.as<uint8_t>());
      tok.release();
      DBuf p0(ntok * 4 + 4, st), p1(ntok * 4 + 4, st), a(ntok * 8 + 8, st), b(ntok * 8 + 8, st);
      select_flagged_index(val.as<uint8_t>(), p0.as<u32>(), cnt.as<u64>(), ntok, st);
      const u64 nk = rd<u64>(cnt.p, st);
      NK(k_gather64, nk, p0.as<u32>(), nk, klo.as<u64>(), a.as<u64>());
      sort_pairs_u64_u32(a.as<u64>(), b.as<u64>(), p0.as<u32>(), p1.as<u32>(), nk, 64, st);
      NK(k_gather64, nk, p1.as<u32>(), nk, khi.as<u64>(), a.as<u64>());
      sort_pairs_u64_u32(a.as<u64>(), b.as<u64>(), p1.as<u32>(), p0.as<u32>(), nk, std::max(1, GB - 64), st);
      DBuf f1b(ntok * 4 + 4, st), f2b(ntok * 4 + 4, st);
      NK(k_gather32, nk, p0.as<u32>(), nk, kf.as<u32>(), f1b.as<u32>());
      sort_pairs_u32_u32(f1b.as<u32>(), f2b.as<u32>(), p0.as<u32>(), p1.as<u32>(), nk, FB, st);
      // p1: window order by (file, hi, lo); f2b: the sorted files
      NK(k_gather64, nk, p1.as<u32>(), nk, khi.as<u64>(), a.as<u64>());
      NK(k_gather64, nk, p1.as<u32>(), nk, klo.as<u64>(), b.as<u64>());
      DBuf hd(nk + 1, st), hidx(nk * 4 + 4, st);
      NK(k_heads_wide, nk, f2b.as<u32>(), a.as<u64>(), b.as<u64>(), nk, hd.as<uint8_t>());
      select_flagged_index(hd.as<uint8_t>(), hidx.as<u32>(), cnt.as<u64>(), nk, st);
      const u64 U = rd<u64>(cnt.p, st);
      DBuf of(U * 4 + 4, st), oh(U * 8 + 8, st), ol(U * 8 + 8, st), oc(U * 8 + 8, st);
      NK(k_runs_wide, U, f2b.as<u32>(), a.as<u64>(), b.as<u64>(), hidx.as<u32>(), U, nk, f0, of.as<u32>(),
         oh.as<u64>(), ol.as<u64>(), oc.as<u64>());
      rf.push_back(std::move(of));
      rk.push_back(std::move(ol));
      rh.push_back(std::move(oh));
      rc.push_back(std::move(oc));
      rn.push_back(U);
      f0 = f1;
      continue;
    }
    DBuf keys, valid;
    u64 nk = ntok;
    int kbits;
    if (gram_task) {
      keys.alloc(ntok * 8 + 8, st);
      valid.alloc(ntok + 1, st);
      NK(k_window_keys, ntok, tok.as<u32>(), ntok, fstart.as<u64>(), fendd.as<u64>(), nf, l, wbits,
         (int)(l * wbits), keys.as<u64>(), valid.as<uint8_t>());
      // drop the windows that would cross a file end
      DBuf sel(ntok * 4 + 4, st), k2(ntok * 8 + 8, st);
      select_flagged_index(valid.as<uint8_t>(), sel.as<u32>(), cnt.as<u64>(), ntok, st);
      nk = rd<u64>(cnt.p, st);
      NK(k_gather64, nk, sel.as<u32>(), nk, keys.as<u64>(), k2.as<u64>());
      keys = std::move(k2);
      kbits = (int)(l * wbits) + std::max(1, bitlen(nf ? nf - 1 : 0));
      if (kbits > 64) fail(GT_E_USAGE, "naive sequence counting: chunk file bits + gram bits exceed 64");
    } else {
      keys.alloc(ntok * 8 + 8, st);
      NK(k_token_keys, ntok, tok.as<u32>(), ntok, fstart.as<u64>(), nf, WB, keys.as<u64>());
      kbits = WB + std::max(1, bitlen(nf ? nf - 1 : 0));
    }
    tok.release();
    DBuf sk(nk * 8 + 8, st), hd(nk + 1, st), hidx(nk * 4 + 4, st);
    sort_keys_u64(keys.as<u64>(), sk.as<u64>(), nk, kbits, st);
    keys.release();
    NK(k_heads64, nk, sk.as<u64>(), nk, hd.as<uint8_t>());
    select_flagged_index(hd.as<uint8_t>(), hidx.as<u32>(), cnt.as<u64>(), nk, st);
    const u64 U = rd<u64>(cnt.p, st);
    DBuf of(U * 4 + 4, st), ok(U * 8 + 8, st), oc(U * 8 + 8, st);
    const int SH = gram_task ? (int)(l * wbits) : WB;
    NK(k_runs, U, sk.as<u64>(), hidx.as<u32>(), U, nk, f0, SH, of.as<u32>(), ok.as<u64>(), oc.as<u64>());
    if (task == GT_WORDCOUNT || task == GT_SORT) {
      NK(k_add_dense, U, ok.as<u64>(), oc.as<u64>(), U, dense.as<u64>());
    } else {
      rf.push_back(std::move(of));
      rk.push_back(std::move(ok));
      rc.push_back(std::move(oc));
      rn.push_back(U);
    }
    f0 = f1;
  }
  pre.release();
  if (task == GT_WORDCOUNT || task == GT_SORT) {
    assemble_counts(d, dense.as<u64>(), V, 0, task == GT_SORT, Rr);
    return;
  }
  // concatenate the chunks' (file, word-or-gram, count) records: already in
  // (file, word-or-gram) order
  u64 n = 0;
  for (u64 x : rn) n += x;
  DBuf file(n * 4 + 4, st), low(n * 8 + 8, st), count(n * 8 + 8, st), high(wide ? n * 8 + 8 : 8, st);
  {
    u64 o = 0;
    for (size_t k = 0; k < rk.size(); k++) {
      if (rn[k]) {
        GT_CUDA(cudaMemcpyAsync(file.as<u32>() + o, rf[k].p, rn[k] * 4, cudaMemcpyDeviceToDevice, st));
        GT_CUDA(cudaMemcpyAsync(low.as<u64>() + o, rk[k].p, rn[k] * 8, cudaMemcpyDeviceToDevice, st));
        GT_CUDA(cudaMemcpyAsync(count.as<u64>() + o, rc[k].p, rn[k] * 8, cudaMemcpyDeviceToDevice, st));
        if (wide) GT_CUDA(cudaMemcpyAsync(high.as<u64>() + o, rh[k].p, rn[k] * 8, cudaMemcpyDeviceToDevice, st));
      }
      o += rn[k];
    }
    rf.clear();
    rk.clear();
    rc.clear();
    rh.clear();
  }
  const int SH = gram_task ? (int)(l * wbits) : WB;
  const u64 Wt = text ? std::max<u64>(hoff[d->F], 1) : d->W;
  const int CB = std::max(1, bitlen(Wt));
  DBuf idx(n * 4 + 4, st), idx2(n * 4 + 4, st), k1(n * 8 + 8, st), k2(n * 8 + 8, st);
  NK(k_iota32, n, idx.as<u32>(), n);
  Rr->n = n;
  if (task == GT_TERMVECTOR || task == GT_SEQCOUNT) {
    // per file: (-count, word-or-gram), stable over the (file, key) order
    NK(k_inv_count_key, n, count.as<u64>(), n, Wt, k1.as<u64>());
    DBuf kk(n * 8 + 8, st);  // (file << CB) | (W - count)
    NK(k_files_counts_key, n, file.as<u32>(), k1.as<u64>(), n, CB, kk.as<u64>());
    sort_pairs_u64_u32(kk.as<u64>(), k2.as<u64>(), idx.as<u32>(), idx2.as<u32>(), n, CB + FB, st);
    Rr->count.alloc(n * 8 + 8, st);
    NK(k_gather64, n, idx2.as<u32>(), n, count.as<u64>(), Rr->count.as<u64>());
    DBuf f2(n * 4 + 4, st);
    NK(k_gather32, n, idx2.as<u32>(), n, file.as<u32>(), f2.as<u32>());
    if (task == GT_TERMVECTOR) {
      DBuf w32(n * 4 + 4, st);
      NK(k_lo32, n, low.as<u64>(), n, w32.as<u32>());
      Rr->id.alloc(n * 4 + 4, st);
      NK(k_gather32, n, idx2.as<u32>(), n, w32.as<u32>(), Rr->id.as<u32>());
    } else if (wide) {
      Rr->gram.alloc(n * l * 4 + 4, st);
      NK(k_decode_wide, n, idx2.as<u32>(), n, high.as<u64>(), low.as<u64>(), l, wbits, Rr->gram.as<u32>());
    } else {
      Rr->key.alloc(n * 8 + 8, st);
      NK(k_gather64, n, idx2.as<u32>(), n, low.as<u64>(), Rr->key.as<u64>());
    }
    Rr->n_groups = nseg;
    Rr->group_off.alloc(((u64)nseg + 1) * 8, st);
    NK(k_csr_offsets, (u64)nseg + 1, f2.as<u32>(), n, (u64)nseg, Rr->group_off.as<u64>());
  } else if (task == GT_INVERTEDINDEX) {
    // by (word, file): LSD, the records are in (file, word) order
    DBuf w32(n * 4 + 4, st), w2(n * 4 + 4, st);
    NK(k_lo32, n, low.as<u64>(), n, w32.as<u32>());
    sort_pairs_u32_u32(w32.as<u32>(), w2.as<u32>(), idx.as<u32>(), idx2.as<u32>(), n, WB, st);
    Rr->id.alloc(n * 4 + 4, st);
    NK(k_gather32, n, idx2.as<u32>(), n, file.as<u32>(), Rr->id.as<u32>());
    NK(k_add32, n, Rr->id.as<u32>(), n, (u32)d->file_lo);
    DBuf hd(n + 1, st), sel(n * 4 + 4, st), ng(8, st);
    NK(k_group_heads_u32, n, w2.as<u32>(), n, hd.as<uint8_t>());
    select_flagged_index(hd.as<uint8_t>(), sel.as<u32>(), ng.as<u64>(), n, st);
    const u64 G = rd<u64>(ng.p, st);
    Rr->n_groups = G;
    Rr->group_id.alloc(G * 4 + 4, st);
    Rr->group_off.alloc((G + 1) * 8, st);
    NK(k_groups_out, G + 1, sel.as<u32>(), ng.as<u64>(), n, w2.as<u32>(), (const u64*)nullptr,
       Rr->group_id.as<u32>(), (u64*)nullptr, Rr->group_off.as<u64>());
  } else if (wide) {
    // ranked inverted index on wide grams: LSD by W - count, then lo, then hi
    NK(k_inv_count_key, n, count.as<u64>(), n, Wt, k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), idx.as<u32>(), idx2.as<u32>(), n, CB, st);
    NK(k_gather64, n, idx2.as<u32>(), n, low.as<u64>(), k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), idx2.as<u32>(), idx.as<u32>(), n, 64, st);
    NK(k_gather64, n, idx.as<u32>(), n, high.as<u64>(), k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), idx.as<u32>(), idx2.as<u32>(), n, std::max(1, (int)(l * wbits) - 64), st);
    // idx2: the final order
    Rr->count.alloc(n * 8 + 8, st);
    NK(k_gather64, n, idx2.as<u32>(), n, count.as<u64>(), Rr->count.as<u64>());
    Rr->id.alloc(n * 4 + 4, st);
    NK(k_gather32, n, idx2.as<u32>(), n, file.as<u32>(), Rr->id.as<u32>());
    NK(k_add32, n, Rr->id.as<u32>(), n, (u32)d->file_lo);
    DBuf sh(n * 8 + 8, st), sl(n * 8 + 8, st);
    NK(k_gather64, n, idx2.as<u32>(), n, high.as<u64>(), sh.as<u64>());
    NK(k_gather64, n, idx2.as<u32>(), n, low.as<u64>(), sl.as<u64>());
    DBuf hd(n + 1, st), sel(n * 4 + 4, st), ng(8, st);
    NK(k_heads_wide2, n, sh.as<u64>(), sl.as<u64>(), n, hd.as<uint8_t>());
    select_flagged_index(hd.as<uint8_t>(), sel.as<u32>(), ng.as<u64>(), n, st);
    const u64 G = rd<u64>(ng.p, st);
    Rr->n_groups = G;
    Rr->group_gram.alloc(G * l * 4 + 4, st);
    Rr->group_off.alloc((G + 1) * 8, st);
    NK(k_groups_out, G + 1, sel.as<u32>(), ng.as<u64>(), n, (const u32*)nullptr, (const u64*)nullptr,
       (u32*)nullptr, (u64*)nullptr, Rr->group_off.as<u64>());
    NK(k_decode_wide, G, sel.as<u32>(), G, sh.as<u64>(), sl.as<u64>(), l, wbits, Rr->group_gram.as<u32>());
  } else {
    // ranked inverted index: gram asc, then (-count, file): LSD over the
    // (file, gram)-ordered records: by W - count, then by gram
    NK(k_inv_count_key, n, count.as<u64>(), n, Wt, k1.as<u64>());
    sort_pairs_u64_u32(k1.as<u64>(), k2.as<u64>(), idx.as<u32>(), idx2.as<u32>(), n, CB, st);
    DBuf g1(n * 8 + 8, st), g2(n * 8 + 8, st);
    NK(k_gather64, n, idx2.as<u32>(), n, low.as<u64>(), g1.as<u64>());
    sort_pairs_u64_u32(g1.as<u64>(), g2.as<u64>(), idx2.as<u32>(), idx.as<u32>(), n, SH, st);
    Rr->count.alloc(n * 8 + 8, st);
    NK(k_gather64, n, idx.as<u32>(), n, count.as<u64>(), Rr->count.as<u64>());
    Rr->id.alloc(n * 4 + 4, st);
    NK(k_gather32, n, idx.as<u32>(), n, file.as<u32>(), Rr->id.as<u32>());
    NK(k_add32, n, Rr->id.as<u32>(), n, (u32)d->file_lo);
    DBuf hd(n + 1, st), sel(n * 4 + 4, st), ng(8, st);
    NK(k_group_heads_u64, n, g2.as<u64>(), n, hd.as<uint8_t>());
    select_flagged_index(hd.as<uint8_t>(), sel.as<u32>(), ng.as<u64>(), n, st);
    const u64 G = rd<u64>(ng.p, st);
    Rr->n_groups = G;
    Rr->group_key.alloc(G * 8 + 8, st);
    Rr->group_off.alloc((G + 1) * 8, st);
    NK(k_groups_out, G + 1, sel.as<u32>(), ng.as<u64>(), n, (const u32*)nullptr, g2.as<u64>(), (u32*)nullptr,
       Rr->group_key.as<u64>(), Rr->group_off.as<u64>());
  }
  GT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gt
