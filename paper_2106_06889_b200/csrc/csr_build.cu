// csr_build.cu — per-rule (symbol, multiplicity) lists: the own / sub CSR of
// dag.py:131-230 (own_ids/own_freqs: distinct words of a body with their
// counts, ascending; sub_ids/sub_freqs: distinct child rules) built without a
// global sort of the grammar.
//
// Bodies are contiguous per rule, so the (rule, symbol) order only needs each
// body sorted by symbol.  Sequitur bodies are short (digram rules: 2 symbols;
// the composed configs: <= 6), so
//   * bodies of <= 32 symbols (all but a handful of rules) are sorted in
//     registers by one thread with a bitonic network and run-length encoded
//     on the spot;
//   * the root (rule 0, body positions [0, L0)) is sorted in place with one
//     32-bit radix sort; other bodies of 33..kGiant symbols go through a
//     segmented sort (CUB, only those segments), longer ones through one
//     radix sort of their (giant rank, symbol) keys; the runs of all long
//     bodies are then found element-parallel (head flags, select).
// Every rule writes its runs in place at its body offset (own words first,
// then the child rules: words sort below splitters below rules), the per-rule
// counts are scanned into own_off / sub_off directly, and one element-
// parallel pass compacts the runs into the CSR arrays.  own_tok (words in a
// body) and num_out (child references) fall out of the same pass.
#include <algorithm>

#include "kernels_common.cuh"

namespace gt {

constexpr u32 kShort = 32;
constexpr u64 kGiant = 4096;  // above: one device-wide radix sort (a block-per-segment sort of 10^5 is slow)

template <int N>
__device__ __forceinline__ void bitonic_sort(u32 (&v)[N]) {
#pragma unroll
  for (int k = 2; k <= N; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < N; i++) {
        const int l = i ^ j;
        if (l > i) {
          const u32 a = v[i], b = v[l];
          const u32 lo = a < b ? a : b, hi = a < b ? b : a;
          if ((i & k) == 0) {
            v[i] = lo;
            v[l] = hi;
          } else {
            v[i] = hi;
            v[l] = lo;
          }
        }
      }
}

struct RunOut {
  u32* tsym;
  u32* tcnt;
  u64 nw, base;
  u32 no = 0, nsu = 0;
  u64 otok = 0, nout = 0;
  u64 at;  // body offset of the rule
  __device__ __forceinline__ void emit(u32 sym, u32 c) {
    if (sym < nw) {
      tsym[at + no] = sym;
      tcnt[at + no] = c;
      no++;
      otok += c;
    } else if (sym >= base) {
      tsym[at + no + nsu] = (u32)(sym - base);
      tcnt[at + no + nsu] = c;
      nsu++;
      nout += c;
    }  // splitters (root only) are neither
  }
};

template <int N>
__device__ __forceinline__ void short_rule(const u32* __restrict__ body, u64 b, u32 len, RunOut& o) {
  u32 v[N];
#pragma unroll
  for (int i = 0; i < N; i++) v[i] = (u32)i < len ? body[b + i] : 0xFFFFFFFFu;
  bitonic_sort<N>(v);
  u32 cur = v[0], c = 1;
#pragma unroll
  for (int i = 1; i < N; i++) {
    if ((u32)i < len) {
      if (v[i] == cur) {
        c++;
      } else {
        o.emit(cur, c);
        cur = v[i];
        c = 1;
      }
    }
  }
  o.emit(cur, c);
}

// one thread per rule: short bodies done here; longer ones flagged
// (lflag: 1 = segmented sort, 2 = giant)
__global__ void k_rules_short(const u32* __restrict__ body, const u64* __restrict__ boff, u64 R, u64 nw, u64 base,
                              u32* tsym, u32* tcnt, u32* n_own, u32* n_sub, u64* own_tok, u64* num_out,
                              uint8_t* lflag, u32* nlong) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 r = (u64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride) {
    const u64 b = boff[r], len = boff[r + 1] - b;
    RunOut o{tsym, tcnt, nw, base};
    o.at = b;
    uint8_t f = 0;
    if (len == 0) {
    } else if (len <= 4) {
      short_rule<4>(body, b, (u32)len, o);
    } else if (len <= 8) {
      short_rule<8>(body, b, (u32)len, o);
    } else if (len <= 16) {
      short_rule<16>(body, b, (u32)len, o);
    } else if (len <= kShort) {
      short_rule<32>(body, b, (u32)len, o);
    } else {
      // the root (rule 0, body positions [0, L0)) is sorted on its own, in
      // place and without keys to gather: it is the one long body of a
      // Sequitur grammar
      f = r == 0 ? 3 : (len > kGiant ? 2 : 1);
      if (f != 3 && nlong) atomicAdd(nlong, 1u);
    }
    lflag[r] = f;
    n_own[r] = o.no;
    n_sub[r] = o.nsu;
    own_tok[r] = o.otok;
    num_out[r] = o.nout;
  }
}

__global__ void k_eq_u8(const uint8_t* a, u64 n, uint8_t v, uint8_t* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = a[i] == v;
}

__global__ void k_giant_elems(const u32* __restrict__ owner, const uint8_t* __restrict__ lflag, u64 E,
                              uint8_t* gflag) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += stride) gflag[p] = lflag[owner[p]] == 2;
}

__global__ void k_seg_bounds(const u32* __restrict__ ids, u64 n, const u64* __restrict__ boff, int* beg, int* end) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 r = ids[i];
    beg[i] = (int)boff[r];
    end[i] = (int)boff[r + 1];
  }
}

__global__ void k_scatter_rank(const u32* __restrict__ ids, u64 n, u32* rank) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) rank[ids[i]] = (u32)i;
}

// key = (rank of the giant rule, symbol): log2(#giants) + SB bits, so a
// single giant (the usual root) sorts on the symbol bits alone
__global__ void k_giant_keys(const u32* __restrict__ pos, u64 n, const u32* __restrict__ owner,
                             const u32* __restrict__ grank, const u32* __restrict__ body, int SB, u64* key) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 p = pos[i];
    key[i] = ((u64)grank[owner[p]] << SB) | body[p];
  }
}

// the sorted keys of the giant rules go back to their (contiguous, rule-
// ordered) positions
__global__ void k_giant_scatter(const u64* __restrict__ key, const u32* __restrict__ pos, u64 n, int SB, u32* sbody) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 m = (1ull << SB) - 1;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) sbody[pos[i]] = (u32)(key[i] & m);
}

__global__ void k_long_heads(const u32* __restrict__ owner, const uint8_t* __restrict__ lflag,
                             const u64* __restrict__ boff, const u32* __restrict__ sbody, u64 E, uint8_t* head) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += stride) {
    const u32 r = owner[p];
    head[p] = lflag[r] && (p == boff[r] || sbody[p - 1] != sbody[p]);
  }
}

// warp segmented sum over lanes with equal ascending keys; true on the last
// lane of each key run
__device__ __forceinline__ bool warp_key_sum(u32 key, u64& v) {
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const u64 ov = __shfl_up_sync(0xFFFFFFFFu, v, s);
    const u32 ok = __shfl_up_sync(0xFFFFFFFFu, key, s);
    if (lane >= (unsigned)s && ok == key) v += ov;
  }
  const u32 nk = __shfl_down_sync(0xFFFFFFFFu, key, 1);
  return lane == 31 || nk != key;
}

struct LongRun {
  u32 r, sym, cnt;
  bool ok;
};

__device__ __forceinline__ LongRun long_run(u64 u, u64 nh, const u32* hidx, const u32* owner, const u64* boff,
                                            const u32* sbody) {
  LongRun x{0xFFFFFFFFu, 0, 0, false};
  if (u >= nh) return x;
  const u32 j = hidx[u];
  x.r = owner[j];
  const u64 nx = (u + 1 < nh && owner[hidx[u + 1]] == x.r) ? hidx[u + 1] : boff[x.r + 1];
  x.cnt = (u32)(nx - j);
  x.sym = sbody[j];
  x.ok = true;
  return x;
}

// per long rule: runs by class (own / splitter / sub), symbol totals, and the
// index of its first run
__global__ void k_long_count(const u32* __restrict__ hidx, const u64* __restrict__ nh_d,
                             const u32* __restrict__ owner, const u64* __restrict__ boff,
                             const u32* __restrict__ sbody, u64 nw, u64 base, u32* n_own, u32* n_sub, u32* n_spl,
                             u64* own_tok, u64* num_out, u32* rfirst) {
  const u64 nh = *nh_d;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 b0 = (u64)blockIdx.x * blockDim.x; b0 < nh; b0 += stride) {
    const u64 u = b0 + threadIdx.x;
    const LongRun x = long_run(u, nh, hidx, owner, boff, sbody);
    if (x.ok && hidx[u] == boff[x.r]) rfirst[x.r] = (u32)u;
    const bool own = x.ok && x.sym < nw, sub = x.ok && x.sym >= base, spl = x.ok && !own && !sub;
    u64 a = own, b = sub, c = spl, t = own ? x.cnt : 0, o = sub ? x.cnt : 0;
    bool last = warp_key_sum(x.r, a);
    warp_key_sum(x.r, b);
    warp_key_sum(x.r, c);
    warp_key_sum(x.r, t);
    warp_key_sum(x.r, o);
    if (x.ok && last) {
      if (a) atomicAdd(&n_own[x.r], (u32)a);
      if (b) atomicAdd(&n_sub[x.r], (u32)b);
      if (c) atomicAdd(&n_spl[x.r], (u32)c);
      if (t) atomicAdd((unsigned long long*)&own_tok[x.r], (unsigned long long)t);
      if (o) atomicAdd((unsigned long long*)&num_out[x.r], (unsigned long long)o);
    }
  }
}

__global__ void k_long_write(const u32* __restrict__ hidx, const u64* __restrict__ nh_d,
                             const u32* __restrict__ owner, const u64* __restrict__ boff,
                             const u32* __restrict__ sbody, u64 nw, u64 base, const u32* __restrict__ n_spl,
                             const u32* __restrict__ rfirst, u32* tsym, u32* tcnt) {
  const u64 nh = *nh_d;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < nh; u += stride) {
    const LongRun x = long_run(u, nh, hidx, owner, boff, sbody);
    const u64 k = u - rfirst[x.r], at = boff[x.r];
    if (x.sym < nw) {
      tsym[at + k] = x.sym;
      tcnt[at + k] = x.cnt;
    } else if (x.sym >= base) {
      tsym[at + k - n_spl[x.r]] = (u32)(x.sym - base);
      tcnt[at + k - n_spl[x.r]] = x.cnt;
    }
  }
}

// The root's distinct symbols by a dense histogram over the symbol space
// when that space is not much larger than the root (C2: 9.4·10^5 symbols
// for a 5.5·10^4-symbol root, C3: 2.0·10^5 for 6.5·10^6): one memset, one
// atomic pass (one atomic per (warp, symbol)), one ordered select of the
// nonzero counts — instead of radix-sorting the root.
__global__ void k_root_hist(const u32* __restrict__ body, u64 L0, u32* hist) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 b = (u64)blockIdx.x * blockDim.x; b < L0; b += stride) {
    const u64 p = b + threadIdx.x;
    const bool ok = p < L0;
    const u32 sym = ok ? body[p] : 0xFFFFFFFFu;
    const unsigned same = __match_any_sync(0xFFFFFFFFu, sym);
    if (ok && (threadIdx.x & 31u) == (unsigned)(__ffs(same) - 1)) atomicAdd(&hist[sym], (u32)__popc(same));
  }
}

// the root's runs (ascending symbols: words, then rules; the splitter range
// was cleared) into its tsym / tcnt rows at body offset 0, and its counts
__global__ void k_root_runs(const u32* __restrict__ idx, const u64* __restrict__ n_dev,
                            const u32* __restrict__ hist, u64 nw, u64 base, u32* tsym, u32* tcnt, u32* n_own,
                            u32* n_sub, u64* own_tok, u64* num_out) {
  const u64 n = *n_dev;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 b = (u64)blockIdx.x * blockDim.x; b < n; b += stride) {
    const u64 u = b + threadIdx.x;
    u32 a = 0, c = 0;
    u64 t = 0, o = 0;
    if (u < n) {
      const u32 sym = idx[u], k = hist[sym];
      const bool own = sym < nw;
      tsym[u] = own ? sym : (u32)(sym - base);
      tcnt[u] = k;
      a = own, c = !own;
      t = own ? k : 0;
      o = own ? 0 : k;
    }
    a = __reduce_add_sync(0xFFFFFFFFu, a);
    c = __reduce_add_sync(0xFFFFFFFFu, c);
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      t += __shfl_xor_sync(0xFFFFFFFFu, t, d);
      o += __shfl_xor_sync(0xFFFFFFFFu, o, d);
    }
    if ((threadIdx.x & 31u) == 0) {
      if (a) atomicAdd(&n_own[0], a);
      if (c) atomicAdd(&n_sub[0], c);
      if (t) atomicAdd((unsigned long long*)&own_tok[0], (unsigned long long)t);
      if (o) atomicAdd((unsigned long long*)&num_out[0], (unsigned long long)o);
    }
  }
}

__global__ void k_widen_u32(const u32* a, u64 n, u64* b) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += stride) b[i] = i < n ? a[i] : 0;
}

// both per-rule counts in one u64 (own | sub << 32): one scan gives both CSR
// offset arrays (every sum < 2^31 on this path)
__global__ void k_pack_counts(const u32* __restrict__ a, const u32* __restrict__ b, u64 R, u64* out) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i <= R; i += stride)
    out[i] = i < R ? ((u64)a[i] | ((u64)b[i] << 32)) : 0ull;
}

__global__ void k_split_offsets(const u64* __restrict__ x, u64 n, u64* own_off, u64* sub_off) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    own_off[i] = x[i] & 0xFFFFFFFFull;
    sub_off[i] = x[i] >> 32;
  }
}

// element-parallel compaction of the in-place runs into the CSR arrays
__global__ void k_rules_compact(const u32* __restrict__ owner, const u64* __restrict__ boff, u64 E,
                                const u32* __restrict__ n_own, const u32* __restrict__ n_sub,
                                const u64* __restrict__ own_off, const u64* __restrict__ sub_off,
                                const u32* __restrict__ tsym, const u32* __restrict__ tcnt, u32* own_ids,
                                u32* own_freqs, u32* own_rule, u32* sub_ids, u32* sub_freqs, u32* sub_rule) {
  u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < E; p += stride) {
    const u32 r = owner[p];
    const u64 k = p - boff[r];
    const u32 no = n_own[r];
    if (k < no) {
      const u64 i = own_off[r] + k;
      own_ids[i] = tsym[p];
      own_freqs[i] = tcnt[p];
      own_rule[i] = r;
    } else if (k < (u64)no + n_sub[r]) {
      const u64 i = sub_off[r] + (k - no);
      sub_ids[i] = tsym[p];
      sub_freqs[i] = tcnt[p];
      sub_rule[i] = r;
    }
  }
}

#define CK(k, n, ...) GT_KLAUNCH(#k, k, grid_for((n), 256), 256, st, __VA_ARGS__)

// the root's body length, known on the host before the device DAG is built
static u64 boff_host_root_len(const DeviceDag* d) { return d->L0; }

// The common shape first, without a host round trip: every body but the
// root is at most kShort symbols (Sequitur rules; the composed configs),
// so the only long body is the root, sorted in place and run-length encoded
// over its L0 positions — no selects over R or E and no count read-back
// before the offsets.  One read-back then returns the pair totals AND the
// number of long non-root bodies; when there are any, the caller redoes
// the build on the general path.
static bool rule_pairs_root_only(DeviceDag* d, const u32* owner, DBuf& own_rule, DBuf& sub_rule, cudaStream_t st) {
  const u64 R = d->R, E = d->E, nw = d->nw, base = d->nw + d->ns, L0 = d->L0;
  const u32* body = d->body.as<u32>();
  const u64* boff = d->boff.as<u64>();
  enum { TSYM, TCNT, NOWN, NSUB, LFLAG, CNT, PACK, PACKS, SBODY, HEAD, HIDX, NSPL, RFIRST };
  const Carve a(st, {E * 4 + 4, E * 4 + 4, R * 4 + 4, R * 4 + 4, R + 1, 64, (R + 1) * 8, (R + 1) * 8, L0 * 4 + 4,
                     L0 + 1, L0 * 4 + 4, 8, 8});
  u32 *tsym = a.at<u32>(TSYM), *tcnt = a.at<u32>(TCNT), *n_own = a.at<u32>(NOWN), *n_sub = a.at<u32>(NSUB);
  uint8_t* lflag = a.at<uint8_t>(LFLAG);
  u64* cnt = a.at<u64>(CNT);  // [0] nlong (u32), [2] run heads of the root
  GT_CUDA(cudaMemsetAsync(cnt, 0, 64, st));
  d->own_tok.alloc(R * 8, st);
  d->num_out.alloc(R * 8, st);
  CK(k_rules_short, R, body, boff, R, nw, base, tsym, tcnt, n_own, n_sub, d->own_tok.as<u64>(),
     d->num_out.as<u64>(), lflag, reinterpret_cast<u32*>(cnt));
  const u64 limit = nw + d->ns + R;
  static const bool root_sort = getenv("GT_ROOT_SORT") != nullptr;  // diagnostics: always sort the root
  if (L0 > kShort && !root_sort && limit <= std::max<u64>(4 * L0, 1ull << 22)) {
    // the root's runs from a dense histogram (k_root_hist)
    DBuf hist(limit * 4 + 4, st), idx(std::min(limit, L0) * 4 + 4, st);
    GT_CUDA(cudaMemsetAsync(hist.p, 0, limit * 4, st));
    CK(k_root_hist, L0, body, L0, hist.as<u32>());
    if (d->ns) GT_CUDA(cudaMemsetAsync(hist.as<u32>() + nw, 0, d->ns * 4, st));  // splitters are no pairs
    select_nonzero_index(hist.p, true, idx.as<u32>(), cnt + 2, limit, st);
    CK(k_root_runs, std::min(limit, L0), idx.as<u32>(), cnt + 2, hist.as<u32>(), nw, base, tsym, tcnt, n_own, n_sub,
       d->own_tok.as<u64>(), d->num_out.as<u64>());
  } else if (L0 > kShort) {  // the root: sorted in place, its runs written at offset 0
    u32* sbody = a.at<u32>(SBODY);
    sort_keys_u32(body, sbody, L0, std::max(1, bitlen(d->nw + d->ns + R - 1)), st);
    CK(k_long_heads, L0, owner, lflag, boff, sbody, L0, a.at<uint8_t>(HEAD));
    select_flagged_index(a.at<uint8_t>(HEAD), a.at<u32>(HIDX), cnt + 2, L0, st);
    GT_CUDA(cudaMemsetAsync(a.at<u32>(NSPL), 0, 8, st));
    CK(k_long_count, L0, a.at<u32>(HIDX), cnt + 2, owner, boff, sbody, nw, base, n_own, n_sub, a.at<u32>(NSPL),
       d->own_tok.as<u64>(), d->num_out.as<u64>(), a.at<u32>(RFIRST));
    CK(k_long_write, L0, a.at<u32>(HIDX), cnt + 2, owner, boff, sbody, nw, base, a.at<u32>(NSPL),
       a.at<u32>(RFIRST), tsym, tcnt);
  }
  CK(k_pack_counts, R + 1, n_own, n_sub, R, a.at<u64>(PACK));
  exclusive_scan_u64(a.at<u64>(PACK), a.at<u64>(PACKS), R + 1, st);
  u64 h[2];
  GT_CUDA(cudaMemcpyAsync(&h[0], a.at<u64>(PACKS) + R, 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(&h[1], cnt, 8, cudaMemcpyDeviceToHost, st));
  stream_sync(st);
  if ((u32)h[1] != 0) return false;  // long non-root bodies: the general path
  d->own_off.alloc((R + 1) * 8, st);
  d->sub_off.alloc((R + 1) * 8, st);
  CK(k_split_offsets, R + 1, a.at<u64>(PACKS), R + 1, d->own_off.as<u64>(), d->sub_off.as<u64>());
  d->E_own = h[0] & 0xFFFFFFFFull;
  d->E_sub = h[0] >> 32;
  const u64 Eo = d->E_own, Es = d->E_sub;
  d->own_ids.alloc(Eo * 4 + 4, st);
  d->own_freqs.alloc(Eo * 4 + 4, st);
  own_rule.alloc(Eo * 4 + 4, st);
  d->sub_ids.alloc(Es * 4 + 4, st);
  d->sub_freqs.alloc(Es * 4 + 4, st);
  sub_rule.alloc(Es * 4 + 4, st);
  CK(k_rules_compact, E, owner, boff, E, n_own, n_sub, d->own_off.as<u64>(), d->sub_off.as<u64>(), tsym, tcnt,
     d->own_ids.as<u32>(), d->own_freqs.as<u32>(), own_rule.as<u32>(), d->sub_ids.as<u32>(),
     d->sub_freqs.as<u32>(), sub_rule.as<u32>());
  return true;
}

void build_rule_pairs(DeviceDag* d, const u32* owner, DBuf& own_rule, DBuf& sub_rule, cudaStream_t st) {
  static const bool nospec = getenv("GT_CSR_GENERAL") != nullptr;  // diagnostics: always the general path
  if (!nospec && (u64)d->E < (1ull << 31) && rule_pairs_root_only(d, owner, own_rule, sub_rule, st)) return;
  const u64 R = d->R, E = d->E, nw = d->nw, base = d->nw + d->ns;
  const u32* body = d->body.as<u32>();
  const u64* boff = d->boff.as<u64>();
  // this phase's temporaries in one allocation
  enum { TSYM, TCNT, NOWN, NSUB, LFLAG, GFLAG, LIDS, GIDS, GPOS, CNT, MEDF, WIDE };
  const Carve a(st, {E * 4 + 4, E * 4 + 4, R * 4 + 4, R * 4 + 4, R + 1, E + 1, R * 4 + 4, R * 4 + 4, E * 4 + 4, 32,
                     R + 1, (R + 1) * 8});
  u32 *tsym = a.at<u32>(TSYM), *tcnt = a.at<u32>(TCNT), *n_own = a.at<u32>(NOWN), *n_sub = a.at<u32>(NSUB);
  uint8_t* lflag = a.at<uint8_t>(LFLAG);
  u64* cnt = a.at<u64>(CNT);
  d->own_tok.alloc(R * 8, st);
  d->num_out.alloc(R * 8, st);
  CK(k_rules_short, R, body, boff, R, nw, base, tsym, tcnt, n_own, n_sub, d->own_tok.as<u64>(),
     d->num_out.as<u64>(), lflag, (u32*)nullptr);
  // the longer bodies: one host round trip for their number and size
  CK(k_eq_u8, R, lflag, R, (uint8_t)1, a.at<uint8_t>(MEDF));
  select_flagged_index(a.at<uint8_t>(MEDF), a.at<u32>(LIDS), cnt, R, st);
  CK(k_eq_u8, R, lflag, R, (uint8_t)2, a.at<uint8_t>(MEDF));
  select_flagged_index(a.at<uint8_t>(MEDF), a.at<u32>(GIDS), cnt + 3, R, st);
  CK(k_giant_elems, E, owner, lflag, E, a.at<uint8_t>(GFLAG));
  select_flagged_index(a.at<uint8_t>(GFLAG), a.at<u32>(GPOS), cnt + 1, E, st);
  u64 h[4];
  GT_CUDA(cudaMemcpyAsync(h, cnt, 32, cudaMemcpyDeviceToHost, st));
  stream_sync(st);
  const u64 nmed = h[0], ngel = h[1], ngiant = h[3];
  const u64 L0 = boff_host_root_len(d);
  const bool root_long = L0 > kShort;
  if (nmed || ngel || root_long) {
    enum { SBODY, BEG, END, K1, K2, GRANK, HEAD, HIDX, NSPL, RFIRST };
    const Carve b(st, {E * 4 + 4, nmed * 4 + 4, nmed * 4 + 4, ngel * 8 + 8, ngel * 8 + 8, R * 4 + 4, E + 1,
                       E * 4 + 4, R * 4 + 4, R * 4 + 4});
    u32* sbody = b.at<u32>(SBODY);
    if (root_long) sort_keys_u32(body, sbody, L0, std::max(1, bitlen(d->nw + d->ns + R - 1)), st);
    if (nmed) {
      CK(k_seg_bounds, nmed, a.at<u32>(LIDS), nmed, boff, b.at<int>(BEG), b.at<int>(END));
      sort_segments_listed_u32(body, sbody, E, nmed, b.at<int>(BEG), b.at<int>(END), st);
    }
    if (ngel) {
      const int SB = std::max(1, bitlen(d->nw + d->ns + R - 1));
      const int KB = SB + bitlen(ngiant - 1);
      CK(k_scatter_rank, ngiant, a.at<u32>(GIDS), ngiant, b.at<u32>(GRANK));
      CK(k_giant_keys, ngel, a.at<u32>(GPOS), ngel, owner, b.at<u32>(GRANK), body, SB, b.at<u64>(K1));
      sort_keys_u64(b.at<u64>(K1), b.at<u64>(K2), ngel, KB, st);
      CK(k_giant_scatter, ngel, b.at<u64>(K2), a.at<u32>(GPOS), ngel, SB, sbody);
    }
    CK(k_long_heads, E, owner, lflag, boff, sbody, E, b.at<uint8_t>(HEAD));
    select_flagged_index(b.at<uint8_t>(HEAD), b.at<u32>(HIDX), cnt + 2, E, st);
    GT_CUDA(cudaMemsetAsync(b.at<u32>(NSPL), 0, R * 4 + 4, st));
    CK(k_long_count, E, b.at<u32>(HIDX), cnt + 2, owner, boff, sbody, nw, base, n_own, n_sub, b.at<u32>(NSPL),
       d->own_tok.as<u64>(), d->num_out.as<u64>(), b.at<u32>(RFIRST));
    CK(k_long_write, E, b.at<u32>(HIDX), cnt + 2, owner, boff, sbody, nw, base, b.at<u32>(NSPL),
       b.at<u32>(RFIRST), tsym, tcnt);
  }
  // per-rule counts -> CSR offsets (no search: the scan IS the offsets)
  d->own_off.alloc((R + 1) * 8, st);
  d->sub_off.alloc((R + 1) * 8, st);
  u64* wide = a.at<u64>(WIDE);
  CK(k_widen_u32, R + 1, n_own, R, wide);
  exclusive_scan_u64(wide, d->own_off.as<u64>(), R + 1, st);
  CK(k_widen_u32, R + 1, n_sub, R, wide);
  exclusive_scan_u64(wide, d->sub_off.as<u64>(), R + 1, st);
  u64 tot[2];
  GT_CUDA(cudaMemcpyAsync(&tot[0], d->own_off.as<u64>() + R, 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(&tot[1], d->sub_off.as<u64>() + R, 8, cudaMemcpyDeviceToHost, st));
  stream_sync(st);
  d->E_own = tot[0];
  d->E_sub = tot[1];
  const u64 Eo = tot[0], Es = tot[1];
  d->own_ids.alloc(Eo * 4 + 4, st);
  d->own_freqs.alloc(Eo * 4 + 4, st);
  own_rule.alloc(Eo * 4 + 4, st);
  d->sub_ids.alloc(Es * 4 + 4, st);
  d->sub_freqs.alloc(Es * 4 + 4, st);
  sub_rule.alloc(Es * 4 + 4, st);
  CK(k_rules_compact, E, owner, boff, E, n_own, n_sub, d->own_off.as<u64>(), d->sub_off.as<u64>(), tsym, tcnt,
     d->own_ids.as<u32>(), d->own_freqs.as<u32>(), own_rule.as<u32>(), d->sub_ids.as<u32>(),
     d->sub_freqs.as<u32>(), sub_rule.as<u32>());
}

}  // namespace gt
