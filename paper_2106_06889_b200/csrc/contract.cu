// contract.cu — the single-parent contraction of the top-down pass.
//
// The top-down pass (Alg. 1, engine.py:196-227; word count / inverted index,
// tasks.py:24-84) pushes every rule's weight to its children level by level:
// its cost on a small grammar is the chain of dependent levels, not the
// bytes.  Most rules of a Sequitur grammar are referenced from exactly one
// place (C2: 756k of 840k rules): a rule r with exactly one non-root parent
// edge (p, f) and no root reference has w(r) = f·w(p), so by induction
// w(r) = M(r)·w(H(r)) for its nearest ancestor H(r) with several parents or
// a root reference (its "head", M(r) the product of the frequencies on the
// way).  Every word-count / presence consumer only needs Σ_r own(r,w)·w(r)
// = Σ_r own(r,w)·M(r)·w(H(r)) (presence: M >= 1 keeps the bits), so the pass
// can run over the heads only:
//   - heads by contracted level L' (1 + max L' over the heads of their
//     parents; the root is level 0): C2 84k rules in 17 levels instead of
//     840k in 24;
//   - edges H(p) -> c with frequency f·M(p) for every non-root edge p -> c
//     into a head c (C2: 325k of 1.08M);
//   - own pairs (word, H(r), f·M(r)), pairs of one word whose rules share a
//     head merged into one (word-major like ow).
// The per-file columns (per-file counts, presence bitsets) are linear in the
// same way, column by column.  A product f·M(p) or f·M(r) of 2^32 or more
// turns the contraction off (the lists stay u32).
//
// Built lazily from the loader's top-down lists (tid space), once a DAG
// serves repeated runs: gt_open stays as it was (a one-shot open + query
// pays nothing), the first top-down word task of the DAG's second public run
// call (gt_run / gt_run_many) builds the lists (C2 0.85 ms, C5 8 ms) and
// every later run takes the shorter chain.  GT_CONTRACT=0 never
// builds them, GT_CONTRACT=2 builds them on the first run.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <chrono>

#include <cooperative_groups.h>

#include "kernels_common.cuh"

namespace cg = cooperative_groups;

namespace gt {

#define LAUNCH(k, n, ...) GT_KLAUNCH(#k, k, grid_for((n), 256), 256, st, __VA_ARGS__)

namespace {

// non-root parent edges per child (tid).  A child's edges are contiguous in
// the td lists, so one atomic per (warp, child) run: same-address atomics of
// a warp would serialise in one L2 slice
__global__ void k_c_count(const u32* __restrict__ child, u64 n, u32* cnt) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 b = (u64)blockIdx.x * blockDim.x; b < n; b += stride) {
    const u64 i = b + threadIdx.x;
    const bool ok = i < n;
    const u32 c = ok ? child[i] : 0xFFFFFFFFu;
    const unsigned same = __match_any_sync(0xFFFFFFFFu, c);
    if (ok && (threadIdx.x & 31u) == (unsigned)(__ffs(same) - 1)) atomicAdd(&cnt[c], (u32)__popc(same));
  }
}

// rules the root references (the unfiltered root lists)
__global__ void k_c_rootp(const u32* __restrict__ rs_rule, u64 n, const u32* __restrict__ tid, uint8_t* flag) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) flag[tid[rs_rule[i]]] = 1;
}

// flag: 1 = single (exactly one non-root parent edge, no root reference)
__global__ void k_c_single(const u32* __restrict__ cnt, u64 R, uint8_t* flag) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < R; t += stride)
    flag[t] = t != 0 && cnt[t] == 1 && !flag[t];
}

// one top-down level's edges p -> c (every parent lies in an earlier level,
// so its H / M / L' are final): a single child inherits (H(p), M(p)·f,
// L'(p)); a head child raises its running max of L'(p) (lv holds the max
// until k_c_final turns it into the head's own level).
// Every level in ONE cooperative launch (grid barriers between levels;
// parents' H / M / L' written by other SMs are read through L2).
__global__ void __launch_bounds__(512) k_c_levels(const u32* __restrict__ child, const u32* __restrict__ par,
                                                  const u32* __restrict__ freq, const u64* __restrict__ off, int nl,
                                                  const uint8_t* __restrict__ single, u32* hd, u32* ml, u32* lv,
                                                  u32* ovf) {
  cg::grid_group grid = cg::this_grid();
  const u64 stride = (u64)gridDim.x * blockDim.x, t0 = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  bool o = false;
  for (int L = 1; L <= nl; L++) {
    const u64 a = off[L], e = off[L + 1];
    for (u64 i = a + t0; i < e; i += stride) {
      const u32 c = child[i], p = par[i];
      const bool ps = single[p];
      const u32 H = ps ? __ldcg(hd + p) : p, M = ps ? __ldcg(ml + p) : 1u;
      const u32 L2 = ps ? __ldcg(lv + p) : __ldcg(lv + p) + 1u;
      if (single[c]) {
        const u64 m = (u64)M * freq[i];
        o |= m > 0xFFFFFFFFull;
        hd[c] = H;
        ml[c] = (u32)m;
        lv[c] = L2;
      } else {
        atomicMax(&lv[c], L2);
      }
    }
    if (L < nl) grid.sync();
  }
  if (o) *ovf = 1;
}

// heads: H = itself, M = 1, L' = 1 + max over parents (the root: 0); the
// tid' sort key (heads by L', singles after every level)
__global__ void k_c_final(const uint8_t* __restrict__ single, u64 R, u32 drop, u32* hd, u32* ml, u32* lv, u32* key) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < R; t += stride) {
    if (single[t]) {
      key[t] = drop;
    } else {
      const u32 L = t ? lv[t] + 1u : 0u;
      hd[t] = (u32)t;
      ml[t] = 1u;
      lv[t] = L;
      key[t] = L;
    }
  }
}

// in-degrees in tid' order (singles have no list of their own)
__global__ void k_c_degt(const u32* __restrict__ ord, u64 R, const uint8_t* __restrict__ single,
                         const u32* __restrict__ cnt, u32* degt) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 j = (u64)blockIdx.x * blockDim.x + threadIdx.x; j < R; j += stride) {
    const u32 t = ord[j];
    degt[j] = single[t] ? 0u : cnt[t];
  }
}

// the heads' edges H(p) -> c, f·M(p), scattered into per-child slot ranges
// (one 12-byte record per edge, unpacked afterwards like the loader's lists)
__global__ void k_c_scatter(const u32* __restrict__ child, const u32* __restrict__ par, const u32* __restrict__ freq,
                            u64 n, const uint8_t* __restrict__ single, const u32* __restrict__ ctid,
                            const u32* __restrict__ hd, const u32* __restrict__ ml, u32* cur, U3* te, u32* ovf) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  bool o = false;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 c = child[i];
    if (single[c]) continue;
    const u32 p = par[i];
    const u64 m = (u64)freq[i] * ml[p];
    o |= m > 0xFFFFFFFFull;
    const u32 tc = ctid[c];
    const u32 slot = atomicAdd(&cur[tc], 1u);
    te[slot] = U3{tc, ctid[hd[p]], (u32)m};
  }
  if (o) *ovf = 1;
}

// own pairs keyed (word, tid'(H(r))) with f·M(r): pairs of the same word
// whose rules share a head merge into one (sort + reduce by key)
__global__ void k_c_own_keys(const u32* __restrict__ word, const u32* __restrict__ rule_t,
                             const u32* __restrict__ freq, u64 n, const u32* __restrict__ ctid,
                             const u32* __restrict__ hd, const u32* __restrict__ ml, int sb, u64* key, u64* val) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 t = rule_t[i];
    key[i] = ((u64)word[i] << sb) | ctid[hd[t]];
    val[i] = (u64)freq[i] * ml[t];
  }
}

__global__ void k_c_own_unpack(const u64* __restrict__ key, const u64* __restrict__ sum,
                               const u64* __restrict__ n_dev, int sb, u32* word, u32* src, u32* fr, u32* ovf) {
  const u64 n = *n_dev, stride = (u64)gridDim.x * blockDim.x;
  bool o = false;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 k = key[i], v = sum[i];
    o |= v > 0xFFFFFFFFull;
    word[i] = (u32)(k >> sb);
    src[i] = (u32)(k & ((1ull << sb) - 1));
    fr[i] = (u32)v;
  }
  if (o) *ovf = 1;
}

}  // namespace

void ensure_contracted(DeviceDag* d) {
  if (d->c_tried) return;
  d->c_tried = true;
  const auto t0 = std::chrono::steady_clock::now();
  GT_CUDA(cudaSetDevice(d->device));
  cudaStream_t st = d->stream;
  const u64 R = d->R;
  const int nl = d->td.nl;
  const u64 Etd = d->te_off.empty() ? 0 : d->te_off.back();
  const u64 Eo = d->E_own;
  if (R < 2 || nl < 1) return;
  const Carve cv(st, {R * 4, R + 16, R * 4, R * 4, R * 4, R * 4, R * 4 + 4, R * 4 + 4, R * 4 + 4,
                      ((u64)nl + 3) * 8, 16});
  u32 *cnt = cv.at<u32>(0), *key = cv.at<u32>(2), *key2 = cv.at<u32>(3), *iota = cv.at<u32>(4),
      *ord = cv.at<u32>(5), *degt = cv.at<u32>(6), *incl = cv.at<u32>(7), *cur = cv.at<u32>(8),
      *ovf = cv.at<u32>(10);
  uint8_t* single = cv.at<uint8_t>(1);
  u64* ls = cv.at<u64>(9);
  GT_CUDA(cudaMemsetAsync(cnt, 0, R * 4, st));
  GT_CUDA(cudaMemsetAsync(single, 0, R, st));
  GT_CUDA(cudaMemsetAsync(ovf, 0, 16, st));
  d->c_hd.alloc(R * 4 + 4, st);
  d->c_ml.alloc(R * 4 + 4, st);
  d->c_lvp.alloc(R * 4 + 4, st);
  u32 *hd = d->c_hd.as<u32>(), *ml = d->c_ml.as<u32>(), *lv = d->c_lvp.as<u32>();
  GT_CUDA(cudaMemsetAsync(lv, 0, R * 4, st));
  // singles: one non-root parent edge and no root reference (any file: the
  // owned range only filters the seeds)
  if (Etd) LAUNCH(k_c_count, Etd, d->te_child.as<u32>(), Etd, cnt);
  const auto& rs = d->full.saved ? d->full.rs_rule : d->rs_rule;
  const u64 nrs = d->full.saved ? d->full.n_rs : d->n_rs;
  if (nrs) LAUNCH(k_c_rootp, nrs, rs.as<u32>(), nrs, d->tid.as<u32>(), single);
  LAUNCH(k_c_single, R, cnt, R, single);
  // H / M / L' level by level (one launch per level; built once per DAG)
  {
    static int per_sm = -1;
    if (per_sm < 0) {
      GT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_c_levels, 512, 0));
      per_sm = std::max(1, std::min(per_sm, 4));
    }
    int nsm = 148;
    GT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, d->device));
    const u32* tc = d->te_child.as<u32>();
    const u32* tp = d->te_par.as<u32>();
    const u32* tf = d->te_freq.as<u32>();
    const u64* to = d->te_off_dev.as<u64>();
    int nlv = nl;
    const uint8_t* sg = single;
    void* args[] = {(void*)&tc, (void*)&tp, (void*)&tf, (void*)&to, (void*)&nlv, (void*)&sg,
                    (void*)&hd, (void*)&ml, (void*)&lv, (void*)&ovf};
    ProfScope ps("k_c_levels", st);
    GT_CUDA(cudaLaunchCooperativeKernel((const void*)k_c_levels, dim3((unsigned)(nsm * per_sm)), dim3(512), args, 0,
                                        st));
    g_launches++;
  }
  LAUNCH(k_c_final, R, single, R, (u32)nl + 1, hd, ml, lv, key);
  // tid': heads by (L', tid) (stable radix sort), singles last
  LAUNCH(k_iota_u32, R, iota, R);
  sort_pairs_u32_u32(key, key2, iota, ord, R, std::max(1, bitlen((u64)nl + 1)), st);
  d->c_tid.alloc(R * 4 + 4, st);
  LAUNCH(k_rank_of, R, ord, R, d->c_tid.as<u32>());
  LAUNCH(k_csr_offsets, (u64)nl + 3, key2, R, (u64)nl + 2, ls);  // ls[L]: first tid' of level >= L
  LAUNCH(k_c_degt, R, ord, R, single, cnt, degt);
  inclusive_scan_u32(degt, incl, R, st);
  LAUNCH(k_cursor, R, degt, incl, R, cur);
  // (+ 16: the TMA-staged level loop copies whole 16-byte words)
  d->c_te_child.alloc(Etd * 4 + 16, st);
  d->c_te_par.alloc(Etd * 4 + 16, st);
  d->c_te_freq.alloc(Etd * 4 + 16, st);
  if (Etd) {
    DBuf te(Etd * 12 + 12, st);
    LAUNCH(k_c_scatter, Etd, d->te_child.as<u32>(), d->te_par.as<u32>(), d->te_freq.as<u32>(), Etd, single,
           d->c_tid.as<u32>(), hd, ml, cur, te.as<U3>(), ovf);
    LAUNCH(k_unpack3_n, Etd, te.as<U3>(), incl + (R - 1), d->c_te_child.as<u32>(), d->c_te_par.as<u32>(),
           d->c_te_freq.as<u32>());
  }
  d->c_te_off_dev.alloc(((u64)nl + 3) * 8, st);
  LAUNCH(k_te_level_off, (u64)nl + 3, ls, incl, degt, R, (u64)nl, d->c_te_off_dev.as<u64>());
  d->c_ow_word.alloc(Eo * 4 + 4, st);
  d->c_ow_src.alloc(Eo * 4 + 4, st);
  d->c_ow_freq.alloc(Eo * 4 + 4, st);
  u64* n_own_dev = reinterpret_cast<u64*>(ovf) + 1;
  GT_CUDA(cudaMemsetAsync(n_own_dev, 0, 8, st));
  if (Eo) {
    const Carve ow(st, {Eo * 8, Eo * 8, Eo * 8, Eo * 8});
    u64 *k1 = ow.at<u64>(0), *k2 = ow.at<u64>(1), *v1 = ow.at<u64>(2), *v2 = ow.at<u64>(3);
    // key (word, tid'): bitlen(R) + bitlen(V) bits (C2: 37, 5 radix passes)
    const int sb = std::max(1, bitlen(R - 1));
    LAUNCH(k_c_own_keys, Eo, d->ow_word.as<u32>(), d->ow_rule_t.as<u32>(), d->ow_freq.as<u32>(), Eo,
           d->c_tid.as<u32>(), hd, ml, sb, k1, v1);
    sort_pairs_u64_u64(k1, k2, v1, v2, Eo, sb + std::max(1, bitlen(d->nw ? d->nw - 1 : 0)), st);
    reduce_by_key_u64(k2, v2, k1, v1, n_own_dev, Eo, st);
    LAUNCH(k_c_own_unpack, Eo, k1, v1, n_own_dev, sb, d->c_ow_word.as<u32>(), d->c_ow_src.as<u32>(),
           d->c_ow_freq.as<u32>(), ovf);
  }
  d->contracted = true;  // (refresh_contracted_seeds maps the current seeds)
  refresh_contracted_seeds(d);
  std::vector<u64> h(2 * ((u64)nl + 3) + 2);
  GT_CUDA(cudaMemcpyAsync(h.data(), ls, ((u64)nl + 3) * 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(h.data() + nl + 3, d->c_te_off_dev.p, ((u64)nl + 3) * 8, cudaMemcpyDeviceToHost, st));
  GT_CUDA(cudaMemcpyAsync(h.data() + 2 * (nl + 3), ovf, 16, cudaMemcpyDeviceToHost, st));
  stream_sync(st);
  if ((u32)h[2 * (nl + 3)]) {  // a product outgrew 32 bits: the full lists stay in use
    d->contracted = false;
    DBuf* bufs[] = {&d->c_tid, &d->c_te_child, &d->c_te_par, &d->c_te_freq, &d->c_te_off_dev, &d->c_ow_word,
                    &d->c_ow_src, &d->c_ow_freq, &d->c_rs_rule_t};
    for (DBuf* b : bufs) b->release();
    if (getenv("GT_TRACE")) fprintf(stderr, "[contract] off: a frequency times multiplier needs 64 bits\n");
    return;
  }
  int ncl = 0;  // the highest level holding a head
  for (int L = 1; L <= nl; L++)
    if (h[L + 1] > h[L]) ncl = L;
  d->c_levels = (u32)ncl;
  d->c_R = h[nl + 1];
  d->c_n_own = h[2 * (nl + 3) + 1];
  d->c_te_off.assign(h.begin() + (nl + 3), h.begin() + (nl + 3) + (ncl + 3));
  d->load_flags |= 4;
  if (getenv("GT_TRACE"))
    fprintf(stderr,
            "[contract] %llu heads of %llu rules, %llu of %llu edges, %d of %d levels, %llu of %llu own pairs; "
            "built in %.3f ms\n",
            (unsigned long long)d->c_R, (unsigned long long)R, (unsigned long long)d->c_te_off.back(),
            (unsigned long long)Etd, ncl, nl, (unsigned long long)d->c_n_own, (unsigned long long)Eo,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
}

void refresh_contracted_seeds(DeviceDag* d) {
  if (!d->contracted) return;
  cudaStream_t st = d->stream;
  d->c_rs_rule_t.alloc(d->n_rs * 4 + 4, st);
  if (d->n_rs)
    LAUNCH(k_map_u32, d->n_rs, d->rs_rule_t.as<u32>(), d->n_rs, d->c_tid.as<u32>(), d->c_rs_rule_t.as<u32>());
}

TdLists td_lists(DeviceDag* d, bool contract) {
  if (contract && !d->c_tried) {
    static const int policy = getenv("GT_CONTRACT") ? atoi(getenv("GT_CONTRACT")) : 1;
    if (policy == 2 || (policy == 1 && d->runs >= 2)) ensure_contracted(d);
  }
  TdLists t;
  if (contract && d->contracted) {
    t.n_own = d->c_n_own;
    t.ow_word = d->c_ow_word.as<u32>();
    t.rows = d->c_R;
    t.te_child = d->c_te_child.as<u32>(), t.te_par = d->c_te_par.as<u32>(), t.te_freq = d->c_te_freq.as<u32>();
    t.te_off_dev = d->c_te_off_dev.as<u64>(), t.te_off = &d->c_te_off, t.nl = (int)d->c_levels;
    t.ow_src = d->c_ow_src.as<u32>(), t.ow_freq = d->c_ow_freq.as<u32>();
    t.rs_rule_t = d->c_rs_rule_t.as<u32>();
    t.contracted = true;
    return t;
  }
  t.rows = d->R;
  t.n_own = d->E_own;
  t.ow_word = d->ow_word.as<u32>();
  t.te_child = d->te_child.as<u32>(), t.te_par = d->te_par.as<u32>(), t.te_freq = d->te_freq.as<u32>();
  t.te_off_dev = d->te_off_dev.as<u64>(), t.te_off = &d->te_off, t.nl = d->td.nl;
  t.ow_src = d->ow_rule_t.as<u32>(), t.ow_freq = d->ow_freq.as<u32>();
  t.rs_rule_t = d->rs_rule_t.as<u32>();
  return t;
}

}  // namespace gt
