/*
 * gt_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * CPU restatement (C11 + OpenMP) of the reference gtadoc engine's
 * analytics-on-compression path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it, as the checker
 * and as the timed CPU baseline ("kind": "port").  The product path
 * (paper_2106_06889_b200, libgtadoc_b200.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every output of this
 * file against tests/golden/expected.json, which tools/make_golden.py
 * produced by running the reference itself (numba backend, both strategies,
 * cross-checked with the reference's decompress-then-count oracle).
 *
 * Every function cites the reference (paths relative to
 * /root/reference/pkg/src/gtadoc).  Data layout follows the reference: all
 * arrays int64, tables are CountTableSet arenas of per-entry-locked chained
 * hash tables (table.py), rounds are bulk-synchronous with mask readiness
 * (engine.py), and the round kernels (_kernels.py) run OpenMP-parallel over
 * partition_work units, like Runner.run's worker threads (engine.py:109-147).
 * Two representational changes with identical results: empty bucket/next
 * links are stored as node+1 with 0 = empty (so calloc gives lazily
 * committed zero pages instead of np.full(-1)), and the dictionary strings
 * are not kept (rendering happens in Python).
 */
#define _GNU_SOURCE
#include <omp.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../include/gtadoc_b200.h"

typedef int64_t i64;
typedef uint64_t u64;

/* ------------------------------------------------------------------------ */
/* errors (errors.py)                                                        */
/* ------------------------------------------------------------------------ */

static __thread char g_err[512];
static __thread jmp_buf* g_jb;
static __thread int g_code;

static void die(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  g_code = code;
  longjmp(*g_jb, 1);
}

const char* gto_last_error(void) { return g_err; }

/* allocation registry so an error (longjmp) frees everything of the call */
typedef struct {
  void** p;
  size_t n, cap;
} Arena;

static void arena_free(Arena* a) {
  for (size_t i = 0; i < a->n; i++) free(a->p[i]);
  free(a->p);
  a->p = NULL;
  a->n = a->cap = 0;
}

static void* acalloc(Arena* a, size_t n, size_t sz) {
  if (n == 0) n = 1;
  void* p = calloc(n, sz);
  if (!p) die(GT_E_RESOURCE, "out of host memory (%zu x %zu bytes)", n, sz);
  if (a->n == a->cap) {
    size_t nc = a->cap ? a->cap * 2 : 64;
    void** q = realloc(a->p, nc * sizeof(void*));
    if (!q) {
      free(p);
      die(GT_E_RESOURCE, "out of host memory");
    }
    a->p = q;
    a->cap = nc;
  }
  a->p[a->n++] = p;
  return p;
}
#define ANEW(a, T, n) ((T*)acalloc((a), (size_t)(n), sizeof(T)))

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* ------------------------------------------------------------------------ */
/* grammar (grammar.py)                                                      */
/* ------------------------------------------------------------------------ */

typedef struct {
  i64 nw, ns, R, base; /* base = rule_base = nw + ns (grammar.py:40-43) */
  i64* boff;           /* R+1 */
  i64* body;           /* E */
} Grammar;

typedef struct {
  const uint8_t* d;
  size_t n, pos;
} Reader;

static const uint8_t* take(Reader* r, u64 n, const char* what, i64 idx) {
  if ((u64)r->pos + n > (u64)r->n) {
    if (idx >= 0) {
      char buf[96];
      snprintf(buf, sizeof buf, what, (long long)idx);
      die(GT_E_FORMAT, "truncated input while reading %s", buf);
    }
    die(GT_E_FORMAT, "truncated input while reading %s", what);
  }
  const uint8_t* p = r->d + r->pos;
  r->pos += (size_t)n;
  return p;
}

static uint32_t rd_u32(Reader* r, const char* what, i64 idx) {
  uint32_t v;
  memcpy(&v, take(r, 4, what, idx), 4);
  return v;
}

/* strict UTF-8 as CPython's bytes.decode("utf-8") */
static int utf8_ok(const uint8_t* s, size_t n) {
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
    else return 0;
    if (i + (size_t)k >= n) return 0;
    if (s[i + 1] < lo || s[i + 1] > hi) return 0;
    for (int j = 2; j <= k; j++)
      if (s[i + j] < 0x80 || s[i + j] > 0xBF) return 0;
    i += (size_t)k + 1;
  }
  return 1;
}

/* deserialize_grammar, grammar.py:193-228 */
static void deserialize(Arena* A, const uint8_t* d, size_t n, Grammar* g) {
  if (n < 4 || memcmp(d, "GTDC", 4) != 0) die(GT_E_FORMAT, "bad magic: not a GTDC file");
  Reader r = {d, n, 4};
  uint8_t version = *take(&r, 1, "version", -1);
  if (version != 1) die(GT_E_FORMAT, "unsupported version %d", (int)version);
  u64 nw = rd_u32(&r, "word count", -1);
  u64 ns = rd_u32(&r, "splitter count", -1);
  u64 R = rd_u32(&r, "rule count", -1);
  if (R < 1) die(GT_E_FORMAT, "grammar must contain a root rule");
  for (u64 i = 0; i < nw; i++) {
    uint32_t ln = rd_u32(&r, "word %lld length", (i64)i);
    const uint8_t* w = take(&r, ln, "word %lld", (i64)i);
    if (!utf8_ok(w, ln)) die(GT_E_FORMAT, "word %lld is not valid UTF-8", (long long)i);
  }
  g->nw = (i64)nw;
  g->ns = (i64)ns;
  g->R = (i64)R;
  g->base = (i64)(nw + ns);
  u64 limit = nw + ns + R;
  /* first pass over the lengths to size the body array */
  size_t save = r.pos;
  u64 E = 0;
  for (u64 i = 0; i < R; i++) {
    uint32_t ln = rd_u32(&r, "rule %lld body length", (i64)i);
    const uint8_t* b = take(&r, 4ull * ln, "rule %lld body", (i64)i);
    u64 mx = 0;
    for (uint32_t j = 0; j < ln; j++) {
      uint32_t s;
      memcpy(&s, b + 4ull * j, 4);
      if (s > mx) mx = s;
    }
    if (ln && mx >= limit)
      die(GT_E_FORMAT, "rule %lld contains symbol %llu out of range", (long long)i,
          (unsigned long long)mx);
    E += ln;
  }
  if (r.pos != r.n)
    die(GT_E_FORMAT, "%lld trailing bytes after rules section", (long long)(r.n - r.pos));
  g->boff = ANEW(A, i64, R + 1);
  g->body = ANEW(A, i64, E);
  r.pos = save;
  u64 k = 0;
  for (u64 i = 0; i < R; i++) {
    uint32_t ln = rd_u32(&r, "", -1);
    const uint8_t* b = take(&r, 4ull * ln, "", -1);
    g->boff[i] = (i64)k;
    for (uint32_t j = 0; j < ln; j++) {
      uint32_t s;
      memcpy(&s, b + 4ull * j, 4);
      g->body[k++] = s;
    }
  }
  g->boff[R] = (i64)k;
}

/* _topo_order, grammar.py:127-161 (reverse postorder, cycle check) */
static i64* topo_order(Arena* A, const Grammar* g) {
  i64 R = g->R, base = g->base;
  int8_t* state = ANEW(A, int8_t, R);
  i64* order = ANEW(A, i64, R);
  i64 no = 0;
  i64* st_r = ANEW(A, i64, R + 1);
  i64* st_p = ANEW(A, i64, R + 1);
  for (i64 start = 0; start < R; start++) {
    if (state[start]) continue;
    i64 sp = 0;
    st_r[sp] = start;
    st_p[sp] = 0;
    sp++;
    state[start] = 1;
    while (sp) {
      sp--;
      i64 r = st_r[sp], pos = st_p[sp];
      i64 lo = g->boff[r], len = g->boff[r + 1] - lo;
      int advanced = 0;
      while (pos < len) {
        i64 s = g->body[lo + pos];
        pos++;
        if (s >= base) {
          i64 c = s - base;
          if (state[c] == 1) die(GT_E_CORRUPTION, "rule reference cycle through rule %lld", (long long)c);
          if (state[c] == 0) {
            st_r[sp] = r;
            st_p[sp] = pos;
            sp++;
            st_r[sp] = c;
            st_p[sp] = 0;
            sp++;
            state[c] = 1;
            advanced = 1;
            break;
          }
        }
      }
      if (!advanced) {
        state[r] = 2;
        order[no++] = r;
      }
    }
  }
  for (i64 i = 0; i < no / 2; i++) {
    i64 t = order[i];
    order[i] = order[no - 1 - i];
    order[no - 1 - i] = t;
  }
  return order;
}

/* ------------------------------------------------------------------------ */
/* DAG (dag.py)                                                              */
/* ------------------------------------------------------------------------ */

typedef struct {
  Grammar g;
  i64 R, E;
  i64 *own_ids, *own_freqs, *own_off, *own_tok;
  i64 *sub_ids, *sub_freqs, *sub_off;
  i64 *par_ids, *par_freqs, *par_off;
  i64 *num_in, *num_out, *root_freq, *height, *exp_len;
  i64 depth;
  i64 F;
  i64 *seg_lo, *seg_hi;
  i64 *seg_tokens; /* segment_token_counts, dag.py:88-104 */
  i64* td_level;   /* per-rule reference top-down round (0 = never visited) */
  i64* bu_level;   /* per-rule reference bottom-up round */
  i64 td_levels, bu_levels;
} Dag;

static int cmp_i64(const void* a, const void* b) {
  i64 x = *(const i64*)a, y = *(const i64*)b;
  return (x > y) - (x < y);
}

static void sort_i64(i64* a, i64 n) {
  if (n < 24) {
    for (i64 i = 1; i < n; i++) {
      i64 v = a[i], j = i - 1;
      while (j >= 0 && a[j] > v) {
        a[j + 1] = a[j];
        j--;
      }
      a[j + 1] = v;
    }
  } else {
    qsort(a, (size_t)n, sizeof(i64), cmp_i64);
  }
}

/* _segments_of_root, dag.py:107-128 */
static void segments_of_root(Arena* A, Dag* d) {
  const Grammar* g = &d->g;
  i64 lo = g->boff[0], len = g->boff[1] - lo;
  if (g->ns == 0) {
    d->F = 1;
    d->seg_lo = ANEW(A, i64, 1);
    d->seg_hi = ANEW(A, i64, 1);
    d->seg_hi[0] = len;
    return;
  }
  d->seg_lo = ANEW(A, i64, g->ns);
  d->seg_hi = ANEW(A, i64, g->ns);
  i64 start = 0, expected = 0;
  for (i64 pos = 0; pos < len; pos++) {
    i64 s = g->body[lo + pos];
    if (s >= g->nw && s < g->base) {
      if (s - g->nw != expected)
        die(GT_E_CORRUPTION, "splitter %lld out of order at root position %lld", (long long)s,
            (long long)pos);
      d->seg_lo[expected] = start;
      d->seg_hi[expected] = pos;
      start = pos + 1;
      expected++;
    }
  }
  if (expected != g->ns) die(GT_E_CORRUPTION, "root body is missing file splitters");
  if (start != len) die(GT_E_CORRUPTION, "root body has content after the last splitter");
  d->F = g->ns;
}

static void td_levels_of(Arena* A, Dag* d);
static void bu_levels_of(Arena* A, Dag* d);

/* build_dag, dag.py:131-230 */
static void build_dag(Arena* A, Dag* d, int nt) {
  Grammar* g = &d->g;
  i64 R = g->R, base = g->base, nw = g->nw;
  d->R = R;
  d->E = g->boff[R];
  i64* order = topo_order(A, g); /* cycle check happens here */
  /* per-rule sorted copies of the body: words first, then splitters, rules */
  i64* srt = ANEW(A, i64, d->E);
  memcpy(srt, g->body, sizeof(i64) * (size_t)d->E);
  i64* nown = ANEW(A, i64, R + 1);
  i64* nsub = ANEW(A, i64, R + 1);
  d->own_tok = ANEW(A, i64, R);
#pragma omp parallel for schedule(dynamic, 256) num_threads(nt)
  for (i64 r = 0; r < R; r++) {
    i64 lo = g->boff[r], hi = g->boff[r + 1];
    sort_i64(srt + lo, hi - lo);
    i64 a = 0, b = 0, tok = 0;
    for (i64 i = lo; i < hi; i++) {
      i64 s = srt[i];
      int first = (i == lo) || srt[i - 1] != s;
      if (s < nw) {
        tok++;
        a += first;
      } else if (s >= base) {
        b += first;
      }
    }
    nown[r] = a;
    nsub[r] = b;
    d->own_tok[r] = tok;
  }
  d->own_off = ANEW(A, i64, R + 1);
  d->sub_off = ANEW(A, i64, R + 1);
  for (i64 r = 0; r < R; r++) {
    d->own_off[r + 1] = d->own_off[r] + nown[r];
    d->sub_off[r + 1] = d->sub_off[r] + nsub[r];
  }
  d->own_ids = ANEW(A, i64, d->own_off[R]);
  d->own_freqs = ANEW(A, i64, d->own_off[R]);
  d->sub_ids = ANEW(A, i64, d->sub_off[R]);
  d->sub_freqs = ANEW(A, i64, d->sub_off[R]);
#pragma omp parallel for schedule(dynamic, 256) num_threads(nt)
  for (i64 r = 0; r < R; r++) {
    i64 lo = g->boff[r], hi = g->boff[r + 1];
    i64 a = d->own_off[r] - 1, b = d->sub_off[r] - 1;
    for (i64 i = lo; i < hi; i++) {
      i64 s = srt[i];
      int first = (i == lo) || srt[i - 1] != s;
      if (s < nw) {
        if (first) d->own_ids[++a] = s;
        d->own_freqs[a]++;
      } else if (s >= base) {
        if (first) d->sub_ids[++b] = s - base;
        d->sub_freqs[b]++;
      }
    }
  }
  /* parents: for p ascending, for c in subs[p] -> parents[c].append(p) */
  i64 Es = d->sub_off[R];
  d->par_off = ANEW(A, i64, R + 1);
  for (i64 j = 0; j < Es; j++) d->par_off[d->sub_ids[j] + 1]++;
  for (i64 r = 0; r < R; r++) d->par_off[r + 1] += d->par_off[r];
  d->par_ids = ANEW(A, i64, Es);
  d->par_freqs = ANEW(A, i64, Es);
  i64* fill = ANEW(A, i64, R);
  for (i64 p = 0; p < R; p++)
    for (i64 j = d->sub_off[p]; j < d->sub_off[p + 1]; j++) {
      i64 c = d->sub_ids[j];
      i64 at = d->par_off[c] + fill[c]++;
      d->par_ids[at] = p;
      d->par_freqs[at] = d->sub_freqs[j];
    }
  /* reachability from the root (dag.py:173-184) */
  int8_t* reach = ANEW(A, int8_t, R);
  i64* stack = ANEW(A, i64, R);
  i64 sp = 0;
  reach[0] = 1;
  stack[sp++] = 0;
  while (sp) {
    i64 p = stack[--sp];
    for (i64 j = d->sub_off[p]; j < d->sub_off[p + 1]; j++) {
      i64 c = d->sub_ids[j];
      if (!reach[c]) {
        reach[c] = 1;
        stack[sp++] = c;
      }
    }
  }
  for (i64 r = 0; r < R; r++)
    if (!reach[r]) die(GT_E_CORRUPTION, "rule %lld is not reachable from the root", (long long)r);
  d->num_in = ANEW(A, i64, R);
  d->num_out = ANEW(A, i64, R);
  d->root_freq = ANEW(A, i64, R);
  for (i64 r = 0; r < R; r++) {
    i64 s = 0;
    for (i64 j = d->par_off[r]; j < d->par_off[r + 1]; j++)
      if (d->par_ids[j] != 0) s += d->par_freqs[j];
    d->num_in[r] = s;
    s = 0;
    for (i64 j = d->sub_off[r]; j < d->sub_off[r + 1]; j++) s += d->sub_freqs[j];
    d->num_out[r] = s;
  }
  for (i64 j = d->sub_off[0]; j < d->sub_off[1]; j++) d->root_freq[d->sub_ids[j]] = d->sub_freqs[j];
  d->height = ANEW(A, i64, R);
  for (i64 k = R - 1; k >= 0; k--) { /* reversed(order): children first */
    i64 r = order[k], h = 0;
    if (d->sub_off[r + 1] > d->sub_off[r]) {
      for (i64 j = d->sub_off[r]; j < d->sub_off[r + 1]; j++)
        if (d->height[d->sub_ids[j]] > h) h = d->height[d->sub_ids[j]];
      d->height[r] = 1 + h;
    }
  }
  d->depth = d->height[0];
  segments_of_root(A, d);
  /* expand_rule_lengths, grammar.py:109-124 */
  d->exp_len = ANEW(A, i64, R);
  for (i64 k = R - 1; k >= 0; k--) {
    i64 r = order[k], t = 0;
    for (i64 i = g->boff[r]; i < g->boff[r + 1]; i++) {
      i64 s = g->body[i];
      if (s < nw) t++;
      else if (s >= base) t += d->exp_len[s - base];
    }
    d->exp_len[r] = t;
  }
  /* segment_token_counts, dag.py:88-104 */
  d->seg_tokens = ANEW(A, i64, d->F);
  for (i64 f = 0; f < d->F; f++) {
    i64 t = 0;
    for (i64 i = d->seg_lo[f]; i < d->seg_hi[f]; i++) {
      i64 s = g->body[g->boff[0] + i];
      if (s < nw) t++;
      else if (s >= base) t += d->exp_len[s - base];
    }
    d->seg_tokens[f] = t;
  }
  td_levels_of(A, d);
  bu_levels_of(A, d);
}

/* ------------------------------------------------------------------------ */
/* tables (table.py)                                                         */
/* ------------------------------------------------------------------------ */

enum { T_OK = 0, T_RETRY = 1, T_FULL = 2 }; /* table.py:35-37 */

static inline u64 mix64(u64 z) { /* table.py:41-49 */
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

static inline i64 fingerprint(const i64* w, i64 start, i64 width) { /* _kernels.py:45-50 */
  u64 h = 0x9E3779B97F4A7C15ull;
  for (i64 j = 0; j < width; j++) h = mix64(h ^ (u64)(w[start + j] + 0x100000001B3ll));
  return (i64)(h & 0x7FFFFFFFFFFFFFFFull);
}

static inline i64 pack_key(const i64* w, i64 start, i64 width, i64 wbits) { /* _kernels.py:53-58 */
  i64 k = 0;
  for (i64 j = 0; j < width; j++) k = (k << wbits) | w[start + j];
  return k;
}

typedef struct {
  i64 T, gw;
  i64 *entries, *locks, *keys, *vals, *nxt, *grams; /* entries/nxt: node+1, 0 empty */
  i64 *cursor, *entry_off, *entry_mask, *node_off, *node_cap;
} Tables;

static i64 entry_capacity(i64 bound) { /* table.py:63-66 */
  i64 need = 2 * bound;
  if (need < 1) need = 1;
  i64 c = 1;
  while (c < need) c <<= 1;
  return c;
}

/* CountTableSet.__init__, table.py:72-107 */
static void tables_init(Arena* A, Tables* t, const i64* bounds, i64 T, i64 gw) {
  memset(t, 0, sizeof *t);
  t->T = T;
  t->gw = gw;
  t->entry_off = ANEW(A, i64, T);
  t->entry_mask = ANEW(A, i64, T);
  t->node_off = ANEW(A, i64, T);
  t->node_cap = ANEW(A, i64, T);
  t->cursor = ANEW(A, i64, T);
  i64 te = 0, tn = 0;
  for (i64 i = 0; i < T; i++) {
    if (bounds[i] < 0) die(GT_E_RESOURCE, "negative table bound");
    i64 c = entry_capacity(bounds[i]);
    t->entry_off[i] = te;
    t->entry_mask[i] = c - 1;
    t->node_off[i] = tn;
    t->node_cap[i] = bounds[i];
    te += c;
    tn += bounds[i];
  }
  t->entries = ANEW(A, i64, te);
  t->locks = ANEW(A, i64, te);
  t->keys = ANEW(A, i64, tn);
  t->vals = ANEW(A, i64, tn);
  t->nxt = ANEW(A, i64, tn);
  t->grams = ANEW(A, i64, tn * (gw ? gw : 0) + 1);
}

static inline i64 tsize(const Tables* t, i64 i) { /* CountTableSet.size, table.py:110-111 */
  i64 c = __atomic_load_n(&t->cursor[i], __ATOMIC_RELAXED);
  return c < t->node_cap[i] ? c : t->node_cap[i];
}

static inline int gram_eq(const Tables* t, i64 node, const i64* gsrc, i64 gstart) {
  for (i64 j = 0; j < t->gw; j++)
    if (t->grams[node * t->gw + j] != gsrc[gstart + j]) return 0;
  return 1;
}

/* table_add, _kernels.py:61-114 (per-entry-locked chained insert-or-add) */
static int table_add(Tables* ts, i64 t, i64 key, i64 delta, const i64* gsrc, i64 gstart,
                     int blocking) {
  i64 b = ts->entry_off[t] + (i64)(mix64((u64)key) & (u64)ts->entry_mask[t]);
  i64 node = __atomic_load_n(&ts->entries[b], __ATOMIC_ACQUIRE) - 1;
  while (node != -1) {
    if (ts->keys[node] == key && gram_eq(ts, node, gsrc, gstart)) {
      __atomic_fetch_add(&ts->vals[node], delta, __ATOMIC_RELAXED);
      return T_OK;
    }
    node = ts->nxt[node] - 1;
  }
  i64 zero = 0;
  if (blocking) {
    while (!__atomic_compare_exchange_n(&ts->locks[b], &zero, 1, 0, __ATOMIC_ACQ_REL,
                                        __ATOMIC_RELAXED))
      zero = 0;
  } else if (!__atomic_compare_exchange_n(&ts->locks[b], &zero, 1, 0, __ATOMIC_ACQ_REL,
                                          __ATOMIC_RELAXED)) {
    return T_RETRY;
  }
  i64 head = __atomic_load_n(&ts->entries[b], __ATOMIC_ACQUIRE) - 1;
  node = head;
  while (node != -1) {
    if (ts->keys[node] == key && gram_eq(ts, node, gsrc, gstart)) {
      __atomic_fetch_add(&ts->vals[node], delta, __ATOMIC_RELAXED);
      __atomic_store_n(&ts->locks[b], 0, __ATOMIC_RELEASE);
      return T_OK;
    }
    node = ts->nxt[node] - 1;
  }
  i64 n = __atomic_fetch_add(&ts->cursor[t], 1, __ATOMIC_RELAXED);
  if (n >= ts->node_cap[t]) {
    __atomic_store_n(&ts->locks[b], 0, __ATOMIC_RELEASE);
    return T_FULL;
  }
  i64 an = ts->node_off[t] + n;
  ts->keys[an] = key;
  ts->vals[an] = delta;
  ts->nxt[an] = head + 1;
  for (i64 j = 0; j < ts->gw; j++) ts->grams[an * ts->gw + j] = gsrc[gstart + j];
  __atomic_store_n(&ts->entries[b], an + 1, __ATOMIC_RELEASE);
  __atomic_store_n(&ts->locks[b], 0, __ATOMIC_RELEASE);
  return T_OK;
}

static void check_capacity(int st, const char* msg) { /* engine.py:521-530 */
  if (st == T_FULL) die(GT_E_RESOURCE, "%s", msg);
}
#define CAP_MSG "result table capacity exhausted"
#define BOUNDS_MSG "local table overflow: the sizing pass under-reserved (corrupt DAG?)"
#define SEQ_MSG "sequence table capacity exhausted"

/* ------------------------------------------------------------------------ */
/* engine (engine.py)                                                        */
/* ------------------------------------------------------------------------ */

typedef struct {
  int strategy; /* GT_TOPDOWN / GT_BOTTOMUP after selection */
  int workers;
  i64 chunk_factor;   /* engine.py:38 */
  i64 file_set_width; /* engine.py:39 */
} Cfg;

typedef struct {
  i64 n;
  i64 *id, *start, *end;
} Units;

/* partition_work, engine.py:74-106 */
static Units partition_work(Arena* A, const i64* ids, const i64* lengths, i64 count, i64 total,
                            i64 cf) {
  Units u = {0, 0, 0, 0};
  if (count == 0) return u;
  i64 avg = total / count;
  if (avg < 1) avg = 1;
  i64 th = cf * avg, n = 0;
  for (i64 i = 0; i < count; i++) n += lengths[i] <= th ? 1 : (lengths[i] + th - 1) / th;
  u.n = n;
  u.id = ANEW(A, i64, n);
  u.start = ANEW(A, i64, n);
  u.end = ANEW(A, i64, n);
  i64 k = 0;
  for (i64 i = 0; i < count; i++) {
    i64 ln = lengths[i];
    if (ln <= th) {
      u.id[k] = ids[i];
      u.start[k] = 0;
      u.end[k] = ln;
      k++;
    } else {
      for (i64 p = 0; p < (ln + th - 1) / th; p++) {
        u.id[k] = ids[i];
        u.start[k] = p * th;
        u.end[k] = (p + 1) * th < ln ? (p + 1) * th : ln;
        k++;
      }
    }
  }
  return u;
}

/* Level schedules as the reference discovers them round by round
 * (engine.py:196-227 top-down, engine.py:313-335 bottom-up); recorded once so
 * tests can pin the device level scheduler against them. */
static void td_levels_of(Arena* A, Dag* d) {
  i64 R = d->R;
  d->td_level = ANEW(A, i64, R);
  i64* cur = ANEW(A, i64, R);
  i64* fr = ANEW(A, i64, R);
  i64* nx = ANEW(A, i64, R);
  i64 nf = 0, k = 0;
  for (i64 r = 1; r < R; r++)
    if (d->num_in[r] == 0) fr[nf++] = r;
  while (nf) {
    k++;
    i64 nn = 0;
    for (i64 i = 0; i < nf; i++) {
      i64 r = fr[i];
      d->td_level[r] = k;
      for (i64 j = d->sub_off[r]; j < d->sub_off[r + 1]; j++) {
        i64 c = d->sub_ids[j];
        cur[c] += d->sub_freqs[j];
        if (cur[c] == d->num_in[c]) nx[nn++] = c;
      }
    }
    i64* t = fr;
    fr = nx;
    nx = t;
    nf = nn;
  }
  d->td_levels = k;
}

static void bu_levels_of(Arena* A, Dag* d) {
  i64 R = d->R;
  d->bu_level = ANEW(A, i64, R);
  i64* cur = ANEW(A, i64, R);
  i64* fr = ANEW(A, i64, R);
  i64* nx = ANEW(A, i64, R);
  i64 nf = 0, k = 0;
  for (i64 r = 1; r < R; r++)
    if (d->sub_off[r + 1] == d->sub_off[r]) fr[nf++] = r;
  while (nf) {
    k++;
    i64 nn = 0;
    for (i64 i = 0; i < nf; i++) {
      i64 r = fr[i];
      d->bu_level[r] = k;
      for (i64 j = d->par_off[r]; j < d->par_off[r + 1]; j++) {
        i64 p = d->par_ids[j];
        cur[p] += d->par_freqs[j];
        if (p != 0 && cur[p] == d->num_out[p]) nx[nn++] = p;
      }
    }
    i64* t = fr;
    fr = nx;
    nx = t;
    nf = nn;
  }
  d->bu_levels = k;
}

/* select_strategy, engine.py:63-71 (+ tasks.py:47-56 hooks) */
static int select_strategy(const Dag* d, int task, int requested, i64 fsw) {
  if (requested == GT_TOPDOWN || requested == GT_BOTTOMUP) return requested;
  int needs_file_info = task >= GT_INVERTEDINDEX;
  if (needs_file_info) return d->F > fsw ? GT_BOTTOMUP : GT_TOPDOWN;
  return GT_TOPDOWN; /* reduce == "global" */
}

typedef struct {
  i64 nf;
  i64 *wmat, *cur_in, *cur_out, *mask;
} State; /* TraversalState, engine.py:150-175 */

static void state_init(Arena* A, State* s, const Dag* d, i64 nf) {
  s->nf = nf;
  s->wmat = ANEW(A, i64, d->R * nf);
  s->cur_in = ANEW(A, i64, d->R);
  s->cur_out = ANEW(A, i64, d->R);
  s->mask = ANEW(A, i64, d->R);
}

/* segment_rule_counts, dag.py:75-86 (dense R x F) */
static i64* segment_rule_counts(Arena* A, const Dag* d) {
  i64* c = ANEW(A, i64, d->R * d->F);
  const Grammar* g = &d->g;
  for (i64 f = 0; f < d->F; f++)
    for (i64 i = d->seg_lo[f]; i < d->seg_hi[f]; i++) {
      i64 s = g->body[g->boff[0] + i];
      if (s >= g->base) c[(s - g->base) * d->F + f]++;
    }
  return c;
}

/* init_top_down_masks, engine.py:178-193 */
static void init_top_down(Arena* A, const Dag* d, State* s) {
  i64 R = d->R, nf = s->nf;
  memset(s->cur_in, 0, sizeof(i64) * R);
  memset(s->mask, 0, sizeof(i64) * R);
  if (nf == 1) {
    for (i64 r = 0; r < R; r++) s->wmat[r] = d->root_freq[r];
    s->wmat[0] = 1;
  } else {
    i64* src = segment_rule_counts(A, d);
    memcpy(s->wmat, src, sizeof(i64) * R * nf);
    for (i64 f = 0; f < nf; f++) s->wmat[f] = 1;
  }
  for (i64 r = 1; r < R; r++) s->mask[r] = d->num_in[r] == 0;
}

static i64 frontier_of(const i64* mask, i64 R, i64* out) {
  i64 n = 0;
  for (i64 r = 0; r < R; r++)
    if (mask[r]) out[n++] = r;
  return n;
}

/* top_down_traverse, engine.py:196-227 + topdown_round, _kernels.py:129-151 */
static i64 top_down_traverse(Arena* A, const Dag* d, State* s, const Cfg* cfg) {
  i64 R = d->R, nf = s->nf, rounds = 0;
  i64* fr = ANEW(A, i64, R);
  i64* len = ANEW(A, i64, R);
  for (;;) {
    i64 n = frontier_of(s->mask, R, fr);
    if (!n) break;
    rounds++;
    if (rounds > d->depth + 1) die(GT_E_CORRUPTION, "top-down traversal exceeded depth bound");
    i64 tot = 0;
    for (i64 i = 0; i < n; i++) tot += len[i] = d->sub_off[fr[i] + 1] - d->sub_off[fr[i]];
    Arena U = {0};
    Units u = partition_work(&U, fr, len, n, tot, cfg->chunk_factor);
#pragma omp parallel for schedule(dynamic, 16) num_threads(cfg->workers)
    for (i64 ui = 0; ui < u.n; ui++) {
      i64 r = u.id[ui], base = d->sub_off[r];
      for (i64 j = u.start[ui]; j < u.end[ui]; j++) {
        i64 c = d->sub_ids[base + j], f = d->sub_freqs[base + j];
        for (i64 k = 0; k < nf; k++) {
          i64 w = s->wmat[r * nf + k];
          if (w != 0) __atomic_fetch_add(&s->wmat[c * nf + k], f * w, __ATOMIC_RELAXED);
        }
        i64 old = __atomic_fetch_add(&s->cur_in[c], f, __ATOMIC_RELAXED);
        if (old + f == d->num_in[c]) s->mask[c] = 1;
      }
    }
    arena_free(&U);
    for (i64 i = 0; i < n; i++) s->mask[fr[i]] = 0;
  }
  return rounds;
}

/* word_table_bounds, engine.py:257-263 */
static i64* word_table_bounds(Arena* A, const Dag* d, int per_file, i64* T) {
  i64 V = d->g.nw;
  if (!per_file) {
    i64* b = ANEW(A, i64, 1);
    b[0] = V;
    *T = 1;
    return b;
  }
  i64* b = ANEW(A, i64, d->F);
  for (i64 f = 0; f < d->F; f++) b[f] = d->seg_tokens[f] < V ? d->seg_tokens[f] : V;
  *T = d->F;
  return b;
}

/* _root_word_units + _split_root_units, engine.py:230-254 ->
 * root_words_round, _kernels.py:175-188 */
static int root_words(Arena* A, const Dag* d, Tables* out, int per_file, i64 out_base,
                      const Cfg* cfg) {
  i64 F = d->F;
  i64* ids = ANEW(A, i64, F);
  i64* lens = ANEW(A, i64, F);
  i64 tot = 0;
  for (i64 f = 0; f < F; f++) {
    ids[f] = f;
    tot += lens[f] = d->seg_hi[f] - d->seg_lo[f];
  }
  Units u = partition_work(A, ids, lens, F, tot, cfg->chunk_factor);
  const i64* body = d->g.body + d->g.boff[0];
  i64 nw = d->g.nw;
  int worst = T_OK;
#pragma omp parallel for schedule(dynamic, 4) num_threads(cfg->workers) reduction(max : worst)
  for (i64 ui = 0; ui < u.n; ui++) {
    i64 f = u.id[ui];
    i64 t = per_file ? out_base + f : out_base;
    for (i64 p = d->seg_lo[f] + u.start[ui]; p < d->seg_lo[f] + u.end[ui]; p++) {
      i64 s = body[p];
      if (s < nw) {
        int st = table_add(out, t, s, 1, NULL, 0, 1);
        if (st > worst) worst = st;
      }
    }
  }
  return worst;
}

/* reduce_top_down, engine.py:266-302 + reduce_words_round, _kernels.py:154-172 */
static void reduce_top_down(Arena* A, const Dag* d, const State* s, const Cfg* cfg, Tables* out) {
  i64 per_file = s->nf > 1, T, R = d->R, nf = s->nf;
  i64* bounds = word_table_bounds(A, d, (int)per_file, &T);
  tables_init(A, out, bounds, T, 0);
  if (R > 1) {
    i64* rules = ANEW(A, i64, R - 1);
    i64* lens = ANEW(A, i64, R - 1);
    i64 tot = 0;
    for (i64 r = 1; r < R; r++) {
      rules[r - 1] = r;
      tot += lens[r - 1] = d->own_off[r + 1] - d->own_off[r];
    }
    Units u = partition_work(A, rules, lens, R - 1, tot, cfg->chunk_factor);
    int worst = T_OK;
#pragma omp parallel for schedule(dynamic, 16) num_threads(cfg->workers) reduction(max : worst)
    for (i64 ui = 0; ui < u.n; ui++) {
      i64 r = u.id[ui], base = d->own_off[r];
      for (i64 j = u.start[ui]; j < u.end[ui]; j++) {
        i64 k = d->own_ids[base + j], fr = d->own_freqs[base + j];
        for (i64 f = 0; f < nf; f++) {
          i64 w = s->wmat[r * nf + f];
          if (w > 0) {
            int st = table_add(out, f, k, fr * w, NULL, 0, 1);
            if (st > worst) worst = st;
          }
        }
      }
    }
    check_capacity(worst, CAP_MSG);
  }
  check_capacity(root_words(A, d, out, (int)per_file, 0, cfg), CAP_MSG);
}

/* init_bottom_up_masks, engine.py:305-310 */
static void init_bottom_up(const Dag* d, State* s) {
  memset(s->cur_out, 0, sizeof(i64) * d->R);
  memset(s->mask, 0, sizeof(i64) * d->R);
  for (i64 r = 1; r < d->R; r++) s->mask[r] = d->sub_off[r + 1] == d->sub_off[r];
}

typedef void (*VisitFn)(Arena* A, const Dag* d, const Cfg* cfg, const i64* ready, i64 n,
                        void* ctx);

/* _bottom_up_rounds, engine.py:313-335 + finalize_round, _kernels.py:205-216 */
static i64 bottom_up_rounds(Arena* A, const Dag* d, State* s, const Cfg* cfg, VisitFn visit,
                            void* vctx, const char* label) {
  i64 R = d->R, rounds = 0;
  i64* ready = ANEW(A, i64, R);
  for (;;) {
    i64 n = frontier_of(s->mask, R, ready);
    if (!n) break;
    rounds++;
    if (rounds > d->depth + 1) die(GT_E_CORRUPTION, "%s pass exceeded depth bound", label);
    visit(A, d, cfg, ready, n, vctx);
#pragma omp parallel for schedule(dynamic, 64) num_threads(cfg->workers)
    for (i64 ri = 0; ri < n; ri++) {
      i64 r = ready[ri];
      for (i64 j = d->par_off[r]; j < d->par_off[r + 1]; j++) {
        i64 p = d->par_ids[j];
        i64 old = __atomic_fetch_add(&s->cur_out[p], d->par_freqs[j], __ATOMIC_RELAXED);
        if (p != 0 && old + d->par_freqs[j] == d->num_out[p]) s->mask[p] = 1;
      }
    }
    for (i64 i = 0; i < n; i++) s->mask[ready[i]] = 0;
  }
  return rounds;
}

typedef struct {
  const i64 *own_sizes, *caps;
  i64* bound;
} BoundsCtx;

/* bounds_round, _kernels.py:191-202 */
static void bounds_visit(Arena* A, const Dag* d, const Cfg* cfg, const i64* ready, i64 n,
                         void* vctx) {
  (void)A;
  BoundsCtx* c = vctx;
#pragma omp parallel for schedule(dynamic, 64) num_threads(cfg->workers)
  for (i64 ri = 0; ri < n; ri++) {
    i64 r = ready[ri], b = c->own_sizes[r];
    for (i64 j = d->sub_off[r]; j < d->sub_off[r + 1]; j++) b += c->bound[d->sub_ids[j]];
    if (b > c->caps[r]) b = c->caps[r];
    c->bound[r] = b;
  }
}

/* local_table_bounds, engine.py:338-367 */
static i64* local_table_bounds(Arena* A, const Dag* d, State* s, const Cfg* cfg,
                               const i64* own_sizes, const i64* caps) {
  i64 R = d->R;
  i64* os = (i64*)own_sizes;
  i64* cp = (i64*)caps;
  if (!os) {
    os = ANEW(A, i64, R);
    for (i64 r = 0; r < R; r++) os[r] = d->own_off[r + 1] - d->own_off[r];
  }
  if (!cp) {
    cp = ANEW(A, i64, R);
    for (i64 r = 0; r < R; r++) cp[r] = d->exp_len[r] < d->g.nw ? d->exp_len[r] : d->g.nw;
  }
  BoundsCtx c = {os, cp, ANEW(A, i64, R)};
  init_bottom_up(d, s);
  bottom_up_rounds(A, d, s, cfg, bounds_visit, &c, "bounds");
  return c.bound;
}

typedef struct {
  i64 n;
  i64 *dst, *src, *scale, *start, *end;
} MUnits;

/* _merge_units + _split_merge_units, engine.py:380-406 */
static MUnits merge_units(Arena* A, const i64* pd, const i64* ps, const i64* pscale, i64 np,
                          const Tables* src, const Cfg* cfg) {
  MUnits m = {0};
  i64* keep = ANEW(A, i64, np);
  i64* lens = ANEW(A, i64, np);
  i64 k = 0, tot = 0;
  for (i64 i = 0; i < np; i++) {
    i64 n = tsize(src, ps[i]);
    if (n == 0) continue;
    keep[k] = i;
    tot += lens[k] = n;
    k++;
  }
  if (!k) return m;
  i64* ids = ANEW(A, i64, k);
  for (i64 i = 0; i < k; i++) ids[i] = i;
  Units u = partition_work(A, ids, lens, k, tot, cfg->chunk_factor);
  m.n = u.n;
  m.dst = ANEW(A, i64, u.n);
  m.src = ANEW(A, i64, u.n);
  m.scale = ANEW(A, i64, u.n);
  m.start = u.start;
  m.end = u.end;
  for (i64 i = 0; i < u.n; i++) {
    i64 p = keep[u.id[i]];
    m.dst[i] = pd[p];
    m.src[i] = ps[p];
    m.scale[i] = pscale[p];
  }
  return m;
}

/* merge_round, _kernels.py:236-250 (blocking scaled merge) */
static int merge_round(Tables* dst, const Tables* src, const MUnits* m, const Cfg* cfg) {
  int worst = T_OK;
  i64 gw = src->gw;
#pragma omp parallel for schedule(dynamic, 16) num_threads(cfg->workers) reduction(max : worst)
  for (i64 ui = 0; ui < m->n; ui++) {
    i64 sb = src->node_off[m->src[ui]], sc = m->scale[ui], dd = m->dst[ui];
    for (i64 i = m->start[ui]; i < m->end[ui]; i++) {
      i64 n = sb + i;
      int st = table_add(dst, dd, src->keys[n], src->vals[n] * sc, src->grams, n * gw, 1);
      if (st > worst) worst = st;
    }
  }
  return worst;
}

/* merge_with_retries, engine.py:449-475 + merge_try_round, _kernels.py:253-276 */
static i64 merge_with_retries(Arena* A, Tables* dst, const Tables* src, const i64* pd,
                              const i64* ps, const i64* pscale, i64 np, const Cfg* cfg,
                              const char* msg) {
  MUnits m = merge_units(A, pd, ps, pscale, np, src, cfg);
  if (!m.n) return 0;
  i64* u_done = ANEW(A, i64, m.n);
  i64 tot = 0;
  for (i64 i = 0; i < m.n; i++) {
    u_done[i] = tot;
    tot += m.end[i] - m.start[i];
  }
  int8_t* done = ANEW(A, int8_t, tot);
  i64 launches = 0, gw = src->gw;
  for (;;) {
    launches++;
    i64 pending = 0;
    int worst = T_OK;
#pragma omp parallel for schedule(dynamic, 16) num_threads(cfg->workers) \
    reduction(max : worst) reduction(+ : pending)
    for (i64 ui = 0; ui < m.n; ui++) {
      i64 sb = src->node_off[m.src[ui]], sc = m.scale[ui], dd = m.dst[ui];
      i64 dbase = u_done[ui] - m.start[ui];
      for (i64 i = m.start[ui]; i < m.end[ui]; i++) {
        if (done[dbase + i]) continue;
        i64 n = sb + i;
        int st = table_add(dst, dd, src->keys[n], src->vals[n] * sc, src->grams, n * gw, 0);
        if (st == T_RETRY) pending++;
        else if (st == T_FULL) worst = T_FULL;
        else done[dbase + i] = 1;
      }
    }
    check_capacity(worst, msg);
    if (!pending) break;
  }
  return launches;
}

typedef struct {
  Tables* pool;
} BuCtx;

/* bottom_up_traverse visit, engine.py:419-439: own_insert_round
 * (_kernels.py:219-233) then merge_round over (ready r, child c, freq) */
static void loctbl_visit(Arena* A, const Dag* d, const Cfg* cfg, const i64* ready, i64 n,
                         void* vctx) {
  Tables* pool = ((BuCtx*)vctx)->pool;
  i64* lens = ANEW(A, i64, n);
  i64 tot = 0, np = 0;
  for (i64 i = 0; i < n; i++) {
    tot += lens[i] = d->own_off[ready[i] + 1] - d->own_off[ready[i]];
    np += d->sub_off[ready[i] + 1] - d->sub_off[ready[i]];
  }
  Units u = partition_work(A, ready, lens, n, tot, cfg->chunk_factor);
  int worst = T_OK;
#pragma omp parallel for schedule(dynamic, 16) num_threads(cfg->workers) reduction(max : worst)
  for (i64 ui = 0; ui < u.n; ui++) {
    i64 r = u.id[ui], base = d->own_off[r];
    for (i64 j = u.start[ui]; j < u.end[ui]; j++) {
      int st = table_add(pool, r, d->own_ids[base + j], d->own_freqs[base + j], NULL, 0, 1);
      if (st > worst) worst = st;
    }
  }
  check_capacity(worst, BOUNDS_MSG);
  i64* pd = ANEW(A, i64, np);
  i64* ps = ANEW(A, i64, np);
  i64* pf = ANEW(A, i64, np);
  i64 k = 0;
  for (i64 i = 0; i < n; i++)
    for (i64 j = d->sub_off[ready[i]]; j < d->sub_off[ready[i] + 1]; j++) {
      pd[k] = ready[i];
      ps[k] = d->sub_ids[j];
      pf[k] = d->sub_freqs[j];
      k++;
    }
  MUnits m = merge_units(A, pd, ps, pf, np, pool, cfg);
  check_capacity(merge_round(pool, pool, &m, cfg), BOUNDS_MSG);
}

/* reduce_bottom_up, engine.py:478-518 (output tables inside the pool) */
static void reduce_bottom_up(Arena* A, const Dag* d, const Cfg* cfg, Tables* pool, int per_file,
                             i64 out_base) {
  check_capacity(root_words(A, d, pool, per_file, out_base, cfg), CAP_MSG);
  i64 F = d->F;
  i64 nc = d->sub_off[1] - d->sub_off[0];
  i64 cap = per_file ? nc * F : nc;
  i64* pd = ANEW(A, i64, cap + 1);
  i64* ps = ANEW(A, i64, cap + 1);
  i64* pf = ANEW(A, i64, cap + 1);
  i64 k = 0;
  if (per_file) {
    i64* seg = segment_rule_counts(A, d);
    for (i64 j = d->sub_off[0]; j < d->sub_off[1]; j++) {
      i64 c = d->sub_ids[j];
      for (i64 f = 0; f < F; f++) {
        i64 fr = seg[c * F + f];
        if (fr > 0) {
          pd[k] = out_base + f;
          ps[k] = c;
          pf[k] = fr;
          k++;
        }
      }
    }
  } else {
    for (i64 j = d->sub_off[0]; j < d->sub_off[1]; j++) {
      pd[k] = out_base;
      ps[k] = d->sub_ids[j];
      pf[k] = d->sub_freqs[j];
      k++;
    }
  }
  merge_with_retries(A, pool, pool, pd, ps, pf, k, cfg, CAP_MSG);
}

/* tasks.py:91-119 word tables: returns the table set and the index of the
 * first output table */
static Tables* word_tables(Arena* A, const Dag* d, const Cfg* cfg, int per_file, i64* first) {
  Tables* t = ANEW(A, Tables, 1);
  State s;
  if (cfg->strategy == GT_TOPDOWN) {
    state_init(A, &s, d, per_file ? d->F : 1);
    init_top_down(A, d, &s);
    top_down_traverse(A, d, &s, cfg);
    reduce_top_down(A, d, &s, cfg, t);
    *first = 0;
    return t;
  }
  state_init(A, &s, d, 1);
  i64* bound = local_table_bounds(A, d, &s, cfg, NULL, NULL);
  i64 T;
  i64* extra = word_table_bounds(A, d, per_file, &T);
  i64* all = ANEW(A, i64, d->R + T);
  memcpy(all, bound, sizeof(i64) * d->R);
  memcpy(all + d->R, extra, sizeof(i64) * T);
  tables_init(A, t, all, d->R + T, 0); /* plan_pool, engine.py:370-377 */
  BuCtx bc = {t};
  init_bottom_up(d, &s);
  bottom_up_rounds(A, d, &s, cfg, loctbl_visit, &bc, "loctbl");
  reduce_bottom_up(A, d, cfg, t, per_file, d->R);
  *first = d->R;
  return t;
}

/* ------------------------------------------------------------------------ */
/* sequences (sequence.py)                                                   */
/* ------------------------------------------------------------------------ */

#define GAP (-2)
#define OWN (-1)

static i64 head_tail_bound(i64 word_size, i64 l, i64 sub_rule_size) { /* sequence.py:50-55 */
  i64 v = word_size + (l - 1) * sub_rule_size - (l - 1);
  return v > 0 ? v : 0;
}

typedef struct {
  i64 m;              /* l - 1 */
  i64 *head, *tail;   /* R x m */
  i64 *hlen, *tlen;   /* lengths */
  int8_t* ready;
} HeadTail;

/* _prefix, sequence.py:72-89; returns 0 if blocked by an unready child */
static int prefix_of(const Dag* d, HeadTail* h, i64 r, i64 target, i64* acc, i64* nacc) {
  const Grammar* g = &d->g;
  i64 n = 0;
  for (i64 i = g->boff[r]; i < g->boff[r + 1]; i++) {
    if (n >= target) break;
    i64 s = g->body[i];
    if (s < g->nw) {
      acc[n++] = s;
    } else if (s >= g->base) {
      i64 c = s - g->base;
      if (!h->ready[c]) return 0;
      for (i64 j = 0; j < h->hlen[c]; j++) acc[n++] = h->head[c * h->m + j];
    }
  }
  *nacc = n < target ? n : target;
  return 1;
}

/* _suffix, sequence.py:92-107 (acc built reversed) */
static int suffix_of(const Dag* d, HeadTail* h, i64 r, i64 target, i64* acc, i64* nacc) {
  const Grammar* g = &d->g;
  i64 n = 0;
  for (i64 i = g->boff[r + 1] - 1; i >= g->boff[r]; i--) {
    if (n >= target) break;
    i64 s = g->body[i];
    if (s < g->nw) {
      acc[n++] = s;
    } else if (s >= g->base) {
      i64 c = s - g->base;
      if (!h->ready[c]) return 0;
      for (i64 j = h->tlen[c] - 1; j >= 0; j--) acc[n++] = h->tail[c * h->m + j];
    }
  }
  *nacc = n < target ? n : target; /* acc[:target][::-1] */
  return 1;
}

/* init_head_tail, sequence.py:110-140 */
static void init_head_tail(Arena* A, const Dag* d, i64 l, HeadTail* h) {
  i64 R = d->R, m = l - 1;
  h->m = m > 0 ? m : 0;
  i64 mm = h->m ? h->m : 1;
  h->head = ANEW(A, i64, R * mm);
  h->tail = ANEW(A, i64, R * mm);
  h->hlen = ANEW(A, i64, R);
  h->tlen = ANEW(A, i64, R);
  h->ready = ANEW(A, int8_t, R);
  int8_t* hdone = ANEW(A, int8_t, R);
  int8_t* tdone = ANEW(A, int8_t, R);
  h->ready[0] = hdone[0] = tdone[0] = 1;
  i64* pend = ANEW(A, i64, R);
  i64 np = 0;
  for (i64 r = 1; r < R; r++) pend[np++] = r;
  /* acc buffers: at most target-1 + (l-1) words */
  i64* acc = ANEW(A, i64, 2 * mm + 2);
  i64 rounds = 0;
  while (np) {
    rounds++;
    if (rounds > d->depth + 1) die(GT_E_CORRUPTION, "head/tail initialization exceeded depth bound");
    i64 still = 0;
    for (i64 i = 0; i < np; i++) {
      i64 r = pend[i];
      i64 target = d->exp_len[r] < m ? d->exp_len[r] : m;
      if (target < 0) target = 0;
      i64 n;
      if (!hdone[r] && prefix_of(d, h, r, target, acc, &n)) {
        for (i64 j = 0; j < n; j++) h->head[r * mm + j] = acc[j];
        h->hlen[r] = n;
        hdone[r] = 1;
      }
      if (!tdone[r] && suffix_of(d, h, r, target, acc, &n)) {
        for (i64 j = 0; j < n; j++) h->tail[r * mm + j] = acc[n - 1 - j];
        h->tlen[r] = n;
        tdone[r] = 1;
      }
      if (hdone[r] && tdone[r]) h->ready[r] = 1;
      else pend[still++] = r;
    }
    np = still;
  }
}

typedef struct {
  i64 n;       /* total stream length */
  i64* words;
  i64* region;
  i64* start;  /* per stream, n_streams + 1 */
} Streams;

/* length of _stream_of(body) without building it */
static i64 stream_len(const Dag* d, const HeadTail* h, i64 lo, i64 hi, i64 l) {
  const Grammar* g = &d->g;
  i64 n = 0;
  for (i64 i = lo; i < hi; i++) {
    i64 s = g->body[i];
    if (s < g->base) n++;
    else {
      i64 c = s - g->base, el = d->exp_len[c];
      if (el < l) n += el;
      else if (el <= 2 * (l - 1)) n += el;
      else n += h->hlen[c] + 1 + h->tlen[c];
    }
  }
  return n;
}

/* _stream_of, sequence.py:162-201 */
static void stream_fill(const Dag* d, const HeadTail* h, i64 lo, i64 hi, i64 l, i64* w, i64* rg) {
  const Grammar* g = &d->g;
  i64 k = 0, span = 0, mm = h->m ? h->m : 1;
  for (i64 i = lo; i < hi; i++) {
    i64 s = g->body[i];
    if (s < g->nw) {
      w[k] = s;
      rg[k++] = OWN;
    } else if (s < g->base) {
      w[k] = 0;
      rg[k++] = GAP;
    } else {
      i64 c = s - g->base, el = d->exp_len[c];
      if (el < l) {
        for (i64 j = 0; j < el; j++) {
          w[k] = h->head[c * mm + j];
          rg[k++] = OWN;
        }
      } else if (el <= 2 * (l - 1)) {
        i64 overlap = 2 * (l - 1) - el;
        for (i64 j = 0; j < h->hlen[c]; j++) {
          w[k] = h->head[c * mm + j];
          rg[k++] = span;
        }
        for (i64 j = overlap; j < h->tlen[c]; j++) {
          w[k] = h->tail[c * mm + j];
          rg[k++] = span;
        }
        span++;
      } else {
        for (i64 j = 0; j < h->hlen[c]; j++) {
          w[k] = h->head[c * mm + j];
          rg[k++] = span;
        }
        w[k] = 0;
        rg[k++] = GAP;
        for (i64 j = 0; j < h->tlen[c]; j++) {
          w[k] = h->tail[c * mm + j];
          rg[k++] = span;
        }
        span++;
      }
    }
  }
}

/* build_local_stream for r in 1..R-1 (or build_segment_stream per file),
 * concatenated like _concat_streams, sequence.py:259-274 */
static Streams build_streams(Arena* A, const Dag* d, const HeadTail* h, i64 l, int segments) {
  Streams s;
  i64 ns = segments ? d->F : d->R;
  s.start = ANEW(A, i64, ns + 1);
  const Grammar* g = &d->g;
  for (i64 i = 0; i < ns; i++) {
    i64 lo, hi;
    if (segments) {
      lo = g->boff[0] + d->seg_lo[i];
      hi = g->boff[0] + d->seg_hi[i];
    } else {
      lo = g->boff[i];
      hi = i ? g->boff[i + 1] : lo; /* the root has no rule stream */
    }
    s.start[i + 1] = s.start[i] + stream_len(d, h, lo, hi, l);
  }
  s.n = s.start[ns];
  s.words = ANEW(A, i64, s.n);
  s.region = ANEW(A, i64, s.n);
  for (i64 i = 0; i < ns; i++) {
    i64 lo, hi;
    if (segments) {
      lo = g->boff[0] + d->seg_lo[i];
      hi = g->boff[0] + d->seg_hi[i];
    } else {
      lo = g->boff[i];
      hi = i ? g->boff[i + 1] : lo;
    }
    stream_fill(d, h, lo, hi, l, s.words + s.start[i], s.region + s.start[i]);
  }
  return s;
}

static inline i64 window_starts(const Streams* s, i64 i, i64 l) { /* LocalStream.window_starts */
  i64 v = s->start[i + 1] - s->start[i] - (l - 1);
  return v > 0 ? v : 0;
}

/* _window_units (sequence.py:277-289) + window_count_round (_kernels.py:279-309)
 * over the listed streams; dst[i]/scale 1 as in every call site */
static int window_count(Arena* A, const Streams* s, const i64* which, i64 nwhich,
                        const i64* dst_of, i64 l, i64 wbits, i64 gw, Tables* t, const Cfg* cfg) {
  i64* lens = ANEW(A, i64, nwhich + 1);
  i64 tot = 0;
  for (i64 i = 0; i < nwhich; i++) tot += lens[i] = window_starts(s, which[i], l);
  Units u = partition_work(A, which, lens, nwhich, tot, cfg->chunk_factor);
  int worst = T_OK;
#pragma omp parallel for schedule(dynamic, 16) num_threads(cfg->workers) reduction(max : worst)
  for (i64 ui = 0; ui < u.n; ui++) {
    i64 key_i = u.id[ui], tt = dst_of[key_i], base = s->start[key_i];
    for (i64 p = base + u.start[ui]; p < base + u.end[ui]; p++) {
      int blocked = 0;
      for (i64 j = 0; j < l; j++)
        if (s->region[p + j] == GAP) {
          blocked = 1;
          break;
        }
      if (blocked) continue;
      if (s->region[p] >= 0 && s->region[p] == s->region[p + l - 1]) continue;
      i64 key = gw == 0 ? pack_key(s->words, p, l, wbits) : fingerprint(s->words, p, l);
      int st = table_add(t, tt, key, 1, s->words, p, 1);
      if (st > worst) worst = st;
    }
  }
  return worst;
}

typedef struct {
  Tables* pool;
  const Streams* rs;
  i64 l, wbits, gw;
  const i64* ident;
} SeqBuCtx;

/* count_sequences bottom-up visit, sequence.py:378-403 */
static void seq_visit(Arena* A, const Dag* d, const Cfg* cfg, const i64* ready, i64 n, void* vctx) {
  SeqBuCtx* c = vctx;
  check_capacity(window_count(A, c->rs, ready, n, c->ident, c->l, c->wbits, c->gw, c->pool, cfg),
                 SEQ_MSG);
  i64 np = 0;
  for (i64 i = 0; i < n; i++) np += d->sub_off[ready[i] + 1] - d->sub_off[ready[i]];
  i64* pd = ANEW(A, i64, np + 1);
  i64* ps = ANEW(A, i64, np + 1);
  i64* pf = ANEW(A, i64, np + 1);
  i64 k = 0;
  for (i64 i = 0; i < n; i++)
    for (i64 j = d->sub_off[ready[i]]; j < d->sub_off[ready[i] + 1]; j++) {
      pd[k] = ready[i];
      ps[k] = d->sub_ids[j];
      pf[k] = d->sub_freqs[j];
      k++;
    }
  MUnits m = merge_units(A, pd, ps, pf, np, c->pool, cfg);
  check_capacity(merge_round(c->pool, c->pool, &m, cfg), SEQ_MSG);
}

/* pack_width, sequence.py:229-231 */
static i64 pack_width(const Dag* d) {
  i64 v = d->g.nw - 1, b = 0;
  if (v < 0) v = -v; /* int(-1).bit_length() == 1 */
  while (v) {
    b++;
    v >>= 1;
  }
  return b > 1 ? b : 1;
}

/* count_sequences, sequence.py:292-417 -> per-file output tables */
static Tables* count_sequences(Arena* A, const Dag* d, const Cfg* cfg, i64 l, i64* wbits_out) {
  if (l < 1) die(GT_E_USAGE, "sequence length must be >= 1");
  i64 F = d->F, R = d->R;
  HeadTail h;
  init_head_tail(A, d, l, &h);
  i64 wbits = pack_width(d);
  int packed = l * wbits <= 63;
  i64 gw = packed ? 0 : l;
  i64 kw = packed ? wbits : 0;
  *wbits_out = kw;
  Streams rs = build_streams(A, d, &h, l, 0);
  Streams ss = build_streams(A, d, &h, l, 1);
  i64* ob = ANEW(A, i64, F);
  for (i64 f = 0; f < F; f++) ob[f] = d->seg_tokens[f] - (l - 1) > 0 ? d->seg_tokens[f] - (l - 1) : 0;
  Tables* out = ANEW(A, Tables, 1);
  tables_init(A, out, ob, F, gw);
  i64* own_c = ANEW(A, i64, R);
  for (i64 r = 1; r < R; r++) own_c[r] = window_starts(&rs, r, l);
  i64* ident = ANEW(A, i64, R > F ? R : F);
  for (i64 i = 0; i < (R > F ? R : F); i++) ident[i] = i;
  i64* segs = ANEW(A, i64, F);
  for (i64 f = 0; f < F; f++) segs[f] = f;
  Tables* pool = ANEW(A, Tables, 1);
  if (cfg->strategy == GT_TOPDOWN) {
    State s;
    state_init(A, &s, d, F);
    init_top_down(A, d, &s);
    top_down_traverse(A, d, &s, cfg);
    i64* b = ANEW(A, i64, R);
    for (i64 r = 1; r < R; r++) {
      i64 x = head_tail_bound(d->own_tok[r], l, d->num_out[r]);
      b[r] = x > own_c[r] ? x : own_c[r];
    }
    tables_init(A, pool, b, R, gw);
    i64* rules = ANEW(A, i64, R);
    for (i64 r = 1; r < R; r++) rules[r - 1] = r;
    check_capacity(window_count(A, &rs, rules, R - 1, ident, l, kw, gw, pool, cfg), SEQ_MSG);
    i64 np = 0;
    for (i64 r = 1; r < R; r++)
      for (i64 f = 0; f < F; f++) np += s.wmat[r * F + f] > 0;
    i64* pd = ANEW(A, i64, np + 1);
    i64* ps = ANEW(A, i64, np + 1);
    i64* pf = ANEW(A, i64, np + 1);
    i64 k = 0;
    for (i64 r = 1; r < R; r++)
      for (i64 f = 0; f < F; f++)
        if (s.wmat[r * F + f] > 0) {
          pd[k] = f;
          ps[k] = r;
          pf[k] = s.wmat[r * F + f];
          k++;
        }
    check_capacity(window_count(A, &ss, segs, F, ident, l, kw, gw, out, cfg), SEQ_MSG);
    merge_with_retries(A, out, pool, pd, ps, pf, np, cfg, CAP_MSG);
  } else {
    State s;
    state_init(A, &s, d, 1);
    i64* caps = ANEW(A, i64, R);
    for (i64 r = 0; r < R; r++) caps[r] = d->exp_len[r] - (l - 1) > 0 ? d->exp_len[r] - (l - 1) : 0;
    i64* bound = local_table_bounds(A, d, &s, cfg, own_c, caps);
    tables_init(A, pool, bound, R, gw);
    init_bottom_up(d, &s);
    SeqBuCtx c = {pool, &rs, l, kw, gw, ident};
    bottom_up_rounds(A, d, &s, cfg, seq_visit, &c, "seq-loctbl");
    check_capacity(window_count(A, &ss, segs, F, ident, l, kw, gw, out, cfg), SEQ_MSG);
    i64* seg = segment_rule_counts(A, d);
    i64 nc = d->sub_off[1] - d->sub_off[0];
    i64* pd = ANEW(A, i64, nc * F + 1);
    i64* ps = ANEW(A, i64, nc * F + 1);
    i64* pf = ANEW(A, i64, nc * F + 1);
    i64 k = 0;
    for (i64 j = d->sub_off[0]; j < d->sub_off[1]; j++) {
      i64 cc = d->sub_ids[j];
      for (i64 f = 0; f < F; f++)
        if (seg[cc * F + f] > 0) {
          pd[k] = f;
          ps[k] = cc;
          pf[k] = seg[cc * F + f];
          k++;
        }
    }
    merge_with_retries(A, out, pool, pd, ps, pf, k, cfg, CAP_MSG);
  }
  return out;
}

/* ------------------------------------------------------------------------ */
/* result assembly (tasks.py:91-185)                                         */
/* ------------------------------------------------------------------------ */

typedef struct {
  gt_view v;
  void* bufs[8];
} ORes;

static void* rmalloc(ORes* o, int slot, size_t n, size_t sz) {
  if (n == 0) n = 1;
  void* p = calloc(n, sz);
  if (!p) die(GT_E_RESOURCE, "out of host memory for results");
  o->bufs[slot] = p;
  return p;
}

typedef struct {
  i64 a, b, c; /* sort record */
} Rec3;

static int cmp_word(const void* x, const void* y) { /* by word id */
  const Rec3 *p = x, *q = y;
  return (p->a > q->a) - (p->a < q->a);
}
static int cmp_negcount_word(const void* x, const void* y) { /* (-count, id) */
  const Rec3 *p = x, *q = y;
  if (p->b != q->b) return p->b < q->b ? 1 : -1;
  return (p->a > q->a) - (p->a < q->a);
}
static int cmp_word_file(const void* x, const void* y) {
  const Rec3 *p = x, *q = y;
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  return (p->b > q->b) - (p->b < q->b);
}

static void word_result(Arena* A, const Dag* d, const Cfg* cfg, int task, ORes* o) {
  int per_file = task == GT_INVERTEDINDEX || task == GT_TERMVECTOR;
  i64 first;
  Tables* t = word_tables(A, d, cfg, per_file, &first);
  gt_view* v = &o->v;
  if (!per_file) {
    i64 n = tsize(t, first), b = t->node_off[first];
    Rec3* rec = ANEW(A, Rec3, n);
    for (i64 i = 0; i < n; i++) rec[i] = (Rec3){t->keys[b + i], t->vals[b + i], 0};
    qsort(rec, (size_t)n, sizeof(Rec3), task == GT_SORT ? cmp_negcount_word : cmp_word);
    uint32_t* id = rmalloc(o, 0, n, 4);
    uint64_t* cnt = rmalloc(o, 1, n, 8);
    for (i64 i = 0; i < n; i++) {
      id[i] = (uint32_t)rec[i].a;
      cnt[i] = (u64)rec[i].b;
    }
    v->n = (u64)n;
    v->id = id;
    v->count = cnt;
    return;
  }
  i64 F = d->F, tot = 0;
  for (i64 f = 0; f < F; f++) tot += tsize(t, first + f);
  if (task == GT_TERMVECTOR) {
    uint64_t* off = rmalloc(o, 0, F + 1, 8);
    uint32_t* id = rmalloc(o, 1, tot, 4);
    uint64_t* cnt = rmalloc(o, 2, tot, 8);
    i64 k = 0;
    for (i64 f = 0; f < F; f++) {
      i64 n = tsize(t, first + f), b = t->node_off[first + f];
      Rec3* rec = ANEW(A, Rec3, n);
      for (i64 i = 0; i < n; i++) rec[i] = (Rec3){t->keys[b + i], t->vals[b + i], 0};
      qsort(rec, (size_t)n, sizeof(Rec3), cmp_negcount_word);
      off[f] = (u64)k;
      for (i64 i = 0; i < n; i++) {
        id[k] = (uint32_t)rec[i].a;
        cnt[k++] = (u64)rec[i].b;
      }
    }
    off[F] = (u64)k;
    v->n_groups = (u64)F;
    v->group_off = off;
    v->n = (u64)tot;
    v->id = id;
    v->count = cnt;
    return;
  }
  /* inverted index: word -> ascending files (tasks.py:133-140) */
  Rec3* rec = ANEW(A, Rec3, tot);
  i64 k = 0;
  for (i64 f = 0; f < F; f++) {
    i64 n = tsize(t, first + f), b = t->node_off[first + f];
    for (i64 i = 0; i < n; i++) rec[k++] = (Rec3){t->keys[b + i], f, 0};
  }
  qsort(rec, (size_t)tot, sizeof(Rec3), cmp_word_file);
  i64 ng = 0;
  for (i64 i = 0; i < tot; i++) ng += (i == 0 || rec[i].a != rec[i - 1].a);
  uint64_t* off = rmalloc(o, 0, ng + 1, 8);
  uint32_t* gid = rmalloc(o, 1, ng, 4);
  uint32_t* id = rmalloc(o, 2, tot, 4);
  i64 g = -1;
  for (i64 i = 0; i < tot; i++) {
    if (i == 0 || rec[i].a != rec[i - 1].a) {
      g++;
      gid[g] = (uint32_t)rec[i].a;
      off[g] = (u64)i;
    }
    id[i] = (uint32_t)rec[i].b;
  }
  off[ng] = (u64)tot;
  v->n_groups = (u64)ng;
  v->group_off = off;
  v->group_id = gid;
  v->n = (u64)tot;
  v->id = id;
  v->count = NULL;
}

/* gram records: key or gram words + count + file */
typedef struct {
  i64 key;  /* packed key, or node index into the gram table (gram mode) */
  i64 count;
  i64 file;
} GRec;

static __thread const i64* g_gr; /* gram-mode comparison context */
static __thread i64 g_gw;

static int gram_cmp(const GRec* p, const GRec* q) {
  if (!g_gw) return (p->key > q->key) - (p->key < q->key);
  for (i64 j = 0; j < g_gw; j++) {
    i64 a = g_gr[p->key * g_gw + j], b = g_gr[q->key * g_gw + j];
    if (a != b) return a < b ? -1 : 1;
  }
  return 0;
}
static int cmp_negcount_gram(const void* x, const void* y) { /* render order, tasks.py:250-255 */
  const GRec *p = x, *q = y;
  if (p->count != q->count) return p->count < q->count ? 1 : -1;
  return gram_cmp(p, q);
}
static int cmp_gram_negcount_file(const void* x, const void* y) { /* tasks.py:162-168,256 */
  const GRec *p = x, *q = y;
  int c = gram_cmp(p, q);
  if (c) return c;
  if (p->count != q->count) return p->count < q->count ? 1 : -1;
  return (p->file > q->file) - (p->file < q->file);
}

static void seq_result(Arena* A, const Dag* d, const Cfg* cfg, int task, i64 l, ORes* o) {
  i64 wbits;
  Tables* t = count_sequences(A, d, cfg, l, &wbits);
  gt_view* v = &o->v;
  v->wbits = (int32_t)wbits;
  i64 F = d->F, gw = t->gw, tot = 0;
  for (i64 f = 0; f < F; f++) tot += tsize(t, f);
  GRec* rec = ANEW(A, GRec, tot);
  i64 k = 0;
  for (i64 f = 0; f < F; f++) {
    i64 n = tsize(t, f), b = t->node_off[f];
    for (i64 i = 0; i < n; i++) rec[k++] = (GRec){gw ? b + i : t->keys[b + i], t->vals[b + i], f};
  }
  g_gr = t->grams;
  g_gw = gw;
  if (task == GT_SEQCOUNT) {
    uint64_t* off = rmalloc(o, 0, F + 1, 8);
    uint64_t* cnt = rmalloc(o, 1, tot, 8);
    uint64_t* key = gw ? NULL : rmalloc(o, 2, tot, 8);
    uint32_t* gram = gw ? rmalloc(o, 3, tot * gw, 4) : NULL;
    for (i64 f = 0, s = 0; f < F; f++) {
      i64 n = tsize(t, f);
      qsort(rec + s, (size_t)n, sizeof(GRec), cmp_negcount_gram);
      off[f] = (u64)s;
      s += n;
    }
    off[F] = (u64)tot;
    for (i64 i = 0; i < tot; i++) {
      cnt[i] = (u64)rec[i].count;
      if (gw)
        for (i64 j = 0; j < gw; j++) gram[i * gw + j] = (uint32_t)t->grams[rec[i].key * gw + j];
      else key[i] = (u64)rec[i].key;
    }
    v->n_groups = (u64)F;
    v->group_off = off;
    v->n = (u64)tot;
    v->count = cnt;
    v->key = key;
    v->gram = gram;
    return;
  }
  qsort(rec, (size_t)tot, sizeof(GRec), cmp_gram_negcount_file);
  i64 ng = 0;
  for (i64 i = 0; i < tot; i++) ng += (i == 0 || gram_cmp(&rec[i], &rec[i - 1]) != 0);
  uint64_t* off = rmalloc(o, 0, ng + 1, 8);
  uint32_t* fid = rmalloc(o, 1, tot, 4);
  uint64_t* cnt = rmalloc(o, 2, tot, 8);
  uint64_t* gkey = gw ? NULL : rmalloc(o, 3, ng, 8);
  uint32_t* ggram = gw ? rmalloc(o, 4, ng * gw, 4) : NULL;
  i64 g = -1;
  for (i64 i = 0; i < tot; i++) {
    if (i == 0 || gram_cmp(&rec[i], &rec[i - 1]) != 0) {
      g++;
      off[g] = (u64)i;
      if (gw)
        for (i64 j = 0; j < gw; j++) ggram[g * gw + j] = (uint32_t)t->grams[rec[i].key * gw + j];
      else gkey[g] = (u64)rec[i].key;
    }
    fid[i] = (uint32_t)rec[i].file;
    cnt[i] = (u64)rec[i].count;
  }
  off[ng] = (u64)tot;
  v->n_groups = (u64)ng;
  v->group_off = off;
  v->group_key = gkey;
  v->group_gram = ggram;
  v->n = (u64)tot;
  v->id = fid;
  v->count = cnt;
}

/* ------------------------------------------------------------------------ */
/* exported oracle API (mirrors include/gtadoc_b200.h with a gto_ prefix)     */
/* ------------------------------------------------------------------------ */

typedef struct {
  Arena A;
  Dag d;
  double init_ms;
} OCtx;

int gto_open(const uint8_t* data, size_t n, int workers, OCtx** out) {
  jmp_buf jb;
  jmp_buf* prev = g_jb;
  OCtx* c = calloc(1, sizeof(OCtx));
  if (!c) return GT_E_RESOURCE;
  g_jb = &jb;
  double t0 = now_ms();
  if (setjmp(jb)) {
    arena_free(&c->A);
    free(c);
    g_jb = prev;
    return g_code;
  }
  deserialize(&c->A, data, n, &c->d.g);
  build_dag(&c->A, &c->d, workers > 0 ? workers : 1);
  c->init_ms = now_ms() - t0;
  g_jb = prev;
  *out = c;
  return GT_OK;
}

void gto_close(OCtx* c) {
  if (!c) return;
  arena_free(&c->A);
  free(c);
}

int gto_info(const OCtx* c, gt_info* o) {
  const Dag* d = &c->d;
  memset(o, 0, sizeof *o);
  o->num_words = (u64)d->g.nw;
  o->num_splitters = (u64)d->g.ns;
  o->num_rules = (u64)d->R;
  o->num_files = (u64)d->F;
  o->total_elements = (u64)d->E;
  o->root_len = (u64)(d->g.boff[1] - d->g.boff[0]);
  o->sub_pairs = (u64)d->sub_off[d->R];
  o->own_pairs = (u64)d->own_off[d->R];
  o->words = (u64)d->exp_len[0];
  o->depth = d->depth;
  o->td_levels = d->td_levels;
  o->bu_levels = d->bu_levels;
  o->init_ms = c->init_ms;
  o->td_edges = (u64)(d->sub_off[d->R] - d->sub_off[d->R > 1 ? 1 : d->R]);
  return GT_OK;
}

int64_t gto_dag_array(OCtx* c, const char* name, int64_t* out, int64_t cap) {
  const Dag* d = &c->d;
  const i64* src = NULL;
  i64 n = 0, R = d->R;
  i64 tmp_n = 0;
  if (!strcmp(name, "own_ids")) src = d->own_ids, n = d->own_off[R];
  else if (!strcmp(name, "own_freqs")) src = d->own_freqs, n = d->own_off[R];
  else if (!strcmp(name, "own_off")) src = d->own_off, n = R + 1;
  else if (!strcmp(name, "own_token_count")) src = d->own_tok, n = R;
  else if (!strcmp(name, "sub_ids")) src = d->sub_ids, n = d->sub_off[R];
  else if (!strcmp(name, "sub_freqs")) src = d->sub_freqs, n = d->sub_off[R];
  else if (!strcmp(name, "sub_off")) src = d->sub_off, n = R + 1;
  else if (!strcmp(name, "par_ids")) src = d->par_ids, n = d->sub_off[R];
  else if (!strcmp(name, "par_freqs")) src = d->par_freqs, n = d->sub_off[R];
  else if (!strcmp(name, "par_off")) src = d->par_off, n = R + 1;
  else if (!strcmp(name, "num_in_edge")) src = d->num_in, n = R;
  else if (!strcmp(name, "num_out_edge")) src = d->num_out, n = R;
  else if (!strcmp(name, "root_freq")) src = d->root_freq, n = R;
  else if (!strcmp(name, "exp_len")) src = d->exp_len, n = R;
  else if (!strcmp(name, "td_level")) src = d->td_level, n = R;
  else if (!strcmp(name, "bu_level")) src = d->bu_level, n = R;
  else if (!strcmp(name, "segment_token_counts")) src = d->seg_tokens, n = d->F;
  else if (!strcmp(name, "segments")) tmp_n = 2 * d->F, n = tmp_n;
  else return -1;
  if (!out) return n;
  if (cap < n) return -1;
  if (tmp_n) {
    for (i64 f = 0; f < d->F; f++) {
      out[2 * f] = d->seg_lo[f];
      out[2 * f + 1] = d->seg_hi[f];
    }
  } else {
    memcpy(out, src, sizeof(i64) * (size_t)n);
  }
  return n;
}

int gto_run(OCtx* c, int task, int seq_len, int strategy, int file_set_width, int workers,
            ORes** out) {
  jmp_buf jb;
  jmp_buf* prev = g_jb;
  Arena A = {0};
  ORes* o = calloc(1, sizeof(ORes));
  if (!o) return GT_E_RESOURCE;
  g_jb = &jb;
  if (setjmp(jb)) {
    arena_free(&A);
    for (int i = 0; i < 8; i++) free(o->bufs[i]);
    free(o);
    g_jb = prev;
    return g_code;
  }
  if (task < 0 || task > GT_RANKEDINVERTEDINDEX) die(GT_E_USAGE, "unknown task %d", task);
  if (strategy < GT_AUTO || strategy > GT_BOTTOMUP) die(GT_E_USAGE, "unknown strategy %d", strategy);
  double t0 = now_ms();
  Cfg cfg = {0, workers > 0 ? workers : 1, 16, file_set_width};
  cfg.strategy = select_strategy(&c->d, task, strategy, file_set_width);
  o->v.task = task;
  o->v.seq_len = seq_len;
  o->v.strategy = cfg.strategy;
  if (task <= GT_TERMVECTOR) word_result(&A, &c->d, &cfg, task, o);
  else seq_result(&A, &c->d, &cfg, task, seq_len, o);
  o->v.total_ms = now_ms() - t0;
  arena_free(&A);
  g_jb = prev;
  *out = o;
  return GT_OK;
}

int gto_view(const ORes* o, gt_view* v) {
  *v = o->v;
  return GT_OK;
}

void gto_free(ORes* o) {
  if (!o) return;
  for (int i = 0; i < 8; i++) free(o->bufs[i]);
  free(o);
}
