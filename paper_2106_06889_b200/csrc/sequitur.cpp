// sequitur.cpp — native corpus ingestion and Sequitur grammar inference
// (host code), producing the reference's GTDC bytes bit for bit.
//
// the reference compressor (sequitur.py:46-258, in
// Python) runs at ~10^5 symbols/s, so real GB-scale corpora are out of its
// reach.  This is the same online algorithm — digram uniqueness + rule
// utility, folding a repeated digram into a rule, inlining a rule whose
// reference count drops to one, lowest-free rule ids (so the grammar is a
// pure function of the stream) — over an index-based node pool instead of
// Python objects: rule references keep an intrusive per-rule list (the
// reference's `uses` sets; the single survivor of an inline is its head),
// the digram index is a hash map keyed by the packed symbol pair, the free
// ids a min-heap.  Every step happens in the reference's order, which the
// output bytes depend on; tests/test_sequitur_native.py compares the bytes
// with the reference-generated golden grammars.
//
// Ingestion (ingest.py:30-121): UTF-8 validation with the decoder's error
// offset, whitespace tokenization with Python str.split() semantics (the
// Unicode White_Space set), first-appearance word ids, one splitter after
// every file; serialization grammar.py:164-174.
#include <stdint.h>
#include <string.h>

#include <functional>
#include <queue>
#include <string>
#include <string_view>
#include <unordered_map>
#include <stdexcept>
#include <vector>

#include "../../include/gtadoc_b200.h"

namespace gt {
namespace {

constexpr uint32_t NIL = 0xFFFFFFFFu;

struct Node {
  int32_t sym;      // >= 0 terminal (stream id), < 0 reference to rule -sym
  int32_t rule_id;  // >= 0 on guard nodes only
  uint32_t prev, next;
  uint32_t use_prev, use_next;  // intrusive list of a rule's references
  bool dead, in_uses;
};

// open-addressing digram index: linear probing, backward-shift deletion
// (no tombstones), load <= 1/2; keys are biased so no key equals kEmptyKey
struct DigramMap {
  static constexpr uint64_t kEmptyKey = ~0ull;
  std::vector<uint64_t> keys;
  std::vector<uint32_t> vals;
  uint64_t mask = 0, size = 0;
  DigramMap() { rehash(1 << 16); }
  static uint64_t mix(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return k;
  }
  void rehash(uint64_t cap) {
    std::vector<uint64_t> ok = std::move(keys);
    std::vector<uint32_t> ov = std::move(vals);
    keys.assign(cap, kEmptyKey);
    vals.assign(cap, 0);
    mask = cap - 1;
    size = 0;
    for (size_t i = 0; i < ok.size(); i++)
      if (ok[i] != kEmptyKey) put(ok[i], ov[i]);
  }
  // slot of key, or of the empty slot where it would go
  uint64_t slot(uint64_t k) const {
    uint64_t i = mix(k) & mask;
    while (keys[i] != kEmptyKey && keys[i] != k) i = (i + 1) & mask;
    return i;
  }
  bool get(uint64_t k, uint32_t* v) const {
    const uint64_t i = slot(k);
    if (keys[i] == kEmptyKey) return false;
    *v = vals[i];
    return true;
  }
  void put(uint64_t k, uint32_t v) {
    if (2 * (size + 1) > mask + 1) rehash(2 * (mask + 1));
    const uint64_t i = slot(k);
    if (keys[i] == kEmptyKey) {
      keys[i] = k;
      size++;
    }
    vals[i] = v;
  }
  void erase(uint64_t k) {
    uint64_t i = slot(k);
    if (keys[i] == kEmptyKey) return;
    // backward shift: pull later entries of the probe run into the hole
    uint64_t j = i;
    for (;;) {
      j = (j + 1) & mask;
      if (keys[j] == kEmptyKey) break;
      const uint64_t h = mix(keys[j]) & mask;
      // move j to i unless its home h lies cyclically in (i, j]
      if ((j > i && (h <= i || h > j)) || (j < i && (h <= i && h > j))) {
        keys[i] = keys[j];
        vals[i] = vals[j];
        i = j;
      }
    }
    keys[i] = kEmptyKey;
    size--;
  }
};

struct Builder {
  std::vector<Node> nodes;
  std::vector<uint32_t> guard;  // rule id -> guard node (NIL if not live)
  struct Uses {
    uint32_t head = NIL;
    uint32_t count = 0;
    bool live = false;
  };
  std::vector<Uses> uses;
  DigramMap index;
  int32_t next_id = 1;
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> free_ids;

  static uint64_t key_of(int32_t a, int32_t b) {
    return ((uint64_t)((uint32_t)a + 0x80000000u) << 32) | ((uint32_t)b + 0x80000000u);
  }

  uint32_t make(int32_t sym, int32_t rule_id = -1) {
    // node ids are u32 with NIL = 2^32 - 1; dead nodes are not reused, so a
    // corpus of ~10^9+ tokens could run out of ids: fail, never wrap
    if (nodes.size() >= (size_t)NIL - 1) throw std::length_error("grammar node pool exceeds 2^32 - 2 nodes");
    nodes.push_back(Node{sym, rule_id, NIL, NIL, NIL, NIL, false, false});
    return (uint32_t)nodes.size() - 1;
  }
  void join(uint32_t a, uint32_t b) {
    nodes[a].next = b;
    nodes[b].prev = a;
  }
  bool is_guard(uint32_t n) const { return nodes[n].rule_id >= 0; }

  Builder() {
    nodes.reserve(1 << 16);
    const uint32_t root = make(0, 0);
    join(root, root);
    set_rule(0, root);
  }
  void set_rule(int32_t rid, uint32_t g) {
    if ((size_t)rid >= guard.size()) {
      guard.resize(rid + 1, NIL);
      uses.resize(rid + 1);
    }
    guard[rid] = g;
  }

  // -- uses ------------------------------------------------------------------
  void use_add(int32_t rid, uint32_t n) {
    Uses& u = uses[rid];
    Node& x = nodes[n];
    x.use_prev = NIL;
    x.use_next = u.head;
    if (u.head != NIL) nodes[u.head].use_prev = n;
    u.head = n;
    u.count++;
    x.in_uses = true;
  }
  void use_discard(int32_t rid, uint32_t n) {
    Node& x = nodes[n];
    if (!x.in_uses) return;
    Uses& u = uses[rid];
    if (x.use_prev != NIL) nodes[x.use_prev].use_next = x.use_next;
    else u.head = x.use_next;
    if (x.use_next != NIL) nodes[x.use_next].use_prev = x.use_prev;
    u.count--;
    x.in_uses = false;
  }
  void track(uint32_t n) {
    if (nodes[n].sym < 0) use_add(-nodes[n].sym, n);
  }

  int32_t alloc_id() {
    if (!free_ids.empty()) {
      const int32_t r = free_ids.top();
      free_ids.pop();
      return r;
    }
    return next_id++;
  }

  // -- digram index (sequitur.py _check) ------------------------------------
  bool check(uint32_t a) {
    const uint32_t b = nodes[a].next;
    if (is_guard(a) || is_guard(b)) return false;
    const uint64_t key = key_of(nodes[a].sym, nodes[b].sym);
    uint32_t ex;
    if (!index.get(key, &ex)) {
      index.put(key, a);
      return false;
    }
    if (ex == a || nodes[ex].next == a || b == ex) return false;  // same / overlapping
    match(a, ex, nodes[a].sym, nodes[b].sym);
    return true;
  }

  void match(uint32_t a, uint32_t ex, int32_t k0, int32_t k1) {
    const uint32_t g = nodes[ex].prev;
    if (is_guard(g) && nodes[nodes[ex].next].next == g) {
      substitute(a, nodes[g].rule_id);  // the indexed occurrence is a whole rule body
    } else {
      const int32_t rid = alloc_id();
      const uint32_t ng = make(0, rid);
      const uint32_t x = make(k0), y = make(k1);
      join(ng, x);
      join(x, y);
      join(y, ng);
      set_rule(rid, ng);
      uses[rid] = Uses{NIL, 0, true};
      track(x);
      track(y);
      index.put(key_of(k0, k1), x);  // the canonical occurrence now lives in the body
      substitute(ex, rid);
      substitute(a, rid);
    }
    enforce(k0);
    enforce(k1);
  }

  uint32_t drop_entry(uint32_t first, uint32_t second) {
    if (is_guard(first) || is_guard(second)) return NIL;
    const uint64_t key = key_of(nodes[first].sym, nodes[second].sym);
    uint32_t cur;
    if (!index.get(key, &cur) || cur != first) return NIL;
    index.erase(key);
    const uint32_t o = nodes[first].prev;
    const int32_t fs = nodes[first].sym;
    if (!is_guard(o) && nodes[o].sym == fs && fs == nodes[second].sym) return o;  // left shadow
    const uint32_t nn = nodes[second].next;
    if (!is_guard(nn) && fs == nodes[second].sym && nodes[second].sym == nodes[nn].sym)
      return second;  // right shadow
    return NIL;
  }

  void substitute(uint32_t a, int32_t rid) {
    const uint32_t b = nodes[a].next;
    const uint32_t p = nodes[a].prev, n = nodes[b].next;
    const uint32_t left = drop_entry(p, a);
    {
      const uint64_t key = key_of(nodes[a].sym, nodes[b].sym);
      uint32_t cur;
      if (index.get(key, &cur) && cur == a) index.erase(key);
    }
    const uint32_t right = drop_entry(b, n);
    if (nodes[a].sym < 0) use_discard(-nodes[a].sym, a);
    if (nodes[b].sym < 0) use_discard(-nodes[b].sym, b);
    nodes[a].dead = nodes[b].dead = true;
    const uint32_t m = make(-rid);
    use_add(rid, m);
    nodes[p].next = m;
    nodes[m].prev = p;
    nodes[m].next = n;
    nodes[n].prev = m;
    check(p);
    if (!nodes[m].dead) check(m);
    for (uint32_t sh : {left, right})
      if (sh != NIL && !nodes[sh].dead && !nodes[nodes[sh].next].dead) check(sh);
  }

  void enforce(int32_t sym) {
    if (sym >= 0) return;
    const int32_t rid = -sym;
    if ((size_t)rid < uses.size() && uses[rid].live && guard[rid] != NIL && uses[rid].count == 1)
      inline_rule(rid, uses[rid].head);
  }

  void inline_rule(int32_t rid, uint32_t u) {
    const uint32_t g = guard[rid];
    guard[rid] = NIL;
    uses[rid] = Uses{};
    const uint32_t first = nodes[g].next, last = nodes[g].prev;
    const uint32_t p = nodes[u].prev, n = nodes[u].next;
    const uint32_t left = drop_entry(p, u);
    const uint32_t right = drop_entry(u, n);
    nodes[u].dead = true;
    nodes[u].in_uses = false;
    join(p, first);
    join(last, n);
    free_ids.push(rid);
    check(p);
    if (!nodes[last].dead) check(last);
    for (uint32_t sh : {left, right})
      if (sh != NIL && !nodes[sh].dead && !nodes[nodes[sh].next].dead) check(sh);
  }

  void append(int32_t sym) {
    const uint32_t root = guard[0];
    const uint32_t last = nodes[root].prev;
    const uint32_t x = make(sym);
    join(last, x);
    join(x, root);
    check(last);
  }
};

// Python str.isspace() code points (the separators of str.split())
bool py_space(uint32_t c) {
  if (c == 0x20 || (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x1F) || c == 0x85 || c == 0xA0) return true;
  if (c < 0x1680) return false;
  return c == 0x1680 || (c >= 0x2000 && c <= 0x200A) || c == 0x2028 || c == 0x2029 || c == 0x202F ||
         c == 0x205F || c == 0x3000;
}

// strict UTF-8 decode (CPython's rules); returns the first bad byte offset
// or -1, and the tokens (byte ranges) split on Python whitespace
int64_t tokenize(const uint8_t* s, size_t n, std::vector<std::string_view>* toks) {
  size_t i = 0, tok_start = 0;
  bool in_tok = false;
  while (i < n) {
    const uint8_t c = s[i];
    uint32_t cp;
    size_t k;
    if (c < 0x80) {
      cp = c;
      k = 1;
    } else {
      uint8_t lo = 0x80, hi = 0xBF;
      if (c >= 0xC2 && c <= 0xDF) k = 2, cp = c & 0x1F;
      else if (c == 0xE0) k = 3, lo = 0xA0, cp = c & 0x0F;
      else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) k = 3, cp = c & 0x0F;
      else if (c == 0xED) k = 3, hi = 0x9F, cp = c & 0x0F;
      else if (c == 0xF0) k = 4, lo = 0x90, cp = c & 0x07;
      else if (c >= 0xF1 && c <= 0xF3) k = 4, cp = c & 0x07;
      else if (c == 0xF4) k = 4, hi = 0x8F, cp = c & 0x07;
      else return (int64_t)i;
      for (size_t j = 1; j < k; j++) {
        if (i + j >= n) return (int64_t)i;
        const uint8_t cc = s[i + j];
        if (cc < (j == 1 ? lo : 0x80) || cc > (j == 1 ? hi : 0xBF)) return (int64_t)i;
        cp = (cp << 6) | (cc & 0x3F);
      }
    }
    const bool sp = py_space(cp);
    if (sp && in_tok) {
      toks->emplace_back((const char*)s + tok_start, i - tok_start);
      in_tok = false;
    } else if (!sp && !in_tok) {
      tok_start = i;
      in_tok = true;
    }
    i += k;
  }
  if (in_tok) toks->emplace_back((const char*)s + tok_start, n - tok_start);
  return -1;
}

thread_local std::string t_seq_err;

}  // namespace
}  // namespace gt

extern "C" {

const char* gt_compress_last_error(void) { return gt::t_seq_err.c_str(); }

int gt_compress(const uint8_t* const* files, const uint64_t* lens, uint64_t nfiles, uint8_t** out,
                uint64_t* out_len, uint64_t* stats) {
  using namespace gt;
  *out = nullptr;
  *out_len = 0;
  if (nfiles == 0) {
    t_seq_err = "corpus must contain at least one file";
    return GT_E_USAGE;
  }
  // ingest: first-appearance word ids, one splitter after every file
  std::unordered_map<std::string_view, int32_t> ids;
  std::vector<std::string_view> words;
  std::vector<int32_t> stream;
  std::vector<std::string_view> toks;
  for (uint64_t f = 0; f < nfiles; f++) {
    toks.clear();
    const int64_t bad = tokenize(files[f], lens[f], &toks);
    if (bad >= 0) {
      t_seq_err = "file " + std::to_string(f) + ": invalid UTF-8 at byte offset " + std::to_string(bad);
      if (stats) stats[0] = f;
      return GT_E_USAGE + 100;  // ingest error (exit code 2) — mapped by the caller
    }
    for (const auto& t : toks) {
      auto it = ids.find(t);
      int32_t w;
      if (it == ids.end()) {
        w = (int32_t)words.size();
        ids.emplace(t, w);
        words.push_back(t);
      } else {
        w = it->second;
      }
      stream.push_back(w);
    }
    stream.push_back(-1);
  }
  if ((uint64_t)words.size() + nfiles >= (1ull << 31)) {
    t_seq_err = "vocabulary + files exceed the 2^31 symbol ids of the compressor";
    return GT_E_RESOURCE;
  }
  const int32_t nw = (int32_t)words.size();
  for (uint64_t i = 0, f = 0; i < stream.size(); i++)
    if (stream[i] < 0) stream[i] = nw + (int32_t)(f++);
  // grammar inference
  Builder b;
  try {
    for (int32_t s : stream) b.append(s);
  } catch (const std::length_error& e) {
    t_seq_err = e.what();
    return GT_E_RESOURCE;
  } catch (const std::bad_alloc&) {
    t_seq_err = "out of host memory";
    return GT_E_RESOURCE;
  }
  // finalize: live rules in id order, compacted
  std::vector<int32_t> compact(b.guard.size(), -1);
  std::vector<int32_t> live;
  for (size_t r = 0; r < b.guard.size(); r++)
    if (b.guard[r] != NIL) {
      compact[r] = (int32_t)live.size();
      live.push_back((int32_t)r);
    }
  const uint32_t base = (uint32_t)nw + (uint32_t)nfiles;
  // serialize (grammar.py:164-174)
  std::string o;
  o.append("GTDC", 4);
  auto put32 = [&](uint32_t v) { o.append((const char*)&v, 4); };
  o.push_back((char)1);
  put32((uint32_t)nw);
  put32((uint32_t)nfiles);
  put32((uint32_t)live.size());
  for (const auto& w : words) {
    put32((uint32_t)w.size());
    o.append(w.data(), w.size());
  }
  std::vector<uint32_t> body;
  for (size_t k = 0; k < live.size(); k++) {
    body.clear();
    const uint32_t g = b.guard[live[k]];
    for (uint32_t x = b.nodes[g].next; x != g; x = b.nodes[x].next) {
      const int32_t s = b.nodes[x].sym;
      const uint32_t v = s >= 0 ? (uint32_t)s : base + (uint32_t)compact[-s];
      // _validate_splitters (sequitur.py): splitters only in the root, in order
      if (k != 0 && s >= 0 && s >= nw) {
        t_seq_err = "splitter " + std::to_string(s) + " escaped into rule " + std::to_string(k);
        return GT_E_CORRUPTION;
      }
      body.push_back(v);
    }
    put32((uint32_t)body.size());
    o.append((const char*)body.data(), body.size() * 4);
  }
  uint8_t* p = (uint8_t*)malloc(o.size());
  if (!p) {
    t_seq_err = "out of host memory";
    return GT_E_RESOURCE;
  }
  memcpy(p, o.data(), o.size());
  *out = p;
  *out_len = o.size();
  if (stats) {
    stats[0] = nfiles;
    stats[1] = live.size();
    stats[2] = (uint64_t)nw;
    stats[3] = stream.size();
  }
  return GT_OK;
}

void gt_compress_free(uint8_t* p) { free(p); }

// The ingest half of gt_compress alone: the corpus as word-id token streams
// (first-appearance ids — the dictionary order of the grammar gt_compress
// writes for the same files), one stream per file, no splitters.
int gt_tokenize(const uint8_t* const* files, const uint64_t* lens, uint64_t nfiles, uint32_t** tokens,
                uint64_t* file_off) {
  using namespace gt;
  *tokens = nullptr;
  std::unordered_map<std::string_view, uint32_t> ids;
  std::vector<uint32_t> stream;
  std::vector<std::string_view> toks;
  file_off[0] = 0;
  for (uint64_t f = 0; f < nfiles; f++) {
    toks.clear();
    const int64_t bad = tokenize(files[f], lens[f], &toks);
    if (bad >= 0) {
      t_seq_err = "file " + std::to_string(f) + ": invalid UTF-8 at byte offset " + std::to_string(bad);
      return GT_E_USAGE;
    }
    for (const auto& t : toks) {
      auto it = ids.find(t);
      uint32_t w;
      if (it == ids.end()) {
        w = (uint32_t)ids.size();
        ids.emplace(t, w);
      } else {
        w = it->second;
      }
      stream.push_back(w);
    }
    file_off[f + 1] = stream.size();
  }
  uint32_t* p = (uint32_t*)malloc(std::max<size_t>(stream.size(), 1) * 4);
  if (!p) {
    t_seq_err = "out of host memory";
    return GT_E_RESOURCE;
  }
  if (!stream.empty()) memcpy(p, stream.data(), stream.size() * 4);
  *tokens = p;
  return GT_OK;
}

}  // extern "C"
