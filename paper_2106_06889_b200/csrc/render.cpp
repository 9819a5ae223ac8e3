// render.cpp — native TSV rendering and SHA-256 output digest (host code).
//
// Byte-identical to the reference's `render` (tasks.py:233-263), whose
// sha256 is the CLI manifest's `outputDigest` (cli.py:121-133).  The result
// arrays of a gt_view are already in render order, so rendering is pure
// formatting: records are split into chunks at group boundaries, chunks are
// formatted on all host threads, and the digest streams over the chunks in
// order (SHA-NI when the CPU has it, FIPS 180-4 scalar otherwise).  This is
// at 10^7–10^8 output lines the Python render is the
// bottleneck of an end-to-end run, and digests make bit-exact comparison
// cheap at every scale.
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include <immintrin.h>

#include "../../include/gtadoc_b200.h"
#include "render.h"

namespace gt {

// ---------------------------------------------------------------------------
// SHA-256
// ---------------------------------------------------------------------------
namespace {

const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void blocks_scalar(uint32_t st[8], const uint8_t* p, size_t nblocks) {
  for (size_t b = 0; b < nblocks; b++, p += 64) {
    uint32_t w[64];
    for (int i = 0; i < 16; i++)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; i++) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = st[0], bb = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
    for (int i = 0; i < 64; i++) {
      const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
      const uint32_t ch = (e & f) ^ (~e & g);
      const uint32_t t1 = h + S1 + ch + K256[i] + w[i];
      const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
      const uint32_t mj = (a & bb) ^ (a & c) ^ (bb & c);
      const uint32_t t2 = S0 + mj;
      h = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = bb;
      bb = a;
      a = t1 + t2;
    }
    st[0] += a, st[1] += bb, st[2] += c, st[3] += d, st[4] += e, st[5] += f, st[6] += g, st[7] += h;
  }
}

// SHA-NI: 16 groups of 4 rounds; W_g = msg2(msg1(W_{g-4}, W_{g-3}) +
// alignr(W_{g-1}, W_{g-2}, 4), W_{g-1}) for g >= 4
__attribute__((target("sha,sse4.1,ssse3"))) void blocks_shani(uint32_t st[8], const uint8_t* p,
                                                                size_t nblocks) {
  const __m128i MASK = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
  __m128i tmp = _mm_loadu_si128((const __m128i*)&st[0]);
  __m128i s1 = _mm_loadu_si128((const __m128i*)&st[4]);
  tmp = _mm_shuffle_epi32(tmp, 0xB1);       // CDAB
  s1 = _mm_shuffle_epi32(s1, 0x1B);         // EFGH
  __m128i s0 = _mm_alignr_epi8(tmp, s1, 8);  // ABEF
  s1 = _mm_blend_epi16(s1, tmp, 0xF0);       // CDGH
  for (size_t b = 0; b < nblocks; b++, p += 64) {
    const __m128i abef = s0, cdgh = s1;
    __m128i W[4];
    for (int g = 0; g < 16; g++) {
      __m128i wg;
      if (g < 4) {
        wg = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i*)(p + 16 * g)), MASK);
      } else {
        const __m128i w4 = W[g & 3], w3 = W[(g + 1) & 3], w2 = W[(g + 2) & 3], w1 = W[(g + 3) & 3];
        wg = _mm_sha256msg1_epu32(w4, w3);
        wg = _mm_add_epi32(wg, _mm_alignr_epi8(w1, w2, 4));
        wg = _mm_sha256msg2_epu32(wg, w1);
      }
      W[g & 3] = wg;
      const __m128i k = _mm_set_epi32((int)K256[4 * g + 3], (int)K256[4 * g + 2], (int)K256[4 * g + 1],
                                      (int)K256[4 * g]);
      __m128i msg = _mm_add_epi32(wg, k);
      s1 = _mm_sha256rnds2_epu32(s1, s0, msg);
      msg = _mm_shuffle_epi32(msg, 0x0E);
      s0 = _mm_sha256rnds2_epu32(s0, s1, msg);
    }
    s0 = _mm_add_epi32(s0, abef);
    s1 = _mm_add_epi32(s1, cdgh);
  }
  tmp = _mm_shuffle_epi32(s0, 0x1B);     // FEBA
  s1 = _mm_shuffle_epi32(s1, 0xB1);      // DCHG
  s0 = _mm_blend_epi16(tmp, s1, 0xF0);   // DCBA
  s1 = _mm_alignr_epi8(s1, tmp, 8);      // ABEF -> HGFE
  _mm_storeu_si128((__m128i*)&st[0], s0);
  _mm_storeu_si128((__m128i*)&st[4], s1);
}

bool have_shani() {
  static const int v = __builtin_cpu_supports("sha") ? 1 : 0;
  return v && !getenv("GT_SHA_SCALAR");
}

}  // namespace

void Sha256::init() {
  static const uint32_t H0[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  memcpy(h, H0, sizeof h);
  nbuf = 0;
  total = 0;
}

void Sha256::blocks(const uint8_t* p, size_t n) {
  if (have_shani()) blocks_shani(h, p, n);
  else blocks_scalar(h, p, n);
}

void Sha256::update(const void* data, size_t len) {
  const uint8_t* p = (const uint8_t*)data;
  total += len;
  if (nbuf) {
    const size_t k = std::min(len, (size_t)64 - nbuf);
    memcpy(buf + nbuf, p, k);
    nbuf += k, p += k, len -= k;
    if (nbuf == 64) {
      blocks(buf, 1);
      nbuf = 0;
    }
  }
  if (len >= 64) {
    const size_t nb = len / 64;
    blocks(p, nb);
    p += nb * 64, len -= nb * 64;
  }
  if (len) {
    memcpy(buf, p, len);
    nbuf = len;
  }
}

void Sha256::final(uint8_t out[32]) {
  const uint64_t bits = total * 8;
  const uint8_t pad = 0x80;
  update(&pad, 1);
  const uint8_t zero[64] = {};
  update(zero, (nbuf <= 56) ? 56 - nbuf : 120 - nbuf);
  uint8_t lenb[8];
  for (int i = 0; i < 8; i++) lenb[i] = (uint8_t)(bits >> (56 - 8 * i));
  update(lenb, 8);
  for (int i = 0; i < 8; i++) {
    out[4 * i] = (uint8_t)(h[i] >> 24);
    out[4 * i + 1] = (uint8_t)(h[i] >> 16);
    out[4 * i + 2] = (uint8_t)(h[i] >> 8);
    out[4 * i + 3] = (uint8_t)h[i];
  }
}

// ---------------------------------------------------------------------------
// dictionary (grammar.py:193-228 layout; validation is gt_open's job)
// ---------------------------------------------------------------------------
bool Dict::parse(const uint8_t* d, size_t n, std::string* err) {
  auto rd32 = [&](size_t p) {
    uint32_t v;
    memcpy(&v, d + p, 4);
    return v;
  };
  if (n < 17 || memcmp(d, "GTDC", 4) != 0 || d[4] != 1) {
    *err = "not a GTDC version 1 blob";
    return false;
  }
  const uint32_t nw = rd32(5);
  size_t pos = 17;
  off.assign(1, 0);
  off.reserve((size_t)nw + 1);
  bytes.clear();
  for (uint32_t i = 0; i < nw; i++) {
    if (pos + 4 > n) {
      *err = "truncated dictionary";
      return false;
    }
    const uint32_t ln = rd32(pos);
    pos += 4;
    if (pos + ln > n) {
      *err = "truncated dictionary";
      return false;
    }
    bytes.insert(bytes.end(), d + pos, d + pos + ln);
    pos += ln;
    off.push_back((uint32_t)bytes.size());
  }
  return true;
}

// ---------------------------------------------------------------------------
// rendering (tasks.py:233-263)
// ---------------------------------------------------------------------------
namespace {

inline void put_u64(std::string& s, uint64_t v) {
  char b[24];
  int n = 0;
  do {
    b[n++] = (char)('0' + v % 10);
    v /= 10;
  } while (v);
  while (n) s.push_back(b[--n]);
}

struct Renderer {
  const Dict& dict;
  const gt_view& v;
  uint64_t wmask = 0;

  void word(std::string& s, uint64_t w) const {
    s.append(dict.bytes.data() + dict.off[w], dict.off[w + 1] - dict.off[w]);
  }
  // counts and group offsets arrive as u64, or narrowed to u32 (ABI 2)
  uint64_t cnt(uint64_t i) const { return v.count ? v.count[i] : (uint64_t)v.count32[i]; }
  uint64_t idv(uint64_t i) const {  // (ABI 3: ids may travel 1 / 2 bytes wide)
    if (v.id) return v.id[i];
    if (!v.id_narrow) return 0;
    return v.id_bytes == 1 ? (uint64_t) static_cast<const uint8_t*>(v.id_narrow)[i]
                           : (uint64_t) static_cast<const uint16_t*>(v.id_narrow)[i];
  }
  uint64_t goff(uint64_t g) const { return v.group_off ? v.group_off[g] : (uint64_t)v.group_off32[g]; }
  void gram_of_key(std::string& s, uint64_t key) const {
    const int l = v.seq_len;
    for (int j = 0; j < l; j++) {
      if (j) s.push_back(' ');
      word(s, (key >> ((l - 1 - j) * v.wbits)) & wmask);
    }
  }
  void gram_of_words(std::string& s, const uint32_t* g) const {
    for (int j = 0; j < v.seq_len; j++) {
      if (j) s.push_back(' ');
      word(s, g[j]);
    }
  }

  // units: records (ungrouped tasks) or groups; chunk [a, b) of units
  void chunk(std::string& s, uint64_t a, uint64_t b) const {
    switch (v.task) {
      case GT_WORDCOUNT:
      case GT_SORT:
        for (uint64_t i = a; i < b; i++) {
          word(s, idv(i));
          s.push_back('\t');
          put_u64(s, cnt(i));
          s.push_back('\n');
        }
        break;
      case GT_INVERTEDINDEX:
        for (uint64_t g = a; g < b; g++) {
          word(s, v.group_id[g]);
          for (uint64_t i = goff(g); i < goff(g + 1); i++) {
            s.push_back('\t');
            put_u64(s, idv(i));
          }
          s.push_back('\n');
        }
        break;
      case GT_TERMVECTOR:
        for (uint64_t f = a; f < b; f++)
          for (uint64_t i = goff(f); i < goff(f + 1); i++) {
            put_u64(s, f);
            s.push_back('\t');
            word(s, idv(i));
            s.push_back('\t');
            put_u64(s, cnt(i));
            s.push_back('\n');
          }
        break;
      case GT_SEQCOUNT:
        for (uint64_t f = a; f < b; f++)
          for (uint64_t i = goff(f); i < goff(f + 1); i++) {
            put_u64(s, f);
            s.push_back('\t');
            if (v.wbits) gram_of_key(s, v.key[i]);
            else gram_of_words(s, v.gram + i * (uint64_t)v.seq_len);
            s.push_back('\t');
            put_u64(s, cnt(i));
            s.push_back('\n');
          }
        break;
      case GT_RANKEDINVERTEDINDEX:
        for (uint64_t g = a; g < b; g++) {
          if (v.wbits) gram_of_key(s, v.group_key[g]);
          else gram_of_words(s, v.group_gram + g * (uint64_t)v.seq_len);
          for (uint64_t i = goff(g); i < goff(g + 1); i++) {
            s.push_back('\t');
            put_u64(s, idv(i));
            s.push_back(':');
            put_u64(s, cnt(i));
          }
          s.push_back('\n');
        }
        break;
      default:
        break;
    }
  }

  uint64_t units() const {
    return (v.task == GT_WORDCOUNT || v.task == GT_SORT) ? v.n : v.n_groups;
  }
  // records covered by units [0, u): for balancing chunks by output size
  uint64_t recs_before(uint64_t u) const {
    if (v.task == GT_WORDCOUNT || v.task == GT_SORT) return u;
    return (v.group_off || v.group_off32) ? goff(u) + u : u;
  }
};

// chunk boundaries balanced by records (+ groups)
std::vector<uint64_t> split_units(const Renderer& r, int parts) {
  const uint64_t U = r.units();
  std::vector<uint64_t> cut{0};
  const uint64_t total = r.recs_before(U);
  for (int k = 1; k < parts; k++) {
    const uint64_t target = total * (uint64_t)k / (uint64_t)parts;
    uint64_t lo = cut.back(), hi = U;
    while (lo < hi) {
      const uint64_t m = (lo + hi) / 2;
      if (r.recs_before(m) < target) lo = m + 1;
      else hi = m;
    }
    cut.push_back(lo);
  }
  cut.push_back(U);
  return cut;
}

int host_threads() {
  static int t = [] {
    int n = (int)std::thread::hardware_concurrency();
    if (const char* e = getenv("GT_RENDER_THREADS")) n = atoi(e);
    return std::max(1, std::min(n, 64));
  }();
  return t;
}

template <class Sink>
void render_all(const Dict& dict, const gt_view& v, Sink sink) {
  Renderer r{dict, v};
  r.wmask = v.wbits ? ((1ull << v.wbits) - 1) : 0;
  const uint64_t U = r.units();
  if (!U) return;
  const int T = host_threads();
  // rounds of T chunks of ~8 MB of output each: bounded memory, ordered sink
  const uint64_t recs = r.recs_before(U);
  const int parts = (int)std::max<uint64_t>(1, std::min<uint64_t>(recs / 200000 + 1, 1u << 16));
  std::vector<uint64_t> cut = split_units(r, parts);
  std::vector<std::string> buf(T);
  for (int base = 0; base < parts; base += T) {
    const int m = std::min(T, parts - base);
    std::vector<std::thread> th;
    for (int k = 1; k < m; k++)
      th.emplace_back([&, k] {
        buf[k].clear();
        r.chunk(buf[k], cut[base + k], cut[base + k + 1]);
      });
    buf[0].clear();
    r.chunk(buf[0], cut[base], cut[base + 1]);
    for (auto& t : th) t.join();
    for (int k = 0; k < m; k++) sink(buf[k]);
  }
}

}  // namespace

std::string render_text(const Dict& d, const gt_view& v) {
  std::string out;
  render_all(d, v, [&](const std::string& s) { out += s; });
  return out;
}

uint64_t render_digest(const Dict& d, const gt_view& v, uint8_t out[32]) {
  Sha256 h;
  h.init();
  uint64_t n = 0;
  render_all(d, v, [&](const std::string& s) {
    h.update(s.data(), s.size());
    n += s.size();
  });
  h.final(out);
  return n;
}

}  // namespace gt

// ---------------------------------------------------------------------------
// C-ABI (host only: usable without a GPU)
// ---------------------------------------------------------------------------
struct gt_dict {
  gt::Dict d;
};

static thread_local std::string t_render_err;

extern "C" {

int gt_dict_open(const uint8_t* gtdc, size_t n, gt_dict** out) {
  *out = nullptr;
  gt_dict* d = new gt_dict();
  if (!d->d.parse(gtdc, n, &t_render_err)) {
    delete d;
    return GT_E_FORMAT;
  }
  *out = d;
  return GT_OK;
}

void gt_dict_close(gt_dict* d) { delete d; }

int gt_render_view(const gt_dict* d, const gt_view* v, char** text, uint64_t* len) {
  std::string s = gt::render_text(d->d, *v);
  char* p = (char*)malloc(s.size() + 1);
  if (!p) return GT_E_RESOURCE;
  memcpy(p, s.data(), s.size());
  p[s.size()] = 0;
  *text = p;
  *len = s.size();
  return GT_OK;
}

void gt_free_text(char* text) { free(text); }

int gt_digest_view(const gt_dict* d, const gt_view* v, uint8_t sha256[32], uint64_t* len) {
  *len = gt::render_digest(d->d, *v, sha256);
  return GT_OK;
}

int gt_sha256(const void* data, uint64_t n, uint8_t out[32]) {
  gt::Sha256 h;
  h.init();
  h.update(data, n);
  h.final(out);
  return GT_OK;
}

}  // extern "C"
