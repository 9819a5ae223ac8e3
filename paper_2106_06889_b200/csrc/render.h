// render.h — native render + SHA-256 (render.cpp), host only.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gtadoc_b200.h"

namespace gt {

struct Sha256 {
  uint32_t h[8];
  uint8_t buf[64];
  size_t nbuf;
  uint64_t total;
  void init();
  void update(const void* data, size_t len);
  void final(uint8_t out[32]);

 private:
  void blocks(const uint8_t* p, size_t nblocks);
};

// word strings of a GTDC dictionary: word i = bytes[off[i], off[i+1])
struct Dict {
  std::vector<char> bytes;
  std::vector<uint32_t> off;
  bool parse(const uint8_t* gtdc, size_t n, std::string* err);
};

std::string render_text(const Dict& d, const gt_view& v);
uint64_t render_digest(const Dict& d, const gt_view& v, uint8_t out[32]);

}  // namespace gt
