// 128-bit structural fingerprints for the host-side memo tables (plans,
// segment plans, generated kernels): two independent 64-bit multiply-rotate
// streams over the key bytes.  Keys are hashed instead of stored, so a lookup
// costs one pass over the structural fields and no allocation; at 128 bits a
// collision between the (thousands of) entries of a process is not a concern.
#pragma once
#include <cstdint>
#include <cstring>
#include <functional>

namespace svgb {

struct Key128 {
  uint64_t a = 0, b = 0;
  bool operator==(const Key128& o) const { return a == o.a && b == o.b; }
};
struct Key128Hash {
  size_t operator()(const Key128& k) const { return static_cast<size_t>(k.a ^ (k.b * 0x9e3779b97f4a7c15ull)); }
};

class Hasher {
 public:
  void word(uint64_t w) {
    a_ = rotl(a_ ^ (w * 0x87c37b91114253d5ull), 31) * 0x4cf5ad432745937full;
    b_ = rotl(b_ ^ (w * 0x52dce729da3ed7c5ull), 29) * 0x9e3779b97f4a7c15ull + 0x38495ab5ull;
    ++n_;
  }
  void bytes(const void* p, size_t len) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    while (len >= 8) {
      uint64_t w;
      std::memcpy(&w, c, 8);
      word(w);
      c += 8;
      len -= 8;
    }
    if (len) {
      uint64_t w = 0;
      std::memcpy(&w, c, len);
      word(w ^ (uint64_t(len) << 56));
    }
  }
  template <class T>
  void pod(const T& v) {
    bytes(&v, sizeof(T));
  }
  Key128 key() const {
    Key128 k;
    k.a = fmix(a_ ^ n_);
    k.b = fmix(b_ + 0x2545f4914f6cdd1dull * n_);
    return k;
  }

 private:
  static uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
  static uint64_t fmix(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
  }
  uint64_t a_ = 0x243f6a8885a308d3ull, b_ = 0x13198a2e03707344ull, n_ = 0;
};

}  // namespace svgb
