// Open-addressing u64 -> u32 map used by the native CSR builder and the
// generators' duplicate filters.  Linear probing, power-of-two capacity,
// grows at 50% load; keys are arbitrary u64 (an occupancy bitmap marks used
// cells, so 0 and ~0 are ordinary keys).
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

namespace wbc::detail {

class U64Map {
 public:
  explicit U64Map(std::uint64_t expect = 0) { rehash(cap_for(expect)); }

  // Returns {value slot, inserted}.  A fresh slot holds `fresh`.
  std::pair<std::uint32_t*, bool> try_emplace(std::uint64_t key, std::uint32_t fresh) {
    if (2 * (size_ + 1) > cap_) rehash(cap_ * 2);
    std::uint64_t i = mix(key) & mask_;
    for (;;) {
      if (!used(i)) {
        set_used(i);
        keys_[i] = key;
        vals_[i] = fresh;
        ++size_;
        return {&vals_[i], true};
      }
      if (keys_[i] == key) return {&vals_[i], false};
      i = (i + 1) & mask_;
    }
  }

  bool insert(std::uint64_t key) { return try_emplace(key, 0).second; }
  std::uint64_t size() const { return size_; }

 private:
  static std::uint64_t cap_for(std::uint64_t expect) {
    std::uint64_t c = 64;
    while (c < 2 * expect + 2) c <<= 1;
    return c;
  }
  static std::uint64_t mix(std::uint64_t x) {
    x ^= x >> 31;
    x *= 0x7fb5d329728ea185ULL;
    x ^= x >> 27;
    x *= 0x81dadef4bc2dd44dULL;
    return x ^ (x >> 33);
  }
  bool used(std::uint64_t i) const { return (bits_[i >> 6] >> (i & 63)) & 1; }
  void set_used(std::uint64_t i) { bits_[i >> 6] |= 1ULL << (i & 63); }

  void rehash(std::uint64_t cap) {
    std::vector<std::uint64_t> ok = std::move(keys_);
    std::vector<std::uint32_t> ov = std::move(vals_);
    std::vector<std::uint64_t> ob = std::move(bits_);
    const std::uint64_t old_cap = cap_;
    cap_ = cap;
    mask_ = cap - 1;
    keys_.assign(cap, 0);
    vals_.assign(cap, 0);
    bits_.assign((cap + 63) / 64, 0);
    size_ = 0;
    for (std::uint64_t i = 0; i < old_cap; ++i) {
      if (!((ob[i >> 6] >> (i & 63)) & 1)) continue;
      std::uint64_t j = mix(ok[i]) & mask_;
      while (used(j)) j = (j + 1) & mask_;
      set_used(j);
      keys_[j] = ok[i];
      vals_[j] = ov[i];
      ++size_;
    }
  }

  std::vector<std::uint64_t> keys_;
  std::vector<std::uint32_t> vals_;
  std::vector<std::uint64_t> bits_;
  std::uint64_t cap_ = 0, mask_ = 0, size_ = 0;
};

}  // namespace wbc::detail
