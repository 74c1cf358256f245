// Thread helpers for the host-side graph builders (generators, CSR build).
// Parallel paths produce output identical to the serial ones (the reference's
// streams and orders); they engage above a size threshold.
//   WBC_HOST_THREADS       worker threads (default: hardware threads, <= 64)
//   WBC_HOST_PARALLEL_MIN  smallest input (entries) that takes a parallel
//                          path (default 2^21; tests set it low to exercise
//                          the parallel code on small graphs)
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <thread>
#include <vector>

namespace wbc::detail {

inline unsigned host_threads() {
  if (const char* e = std::getenv("WBC_HOST_THREADS")) {
    const long v = std::strtol(e, nullptr, 10);
    if (v >= 1) return static_cast<unsigned>(std::min<long>(v, 64));
  }
  return std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
}

inline std::uint64_t parallel_min_entries() {
  if (const char* e = std::getenv("WBC_HOST_PARALLEL_MIN")) return std::strtoull(e, nullptr, 10);
  return 1ULL << 21;
}

// f(t, begin, end) on T contiguous chunks of [0, n), one thread each.
template <class F>
void parallel_chunks(std::uint64_t n, unsigned T, F&& f) {
  if (T <= 1 || n < 2) {
    f(0u, std::uint64_t{0}, n);
    return;
  }
  std::vector<std::thread> ts;
  ts.reserve(T);
  for (unsigned t = 0; t < T; ++t) {
    const std::uint64_t b = n * t / T, e = n * (t + 1) / T;
    ts.emplace_back([&f, t, b, e] { f(t, b, e); });
  }
  for (auto& th : ts) th.join();
}

inline std::uint64_t mix64(std::uint64_t x) {
  x ^= x >> 31;
  x *= 0x7fb5d329728ea185ULL;
  x ^= x >> 27;
  x *= 0x81dadef4bc2dd44dULL;
  return x ^ (x >> 33);
}

}  // namespace wbc::detail
