// Drop-in for reference proj/include/vitdec/parallel.hpp:11-29 (used by the
// reference's BER harness, berlab.cpp). The decoder itself no longer uses it:
// frames are spread over the GPU grid instead of std::threads.
#pragma once

#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

namespace vitdec {

/// fn(first, last) over contiguous chunks of [0, n), one std::thread per
/// chunk (at most `workers`), joined before returning.
template <typename Fn>
void parallel_for_chunks(std::int64_t n, int workers, Fn&& fn) {
  if (n <= 0) return;
  const std::int64_t w = std::min<std::int64_t>(std::max(workers, 1), n);
  if (w == 1) {
    fn(std::int64_t{0}, n);
    return;
  }
  const std::int64_t per = (n + w - 1) / w;
  std::vector<std::thread> pool;
  pool.reserve(static_cast<std::size_t>(w));
  for (std::int64_t lo = 0; lo < n; lo += per) {
    const std::int64_t hi = std::min(lo + per, n);
    pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (std::thread& t : pool) t.join();
}

}  // namespace vitdec
