// Host memcpy bandwidth vs thread count (pageable source -> destination), the
// staging step of decode_host for pageable caller buffers.
//   g++ -O2 -pthread tools/memcpy_probe.cpp -o /tmp/memcpy_probe && /tmp/memcpy_probe
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

int main() {
  const std::size_t bytes = std::size_t{32} << 20;  // one 2^24-stage r1/2 chunk
  std::vector<char> src(std::size_t{1} << 30, 1), dst(bytes * 2, 0);
  std::printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
  for (int nt : {1, 2, 4, 8, 12, 16, 24, 32}) {
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
      const char* s = src.data() + (static_cast<std::size_t>(rep) * bytes) % (src.size() - bytes);
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      const std::size_t part = (bytes + nt - 1) / nt;
      for (int i = 0; i < nt; ++i)
        th.emplace_back([&, i] { std::memcpy(dst.data() + i * part, s + i * part, std::min(part, bytes - i * part)); });
      for (auto& t : th) t.join();
      const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      best = std::max(best, bytes / sec / 1e9);
    }
    std::printf("threads %2d: %.1f GB/s\n", nt, best);
  }
}
