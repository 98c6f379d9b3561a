// End-to-end throughput of the reference-facing C++ drop-in call,
// vitdec::framed_decode(const LlrBlock&, const Trellis&, const FrameConfig&,
// int workers) (reference decoder.hpp:74-79): a B x N block of doubles in,
// std::vector<uint8_t> bits out, everything in between (the integer-valued
// check and double -> int8 conversion, pageable-to-pinned staging, H2D, the
// decode, D2H, the byte unpack) inside the timed call. Built by
// `make -C paper_2011_09337_b200` next to the library; bench.py reports it
// as e2e_reference_api.
//
//   bench_dropin [n_stages = 2^26] [reps = 3] [workers = hardware threads]
//
// Workload: K=7 (171,133) r1/2, f=256 v1=20 v2=20, int8-valued LLRs
// q = clamp(rint(32 y), -127, 127) of BPSK + AWGN at 3 dB over a random
// message (the C5 workload's statistics; a stand-alone generator, since the
// reference's channel.cpp is a test harness, not part of this library).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>

#include "vitdec/decoder.hpp"
#include "vitdec/trellis.hpp"

int main(int argc, char** argv) {
  using namespace vitdec;
  const Eigen::Index n = argc > 1 ? std::atoll(argv[1]) : (Eigen::Index{1} << 26);
  const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
  const int workers = argc > 3 ? std::atoi(argv[3]) : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const Trellis t = build_trellis(CodeSpec::from_octal(7, "171,133"));
  LlrBlock llr(2, n);
  {
    // encoder state machine of (171, 133) + BPSK + AWGN, quantised
    std::mt19937_64 rng(20261017);
    std::normal_distribution<double> noise(0.0, std::sqrt(1.0 / (2.0 * 0.5 * std::pow(10.0, 0.3))));
    std::uint32_t state = 0;
    for (Eigen::Index i = 0; i < n; ++i) {
      const std::uint32_t u = static_cast<std::uint32_t>(rng() & 1u);
      const std::uint32_t reg = (u << 6) | state;
      for (int b = 0; b < 2; ++b) {
        const std::uint32_t poly = b == 0 ? 0171u : 0133u;
        const int bit = __builtin_popcount(reg & poly) & 1;
        const double y = (bit ? -1.0 : 1.0) + noise(rng);
        llr.data()[2 * i + b] = std::clamp(std::nearbyint(32.0 * y), -127.0, 127.0);
      }
      state = reg >> 1;
    }
  }
  FrameConfig cfg;
  cfg.f = 256;
  cfg.v1 = 20;
  cfg.v2 = 20;
  DecodeOutput out = framed_decode(llr, t, cfg, workers);  // warm-up (device context, pools, JIT-free)
  std::vector<double> secs;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    out = framed_decode(llr, t, cfg, workers);
    const auto t1 = std::chrono::steady_clock::now();
    secs.push_back(std::chrono::duration<double>(t1 - t0).count());
  }
  std::sort(secs.begin(), secs.end());
  const double med = secs[secs.size() / 2];
  // breakdown: a fresh BitVec of n bytes (what the API returns), and the
  // native int8 overload on a pre-converted pageable block (decode + staging)
  auto timed = [&](auto&& fn) {
    std::vector<double> v;
    for (int r = 0; r < reps; ++r) {
      const auto a = std::chrono::steady_clock::now();
      fn();
      v.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
    }
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  std::vector<std::int8_t> q8(static_cast<std::size_t>(2 * n));
  for (Eigen::Index i = 0; i < 2 * n; ++i) q8[i] = static_cast<std::int8_t>(llr.data()[i]);
  std::vector<std::uint32_t> packed(static_cast<std::size_t>((n + 31) / 32));
  const double t_native = timed([&] { framed_decode(q8.data(), n, t, cfg, packed.data()); });
  const double t_bitvec = timed([&] {
    BitVec b(static_cast<std::size_t>(n));
    if (b[n / 2] == 7) std::printf("?");
  });
  std::printf("{\"value\": %.4f, \"unit\": \"Gbps\", \"info_bits\": %lld, \"workers\": %d, \"reps\": %d, "
              "\"median_s\": %.6f, \"frames\": %lld, \"h2d_bytes_per_call\": %lld, \"d2h_bytes_per_call\": %lld, "
              "\"breakdown_s\": {\"native_int8_pageable_call\": %.6f, \"fresh_bitvec_alloc\": %.6f}}\n",
              static_cast<double>(n) / med / 1e9, static_cast<long long>(n), workers, reps, med,
              static_cast<long long>(out.stats.frames), static_cast<long long>(2 * n),
              static_cast<long long>((n + 31) / 32 * 4), t_native, t_bitvec);
  return 0;
}
