// Drop-in C++ API check (built by `make -C oracle dropin`, run by
// tests/test_dropin_gpu.py on a B200): a multi-million-stage LlrBlock through
// vitdec::framed_decode with workers = 1 and workers = 8 (host threads for the
// block conversion / bit unpacking) gives identical bits and stats, equal to
// the native int8 entry point; a real-valued block takes the FP64 kernel.
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "vitdec/decoder.hpp"
#include "vitdec/trellis.hpp"

int main() {
  using namespace vitdec;
  const Trellis t = build_trellis(CodeSpec::from_octal(7, "171,133"));
  const Eigen::Index n = 3 << 20;
  LlrBlock llr(2, n);
  std::mt19937_64 rng(7);
  std::uniform_int_distribution<int> dist(-60, 60);
  std::vector<std::int8_t> q(static_cast<std::size_t>(2 * n));
  for (Eigen::Index i = 0; i < 2 * n; ++i) {
    q[i] = static_cast<std::int8_t>(dist(rng));
    llr.data()[i] = q[i];
  }
  FrameConfig cfg;
  cfg.f = 256;
  cfg.v1 = 20;
  cfg.v2 = 20;
  const DecodeOutput a = framed_decode(llr, t, cfg, 1);
  const DecodeOutput b = framed_decode(llr, t, cfg, 8);
  std::vector<std::uint32_t> packed(static_cast<std::size_t>((n + 31) / 32));
  const DecodeStats st = framed_decode(q.data(), n, t, cfg, packed.data());
  int bad = 0;
  for (Eigen::Index i = 0; i < n; ++i) {
    const std::uint8_t c = (packed[i >> 5] >> (i & 31)) & 1u;
    bad += a.bits[i] != b.bits[i] || a.bits[i] != c;
  }
  bad += a.stats.frames != b.stats.frames || a.stats.stages != b.stats.stages || a.stats.frames != st.frames;
  // real-valued block (FP64 kernel) on a short prefix: workers-invariant too
  LlrBlock r = llr.leftCols(4096) * 0.37;
  const DecodeOutput ra = framed_decode(r, t, cfg, 1), rb = framed_decode(r, t, cfg, 8);
  bad += ra.bits != rb.bits;
  std::printf("%s: %d mismatches\n", bad ? "FAIL" : "OK", bad);
  return bad ? 1 : 0;
}
