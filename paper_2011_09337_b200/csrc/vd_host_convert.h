// Host-side conversion of the drop-in API's double LLR blocks to int8 (header
// so that tests/cpp/host_convert_check.cpp exercises the same code on CPU).
#pragma once

#include <cmath>
#include <cstdint>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace vitdec {
namespace host {

// One value: clamp (NaN -> -127), truncate; v is an integer in [-127, 127]
// iff the truncated value equals it.
inline int int8_one(double v, std::int8_t* out) {
  const int iv = static_cast<int>(std::fmin(std::fmax(v, -127.0), 127.0));
  *out = static_cast<std::int8_t>(iv);
  return static_cast<double>(iv) != v;
}

// Range [lo, hi) of int8_exact; nonzero if a value is not an int8 integer.
// SSE2 (every x86-64): 16 doubles per iteration, clamp by MINPD / MAXPD (a
// NaN clamps to 127 and then fails the equality test), CVTTPD2DQ, the
// round-trip compare, and saturating packs (exact: the values are already in
// [-127, 127]). The scalar libm fmin / fmax loop ran at ~6 ns per value.
inline int int8_range(const double* d, std::int8_t* out, std::int64_t lo, std::int64_t hi) {
  int bad = 0;
  std::int64_t i = lo;
#if defined(__SSE2__)
  const __m128d cmin = _mm_set1_pd(-127.0), cmax = _mm_set1_pd(127.0);
  __m128d badv = _mm_setzero_pd();
  for (; i + 16 <= hi; i += 16) {
    __m128i w[4];
    for (int k = 0; k < 4; ++k) {
      const __m128d v0 = _mm_loadu_pd(d + i + 4 * k), v1 = _mm_loadu_pd(d + i + 4 * k + 2);
      const __m128i i0 = _mm_cvttpd_epi32(_mm_max_pd(_mm_min_pd(v0, cmax), cmin));
      const __m128i i1 = _mm_cvttpd_epi32(_mm_max_pd(_mm_min_pd(v1, cmax), cmin));
      badv = _mm_or_pd(badv, _mm_cmpneq_pd(_mm_cvtepi32_pd(i0), v0));
      badv = _mm_or_pd(badv, _mm_cmpneq_pd(_mm_cvtepi32_pd(i1), v1));
      w[k] = _mm_unpacklo_epi64(i0, i1);
    }
    const __m128i b = _mm_packs_epi16(_mm_packs_epi32(w[0], w[1]), _mm_packs_epi32(w[2], w[3]));
    _mm_storeu_si128(reinterpret_cast<__m128i*>(out + i), b);
  }
  bad |= _mm_movemask_pd(badv);
#endif
  for (; i < hi; ++i) bad |= int8_one(d[i], out + i);
  return bad;
}

}  // namespace host
}  // namespace vitdec
