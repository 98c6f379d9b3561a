// CPU check of the drop-in API's double -> int8 block conversion
// (csrc/vd_host_convert.h): the SSE2 body and the scalar tail agree with the
// per-value rule (an integer in [-127, 127] converts exactly; anything else —
// fractions, +-128 and beyond, infinities, NaN — marks the block as not int8)
// at every offset and length, including a single offending value placed in
// the vector body or in the tail.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <limits>
#include <random>
#include <vector>

#include "vd_host_convert.h"

using vitdec::host::int8_one;
using vitdec::host::int8_range;

int main() {
  std::mt19937_64 rng(2026);
  const double specials[] = {128.0, -128.0, 127.5, -0.5, 1e300, -3e10, std::numeric_limits<double>::infinity(),
                             -std::numeric_limits<double>::infinity(), std::numeric_limits<double>::quiet_NaN(),
                             0.25, 126.999999, -127.000001};
  long fails = 0, cases = 0;
  for (int t = 0; t < 40000; ++t) {
    const int n = 1 + static_cast<int>(rng() % 80);
    const int lo = static_cast<int>(rng() % 3);
    std::vector<double> d(n + lo);
    for (auto& v : d) v = static_cast<double>(static_cast<int>(rng() % 255) - 127);
    if (t % 7 == 0) d[rng() % d.size()] = -0.0;
    const int nbad = t % 3 == 0 ? 0 : 1 + static_cast<int>(rng() % 2);
    for (int j = 0; j < nbad; ++j) d[lo + rng() % n] = specials[rng() % (sizeof(specials) / sizeof(double))];
    std::vector<std::int8_t> want(d.size()), got(d.size());
    int bad_want = 0;
    for (int i = lo; i < lo + n; ++i) bad_want |= int8_one(d[i], &want[i]);
    const int bad_got = int8_range(d.data(), got.data(), lo, lo + n);
    ++cases;
    if ((bad_want != 0) != (bad_got != 0)) {
      ++fails;
      continue;
    }
    // the rule itself: exact integers in range <=> not bad
    bool exp_bad = false;
    for (int i = lo; i < lo + n; ++i) {
      const double v = d[i];
      if (!(v >= -127.0 && v <= 127.0 && std::trunc(v) == v)) exp_bad = true;
    }
    if (exp_bad != (bad_got != 0)) ++fails;
    if (!exp_bad)
      for (int i = lo; i < lo + n; ++i)
        if (got[i] != static_cast<std::int8_t>(d[i]) || want[i] != got[i]) {
          ++fails;
          break;
        }
  }
  std::printf("%s: %ld of %ld cases failed\n", fails ? "FAIL" : "OK", fails, cases);
  return fails ? 1 : 0;
}
