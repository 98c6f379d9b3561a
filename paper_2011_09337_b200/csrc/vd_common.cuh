// Shared host/device helpers: frame geometry and the random-start salt.
//
// Frame geometry restates reference decoder.cpp:170-191 (decode_frame's
// window, subframe split and traceback start stages); mix_seed restates
// reference channel.cpp:85-90 bit-exactly so random-start tracebacks pick the
// same states on the GPU as on the CPU.
#pragma once

#include "vd_std.h"

#ifdef __CUDACC__
#define VD_HD __host__ __device__ __forceinline__
#else
#define VD_HD inline
#endif

namespace vd {

VD_HD std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t salt) {
  std::uint64_t z = seed + 0x9e3779b97f4a7c15ull * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

VD_HD std::int64_t imin(std::int64_t a, std::int64_t b) { return a < b ? a : b; }
VD_HD std::int64_t imax(std::int64_t a, std::int64_t b) { return a > b ? a : b; }

/// Geometry of frame m (reference decoder.cpp:175-183).
struct FrameGeom {
  std::int64_t out_lo, out_hi;  // output stages [out_lo, out_hi)
  std::int64_t beg, end;        // processed stages [beg, end)
  std::int64_t step, num_sub;   // subframe length and count

  VD_HD FrameGeom(std::int64_t m, std::int64_t n, int f, int v1, int v2, int f0) {
    out_lo = m * f;
    out_hi = imin(out_lo + f, n);
    beg = imax(out_lo - v1, 0);
    end = imin(out_hi + v2, n);
    step = f0 > 0 ? f0 : (out_hi - out_lo);
    num_sub = (out_hi - out_lo + step - 1) / step;
  }
  VD_HD std::int64_t len() const { return end - beg; }
  /// Local traceback start stage of subframe s (reference decoder.cpp:187-191).
  VD_HD std::int64_t start_stage(std::int64_t s, int v2) const {
    const std::int64_t sub_hi = imin(out_lo + (s + 1) * step, out_hi);
    return imin(sub_hi + v2, end) - 1 - beg;
  }
  VD_HD std::int64_t sub_lo(std::int64_t s) const { return out_lo + s * step; }
  VD_HD std::int64_t sub_hi(std::int64_t s) const { return imin(out_lo + (s + 1) * step, out_hi); }
};

}  // namespace vd
