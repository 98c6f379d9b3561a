// Fast-kernel instantiations: K7a, K7b, K7c (see vd_fast.cuh).
#include "vd_fast.cuh"

namespace vd {
namespace fast {

bool try_group_k7(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe) {
  Plan pl;
  if (K7a::matches(p.k, p.b, p.polys)) return probe ? plan<K7a, 16>(p, &pl) : try_variant<K7a, 16>(p, stream, err);
  if (K7b::matches(p.k, p.b, p.polys)) return probe ? plan<K7b, 16>(p, &pl) : try_variant<K7b, 16>(p, stream, err);
  if (K7c::matches(p.k, p.b, p.polys)) return probe ? plan<K7c, 16>(p, &pl) : try_variant<K7c, 16>(p, stream, err);
  return false;
}

}  // namespace fast
}  // namespace vd

namespace vd {
namespace fast {

// Fused-depuncture instantiations (K = 7 (171,133) mother code, rates 2/3, 3/4).
bool try_punct_k7(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err, std::int64_t* mi0,
                  std::int64_t* mi1) {
  if (pattern == 23) return try_punct_variant<K7a, 16, PunctR23>(p, stream, err, mi0, mi1);
  if (pattern == 34) return try_punct_variant<K7a, 16, PunctR34>(p, stream, err, mi0, mi1);
  return false;
}

}  // namespace fast
}  // namespace vd
