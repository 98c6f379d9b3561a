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
