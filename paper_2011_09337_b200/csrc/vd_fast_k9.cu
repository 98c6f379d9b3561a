// Fast-kernel instantiations: K9a, K9b, K9c (see vd_fast.cuh).
#include "vd_fast.cuh"

namespace vd {
namespace fast {

bool try_group_k9(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe) {
  Plan pl;
  if (K9a::matches(p.k, p.b, p.polys)) return probe ? plan<K9a, 16>(p, &pl) : try_variant<K9a, 16>(p, stream, err);
  if (K9b::matches(p.k, p.b, p.polys)) return probe ? plan<K9b, 16>(p, &pl) : try_variant<K9b, 16>(p, stream, err);
  if (K9c::matches(p.k, p.b, p.polys)) return probe ? plan<K9c, 16>(p, &pl) : try_variant<K9c, 16>(p, stream, err);
  return false;
}

}  // namespace fast
}  // namespace vd
