// Fast-kernel instantiations: K5a, K6a, K8a (see vd_fast.cuh).
#include "vd_fast.cuh"

namespace vd {
namespace fast {

bool try_group_k568(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe) {
  Plan pl;
  if (K5a::matches(p.k, p.b, p.polys)) return probe ? plan<K5a, 16>(p, &pl) : try_variant<K5a, 16>(p, stream, err);
  if (K6a::matches(p.k, p.b, p.polys)) return probe ? plan<K6a, 16>(p, &pl) : try_variant<K6a, 16>(p, stream, err);
  if (K8a::matches(p.k, p.b, p.polys)) return probe ? plan<K8a, 16>(p, &pl) : try_variant<K8a, 16>(p, stream, err);
  return false;
}

}  // namespace fast
}  // namespace vd
