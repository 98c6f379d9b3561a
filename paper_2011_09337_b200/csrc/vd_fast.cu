// Fast-kernel dispatch (the kernels and their planning: vd_fast.cuh; the
// per-code instantiations: vd_fast_k*.cu) and the zero-padded block-head
// gather used by the batched decode.
#include "vd_fast.cuh"

namespace vd {
namespace fast {

// vd_fast_k*.cu: try the codes of one group; probe == true only plans.
bool try_group_k7(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe);
bool try_group_k9(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe);
bool try_group_k568(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe);
bool try_punct_k7(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err, std::int64_t* mi0,
                  std::int64_t* mi1);

__global__ void head_gather_kernel(const std::int8_t* __restrict__ llr, const std::int64_t* __restrict__ blk_stage,
                                   int nblocks, int b, int v1, std::int64_t pitch, std::int64_t copy,
                                   std::int8_t* __restrict__ head) {
  const std::int64_t pb = pitch * b, total = pb * nblocks;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t j = i / pb, o = i - j * pb - static_cast<std::int64_t>(v1) * b;
    std::int8_t v = 0;
    if (o >= 0) {
      const std::int64_t s0 = __ldg(blk_stage + j), nj = __ldg(blk_stage + j + 1) - s0;
      if (o < (copy < nj ? copy : nj) * b) v = llr[s0 * b + o];
    }
    head[i] = v;
  }
}

}  // namespace fast

cudaError_t launch_head_gather(const std::int8_t* llr, const std::int64_t* blk_stage, int nblocks, int b, int v1,
                               std::int64_t pitch, std::int64_t copy, std::int8_t* head, cudaStream_t stream) {
  const std::int64_t total = pitch * b * nblocks;
  const std::int64_t cap = static_cast<std::int64_t>(sm_count()) * 8;
  const std::int64_t grid = std::min<std::int64_t>((total + 255) / 256, cap);
  if (grid <= 0) return cudaSuccess;
  fast::head_gather_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(llr, blk_stage, nblocks, b, v1, pitch,
                                                                            copy, head);
  note_launch();
  return cudaGetLastError();
}

bool fast_path_supported(const DecodeLaunch& p) {
  using namespace fast;
  if (p.b != 2 && p.b != 3) return false;
  cudaError_t unused = cudaSuccess;
  return try_group_k7(p, nullptr, &unused, true) || try_group_k9(p, nullptr, &unused, true) ||
         try_group_k568(p, nullptr, &unused, true);
}

bool launch_fast_punct_i8(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err,
                          std::int64_t* mi0, std::int64_t* mi1) {
  return fast::try_punct_k7(p, pattern, stream, err, mi0, mi1);
}

cudaError_t launch_fast_i8(const DecodeLaunch& p, cudaStream_t stream) {
  using namespace fast;
  cudaError_t err = cudaErrorNotSupported;
  if (try_group_k7(p, stream, &err, false)) return err;
  if (try_group_k9(p, stream, &err, false)) return err;
  if (try_group_k568(p, stream, &err, false)) return err;
  return cudaErrorNotSupported;
}

}  // namespace vd
