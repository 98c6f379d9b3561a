// Fast-kernel dispatch (the kernels and their planning: vd_fast.cuh; the
// per-code instantiations: vd_fast_k*.cu; other codes: run-time
// instantiations, vd_jit.cu) and the zero-padded block-head gather used by
// the batched decode.
#include "vd_fast.cuh"

namespace vd {
namespace fast {

// vd_fast_k*.cu: try the codes of one group; probe == true only plans.
bool try_group_k7(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe);
bool try_group_k9(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe);
bool try_group_k568(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe);
bool try_punct_k7(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err, std::int64_t* mi0,
                  std::int64_t* mi1);
// vd_small.cu: 8-states-per-lane kernel for latency-bound small launches
bool small_launch_wanted(const DecodeLaunch& p);
bool try_small(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err);
bool small_writes_whole_words(const DecodeLaunch& p);

// ---- run-time instantiations (vd_jit.cu) for other complement-paired codes --
// plan() uses only K and B of its code, so one placeholder code per (K, B)
// class plans every code of the class; the kernel comes from the JIT.
template <int K, int B>
using PlanCode = CodeB<K, B, (1u << (K - 1)) | 1u, (1u << (K - 1)) | 1u, B >= 3 ? ((1u << (K - 1)) | 1u) : 0u,
                       B >= 4 ? ((1u << (K - 1)) | 1u) : 0u>;

struct JitSel {
  const DecodeLaunch* p;
  const void* operator()(bool tm, bool gl, cudaError_t* e) const {
    return jit::fast_kernel(p->k, p->b, p->polys, tm, gl, e);
  }
};

template <int K, int B>
bool try_jit_kb(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe) {
  Plan pl;
  if (!plan<PlanCode<K, B>, 16>(p, &pl)) return false;
  if (!probe) *err = launch_variant<PlanCode<K, B>, 16>(p, stream, JitSel{&p});
  return true;
}

// The fast kernel's envelope: 5 <= K <= 10 (16 states per lane, at most 32
// lanes per frame pair; int16 metric range), B in {2, 3, 4}; any polynomials (complement-paired or
// not: a butterfly's four edge labels are x, x ^ cb(0), x ^ cb(K-1) and
// x ^ cb(0) ^ cb(K-1), all compile-time).
bool jit_code(const DecodeLaunch& p) { return jit::enabled() && fast_envelope_code(p.k, p.b, p.polys); }

bool try_jit(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe) {
  if (!jit_code(p)) return false;
  switch (p.k * 10 + p.b) {
    case 52: return try_jit_kb<5, 2>(p, stream, err, probe);
    case 53: return try_jit_kb<5, 3>(p, stream, err, probe);
    case 62: return try_jit_kb<6, 2>(p, stream, err, probe);
    case 63: return try_jit_kb<6, 3>(p, stream, err, probe);
    case 72: return try_jit_kb<7, 2>(p, stream, err, probe);
    case 73: return try_jit_kb<7, 3>(p, stream, err, probe);
    case 82: return try_jit_kb<8, 2>(p, stream, err, probe);
    case 83: return try_jit_kb<8, 3>(p, stream, err, probe);
    case 92: return try_jit_kb<9, 2>(p, stream, err, probe);
    case 93: return try_jit_kb<9, 3>(p, stream, err, probe);
    case 102: return try_jit_kb<10, 2>(p, stream, err, probe);
    case 103: return try_jit_kb<10, 3>(p, stream, err, probe);
    case 54: return try_jit_kb<5, 4>(p, stream, err, probe);
    case 64: return try_jit_kb<6, 4>(p, stream, err, probe);
    case 74: return try_jit_kb<7, 4>(p, stream, err, probe);
    case 84: return try_jit_kb<8, 4>(p, stream, err, probe);
    case 94: return try_jit_kb<9, 4>(p, stream, err, probe);
    case 104: return try_jit_kb<10, 4>(p, stream, err, probe);
    default: return false;
  }
}

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

bool fast_envelope_code(int k, int b, const std::uint32_t* polys) {
  (void)polys;  // any generator polynomials: the edge labels are compile-time per code
  return k >= 5 && k <= 10 && b >= 2 && b <= 4;
}

bool fast_path_supported(const DecodeLaunch& p) {
  using namespace fast;
  if (p.b < 2 || p.b > 4) return false;
  cudaError_t unused = cudaSuccess;
  return try_group_k7(p, nullptr, &unused, true) || try_group_k9(p, nullptr, &unused, true) ||
         try_group_k568(p, nullptr, &unused, true) || try_jit(p, nullptr, &unused, true);
}

namespace fast {
namespace {
template <int K, class PN>
bool try_jit_punct_pn(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err, std::int64_t* mi0,
                      std::int64_t* mi1) {
  return try_punct_with<PlanCode<K, 2>, 16, PN>(p, stream, err, mi0, mi1, [&](cudaError_t* e) {
    return jit::punct_kernel(p.k, p.polys, pattern, e);
  });
}

template <int K>
bool try_jit_punct_k(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err, std::int64_t* mi0,
                     std::int64_t* mi1) {
  if (pattern == 23) return try_jit_punct_pn<K, PunctR23>(p, pattern, stream, err, mi0, mi1);
  if (pattern == 34) return try_jit_punct_pn<K, PunctR34>(p, pattern, stream, err, mi0, mi1);
  return false;
}

// Fused depuncture for the other K = 7 rate-1/2 codes: a run-time
// instantiation of the same kernel ((133,171) r3/4: 1.03x the separate pass +
// decode). Not for K = 5 / 6 (64 / 32 frames per warp: more than the fills'
// two lanes per frame slot cover, plan()), nor K >= 8: there the decode costs
// 2-4x more per bit, the separate pass is a smaller share than the fused
// staging's per-block cost (K = 9 (561,753): fused 0.94x,
// profiles/r02_ab_notes.md).
bool try_jit_punct(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err, std::int64_t* mi0,
                   std::int64_t* mi1) {
  if (p.b != 2 || p.k != 7 || !jit_code(p)) return false;
  return try_jit_punct_k<7>(p, pattern, stream, err, mi0, mi1);
}
}  // namespace
}  // namespace fast

bool launch_fast_punct_i8(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err,
                          std::int64_t* mi0, std::int64_t* mi1) {
  if (fast::K7a::matches(p.k, p.b, p.polys)) return fast::try_punct_k7(p, pattern, stream, err, mi0, mi1);
  return fast::try_jit_punct(p, pattern, stream, err, mi0, mi1);
}

cudaError_t side_fork(cudaStream_t main, cudaStream_t* side) {
  fast::SideStream* ss = fast::side_stream();
  if (!ss) return cudaErrorUnknown;
  if (cudaError_t e = cudaEventRecord(ss->fork, main); e != cudaSuccess) return e;
  if (cudaError_t e = cudaStreamWaitEvent(ss->s, ss->fork, 0); e != cudaSuccess) return e;
  *side = ss->s;
  return cudaSuccess;
}

cudaError_t side_join(cudaStream_t main) {
  fast::SideStream* ss = fast::side_stream();
  if (!ss) return cudaErrorUnknown;
  if (cudaError_t e = cudaEventRecord(ss->join, ss->s); e != cudaSuccess) return e;
  return cudaStreamWaitEvent(main, ss->join, 0);
}

bool fast_output_whole_words(const DecodeLaunch& p) {
  return fast_path_supported(p) && fast::small_writes_whole_words(p);
}

cudaError_t launch_fast_i8(const DecodeLaunch& p, cudaStream_t stream) {
  using namespace fast;
  cudaError_t err = cudaErrorNotSupported;
  if (small_launch_wanted(p) && try_small(p, stream, &err)) return err;
  if (try_group_k7(p, stream, &err, false)) return err;
  if (try_group_k9(p, stream, &err, false)) return err;
  if (try_group_k568(p, stream, &err, false)) return err;
  if (try_jit(p, stream, &err, false)) return err;
  return cudaErrorNotSupported;
}

}  // namespace vd
