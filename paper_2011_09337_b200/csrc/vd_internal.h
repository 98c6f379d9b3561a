// Internal launch interface between the C-ABI layer (vd_capi.cu) and the
// kernels (vd_generic.cu, vd_fast.cu, vd_synth.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace vd {

/// Everything a decode launch needs. Pointers are device pointers.
struct DecodeLaunch {
  int k = 0, b = 0, s = 0;
  int f = 0, v1 = 0, v2 = 0, f0 = 0, start = 0;
  std::uint64_t seed = 0;
  std::int64_t n = 0;                     // stream length in stages
  std::int64_t frame_begin = 0, frame_end = 0;
  const void* llr = nullptr;              // LLRs of stage llr_stage0
  std::int64_t llr_stage0 = 0;
  std::uint32_t* out = nullptr;           // packed bits of stage out_stage0 (word aligned)
  std::int64_t out_stage0 = 0;
  void* sigma = nullptr;                  // optional final metrics [frames][S]
  const std::uint32_t* in_out = nullptr;  // device copy of Trellis::in_out_ [S*2]
  std::uint32_t polys[8] = {};
  bool complement_paired = false;
};

/// Generic sm_100a kernel (any K in [2, 12], B in [2, 8]); int8 LLRs with
/// int32 metrics or double LLRs with double metrics.
cudaError_t launch_generic_i8(const DecodeLaunch& p, cudaStream_t stream);
cudaError_t launch_generic_f64(const DecodeLaunch& p, cudaStream_t stream);

/// Register-resident fast kernel. Returns cudaErrorNotSupported when the
/// code/config is outside its envelope (caller then uses the generic one).
bool fast_path_supported(const DecodeLaunch& p);
cudaError_t launch_fast_i8(const DecodeLaunch& p, cudaStream_t stream);

cudaError_t launch_synth_i8(int k, int b, const std::uint32_t* polys, std::int64_t n, double sigma, double scale,
                            std::uint64_t seed, std::int8_t* llr, std::uint32_t* bits, cudaStream_t stream);
cudaError_t launch_count_bit_errors(const std::uint32_t* a, const std::uint32_t* b, std::int64_t n_bits,
                                    unsigned long long* count, cudaStream_t stream);

/// SM count of the current device (cached per device).
int sm_count();

}  // namespace vd
