// Internal launch interface between the C-ABI layer (vd_capi.cu) and the
// kernels (vd_generic.cu, vd_fast.cu, vd_synth.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "vd_launch.h"

namespace vd {

/// Generic sm_100a kernels (any K in [2, 16], B in [2, 8]); int8 LLRs with
/// int32 metrics or double LLRs with double metrics. K <= kMaxGenericK: warp
/// per frame (vd_generic.cu); larger K: CTA per frame with the path metrics in
/// a per-CTA global (L2) scratch (vd_bigk.cu, launch_bigk_*).
constexpr int kMaxGenericK = 12;
constexpr int kMaxK = 16;  // reference trellis.cpp:44
cudaError_t launch_generic_i8(const DecodeLaunch& p, cudaStream_t stream);
cudaError_t launch_generic_f64(const DecodeLaunch& p, cudaStream_t stream);
cudaError_t launch_bigk_i8(const DecodeLaunch& p, cudaStream_t stream);
cudaError_t launch_bigk_f64(const DecodeLaunch& p, cudaStream_t stream);

/// Stages a fast-kernel window may read past its end (rounding to 4-stage
/// blocks + the two-block LLR prefetch); callers building padded copies or
/// choosing which frames go to the fast kernel keep this much readable slack.
constexpr int kPfSlackStages = 12;

/// Register-resident fast kernel. Returns cudaErrorNotSupported when the
/// code/config is outside its envelope (caller then uses the generic one).
bool fast_path_supported(const DecodeLaunch& p);
cudaError_t launch_fast_i8(const DecodeLaunch& p, cudaStream_t stream);
/// True when launch_fast_i8(p) writes every output word of its frames whole
/// (the small-launch kernel with 32-aligned frame / subframe boundaries): the
/// caller may then skip zeroing the output.
bool fast_output_whole_words(const DecodeLaunch& p);
/// Fused depuncture (pattern 23: "11;10", 34: "110;101"; B = 2 codes with a
/// fused instantiation): p.llr is the punctured stream; launches the fast
/// kernel over the interior frames [*mi0, *mi1) it takes (stream == nullptr
/// and err == nullptr: plan only). False: not supported for this code/config.
bool launch_fast_punct_i8(const DecodeLaunch& p, int pattern, cudaStream_t stream, cudaError_t* err,
                          std::int64_t* mi0, std::int64_t* mi1);
/// The calling thread's side stream on the current device (the one the fast
/// launches use for edge frames): side_fork makes it wait for the work
/// enqueued on `main` so far and returns it; side_join makes `main` wait for
/// the work enqueued on it so far. (Launches on the side stream may use it
/// themselves: the waits are captured at enqueue time.)
cudaError_t side_fork(cudaStream_t main, cudaStream_t* side);
cudaError_t side_join(cudaStream_t main);
namespace jit {
/// Run-time (NVRTC) instantiation of the fast kernel for a code outside the
/// precompiled list (vd_jit.cu); nullptr + *err (cudaErrorInvalidSource:
/// compile failure, see last_log()) on failure. VITDEC_JIT=0 disables it.
bool enabled();
const void* fast_kernel(int k, int b, const std::uint32_t* polys, bool tm, bool gl, cudaError_t* err);
/// The small-launch kernel (vd_small_dev.cuh, 8 states per lane) for a rate-1/2 code.
const void* small_kernel(int k, const std::uint32_t* polys, cudaError_t* err);
/// Fused-depuncture fast kernel (pattern 23: PunctR23, 34: PunctR34) of a B = 2 code.
const void* punct_kernel(int k, const std::uint32_t* polys, int pattern, cudaError_t* err);
const std::string& last_log();
/// Compile only (no GPU needed): false + last_log() on failure.
bool compile_check(int k, int b, const std::uint32_t* polys);
}  // namespace jit
/// Complement-paired code inside the fast kernel's envelope (vd_fast.cu).
bool fast_envelope_code(int k, int b, const std::uint32_t* polys);

/// Exact segment-parallel decode of one long frame (serial_decode, f >= N;
/// max-plus transfer matrices, vd_serial.cu). S <= 64, B in {2, 3}, int8.
bool serial_parallel_supported(const DecodeLaunch& p);
cudaError_t launch_serial_parallel_i8(const DecodeLaunch& p, cudaStream_t stream);

/// Zero-padded block heads for the fast kernel: for every block j of the
/// batch (blk_stage: device [nblocks + 1]), head[j * pitch * b ...] = v1 zero
/// stages followed by the block's first min(copy, n_j) stages (rest zero).
cudaError_t launch_head_gather(const std::int8_t* llr, const std::int64_t* blk_stage, int nblocks, int b, int v1,
                               std::int64_t pitch, std::int64_t copy, std::int8_t* head, cudaStream_t stream);

/// Device depuncture of stages [t0, t0 + n) (reference decoder.cpp:131-163):
/// out[(t - t0) * b + row] = mask(row, t % period) ? next punctured byte : 0.
/// `in` points at the first kept byte of stage t0, whose absolute offset in
/// the punctured stream is in0. rank[q] (q = col * b + row, the reference's
/// column-major mask order) is the kept index of position q inside its period,
/// or -1 when q is punctured. `in` holds in_len bytes. A unit is
/// unit_periods whole periods: unit_bytes = unit_periods * period * b output
/// bytes (a multiple of 16), unit_in = unit_periods * kept input bytes (a
/// multiple of 4); a tile (one shared-memory staging round) is tu units.
constexpr int kMaxPunctureCells = 1024;  // period * b
struct DepunctureLaunch {
  const std::int8_t* in = nullptr;
  std::int64_t in0 = 0, in_len = 0;
  std::int8_t* out = nullptr;  // 4-byte aligned
  std::int64_t t0 = 0, n = 0;
  int b = 0, period = 0, kept = 0;
  int unit_periods = 0, unit_bytes = 0, unit_in = 0, tu = 0;
  std::int16_t rank[kMaxPunctureCells] = {};
};
cudaError_t launch_depuncture_i8(const DepunctureLaunch& p, cudaStream_t stream);
/// Real-valued depuncture (the drop-in vitdec::depuncture on LlrBlock
/// doubles): one thread per output element, out[t * b + row] =
/// in[(t / period) * kept + rank[(t % period) * b + row]] or 0.
cudaError_t launch_depuncture_f64(const double* in, std::int64_t n_stages, int b, int period, int kept,
                                  const std::int16_t* rank, double* out, cudaStream_t stream);

/// 4-bit wire format: widen `count` signed nibbles (element i in nibble
/// nib_off + i of `in`, low nibble first) to int8 at `out` (8-byte aligned).
cudaError_t launch_unpack_i4(const std::uint8_t* in, int nib_off, std::int64_t count, std::int8_t* out,
                             cudaStream_t stream);

cudaError_t launch_synth_i8(int k, int b, const std::uint32_t* polys, std::int64_t t_begin, std::int64_t n,
                            double sigma, double scale, std::uint64_t seed, std::int8_t* llr, std::uint32_t* bits,
                            cudaStream_t stream);
cudaError_t launch_count_bit_errors(const std::uint32_t* a, const std::uint32_t* b, std::int64_t n_bits,
                                    unsigned long long* count, cudaStream_t stream);

/// Kernel launches issued by this library (every <<<>>> site calls
/// note_launch); exported as vd_kernel_launches() so benchmarks count the
/// launches of their timed region instead of assuming them.
void note_launch(int n = 1);

/// Dynamic shared-memory limit every kernel's cudaFuncAttributeMaxDynamic-
/// SharedMemorySize is set to (sm_100 maximum per CTA). Always the maximum,
/// never the launch's own size: host threads launching different geometries
/// of one kernel at once must not lower the limit under each other.
constexpr int kMaxDynSmem = 232448;
/// Sets kernel `kern`'s dynamic shared-memory limit to kMaxDynSmem on the
/// current device, once per (kernel, device) (a driver call per launch costs
/// microseconds of host time that small, latency-bound launches notice).
cudaError_t allow_max_smem(const void* kern);

/// SM count of the current device (cached per device).
int sm_count();

/// Makes the current device's default memory pool keep freed blocks (release
/// threshold = max), so the per-launch stream-ordered scratch allocations
/// (cudaMallocAsync) of the kernels are pool hits instead of fresh mappings.
cudaError_t retain_async_pool();

}  // namespace vd
