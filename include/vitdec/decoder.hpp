// Drop-in declaration of the vitdec decoder API (reference
// proj/include/vitdec/decoder.hpp:13-79) backed by the B200 kernels.
//
// framed_decode / serial_decode run on the GPU through the C-ABI in
// vitdec_b200.h (no CPU fallback): integer-valued LLR blocks in [-127, 127]
// take the int8 fixed-point kernels, any other real-valued block the
// FP64-metric kernel; both are bit-identical to the reference. The per-stage
// helpers (branch_metric ... acs_stage) are the reference's single-stage
// semantics on the host, kept because the reference's tests call them.
#pragma once

#include <Eigen/Dense>
#include <cstdint>
#include <vector>

#include "vitdec/channel.hpp"
#include "vitdec/codec.hpp"
#include "vitdec/trellis.hpp"

namespace vitdec {

enum class TracebackStart { kStoredMax, kRandom };

/// Overlapped tiling: frames of f output bits, each preceded by v1 warm-up
/// stages and followed by v2 convergence stages; f0 > 0 splits a frame's
/// traceback into subframes of f0 bits (each with its own v2 tail).
struct FrameConfig {
  int f = 0;
  int v1 = 0;
  int v2 = 0;
  int f0 = 0;
  TracebackStart start = TracebackStart::kStoredMax;
  std::uint64_t seed = 0;

  /// std::invalid_argument on bad values; f, v1, v2 must be multiples of a
  /// puncture period > 1.
  void validate(int pattern_period = 1) const;
};

struct DecodeStats {
  std::int64_t frames = 0;
  std::int64_t stages = 0;
  std::int64_t tracebacks = 0;
};

struct DecodeOutput {
  BitVec bits;
  DecodeStats stats;
};

double branch_metric(std::uint32_t bo, const Eigen::Ref<const Eigen::ArrayXd>& llr_t);
Eigen::ArrayXd stage_metrics(const Eigen::Ref<const Eigen::ArrayXd>& llr_t);
void fill_stage_table(const Eigen::Ref<const Eigen::ArrayXd>& llr_t, double* table);
void acs_stage(const Eigen::ArrayXd& sigma_prev, const double* stage_table, const Trellis& trellis,
               Eigen::ArrayXd& sigma_cur, std::uint16_t* pi_col);

DecodeOutput serial_decode(const LlrBlock& llr, const Trellis& trellis);

LlrBlock depuncture(const Eigen::Ref<const Eigen::ArrayXd>& punctured, const PuncturePattern& pattern);

/// `workers` is accepted for API compatibility; parallelism is the GPU grid.
/// The number of GPUs the frames are sharded over is VITDEC_GPUS (default 1).
DecodeOutput framed_decode(const LlrBlock& llr, const Trellis& trellis, const FrameConfig& cfg, int workers = 1);

// ---- native extension (this build) ---------------------------------------

/// Execution options for the native entry point.
struct ExecOptions {
  int gpus = 0;                  // > 0: frames sharded over devices 0 .. gpus-1; 0: the current device
  std::int64_t chunk_stages = 0; // streaming chunk per device (0 = automatic)
};

/// framed_decode on a stage-major int8 stream (B values per stage) with
/// bit-packed output: bit i -> (packed_out[i / 32] >> (i % 32)) & 1, which
/// must hold ceil(n_stages / 32) words. Pinned host memory streams at full
/// PCIe rate.
DecodeStats framed_decode(const std::int8_t* llr, std::int64_t n_stages, const Trellis& trellis,
                          const FrameConfig& cfg, std::uint32_t* packed_out, const ExecOptions& exec = {});

/// framed_decode(depuncture(stream, pattern), trellis, cfg) — the chain the
/// reference BER harness and CLI run (berlab.cpp:79-84, vitdec_cli.cpp:172-176)
/// — on an int8 punctured stream: only the punctured bytes cross PCIe and the
/// depuncture runs on the device. packed_out holds ceil(n_stages / 32) words,
/// n_stages as reference depuncture derives it (decoder.cpp:141-152).
DecodeStats framed_decode_punctured(const std::int8_t* punctured, std::int64_t n_punctured,
                                    const PuncturePattern& pattern, const Trellis& trellis, const FrameConfig& cfg,
                                    std::uint32_t* packed_out, const ExecOptions& exec = {});

}  // namespace vitdec
