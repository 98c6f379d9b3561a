/* vitdec_b200 — C-ABI of the B200-native framed soft-decision Viterbi decoder.
 *
 * This is the drop-in boundary between the reference's C++ decoder API
 * (reference proj/include/vitdec/decoder.hpp, trellis.hpp) and the sm_100a
 * kernels. The reference has no FFI of its own — its entry points are plain
 * C++ functions — so each symbol below names the reference function whose
 * body it replaces. The C++ API in include/vitdec/ (implemented in
 * paper_2011_09337_b200/csrc/vitdec_api.cpp) is a thin wrapper over these
 * calls, and Python binds the same symbols via ctypes.
 *
 * Conventions
 *  - LLR streams are stage-major, B values per stage (element (b, t) at
 *    t*B + b), positive = bit 0 more likely. This is the memory order of the
 *    reference LlrBlock (Eigen::ArrayXXd B x N column-major,
 *    reference channel.hpp:11-13, channel.cpp:55-62).
 *  - Decoded bits are bit-packed LSB-first into uint32 words: bit i of the
 *    stream is (out[i / 32] >> (i % 32)) & 1.
 *  - Every call returns a vd_status; VD_OK == 0. On failure
 *    vd_last_error() returns a thread-local message. VD_EINVAL carries the
 *    exact std::invalid_argument message the reference throws.
 *  - All entry points are re-entrant and thread-safe (the reference calls
 *    framed_decode concurrently from BER-sweep worker threads,
 *    reference berlab.cpp:63-88): no mutable global state except the
 *    per-thread error string and a per-(thread, device) stream cache.
 *  - There is no CPU fallback: without a usable CUDA device every decode
 *    entry point returns VD_ECUDA.
 */
#ifndef VITDEC_B200_H
#define VITDEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VD_OK = 0,
  VD_EINVAL = 1,       /* invalid argument (reference std::invalid_argument) */
  VD_ECUDA = 2,        /* CUDA runtime/launch failure or no device */
  VD_EUNSUPPORTED = 3, /* valid for the reference but outside the GPU path (K > 12, B > 8) */
  VD_ENOMEM = 4
} vd_status;

/* reference decoder.hpp:13 (enum class TracebackStart) */
typedef enum { VD_TB_STORED_MAX = 0, VD_TB_RANDOM = 1 } vd_tb_start;

/* reference decoder.hpp:20-31 (struct FrameConfig) */
typedef struct {
  int32_t f;     /* output bits per frame, >= 1 */
  int32_t v1;    /* warm-up stages left of the frame, >= 0 */
  int32_t v2;    /* convergence stages right of each (sub)frame, >= 0 */
  int32_t f0;    /* subframe size for parallel traceback; 0 = one traceback per frame */
  int32_t start; /* vd_tb_start */
  int32_t reserved;
  uint64_t seed; /* random-start salt seed (used only with VD_TB_RANDOM) */
} vd_frame_cfg;

/* reference decoder.hpp:33-37 (struct DecodeStats) */
typedef struct {
  int64_t frames;
  int64_t stages;
  int64_t tracebacks;
} vd_stats;

/* Execution options for the host-buffer entry points. */
typedef struct {
  int32_t num_devices;    /* 0 = current device only */
  const int32_t* devices; /* NULL = devices 0 .. num_devices-1 */
  int64_t chunk_stages;   /* streaming chunk size per device; 0 = automatic */
} vd_exec;

/* Opaque compiled code: trellis tables + device-side constants. Immutable
 * and shareable across threads after creation (reference SPEC: Trellis is
 * immutable). */
typedef struct vd_code vd_code;

/* ---- trellis (replaces reference trellis.cpp:38-103) ---------------------- */

/* Validate (K, B, polys) exactly as reference trellis.cpp:38-53 and build the
 * tables of trellis.cpp:57-101. polys are K-bit, newest-bit tap at the MSB. */
vd_status vd_code_create(int32_t k, int32_t b, const uint32_t* polys, vd_code** out);
void vd_code_destroy(vd_code* code);
int32_t vd_code_k(const vd_code* code);
int32_t vd_code_b(const vd_code* code);
/* Host copies of the [S*2] tables of reference trellis.hpp:66-70 (any
 * pointer may be NULL). complement_paired per trellis.cpp:93-100. */
vd_status vd_code_tables(const vd_code* code, uint32_t* next, uint32_t* out, uint32_t* pred, uint32_t* in_out,
                         int32_t* complement_paired);
/* 1 when the fast register-resident kernel serves this code, else 0 (the
 * generic sm_100a kernel is used). Codes outside the precompiled list with
 * 5 <= K <= 10 and B in {2, 3, 4} are served by a run-time (NVRTC) instantiation
 * of the same kernel, compiled on first use and cached
 * (VITDEC_JIT=0 disables it, VITDEC_JIT_CACHE sets the cubin cache dir). */
int32_t vd_code_fast_path(const vd_code* code);
/* Diagnostics: compiles (without loading) the run-time fast-kernel
 * instantiation for this code with the embedded sources; VD_OK, or
 * VD_EUNSUPPORTED (code outside the fast envelope) / VD_ECUDA (NVRTC missing
 * or the compile failed; vd_last_error() holds the log). Needs no GPU. */
vd_status vd_code_jit_check(const vd_code* code);

/* ---- frame geometry (reference decoder.cpp:10-20, 241-267) ---------------- */

/* FrameConfig::validate(pattern_period), reference decoder.cpp:10-20. */
vd_status vd_frame_cfg_validate(const vd_frame_cfg* cfg, int32_t pattern_period);
/* DecodeStats that framed_decode reports for n_stages (decoder.cpp:256-265). */
vd_status vd_frame_stats(const vd_frame_cfg* cfg, int64_t n_stages, vd_stats* stats);
/* Frame-range partition for sharding frames [0, ceil(n/f)) over `parts`
 * devices: part p gets [first[p], first[p+1]); boundaries are chosen so
 * every part but the first starts on a 32-bit output word when possible. */
vd_status vd_partition_frames(const vd_frame_cfg* cfg, int64_t n_stages, int32_t parts, int64_t* first);

/* ---- device-resident decode: the hot path --------------------------------- */

/* Decode frames [frame_begin, frame_end) of an n_stages stream whose int8
 * LLRs are resident on `device`. Replaces the per-frame loop of reference
 * framed_decode (decoder.cpp:241-254) and decode_frame (decoder.cpp:170-237).
 *   llr_dev     device pointer to the LLRs of stage llr_stage0 (B bytes per
 *               stage); must cover [window_begin(frame_begin),
 *               window_end(frame_end-1)) — use vd_frame_window().
 *   out_dev     device pointer to packed output words for stages starting at
 *               out_stage0 (out_stage0 % 32 == 0). Words overlapping the
 *               decoded output range are overwritten; bits of those words that
 *               lie outside [frame_begin*f, min(frame_end*f, n)) are zero.
 *   sigma_dev   optional (NULL): receives the final path metrics of every
 *               frame, [frame_end-frame_begin][S] int64, renormalisation
 *               offset re-added (metric parity with reference decoder.cpp:195-203).
 *   stream      cudaStream_t (NULL = legacy default stream of `device`).
 * Asynchronous with respect to the host. */
vd_status vd_decode_i8_device(const vd_code* code, const vd_frame_cfg* cfg, int64_t n_stages, const int8_t* llr_dev,
                              int64_t llr_stage0, int64_t frame_begin, int64_t frame_end, uint32_t* out_dev,
                              int64_t out_stage0, int64_t* sigma_dev, int32_t device, void* stream);
/* Same for real-valued LLRs with double path metrics: identical operations
 * and order as reference decoder.cpp:22-76, hence bit-identical to the
 * reference on ANY input. sigma_dev is double here. */
vd_status vd_decode_f64_device(const vd_code* code, const vd_frame_cfg* cfg, int64_t n_stages, const double* llr_dev,
                               int64_t llr_stage0, int64_t frame_begin, int64_t frame_end, uint32_t* out_dev,
                               int64_t out_stage0, double* sigma_dev, int32_t device, void* stream);
/* Stage window [*begin, *end) the frames [frame_begin, frame_end) read. */
vd_status vd_frame_window(const vd_frame_cfg* cfg, int64_t n_stages, int64_t frame_begin, int64_t frame_end,
                          int64_t* begin, int64_t* end);

/* ---- batched independent blocks ------------------------------------------ */

/* Decodes n_blocks independent LLR blocks in one device pass, each exactly as
 * its own framed_decode call would (reference decoder.hpp:74-79): its own
 * frame grid, frames clipped at both ends of the block, random-start salt
 * from the block-local frame index. This is how reference run_ber_sweep
 * decodes a BER point (berlab.cpp:63-88: one framed_decode per block of
 * block_bits). Block j holds block_stages[j] >= 1 stages (host array); the
 * blocks are concatenated in llr_dev, and block j's decoded bits land in
 * out_dev at bit offset block_stages[0] + ... + block_stages[j-1] (the whole
 * ceil(total/32)-word range is overwritten). stats (may be NULL) is the sum
 * over blocks. Asynchronous with respect to the host. */
vd_status vd_decode_batch_i8_device(const vd_code* code, const vd_frame_cfg* cfg, int32_t n_blocks,
                                    const int64_t* block_stages, const int8_t* llr_dev, uint32_t* out_dev,
                                    vd_stats* stats, int32_t device, void* stream);
vd_status vd_decode_batch_f64_device(const vd_code* code, const vd_frame_cfg* cfg, int32_t n_blocks,
                                     const int64_t* block_stages, const double* llr_dev, uint32_t* out_dev,
                                     vd_stats* stats, int32_t device, void* stream);
/* Host-buffer form (one device: exec->devices[0], or the current device):
 * H2D of the concatenated blocks, the batched decode, D2H of the packed bits.
 * Synchronous. */
vd_status vd_decode_batch_i8(const vd_code* code, const vd_frame_cfg* cfg, int32_t n_blocks,
                             const int64_t* block_stages, const int8_t* llr, uint32_t* out_packed, vd_stats* stats,
                             const vd_exec* exec);

/* ---- host-buffer decode: the reference-facing call ------------------------ */

/* framed_decode (reference decoder.hpp:74-79) on host buffers: streams the
 * LLRs to the device(s) in chunks (H2D / kernel / D2H overlapped on
 * separate streams; pinned host memory gives full PCIe rate), shards frames
 * across exec->num_devices GPUs, and writes packed bits for all n_stages
 * stages into out_packed (ceil(n/32) words). stats may be NULL. Output is
 * bit-identical for any device count / chunking. */
vd_status vd_decode_i8(const vd_code* code, const vd_frame_cfg* cfg, const int8_t* llr, int64_t n_stages,
                       uint32_t* out_packed, vd_stats* stats, const vd_exec* exec);
vd_status vd_decode_f64(const vd_code* code, const vd_frame_cfg* cfg, const double* llr, int64_t n_stages,
                        uint32_t* out_packed, vd_stats* stats, const vd_exec* exec);
/* ---- puncturing (reference codec.hpp:13-33, decoder.hpp:69-72) ----------- */

/* PuncturePattern: B rows x period columns, mask[col * b + row] in {0, 1}
 * (1 keeps the bit), column-major as reference codec.hpp:15-21. */
typedef struct {
  int32_t b;
  int32_t period;
  const uint8_t* mask;
} vd_puncture;

/* PuncturePattern::validate (reference codec.cpp:12-23); VD_EUNSUPPORTED when
 * period * b > 1024 (GPU depuncture table limit). */
vd_status vd_puncture_validate(const vd_puncture* pattern);
/* Stages covered by a punctured stream of n_punctured values; VD_EINVAL
 * "punctured length inconsistent with pattern" exactly when reference
 * depuncture throws (decoder.cpp:141-152). */
vd_status vd_depuncture_stages(const vd_puncture* pattern, int64_t n_punctured, int64_t* n_stages);
/* depuncture (reference decoder.cpp:131-163) on the device: llr_dev
 * (4-byte aligned, n_stages * b bytes) receives the stage-major int8 block
 * with 0 at every punctured position. Asynchronous. */
vd_status vd_depuncture_i8_device(const vd_puncture* pattern, const int8_t* punctured_dev, int64_t n_punctured,
                                  int8_t* llr_dev, int32_t device, void* stream);
/* framed_decode(depuncture(stream, pattern), trellis, cfg) — the composition
 * reference run_ber_sweep and the CLI run (berlab.cpp:79-84,
 * vitdec_cli.cpp:172-176) — on host buffers: only the punctured bytes cross
 * PCIe; each streamed chunk is depunctured on the device right before its
 * decode. Output and stats as vd_decode_i8 on the depunctured block. */
vd_status vd_decode_punctured_i8(const vd_code* code, const vd_frame_cfg* cfg, const vd_puncture* pattern,
                                 const int8_t* punctured, int64_t n_punctured, uint32_t* out_packed, vd_stats* stats,
                                 const vd_exec* exec);
/* Device-resident form: every frame is decoded into out_dev (ceil(n_stages
 * / 32) words). For the r2/3 ("11;10") and r3/4 ("110;101") patterns of the
 * K=7 (171,133) code with f0 = 0 and a 4-byte aligned punctured_dev, the
 * depuncture is fused into the fast kernel's LLR staging (the depunctured
 * block never reaches HBM; llr_scratch_dev holds only the edge frames'
 * windows); otherwise, or with VITDEC_PUNCT_FUSED=0, llr_scratch_dev
 * (4-byte aligned, n_stages * b bytes, see vd_depuncture_stages) receives the
 * depunctured block first. Asynchronous; stats (may be NULL) is computed on
 * the host. */
vd_status vd_decode_punctured_i8_device(const vd_code* code, const vd_frame_cfg* cfg, const vd_puncture* pattern,
                                        const int8_t* punctured_dev, int64_t n_punctured, int8_t* llr_scratch_dev,
                                        uint32_t* out_dev, vd_stats* stats, int32_t device, void* stream);

/* ---- 4-bit LLR wire format --------------------------------
 * Two signed 4-bit LLRs per byte, element i of the stage-major stream (t*B + b)
 * in nibble i (low nibble first), values in [-8, 7] (e.g. the quantiser
 * clamp(rint(scale * y), -7, 7)). Decoding is exact for those integer LLRs:
 * identical to vd_decode_i8 on the same values widened to int8. */

/* framed_decode on a 4-bit host stream: only the packed bytes cross PCIe
 * (1 byte per r1/2 stage), each chunk is widened on the device. Same output,
 * stats, sharding and threading as vd_decode_i8. */
vd_status vd_decode_i4(const vd_code* code, const vd_frame_cfg* cfg, const uint8_t* llr4, int64_t n_stages,
                       uint32_t* out_packed, vd_stats* stats, const vd_exec* exec);
/* Widen `count` 4-bit LLRs (device, 4-byte aligned) to int8 (device, 8-byte
 * aligned). Asynchronous. */
vd_status vd_unpack_i4_device(const uint8_t* llr4_dev, int64_t count, int8_t* llr_dev, int32_t device, void* stream);

/* serial_decode (reference decoder.cpp:101-129): one frame, no overlap. */
vd_status vd_serial_decode_f64(const vd_code* code, const double* llr, int64_t n_stages, uint32_t* out_packed,
                               vd_stats* stats, int32_t device);

/* Real-valued depuncture on host buffers (the drop-in vitdec::depuncture,
 * reference decoder.cpp:131-163): n_stages from vd_depuncture_stages;
 * llr_out receives n_stages * B doubles, stage-major, 0.0 at punctured
 * positions. Runs on the current device (no CPU fallback). */
vd_status vd_depuncture_f64(const vd_puncture* pattern, const double* punctured, int64_t n_punctured,
                            double* llr_out);

/* ---- synthetic input (bench / streaming tests; not reference parity data) - */

/* Fills llr_dev with int8 LLRs for n_stages stages of a random message
 * encoded by `code`, BPSK + AWGN at sigma, quantised q = clamp(rint(scale*y),
 * -127, 127); counter-based RNG keyed by seed. If bits_dev != NULL the
 * packed message bits are written too. Device-side, asynchronous. */
vd_status vd_synth_llr_i8_device(const vd_code* code, int64_t n_stages, double sigma, double scale, uint64_t seed,
                                 int8_t* llr_dev, uint32_t* bits_dev, int32_t device, void* stream);

/* Stages [t_begin, t_begin + n_stages) of the same synthetic stream (every
 * value is a pure function of (seed, stage)): a shard's halo window is
 * generated on its own device, identical to the whole-stream values. llr_dev
 * receives stage t at (t - t_begin) * B; bits_dev (t_begin % 32 == 0 only)
 * the packed message bits of the range; llr_dev may be NULL (bits only). */
vd_status vd_synth_llr_i8_range_device(const vd_code* code, int64_t t_begin, int64_t n_stages, double sigma,
                                       double scale, uint64_t seed, int8_t* llr_dev, uint32_t* bits_dev,
                                       int32_t device, void* stream);

/* Number of bit positions where packed a and b differ over n bits (device). */
vd_status vd_count_bit_errors_device(const uint32_t* a_dev, const uint32_t* b_dev, int64_t n_bits,
                                     unsigned long long* count_dev, int32_t device, void* stream);

const char* vd_last_error(void);
const char* vd_version(void);
/* Kernels this library has launched so far in the process (all devices and
 * threads): a benchmark reads it around its timed region. */
uint64_t vd_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* VITDEC_B200_H */
