// Decode-launch descriptor shared by the host dispatch and the kernels. Kept
// free of host-only headers: the fast kernel's device half (vd_fast_dev.cuh)
// includes it and is also compiled at run time by NVRTC (vd_jit.cu).
#pragma once

#include "vd_std.h"

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
  // Batched mode (nblocks > 0): the stream is the concatenation of nblocks
  // independent blocks (reference run_ber_sweep decodes every block with its
  // own framed_decode call, berlab.cpp:63-88). Block j spans stages
  // [blk_stage[j], blk_stage[j+1]) and global frames [blk_frame[j],
  // blk_frame[j+1]); its frames are clipped at the block ends and their
  // random-start salt uses the block-local frame index. Frame indices in
  // [frame_begin, frame_end) are global; n is the total stage count.
  int nblocks = 0;
  const std::int64_t* blk_stage = nullptr;  // device [nblocks + 1]
  const std::int64_t* blk_frame = nullptr;  // device [nblocks + 1]
  const std::int32_t* blk_ilo = nullptr;    // device [nblocks]: fast-kernel frames are local [ilo, ihi)
  const std::int32_t* blk_ihi = nullptr;
  // Generic kernels only: process frame_list[frame_begin .. frame_end) (global
  // frame ids) instead of the index range itself.
  const std::int64_t* frame_list = nullptr;
  std::int64_t safe_stage = 0;  // batched fast launch: window start of some interior frame
  // Fast kernel only: frames whose window is clipped by their block start
  // (m*f < v1) read a zero-padded copy of the block head instead:
  // llr_head[(blk * head_pitch + (t + v1)) * b] = stage t of block blk.
  const std::int8_t* llr_head = nullptr;
  std::int64_t head_pitch = 0;
};

/// A global frame id resolved to its block: block-local frame index, block
/// length and the block's first stage in the concatenated stream.
struct FrameRef {
  std::int64_t m, n, base;
  int blk;
};

#if defined(__CUDACC__) || defined(__CUDACC_RTC__)
__device__ __forceinline__ FrameRef resolve_frame(const DecodeLaunch& p, std::int64_t idx) {
  const std::int64_t g = p.frame_list ? __ldg(p.frame_list + idx) : idx;
  if (p.nblocks == 0) return FrameRef{g, p.n, 0, 0};
  int lo = 0, hi = p.nblocks;  // blk_frame[lo] <= g < blk_frame[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(p.blk_frame + mid) <= g) {
      lo = mid;
    } else {
      hi = mid;
    }
  }
  const std::int64_t b0 = __ldg(p.blk_stage + lo);
  return FrameRef{g - __ldg(p.blk_frame + lo), __ldg(p.blk_stage + lo + 1) - b0, b0, lo};
}
#endif

}  // namespace vd
