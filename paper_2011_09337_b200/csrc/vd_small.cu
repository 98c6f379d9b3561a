// Host planning and launch of the small-launch kernel (vd_small_dev.cuh) and
// its instantiations. Used by launch_fast_i8 when the 16-states-per-lane fast
// kernel would run less than one warp per scheduler (e.g. the reference's
// 1 M-bit default: 3907 frames = 245 warps of 16 frames), where a warp's
// dependency chain, not throughput, sets the time; VITDEC_SMALL=0 disables it.
#include <algorithm>
#include <cstdlib>

#include "vd_fast.cuh"
#include "vd_small_dev.cuh"

namespace vd {
namespace fast {
namespace {

constexpr int kSmallSmemMax = 232448;

// Layout and grid for frames [mi0, mi1) that share one geometry (window L,
// output length f_out).
template <class C, int R>
bool plan_geom(const DecodeLaunch& p, std::int64_t mi0, std::int64_t mi1, int L, int f_out, SmallParams* out) {
  using GEO = Geo<C, R>;
  using SG = SmallGeo<R>;
  SmallParams sp{};
  sp.p = p;
  sp.m1 = 0xffffffffu;
  sp.L = L;
  sp.f_out = f_out;
  sp.nsb = (L + SG::SB - 1) / SG::SB;
  sp.step = p.f0 > 0 ? p.f0 : p.f;
  sp.num_sub = (f_out + sp.step - 1) / sp.step;
  if (sp.num_sub > 64 || L < 6 || SG::SB * sp.nsb > kSmallMaxStages || mi1 <= mi0) return false;
  sp.mi0 = mi0;
  sp.mi1 = mi1;
  sp.safe_stage = (mi1 - 1) * p.f - p.v1;  // the last frame's window (empty slots)
  // per-warp shared memory: staged windows, survivor rows, relayout buffer, start states
  sp.pitch = 4 * SG::WSB * sp.nsb + 4;  // (+ 1 word: keeps the rows of different frames on different banks)
  // survivor words: stages [SB floor(v1 / SB), SB nsb) + the traceback's over-read
  const int rows = (SG::SB * sp.nsb - SG::SB * (p.v1 / SG::SB)) / SG::SPW + 3;
  sp.llr_off = 0;
  sp.dec_off = (GEO::FPW * sp.pitch + 15) & ~15;  // (16-byte rows below: the relayout's LDS.128)
  sp.x_off = sp.dec_off + rows * 32 * 4;
  sp.ss_off = sp.x_off + GEO::GROUPS * GEO::XSTRIDE * 4;
  sp.smem_per_warp = (sp.ss_off + GEO::FPW * sp.num_sub * 2 + 15) & ~15;
  *out = sp;
  return true;
}

// The launch's frames in segments: [frame_begin, mi1) with the full window
// (interior and, when the buffer starts at stage 0, head frames), then every
// clipped tail frame with its own geometry (FrameGeom, reference
// decoder.cpp:175-191), all in ONE launch (the tail frames' warps run on other
// SMs beside the main segment's; no side stream, no events).
template <class C, int R>
bool plan_small(const DecodeLaunch& p, SmallLaunch* out) {
  using GEO = Geo<C, R>;
  if (GEO::B != 2 || p.nblocks > 0 || p.sigma || p.frame_list) return false;
  SmallLaunch sl{};
  const int L = p.f + p.v1 + p.v2;
  const std::int64_t lo = p.llr_stage0 == 0 ? 0 : (p.llr_stage0 + p.v1 + p.f - 1) / p.f;
  if (std::max(lo, p.frame_begin) != p.frame_begin) return false;  // windows before the buffer
  const std::int64_t hi = (p.n - p.f - p.v2 >= 0) ? (p.n - p.f - p.v2) / p.f + 1 : 0;  // full windows below
  const std::int64_t mi1 = std::min<std::int64_t>(hi, p.frame_end);
  std::int64_t warps = 0;
  int smem = 0;
  auto add = [&](std::int64_t m0, std::int64_t m1, int len, int f_out) {
    if (sl.nseg == kSmallSegs) return false;
    SmallParams& sp = sl.seg[sl.nseg];
    if (!plan_geom<C, R>(p, m0, m1, len, f_out, &sp)) return false;
    sl.warp_begin[sl.nseg] = static_cast<int>(warps);
    warps += (m1 - m0 + GEO::FPW - 1) / GEO::FPW;
    smem = std::max(smem, sp.smem_per_warp);
    ++sl.nseg;
    return true;
  };
  if (mi1 > p.frame_begin && !add(p.frame_begin, mi1, L, p.f)) return false;
  for (std::int64_t m = std::max(mi1, p.frame_begin); m < p.frame_end; ++m) {
    const FrameGeom g(m, p.n, p.f, p.v1, p.v2, p.f0);
    const std::int64_t ws = m * p.f - p.v1;  // virtual window start (zero-filled below stage 0)
    if (!add(m, m + 1, static_cast<int>(g.end - ws), static_cast<int>(g.out_hi - g.out_lo))) return false;
  }
  if (sl.nseg == 0 || warps > (1 << 30)) return false;
  sl.warp_begin[sl.nseg] = static_cast<int>(warps);
  const int sms = sm_count();
  int wpc = static_cast<int>(std::min<std::int64_t>((warps + sms - 1) / sms, kSmallMaxWarps));
  wpc = std::max(wpc, 1);
  while (wpc > 1 && smem * wpc > kSmallSmemMax) --wpc;
  if (smem * wpc > kSmallSmemMax) return false;
  // one round of CTAs only: beyond that the 16-states-per-lane kernel in one
  // round of 4- / 8-warp CTAs is faster (2^21 stages: 75.6 -> see
  // profiles/r02_ab_notes.md), and its edge frames come back here
  if ((warps + wpc - 1) / wpc > sms) return false;
  sl.warps_per_cta = wpc;
  sl.smem_per_warp = smem;
  // every output word written whole by one task: frame and subframe
  // boundaries on 32-bit words (frame m's output starts at m * f), and a
  // stream end inside the launch on one too (tasks emit from their top stage
  // down, so a subframe ending at n must span whole words)
  const int step = p.f0 > 0 ? p.f0 : p.f;
  const bool ends_in = p.frame_end * static_cast<std::int64_t>(p.f) >= p.n;
  sl.whole_words = p.f % 32 == 0 && step % 32 == 0 && p.out_stage0 % 32 == 0 && (!ends_in || p.n % 32 == 0);
  *out = sl;
  return true;
}

cudaError_t launch_kernel(const void* kern, const SmallLaunch& sl, cudaStream_t stream) {
  const std::int64_t warps = sl.warp_begin[sl.nseg];
  const std::int64_t blocks = (warps + sl.warps_per_cta - 1) / sl.warps_per_cta;
  const std::size_t smem = static_cast<std::size_t>(sl.smem_per_warp) * sl.warps_per_cta;
  cudaError_t e = allow_max_smem(kern);
  if (e != cudaSuccess) return e;
  SmallLaunch arg = sl;
  void* args[] = {&arg};
  e = cudaLaunchKernel(kern, dim3(static_cast<unsigned>(blocks)), dim3(sl.warps_per_cta * 32), args, smem, stream);
  note_launch();
  return e;
}

template <class C, int R>
cudaError_t launch_small(const SmallLaunch& sl, cudaStream_t stream) {
  return launch_kernel(reinterpret_cast<const void*>(small_kernel<C, R>), sl, stream);
}

// Placeholder code of a K class for planning (plan_small uses only K and B);
// the kernel of any other rate-1/2 code comes from the run-time instantiation.
template <int K>
using SmallPlanCode = CodeB<K, 2, (1u << (K - 1)) | 1u, (1u << (K - 1)) | 1u>;

template <int K>
bool try_jit_small(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe, bool* whole) {
  SmallLaunch sl;
  if (!plan_small<SmallPlanCode<K>, 8>(p, &sl)) return false;
  if (whole) *whole = sl.whole_words;
  if (probe) return true;
  cudaError_t ek = cudaSuccess;
  const void* kern = jit::small_kernel(p.k, p.polys, &ek);
  *err = kern ? launch_kernel(kern, sl, stream) : (ek != cudaSuccess ? ek : cudaErrorInvalidSource);
  return true;
}

bool jit_small(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, bool probe, bool* whole) {
  if (p.b != 2 || !jit::enabled()) return false;
  switch (p.k) {
    case 5: return try_jit_small<5>(p, stream, err, probe, whole);
    case 6: return try_jit_small<6>(p, stream, err, probe, whole);
    case 7: return try_jit_small<7>(p, stream, err, probe, whole);
    // K = 8 / 9 instantiate and decode correctly, but lose to the
    // 16-states-per-lane kernel at every small-launch size measured (C1:
    // 13.1 vs 19.7 Gbps at K = 8, 9.3 vs 10.8 at K = 9; profiles/r02_ab_notes.md):
    // twice the warps and a 16 / 32-lane relayout per 3 stages. They stay on it.
    default: return false;
  }
}

}  // namespace

bool small_launch_wanted(const DecodeLaunch& p) {
  const char* env = std::getenv("VITDEC_SMALL");
  if (env && std::atoi(env) == 0) return false;
  if (p.nblocks > 0 || p.sigma || p.frame_list || p.b != 2) return false;
  // the 16-states-per-lane kernel would run fewer warps than the GPU has schedulers
  const std::int64_t warps16 = (p.frame_end - p.frame_begin + 15) / 16;
  return warps16 < static_cast<std::int64_t>(sm_count()) * 4;
}

// Which small-kernel plan serves p (nullptr: none); fills *sl.
bool plan_any(const DecodeLaunch& p, SmallLaunch* sl, int* code) {
  if (K7a::matches(p.k, p.b, p.polys) && plan_small<K7a, 8>(p, sl)) {
    *code = 0;
    return true;
  }
  if (K7b::matches(p.k, p.b, p.polys) && plan_small<K7b, 8>(p, sl)) {
    *code = 1;
    return true;
  }
  return false;
}

bool try_small(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err) {
  SmallLaunch sl;
  int code = -1;
  if (plan_any(p, &sl, &code)) {
    *err = code == 0 ? launch_small<K7a, 8>(sl, stream) : launch_small<K7b, 8>(sl, stream);
    return true;
  }
  if (K7a::matches(p.k, p.b, p.polys) || K7b::matches(p.k, p.b, p.polys)) return false;
  return jit_small(p, stream, err, false, nullptr);
}

bool small_can_take(const DecodeLaunch& p) {
  const char* env = std::getenv("VITDEC_SMALL");
  if (env && std::atoi(env) == 0) return false;
  if (p.nblocks > 0 || p.sigma || p.frame_list || p.b != 2) return false;
  SmallLaunch sl;
  int code = -1;
  if (plan_any(p, &sl, &code)) return true;
  if (K7a::matches(p.k, p.b, p.polys) || K7b::matches(p.k, p.b, p.polys)) return false;
  bool whole = false;
  return jit_small(p, nullptr, nullptr, true, &whole);
}

bool small_writes_whole_words(const DecodeLaunch& p) {
  if (!small_launch_wanted(p)) return false;
  SmallLaunch sl;
  int code = -1;
  if (plan_any(p, &sl, &code)) return sl.whole_words;
  if (K7a::matches(p.k, p.b, p.polys) || K7b::matches(p.k, p.b, p.polys)) return false;
  bool whole = false;
  return jit_small(p, nullptr, nullptr, true, &whole) && whole;
}

}  // namespace fast
}  // namespace vd
