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
  sp.dec_off = GEO::FPW * sp.pitch;
  sp.x_off = sp.dec_off + rows * 32 * 4;
  sp.ss_off = sp.x_off + GEO::GROUPS * GEO::XSTRIDE * 4;
  sp.smem_per_warp = (sp.ss_off + GEO::FPW * sp.num_sub * 2 + 15) & ~15;
  const std::int64_t warps = (mi1 - mi0 + GEO::FPW - 1) / GEO::FPW;
  const int sms = sm_count();
  int wpc = static_cast<int>(std::min<std::int64_t>((warps + sms - 1) / sms, kSmallMaxWarps));
  wpc = std::max(wpc, 1);
  while (wpc > 1 && sp.smem_per_warp * wpc > kSmallSmemMax) --wpc;
  if (sp.smem_per_warp * wpc > kSmallSmemMax) return false;
  sp.warps_per_cta = wpc;
  *out = sp;
  return true;
}

// The launch's frames: [mi0, mi1) with the full window (interior and, when the
// buffer starts at stage 0, head frames), then every clipped tail frame with
// its own geometry (FrameGeom, reference decoder.cpp:175-191).
struct SmallPlan {
  SmallParams main;
  bool has_main = false;
  SmallParams tail[4];
  int ntail = 0;
};

template <class C, int R>
bool plan_small(const DecodeLaunch& p, SmallPlan* out) {
  using GEO = Geo<C, R>;
  if (GEO::B != 2 || p.nblocks > 0 || p.sigma || p.frame_list) return false;
  SmallPlan pl;
  const int L = p.f + p.v1 + p.v2;
  const std::int64_t lo = p.llr_stage0 == 0 ? 0 : (p.llr_stage0 + p.v1 + p.f - 1) / p.f;
  if (std::max(lo, p.frame_begin) != p.frame_begin) return false;  // windows before the buffer
  const std::int64_t hi = (p.n - p.f - p.v2 >= 0) ? (p.n - p.f - p.v2) / p.f + 1 : 0;  // full windows below
  const std::int64_t mi1 = std::min<std::int64_t>(hi, p.frame_end);
  if (mi1 > p.frame_begin) {
    if (!plan_geom<C, R>(p, p.frame_begin, mi1, L, p.f, &pl.main)) return false;
    pl.has_main = true;
  }
  for (std::int64_t m = std::max(mi1, p.frame_begin); m < p.frame_end; ++m) {
    if (pl.ntail == 4) return false;
    const FrameGeom g(m, p.n, p.f, p.v1, p.v2, p.f0);
    const std::int64_t ws = m * p.f - p.v1;  // virtual window start (zero-filled below stage 0)
    if (!plan_geom<C, R>(p, m, m + 1, static_cast<int>(g.end - ws), static_cast<int>(g.out_hi - g.out_lo),
                      &pl.tail[pl.ntail]))
      return false;
    ++pl.ntail;
  }
  if (!pl.has_main && pl.ntail == 0) return false;
  *out = pl;
  return true;
}

template <class C, int R>
cudaError_t launch_one(const SmallParams& sp, cudaStream_t stream) {
  using GEO = Geo<C, R>;
  const std::int64_t warps = (sp.mi1 - sp.mi0 + GEO::FPW - 1) / GEO::FPW;
  const std::int64_t blocks = (warps + sp.warps_per_cta - 1) / sp.warps_per_cta;
  const std::size_t smem = static_cast<std::size_t>(sp.smem_per_warp) * sp.warps_per_cta;
  // (always the maximum: host threads launching different geometries at once
  // must not lower the limit under each other's launches)
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(small_kernel<C, R>));
  if (e != cudaSuccess) return e;
  small_kernel<C, R><<<static_cast<unsigned>(blocks), sp.warps_per_cta * 32, smem, stream>>>(sp);
  note_launch();
  return cudaGetLastError();
}

template <class C, int R>
cudaError_t launch_small(const SmallPlan& pl, cudaStream_t stream) {
  // tail frames (one warp each) on a side stream, concurrently with the main launch
  SideStream* side = nullptr;
  if (pl.ntail > 0) {
    side = side_stream();
    if (!side) return cudaErrorUnknown;
    if (cudaError_t err = cudaEventRecord(side->fork, stream); err != cudaSuccess) return err;
    if (cudaError_t err = cudaStreamWaitEvent(side->s, side->fork, 0); err != cudaSuccess) return err;
    for (int i = 0; i < pl.ntail; ++i) {
      if (cudaError_t err = launch_one<C, R>(pl.tail[i], side->s); err != cudaSuccess) return err;
    }
    if (cudaError_t err = cudaEventRecord(side->join, side->s); err != cudaSuccess) return err;
  }
  if (pl.has_main) {
    if (cudaError_t err = launch_one<C, R>(pl.main, stream); err != cudaSuccess) return err;
  }
  if (side) return cudaStreamWaitEvent(stream, side->join, 0);
  return cudaSuccess;
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

bool try_small(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err) {
  SmallPlan pl;
  if (K7a::matches(p.k, p.b, p.polys)) {
    if (!plan_small<K7a, 8>(p, &pl)) return false;
    *err = launch_small<K7a, 8>(pl, stream);
    return true;
  }
  if (K7b::matches(p.k, p.b, p.polys)) {
    if (!plan_small<K7b, 8>(p, &pl)) return false;
    *err = launch_small<K7b, 8>(pl, stream);
    return true;
  }
  return false;
}

}  // namespace fast
}  // namespace vd
