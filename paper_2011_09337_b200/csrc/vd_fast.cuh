#pragma once
// Host half of the fast kernel: dispatch over the precompiled codes, launch
// planning (survivor-store layout, warps per CTA) and the launch itself. The
// kernel template is in vd_fast_dev.cuh; instantiations in vd_fast_k*.cu, and
// run-time (NVRTC) instantiations for other codes in vd_jit.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>

#include "vd_fast_dev.cuh"
#include "vd_internal.h"

namespace vd {
namespace fast {

// ---- dispatch ----------------------------------------------------------------

template <class C, int R>
struct Variant {
  using GEO = Geo<C, R>;
  static bool matches(const DecodeLaunch& p) { return C::matches(p.k, p.b, p.polys); }
};

using K7a = Code2<7, 0171, 0133>;
using K7b = Code2<7, 0133, 0171>;
using K9a = Code2<9, 0561, 0753>;
using K9b = Code2<9, 0753, 0561>;
using K5a = Code2<5, 023, 035>;
using K6a = Code2<6, 053, 075>;
using K8a = Code2<8, 0247, 0371>;
using K9c = Code3<9, 0557, 0663, 0711>;  // UMTS / 3GPP rate 1/3
using K7c = Code3<7, 0133, 0171, 0165>;  // LTE rate 1/3
static_assert(K7a::sym() && K7b::sym() && K9a::sym() && K9b::sym() && K5a::sym() && K6a::sym() && K8a::sym() &&
                  K7c::sym() && K9c::sym(),
              "fast-path codes must tap the newest and oldest register bits");

constexpr int kMaxWarpsSmem = 8;   // smem-only survivor store
constexpr int kSmemMax = 232448;   // sm_100 max dynamic shared memory per CTA
constexpr int kHeader = 16;        // CTA header: TMEM base address

// Per-(host thread, device) side stream + fork/join events for the edge-frame
// launches (re-entrant: every host thread has its own).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

inline SideStream* side_stream() {
  struct Cache {
    std::map<int, SideStream> m;
    ~Cache() {
      for (auto& kv : m) {
        if (cudaSetDevice(kv.first) != cudaSuccess) continue;
        cudaEventDestroy(kv.second.fork);
        cudaEventDestroy(kv.second.join);
        cudaStreamDestroy(kv.second.s);
      }
    }
  };
  thread_local Cache cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  auto it = cache.m.find(dev);
  if (it != cache.m.end()) return &it->second;
  SideStream ss;
  if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  if (cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
  if (cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) return nullptr;
  return &(cache.m[dev] = ss);
}

// Small-launch kernel (vd_small.cu): a single-round launch's edge frames, and
// the partial last round of a multi-round launch.
bool small_launch_wanted(const DecodeLaunch& p);
bool try_small(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err);
bool small_can_take(const DecodeLaunch& p);  // plan only: one round of the small kernel

struct Plan {
  FastParams fp;
  std::size_t smem;
  bool tm, gl;
};

template <class C, int R, class PN = NoPunct>
bool plan(const DecodeLaunch& p, Plan* out, bool pad_head = false) {
  using GEO = Geo<C, R>;
  if (PN::kActive && (GEO::B != 2 || pad_head || p.nblocks > 0 || p.llr_stage0 != 0 || p.sigma)) return false;
  if (PN::kActive && 2 * GEO::FPW > 32) return false;  // fills: two lanes per frame slot
  FastParams fp{};
  fp.llr_head = p.llr_head;
  fp.head_pitch = p.head_pitch;
  fp.p = p;
  fp.m1 = 0xffffffffu;
  fp.L = p.f + p.v1 + p.v2;
  fp.nblk = (fp.L + GEO::LB - 1) / GEO::LB;
  fp.step = p.f0 > 0 ? p.f0 : p.f;
  fp.num_sub = (p.f + fp.step - 1) / fp.step;
  if (fp.num_sub > 64) return false;
  if (fp.L < 2 * GEO::LB) return false;  // the first two blocks are loaded unclamped
  // Interior frames: full window, 4-byte aligned LLRs, prefetch in bounds.
  constexpr int B = GEO::B;
  if ((static_cast<std::int64_t>(p.f) * B) % 4 != 0 || (static_cast<std::int64_t>(p.v1) * B) % 4 != 0) return false;
  if ((p.llr_stage0 * B) % 4 != 0) return false;
  if (p.nblocks > 0) {
    // Batched: the caller launches every global frame and marks the interior
    // ones per block (blk_ilo / blk_ihi); edge frames go to the generic kernel.
    fp.mi0 = p.frame_begin;
    fp.mi1 = p.frame_end;
    fp.safe_stage = p.safe_stage;
    if (p.sigma) return false;
  } else {
  // stages read per frame: the window rounded up to whole blocks, plus the
  // two-block prefetch overrun; fused depuncture: whole 24-stage chunks of
  // blocks 0 .. nblk + 1, plus the fill's 6-word read slack (<= 24 stages)
  const std::int64_t span = PN::kActive ? static_cast<std::int64_t>((fp.nblk + 1) / 6 + 1) * 24 + 24
                                        : static_cast<std::int64_t>(fp.nblk) * GEO::LB + 2 * GEO::LB;
  std::int64_t lo = pad_head ? p.frame_begin : (p.v1 + p.f - 1) / p.f;  // first m with m*f >= v1 (or padded head)
  std::int64_t hi_excl = (p.n - p.f - p.v2 >= 0) ? (p.n - p.f - p.v2) / p.f + 1 : 0;  // m*f + f + v2 <= n
  // the caller guarantees LLRs up to the window end of the last launched frame
  const std::int64_t avail = std::min<std::int64_t>(p.frame_end * static_cast<std::int64_t>(p.f) + p.v2, p.n);
  const std::int64_t hi2 = (avail + p.v1 - span >= 0) ? (avail + p.v1 - span) / p.f + 1 : 0;  // m*f - v1 + span <= avail
  if (hi2 < hi_excl) hi_excl = hi2;
  fp.mi0 = lo > p.frame_begin ? lo : p.frame_begin;
  fp.mi1 = hi_excl < p.frame_end ? hi_excl : p.frame_end;
  if (fp.mi1 - fp.mi0 < GEO::FPW) return false;  // not worth it
  // also the llr window must start at or before the first interior frame's beg
  if (!pad_head && p.llr_stage0 > fp.mi0 * p.f - p.v1) return false;
  fp.safe_stage = fp.mi0 * p.f - p.v1;
  }
  const int x_bytes = GEO::g > 0 ? GEO::GROUPS * GEO::XSTRIDE * 4 : 0;
  const int ss_bytes = (((GEO::FPW * fp.num_sub * 2) + 15) & ~15) + (PN::kActive ? 2 * GEO::FPW * 48 : 0);
  auto layout = [&](int smem_rows) {
    const int dec_bytes = smem_rows * 32 * 4;
    fp.smem_rows = smem_rows;
    fp.dec_off = 0;
    fp.x_off = dec_bytes;
    fp.ss_off = dec_bytes + x_bytes;
    fp.stg_off = fp.ss_off + (((GEO::FPW * fp.num_sub * 2) + 15) & ~15);  // staging ring after the start states
    fp.smem_per_warp = (dec_bytes + x_bytes + ss_bytes + 15) & ~15;
  };
  // Tensor-memory survivor store: W warps per CTA (W/4 per TMEM lane quarter)
  // share `alloc` columns. Large launches take 12 warps / 512 columns (one CTA
  // and 12 warps per SM); small launches spread over more SMs.
  const std::int64_t warps_needed = (fp.mi1 - fp.mi0 + GEO::FPW - 1) / GEO::FPW;
  struct Cand {
    int w, alloc;
  };
  const Cand cands[] = {{12, 512}, {8, 512}, {4, 256}};
  fp.t_gl = fp.L;  // no global rows unless a spill layout is chosen below
  fp.g_rows = 0;
  fp.gscratch = nullptr;
  // TMEM + smem rows for candidate c; with `spill`, the rows that do not fit in
  // shared memory go to global scratch (stages [t_gl, L), t_gl % 4 == 0).
  // Test hook: VITDEC_SPILL_ROWS=N caps the shared-memory rows at N and forces
  // the spill layout, so small parity tests exercise the global tier.
  const char* env_rows = std::getenv("VITDEC_SPILL_ROWS");
  const int cap_rows = env_rows ? std::atoi(env_rows) : -1;
  auto try_cand = [&](const Cand& c, bool spill) {
    fp.tm_alloc = c.alloc;
    fp.tcols = ((c.alloc / (c.w / 4)) & ~3);
    fp.t_first = p.v1 & ~3;
    fp.t_split = fp.t_first + fp.tcols;
    fp.s_base = fp.t_split;
    fp.t_gl = fp.L;
    fp.g_rows = 0;
    layout(std::max(fp.L - fp.t_split, 0) + 1);
    const bool fits = kHeader + static_cast<std::size_t>(fp.smem_per_warp) * c.w <= static_cast<std::size_t>(kSmemMax);
    if (fits && (cap_rows < 0 || fp.L - fp.t_split <= cap_rows)) return true;
    if (!spill) return false;
    const int budget = (kSmemMax - kHeader) / c.w - x_bytes - ss_bytes - 16;  // bytes of smem rows per warp
    int rows = budget / 128 - 1;                                               // minus the dummy row
    if (cap_rows >= 0) rows = std::min(rows, cap_rows);
    if (rows < 0) return false;
    fp.t_gl = std::max(fp.t_split, (fp.t_split + rows) & ~3);
    if (fp.t_gl >= fp.L) return false;
    fp.g_rows = fp.L - fp.t_gl + 4;  // + 4 rows of padding: the general traceback reads whole blocks
    layout(fp.t_gl - fp.t_split + 1);
    return kHeader + static_cast<std::size_t>(fp.smem_per_warp) * c.w <= static_cast<std::size_t>(kSmemMax);
  };
  bool ok = false;
  // Large launches: 12 warps per SM, TMEM + smem rows, and global rows for
  // what does not fit (prefer the spill tier to fewer resident warps)
  if (warps_needed >= 12 * 148 || cap_rows >= 0) {
    ok = try_cand(cands[0], true);
    fp.warps_per_cta = 12;
  }
  // Smaller launches: the fewest warps per CTA that still hold every frame
  // group in one round (the runtime keeps one TMEM kernel CTA per SM:
  // cudaOccupancyMaxActiveBlocksPerMultiprocessor = 1 even for 4-warp CTAs),
  // which also leaves shared memory beside it for the edge frames' launch.
  const std::int64_t sms = sm_count();
  for (int i = 2; i >= 0 && !ok; --i) {  // 4, 8, 12 warps
    const Cand& c = cands[i];
    if (i > 0 && warps_needed > static_cast<std::int64_t>(c.w) * sms) continue;  // would need more rounds
    if (try_cand(c, false)) {
      fp.warps_per_cta = c.w;
      ok = true;
    }
  }
  if (!ok) {
    // Long frames: 12 (or fewer for small launches) warps with TMEM + smem + global rows.
    for (int i = 2; i >= 0 && !ok; --i) {
      const Cand& c = cands[i];
      if (i > 0 && warps_needed > static_cast<std::int64_t>(c.w) * sms) continue;
      if (try_cand(c, true)) {
        fp.warps_per_cta = c.w;
        ok = true;
      }
    }
  }
  if (ok) out->tm = true;
  out->gl = ok && fp.g_rows > 0;
  if (!ok) {
    // Long frames: shared memory only, as many warps as fit.
    fp.tcols = 0;
    fp.tm_alloc = 0;
    fp.t_first = fp.t_split = fp.s_base = p.v1;
    fp.t_gl = fp.L;
    fp.g_rows = 0;
    layout(p.f + p.v2 + 1);
    const int w = (kSmemMax - kHeader) / fp.smem_per_warp;
    if (w < 1) return false;
    fp.warps_per_cta = std::min(w, kMaxWarpsSmem);
    out->tm = false;
  }
  out->fp = fp;
  out->smem = kHeader + static_cast<std::size_t>(fp.smem_per_warp) * fp.warps_per_cta;
  return true;
}

// Kernel of code C for a plan's survivor-store layout (TMEM, global spill
// tier): the precompiled instantiations.
template <class C, int R>
struct Precompiled {
  const void* operator()(bool tm, bool gl, cudaError_t*) const {
    return !tm ? reinterpret_cast<const void*>(fast_kernel<C, R, false, false>)
               : gl ? reinterpret_cast<const void*>(fast_kernel<C, R, true, true>)
                    : reinterpret_cast<const void*>(fast_kernel<C, R, true, false>);
  }
};

template <class C, int R, class KSel = Precompiled<C, R>>
cudaError_t launch_variant(const DecodeLaunch& p, cudaStream_t stream, KSel ksel = KSel()) {
  using GEO = Geo<C, R>;
  Plan pl;
  // Head frames on the fast path via a zero-padded copy of the stream head
  // (exact, see FastParams::llr_head); otherwise they go to the generic kernel.
  const std::int64_t head_end = std::min<std::int64_t>((p.v1 + p.f - 1) / p.f, p.frame_end);
  bool pad = p.nblocks == 0 && p.llr_stage0 == 0 && p.frame_begin < head_end &&
             plan<C, R>(p, &pl, true) && pl.fp.mi0 == p.frame_begin && pl.fp.mi1 >= head_end;
  if (!pad && !plan<C, R>(p, &pl)) return cudaErrorNotSupported;
  cudaError_t ek = cudaSuccess;
  const void* kern = ksel(pl.tm, pl.gl, &ek);  // before any launch: a JIT failure launches nothing
  if (!kern) return ek != cudaSuccess ? ek : cudaErrorInvalidSource;
  std::int8_t* head_buf = nullptr;
  if (pad) {
    constexpr int B = GEO::B;
    const std::int64_t stages = head_end * p.f + p.v2;  // window end of the last head frame (<= n: mi1 >= head_end)
    if (cudaError_t e = retain_async_pool(); e != cudaSuccess) return e;
    // (+16 bytes: the last LLR word of a window may extend past the window's last stage)
    if (cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&head_buf), (p.v1 + stages + kPfSlackStages) * B + 16,
                                        stream);
        e != cudaSuccess)
      return e;
    if (cudaError_t e = cudaMemsetAsync(head_buf, 0, static_cast<std::size_t>(p.v1) * B, stream); e != cudaSuccess)
      return e;
    if (cudaError_t e = cudaMemcpyAsync(head_buf + p.v1 * B, p.llr, stages * B, cudaMemcpyDeviceToDevice, stream);
        e != cudaSuccess)
      return e;
    pl.fp.llr_head = head_buf;
  }
  const FastParams& fp = pl.fp;
  const std::int64_t warps = (fp.mi1 - fp.mi0 + GEO::FPW - 1) / GEO::FPW;
  std::int64_t blocks = (warps + fp.warps_per_cta - 1) / fp.warps_per_cta;
  // (always the maximum: host threads launching different plans at once must
  // not lower the limit under each other's launches)
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return e;
  // persistent grid: as many CTAs as are co-resident (one per SM with TMEM)
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fp.warps_per_cta * 32, pl.smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  const std::int64_t resident = static_cast<std::int64_t>(sm_count()) * per_sm;
  // Edge frames (clipped windows) run on a side stream, concurrently with the
  // fast kernel. Generic kernel (one warp per frame, fits beside the fast
  // kernel's CTAs; ~100 us for a 296-stage window) by default; when the fast
  // launch is a single round of partly filled CTAs (mid-size decodes, where
  // that latency would be the critical path) the small-launch kernel (~30 us)
  // takes them instead, beside it.
  // Multi-round launches whose last round would hold only a few frame groups
  // (on a few SMs, at the full per-round time): those groups and the tail
  // edge frames go to one small-kernel launch after the fast kernel instead
  // (2^23 stages: 2048 groups = 1776 + 272, see profiles/r02_ab_notes.md).
  std::int64_t mi1_fast = fp.mi1;
  DecodeLaunch rest = p;
  bool small_rest = false;
  if (p.nblocks == 0 && blocks > resident) {
    const std::int64_t slots = resident * fp.warps_per_cta;
    const std::int64_t r = warps % slots;
    rest.frame_begin = fp.mi0 + (warps - r) * GEO::FPW;
    if (r > 0 && small_can_take(rest)) {
      small_rest = true;
      mi1_fast = rest.frame_begin;
    }
  }
  const bool edges = p.nblocks == 0 && (fp.mi0 > p.frame_begin || (!small_rest && fp.mi1 < p.frame_end));
  const bool small_edges = blocks <= resident && fp.warps_per_cta < 12;
  SideStream* side = nullptr;
  if (edges) {
    side = side_stream();
    if (!side) return cudaErrorUnknown;
    if (cudaError_t err = cudaEventRecord(side->fork, stream); err != cudaSuccess) return err;
    if (cudaError_t err = cudaStreamWaitEvent(side->s, side->fork, 0); err != cudaSuccess) return err;
  }
  auto edge = [&](const DecodeLaunch& ed) {
    cudaError_t err = cudaSuccess;
    if (small_edges && small_launch_wanted(ed) && try_small(ed, side->s, &err)) return err;
    return launch_generic_i8(ed, side->s);
  };
  if (edges && fp.mi0 > p.frame_begin) {
    DecodeLaunch ed = p;
    ed.frame_end = fp.mi0;
    if (cudaError_t err = edge(ed); err != cudaSuccess) return err;
  }
  if (edges && !small_rest && fp.mi1 < p.frame_end) {
    DecodeLaunch ed = p;
    ed.frame_begin = fp.mi1;
    if (p.sigma) ed.sigma = static_cast<std::int64_t*>(p.sigma) + (fp.mi1 - p.frame_begin) * p.s;
    if (cudaError_t err = edge(ed); err != cudaSuccess) return err;
  }
  if (edges) {
    if (cudaError_t err = cudaEventRecord(side->join, side->s); err != cudaSuccess) return err;
  }
  FastParams fpl = fp;
  fpl.mi1 = mi1_fast;
  blocks = std::min<std::int64_t>(blocks, resident);
  if (fp.g_rows > 0) {
    // stream-ordered scratch for the spilled survivor rows (the pool keeps it
    // cached across launches, see retain_async_pool())
    const std::size_t bytes = static_cast<std::size_t>(blocks) * fp.warps_per_cta * fp.g_rows * 32 * 4;
    if (cudaError_t ea = retain_async_pool(); ea != cudaSuccess) return ea;
    if (cudaError_t ea = cudaMallocAsync(reinterpret_cast<void**>(&fpl.gscratch), bytes, stream); ea != cudaSuccess)
      return ea;
  }
  void* args[] = {&fpl};
  e = cudaLaunchKernel(kern, dim3(static_cast<unsigned>(blocks)), dim3(fp.warps_per_cta * 32), args, pl.smem, stream);
  note_launch();
  if (fpl.gscratch) {
    const cudaError_t ef = cudaFreeAsync(fpl.gscratch, stream);
    if (e == cudaSuccess) e = ef;
  }
  if (head_buf) {
    const cudaError_t ef = cudaFreeAsync(head_buf, stream);
    if (e == cudaSuccess) e = ef;
  }
  if (e == cudaSuccess && small_rest && !try_small(rest, stream, &e)) e = cudaErrorNotSupported;
  if (e == cudaSuccess && edges) e = cudaStreamWaitEvent(stream, side->join, 0);
  return e;
}

template <class C, int R>
bool try_variant(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err) {
  if (!C::matches(p.k, p.b, p.polys)) return false;
  Plan pl;
  if (!plan<C, R>(p, &pl)) return false;
  if (err) *err = launch_variant<C, R>(p, stream);
  return true;
}

/// Fused-depuncture launch: p.llr is the PUNCTURED stream (pattern PN, stage
/// 0 at byte 0); the fast kernel decodes the interior frames [*mi0, *mi1)
/// it can take, the caller decodes the rest from a dense copy. Returns false
/// (nothing launched) when the plan needs more than TMEM + shared memory.
// Fused-depuncture launch of code class C's plan with the kernel kfn(&err)
// returns (precompiled or run-time instantiated).
template <class C, int R, class PN, class KFn>
bool try_punct_with(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, std::int64_t* mi0,
                    std::int64_t* mi1, KFn kfn) {
  using GEO = Geo<C, R>;
  if (p.f % PN::P || p.v1 % PN::P || p.v2 % PN::P) return false;
  Plan pl;
  if (!plan<C, R, PN>(p, &pl) || !pl.tm || pl.gl) return false;
  *mi0 = pl.fp.mi0;
  *mi1 = pl.fp.mi1;
  if (!stream && !err) return true;  // probe
  const FastParams& fp = pl.fp;
  cudaError_t e = cudaSuccess;
  const void* kern = kfn(&e);
  if (!kern) {
    *err = e != cudaSuccess ? e : cudaErrorInvalidSource;
    return true;
  }
  e = allow_max_smem(kern);
  if (e == cudaSuccess) {
    const std::int64_t warps = (fp.mi1 - fp.mi0 + GEO::FPW - 1) / GEO::FPW;
    std::int64_t blocks = (warps + fp.warps_per_cta - 1) / fp.warps_per_cta;
    blocks = std::min<std::int64_t>(blocks, static_cast<std::int64_t>(sm_count()));
    FastParams fpl = fp;
    void* args[] = {&fpl};
    e = cudaLaunchKernel(kern, dim3(static_cast<unsigned>(blocks)), dim3(fp.warps_per_cta * 32), args, pl.smem, stream);
    note_launch();
  }
  *err = e;
  return true;
}

template <class C, int R, class PN>
bool try_punct_variant(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err, std::int64_t* mi0,
                       std::int64_t* mi1) {
  if (!C::matches(p.k, p.b, p.polys)) return false;
  return try_punct_with<C, R, PN>(p, stream, err, mi0, mi1, [](cudaError_t*) {
    return reinterpret_cast<const void*>(fast_kernel<C, R, true, false, PN>);
  });
}

}  // namespace fast
}  // namespace vd
