#pragma once
// Small-launch variant of the fast kernel (latency-bound decodes such as the
// reference's own 1 M-bit default, BASELINE C1): 8 states per lane instead of
// 16, so a warp carries 8 frames instead of 16 and a frame's forward pass is
// about half as many instructions per stage on the warp's dependency chain.
//
// Same algorithm and exactness argument as fast_kernel (vd_fast_dev.cuh):
// frame-pair packed offset-binary int16 metrics, packed VIADD.16x2 /
// VIADDMNMX.S16x2 butterflies with ties to the second predecessor
// (reference decoder.cpp:53-76), stored-max argmax with the lowest index on
// ties (decoder.cpp:80-90), subframe traceback (decoder.cpp:214-236). What
// changes with R = 8 (Geo<C, 8>: LB = 3 in-register stages between the
// shared-memory relayouts):
//  * the frames' windows are first copied into shared memory (one
//    cooperative pass), so 6-stage super-blocks (two relayout blocks, 12 LLR
//    bytes per frame) read aligned words without any prefetch bookkeeping;
//  * a lane's 16 decisions per stage (8 registers x 2 frames) are merged by
//    4 PRMT + 4 IMAD into one 32-bit survivor word (bit (reg & 3) +
//    8 (reg >> 2) + 16 half), stored in shared memory (small launches have
//    few warps per SM, so no tensor memory is needed);
//  * the traceback walks 3-stage blocks: within one the traced state's lane
//    is fixed (only register bits change), as in the fast kernel.
// Every frame of a small launch is taken: interior and head frames (window
// clipped at the stream start: the staging reads zeros before stage 0) in one
// launch, each clipped tail frame in a launch of its own geometry (its output
// length f_out and window L, with the start stages clipped to the window as
// decoder.cpp:187-191 does).
#include "vd_fast_dev.cuh"

namespace vd {
namespace fast {

struct SmallParams {
  DecodeLaunch p;
  std::int64_t mi0, mi1;  // frames of this launch
  int L;                  // window length: f + v1 + v2, or a clipped tail frame's
  int f_out;              // output stages per frame (f, or a partial last frame's)
  int nsb;                // 6-stage super-blocks per frame
  int step, num_sub;      // subframe geometry
  int smem_per_warp;      // bytes per warp this geometry needs
  int llr_off, dec_off, x_off, ss_off;  // regions of a warp's area
  int pitch;              // bytes per staged frame row (multiple of 12, >= 12 * nsb)
  std::int64_t safe_stage;      // window start of an interior frame (empty slots)
  std::uint32_t m1;             // -1 from the parameter bank
};

constexpr int kSmallMaxWarps = 8;
constexpr int kSmallSegs = 4;  // frame segments per launch: the full-window frames + up to 3 clipped tail frames

// One launch: segment i (its own window / output geometry) owns the grid's
// warps [warp_begin[i], warp_begin[i + 1]); every warp's area is the largest
// segment's. whole_words: every output word belongs to one traceback task
// (32-aligned frame and subframe boundaries), so the host skips zeroing the
// output and partial last words are stored, not OR-ed.
struct SmallLaunch {
  SmallParams seg[kSmallSegs];
  int warp_begin[kSmallSegs + 1];
  int nseg;
  int warps_per_cta;
  int smem_per_warp;
  int whole_words;
};
constexpr int kSmallMaxStages = 1032;  // largest staged window (f + v1 + v2 rounded up to 6 stages)

// Geometry of the small kernel for R states per lane. Launched with R = 8;
// R = 4 (16 lanes per frame pair, 4 frames per warp) is parity-clean but was
// measured slower on C1 (19.5 vs 25.6 Gbps: the per-lane table and relayout
// work no longer halves, profiles/r02_ab_notes.md).
// Survivor-word layout of SmallGeo<R>: a stage's 2R decisions (R registers x
// 2 frames) are merged by Q = R / 2 PRMTs (registers q and q + Q) and IMADs
// into bit (rho % Q) + Q p + 8 (rho / Q) + 16 half, p = the stage's index
// among the SPW stages that share the word.
template <int R>
struct SmallGeo {
  static constexpr int LB = R == 8 ? 3 : 2;        // in-register stages between relayouts
  static constexpr int SB = LB % 2 ? 2 * LB : LB;  // stages per super-block (whole LLR words at B = 2)
  static constexpr int WSB = SB * 2 / 4;           // LLR words per frame and super-block
  static constexpr int Q = R / 2;                  // PRMTs per stage
  static constexpr int SPW = R == 8 ? 1 : 2;       // stages per survivor word (16 bits used each)
  static_assert(SB % SPW == 0, "survivor words must not straddle super-blocks");
  // bit index of register rho (p = 0), half h
  __device__ static __forceinline__ std::uint32_t bit(std::uint32_t rho, std::uint32_t hsh) {
    return (rho & (Q - 1)) | ((rho / Q) << 3) | hsh;
  }
  // bit of register bit j in that index: j < LB - 1 -> j, the top bit -> 3
  static constexpr std::uint32_t pos(int j) { return j < LB - 1 ? j : 3u; }
  // register index back from a bit index
  __device__ static __forceinline__ std::uint32_t reg(std::uint32_t bx) {
    return (bx & (Q - 1)) | (((bx >> 3) & 1u) << (LB - 1));
  }
};

template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

// acc += y[q] * (0x01010101 << (q + Q ph)) for the Q PRMTs of one stage
template <int Q, int PH, int q = 0>
__device__ __forceinline__ void small_merge(const std::uint32_t* w, std::uint32_t& acc) {
  if constexpr (q < Q) {
    acc = mad_imm<(0x01010101u << (q + Q * PH))>(prmt(w[q], w[q + Q], 0xFBD9u), acc);
    small_merge<Q, PH, q + 1>(w, acc);
  }
}

template <class C, int R_>
__global__ void __launch_bounds__(kSmallMaxWarps * 32, 1) small_kernel(const SmallLaunch sl_) {
  using GEO = Geo<C, R_>;
  using SG = SmallGeo<R_>;
  constexpr int M = GEO::M, S = GEO::S, G = GEO::G, LB = GEO::LB, R = GEO::R, r = GEO::r, g = GEO::g;
  constexpr int B = GEO::B, FPW = GEO::FPW;
  constexpr int SB = SG::SB, WSB = SG::WSB, Q = SG::Q, SPW = SG::SPW;
  static_assert(B == 2, "small kernel: rate-1/2 codes");
  static_assert(LB == SG::LB && (R == 8 || R == 4), "small kernel geometry");
  constexpr std::uint32_t BASE = 0x20002000u;
  constexpr std::uint32_t XM = C::kXM;
  constexpr std::uint32_t CB0 = C::cb(0), CBT = C::cb(C::kK - 1);
  constexpr std::uint32_t OFFB = static_cast<std::uint32_t>(256 * B) * 0x00010001u;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  // (opaque: keeps the lane-derived values in registers instead of
  // re-reading SR_TID inside the stage loop)
  const int lane = static_cast<int>(opaque(threadIdx.x & 31u));
  const int warp = threadIdx.x >> 5;
  const int grp = lane / G;
  const int lam = lane % G;
  unsigned char* wbase = smem_raw + static_cast<std::size_t>(warp) * sl_.smem_per_warp;
  const int gwarp = static_cast<int>(blockIdx.x) * sl_.warps_per_cta + warp;
  int si = 0;
  while (si + 1 < sl_.nseg && gwarp >= sl_.warp_begin[si + 1]) ++si;
  const SmallParams& sp = sl_.seg[si];
  const DecodeLaunch& p = sp.p;
  unsigned char* llr_s = wbase + sp.llr_off;
  std::uint32_t* dec = reinterpret_cast<std::uint32_t*>(wbase + sp.dec_off);
  std::uint32_t* xbuf = reinterpret_cast<std::uint32_t*>(wbase + sp.x_off);
  std::uint16_t* sstate = reinterpret_cast<std::uint16_t*>(wbase + sp.ss_off);

  const std::int64_t mbase = sp.mi0 + static_cast<std::int64_t>(gwarp - sl_.warp_begin[si]) * FPW;
  if (mbase >= sp.mi1) return;

  const int f = static_cast<int>(opaque(static_cast<std::uint32_t>(p.f)));
  const int v1 = static_cast<int>(opaque(static_cast<std::uint32_t>(p.v1)));
  const int v2 = static_cast<int>(opaque(static_cast<std::uint32_t>(p.v2)));
  const int L = static_cast<int>(opaque(static_cast<std::uint32_t>(sp.L)));
  const int nsb = sp.nsb;
  const int num_sub = sp.num_sub;
  const int step = sp.step;
  const int pitch = sp.pitch;

  struct Slot {
    std::int64_t ws, m;  // window start stage (negative for head frames), frame index
  };
  const Slot empty{sp.safe_stage, 0};
  auto frame_slot = [&](std::int64_t mg, bool valid) -> Slot {
    if (!valid) return empty;
    const FrameRef fr = resolve_frame(p, mg);
    return Slot{fr.base + fr.m * p.f - p.v1, fr.m};
  };

  // ---- stage the FPW frames' windows into shared memory (zero past L) -------
  // LPS = 32 / FPW lanes per frame slot, each taking every LPS-th word of its
  // row, 16 words per chunk (40: more registers, a slower stage loop): a
  // chunk's global loads are all issued before its stores (one memory latency
  // per chunk); a window starting on an odd stage
  // (byte offset 2) is re-aligned with one PRMT per word.
  {
    constexpr int kChunk = 16, LPS = 32 / FPW;
    const int fs = lane / LPS, sub = lane % LPS;
    const bool v = mbase + fs < sp.mi1;
    const Slot sl = frame_slot(mbase + fs, v);
    // head frames (window start before stage 0 of the stream) read zeros
    // there: all-zero branch metrics keep every path metric at 0, so the
    // frame's metrics at stage 0 are the reference's clipped start
    // (decoder.cpp:195) and its traceback ends at stage 0 anyway.
    const std::int8_t* llr0 = static_cast<const std::int8_t*>(p.llr);
    const std::int8_t* b8 = llr0 + (sl.ws - p.llr_stage0) * B;
    const int mis = static_cast<int>(reinterpret_cast<std::uintptr_t>(b8) & 3u);  // 0 or 2
    const std::uint32_t* w = reinterpret_cast<const std::uint32_t*>(b8 - mis);
    // first row word at or after the stream start (aligned words never straddle it)
    const int ifirst = sl.ws < 0 ? static_cast<int>((static_cast<std::int64_t>(llr0 - (b8 - mis)) + 3) / 4) : 0;
    const int nw = pitch / 4;  // words of the row
    const int nbytes = L * B;  // window bytes
    // bytes from w[0] to the end of the stream: a word past it is read as its
    // valid lower half only (no read beyond the caller's buffer)
    const std::int64_t avail = (p.n - sl.ws) * B + mis;
    auto ld = [&](int i) -> std::uint32_t {
      const std::int64_t e = 4 * static_cast<std::int64_t>(i) + 4;
      if (e <= avail) return __ldg(w + i);
      return e - 2 <= avail ? static_cast<std::uint32_t>(__ldg(reinterpret_cast<const std::uint16_t*>(w + i))) : 0u;
    };
    std::uint32_t* row = reinterpret_cast<std::uint32_t*>(llr_s + fs * pitch);
    // Common case, uniform over the warp: every window 4-byte aligned and
    // wholly inside the stream -> plain loads, no per-word checks.
    const bool simple = __all_sync(kFull, mis == 0 && sl.ws >= 0 && avail >= 4 * static_cast<std::int64_t>(nw));
    if (simple) {
      for (int c0 = 0; c0 < nw; c0 += LPS * kChunk) {
        std::uint32_t x[kChunk];
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
          const int i = c0 + sub + LPS * j;
          x[j] = i < nw ? __ldg(w + i) : 0u;
        }
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
          const int i = c0 + sub + LPS * j;
          const int nb = nbytes - 4 * i;  // window bytes in this word
          const std::uint32_t v = nb >= 4 ? x[j] : (nb > 0 ? (x[j] & 0xffffu) : 0u);
          if (i < nw) row[i] = v;
        }
      }
    }
    for (int c0 = 0; c0 < (simple ? 0 : nw); c0 += LPS * kChunk) {
      std::uint32_t lo[kChunk], hi[kChunk];
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const int i = c0 + sub + LPS * j;
        lo[j] = (i >= ifirst && 4 * i - mis < nbytes) ? ld(i) : 0u;
        hi[j] = (mis && i + 1 >= ifirst && 4 * i + 2 < nbytes) ? ld(i + 1) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const int i = c0 + sub + LPS * j;
        std::uint32_t x = mis ? prmt(lo[j], hi[j], 0x5432u) : lo[j];
        const int nb = nbytes - 4 * i;  // window bytes in this word
        x = nb >= 4 ? x : (nb > 0 ? (x & 0xffffu) : 0u);
        if (i < nw) row[i] = x;
      }
    }
  }
  __syncwarp();

  // ---- per-lane constants: LLR sign flips of the lane part of the branch
  // index (phase k = stage % LB of each of the super-block's SB stages)
  std::uint32_t fw[WSB];
  std::uint32_t kc[SB][2];
  {
    std::uint32_t w[WSB];
#pragma unroll
    for (int j = 0; j < WSB; ++j) w[j] = 0x80808080u;
#pragma unroll
    for (int k6 = 0; k6 < SB; ++k6) {
      const int k = k6 % LB;
      std::uint32_t z = 0;
#pragma unroll
      for (int i = 0; i < g; ++i) {
        if ((lam >> i) & 1) z ^= C::cb(r + i - k);
      }
      const std::uint32_t phi0 = (z >> 1) & 1u, phi1 = z & 1u;
      const int q0 = k6 * 2, q1 = k6 * 2 + 1;
      if (phi0) w[q0 >> 2] ^= 0xffu << (8 * (q0 & 3));
      if (phi1) w[q1 >> 2] ^= 0xffu << (8 * (q1 & 3));
      kc[k6][0] = opaque((phi0 + phi1) * 0x00010001u);
      kc[k6][1] = opaque((256u + phi0 - phi1) * 0x00010001u);
    }
#pragma unroll
    for (int j = 0; j < WSB; ++j) fw[j] = opaque(w[j]);
  }
  const std::uint32_t m1 = opaque(sp.m1);
  std::uint32_t sig[R];
#pragma unroll
  for (int i = 0; i < R; ++i) sig[i] = BASE;
  std::uint32_t corr = 0u;
  std::int32_t subA = 0, subB = 0;
  (void)subA;
  (void)subB;

  // stored-max start stages (decoder.cpp:187-191, 205-211)
  // (f_out / L: the frame's own output length and window, which a clipped
  // tail frame launch sets below f / f + v1 + v2: decoder.cpp:175-191)
  const int f_out = sp.f_out;
  auto sub_start = [&](int s) { return min(v1 + min((s + 1) * step, f_out) + v2, L) - 1; };
  auto needs_record = [&](int s) { return !(p.f0 > 0 && p.start == 1 && sub_start(s) < L - 1); };
  int next_sub = 0;
  while (next_sub < num_sub && !needs_record(next_sub)) ++next_sub;
  int next_rec = next_sub < num_sub ? sub_start(next_sub) : 0x7fffffff;
  auto rec = [&](int t, int k) {
    if (t != next_rec) return;
    const int sh = (k + 1) % M;
    const std::uint32_t lanepart =
        ((static_cast<std::uint32_t>(lam * R) >> sh) | (static_cast<std::uint32_t>(lam * R) << (M - sh))) & GEO::SMASK;
    std::uint32_t bestA = 0, bestB = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const std::uint32_t regpart = static_cast<std::uint32_t>(GEO::rotr(i, k + 1));
      const std::uint32_t ck = (lanepart | regpart) ^ 0xffffu;
      bestA = max(bestA, prmt(ck, sig[i], 0x5410u));
      bestB = max(bestB, prmt(ck, sig[i], 0x7610u));
    }
#pragma unroll
    for (int o2 = 1; o2 < G; o2 <<= 1) {
      bestA = max(bestA, __shfl_xor_sync(kFull, bestA, o2));
      bestB = max(bestB, __shfl_xor_sync(kFull, bestB, o2));
    }
    do {  // (subframes of a clipped tail frame can share the start stage L - 1)
      if (lam == 0) {
        sstate[(2 * grp) * num_sub + next_sub] = static_cast<std::uint16_t>(0xffffu - (bestA & 0xffffu));
        sstate[(2 * grp + 1) * num_sub + next_sub] = static_cast<std::uint16_t>(0xffffu - (bestB & 0xffffu));
      }
      ++next_sub;
      while (next_sub < num_sub && !needs_record(next_sub)) ++next_sub;
      next_rec = next_sub < num_sub ? sub_start(next_sub) : 0x7fffffff;
    } while (next_rec == t);
  };

  std::uint32_t* const xb = xbuf + opaque(static_cast<std::uint32_t>(grp * GEO::XSTRIDE));
  auto relayout = [&]() {  // back to the canonical layout (P_new = rotr(P_old, r))
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int pn_reg = ((i << g) & (R - 1));
      const int pn_lane = (i << g) >> r;
      xb[(pn_lane + (lam >> r)) * GEO::LSTRIDE + pn_reg + (lam & (R - 1))] = sig[i];
    }
    __syncwarp();
    const uint4* src = reinterpret_cast<const uint4*>(xb + lam * GEO::LSTRIDE);
#pragma unroll
    for (int i = 0; i < R / 4; ++i) {
      const uint4 v = src[i];
      sig[4 * i] = v.x;
      sig[4 * i + 1] = v.y;
      sig[4 * i + 2] = v.z;
      sig[4 * i + 3] = v.w;
    }
    __syncwarp();
  };

  const std::uint32_t* rowA = reinterpret_cast<const std::uint32_t*>(llr_s + (2 * grp) * pitch);
  const std::uint32_t* rowB = reinterpret_cast<const std::uint32_t*>(llr_s + (2 * grp + 1) * pitch);
  // Survivor rows (one word per SPW stages): every stage of the super-blocks
  // that hold a stage >= v1 (from stage t_first = SB * floor(v1 / SB)), so the
  // stores need no range checks (the traceback reads only stages in [v1, L),
  // decoder.cpp:229-235).
  const int sb_warm = v1 / SB;  // super-blocks entirely before stage v1
  const int t_first = SB * sb_warm;
  std::uint32_t* const drow = dec + lane - (t_first / SPW) * 32;

  // One SB-stage super-block, straight-line: STORE keeps decision words; REC
  // checks every stage for a stored-max start stage (only the super-blocks
  // that hold one).
  auto super_block = [&](int sb, auto store_tag, auto rec_tag) {
    constexpr bool STORE = decltype(store_tag)::value;
    constexpr bool REC = decltype(rec_tag)::value;
    // tables of the SB stages for both frames (reference decoder.cpp:22-51):
    // PT[k][x] = T_k[x ^ lane part] + 256 per half
    std::uint32_t il[WSB][2];
#pragma unroll
    for (int j = 0; j < WSB; ++j) {
      const std::uint32_t a = rowA[sb * WSB + j] ^ fw[j];
      const std::uint32_t bq = rowB[sb * WSB + j] ^ fw[j];
      il[j][0] = prmt(a, bq, 0x5410u);
      il[j][1] = prmt(a, bq, 0x7632u);
    }
    std::uint32_t PT[SB][4];
#pragma unroll
    for (int k6 = 0; k6 < SB; ++k6) {
      const int q0 = k6 * 2, q1 = k6 * 2 + 1;
      const std::uint32_t x0 = prmt(il[q0 >> 2][(q0 >> 1) & 1], 0u, (q0 & 1) ? 0x4341u : 0x4240u);
      const std::uint32_t x1 = prmt(il[q1 >> 2][(q1 >> 1) & 1], 0u, (q1 & 1) ? 0x4341u : 0x4240u);
      PT[k6][0] = x0 + x1 + kc[k6][0];
      PT[k6][1] = x0 - x1 + kc[k6][1];
      PT[k6][XM ^ 0] = mad_u32(PT[k6][0], m1, OFFB);
      PT[k6][XM ^ 1] = mad_u32(PT[k6][1], m1, OFFB);
    }
    std::uint32_t PA0[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) PA0[x] = __vadd2(PT[0][x], corr);  // renormalisation, folded
    std::uint32_t acc = 0u;  // survivor word being merged (SPW stages)
    static_for<0, SB>([&](auto k6c) {
      constexpr int k6 = decltype(k6c)::value;
      constexpr int k = k6 % LB;
      const int t = sb * SB + k6;
      auto pa = [&](std::uint32_t x) { return k6 == 0 ? PA0[x] : PT[k6][x]; };
      std::uint32_t w[R];
      (void)t;
      (void)w;
#pragma unroll
      for (int e = 0; e < R; ++e) {
        if ((e >> k) & 1) continue;
        const int od = e | (1 << k);
        const std::uint32_t x = GEO::xreg(k, e);
        const std::uint32_t sE = sig[e], sO = sig[od];
        const std::uint32_t s2L = __vadd2(sO, pa(x ^ CB0));  // edge labels: see run_block
        const std::uint32_t s2H = __vadd2(sO, pa(x ^ CB0 ^ CBT));
        const std::uint32_t nL = __viaddmax_s16x2(sE, pa(x), s2L);
        const std::uint32_t nH = __viaddmax_s16x2(sE, pa(x ^ CBT), s2H);
        if constexpr (STORE) {
          w[e] = nL - s2L + 0x7fff7fffu;  // bit 15 / 31: the first predecessor won
          w[od] = nH - s2H + 0x7fff7fffu;
        }
        sig[e] = nL;
        sig[od] = nH;
      }
      if constexpr (STORE) {
        // 2R decisions -> the word's Q bits of this stage (see compact16):
        // y[q] = 255 * N_q, merged at bit q + Q p of each byte
        constexpr int ph = k6 % SPW;
        if constexpr (ph == 0) acc = m1;
        small_merge<Q, ph>(w, acc);
        if constexpr (ph == SPW - 1) drow[(t / SPW) * 32] = acc;
      }
      if constexpr (REC) rec(t, k);
      if constexpr (k == LB - 1) relayout();
    });
    // renormalisation after every super-block (group-wide reference)
    const std::uint32_t ref = __shfl_sync(kFull, sig[0], grp * G);
    corr = __vsub2(BASE, ref);
  };
  using F = std::integral_constant<bool, false>;
  using T = std::integral_constant<bool, true>;
  int sb = 0;
  for (; sb < sb_warm; ++sb) super_block(sb, F{}, F{});  // (start stages are >= v1)
  for (; sb < nsb; ++sb) {
    if (next_rec < 6 * sb + 6) {
      super_block(sb, T{}, T{});
    } else {
      super_block(sb, T{}, F{});
    }
  }
  __syncwarp();

  // ---- subframe traceback (decoder.cpp:214-236) ------------------------------
  // Tasks (frame slot, subframe) over the lanes; each lane walks its own range
  // (the survivor words are per-lane shared-memory loads, so no warp-uniform
  // loop is needed). Within a 3-stage block the traced state's lane is fixed;
  // its register index rho is tracked as the survivor-word bit index
  // B = (rho & 3) | ((rho & 4) << 1) | 16 half, so a step is a funnel shift
  // (bit B -> bit pos(j)) and a bit select, pos = {0, 1, 3}. The decoded bit of
  // stage tb0 + j is register bit j at block entry (as in the fast kernel).
  const int ntask = FPW * num_sub;
  for (int base = 0; base < ntask; base += 32) {
    const int task = base + lane;
    if (task >= ntask) break;
    const int fr = task % FPW;
    const int s = task / FPW;
    const int half = fr & 1;
    const bool valid = mbase + fr < sp.mi1;
    const Slot sl = frame_slot(mbase + fr, valid);
    const int st_t = sub_start(s);
    const int sub_lo = v1 + s * step;
    const int sub_hi = v1 + min((s + 1) * step, f_out);
    std::uint32_t state;
    if (p.f0 > 0 && p.start == 1 && st_t < L - 1) {
      state = static_cast<std::uint32_t>(mix_seed(p.seed, static_cast<std::uint64_t>(sl.m) * 0x10001ull +
                                                              static_cast<std::uint64_t>(s)) %
                                         static_cast<std::uint64_t>(S));
    } else {
      state = sstate[fr * num_sub + s];
    }
    const int sh = st_t % LB + 1;
    const std::uint32_t P0 = ((state << sh) | (state >> (M - sh))) & GEO::SMASK;
    const std::uint32_t hsh = half ? 16u : 0u;
    std::uint32_t lp = P0 >> r;
    std::uint32_t Bx = SG::bit(P0 & (R - 1), hsh);
    // word of stage t: dcol[(t / SPW) * 32 + lp], its bits at + Q (t % SPW)
    const std::uint32_t* dcol = dec + (fr >> 1) * G - (t_first / SPW) * 32;
    const std::int64_t obase = sl.ws - p.out_stage0;
    std::uint64_t acc = 0;  // emitted bits, lowest stage at bit 0
    int nb = 0;
    auto emit = [&](int t0, int n, std::uint32_t bits) {  // stages t0 .. t0 + n - 1
      acc = (acc << n) | bits;
      nb += n;
      if (nb >= 32) {
        const std::uint32_t word = static_cast<std::uint32_t>(acc >> (nb - 32));
        const std::int64_t ol = obase + t0 + (nb - 32);
        const std::int64_t w0 = ol >> 5;
        const int o = static_cast<int>(ol & 31);
        if (valid) {
          if (o == 0) {
            p.out[w0] = word;
          } else {
            atomicOr(p.out + w0, word << o);
            atomicOr(p.out + w0 + 1, word >> (32 - o));
          }
        }
        nb -= 32;
      }
    };
    // register bits of the bit index at block entry -> decoded bits of the block
    auto block_bits = [](std::uint32_t bx) { return SG::reg(bx); };
    // the relayout undone: P -> rotl(P, r) for the block below
    auto next_block = [&]() {
      const std::uint32_t P = (lp << r) | block_bits(Bx);
      const std::uint32_t Pn = ((P << r) | (P >> (M - r))) & GEO::SMASK;
      lp = Pn >> r;
      Bx = SG::bit(Pn & (R - 1), hsh);
    };
    // one step at phase j of a block (blocks start at multiples of LB, so the
    // stage's position in its survivor word is j % SPW)
    auto step_j = [&](std::uint32_t word, int j) {
      const std::uint32_t pos = SG::pos(j);
      const std::uint32_t x = __funnelshift_r(word, word, Bx + Q * (j % SPW) - pos);  // bit -> bit pos
      Bx = bitsel_m(x, Bx, 1u << pos);
    };
    int tb0 = st_t - st_t % LB;
    // top block: phases st_t % LB .. max(sub_lo - tb0, 0)
    {
      const int jhi = st_t - tb0, jlo = max(sub_lo - tb0, 0);
      const std::uint32_t bin = block_bits(Bx);
#pragma unroll
      for (int j = LB - 1; j >= 0; --j) {
        if (j <= jhi && j >= jlo) step_j(dcol[((tb0 + j) / SPW) * 32 + lp], j);
      }
      const int ehi = min(jhi, sub_hi - 1 - tb0);
      if (ehi >= jlo) emit(tb0 + jlo, ehi - jlo + 1, (bin >> jlo) & ((1u << (ehi - jlo + 1)) - 1u));
      next_block();
      tb0 -= LB;
    }
    // whole blocks above sub_lo
    for (; tb0 >= sub_lo; tb0 -= LB) {
      const std::uint32_t* src = dcol + (tb0 / SPW) * 32 + lp;
      std::uint32_t wd[LB];
#pragma unroll
      for (int j = 0; j < LB; ++j) wd[j] = src[(j / SPW) * 32];
      const std::uint32_t bin = block_bits(Bx);
#pragma unroll
      for (int j = LB - 1; j >= 0; --j) step_j(wd[j], j);
      if (tb0 + LB <= sub_hi) {
        emit(tb0, LB, bin);
      } else if (tb0 < sub_hi) {
        const int n = sub_hi - tb0;
        emit(tb0, n, bin & ((1u << n) - 1u));
      }
      next_block();
    }
    // bottom block (sub_lo inside it)
    if (tb0 + LB > sub_lo) {
      const int jlo = sub_lo - tb0;
      const std::uint32_t bin = block_bits(Bx);
      const int ehi = min(LB - 1, sub_hi - 1 - tb0);
      if (ehi >= jlo) emit(sub_lo, ehi - jlo + 1, (bin >> jlo) & ((1u << (ehi - jlo + 1)) - 1u));
    }
    if (nb > 0 && valid) {
      const std::uint32_t word = static_cast<std::uint32_t>(acc) & ((nb == 32) ? 0xffffffffu : ((1u << nb) - 1u));
      const std::int64_t ol = obase + sub_lo;
      const std::int64_t w0 = ol >> 5;
      const int o = static_cast<int>(ol & 31);
      if (o == 0 && sl_.whole_words) {
        p.out[w0] = word;  // the stream's last, partial word: ours alone
      } else {
        atomicOr(p.out + w0, word << o);
        if (o + nb > 32) atomicOr(p.out + w0 + 1, word >> (32 - o));
      }
    }
  }
}

}  // namespace fast
}  // namespace vd
