// Register-resident unified Viterbi kernel for sm_100a (the throughput path).
//
// One kernel per launch does, for every frame (reference decode_frame,
// decoder.cpp:170-237): forward add-compare-select over the frame window,
// stored-max argmax at every subframe start stage, bit-packed survivor
// decisions in shared memory, and the subframe-parallel traceback, writing
// only bit-packed decoded bits to HBM. Frames whose window is clipped by the
// stream ends (the first and last few) are left to the generic kernel.
//
// Data layout:
//  * FRAME-PAIR PACKING: every 32-bit register holds the 16-bit path metric of
//    the SAME trellis state for two frames (lo = frame A, hi = frame B), so the
//    packed VIADD.16x2 / VIADDMNMX.S16x2 instructions advance two frames at
//    once and a butterfly's branch metrics are plain table entries.
//  * A lane group of G = S / R lanes owns a frame pair; each lane holds R
//    registers = R states. The physical index P = lane * R + reg of a state
//    is a rotation of its state index: after k stages of a block,
//    P = rotl_{K-1}(state, k). In-place butterflies (E/O registers -> NL/NH)
//    keep every stage inside a lane for LB = log2(R) stages; one shared-memory
//    relayout (STS.32 x R + LDS.128 x R/4 per lane) then restores the
//    canonical layout, so the code for a block of LB stages repeats forever.
//  * Path metrics are offset-binary int16 (kept in [~4k, ~16k] by a group-wide
//    renormalisation every 2 blocks), which lets one 32-bit IADD3 produce both
//    halves' decision bits: w = sigma_O - sigma_E + C has bit 15 / 31 set iff
//    the second predecessor wins, ties included (reference decoder.cpp:67-74).
//  * Decision bits are gathered with PRMT sign-replication + LOP3 merges into
//    one 32-bit word per lane per stage (32 decisions) and stored to shared
//    memory: (f + v2) stages x 32 lanes x 4 B per warp.
//  * The lane-dependent part of every butterfly's branch index is folded into
//    per-lane LLR sign flips, so all table selections are compile-time.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "vd_common.cuh"
#include "vd_internal.h"

namespace vd {
namespace fast {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t s) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

/// Rate-1/2 code with compile-time generator polynomials.
template <int K_, std::uint32_t P0, std::uint32_t P1>
struct Code2 {
  static constexpr int kK = K_;
  static constexpr int kB = 2;
  // Branch-index bits contributed by register bit q (poly 0 -> MSB of the
  // index, as reference trellis.cpp:70-73 packs branch outputs).
  static constexpr std::uint32_t cb(int q) { return (((P0 >> q) & 1u) << 1) | ((P1 >> q) & 1u); }
  static constexpr bool sym() { return cb(0) == 3u && cb(K_ - 1) == 3u; }
  static constexpr bool matches(int k, int b, const std::uint32_t* p) {
    return k == K_ && b == 2 && p[0] == P0 && p[1] == P1;
  }
};

template <class C, int R_>
struct Geo {
  static constexpr int M = C::kK - 1;
  static constexpr int S = 1 << M;
  static constexpr int R = R_;
  static constexpr int r = ilog2(R);
  static constexpr int g = M - r;
  static constexpr int G = 1 << g;
  static constexpr int LB = r;            // stages per block
  static constexpr int GROUPS = 32 / G;   // lane groups (frame pairs) per warp
  static constexpr int FPW = 2 * GROUPS;  // frames per warp
  static constexpr std::uint32_t SMASK = S - 1;
  static constexpr int XSTRIDE = S + 4;   // relayout buffer words per group (bank padding)
  static_assert(R <= S && R >= 4 && (R & (R - 1)) == 0, "R must be a power of two in [4, S]");
  static_assert(G <= 32, "at most one frame pair per 32 lanes");
  static_assert(R % 4 == 0, "relayout reads use 128-bit loads");

  static constexpr int rotl(int v, int s) {
    s = ((s % M) + M) % M;
    return s == 0 ? v : (((v << s) | (v >> (M - s))) & static_cast<int>(SMASK));
  }
  static constexpr int rotr(int v, int s) { return rotl(v, M - (s % M)); }

  /// Register part of the branch index of the butterfly whose E register is
  /// rho (bit k clear) at block phase k: XOR over the other register bits c of
  /// cb(state position of c), state position = (c - k) mod M.
  static constexpr std::uint32_t xreg(int k, int rho) {
    std::uint32_t x = 0;
    for (int c = 0; c < r; ++c) {
      if (c != k && ((rho >> c) & 1)) x ^= C::cb(((c - k) % M + M) % M);
    }
    return x;
  }
  /// Lane part at phase k for lane-in-group lam.
  static constexpr std::uint32_t xlane(int k, int lam) {
    std::uint32_t x = 0;
    for (int i = 0; i < g; ++i) {
      if ((lam >> i) & 1) x ^= C::cb(r + i - k);
    }
    return x;
  }
};

struct FastParams {
  DecodeLaunch p;
  std::int64_t mi0, mi1;  // interior frames handled by this launch
  int L;                  // frame window length f + v1 + v2
  int nblk;               // blocks per frame (ceil(L / LB))
  int step, num_sub;      // subframe geometry
  int warps_per_cta;
  int smem_per_warp;      // bytes
  int dec_off, x_off, ss_off;  // byte offsets of the regions inside a warp's area
};

// Opaque copy: keeps a per-lane constant in a register instead of letting the
// compiler rematerialise it from threadIdx every block.
__device__ __forceinline__ std::uint32_t opaque(std::uint32_t x) {
  asm volatile("" : "+r"(x));
  return x;
}

// (a & m) | (b & ~m) as one LOP3 that the compiler cannot re-associate into a
// serial chain (keeps the decision-compaction tree 3 deep).
template <std::uint32_t MASK>
__device__ __forceinline__ std::uint32_t bitsel(std::uint32_t a, std::uint32_t b) {
  std::uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "n"(MASK));  // 0xE4: c ? a : b
  return r;
}

// 32 decisions (16 registers x 2 frames) -> one word, bit (rho + 16 * half).
__device__ __forceinline__ std::uint32_t compact16(const std::uint32_t* w) {
  std::uint32_t y[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) y[q] = prmt(w[q], w[q + 8], 0xFBD9u);
  const std::uint32_t a = bitsel<0x01010101u>(y[0], y[1]);
  const std::uint32_t b = bitsel<0x04040404u>(y[2], y[3]);
  const std::uint32_t c = bitsel<0x10101010u>(y[4], y[5]);
  const std::uint32_t d = bitsel<0x40404040u>(y[6], y[7]);
  const std::uint32_t ab = bitsel<0x03030303u>(a, b);
  const std::uint32_t cd = bitsel<0x30303030u>(c, d);
  return bitsel<0x0f0f0f0fu>(ab, cd);
}

template <class GEO>
struct FrameState {
  std::uint32_t sig[GEO::R];
  std::uint32_t wv[2][GEO::R];
  std::uint32_t fm[GEO::LB], k0[GEO::LB], k1[GEO::LB];  // per-lane LLR flip constants per phase
  std::uint32_t cur[2][GEO::LB / 2];                     // LLR words of this block (frame A, B)
  std::uint32_t nxt[2][GEO::LB / 2];                     // and of the next block
};

struct BlockCtx {
  int v1, L;
  std::uint32_t* drow_lane;  // dec + lane
  int dummy_row;             // row index receiving out-of-range decision words
};

// One block of LB stages. SLOW adds the per-stage range checks and the
// stored-max argmax hook; FAST blocks (fully inside the stored range, no
// argmax) are straight-line code.
template <class C, class GEO, bool SLOW, class RecFn>
__device__ __forceinline__ void run_block(FrameState<GEO>& st, int blk, const BlockCtx& bc, int& tprev, RecFn&& rec) {
  constexpr int LB = GEO::LB, R = GEO::R;
  constexpr std::uint32_t BIAS = 0x80008000u;
  constexpr std::uint32_t OFF2 = 0x02000200u;
  // ---- branch-metric tables for the LB stages of this block (both frames) ---
  std::uint32_t PT[LB][4], CL[LB][4];
#pragma unroll
  for (int k = 0; k < LB; ++k) {
    const std::uint32_t wA = st.cur[0][k >> 1], wB = st.cur[1][k >> 1];
    const std::uint32_t o = (k & 1) * 2;
    const std::uint32_t sel = o | ((o + 1) << 4) | ((o + 4) << 8) | ((o + 5) << 12);
    const std::uint32_t tmp = prmt(wA, wB, sel) ^ st.fm[k];
    const std::uint32_t X = prmt(tmp, 0u, 0x4240u);  // (L0A, L0B) offset-binary, zero-extended
    const std::uint32_t Y = prmt(tmp, 0u, 0x4341u);  // (L1A, L1B)
    PT[k][0] = X + Y + st.k0[k];                     // T0 + 256 = l0 + l1 + 256
    PT[k][1] = X + (Y ^ 0x00ff00ffu) + st.k1[k];     // T1 + 256 = l0 - l1 + 256
    PT[k][3] = OFF2 - PT[k][0];                      // T3 = -T0
    PT[k][2] = OFF2 - PT[k][1];                      // T2 = -T1
#pragma unroll
    for (int x = 0; x < 4; ++x) CL[k][x] = PT[k][x ^ 3] - PT[k][x] + BIAS;
  }
#pragma unroll
  for (int k = 0; k < LB; ++k) {
    const int t = blk * LB + k;
    std::uint32_t* w = st.wv[k & 1];
    // ---- add-compare-select, in place: E/O registers differ in bit k -------
#pragma unroll
    for (int e = 0; e < R; ++e) {
      if ((e >> k) & 1) continue;
      const int od = e | (1 << k);
      const std::uint32_t x = GEO::xreg(k, e);
      const std::uint32_t sE = st.sig[e], sO = st.sig[od];
      const std::uint32_t s2L = __vadd2(sO, PT[k][x ^ 3]);
      const std::uint32_t s2H = __vadd2(sO, PT[k][x]);
      w[e] = sO - sE + CL[k][x];
      w[od] = sO - sE + CL[k][x ^ 3];
      st.sig[e] = __viaddmax_s16x2(sE, PT[k][x], s2L);
      st.sig[od] = __viaddmax_s16x2(sE, PT[k][x ^ 3], s2H);
    }
    // ---- previous stage's decisions -> shared memory (overlaps this ACS) ---
    const std::uint32_t word = compact16(st.wv[(k + 1) & 1]);
    if constexpr (SLOW) {
      const int row = (tprev >= bc.v1 && tprev < bc.L) ? tprev - bc.v1 : bc.dummy_row;
      bc.drow_lane[row * 32] = word;
      tprev = t;
      rec(t, k);
    } else {
      bc.drow_lane[(t - 1 - bc.v1) * 32] = word;
    }
  }
  if constexpr (!SLOW) tprev = blk * LB + LB - 1;
}

template <class C, int R>
__global__ void __launch_bounds__(256) fast_kernel(const FastParams fp) {
  using GEO = Geo<C, R>;
  constexpr int M = GEO::M, S = GEO::S, G = GEO::G, LB = GEO::LB, r = GEO::r, g = GEO::g;
  constexpr std::uint32_t BASE = 0x20002000u;  // offset-binary metric origin (8192 per half)
  constexpr int WPB = LB / 2;
  static_assert(LB % 2 == 0, "B=2 fast path needs an even block length");
  static_assert(R == 16, "one 32-bit decision word per lane per stage");
  const DecodeLaunch& p = fp.p;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int grp = lane / G;
  const int lam = lane % G;
  unsigned char* wbase = smem_raw + static_cast<std::size_t>(warp) * fp.smem_per_warp;
  std::uint32_t* dec = reinterpret_cast<std::uint32_t*>(wbase + fp.dec_off);
  std::uint32_t* xbuf = reinterpret_cast<std::uint32_t*>(wbase + fp.x_off);
  std::uint16_t* sstate = reinterpret_cast<std::uint16_t*>(wbase + fp.ss_off);

  const std::int64_t gwarp = static_cast<std::int64_t>(blockIdx.x) * fp.warps_per_cta + warp;
  const std::int64_t mbase = fp.mi0 + gwarp * GEO::FPW;
  if (mbase >= fp.mi1) return;  // whole warp idle (uniform)
  const std::int64_t mA = mbase + 2 * grp, mB = mA + 1;
  const bool validA = mA < fp.mi1, validB = mB < fp.mi1;
  const std::int64_t lA = validA ? mA : fp.mi0, lB = validB ? mB : fp.mi0;  // clamp loads

  const int f = p.f, v1 = p.v1, v2 = p.v2, L = fp.L;
  // Frame-relative LLR word pointers (frame start is 4-byte aligned: checked at launch).
  const std::uint32_t* llrA = reinterpret_cast<const std::uint32_t*>(static_cast<const std::int8_t*>(p.llr) +
                                                                     (lA * f - v1 - p.llr_stage0) * 2);
  const std::uint32_t* llrB = reinterpret_cast<const std::uint32_t*>(static_cast<const std::int8_t*>(p.llr) +
                                                                     (lB * f - v1 - p.llr_stage0) * 2);

  FrameState<GEO> st;
  // Per-phase flip constants for this lane (lane part of the branch index).
#pragma unroll
  for (int k = 0; k < LB; ++k) {
    std::uint32_t z = 0;
#pragma unroll
    for (int i = 0; i < g; ++i) {
      if ((lam >> i) & 1) z ^= C::cb(r + i - k);
    }
    const std::uint32_t f0b = (z >> 1) & 1u, f1b = z & 1u;  // flip l0 / flip l1
    st.fm[k] = opaque(0x80808080u ^ (f0b ? 0x00ff00ffu : 0u) ^ (f1b ? 0xff00ff00u : 0u));
    st.k0[k] = opaque((f0b + f1b) * 0x00010001u);
    st.k1[k] = opaque((f0b + 1u - f1b) * 0x00010001u);
  }
#pragma unroll
  for (int i = 0; i < R; ++i) st.sig[i] = BASE;
#pragma unroll
  for (int i = 0; i < R; ++i) st.wv[1][i] = 0u;
  std::int32_t subA = 0, subB = 0;  // accumulated renormalisation (ref - BASE) per half

#pragma unroll
  for (int i = 0; i < WPB; ++i) {
    st.cur[0][i] = __ldg(llrA + i);
    st.cur[1][i] = __ldg(llrB + i);
    st.nxt[0][i] = __ldg(llrA + WPB + i);
    st.nxt[1][i] = __ldg(llrB + WPB + i);
  }
  const std::uint32_t* pfA = llrA + 2 * WPB;
  const std::uint32_t* pfB = llrB + 2 * WPB;

  int next_sub = 0;
  // subframes whose traceback starts from the stored max state
  auto sub_start = [&](int s) { return v1 + min((s + 1) * fp.step, f) + v2 - 1; };
  auto needs_record = [&](int s) {
    const int sst = sub_start(s);
    return !(p.f0 > 0 && p.start == 1 && sst < L - 1);
  };
  while (next_sub < fp.num_sub && !needs_record(next_sub)) ++next_sub;
  int next_rec = next_sub < fp.num_sub ? sub_start(next_sub) : 0x7fffffff;

  // stored-max argmax at start stages (decoder.cpp:205-211)
  auto rec = [&](int t, int k) {
    if (t != next_rec) return;
    // key = (metric << 16) | (0xFFFF - state): max -> best metric, lowest state.
    const int sh = (k + 1) % M;
    const std::uint32_t lanepart =
        ((static_cast<std::uint32_t>(lam * R) >> sh) | (static_cast<std::uint32_t>(lam * R) << (M - sh))) &
        GEO::SMASK;
    std::uint32_t bestA = 0, bestB = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const std::uint32_t regpart = static_cast<std::uint32_t>(GEO::rotr(i, k + 1));
      const std::uint32_t ck = (lanepart | regpart) ^ 0xffffu;
      bestA = max(bestA, prmt(ck, st.sig[i], 0x5410u));
      bestB = max(bestB, prmt(ck, st.sig[i], 0x7610u));
    }
#pragma unroll
    for (int o2 = 1; o2 < G; o2 <<= 1) {
      bestA = max(bestA, __shfl_xor_sync(kFull, bestA, o2));
      bestB = max(bestB, __shfl_xor_sync(kFull, bestB, o2));
    }
    if (lam == 0) {
      sstate[(2 * grp) * fp.num_sub + next_sub] = static_cast<std::uint16_t>(0xffffu - (bestA & 0xffffu));
      sstate[(2 * grp + 1) * fp.num_sub + next_sub] = static_cast<std::uint16_t>(0xffffu - (bestB & 0xffffu));
    }
    if (t == L - 1 && p.sigma != nullptr) {
      // final metrics: true = stored - BASE - 256 * L + sum(ref - BASE)
      std::int64_t* sg = static_cast<std::int64_t*>(p.sigma);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int sidx = static_cast<int>(lanepart | static_cast<std::uint32_t>(GEO::rotr(i, k + 1)));
        const std::int64_t a = static_cast<std::int64_t>(st.sig[i] & 0xffffu) - 8192 - 256LL * L + subA;
        const std::int64_t b = static_cast<std::int64_t>(st.sig[i] >> 16) - 8192 - 256LL * L + subB;
        if (validA) sg[(mA - p.frame_begin) * S + sidx] = a;
        if (validB) sg[(mB - p.frame_begin) * S + sidx] = b;
      }
    }
    ++next_sub;
    while (next_sub < fp.num_sub && !needs_record(next_sub)) ++next_sub;
    next_rec = next_sub < fp.num_sub ? sub_start(next_sub) : 0x7fffffff;
  };

  BlockCtx bc;
  bc.v1 = v1;
  bc.L = L;
  bc.drow_lane = dec + lane;
  bc.dummy_row = f + v2;  // one spare row after the stored range
  int tprev = -1;

  for (int blk = 0; blk < fp.nblk; ++blk) {
    const int t0 = blk * LB;
    // fast block: every pending store (stages t0-1 .. t0+LB-2) is in range and
    // no start stage falls inside the block
    const bool fast = (t0 - 1 >= v1) && (t0 + LB - 2 < L) && !(next_rec >= t0 && next_rec < t0 + LB);
    if (fast) {
      run_block<C, GEO, false>(st, blk, bc, tprev, rec);
    } else {
      run_block<C, GEO, true>(st, blk, bc, tprev, rec);
    }
    // ---- LLR pipeline: advance one block, prefetch the block after next ----
#pragma unroll
    for (int i = 0; i < WPB; ++i) {
      st.cur[0][i] = st.nxt[0][i];
      st.cur[1][i] = st.nxt[1][i];
      st.nxt[0][i] = __ldg(pfA + i);
      st.nxt[1][i] = __ldg(pfB + i);
    }
    pfA += WPB;
    pfB += WPB;
    // ---- renormalisation every 2 blocks (group-wide reference) ------------
    if (blk & 1) {
      const std::uint32_t ref = __shfl_sync(kFull, st.sig[0], grp * G);
      subA += static_cast<std::int32_t>(ref & 0xffffu) - 8192;
      subB += static_cast<std::int32_t>(ref >> 16) - 8192;
#pragma unroll
      for (int i = 0; i < R; ++i) st.sig[i] = st.sig[i] - ref + BASE;
    }
    // ---- relayout: back to the canonical layout (P_new = rotr(P_old, r)) --
    if constexpr (g > 0) {
      std::uint32_t* xb = xbuf + grp * GEO::XSTRIDE;
#pragma unroll
      for (int i = 0; i < R; ++i) xb[(i << g) | lam] = st.sig[i];
      __syncwarp();
      const uint4* src = reinterpret_cast<const uint4*>(xb + lam * R);
#pragma unroll
      for (int i = 0; i < R / 4; ++i) {
        const uint4 v = src[i];
        st.sig[4 * i] = v.x;
        st.sig[4 * i + 1] = v.y;
        st.sig[4 * i + 2] = v.z;
        st.sig[4 * i + 3] = v.w;
      }
      __syncwarp();
    }
  }
  // decisions of the last processed stage
  {
    const std::uint32_t word = compact16(st.wv[(fp.nblk * LB - 1) & 1]);
    const int row = (tprev >= v1 && tprev < L) ? tprev - v1 : bc.dummy_row;
    bc.drow_lane[row * 32] = word;
  }
  __syncwarp();

  // ---- subframe-parallel traceback (decoder.cpp:214-236) --------------------
  // Tasks (frame, subframe) are spread over all 32 lanes of the warp, frames
  // fastest: in a round every lane traces one task, reading any group's
  // decision words from shared memory. Within a block of LB stages the lane
  // index of the traced state (P >> r) is fixed (only register bits are
  // rewritten), so the block's words are fetched together: one shared-memory
  // latency per LB steps, and the per-step work is branch-free.
  const int ntask = GEO::FPW * fp.num_sub;
  for (int task = lane; task - lane < ntask; task += 32) {
    const bool active = task < ntask;
    const int fr = active ? task % GEO::FPW : 0;  // frame slot in the warp (2 * group + half)
    const int s = active ? task / GEO::FPW : 0;
    const int half = fr & 1;
    const std::int64_t m = mbase + fr;
    const bool valid = active && m < fp.mi1;
    const int st = sub_start(s);
    const int sub_lo = v1 + s * fp.step;
    const int sub_hi = v1 + min((s + 1) * fp.step, f);
    std::uint32_t state;
    if (p.f0 > 0 && p.start == 1 && st < L - 1) {
      state = static_cast<std::uint32_t>(mix_seed(p.seed, static_cast<std::uint64_t>(m) * 0x10001ull +
                                                              static_cast<std::uint64_t>(s)) %
                                         static_cast<std::uint64_t>(S));
    } else {
      state = sstate[fr * fp.num_sub + s];
    }
    // physical index after stage st (phase st % LB): rotl(state, phase + 1)
    const int sh = ((st & (LB - 1)) + 1) % M;
    std::uint32_t P = sh == 0 ? state : (((state << sh) | (state >> (M - sh))) & GEO::SMASK);
    const std::uint32_t hsh = half ? 16u : 0u;
    const std::uint32_t* gdec = dec + (fr >> 1) * G;  // this frame's group columns
    const std::int64_t obase = m * f - v1 - p.out_stage0;  // output bit index of frame-relative stage 0
    std::uint32_t acc = 0;
    int nb = 0;
    int t = st;
    while (t >= sub_lo) {
      const int tb0 = t & ~(LB - 1);
      const std::uint32_t lp = P >> r;
      std::uint32_t wd[LB];
#pragma unroll
      for (int j = 0; j < LB; ++j) {
        const int row = max(tb0 + j - v1, 0);
        wd[j] = gdec[row * 32 + lp];
      }
#pragma unroll
      for (int j = LB - 1; j >= 0; --j) {
        const int sj = tb0 + j;
        const bool in = sj <= t && sj >= sub_lo;
        const std::uint32_t dbit = (wd[j] >> ((P & (R - 1)) | hsh)) & 1u;
        const bool em = in && sj < sub_hi;
        const std::uint32_t ob = (P >> j) & 1u;
        acc = em ? ((acc << 1) | ob) : acc;
        nb += em ? 1 : 0;
        const std::uint32_t Pn = (P & ~(1u << j)) | (dbit << j);
        P = in ? Pn : P;
        if (nb == 32) {
          const std::int64_t ol = obase + sj;  // lowest output index held in acc
          const std::int64_t w0 = ol >> 5;
          const int o = static_cast<int>(ol & 31);
          if (valid) {
            if (o == 0) {
              p.out[w0] = acc;
            } else {
              atomicOr(p.out + w0, acc << o);
              atomicOr(p.out + w0 + 1, acc >> (32 - o));
            }
          }
          acc = 0;
          nb = 0;
        }
      }
      if (tb0 >= sub_lo) P = ((P << r) | (P >> (M - r))) & GEO::SMASK;  // undo the block relayout
      t = tb0 - 1;
    }
    if (nb > 0 && valid) {
      const std::int64_t ol = obase + sub_lo;
      const std::int64_t w0 = ol >> 5;
      const int o = static_cast<int>(ol & 31);
      atomicOr(p.out + w0, acc << o);
      if (o + nb > 32) atomicOr(p.out + w0 + 1, acc >> (32 - o));
    }
  }
}

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
static_assert(K7a::sym() && K7b::sym() && K9a::sym() && K9b::sym() && K5a::sym() && K6a::sym() && K8a::sym(),
              "fast-path codes must tap the newest and oldest register bits");

constexpr int kWarpsPerCta = 4;
constexpr int kMaxWarpsPerCta = 8;
constexpr int kSmemMax = 232448;  // sm_100 max dynamic shared memory per CTA

struct Plan {
  FastParams fp;
  std::size_t smem;
};

template <class C, int R>
bool plan(const DecodeLaunch& p, Plan* out) {
  using GEO = Geo<C, R>;
  FastParams fp{};
  fp.p = p;
  fp.L = p.f + p.v1 + p.v2;
  fp.nblk = (fp.L + GEO::LB - 1) / GEO::LB;
  fp.step = p.f0 > 0 ? p.f0 : p.f;
  fp.num_sub = (p.f + fp.step - 1) / fp.step;
  if (fp.num_sub > 64) return false;
  // Interior frames: full window, 4-byte aligned LLRs, prefetch in bounds.
  if ((static_cast<std::int64_t>(p.f) * 2) % 4 != 0 || (static_cast<std::int64_t>(p.v1) * 2) % 4 != 0) return false;
  if ((p.llr_stage0 * 2) % 4 != 0) return false;
  const std::int64_t span = static_cast<std::int64_t>(fp.nblk + 2) * GEO::LB;  // stages read per frame
  std::int64_t lo = (p.v1 + p.f - 1) / p.f;                                    // first m with m*f >= v1
  std::int64_t hi_excl = (p.n - p.f - p.v2 >= 0) ? (p.n - p.f - p.v2) / p.f + 1 : 0;  // m*f + f + v2 <= n
  // the caller guarantees LLRs up to the window end of the last launched frame
  const std::int64_t avail = std::min<std::int64_t>(p.frame_end * static_cast<std::int64_t>(p.f) + p.v2, p.n);
  const std::int64_t hi2 = (avail + p.v1 - span >= 0) ? (avail + p.v1 - span) / p.f + 1 : 0;  // m*f - v1 + span <= avail
  if (hi2 < hi_excl) hi_excl = hi2;
  fp.mi0 = lo > p.frame_begin ? lo : p.frame_begin;
  fp.mi1 = hi_excl < p.frame_end ? hi_excl : p.frame_end;
  if (fp.mi1 - fp.mi0 < GEO::FPW) return false;  // not worth it
  // also the llr window must start at or before the first interior frame's beg
  if (p.llr_stage0 > fp.mi0 * p.f - p.v1) return false;
  fp.warps_per_cta = kWarpsPerCta;  // refined below from the shared-memory footprint
  const int dec_bytes = (p.f + p.v2 + 1) * (R / 16 > 0 ? R / 16 : 1) * 32 * 4;  // + dummy row
  const int x_bytes = GEO::g > 0 ? GEO::GROUPS * GEO::XSTRIDE * 4 : 0;
  const int ss_bytes = ((GEO::FPW * fp.num_sub * 2) + 15) & ~15;
  fp.dec_off = 0;
  fp.x_off = dec_bytes;
  fp.ss_off = dec_bytes + x_bytes;
  fp.smem_per_warp = (dec_bytes + x_bytes + ss_bytes + 15) & ~15;
  // As many warps per CTA as fit in the 227 KB opt-in shared memory (one CTA
  // per SM when the decision store is large), at most 8.
  int w = kSmemMax / fp.smem_per_warp;
  if (w < 1) return false;
  fp.warps_per_cta = w < kMaxWarpsPerCta ? w : kMaxWarpsPerCta;
  out->fp = fp;
  out->smem = static_cast<std::size_t>(fp.smem_per_warp) * fp.warps_per_cta;
  return true;
}

template <class C, int R>
cudaError_t launch_variant(const DecodeLaunch& p, cudaStream_t stream) {
  using GEO = Geo<C, R>;
  Plan pl;
  if (!plan<C, R>(p, &pl)) return cudaErrorNotSupported;
  const FastParams& fp = pl.fp;
  // Edge frames (clipped windows) go to the generic kernel, on the same stream.
  if (fp.mi0 > p.frame_begin) {
    DecodeLaunch e = p;
    e.frame_end = fp.mi0;
    if (cudaError_t err = launch_generic_i8(e, stream); err != cudaSuccess) return err;
  }
  if (fp.mi1 < p.frame_end) {
    DecodeLaunch e = p;
    e.frame_begin = fp.mi1;
    if (p.sigma) e.sigma = static_cast<std::int64_t*>(p.sigma) + (fp.mi1 - p.frame_begin) * p.s;
    if (cudaError_t err = launch_generic_i8(e, stream); err != cudaSuccess) return err;
  }
  if (p.sigma && fp.mi0 > p.frame_begin) {
    // the head launch above wrote sigma for frames [frame_begin, mi0) at offset 0 (correct)
  }
  const std::int64_t warps = (fp.mi1 - fp.mi0 + GEO::FPW - 1) / GEO::FPW;
  const std::int64_t blocks = (warps + fp.warps_per_cta - 1) / fp.warps_per_cta;
  auto kern = fast_kernel<C, R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(pl.smem));
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(blocks), fp.warps_per_cta * 32, pl.smem, stream>>>(fp);
  return cudaGetLastError();
}

template <class C, int R>
bool try_variant(const DecodeLaunch& p, cudaStream_t stream, cudaError_t* err) {
  if (!C::matches(p.k, p.b, p.polys)) return false;
  Plan pl;
  if (!plan<C, R>(p, &pl)) return false;
  if (err) *err = launch_variant<C, R>(p, stream);
  return true;
}

}  // namespace fast

bool fast_path_supported(const DecodeLaunch& p) {
  using namespace fast;
  if (p.b != 2) return false;
  Plan pl;
  if (K7a::matches(p.k, p.b, p.polys)) return plan<K7a, 16>(p, &pl);
  if (K7b::matches(p.k, p.b, p.polys)) return plan<K7b, 16>(p, &pl);
  if (K9a::matches(p.k, p.b, p.polys)) return plan<K9a, 16>(p, &pl);
  if (K9b::matches(p.k, p.b, p.polys)) return plan<K9b, 16>(p, &pl);
  if (K5a::matches(p.k, p.b, p.polys)) return plan<K5a, 16>(p, &pl);
  if (K6a::matches(p.k, p.b, p.polys)) return plan<K6a, 16>(p, &pl);
  if (K8a::matches(p.k, p.b, p.polys)) return plan<K8a, 16>(p, &pl);
  return false;
}

cudaError_t launch_fast_i8(const DecodeLaunch& p, cudaStream_t stream) {
  using namespace fast;
  cudaError_t err = cudaErrorNotSupported;
  if (try_variant<K7a, 16>(p, stream, &err)) return err;
  if (try_variant<K7b, 16>(p, stream, &err)) return err;
  if (try_variant<K9a, 16>(p, stream, &err)) return err;
  if (try_variant<K9b, 16>(p, stream, &err)) return err;
  if (try_variant<K5a, 16>(p, stream, &err)) return err;
  if (try_variant<K6a, 16>(p, stream, &err)) return err;
  if (try_variant<K8a, 16>(p, stream, &err)) return err;
  return cudaErrorNotSupported;
}

}  // namespace vd
