#pragma once
// Register-resident unified Viterbi kernel for sm_100a (the throughput path).
// Device half (this file): code traits, geometry and the kernel template. It
// is compiled by nvcc (vd_fast_k*.cu instantiations) and, for codes outside
// the precompiled list, at run time by NVRTC (vd_jit.cu), so it includes
// nothing but vd_std.h / vd_common.cuh / vd_launch.h. Host planning and
// dispatch: vd_fast.cuh.
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
//  * Path metrics are offset-binary int16 (kept in [~4k, ~21k] by a group-wide
//    renormalisation every 4 blocks), which lets one 32-bit IADD3 produce both
//    halves' decision bits: w = sigma_O - sigma_E + C has bit 15 / 31 set iff
//    the second predecessor wins, ties included (reference decoder.cpp:67-74).
//  * Decision bits are gathered with PRMT sign-replication + IMAD merges into
//    one 32-bit word per lane per stage (32 decisions) and stored to tensor /
//    shared memory: (f + v2) stages x 32 lanes x 4 B per warp.
//  * The lane-dependent part of every butterfly's branch index is folded into
//    per-lane LLR sign flips, so all table selections are compile-time.
#include "vd_std.h"
#include "vd_common.cuh"
#include "vd_launch.h"

namespace vd {
namespace fast {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t s) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

/// Rate-1/B code (B = 2, 3 or 4) with compile-time generator polynomials.
template <int K_, int B_, std::uint32_t P0, std::uint32_t P1, std::uint32_t P2 = 0, std::uint32_t P3 = 0>
struct CodeB {
  static constexpr int kK = K_;
  static constexpr int kB = B_;
  static constexpr std::uint32_t kXM = (1u << B_) - 1u;  // complement mask of a branch index
  static constexpr std::uint32_t poly(int i) { return i == 0 ? P0 : i == 1 ? P1 : i == 2 ? P2 : P3; }
  // Branch-index bits contributed by register bit q (poly 0 -> MSB of the
  // index, as reference trellis.cpp:70-73 packs branch outputs).
  static constexpr std::uint32_t cb(int q) {
    std::uint32_t x = 0;
    for (int i = 0; i < B_; ++i) x |= ((poly(i) >> q) & 1u) << (B_ - 1 - i);
    return x;
  }
  static constexpr bool sym() { return cb(0) == kXM && cb(K_ - 1) == kXM; }
  static constexpr bool matches(int k, int b, const std::uint32_t* p) {
    if (k != K_ || b != B_) return false;
    for (int i = 0; i < B_; ++i) {
      if (p[i] != poly(i)) return false;
    }
    return true;
  }
};
template <int K_, std::uint32_t P0, std::uint32_t P1>
using Code2 = CodeB<K_, 2, P0, P1>;
template <int K_, std::uint32_t P0, std::uint32_t P1, std::uint32_t P2>
using Code3 = CodeB<K_, 3, P0, P1, P2>;

/// Puncture pattern of a B = 2 mother code for the fused-depuncture kernel
/// (reference PuncturePattern, codec.hpp:13-33, codec.cpp:57-71): period P
/// stages, KEPT bit (col * 2 + row) set when LLR (row, col) is transmitted
/// (the reference's column-major mask[col * b + row] order). The kernel
/// re-inserts the punctured zeros while it stages the LLR stream into shared
/// memory (reference depuncture, decoder.cpp:131-163), one lane per 12 stages
/// of a frame: every task starts at a stage that is a multiple of P (frames
/// are period-aligned, decoder.cpp:14-19), so the byte gather is a
/// compile-time PRMT pattern plus a runtime byte alignment.
template <int P_, std::uint32_t KEPT_>
struct Punct {
  static constexpr bool kActive = true;
  static constexpr int P = P_;
  static constexpr std::uint32_t KEPT = KEPT_;
  static constexpr int kTaskStages = 12;  // stages per fill task (6 output words)
  static_assert(kTaskStages % P == 0, "a fill task must cover whole periods");
  static constexpr bool kept(int col, int row) { return ((KEPT >> (col * 2 + row)) & 1u) != 0; }
  static constexpr int kept_per_period() {
    int k = 0;
    for (int c = 0; c < P; ++c) k += kept(c, 0) + kept(c, 1);
    return k;
  }
  static constexpr int task_bytes() { return kept_per_period() * (kTaskStages / P); }
  /// Source byte (relative to the task's first transmitted byte) of output
  /// byte j of output word i (stage 2i + j/2, row j%2), or -1 if punctured.
  static constexpr int src(int i, int j) {
    const int t = 2 * i + j / 2, row = j % 2;
    if (!kept(t % P, row)) return -1;
    int n = 0;
    for (int q = 0; q < 2 * t + row; ++q) n += kept((q / 2) % P, q % 2);
    return n;
  }
  static constexpr int lo_src(int i) {
    int m = 1 << 20;
    for (int j = 0; j < 4; ++j) m = (src(i, j) >= 0 && src(i, j) < m) ? src(i, j) : m;
    return m;
  }
  /// PRMT over (u[lo_src / 4], u[lo_src / 4 + 1]) and the byte keep-mask.
  static constexpr std::uint32_t sel(int i) {
    std::uint32_t s = 0;
    const int a = (lo_src(i) / 4) * 4;
    for (int j = 0; j < 4; ++j) s |= static_cast<std::uint32_t>(src(i, j) >= 0 ? src(i, j) - a : 0) << (4 * j);
    return s;
  }
  static constexpr std::uint32_t mask(int i) {
    std::uint32_t m = 0;
    for (int j = 0; j < 4; ++j) m |= (src(i, j) >= 0 ? 0xffu : 0u) << (8 * j);
    return m;
  }
  /// The gather of one fill task's 6 output words as one constant-evaluated
  /// table (called from device code, the functions above were left to run
  /// time for P = 3: ~360 uniform-datapath instructions per block).
  struct Gather {
    int word[6];
    std::uint32_t sel[6], mask[6];
  };
  static constexpr Gather gather() {
    Gather g{};
    for (int i = 0; i < 6; ++i) {
      g.word[i] = lo_src(i) / 4;
      g.sel[i] = sel(i);
      g.mask[i] = mask(i);
    }
    return g;
  }
};
struct NoPunct {
  static constexpr bool kActive = false;
  static constexpr int P = 1;
};
using PunctR23 = Punct<2, 0x07>;  // "11;10"  (reference PuncturePattern::named("r23"))
using PunctR34 = Punct<3, 0x27>;  // "110;101" (named("r34"))
static_assert(PunctR23::task_bytes() == 18 && PunctR34::task_bytes() == 16, "pattern tables");
static_assert(PunctR23::sel(1) == 0x0543u && PunctR23::mask(1) == 0x00ffffffu, "r2/3 gather");
static_assert(PunctR34::mask(1) == 0xffffff00u && PunctR34::mask(2) == 0xff0000ffu, "r3/4 gather");

template <class C, int R_>
struct Geo {
  static constexpr int M = C::kK - 1;
  static constexpr int S = 1 << M;
  static constexpr int R = R_;
  static constexpr int r = ilog2(R);
  static constexpr int g = M - r;
  static constexpr int G = 1 << g;
  static constexpr int LB = r;            // stages per block
  static constexpr int B = C::kB;
  static constexpr int WPB = LB * B / 4;  // LLR words per frame per block (4 stages x B bytes)
  static constexpr int NT = 1 << (B - 1); // direct branch-table entries per stage
  static constexpr int GROUPS = 32 / G;   // lane groups (frame pairs) per warp
  static constexpr int FPW = 2 * GROUPS;  // frames per warp
  static constexpr std::uint32_t SMASK = S - 1;
  // Relayout buffer: new-layout slot (lane', reg') at lane' * LSTRIDE + reg';
  // the 4-word lane pitch and a group pitch = 20 (mod 32) words spread both
  // the per-register STS.32 and the LDS.128 reads evenly over the banks.
  struct Strides {
    int l, x;
  };
  // Cost of one relayout: wavefronts of the LDS.128 reads (per quarter-warp,
  // the max multiplicity of a 4-bank group) plus STS.32 conflict degree.
  static constexpr int relayout_cost(int ls, int xs) {
    int worst = 0;  // LDS.128 is serviced per quarter-warp: 8 lanes x 16 B
    for (int h = 0; h < 4; ++h) {
      int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int ln = 8 * h; ln < 8 * h + 8; ++ln) {
        const int gq = ln / G, lm = ln % G;
        cnt[((gq * xs + lm * ls) % 32) / 4] += 1;
      }
      int wq = 0;
      for (int b = 0; b < 8; ++b) wq = cnt[b] > wq ? cnt[b] : wq;
      worst += wq;
    }
    int sts = 0;
    for (int i = 0; i < R; ++i) {
      int bank[32] = {};
      for (int ln = 0; ln < 32; ++ln) {
        const int gq = ln / G, lm = ln % G;
        const int pn = (i << g) | lm;
        const int addr = gq * xs + (pn >> r) * ls + (pn & (R - 1));
        bank[addr % 32] += 1;
      }
      for (int b = 0; b < 32; ++b) sts = bank[b] > sts ? bank[b] : sts;
    }
    return worst + sts;
  }
  static constexpr Strides pick_strides() {
    Strides best{R, G * R};
    int bc = 1 << 30;
    for (int ls = R; ls < R + 32; ls += 4) {
      for (int xs = G * ls; xs < G * ls + 32; xs += 4) {
        const int c = relayout_cost(ls, xs) * 4096 + xs;  // prefer fewer conflicts, then less memory
        if (c < bc) {
          bc = c;
          best = Strides{ls, xs};
        }
      }
    }
    return best;
  }
  // Chunked relayout (CS = 2^(r-g) >= 4 consecutive registers of an old lane
  // land in one new lane): one STS.128 and one LDS.128 per 4 registers.
  // Chunk (a, lam) = old lane lam's registers a*CS .. a*CS+CS-1, read by new
  // lane a, at word a * AS + lam * CS of the group's area (group pitch XS).
  static constexpr int CS = (g <= r) ? (1 << (r - g)) : 0;
  static constexpr bool kChunked = g > 0 && CS >= 4;
  static constexpr int chunk_cost(int as, int xs) {
    int cost = 0;
    for (int side = 0; side < 2; ++side) {        // 0: writes (fixed a), 1: reads (fixed lam)
      for (int fix = 0; fix < G; ++fix) {
        for (int part = 0; part < CS / 4; ++part) {
          for (int h = 0; h < 4; ++h) {             // quarter-warps: 8 lanes x 16 B
            int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int ln = 8 * h; ln < 8 * h + 8; ++ln) {
              const int gq = ln / G, lm = ln % G;
              const int a = side == 0 ? fix : lm, l2 = side == 0 ? lm : fix;
              const int addr = gq * xs + a * as + l2 * CS + 4 * part;
              cnt[(addr / 4) % 8] += 1;
            }
            int wq = 0;
            for (int b = 0; b < 8; ++b) wq = cnt[b] > wq ? cnt[b] : wq;
            cost += wq;
          }
        }
      }
    }
    return cost;
  }
  static constexpr Strides pick_chunk_strides() {
    Strides best{R, G * R};
    int bc = 1 << 30;
    for (int as = R; as < R + 64; as += 4) {
      for (int xs = G * as; xs < G * as + 64; xs += 4) {
        const int c = chunk_cost(as, xs) * 4096 + xs;
        if (c < bc) {
          bc = c;
          best = Strides{as, xs};
        }
      }
    }
    return best;
  }
  static constexpr int LSTRIDE = kChunked ? pick_chunk_strides().l : pick_strides().l;  // AS when chunked
  static constexpr int XSTRIDE = kChunked ? pick_chunk_strides().x : pick_strides().x;
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
  int smem_per_warp;      // bytes (per-warp area, after the CTA header)
  int dec_off, x_off, ss_off;  // byte offsets of the regions inside a warp's area
  int stg_off;                 // fused depuncture: LLR staging ring (2 chunks x FPW frames x 12 words)
  // Survivor store split: decisions of stages
  // [t_first, t_split) live in tensor memory (tcols columns per warp, 32 TMEM
  // lanes = the warp's lanes), stages [s_base, L) in shared memory rows
  // (row = t - s_base); row smem_rows - 1 is a dummy sink.
  int t_first, t_split, s_base, smem_rows, tcols;
  // Long frames: stages [t_gl, L) spill to a global scratch (L2 / HBM),
  // g_rows rows of 32 words per warp slot (slot = CTA * warps_per_cta + warp);
  // t_gl = L when everything stays on chip.
  int t_gl, g_rows;
  std::uint32_t* gscratch;
  // Head frames (window start m*f - v1 < 0, clipped by the stream start) read
  // a zero-padded copy of the stream head: llr_head[(t + v1) * B] = stage t,
  // zero for t < 0. All-zero branch metrics keep every path metric at 0, so
  // v1 padded stages leave sigma = 0 at stage 0 exactly as the clipped window
  // starts (reference decoder.cpp:195), and the traceback stops at stage 0.
  const std::int8_t* llr_head;
  std::int64_t head_pitch;  // stages per block in llr_head (batched: v1 + head window)
  int tm_alloc;  // TMEM columns allocated per CTA (power of two)
  std::int64_t safe_stage;  // window start of an interior frame (loads of empty frame slots)
  // -1 read from the parameter bank: ptxas cannot constant-fold it, so the
  // table negations written as mad_u32 stay IMADs on the FMA pipe instead of
  // becoming ALU-pipe IADD3s.
  std::uint32_t m1;
};

// Opaque copy: keeps a per-lane constant in a register instead of letting the
// compiler rematerialise it from threadIdx every block.
__device__ __forceinline__ std::uint32_t opaque(std::uint32_t x) {
  asm volatile("" : "+r"(x));
  return x;
}
// LLR prefetch load that the compiler may not sink towards its use (it would
// otherwise trade the two-block prefetch distance for fewer live registers).
__device__ __forceinline__ std::uint32_t ldg_pinned(const std::uint32_t* p) {
  std::uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Fused-depuncture staging: 8-byte shared-memory load / store (shared-space address).
__device__ __forceinline__ void lds_v2(std::uint32_t saddr, std::uint32_t* v) {
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(saddr));
}
__device__ __forceinline__ void sts_v2(std::uint32_t saddr, std::uint32_t a, std::uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(saddr), "r"(a), "r"(b) : "memory");
}

// a * b + c as an IMAD on the FMA pipe (b is an opaque register, so ptxas
// cannot strength-reduce it into an ALU-pipe add or shift).
__device__ __forceinline__ std::uint32_t mad_u32(std::uint32_t a, std::uint32_t b, std::uint32_t c) {
  std::uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Tuning choices are the measured-best settings; every rejected alternative is
// logged in profiles/r01_ab_notes.md / profiles/r02_ab_notes.md and was
// removed from the source: negated branch tables as IMADs with a
// parameter-bank -1 (C5 +0.5 %, C4 +0.9 %); the serial-traceback and
// subframe-traceback fast paths (+6 %, +4-5 %); head frames through a
// zero-padded copy; the long-frame traceback's bulk L2 prefetch.
constexpr int kTbL2Rows = 64;  // rows (stages) per bulk L2 prefetch window
// Warps per CTA (launch bound): 12 = 3 per scheduler, the most the TMEM +
// shared-memory survivor store holds at f=256/20/20; 16 with part of the rows
// spilled to (L2-resident) global scratch measured slower for every code
// (C5 115 vs 123, C4 29.0 vs 29.9 Gbps, profiles/r02_ab_notes.md).
template <class C>
constexpr int max_warps() {
  return 12;
}

// (a & m) | (b & ~m) as one LOP3 (m a compile-time constant after unrolling)
__device__ __forceinline__ std::uint32_t bitsel_m(std::uint32_t a, std::uint32_t b, std::uint32_t m) {
  std::uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "r"(m));
  return r;
}

template <std::uint32_t MUL>
__device__ __forceinline__ std::uint32_t mad_imm(std::uint32_t a, std::uint32_t c) {
  std::uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "n"(MUL), "r"(c));
  return d;
}
// 32 decisions (16 registers x 2 frames) -> one word, bit (rho + 16 * half).
// The source words carry !decision in bits 15 / 31; m1 = -1 (parameter bank).
__device__ __forceinline__ std::uint32_t compact16(const std::uint32_t* w, std::uint32_t m1) {
  std::uint32_t y[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) y[q] = prmt(w[q], w[q + 8], 0xFBD9u);
  // Merge on the FMA pipe: y[q] = 255 * N_q with N_q the 4 !decision bits
  // of PRMT q at bit 8j of byte j, and 255 * 0x01010101 = -1 (mod 2^32), so
  // sum_q y[q] * (0x01010101 << q) = -sum_q N_q << q = -Xn, where Xn holds
  // !decision (reg, half) at bit reg + 16 * half; -1 - Xn = ~Xn is the
  // decision word. Eight IMADs instead of a 7-LOP3 merge tree: the ALU pipe
  // (VIADDMNMX, IADD3, PRMT) was the binding pipe (C5 +4 %, C3 +4 %,
  // profiles/r02_ab_notes.md).
  std::uint32_t acc = mad_imm<0x01010101u>(y[0], m1);
  acc = mad_imm<0x02020202u>(y[1], acc);
  acc = mad_imm<0x04040404u>(y[2], acc);
  acc = mad_imm<0x08080808u>(y[3], acc);
  acc = mad_imm<0x10101010u>(y[4], acc);
  acc = mad_imm<0x20202020u>(y[5], acc);
  acc = mad_imm<0x40404040u>(y[6], acc);
  return mad_imm<0x80808080u>(y[7], acc);
}

template <class GEO>
struct FrameState {
  std::uint32_t sig[GEO::R];
  std::uint32_t wv[2][GEO::R];
  // Per-lane LLR sign flips (lane part of the branch index): fw[j] XORs the
  // block's raw LLR word j (0x80: int8 -> offset binary; 0xff: one's-complement
  // negation), kc[k][e] are the per-phase corrections that make the one's
  // complement exact inside the table sums.
  std::uint32_t fw[GEO::WPB];
  std::uint32_t kc[GEO::LB][GEO::B == 2 ? 2 : GEO::B];
  std::uint32_t llr[2][2][GEO::WPB];  // [buffer][frame A/B][word]: even/odd blocks
  std::uint32_t m1_p;                 // -1 from the parameter bank
  std::uint32_t corr;                 // pending renormalisation (BASE - ref per half)
};

// Branch tables of one block: PT[k][x] = T_k[x ^ lane part] + 128 B per half
// (T = the reference stage table, decoder.cpp:41-51, for frames A | B).
template <class C, class GEO, int BUF>
__device__ __forceinline__ void block_tables(const FrameState<GEO>& st, std::uint32_t (&PT)[GEO::LB][1 << GEO::B]) {
  constexpr int LB = GEO::LB, B = GEO::B, WPB = GEO::WPB;
  constexpr std::uint32_t XM = C::kXM;
  constexpr std::uint32_t OFFB = static_cast<std::uint32_t>(256 * B) * 0x00010001u;
  // interleave frames A / B: lo = (A0, A1, B0, B1), hi = (A2, A3, B2, B3) of each word
  std::uint32_t il[WPB][2];
#pragma unroll
  for (int j = 0; j < WPB; ++j) {
    const std::uint32_t a = st.llr[BUF][0][j] ^ st.fw[j];
    const std::uint32_t b = st.llr[BUF][1][j] ^ st.fw[j];
    il[j][0] = prmt(a, b, 0x5410u);
    il[j][1] = prmt(a, b, 0x7632u);
  }
  // LLR i of phase k, zero-extended per half: byte q = k B + i of the block
  auto X = [&](int k, int i) {
    const int q = k * B + i;
    return prmt(il[q >> 2][(q >> 1) & 1], 0u, (q & 1) ? 0x4341u : 0x4240u);
  };
#pragma unroll
  for (int k = 0; k < LB; ++k) {
    const std::uint32_t x0 = X(k, 0), x1 = X(k, 1);
    if constexpr (B == 2) {
      PT[k][0] = x0 + x1 + st.kc[k][0];             // l0 + l1 + 256
      PT[k][1] = x0 - x1 + st.kc[k][1];             // l0 - l1 + 256
    } else if constexpr (B == 3) {
      const std::uint32_t x2 = X(k, 2) + st.kc[k][2];
      const std::uint32_t a = x0 + x1 + st.kc[k][0];  // l0 + l1 + 256
      const std::uint32_t d = x0 - x1 + st.kc[k][1];  // l0 - l1 + 256
      PT[k][0] = a + x2;
      PT[k][1] = a - x2 + 0x01000100u;
      PT[k][2] = d + x2;
      PT[k][3] = d - x2 + 0x01000100u;
    } else {  // B = 4: T + 512 per half
      const std::uint32_t a = x0 + x1 + st.kc[k][0];  // l0 + l1 + 256
      const std::uint32_t d = x0 - x1 + st.kc[k][1];  // l0 - l1 + 256
      const std::uint32_t x2 = X(k, 2) + st.kc[k][2];  // l2 + 128
      const std::uint32_t x3 = X(k, 3) + st.kc[k][3];  // l3 + 128
      const std::uint32_t pp = x2 + x3;                // l2 + l3 + 256
      const std::uint32_t qq = x2 - x3;                // l2 - l3
      PT[k][0] = a + pp;
      PT[k][1] = a + qq + 0x01000100u;
      PT[k][2] = a - qq + 0x01000100u;
      PT[k][3] = a - pp + 0x02000200u;
      PT[k][4] = d + pp;
      PT[k][5] = d + qq + 0x01000100u;
      PT[k][6] = d - qq + 0x01000100u;
      PT[k][7] = d - pp + 0x02000200u;
    }
#pragma unroll
    for (int x = 0; x < GEO::NT; ++x) {
      // T[x ^ XM] = -T[x]
      PT[k][x ^ XM] = mad_u32(PT[k][x], st.m1_p, OFFB);
    }
  }
}

// ---- tensor-memory survivor store --------------------------------------------
__device__ __forceinline__ void tmem_st1(std::uint32_t taddr, std::uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st4(std::uint32_t taddr, const std::uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(std::uint32_t taddr, std::uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Split form of tmem_ld4: the load, and a wait that names the destination
// registers (so no use of them can be scheduled before the wait).
__device__ __forceinline__ void tmem_ld4_async(std::uint32_t taddr, std::uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld(std::uint32_t (&v)[4]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3])::"memory");
}

struct BlockCtx {
  int v1, L;
  std::uint32_t* drow_lane;  // smem survivor rows of this warp + lane
  int s_base;                // stage of smem row 0
  int dummy_row;             // row index receiving out-of-range decision words
  int t_first, t_split;      // TMEM holds stages [t_first, t_split)
  std::uint32_t taddr;       // TMEM address of this warp's column t_first
  int t_gl;                  // stages [t_gl, L) live in global scratch rows
  std::uint32_t* grow_lane;  // global scratch rows of this warp slot + lane
};

// Decision word of stage t -> its survivor slot (TMEM column or smem row).
template <bool TM, bool GL>
__device__ __forceinline__ void store_dec(const BlockCtx& bc, int t, std::uint32_t word) {
  const bool in = t >= bc.v1 && t < bc.L;
  if (TM && in && t < bc.t_split) {
    tmem_st1(bc.taddr + static_cast<std::uint32_t>(t - bc.t_first), word);
  } else if (GL && in && t >= bc.t_gl) {
    bc.grow_lane[(t - bc.t_gl) * 32] = word;
  } else {
    bc.drow_lane[(in ? t - bc.s_base : bc.dummy_row) * 32] = word;
  }
}

// One block of LB stages. MODE 0 (slow) range-checks every pending store and
// calls the stored-max argmax hook; MODE 1 / 2 / 5 are straight-line blocks
// whose pending stores all go to shared memory / tensor memory / global rows;
// MODE 3 blocks lie entirely in the v1 warm-up (ACS only: no decision words,
// no stores).
template <class C, class GEO, int MODE, bool TM, bool GL, int BUF, class PN, class RecFn>
__device__ __forceinline__ void run_block(FrameState<GEO>& st, int blk, const BlockCtx& bc, int& tprev,
                                          const std::uint32_t* pfA, const std::uint32_t* pfB, std::uint32_t sA,
                                          RecFn&& rec) {
  constexpr int LB = GEO::LB, R = GEO::R, WPB = GEO::WPB;
  constexpr std::uint32_t CB0 = C::cb(0), CBT = C::cb(C::kK - 1);
  // ---- branch-metric tables for the LB stages of this block (both frames) ---
  std::uint32_t PT[LB][1 << GEO::B];
  block_tables<C, GEO, BUF>(st, PT);
  // Renormalisation folded into the ACS tables: the block
  // after a renorm point adds st.corr = BASE - ref per half to its stage-0
  // ACS tables, which subtracts ref - BASE from every new metric (one
  // VIADD.16x2 per table entry instead of one IADD3 per state register).
  // Decision words keep the unshifted tables: both candidates shift equally.
  constexpr bool CORR = BUF == 0;
  std::uint32_t PA0[1 << GEO::B];
#pragma unroll
  for (int x = 0; x < (1 << GEO::B); ++x) PA0[x] = CORR ? __vadd2(PT[0][x], st.corr) : PT[0][x];
  auto pa = [&](int k, std::uint32_t x) { return (CORR && k == 0) ? PA0[x] : PT[k][x]; };
  constexpr std::uint32_t OFFB = static_cast<std::uint32_t>(256 * GEO::B) * 0x00010001u;
  // The words of this buffer are consumed: refill it with block blk + 2 now,
  // so two full blocks of work cover the HBM latency.
  // Every launched window is followed by >= 2 blocks of readable stages
  // (plan() / the head copies / the batch tables guarantee it), so the
  // prefetch never needs clamping; the over-read values are never consumed
  // past stage L-1.
  if constexpr (PN::kActive) {
    // fused depuncture: the block's words come from the warp's staging ring
    // (frame A at sA, frame B one 48-byte frame row later)
    static_assert(WPB == 2, "fused depuncture stages B = 2 streams");
    lds_v2(sA, st.llr[BUF][0]);
    lds_v2(sA + 48u, st.llr[BUF][1]);
  } else {
#pragma unroll
    for (int i = 0; i < WPB; ++i) {
      st.llr[BUF][0][i] = ldg_pinned(pfA + i);
      st.llr[BUF][1][i] = ldg_pinned(pfB + i);
    }
  }
  std::uint32_t tw[4];
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
      // edge labels (reference trellis.cpp:65-91, in_out): E -> L is x; the
      // odd predecessor adds cb(0), input 1 (the H state) adds cb(K - 1)
      // (both XM for complement-paired codes)
      const std::uint32_t s2L = __vadd2(sO, pa(k, x ^ CB0));
      const std::uint32_t s2H = __vadd2(sO, pa(k, x ^ CB0 ^ CBT));
      const std::uint32_t nL = __viaddmax_s16x2(sE, pa(k, x), s2L);
      const std::uint32_t nH = __viaddmax_s16x2(sE, pa(k, x ^ CBT), s2H);
      // Decision words: bit 15 / 31 set iff the FIRST predecessor won, i.e.
      // s1 - s2 >= 1 per half (ties -> second, decoder.cpp:67-74); + 0x7FFF
      // per half keeps each half in [0, 0xFFFE], so no carry crosses halves.
      // (MODE 3: warm-up stages t < v1 keep no decisions, decoder.cpp:229-235
      // never reads them.)
      if constexpr (MODE != 3) {
        // new - s2 (>= 0, 0 iff the second won) + 0x7FFF: one IADD3 per two
        // decisions (measured faster than an FMA-pipe form for some of them)
        w[e] = nL - s2L + 0x7fff7fffu;
        w[od] = nH - s2H + 0x7fff7fffu;
      }
      st.sig[e] = nL;
      st.sig[od] = nH;
    }
    // ---- previous stage's decisions -> survivor store (overlaps this ACS) --
    if constexpr (MODE == 3) continue;
    const std::uint32_t word = compact16(st.wv[(k + 1) & 1], st.m1_p);
    if constexpr (MODE == 0) {
      store_dec<TM, GL>(bc, tprev, word);
      tprev = t;
      rec(t, k);
    } else {
      tw[k] = word;  // stored after the block, below
    }
  }
  if constexpr (MODE == 2) tmem_st4(bc.taddr + static_cast<std::uint32_t>(blk * LB - 1 - bc.t_first), tw);
  if constexpr (MODE == 1) {
    // same register schedule as the TMEM blocks (an in-loop store per stage
    // made ptxas rotate the metric registers with ~30 IMAD.MOVs per block)
#pragma unroll
    for (int k = 0; k < LB; ++k) bc.drow_lane[(blk * LB - 1 + k - bc.s_base) * 32] = tw[k];
  }
  if constexpr (MODE == 5) {
    // global rows: one address per block, coalesced 128-byte rows per warp
    std::uint32_t* const gp = bc.grow_lane + static_cast<std::ptrdiff_t>(blk * LB - 1 - bc.t_gl) * 32;
#pragma unroll
    for (int k = 0; k < LB; ++k) gp[k * 32] = tw[k];
  }
  if constexpr (MODE != 0) tprev = blk * LB + LB - 1;
}

template <class C, int R, bool TM, bool GL, class PN = NoPunct>
__global__ void __launch_bounds__(max_warps<C>() * 32, 1) fast_kernel(const FastParams fp) {
  using GEO = Geo<C, R>;
  constexpr int M = GEO::M, S = GEO::S, G = GEO::G, LB = GEO::LB, r = GEO::r, g = GEO::g;
  constexpr std::uint32_t BASE = 0x20002000u;  // offset-binary metric origin (8192 per half)
  constexpr int WPB = GEO::WPB, B = GEO::B;
  static_assert((LB * B) % 4 == 0, "a block must cover whole LLR words");
  static_assert(LB == 4, "tensor-memory blocks are 4 columns");
  static_assert(R == 16, "one 32-bit decision word per lane per stage");
  const DecodeLaunch& p = fp.p;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int grp = lane / G;
  const int lam = lane % G;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(smem_raw);  // CTA header (16 B)
  unsigned char* wbase = smem_raw + 16 + static_cast<std::size_t>(warp) * fp.smem_per_warp;
  std::uint32_t* dec = reinterpret_cast<std::uint32_t*>(wbase + fp.dec_off);
  std::uint32_t* xbuf = reinterpret_cast<std::uint32_t*>(wbase + fp.x_off);
  std::uint16_t* sstate = reinterpret_cast<std::uint16_t*>(wbase + fp.ss_off);

  // ---- tensor-memory allocation (one warp allocates for the CTA) ------------
  std::uint32_t tbase = 0;
  if constexpr (TM) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(tmem_slot))),
                   "r"(static_cast<unsigned>(fp.tm_alloc)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    tbase = *tmem_slot;
  }

  // Persistent warps: the grid holds at most one CTA per SM and every warp
  // walks frame groups gwarp, gwarp + W, ... (W = warps in the grid), so the
  // TMEM allocation and CTA start-up are paid once per SM, and warps drift out
  // of phase (one warp's traceback overlaps other warps' forward passes).
  // All warps of a CTA run the same number of rounds and meet at a CTA
  // barrier after each one: keeping the warps in phase measured faster than
  // letting them drift (the forward and traceback code then compete for the
  // instruction cache).
  const std::int64_t wtotal = static_cast<std::int64_t>(gridDim.x) * fp.warps_per_cta;
  const std::int64_t groups = (fp.mi1 - fp.mi0 + GEO::FPW - 1) / GEO::FPW;
  const std::int64_t rounds = (groups + wtotal - 1) / wtotal;
  for (std::int64_t rnd = 0; rnd < rounds; ++rnd) {
  if (rnd > 0) __syncthreads();
  const std::int64_t gwarp = rnd * wtotal + static_cast<std::int64_t>(blockIdx.x) * fp.warps_per_cta + warp;
  const std::int64_t mbase = fp.mi0 + gwarp * GEO::FPW;
  if (mbase < fp.mi1) {  // (no early return: TMEM dealloc needs every warp at the barrier)
  const std::int64_t mA = mbase + 2 * grp, mB = mA + 1;
  bool validA = mA < fp.mi1, validB = mB < fp.mi1;
  // Window start stage of a frame slot; empty slots (past the launch, or in
  // batched mode a clipped edge frame of its block) load an interior frame's
  // LLRs and write nothing.
  struct Slot {
    std::int64_t ws, m;  // window start stage (stream), block-local frame index
    int blk;             // block (batched mode)
    bool head;           // window clipped at the block start: read the zero-padded head copy
  };
  // Empty slots read some valid window and write nothing: block 0's padded
  // head when there is one (safe_stage may then be negative), else safe_stage.
  const Slot empty = fp.llr_head ? Slot{-static_cast<std::int64_t>(p.v1), 0, 0, true} : Slot{fp.safe_stage, 0, 0, false};
  auto frame_slot = [&](std::int64_t mg, bool& valid) -> Slot {
    if (!valid) return empty;
    const FrameRef r = resolve_frame(p, mg);
    // batched main launch: only the block's interior frames (a frame list
    // launch takes every listed frame)
    if (p.nblocks > 0 && !p.frame_list) valid = r.m >= __ldg(p.blk_ilo + r.blk) && r.m < __ldg(p.blk_ihi + r.blk);
    if (!valid) return empty;
    return Slot{r.base + r.m * p.f - p.v1, r.m, r.blk, fp.llr_head != nullptr && r.m * p.f < p.v1};
  };
  const Slot slA = frame_slot(mA, validA), slB = frame_slot(mB, validB);


  const int f = static_cast<int>(opaque(static_cast<std::uint32_t>(p.f)));
  const int v1 = static_cast<int>(opaque(static_cast<std::uint32_t>(p.v1)));
  const int v2 = static_cast<int>(opaque(static_cast<std::uint32_t>(p.v2)));
  const int L = static_cast<int>(opaque(static_cast<std::uint32_t>(fp.L)));
  const int nblk = static_cast<int>(opaque(static_cast<std::uint32_t>(fp.nblk)));
  const int num_sub = static_cast<int>(opaque(static_cast<std::uint32_t>(fp.num_sub)));
  const int step = static_cast<int>(opaque(static_cast<std::uint32_t>(fp.step)));
  const int t_split = TM ? static_cast<int>(opaque(static_cast<std::uint32_t>(fp.t_split))) : v1;
  const int t_first = TM ? static_cast<int>(opaque(static_cast<std::uint32_t>(fp.t_first))) : v1;
  const int s_base = static_cast<int>(opaque(static_cast<std::uint32_t>(fp.s_base)));
  const int t_gl = GL ? static_cast<int>(opaque(static_cast<std::uint32_t>(fp.t_gl))) : L;
  // Frame-relative LLR word pointers (frame start is 4-byte aligned: checked at launch).
  auto llr_of = [&](const Slot& sl) {
    const std::int8_t* b8 =
        sl.head ? fp.llr_head + (static_cast<std::int64_t>(sl.blk) * fp.head_pitch + sl.m * p.f) * B
                : static_cast<const std::int8_t*>(p.llr) + (sl.ws - p.llr_stage0) * B;
    return reinterpret_cast<const std::uint32_t*>(b8);
  };
  const std::uint32_t* llrA = PN::kActive ? nullptr : llr_of(slA);
  const std::uint32_t* llrB = PN::kActive ? nullptr : llr_of(slB);

  // ---- fused depuncture: LLR staging ring ----------------------------------
  // Chunks of 24 stages of the warp's FPW frames are depunctured into a
  // 2-chunk ring in shared memory ([chunk & 1][frame slot][12 words]); lane
  // 2q + h fills 12 stages (6 words) of frame slot q. Chunk c + 1 is loaded
  // during the blocks of chunk c (global loads issued at block 6c, gathered
  // and stored at block 6c + 2) and first read by the prefetch of block 6c + 4.
  constexpr std::uint32_t kChunkBytes = static_cast<std::uint32_t>(GEO::FPW) * 48u;
  std::uint32_t stg_s = 0, rbuf = 0;
  int rpos = 2, rc = 0, nch = 0;  // prefetch cursor: block b + 2 = chunk rc, block rpos of it
  const unsigned char* tptr = nullptr;  // this lane's fill task: first transmitted byte of chunk 0
  bool tvalid = false;
  std::uint32_t raw[6] = {0u, 0u, 0u, 0u, 0u, 0u};
  std::uint32_t ralign = 0;
  (void)stg_s;
  (void)rbuf;
  (void)raw;
  auto fill_issue = [&](int c) {
    if constexpr (PN::kActive) {
      const unsigned char* a = tptr + static_cast<std::int64_t>(c) * (2 * PN::task_bytes());
      ralign = static_cast<std::uint32_t>(reinterpret_cast<std::uintptr_t>(a) & 3u);
      const std::uint32_t* w = reinterpret_cast<const std::uint32_t*>(a - ralign);
#pragma unroll
      for (int j = 0; j < 6; ++j) raw[j] = tvalid ? ldg_pinned(w + j) : 0u;
    }
  };
  auto fill_finish = [&](int c) {
    if constexpr (PN::kActive) {
      std::uint32_t u[5];
#pragma unroll
      for (int j = 0; j < 5; ++j) u[j] = __funnelshift_r(raw[j], raw[j + 1], 8u * ralign);
      constexpr typename PN::Gather G = PN::gather();
      std::uint32_t o[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const int a = G.word[i];
        o[i] = prmt(u[a], u[a + 1 < 5 ? a + 1 : 4], G.sel[i]) & G.mask[i];
      }
      if (tvalid) {
        const std::uint32_t s = stg_s + ((c & 1) ? kChunkBytes : 0u) + static_cast<std::uint32_t>(lane >> 1) * 48u +
                                static_cast<std::uint32_t>(lane & 1) * 24u;
        sts_v2(s, o[0], o[1]);
        sts_v2(s + 8u, o[2], o[3]);
        sts_v2(s + 16u, o[4], o[5]);
      }
    }
  };
  if constexpr (PN::kActive) {
    stg_s = static_cast<std::uint32_t>(__cvta_generic_to_shared(wbase + fp.stg_off));
    const int ft = lane >> 1;
    tvalid = ft < GEO::FPW;
    bool vt = tvalid && mbase + ft < fp.mi1;
    const Slot slT = frame_slot(mbase + ft, vt);  // empty slots read some interior window
    // frames are period-aligned: window start ws is a multiple of P
    tptr = static_cast<const unsigned char*>(p.llr) + (slT.ws / PN::P) * PN::kept_per_period() +
           (lane & 1) * PN::task_bytes();
    nch = (fp.nblk + 1) / 6 + 1;  // chunks read: blocks 0 .. nblk + 1
    fill_issue(0);
    fill_finish(0);
    __syncwarp();
  }

  FrameState<GEO> st;
  // Per-phase flip constants for this lane (lane part of the branch index).
  {
    std::uint32_t fw[WPB];
#pragma unroll
    for (int j = 0; j < WPB; ++j) fw[j] = 0x80808080u;
#pragma unroll
    for (int k = 0; k < LB; ++k) {
      std::uint32_t z = 0;  // lane part of the branch index at phase k
#pragma unroll
      for (int i = 0; i < g; ++i) {
        if ((lam >> i) & 1) z ^= C::cb(r + i - k);
      }
      std::uint32_t phi[4] = {0u, 0u, 0u, 0u};  // llr i negated for this lane
#pragma unroll
      for (int i = 0; i < B; ++i) {
        phi[i] = (z >> (B - 1 - i)) & 1u;
        const int q = k * B + i;
        if (phi[i]) fw[q >> 2] ^= 0xffu << (8 * (q & 3));
      }
      // one's complement (255 - u) is the exact negation (256 - u) minus 1
      st.kc[k][0] = opaque((phi[0] + phi[1]) * 0x00010001u);
      st.kc[k][1] = opaque((256u + phi[0] - phi[1]) * 0x00010001u);
      if constexpr (B >= 3) st.kc[k][2] = opaque(phi[2] * 0x00010001u);
      if constexpr (B == 4) st.kc[k][3] = opaque(phi[3] * 0x00010001u);
    }
#pragma unroll
    for (int j = 0; j < WPB; ++j) st.fw[j] = opaque(fw[j]);
  }
  st.m1_p = fp.m1;
  st.corr = 0u;
#pragma unroll
  for (int i = 0; i < R; ++i) st.sig[i] = BASE;
#pragma unroll
  for (int i = 0; i < R; ++i) st.wv[1][i] = 0u;
  std::int32_t subA = 0, subB = 0;  // accumulated renormalisation (ref - BASE) per half

  if constexpr (PN::kActive) {
    const std::uint32_t s0 = stg_s + static_cast<std::uint32_t>(2 * grp) * 48u;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      lds_v2(s0 + 8u * b, st.llr[b][0]);
      lds_v2(s0 + 8u * b + 48u, st.llr[b][1]);
    }
  } else {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
#pragma unroll
      for (int i = 0; i < WPB; ++i) {
        st.llr[b][0][i] = __ldg(llrA + b * WPB + i);
        st.llr[b][1][i] = __ldg(llrB + b * WPB + i);
      }
    }
  }
  // Prefetch pointers: block b + 2 is requested right after block b has
  // built its tables (two blocks of latency cover).
  const std::uint32_t* pfA = PN::kActive ? nullptr : llrA + 2 * WPB;
  const std::uint32_t* pfB = PN::kActive ? nullptr : llrB + 2 * WPB;

  int next_sub = 0;
  // subframes whose traceback starts from the stored max state
  auto sub_start = [&](int s) { return v1 + min((s + 1) * step, f) + v2 - 1; };
  auto needs_record = [&](int s) {
    const int sst = sub_start(s);
    return !(p.f0 > 0 && p.start == 1 && sst < L - 1);
  };
  while (next_sub < num_sub && !needs_record(next_sub)) ++next_sub;
  int next_rec = next_sub < num_sub ? sub_start(next_sub) : 0x7fffffff;

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
      sstate[(2 * grp) * num_sub + next_sub] = static_cast<std::uint16_t>(0xffffu - (bestA & 0xffffu));
      sstate[(2 * grp + 1) * num_sub + next_sub] = static_cast<std::uint16_t>(0xffffu - (bestB & 0xffffu));
    }
    if (t == L - 1 && p.sigma != nullptr) {
      // final metrics: true = stored - BASE - 128 B L + sum(ref - BASE)
      std::int64_t* sg = static_cast<std::int64_t*>(p.sigma);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int sidx = static_cast<int>(lanepart | static_cast<std::uint32_t>(GEO::rotr(i, k + 1)));
        const std::int64_t a = static_cast<std::int64_t>(st.sig[i] & 0xffffu) - 8192 - 128LL * B * L + subA;
        const std::int64_t b = static_cast<std::int64_t>(st.sig[i] >> 16) - 8192 - 128LL * B * L + subB;
        if (validA) sg[(mA - p.frame_begin) * S + sidx] = a;
        if (validB) sg[(mB - p.frame_begin) * S + sidx] = b;
      }
    }
    ++next_sub;
    while (next_sub < num_sub && !needs_record(next_sub)) ++next_sub;
    next_rec = next_sub < num_sub ? sub_start(next_sub) : 0x7fffffff;
  };

  BlockCtx bc;
  bc.v1 = v1;
  bc.L = L;
  bc.drow_lane = dec + lane;
  bc.s_base = s_base;
  bc.dummy_row = fp.smem_rows - 1;
  bc.t_first = t_first;
  bc.t_split = t_split;
  // this warp's TMEM lanes (32 * (warp % 4)) and columns (tcols * (warp / 4))
  bc.t_gl = t_gl;
  bc.grow_lane = fp.gscratch + (static_cast<std::size_t>(blockIdx.x) * fp.warps_per_cta + warp) *
                                   static_cast<std::size_t>(fp.g_rows) * 32 + lane;
  bc.taddr = tbase + ((32u * static_cast<std::uint32_t>(warp & 3)) << 16) +
             static_cast<std::uint32_t>(fp.tcols * (warp >> 2));
  int tprev = -1;

  // (opaque offset, not pointer: the accesses must stay STS/LDS)
  std::uint32_t* const xb = xbuf + opaque(static_cast<std::uint32_t>(grp * GEO::XSTRIDE));
  // chunked relayout: this lane writes its chunks at lam * CS, reads its own at lam * AS
  std::uint32_t* const xw = xbuf + opaque(static_cast<std::uint32_t>(grp * GEO::XSTRIDE + lam * GEO::CS));
  const std::uint32_t* const xr = xbuf + opaque(static_cast<std::uint32_t>(grp * GEO::XSTRIDE + lam * GEO::LSTRIDE));
  auto block_end = [&](int blk, auto buf_tag) {
    // ---- renormalisation every 2 blocks (after each odd block: a compile-time
    // position in the 2-block loop body; group-wide reference): metrics stay
    // within [BASE - spread, BASE + spread + 16 * 510] (< 32768 up to K = 9).
    constexpr int BUFE = decltype(buf_tag)::value;
    if (BUFE == 1) {
      const std::uint32_t ref = __shfl_sync(kFull, st.sig[0], grp * G);
      subA += static_cast<std::int32_t>(ref & 0xffffu) - 8192;
      subB += static_cast<std::int32_t>(ref >> 16) - 8192;
      st.corr = __vsub2(BASE, ref);  // applied by the next (BUF 0) block's stage-0 tables
    }
    // ---- relayout: back to the canonical layout (P_new = rotr(P_old, r)) --
    if constexpr (GEO::kChunked) {
      constexpr int CS = GEO::CS, AS = GEO::LSTRIDE;
#pragma unroll
      for (int a = 0; a < G; ++a) {
#pragma unroll
        for (int q = 0; q < CS / 4; ++q) {
          const int i = a * CS + 4 * q;
          *reinterpret_cast<uint4*>(xw + a * AS + 4 * q) =
              make_uint4(st.sig[i], st.sig[i + 1], st.sig[i + 2], st.sig[i + 3]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int l2 = 0; l2 < G; ++l2) {
#pragma unroll
        for (int q = 0; q < CS / 4; ++q) {
          const uint4 v = *reinterpret_cast<const uint4*>(xr + l2 * CS + 4 * q);
          // old register a*CS + c of old lane l2 -> new register (c << g) | l2
          st.sig[((4 * q + 0) << g) | l2] = v.x;
          st.sig[((4 * q + 1) << g) | l2] = v.y;
          st.sig[((4 * q + 2) << g) | l2] = v.z;
          st.sig[((4 * q + 3) << g) | l2] = v.w;
        }
      }
      __syncwarp();
    } else if constexpr (g > 0) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        // old (lam, i) -> new physical index rotr(lam * R + i, r) = (i << g) | lam
        const int pn_reg = ((i << g) & (R - 1));  // compile-time part of the new register index
        const int pn_lane = (i << g) >> r;        // compile-time part of the new lane index
        xb[(pn_lane + (lam >> r)) * GEO::LSTRIDE + pn_reg + (lam & (R - 1))] = st.sig[i];
      }
      __syncwarp();
      const uint4* src = reinterpret_cast<const uint4*>(xb + lam * GEO::LSTRIDE);
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
  };
  // Store mode of a block: warm-up (3: t0 + LB <= v1); straight-line
  // ("clean": pending stores of stages t0-1 .. t0+LB-2 all inside [v1, L) and
  // on one side of the TMEM / smem / global split, no start stage inside) to
  // global rows (5), smem rows (1) or TMEM (2); else the general block (0).
  // The mode only changes at a few block indices per frame: the end of the warm-up, the first / last clean block,
  // the TMEM / smem / global-row splits, and the block holding the next
  // stored-max start stage (which only moves inside a MODE 0 block). The loop
  // picks the mode once per run of equal-mode blocks and runs them with a
  // fixed body (per-block mode tests had cost ~40 instructions per block pair).
  auto one_block_mode = [&](int blk, auto mode_tag, auto buf_tag) {
    constexpr int MD = decltype(mode_tag)::value, BUF = decltype(buf_tag)::value;
    if constexpr (PN::kActive) {
      const std::uint32_t sA = stg_s + rbuf + static_cast<std::uint32_t>(2 * grp) * 48u + static_cast<std::uint32_t>(rpos) * 8u;
      run_block<C, GEO, MD, TM, GL, BUF, PN>(st, blk, bc, tprev, pfA, pfB, sA, rec);
      // (rpos = (blk + 2) % 6 has the parity of blk: the fills only ever
      // fall on the first block of a pair, and as branches, not predicated
      // every block — ptxas if-converted them for P = 3: +24 issued
      // instructions per block)
      if constexpr (BUF == 0) {
        if (rc + 1 < nch) {
          if (__builtin_expect(rpos == 2, 0)) {
            fill_issue(rc + 1);
          } else if (__builtin_expect(rpos == 4, 0)) {
            fill_finish(rc + 1);
          }
        }
      }
      if (++rpos == 6) {
        rpos = 0;
        rbuf ^= kChunkBytes;
        ++rc;
      }
    } else {
      if constexpr (C::kK == 7 && GEO::B == 2) {
        // prefetch address = the lane's window base + a warp-uniform block
        // offset (K=7 r1/2: 328 instead of 332 instructions per TMEM block,
        // C5 123.1 vs 122.3 Gbps; K=9 and B=3 measured 0.3-0.9 % slower this
        // way, profiles/r02_ab_notes.md)
        const int pfo = (blk + 2) * WPB;
        run_block<C, GEO, MD, TM, GL, BUF, PN>(st, blk, bc, tprev, llrA + pfo, llrB + pfo, 0u, rec);
      } else {
        run_block<C, GEO, MD, TM, GL, BUF, PN>(st, blk, bc, tprev, pfA, pfB, 0u, rec);
        pfA += WPB;
        pfB += WPB;
      }
    }
    block_end(blk, buf_tag);
  };
  auto run_mode = [&](auto mode_tag, int& blk, int end) {
    while (blk < end) {
      if ((blk & 1) == 0) {
        one_block_mode(blk, mode_tag, std::integral_constant<int, 0>{});
        if (++blk >= end) break;
      }
      one_block_mode(blk, mode_tag, std::integral_constant<int, 1>{});
      ++blk;
    }
  };
  // first block index with blk * LB + LB - 2 >= x  /  with blk * LB - 1 >= x
  auto first_hi = [](int x) { return (x + 1) / LB; };
  auto first_lo = [](int x) { return (x + LB) / LB; };
  const int nb_warm = v1 / LB;          // t0 + LB <= v1
  const int cl_lo = first_lo(v1);       // t0 - 1 >= v1
  const int cl_hi = first_hi(L);        // t0 + LB - 2 < L below this
  const int tm_hi = first_hi(t_split);  // t0 + LB - 2 < t_split below this
  const int sm_lo = first_lo(t_split);  // t0 - 1 >= t_split
  const int gl_lo = first_lo(t_gl);     // t0 - 1 >= t_gl
  const int sm_hi = GL ? min(first_hi(t_gl), cl_hi) : cl_hi;
  int blk = 0;
  while (blk < nblk) {
    const int rb = next_rec / LB;  // block holding the next start stage
    int md = 0, end = blk + 1;
    if (blk < nb_warm) {
      md = 3;
      end = nb_warm;
    } else if (blk >= cl_lo && blk < cl_hi && blk != rb) {
      const int rend = rb > blk ? min(cl_hi, rb) : cl_hi;
      if (GL && blk >= gl_lo) {
        md = 5;
        end = rend;
      } else if (blk >= sm_lo && blk < sm_hi) {
        md = 1;
        end = min(rend, sm_hi);
      } else if (TM && blk < tm_hi) {
        md = 2;
        end = min(rend, tm_hi);
      }
    }
    if (md == 2) {
      run_mode(std::integral_constant<int, 2>{}, blk, end);
    } else if (md == 1) {
      run_mode(std::integral_constant<int, 1>{}, blk, end);
    } else if (md == 3) {
      run_mode(std::integral_constant<int, 3>{}, blk, end);
    } else if (GL && md == 5) {
      run_mode(std::integral_constant<int, 5>{}, blk, end);
    } else {
      run_mode(std::integral_constant<int, 0>{}, blk, end);
    }
  }
  // decisions of the last processed stage
  store_dec<TM, GL>(bc, tprev, compact16(st.wv[(nblk * LB - 1) & 1], st.m1_p));
  if constexpr (TM) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  __syncwarp();

  // ---- subframe-parallel traceback (decoder.cpp:214-236) --------------------
  // Tasks (frame, subframe) are spread over all 32 lanes of the warp, frames
  // fastest; the block loop is warp-uniform (the union of the round's task
  // ranges) so tensor-memory loads, which are warp-collective, can be used.
  // Within a block of LB stages the lane index of a traced state (P >> r) is
  // fixed (only register bits are rewritten): the block's 4 words come from
  // one TMEM load + shuffles or 4 independent LDS, then the per-step work is
  // branch-free. Output bit of phase j = bit j of P at block entry.
  const int ntask = GEO::FPW * num_sub;
  for (int base = 0; base < ntask; base += 32) {
    const int task = base + lane;
    const bool active = task < ntask;
    const int fr = active ? task % GEO::FPW : 0;  // frame slot in the warp (2 * group + half)
    const int s = active ? task / GEO::FPW : 0;
    const int half = fr & 1;
    bool valid = active && mbase + fr < fp.mi1;
    const Slot sl = frame_slot(mbase + fr, valid);
    const std::int64_t m = sl.m;  // block-local frame index (random-start salt)
    const int st_t = active ? sub_start(s) : -1;
    const int sub_lo = v1 + s * step;
    const int sub_hi = v1 + min((s + 1) * step, f);
    std::uint32_t state;
    if (p.f0 > 0 && p.start == 1 && st_t < L - 1) {
      state = static_cast<std::uint32_t>(mix_seed(p.seed, static_cast<std::uint64_t>(m) * 0x10001ull +
                                                              static_cast<std::uint64_t>(s)) %
                                         static_cast<std::uint64_t>(S));
    } else {
      state = sstate[fr * num_sub + s];
    }
    // physical index after stage st (phase st % LB): rotl(state, phase + 1)
    const int sh = ((st_t & (LB - 1)) + 1) % M;
    std::uint32_t P = sh == 0 ? state : (((state << sh) | (state >> (M - sh))) & GEO::SMASK);
    const std::uint32_t hsh = half ? 16u : 0u;
    const int gcol = (fr >> 1) * G;  // this frame's group: first lane of its decision columns
    const std::int64_t obase = sl.ws - p.out_stage0;  // output bit index of frame-relative stage 0
    // ---- serial-traceback fast path: one task per frame, whole blocks from
    // stage L-1 down to v1, output words aligned (f % 32 == 0). Per block:
    // one 4-word fetch, 4 x (funnel shift + bit select), 4 emitted bits into
    // a 32-bit accumulator stored with a plain 32-bit write every 8 blocks.
    if (num_sub == 1 && ((L & (LB - 1)) == 0 || v2 >= LB) && (v1 & (LB - 1)) == 0 && (f & 31) == 0 &&
        __all_sync(kFull, ((obase + v1) & 31) == 0)) {
      std::uint32_t lp = P >> r;
      std::uint32_t u = (P & (R - 1)) | hsh;  // bit index into a decision word: register + 16 * half
      std::uint32_t acc32 = 0;
      std::uint32_t* const outw = p.out + ((obase + v1) >> 5);
      const int t_emit = v1 + f;  // blocks below this stage emit their 4 bits
      std::uint32_t* wp = outw + ((t_emit - LB - v1) >> 5);  // word of the first emitting block
      auto step_block = [&](int tb0, const std::uint32_t (&wd)[LB], int jmax = 3 /* LB - 1 */) {
        const std::uint32_t rin = u & (R - 1);  // bit j = decoded bit of stage tb0 + j
#pragma unroll
        for (int j = LB - 1; j >= 0; --j) {
          const std::uint32_t x = __funnelshift_r(wd[j], wd[j], u - static_cast<std::uint32_t>(j));  // bit u -> bit j
          if (j <= jmax) u = bitsel_m(x, u, 1u << j);
        }
        if (tb0 < t_emit) {
          acc32 = (acc32 << LB) | rin;
          // running word pointer (one decrement per store, no address math per block)
          if (((tb0 - v1) & 31) == 0) {
            if (valid) *wp = acc32;
            --wp;
          }
        }
        const std::uint32_t pa = (lp << r) | (u & (R - 1));
        const std::uint32_t pn = ((pa << r) | (pa >> (M - r))) & GEO::SMASK;  // undo the block relayout
        lp = pn >> r;
        u = (pn & (R - 1)) | hsh;
      };
      int tb0 = (L - 1) & ~(LB - 1);
      if ((L & (LB - 1)) != 0) {
        // L % 4 != 0: the top block only walks phases 0 .. (L-1) % 4 (it lies in
        // the v2 tail, v2 >= 4, so it emits nothing); peeled here, then whole blocks
        const int jmax = (L - 1) & (LB - 1);
        std::uint32_t wd[LB];
        if (GL && tb0 >= t_gl) {
#pragma unroll
          for (int j = 0; j < LB; ++j) wd[j] = bc.grow_lane[(tb0 + j - t_gl) * 32 - lane + gcol + static_cast<int>(lp)];
        } else if (!TM || tb0 >= t_split) {
#pragma unroll
          for (int j = 0; j < LB; ++j) wd[j] = dec[(tb0 + j - s_base) * 32 + gcol + lp];
        } else {
          std::uint32_t own[4];
          tmem_ld4(bc.taddr + static_cast<std::uint32_t>(tb0 - t_first), own);
#pragma unroll
          for (int j = 0; j < LB; ++j) wd[j] = __shfl_sync(kFull, own[j], gcol + static_cast<int>(lp));
        }
        step_block(tb0, wd, jmax);
        tb0 -= LB;
      }
      if (GL && t_gl < L) {
        // global scratch rows: a group's G words of a stage are contiguous, so
        // the loads do not depend on the traced lane and run one block ahead;
        // the rows were written a whole forward pass ago (usually evicted to
        // HBM), so lane 0 also pulls the next kTbL2Rows rows into L2 with one
        // bulk prefetch every kTbL2Rows / 2 rows (rows are contiguous)
        const std::uint32_t* grow = bc.grow_lane - lane + gcol;
        const unsigned char* grow_base = reinterpret_cast<const unsigned char*>(bc.grow_lane - lane);
        auto l2_prefetch = [&](int tb) {  // rows [tb - kTbL2Rows, tb) below the current block
          if (lane == 0) {
            const int lo_row = max(tb - kTbL2Rows, t_gl) - t_gl, hi_row = tb - t_gl;
            if (hi_row > lo_row) {
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(grow_base + lo_row * 128),
                           "r"(static_cast<unsigned>((hi_row - lo_row) * 128))
                           : "memory");
            }
          }
        };
        l2_prefetch(tb0 + LB);  // the first window (the block at tb0 and the rows below it)
        if constexpr (G == 4) {
          uint4 cur[LB], nxt[LB];
#pragma unroll
          for (int j = 0; j < LB; ++j) cur[j] = *reinterpret_cast<const uint4*>(grow + (tb0 + j - t_gl) * 32);
          for (; tb0 >= t_gl; tb0 -= LB) {
            if (((tb0 - t_gl) & (kTbL2Rows / 2 - 1)) == 0) l2_prefetch(tb0 - kTbL2Rows / 2);
            if (tb0 - LB >= t_gl) {
#pragma unroll
              for (int j = 0; j < LB; ++j)
                nxt[j] = *reinterpret_cast<const uint4*>(grow + (tb0 - LB + j - t_gl) * 32);
            }
            std::uint32_t wd[LB];
#pragma unroll
            for (int j = 0; j < LB; ++j) {
              const uint4 c = cur[j];
              const std::uint32_t lo = (lp & 1u) ? c.y : c.x, hi = (lp & 1u) ? c.w : c.z;
              wd[j] = (lp & 2u) ? hi : lo;
            }
            step_block(tb0, wd);
#pragma unroll
            for (int j = 0; j < LB; ++j) cur[j] = nxt[j];
          }
        } else {
          for (; tb0 >= t_gl; tb0 -= LB) {
            if (((tb0 - t_gl) & (kTbL2Rows / 2 - 1)) == 0) l2_prefetch(tb0 - kTbL2Rows / 2);
            std::uint32_t wd[LB];
#pragma unroll
            for (int j = 0; j < LB; ++j) wd[j] = grow[(tb0 + j - t_gl) * 32 + lp];
            step_block(tb0, wd);
          }
        }
      }
      {
        for (; tb0 >= v1 && (!TM || tb0 >= t_split); tb0 -= LB) {  // shared-memory rows
          std::uint32_t wd[LB];
          const std::uint32_t* src = dec + (tb0 - s_base) * 32 + gcol + lp;
#pragma unroll
          for (int j = 0; j < LB; ++j) wd[j] = src[j * 32];
          step_block(tb0, wd);
        }
      }
      if constexpr (TM) {
        for (; tb0 >= v1; tb0 -= LB) {  // tensor-memory columns
          std::uint32_t own[4], wd[LB];
          tmem_ld4(bc.taddr + static_cast<std::uint32_t>(tb0 - t_first), own);
#pragma unroll
          for (int j = 0; j < LB; ++j) wd[j] = __shfl_sync(kFull, own[j], gcol + static_cast<int>(lp));
          step_block(tb0, wd);
        }
      }
      continue;
    }
    // ---- subframe-traceback fast path (stored-max parallel traceback, e.g.
    // f=320/20/45/32): every start stage has the same block phase, every
    // subframe emits whole aligned words; one uniform block loop over the
    // round, each lane walking only its own range (its top block partial).
    if (num_sub > 1 && (step & 31) == 0 && (f % step) == 0 && (v1 & (LB - 1)) == 0 && v2 >= LB &&
        __all_sync(kFull, !active || ((obase + sub_lo) & 31) == 0)) {
      const int ph = (v1 + step + v2 - 1) & (LB - 1);  // phase of every start stage
      const int stb = st_t & ~(LB - 1);                // this lane's top block
      std::uint32_t lp = P >> r;
      std::uint32_t u = (P & (R - 1)) | hsh;
      std::uint32_t acc32 = 0;
      std::uint32_t* const outw = p.out + ((obase + sub_lo) >> 5);
      std::uint32_t* wp = outw + ((sub_hi - LB - sub_lo) >> 5);  // word of this lane's first emitting block
      const int tstart = static_cast<int>(__reduce_max_sync(kFull, active ? static_cast<unsigned>(stb) : 0u));
      const int tstop = static_cast<int>(__reduce_min_sync(kFull, active ? static_cast<unsigned>(sub_lo) : 0x7fffffffu));
      for (int tb0 = tstart; tb0 >= tstop; tb0 -= LB) {
        const bool act = active && tb0 <= stb && tb0 >= sub_lo;
        const bool top = tb0 == stb;
        std::uint32_t wd[LB];
        if (TM && tb0 < t_split) {
          std::uint32_t own[4];
          tmem_ld4(bc.taddr + static_cast<std::uint32_t>(tb0 - t_first), own);
#pragma unroll
          for (int j = 0; j < LB; ++j) wd[j] = __shfl_sync(kFull, own[j], gcol + static_cast<int>(lp));
        } else if (GL && tb0 >= t_gl) {
#pragma unroll
          for (int j = 0; j < LB; ++j) wd[j] = bc.grow_lane[(tb0 + j - t_gl) * 32 - lane + gcol + static_cast<int>(lp)];
        } else {
#pragma unroll
          for (int j = 0; j < LB; ++j) wd[j] = dec[(tb0 + j - s_base) * 32 + gcol + lp];
        }
        const std::uint32_t rin = u & (R - 1);
#pragma unroll
        for (int j = LB - 1; j >= 0; --j) {
          const std::uint32_t x = __funnelshift_r(wd[j], wd[j], u - static_cast<std::uint32_t>(j));
          const bool walk = act && (j <= ph || !top);
          if (walk) u = bitsel_m(x, u, 1u << j);
        }
        if (act && tb0 < sub_hi) {
          acc32 = (acc32 << LB) | rin;
          if (((tb0 - sub_lo) & 31) == 0) {
            if (valid) *wp = acc32;
            --wp;
          }
        }
        if (act) {
          const std::uint32_t pa = (lp << r) | (u & (R - 1));
          const std::uint32_t pn = ((pa << r) | (pa >> (M - r))) & GEO::SMASK;  // undo the block relayout
          lp = pn >> r;
          u = (pn & (R - 1)) | hsh;
        }
      }
      continue;
    }
    std::uint64_t acc = 0;  // emitted bits, newest (lowest stage) at bit 0
    int nb = 0;
    // Round-uniform bounds (inactive lanes have st_t = -1 and sub_lo = v1).
    const int thi = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(st_t + 1))) - 1;
    const int tlo = static_cast<int>(__reduce_min_sync(kFull, active ? static_cast<unsigned>(sub_lo) : 0x7fffffffu));
    const int st_min = static_cast<int>(__reduce_min_sync(kFull, active ? static_cast<unsigned>(st_t) : 0x7fffffffu));
    const int lo_max = static_cast<int>(__reduce_max_sync(kFull, active ? static_cast<unsigned>(sub_lo) : 0u));
    const int hi_min = static_cast<int>(__reduce_min_sync(kFull, active ? static_cast<unsigned>(sub_hi) : 0x7fffffffu));
    const int hi_max = static_cast<int>(__reduce_max_sync(kFull, active ? static_cast<unsigned>(sub_hi) : 0u));
    auto emit = [&](int tb0, int jlo, int n, std::uint32_t bits) {
      acc = (acc << n) | bits;
      nb += n;
      if (nb >= 32) {
        // the oldest 32 bits: stages tb0 + jlo + (nb - 32) ... + 31
        const std::uint32_t word = static_cast<std::uint32_t>(acc >> (nb - 32));
        const std::int64_t ol = obase + tb0 + jlo + (nb - 32);
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
    for (int tb0 = thi & ~(LB - 1); tb0 >= (tlo & ~(LB - 1)); tb0 -= LB) {
      const std::uint32_t lp = P >> r;
      std::uint32_t wd[LB];
      if (TM && tb0 < t_split) {
        std::uint32_t own[4];
        tmem_ld4(bc.taddr + static_cast<std::uint32_t>(tb0 - t_first), own);
#pragma unroll
        for (int j = 0; j < LB; ++j) wd[j] = __shfl_sync(kFull, own[j], gcol + static_cast<int>(lp));
      } else if (GL && tb0 >= t_gl) {
#pragma unroll
        for (int j = 0; j < LB; ++j) wd[j] = bc.grow_lane[(tb0 + j - t_gl) * 32 - lane + gcol + static_cast<int>(lp)];
      } else {
#pragma unroll
        for (int j = 0; j < LB; ++j) {
          const int row = max(tb0 + j - s_base, 0);
          wd[j] = dec[row * 32 + gcol + lp];
        }
      }
      const std::uint32_t Pin = P;
      std::uint32_t u = (P & (R - 1)) | hsh;  // bit index into the word: register + 16 * half
      if (tb0 + LB - 1 <= st_min && tb0 >= lo_max) {
        // every task walks all LB phases of this block
#pragma unroll
        for (int j = LB - 1; j >= 0; --j) {
          const std::uint32_t dbit = (wd[j] >> u) & 1u;
          u = (u & ~(1u << j)) | (dbit << j);
        }
        P = (P & ~static_cast<std::uint32_t>(R - 1)) | (u & (R - 1));
        if (tb0 + LB - 1 < hi_min) {
          emit(tb0, 0, LB, Pin & ((1u << LB) - 1u));
        } else if (tb0 < hi_max) {
          const int ejhi = min(sub_hi - 1 - tb0, LB - 1);
          if (ejhi >= 0) emit(tb0, 0, ejhi + 1, Pin & ((1u << (ejhi + 1)) - 1u));
        }
        P = ((P << r) | (P >> (M - r))) & GEO::SMASK;  // undo the block relayout
      } else {
        const int jhi = st_t - tb0;  // phases jlo..jhi of this block are walked
        const int jlo = sub_lo > tb0 ? sub_lo - tb0 : 0;
#pragma unroll
        for (int j = LB - 1; j >= 0; --j) {
          const std::uint32_t dbit = (wd[j] >> u) & 1u;
          const std::uint32_t un = (u & ~(1u << j)) | (dbit << j);
          u = (j <= jhi && j >= jlo) ? un : u;
        }
        P = (P & ~static_cast<std::uint32_t>(R - 1)) | (u & (R - 1));
        const int ejhi = min(min(jhi, sub_hi - 1 - tb0), LB - 1);
        if (ejhi >= jlo) emit(tb0, jlo, ejhi - jlo + 1, (Pin >> jlo) & ((1u << (ejhi - jlo + 1)) - 1u));
        if (tb0 >= sub_lo && tb0 <= st_t) P = ((P << r) | (P >> (M - r))) & GEO::SMASK;  // undo the relayout
      }
    }
    if (nb > 0 && valid) {
      const std::uint32_t word = static_cast<std::uint32_t>(acc) & ((nb == 32) ? 0xffffffffu : ((1u << nb) - 1u));
      const std::int64_t ol = obase + sub_lo;
      const std::int64_t w0 = ol >> 5;
      const int o = static_cast<int>(ol & 31);
      atomicOr(p.out + w0, word << o);
      if (o + nb > 32) atomicOr(p.out + w0 + 1, word >> (32 - o));
    }
  }
  __syncwarp();  // this group's traceback reads are done before the next group's stores
  }  // mbase < mi1
  }  // rounds

  if constexpr (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase),
                   "r"(static_cast<unsigned>(fp.tm_alloc)));
    }
  }
}

}  // namespace fast
}  // namespace vd
