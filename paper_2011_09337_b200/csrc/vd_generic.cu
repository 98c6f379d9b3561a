// Generic unified Viterbi kernel for sm_100a: one warp per frame.
//
// This is the general-envelope path (any K in [2, 12], any B in [2, 8], any
// code, int8 LLRs with int32 metrics or double LLRs with double metrics).
// The throughput path for the benchmark codes is vd_fast.cu; this kernel
// serves every other code/config on the GPU, the FP64 real-valued API, and
// serial_decode's single long frame.
//
// Per frame (reference decode_frame, decoder.cpp:170-237), one warp:
//   forward pass over the clipped window [beg, end):
//     - stage table: lanes < 2^(B-1) evaluate branch_metric (decoder.cpp:22-30)
//       in the reference's add order, the other half by complement symmetry
//       (decoder.cpp:41-51);
//     - ACS over the S states, lane j owning states j, j+32, ... with the
//       reference's strict '>' (ties -> second predecessor, decoder.cpp:67-74);
//     - decisions are warp ballots: one bit per state per stage, bit-packed
//       32 states per word (shared memory when the frame fits, else a global
//       scratch slot per warp);
//     - argmax (lowest index on ties, decoder.cpp:80-90) at every subframe
//       start stage (decoder.cpp:205-211);
//   parallel traceback: subframe s is traced by lane s % 32
//   (decoder.cpp:214-236); output bits are OR-ed into packed words.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "vd_common.cuh"
#include "vd_internal.h"

namespace vd {
namespace {

constexpr int kWarps = 4;     // warps (frames in flight) per CTA
constexpr int kStage = 128;   // LLR staging depth (stages) per warp
constexpr int kTbChunk = 512; // traceback staging chunk (stages) for decisions held in global memory
#ifndef VD_TB1_SMEM
#define VD_TB1_SMEM 0  // 1: single-traceback walk also for shared-memory decisions (measured: FP64 3.6x slower)
#endif
constexpr unsigned kFull = 0xffffffffu;

struct GenericParams {
  DecodeLaunch p;
  int words;           // decision words per stage = ceil(S / 32)
  int len_max;         // max processed stages over the launched frames
  int nsub_max;        // max subframes per frame
  bool dec_in_smem;
  std::uint32_t* dec_global;  // [total_warps][len_max * words] when !dec_in_smem
  int smem_per_warp;          // bytes
  int stage_off, dec_off;     // byte offsets inside a warp's area
  int tb_off;                 // reg_kernel with global decisions: traceback staging (kTbChunk stages)
};

template <typename M>
__device__ __forceinline__ bool better(M v, int i, M bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

template <typename In, typename M>
__global__ void __launch_bounds__(kWarps * 32) generic_kernel(const GenericParams gp) {
  const DecodeLaunch& p = gp.p;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int S = p.s;
  const int words = gp.words;
  const std::uint32_t low_mask = static_cast<std::uint32_t>(S / 2 - 1);
  const int nt = 1 << p.b;
  const std::uint32_t half = 1u << (p.b - 1);
  const std::uint32_t tmask = static_cast<std::uint32_t>(nt - 1);

  unsigned char* base = smem_raw + static_cast<std::size_t>(warp) * gp.smem_per_warp;
  M* sig0 = reinterpret_cast<M*>(base);
  M* sig1 = sig0 + S;
  M* table = sig1 + S;
  int* start_state = reinterpret_cast<int*>(table + nt);
  // LLR staging: kStage stages of this frame's window, loaded cooperatively
  // (coalesced) by the warp once per kStage stages.
  In* stage_buf = reinterpret_cast<In*>(base + gp.stage_off);
  std::uint32_t* dec = reinterpret_cast<std::uint32_t*>(base + gp.dec_off);
  const std::int64_t gwarp = static_cast<std::int64_t>(blockIdx.x) * kWarps + warp;
  if (!gp.dec_in_smem) dec = gp.dec_global + gwarp * static_cast<std::int64_t>(gp.len_max) * words;

  const In* llr = static_cast<const In*>(p.llr);
  const std::int64_t total_warps = static_cast<std::int64_t>(gridDim.x) * kWarps;

  for (std::int64_t mi = p.frame_begin + gwarp; mi < p.frame_end; mi += total_warps) {
    const FrameRef fr = resolve_frame(p, mi);
    const std::int64_t m = fr.m;  // block-local frame index (geometry, random-start salt)
    const FrameGeom g(m, fr.n, p.f, p.v1, p.v2, p.f0);
    const std::int64_t len = g.len();
    M* sp = sig0;
    M* sc = sig1;
    for (int j = lane; j < S; j += 32) sp[j] = M(0);  // sigma_0 = 0 (decoder.cpp:195)
    std::int64_t offset = 0;                            // int32 renormalisation offset
    std::int64_t next_record = 0;
    std::int64_t next_start = g.start_stage(0, p.v2);
    __syncwarp();

    for (std::int64_t t = 0; t < len; ++t) {
      if ((t & (kStage - 1)) == 0) {
        const std::int64_t cnt = imin(kStage, len - t) * p.b;
        const In* src = llr + (fr.base + g.beg + t - p.llr_stage0) * p.b;
        __syncwarp();
        for (std::int64_t i = lane; i < cnt; i += 32) stage_buf[i] = src[i];
        __syncwarp();
      }
      const In* lt = stage_buf + (t & (kStage - 1)) * p.b;
      // Stage table (decoder.cpp:41-51): direct half, then complements.
      for (std::uint32_t bo = lane; bo < half; bo += 32) {
        M acc = M(0);
        for (int i = 0; i < p.b; ++i) {
          const M v = static_cast<M>(lt[i]);
          acc += ((bo >> (p.b - 1 - i)) & 1u) ? -v : v;
        }
        table[bo] = acc;
      }
      __syncwarp();
      for (std::uint32_t bo = half + lane; bo <= tmask; bo += 32) table[bo] = -table[bo ^ tmask];
      __syncwarp();
      // ACS (decoder.cpp:53-76).
      for (int r = 0; r < words; ++r) {
        const int j = r * 32 + lane;
        bool d = false;
        if (j < S) {
          const std::uint32_t i1 = (static_cast<std::uint32_t>(j) & low_mask) << 1;
          const M s1 = sp[i1] + table[__ldg(p.in_out + 2 * j)];
          const M s2 = sp[i1 | 1] + table[__ldg(p.in_out + 2 * j + 1)];
          d = !(s1 > s2);
          sc[j] = d ? s2 : s1;
        }
        const std::uint32_t w = __ballot_sync(kFull, d);
        if (lane == 0) dec[t * words + r] = w;
      }
      __syncwarp();
      M* tmp = sp;
      sp = sc;
      sc = tmp;
      if constexpr (std::is_integral<M>::value) {
        // Keep int32 metrics far from overflow on long frames; the offset is
        // re-added for metric export. Differences (hence decisions) are exact.
        if ((t & 4095) == 4095) {
          const M ref = sp[0];
          __syncwarp();
          for (int j = lane; j < S; j += 32) sp[j] -= ref;
          offset += ref;
          __syncwarp();
        }
      }
      // Stored-max start states (decoder.cpp:205-211).
      while (next_record < g.num_sub && next_start == t) {
        M bv = sp[0];
        int bi = 0;
        bool have = false;
        for (int j = lane; j < S; j += 32) {
          if (!have || sp[j] > bv) {
            bv = sp[j];
            bi = j;
            have = true;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const M ov = __shfl_xor_sync(kFull, bv, o);
          const int oi = __shfl_xor_sync(kFull, bi, o);
          const bool oh = __shfl_xor_sync(kFull, have ? 1 : 0, o) != 0;
          if (oh && (!have || better(ov, oi, bv, bi))) {
            bv = ov;
            bi = oi;
            have = true;
          }
        }
        if (lane == 0) start_state[next_record] = bi;
        ++next_record;
        if (next_record < g.num_sub) next_start = g.start_stage(next_record, p.v2);
      }
    }
    __syncwarp();

    if (p.sigma) {
      for (int j = lane; j < S; j += 32) {
        if constexpr (std::is_integral<M>::value) {
          static_cast<std::int64_t*>(p.sigma)[(mi - p.frame_begin) * S + j] = static_cast<std::int64_t>(sp[j]) + offset;
        } else {
          static_cast<double*>(p.sigma)[(mi - p.frame_begin) * S + j] = sp[j];
        }
      }
    }

    // Parallel traceback (decoder.cpp:214-236): lane owns subframes s = lane mod 32.
    for (std::int64_t s = lane; s < g.num_sub; s += 32) {
      const std::int64_t st = g.start_stage(s, p.v2);
      const std::int64_t lo = g.sub_lo(s), hi = g.sub_hi(s);
      std::uint32_t state;
      if (p.f0 > 0 && p.start == 1 && st < len - 1) {
        state = static_cast<std::uint32_t>(mix_seed(p.seed, static_cast<std::uint64_t>(m) * 0x10001ull +
                                                                static_cast<std::uint64_t>(s)) %
                                           static_cast<std::uint64_t>(S));
      } else {
        state = static_cast<std::uint32_t>(start_state[s]);
      }
      std::uint32_t acc = 0;
      std::int64_t cur = -1;
      for (std::int64_t t = st; t >= lo - g.beg; --t) {
        const std::int64_t stage = g.beg + t;
        if (stage < hi) {
          const std::int64_t rel = fr.base + stage - p.out_stage0;
          const std::int64_t w = rel >> 5;
          if (w != cur) {
            if (cur >= 0 && acc) atomicOr(p.out + cur, acc);
            cur = w;
            acc = 0;
          }
          acc |= (state >> (p.k - 2)) << (rel & 31);
        }
        const std::uint32_t d = (dec[t * words + (state >> 5)] >> (state & 31)) & 1u;
        state = ((state & low_mask) << 1) | d;
      }
      if (cur >= 0 && acc) atomicOr(p.out + cur, acc);
    }
    __syncwarp();
  }
}

// Register-resident variant for S <= 256 (K <= 9), the latency path for the
// few edge frames around every fast-kernel launch and the throughput path for
// the FP64 API. Same algorithm and outputs as generic_kernel above; lane j owns
// states j, j+32, ... in registers, so the critical chain of a stage is
// shuffle -> add -> compare -> select (no shared-memory round trip or
// __syncwarp between stages). Branch metrics are evaluated per lane straight
// from the stage LLRs in the reference's add order (decoder.cpp:41-51).
// BT > 0: B known at compile time (2, 3, 4): the stage's 2^(B-1) direct
// branch metrics are computed once per stage in the reference's add order
// and each state edge picks its entry (+ sign) with a precomputed index
// (BT = 0: any B, evaluated per edge).
template <typename In, typename M, int NPL, int BT>
__global__ void __launch_bounds__(kWarps * 32) reg_kernel(const GenericParams gp) {
  const DecodeLaunch& p = gp.p;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int S = p.s;
  const int b = BT > 0 ? BT : p.b;
  const std::uint32_t half = 1u << (b - 1);
  const std::uint32_t tmask = (1u << b) - 1u;

  unsigned char* base = smem_raw + static_cast<std::size_t>(warp) * gp.smem_per_warp;
  int* start_state = reinterpret_cast<int*>(base);
  In* stage_buf = reinterpret_cast<In*>(base + gp.stage_off);
  std::uint32_t* dec = reinterpret_cast<std::uint32_t*>(base + gp.dec_off);
  const std::int64_t gwarp = static_cast<std::int64_t>(blockIdx.x) * kWarps + warp;
  if (!gp.dec_in_smem) dec = gp.dec_global + gwarp * static_cast<std::int64_t>(gp.len_max) * NPL;

  // Branch labels of this lane's states: table index (sign pattern) and
  // whether the entry is the complement of the direct half.
  std::uint32_t lab[NPL][2];
  bool valid[NPL];
#pragma unroll
  for (int r = 0; r < NPL; ++r) {
    const int j = r * 32 + lane;
    valid[r] = j < S;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const std::uint32_t x = valid[r] ? __ldg(p.in_out + 2 * j + e) : 0u;
      lab[r][e] = x;
    }
  }
  // predecessor lanes
  const int low = S / 2 - 1;
  const int srcA = NPL == 1 ? (((lane & low) << 1) & 31) : ((2 * lane) & 31);
  const int srcB = NPL == 1 ? ((((lane & low) << 1) | 1) & 31) : ((2 * lane + 1) & 31);
  const bool upper = lane >= 16;

  const In* llr = static_cast<const In*>(p.llr);
  const std::int64_t total_warps = static_cast<std::int64_t>(gridDim.x) * kWarps;

  auto bm = [&](const M* v, std::uint32_t x) -> M {
    const bool neg = x >= half;
    const std::uint32_t xs = neg ? (x ^ tmask) : x;
    M acc = M(0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < b) acc += ((xs >> (b - 1 - i)) & 1u) ? -v[i] : v[i];
    }
    return neg ? -acc : acc;
  };
  // compile-time-B form: per edge, direct-table index and complement flag
  constexpr int NT = BT > 0 ? (1 << (BT - 1)) : 1;
  std::uint32_t eidx[NPL][2];
  bool eneg[NPL][2];
#pragma unroll
  for (int r = 0; r < NPL; ++r) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      eneg[r][e] = lab[r][e] >= half;
      eidx[r][e] = eneg[r][e] ? (lab[r][e] ^ tmask) : lab[r][e];
    }
  }
  auto stage_table = [&](const M* v, M (&T)[NT]) {
#pragma unroll
    for (int x = 0; x < NT; ++x) {
      M acc = M(0);  // reference decoder.cpp:22-30 order: 0 + (+/-v0) + (+/-v1) ...
#pragma unroll
      for (int i = 0; i < (BT > 0 ? BT : 1); ++i) acc += ((x >> ((BT > 0 ? BT : 1) - 1 - i)) & 1) ? -v[i] : v[i];
      T[x] = acc;
    }
  };
  auto pick = [&](const M (&T)[NT], std::uint32_t idx, bool neg) -> M {
    M val = T[0];
#pragma unroll
    for (int x = 1; x < NT; ++x) val = idx == static_cast<std::uint32_t>(x) ? T[x] : val;
    return neg ? -val : val;
  };

  for (std::int64_t mi = p.frame_begin + gwarp; mi < p.frame_end; mi += total_warps) {
    const FrameRef fr = resolve_frame(p, mi);
    const std::int64_t m = fr.m;  // block-local frame index (geometry, random-start salt)
    const FrameGeom g(m, fr.n, p.f, p.v1, p.v2, p.f0);
    const std::int64_t len = g.len();
    M sig[NPL];
#pragma unroll
    for (int r = 0; r < NPL; ++r) sig[r] = M(0);  // sigma_0 = 0 (decoder.cpp:195)
    std::int64_t offset = 0;
    int next_record = 0;
    int next_start = static_cast<int>(g.start_stage(0, p.v2));
    const In* src = llr + (fr.base + g.beg - p.llr_stage0) * b;
    const int len32 = static_cast<int>(len);  // frame windows < 2^31 stages (checked at launch)

    auto refill = [&](int t) {
      const int cnt = (kStage < len32 - t ? kStage : len32 - t) * b;
      __syncwarp();
      for (int i = lane; i < cnt; i += 32) stage_buf[i] = src[static_cast<std::int64_t>(t) * b + i];
      __syncwarp();
    };
    M v[8];
    if (len > 0) {
      refill(0);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = i < b ? static_cast<M>(stage_buf[i]) : M(0);
    }
    for (int t = 0; t < len32; ++t) {
      M bmv[NPL][2];
      if constexpr (BT > 0) {
        M T[NT];
        stage_table(v, T);
#pragma unroll
        for (int r = 0; r < NPL; ++r) {
          bmv[r][0] = pick(T, eidx[r][0], eneg[r][0]);
          bmv[r][1] = pick(T, eidx[r][1], eneg[r][1]);
        }
      } else {
#pragma unroll
        for (int r = 0; r < NPL; ++r) {
          bmv[r][0] = bm(v, lab[r][0]);
          bmv[r][1] = bm(v, lab[r][1]);
        }
      }
      if (t + 1 < len32) {  // software pipeline: next stage's LLRs
        if (((t + 1) & (kStage - 1)) == 0) refill(t + 1);
        const In* lt = stage_buf + ((t + 1) & (kStage - 1)) * b;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = i < b ? static_cast<M>(lt[i]) : M(0);
      }
      // ACS (decoder.cpp:53-76): ties -> second predecessor.
      M nsig[NPL];
      bool d[NPL];
#pragma unroll
      for (int q = 0; q < (NPL == 1 ? 1 : NPL / 2); ++q) {
        M pa, pb;
        if constexpr (NPL == 1) {
          pa = __shfl_sync(kFull, sig[0], srcA);
          pb = __shfl_sync(kFull, sig[0], srcB);
        } else {
          const M a0 = __shfl_sync(kFull, sig[2 * q], srcA);
          const M a1 = __shfl_sync(kFull, sig[2 * q + 1], srcA);
          const M b0 = __shfl_sync(kFull, sig[2 * q], srcB);
          const M b1 = __shfl_sync(kFull, sig[2 * q + 1], srcB);
          pa = upper ? a1 : a0;
          pb = upper ? b1 : b0;
        }
#pragma unroll
        for (int h = 0; h < (NPL == 1 ? 1 : 2); ++h) {
          const int r = q + h * (NPL / 2);
          const M s1 = pa + bmv[r][0];
          const M s2 = pb + bmv[r][1];
          d[r] = !(s1 > s2);
          nsig[r] = d[r] ? s2 : s1;
        }
      }
#pragma unroll
      for (int r = 0; r < NPL; ++r) {
        sig[r] = nsig[r];
        const std::uint32_t w = __ballot_sync(kFull, d[r] && valid[r]);
        if (lane == r) dec[t * NPL + r] = w;
      }
      if constexpr (std::is_integral<M>::value) {
        if ((t & 4095) == 4095) {  // int32 renormalisation (exact differences)
          const M ref = __shfl_sync(kFull, sig[0], 0);
#pragma unroll
          for (int r = 0; r < NPL; ++r) sig[r] -= ref;
          offset += ref;
        }
      }
      // Stored-max start states (decoder.cpp:205-211): lowest index on ties.
      while (next_record < g.num_sub && next_start == t) {
        M bv = sig[0];
        int bi = lane;
        bool have = valid[0];
#pragma unroll
        for (int r = 1; r < NPL; ++r) {
          if (valid[r] && (!have || sig[r] > bv)) {
            bv = sig[r];
            bi = r * 32 + lane;
            have = true;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const M ov = __shfl_xor_sync(kFull, bv, o);
          const int oi = __shfl_xor_sync(kFull, bi, o);
          const bool oh = __shfl_xor_sync(kFull, have ? 1 : 0, o) != 0;
          if (oh && (!have || better(ov, oi, bv, bi))) {
            bv = ov;
            bi = oi;
            have = true;
          }
        }
        if (lane == 0) start_state[next_record] = bi;
        ++next_record;
        if (next_record < g.num_sub) next_start = static_cast<int>(g.start_stage(next_record, p.v2));
      }
    }
    __syncwarp();

    if (p.sigma) {
#pragma unroll
      for (int r = 0; r < NPL; ++r) {
        const int j = r * 32 + lane;
        if (!valid[r]) continue;
        if constexpr (std::is_integral<M>::value) {
          static_cast<std::int64_t*>(p.sigma)[(mi - p.frame_begin) * S + j] = static_cast<std::int64_t>(sig[r]) + offset;
        } else {
          static_cast<double*>(p.sigma)[(mi - p.frame_begin) * S + j] = sig[r];
        }
      }
    }

    // Parallel traceback (decoder.cpp:214-236): lane owns subframes s = lane mod 32.
    // The decision words of 4 stages are loaded before the state chain walks
    // them, so the chain is select + shift instead of a load per stage.
    const std::uint32_t lmask = static_cast<std::uint32_t>(S / 2 - 1);
    const bool tb1 = g.num_sub == 1 && (VD_TB1_SMEM || !gp.dec_in_smem);
    if (tb1) {
      // One traceback per frame (f0 == 0, serial_decode): lane 0 walks from
      // the stored-max state with the decision words of 8 stages loaded ahead
      // (they do not depend on the traced path), so the state chain is pure
      // ALU; emitted bits gather in a 32-bit word flushed every 32 stages.
      // Decisions held in global memory (long frames) are first staged into
      // shared memory in chunks of kTbChunk stages with coalesced loads.
      std::uint32_t* tb = reinterpret_cast<std::uint32_t*>(base + gp.tb_off);
      const int st = static_cast<int>(g.start_stage(0, p.v2));
      const int tend = static_cast<int>(g.sub_lo(0) - g.beg);
      const int temit = static_cast<int>(g.sub_hi(0) - g.beg);  // stages t < temit emit a bit
      const std::int64_t rel0 = fr.base + g.beg - p.out_stage0;  // output bit of stage t = 0
      const std::uint32_t rlo = static_cast<std::uint32_t>(rel0);
      const int ksh = p.k - 2;
      std::uint32_t state = static_cast<std::uint32_t>(start_state[0]);  // num_sub == 1: stored max
      std::uint32_t acc = 0;
      auto step = [&](int t, std::uint32_t word) {
        if (t < temit) {
          const std::uint32_t pos = (rlo + static_cast<std::uint32_t>(t)) & 31u;
          acc |= (state >> ksh) << pos;
          if (pos == 0 || t == tend) {
            if (acc) atomicOr(p.out + ((rel0 + t) >> 5), acc);
            acc = 0;
          }
        }
        state = ((state & lmask) << 1) | ((word >> (state & 31)) & 1u);
      };
      for (int chi = st; chi >= tend; chi -= kTbChunk) {
        const int clo = chi - kTbChunk + 1 > tend ? chi - kTbChunk + 1 : tend;
        const std::uint32_t* src = dec;
        if (!gp.dec_in_smem) {
          const int cnt = (chi - clo + 1) * NPL;
          __syncwarp();
          for (int i = lane; i < cnt; i += 32) tb[i] = dec[clo * NPL + i];
          __syncwarp();
          src = tb - clo * NPL;
        }
        if (lane == 0) {
          int t = chi;
          for (; t - 7 >= clo; t -= 8) {
            std::uint32_t wv[8][NPL];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
#pragma unroll
              for (int r = 0; r < NPL; ++r) wv[u][r] = src[(t - u) * NPL + r];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              std::uint32_t word = wv[u][0];
#pragma unroll
              for (int r = 1; r < NPL; ++r) word = (state >> 5) == static_cast<std::uint32_t>(r) ? wv[u][r] : word;
              step(t - u, word);
            }
          }
          for (; t >= clo; --t) step(t, src[t * NPL + (NPL > 1 ? (state >> 5) : 0)]);
        }
      }
    }
    for (std::int64_t s = lane; s < g.num_sub && !tb1; s += 32) {
      const std::int64_t st = g.start_stage(s, p.v2);
      const std::int64_t lo = g.sub_lo(s), hi = g.sub_hi(s);
      std::uint32_t state;
      if (p.f0 > 0 && p.start == 1 && st < len - 1) {
        state = static_cast<std::uint32_t>(mix_seed(p.seed, static_cast<std::uint64_t>(m) * 0x10001ull +
                                                                static_cast<std::uint64_t>(s)) %
                                           static_cast<std::uint64_t>(S));
      } else {
        state = static_cast<std::uint32_t>(start_state[s]);
      }
      std::uint32_t acc = 0;
      std::int64_t cur = -1;
      const std::int64_t tend = lo - g.beg;
      auto step_one = [&](std::int64_t t, std::uint32_t word) {
        const std::int64_t stage = g.beg + t;
        if (stage < hi) {
          const std::int64_t rel = fr.base + stage - p.out_stage0;
          const std::int64_t w = rel >> 5;
          if (w != cur) {
            if (cur >= 0 && acc) atomicOr(p.out + cur, acc);
            cur = w;
            acc = 0;
          }
          acc |= (state >> (p.k - 2)) << (rel & 31);
        }
        state = ((state & lmask) << 1) | ((word >> (state & 31)) & 1u);
      };
      std::int64_t t = st;
      for (; t - 3 >= tend; t -= 4) {
        std::uint32_t wv[4][NPL];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int r = 0; r < NPL; ++r) wv[u][r] = dec[(t - u) * NPL + r];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          std::uint32_t word = wv[u][0];
#pragma unroll
          for (int r = 1; r < NPL; ++r) word = (state >> 5) == static_cast<std::uint32_t>(r) ? wv[u][r] : word;
          step_one(t - u, word);
        }
      }
      for (; t >= tend; --t) step_one(t, dec[t * NPL + (state >> 5)]);
      if (cur >= 0 && acc) atomicOr(p.out + cur, acc);
    }
    __syncwarp();
  }
}

template <typename In, typename M, int NPL, int BT>
cudaError_t launch_reg(GenericParams gp, cudaStream_t stream) {
  const DecodeLaunch& p = gp.p;
  const std::int64_t frames = p.frame_end - p.frame_begin;
  const std::size_t head = (sizeof(int) * gp.nsub_max + 15) & ~std::size_t(15);
  const std::size_t stage_bytes = (sizeof(In) * kStage * p.b + 15) & ~std::size_t(15);
  gp.stage_off = static_cast<int>(head);
  gp.dec_off = static_cast<int>(head + stage_bytes);
  const std::size_t dec_bytes = sizeof(std::uint32_t) * static_cast<std::size_t>(gp.len_max) * NPL;
  constexpr std::size_t kSmemBudget = 200 * 1024;
  gp.dec_in_smem = (head + stage_bytes + dec_bytes) * kWarps <= kSmemBudget;
  const std::size_t tb_bytes = sizeof(std::uint32_t) * kTbChunk * NPL;
  gp.tb_off = static_cast<int>(head + stage_bytes);
  const std::size_t per_warp =
      ((gp.dec_in_smem ? head + stage_bytes + dec_bytes : head + stage_bytes + tb_bytes) + 15) & ~std::size_t(15);
  if (per_warp * kWarps > kSmemBudget) return cudaErrorInvalidValue;
  gp.smem_per_warp = static_cast<int>(per_warp);
  std::int64_t blocks = (frames + kWarps - 1) / kWarps;
  const int occ_blocks = sm_count() * 8;
  if (blocks > occ_blocks) blocks = occ_blocks;
  gp.dec_global = nullptr;
  if (!gp.dec_in_smem) {
    const std::size_t bytes = dec_bytes * static_cast<std::size_t>(blocks) * kWarps;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&gp.dec_global), bytes, stream);
    if (e != cudaSuccess) return e;
  }
  const std::size_t smem = per_warp * kWarps;
  auto kern = reg_kernel<In, M, NPL, BT>;
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
  if (e == cudaSuccess) {
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, stream>>>(gp);
    note_launch();
    e = cudaGetLastError();
  }
  if (gp.dec_global) {
    const cudaError_t e2 = cudaFreeAsync(gp.dec_global, stream);
    if (e == cudaSuccess) e = e2;
  }
  return e;
}

template <typename In, typename M>
cudaError_t launch_generic(const DecodeLaunch& p, cudaStream_t stream) {
  GenericParams gp;
  gp.p = p;
  gp.words = (p.s + 31) / 32;
  // Upper bounds over all frames: the window is at most f + v1 + v2 stages
  // (clipped to the stream) and a frame has at most ceil(f / f0) subframes.
  const std::int64_t len_max = imin(static_cast<std::int64_t>(p.f) + p.v1 + p.v2, p.n);
  const std::int64_t nsub_max = p.f0 > 0 ? (static_cast<std::int64_t>(p.f) + p.f0 - 1) / p.f0 : 1;
  if (len_max > 0x7fffffffLL / gp.words) return cudaErrorInvalidValue;
  gp.len_max = static_cast<int>(len_max);
  gp.nsub_max = static_cast<int>(nsub_max);
  const std::int64_t frames = p.frame_end - p.frame_begin;
  if (frames <= 0) return cudaSuccess;

  if (p.s <= 256) {
    const int npl = p.s <= 32 ? 1 : p.s / 32;
    auto by_b = [&](auto npl_tag) -> cudaError_t {
      constexpr int NPLc = decltype(npl_tag)::value;
      switch (p.b) {
        case 2: return launch_reg<In, M, NPLc, 2>(gp, stream);
        case 3: return launch_reg<In, M, NPLc, 3>(gp, stream);
        default: return launch_reg<In, M, NPLc, 0>(gp, stream);
      }
    };
    switch (npl) {
      case 1: return by_b(std::integral_constant<int, 1>{});
      case 2: return by_b(std::integral_constant<int, 2>{});
      case 4: return by_b(std::integral_constant<int, 4>{});
      case 8: return by_b(std::integral_constant<int, 8>{});
      default: break;
    }
  }
  const std::size_t head = sizeof(M) * (2 * p.s + (1 << p.b)) + sizeof(int) * (gp.nsub_max + (gp.nsub_max & 1));
  const std::size_t head_al = (head + 15) & ~std::size_t(15);
  const std::size_t stage_bytes = (sizeof(In) * kStage * p.b + 15) & ~std::size_t(15);
  gp.stage_off = static_cast<int>(head_al);
  gp.dec_off = static_cast<int>(head_al + stage_bytes);
  const std::size_t dec_bytes = sizeof(std::uint32_t) * static_cast<std::size_t>(len_max) * gp.words;
  constexpr std::size_t kSmemBudget = 200 * 1024;
  gp.dec_in_smem = (head_al + stage_bytes + dec_bytes) * kWarps <= kSmemBudget;
  const std::size_t per_warp =
      ((gp.dec_in_smem ? head_al + stage_bytes + dec_bytes : head_al + stage_bytes) + 15) & ~std::size_t(15);
  if (per_warp * kWarps > kSmemBudget) return cudaErrorInvalidValue;  // K too large for this kernel
  gp.smem_per_warp = static_cast<int>(per_warp);

  std::int64_t blocks = (frames + kWarps - 1) / kWarps;
  const int occ_blocks = sm_count() * 8;
  if (blocks > occ_blocks) blocks = occ_blocks;
  gp.dec_global = nullptr;
  if (!gp.dec_in_smem) {
    const std::size_t bytes = dec_bytes * static_cast<std::size_t>(blocks) * kWarps;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&gp.dec_global), bytes, stream);
    if (e != cudaSuccess) return e;
  }
  const std::size_t smem = per_warp * kWarps;
  auto kern = generic_kernel<In, M>;
  cudaError_t e = allow_max_smem(reinterpret_cast<const void*>(kern));
  if (e == cudaSuccess) {
    kern<<<static_cast<unsigned>(blocks), kWarps * 32, smem, stream>>>(gp);
    note_launch();
    e = cudaGetLastError();
  }
  if (gp.dec_global) {
    const cudaError_t e2 = cudaFreeAsync(gp.dec_global, stream);
    if (e == cudaSuccess) e = e2;
  }
  return e;
}

}  // namespace

cudaError_t launch_generic_i8(const DecodeLaunch& p, cudaStream_t stream) {
  if (p.k > kMaxGenericK) return launch_bigk_i8(p, stream);  // CTA-per-frame path (vd_bigk.cu)
  return launch_generic<std::int8_t, std::int32_t>(p, stream);
}

cudaError_t launch_generic_f64(const DecodeLaunch& p, cudaStream_t stream) {
  if (p.k > kMaxGenericK) return launch_bigk_f64(p, stream);
  return launch_generic<double, double>(p, stream);
}

}  // namespace vd
