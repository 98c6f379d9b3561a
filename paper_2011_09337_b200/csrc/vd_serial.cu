// Exact parallel decode of ONE long frame (reference serial_decode,
// decoder.cpp:101-129, and framed_decode frames with f >= N): the forward
// recursion sigma_t = A_t (x) sigma_{t-1} is a max-plus matrix-vector
// product, and max-plus products are associative and exact on integers, so
// the stage chain is cut into segments:
//
//   A  segment_matrix_kernel  per segment g and start state j (one warp each):
//      the forward pass from the unit vector e_j (0 at j, -inf elsewhere)
//      gives column j of the segment transfer matrix M_g (M_g[i][j] = best
//      metric of a path j -> i through the segment). No decisions.
//   B  boundary metrics sigma_g by a two-level max-plus scan: products of
//      groups of 32 segment matrices (group_product_kernel, parallel), a
//      sequential mat-vec chain over the group products, then each group's
//      own chain from its start metrics in parallel (chain_matvec_kernel).
//   C  segment_forward_kernel per segment (one warp each): the ordinary
//      forward pass from the exact sigma_g, storing the decision words; the
//      last segment also takes the argmax of the final metrics (lowest state
//      on ties, decoder.cpp:80-90).
//   D1 segment_map_kernel     per segment: trace back from every end state
//      through the segment (one chain per state) -> map_g[state].
//   D2 chain_kernel           one warp: end state of every segment by
//      composing the maps from the final argmax (maps prefetched 8 ahead).
//   D3 segment_emit_kernel    per segment: trace back from its end state and
//      write its decoded bits.
//
// Decisions are computed from the same integer metrics up to a per-segment
// common offset, so every decision (ties included, decoder.cpp:67-74) and the
// decoded bits are identical to the sequential decode. int8 LLRs only (double
// sums are not associative).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>

#include "vd_common.cuh"
#include "vd_internal.h"

namespace vd {
namespace {

#ifndef VD_SERIAL_COLS
#define VD_SERIAL_COLS 1
#endif

constexpr unsigned kFull = 0xffffffffu;
constexpr std::int32_t kNeg = -(1 << 28);  // "-inf" for the unit start vectors

struct SerialParams {
  const std::int8_t* llr;  // stage beg of the frame window
  int k, b, s;
  std::int64_t len;        // window stages
  int seg_len, nseg;
  const std::uint32_t* in_out;
  std::uint32_t polys[4];
  std::int32_t* mat;       // [nseg][S (j)][S (i)]: column-major per segment
  std::int64_t* sig0;      // [nseg + 1][S]: metrics before each segment
  std::uint32_t* dec;      // [len][NPL] decision words
  std::int32_t* map;       // [nseg][S]
  std::int32_t* endst;     // [nseg]: traced state at each segment's last stage; endst[nseg] = final argmax
  std::uint32_t* out;      // packed output, bit of window stage t at out_bit0 + t
  std::int64_t out_bit0;
  std::int64_t emit_lo, emit_hi;  // window stages whose bits are written
};

template <int NPL, int BT>
struct Lane {
  std::uint32_t eidx[NPL][2];
  bool eneg[NPL][2];
  int srcA, srcB;
  bool upper;
  __device__ void init(const SerialParams& p, int lane) {
    const std::uint32_t half = 1u << (BT - 1), tmask = (1u << BT) - 1u;
#pragma unroll
    for (int r = 0; r < NPL; ++r) {
      const int j = r * 32 + lane;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const std::uint32_t x = j < p.s ? __ldg(p.in_out + 2 * j + e) : 0u;
        eneg[r][e] = x >= half;
        eidx[r][e] = eneg[r][e] ? (x ^ tmask) : x;
      }
    }
    const int low = p.s / 2 - 1;
    srcA = NPL == 1 ? (((lane & low) << 1) & 31) : ((2 * lane) & 31);
    srcB = NPL == 1 ? ((((lane & low) << 1) | 1) & 31) : ((2 * lane + 1) & 31);
    upper = lane >= 16;
  }
  // one ACS stage (reference decoder.cpp:53-76); returns the decision bits
  __device__ __forceinline__ void stage(const std::int8_t* l, std::int32_t (&sig)[NPL], bool (&d)[NPL]) const {
    constexpr int NT = 1 << (BT - 1);
    std::int32_t v[BT];
#pragma unroll
    for (int i = 0; i < BT; ++i) v[i] = l[i];
    std::int32_t T[NT];
#pragma unroll
    for (int x = 0; x < NT; ++x) {
      std::int32_t acc = 0;
#pragma unroll
      for (int i = 0; i < BT; ++i) acc += ((x >> (BT - 1 - i)) & 1) ? -v[i] : v[i];
      T[x] = acc;
    }
    auto pick = [&](std::uint32_t idx, bool neg) {
      std::int32_t val = T[0];
#pragma unroll
      for (int x = 1; x < NT; ++x) val = idx == static_cast<std::uint32_t>(x) ? T[x] : val;
      return neg ? -val : val;
    };
    std::int32_t ns[NPL];
#pragma unroll
    for (int q = 0; q < (NPL == 1 ? 1 : NPL / 2); ++q) {
      std::int32_t pa, pb;
      if constexpr (NPL == 1) {
        pa = __shfl_sync(kFull, sig[0], srcA);
        pb = __shfl_sync(kFull, sig[0], srcB);
      } else {
        const std::int32_t a0 = __shfl_sync(kFull, sig[2 * q], srcA), a1 = __shfl_sync(kFull, sig[2 * q + 1], srcA);
        const std::int32_t b0 = __shfl_sync(kFull, sig[2 * q], srcB), b1 = __shfl_sync(kFull, sig[2 * q + 1], srcB);
        pa = upper ? a1 : a0;
        pb = upper ? b1 : b0;
      }
#pragma unroll
      for (int h = 0; h < (NPL == 1 ? 1 : 2); ++h) {
        const int r = q + h * (NPL / 2);
        const std::int32_t s1 = pa + pick(eidx[r][0], eneg[r][0]);
        const std::int32_t s2 = pb + pick(eidx[r][1], eneg[r][1]);
        d[r] = !(s1 > s2);  // ties -> second predecessor
        ns[r] = d[r] ? s2 : s1;
      }
    }
#pragma unroll
    for (int r = 0; r < NPL; ++r) sig[r] = ns[r];
  }
};

template <int NPL, int BT>
__global__ void __launch_bounds__(128) segment_matrix_kernel(const SerialParams p) {
  const int lane = threadIdx.x & 31;
  const std::int64_t wid = static_cast<std::int64_t>(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (wid >= static_cast<std::int64_t>(p.nseg) * p.s) return;  // whole warps only
  const int g = static_cast<int>(wid / p.s), j = static_cast<int>(wid % p.s);
  Lane<NPL, BT> ln;
  ln.init(p, lane);
  std::int32_t sig[NPL];
#pragma unroll
  for (int r = 0; r < NPL; ++r) sig[r] = (r * 32 + lane == j) ? 0 : kNeg;
  const std::int64_t t0 = static_cast<std::int64_t>(g) * p.seg_len;
  const std::int64_t t1 = t0 + p.seg_len < p.len ? t0 + p.seg_len : p.len;
  bool d[NPL];
  for (std::int64_t t = t0; t < t1; ++t) ln.stage(p.llr + t * BT, sig, d);
  std::int32_t* col = p.mat + (static_cast<std::int64_t>(g) * p.s + j) * p.s;
#pragma unroll
  for (int r = 0; r < NPL; ++r) {
    const int i = r * 32 + lane;
    if (i < p.s) col[i] = sig[r];
  }
}

// Kernel A for codes known at compile time (the common standards): one LANE
// per column j — all S states of the column live in the lane's registers, so
// a stage is S x (IADD3 + VIADDMNMX-style max) with compile-time branch-table
// picks and no shuffles (the stage's LLRs and table are warp-uniform): ~2
// instructions per column-state instead of ~18 for the warp-per-column form.
template <int K_, int B_, std::uint32_t P0, std::uint32_t P1, std::uint32_t P2 = 0>
struct SCode {
  static constexpr int K = K_, B = B_, S = 1 << (K_ - 1);
  static constexpr std::uint32_t poly(int i) { return i == 0 ? P0 : i == 1 ? P1 : P2; }
  // branch output of (state s, input u), polys[0] at the MSB (trellis.cpp:65-79)
  static constexpr std::uint32_t out(std::uint32_t st, std::uint32_t u) {
    const std::uint32_t reg = (u << (K - 1)) | st;
    std::uint32_t bo = 0;
    for (int b = 0; b < B; ++b) {
      std::uint32_t x = poly(b) & reg, par = 0;
      while (x) {
        par ^= x & 1u;
        x >>= 1;
      }
      bo |= par << (B - 1 - b);
    }
    return bo;
  }
  // incoming output of state j from predecessor w (trellis.cpp:81-91)
  static constexpr std::uint32_t in_out(int j, int w) {
    const std::uint32_t pred = 2u * (static_cast<std::uint32_t>(j) & (S / 2 - 1)) + static_cast<std::uint32_t>(w);
    return out(pred, static_cast<std::uint32_t>(j) >> (K - 2));
  }
  static bool matches(int k, int b, const std::uint32_t* p) {
    if (k != K || b != B) return false;
    for (int i = 0; i < B; ++i) {
      if (p[i] != poly(i)) return false;
    }
    return true;
  }
};

template <class C>
__global__ void __launch_bounds__(64) segment_matrix_cols_kernel(const SerialParams p) {
  constexpr int S = C::S, B = C::B, NT = 1 << (B - 1);
  constexpr std::uint32_t half = 1u << (B - 1), tmask = (1u << B) - 1u;
  const std::int64_t col = static_cast<std::int64_t>(blockIdx.x) * 64 + threadIdx.x;  // g * S + j
  if (col >= static_cast<std::int64_t>(p.nseg) * S) return;
  const int g = static_cast<int>(col / S), j = static_cast<int>(col % S);
  std::int32_t sig[S];
#pragma unroll
  for (int i = 0; i < S; ++i) sig[i] = i == j ? 0 : kNeg;
  const std::int64_t t0 = static_cast<std::int64_t>(g) * p.seg_len;
  const std::int64_t t1 = t0 + p.seg_len < p.len ? t0 + p.seg_len : p.len;
  // one stage: sig <- A_t (x) sig (values only; ties do not matter here)
  auto stage = [&](std::int64_t t) {
    const std::int8_t* l = p.llr + t * B;
    std::int32_t v[B];
#pragma unroll
    for (int i = 0; i < B; ++i) v[i] = l[i];
    std::int32_t T[NT];
#pragma unroll
    for (int x = 0; x < NT; ++x) {
      std::int32_t acc = 0;
#pragma unroll
      for (int i = 0; i < B; ++i) acc += ((x >> (B - 1 - i)) & 1) ? -v[i] : v[i];
      T[x] = acc;
    }
    std::int32_t ns[S];
#pragma unroll
    for (int jj = 0; jj < S; ++jj) {
      const int m = jj & (S / 2 - 1);
      const std::uint32_t x0 = C::in_out(jj, 0), x1 = C::in_out(jj, 1);
      const std::int32_t b0 = x0 >= half ? -T[(x0 ^ tmask)] : T[x0];
      const std::int32_t b1 = x1 >= half ? -T[(x1 ^ tmask)] : T[x1];
      const std::int32_t s1 = sig[2 * m] + b0, s2 = sig[2 * m + 1] + b1;
      ns[jj] = s1 > s2 ? s1 : s2;
    }
#pragma unroll
    for (int jj = 0; jj < S; ++jj) sig[jj] = ns[jj];
  };
  // K-1 stages compose the perfect shuffle to the identity, so an unrolled
  // group of K-1 stages needs no register moves
  constexpr int U = C::K - 1;
  std::int64_t t = t0;
  for (; t + U <= t1; t += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) stage(t + u);
  }
  for (; t < t1; ++t) stage(t);
  std::int32_t* dst = p.mat + col * S;  // column j of segment g: rows i contiguous
#pragma unroll
  for (int i = 0; i < S; i += 4) *reinterpret_cast<int4*>(dst + i) = make_int4(sig[i], sig[i + 1], sig[i + 2], sig[i + 3]);
}

// Sequential max-plus chain sigma <- M_k (x) sigma over `count` matrices
// (mats + k * S * S, column-major), writing the metrics BEFORE each step to
// sig_out + k * S. CTA b handles chain b: mats += b * mat_stride, sig_out +=
// b * out_stride, start vector sig_in + b * S (nullptr: zeros, decoder.cpp:109).
// 256 threads: thread (q, i) = (tid >> 6, tid & 63) takes row i over the
// columns j = q, q + 4, ...; the next matrix is prefetched into registers
// while the current one is reduced from shared memory.
struct ChainArgs {
  const std::int32_t* mats;
  std::int64_t mat_stride;  // matrices per chain
  const std::int64_t* sig_in;
  std::int64_t* sig_out;
  std::int64_t out_stride;  // S-vectors per chain
  int total;                // matrices overall (the last chain may be shorter)
  int per_chain;
  int s;
};

__global__ void __launch_bounds__(256) chain_matvec_kernel(const ChainArgs a) {
  __shared__ std::int32_t m_s[2][64 * 64];
  __shared__ std::int64_t sig_s[64];
  __shared__ std::int64_t part[4][64];
  const int tid = threadIdx.x;
  const int i = tid & 63, q = tid >> 6;
  const int S = a.s, SS = S * S;
  const int b = blockIdx.x;
  const int k0 = b * a.per_chain;
  const int count = a.total - k0 < a.per_chain ? a.total - k0 : a.per_chain;
  const std::int32_t* mats = a.mats + static_cast<std::int64_t>(b) * a.mat_stride * SS;
  std::int64_t* out = a.sig_out + static_cast<std::int64_t>(b) * a.out_stride * S;
  constexpr int kPer = 64 * 64 / 256;  // matrix elements each thread moves
  if (tid < 64) sig_s[tid] = (a.sig_in && tid < S) ? a.sig_in[static_cast<std::int64_t>(b) * S + tid] : 0;
  std::int32_t pre[kPer];
  auto load = [&](int k) {
    const std::int32_t* m = mats + static_cast<std::int64_t>(k) * SS;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int x = tid + 256 * e;
      pre[e] = x < SS ? __ldg(m + x) : 0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int e = 0; e < kPer; ++e) m_s[buf][tid + 256 * e] = pre[e];
  };
  if (count <= 0) return;
  load(0);
  stash(0);
  __syncthreads();
  for (int k = 0; k < count; ++k) {
    if (k + 1 < count) load(k + 1);  // in flight during this step's reduction
    if (tid < S) out[static_cast<std::int64_t>(k) * S + tid] = sig_s[tid];
    std::int64_t best = LLONG_MIN;
    if (i < S) {
      const std::int32_t* m = m_s[k & 1];
      for (int j = q; j < S; j += 4) {
        const std::int64_t c = static_cast<std::int64_t>(m[j * S + i]) + sig_s[j];
        best = c > best ? c : best;
      }
    }
    part[q][i] = best;
    __syncthreads();
    if (tid < S) {
      std::int64_t bb = part[0][tid];
#pragma unroll
      for (int e = 1; e < 4; ++e) bb = part[e][tid] > bb ? part[e][tid] : bb;
      sig_s[tid] = bb;
    }
    if (k + 1 < count) stash((k + 1) & 1);
    __syncthreads();
  }
  if (tid < S) out[static_cast<std::int64_t>(count) * S + tid] = sig_s[tid];
}

// Group products P_b = M_{last} (x) ... (x) M_{first} of kGroup consecutive
// segments (one CTA per group): P <- M_k (x) P, 64 x 64 x 64 max-plus per
// step, register-tiled (each thread a 4 x 4 tile of P: per l one 16-byte
// load of M's column and 4 loads of P's row, 16 add/max pairs). Entries stay
// finite after >= K-1 stages; clamped at kNeg anyway. Matrices are padded to
// 64 x 64 (unused rows / columns hold kNeg).
constexpr int kGroup = 16;
__global__ void __launch_bounds__(256) group_product_kernel(const SerialParams p, std::int32_t* prod) {
  __shared__ __align__(16) std::int32_t P_s[64 * 64];
  __shared__ __align__(16) std::int32_t M_s[64 * 64];
  const int tid = threadIdx.x;
  const int S = p.s, SS = S * S;
  const int i0 = (tid & 15) * 4, j0 = (tid >> 4) * 4;  // tile rows i0..i0+3, cols j0..j0+3
  const int g0 = blockIdx.x * kGroup;
  const int count = p.nseg - g0 < kGroup ? p.nseg - g0 : kGroup;
  auto load64 = [&](std::int32_t* dst, const std::int32_t* src) {  // S x S column-major -> 64 x 64
    for (int x = tid; x < 64 * 64; x += 256) {
      const int i = x & 63, j = x >> 6;
      dst[x] = (i < S && j < S) ? __ldg(src + j * S + i) : kNeg;
    }
  };
  load64(P_s, p.mat + static_cast<std::int64_t>(g0) * SS);
  for (int k = 1; k < count; ++k) {
    load64(M_s, p.mat + static_cast<std::int64_t>(g0 + k) * SS);
    __syncthreads();
    std::int32_t acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c] = kNeg;
    }
    for (int l = 0; l < 64; ++l) {
      const int4 mcol = *reinterpret_cast<const int4*>(M_s + l * 64 + i0);  // M[i0..i0+3][l]
      const std::int32_t m[4] = {mcol.x, mcol.y, mcol.z, mcol.w};
      std::int32_t pr[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) pr[c] = P_s[(j0 + c) * 64 + l];  // P[l][j0 + c]
#pragma unroll
      for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const std::int32_t v = m[a] + pr[c];
          acc[a][c] = v > acc[a][c] ? v : acc[a][c];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      *reinterpret_cast<int4*>(P_s + (j0 + c) * 64 + i0) =
          make_int4(acc[0][c] > kNeg ? acc[0][c] : kNeg, acc[1][c] > kNeg ? acc[1][c] : kNeg,
                    acc[2][c] > kNeg ? acc[2][c] : kNeg, acc[3][c] > kNeg ? acc[3][c] : kNeg);
    }
    __syncthreads();
  }
  __syncthreads();
  for (int x = tid; x < SS; x += 256) {
    const int i = x % S, j = x / S;
    prod[static_cast<std::int64_t>(blockIdx.x) * SS + x] = P_s[j * 64 + i];
  }
}

template <int NPL, int BT>
__global__ void __launch_bounds__(128) segment_forward_kernel(const SerialParams p) {
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (g >= p.nseg) return;
  Lane<NPL, BT> ln;
  ln.init(p, lane);
  // exact start metrics minus a common offset (decisions depend on differences only)
  const std::int64_t* s0 = p.sig0 + static_cast<std::int64_t>(g) * p.s;
  const std::int64_t ref = s0[0];
  std::int32_t sig[NPL];
  bool valid[NPL];
#pragma unroll
  for (int r = 0; r < NPL; ++r) {
    const int i = r * 32 + lane;
    valid[r] = i < p.s;
    sig[r] = valid[r] ? static_cast<std::int32_t>(s0[i] - ref) : 0;
  }
  const std::int64_t t0 = static_cast<std::int64_t>(g) * p.seg_len;
  const std::int64_t t1 = t0 + p.seg_len < p.len ? t0 + p.seg_len : p.len;
  bool d[NPL];
  for (std::int64_t t = t0; t < t1; ++t) {
    ln.stage(p.llr + t * BT, sig, d);
#pragma unroll
    for (int r = 0; r < NPL; ++r) {
      const std::uint32_t w = __ballot_sync(kFull, d[r] && valid[r]);
      if (lane == r) p.dec[t * NPL + r] = w;
    }
  }
  if (g == p.nseg - 1) {
    // final argmax, lowest state on ties (decoder.cpp:80-90)
    std::int32_t bv = sig[0];
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
      const std::int32_t ov = __shfl_xor_sync(kFull, bv, o);
      const int oi = __shfl_xor_sync(kFull, bi, o);
      const bool oh = __shfl_xor_sync(kFull, have ? 1 : 0, o) != 0;
      if (oh && (!have || ov > bv || (ov == bv && oi < bi))) {
        bv = ov;
        bi = oi;
        have = true;
      }
    }
    if (lane == 0) p.endst[p.nseg] = bi;
  }
}

template <int NPL>
__global__ void __launch_bounds__(128) segment_map_kernel(const SerialParams p) {
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (g >= p.nseg) return;
  const std::uint32_t lmask = static_cast<std::uint32_t>(p.s / 2 - 1);
  const std::int64_t t0 = static_cast<std::int64_t>(g) * p.seg_len;
  const std::int64_t t1 = t0 + p.seg_len < p.len ? t0 + p.seg_len : p.len;
  std::uint32_t st[NPL];
#pragma unroll
  for (int r = 0; r < NPL; ++r) st[r] = static_cast<std::uint32_t>((r * 32 + lane) % p.s);
  for (std::int64_t t = t1 - 1; t >= t0; --t) {
    std::uint32_t w[NPL];
#pragma unroll
    for (int r = 0; r < NPL; ++r) w[r] = __ldg(p.dec + t * NPL + r);
#pragma unroll
    for (int r = 0; r < NPL; ++r) {
      std::uint32_t word = w[0];
#pragma unroll
      for (int q = 1; q < NPL; ++q) word = (st[r] >> 5) == static_cast<std::uint32_t>(q) ? w[q] : word;
      st[r] = ((st[r] & lmask) << 1) | ((word >> (st[r] & 31)) & 1u);
    }
  }
#pragma unroll
  for (int r = 0; r < NPL; ++r) {
    if (r * 32 + lane < p.s) p.map[static_cast<std::int64_t>(g) * p.s + r * 32 + lane] = static_cast<std::int32_t>(st[r]);
  }
}

// one warp: the segment maps are fetched kDepth segments ahead (independent
// of the chained state) into a register ring; the state hops by shuffles.
__global__ void __launch_bounds__(32) chain_kernel(const SerialParams p) {
  constexpr int kDepth = 8;
  const int lane = threadIdx.x;
  std::int32_t ring[kDepth][2];
  auto fetch = [&](int g, std::int32_t (&m)[2]) {
    if (g < 0) return;
    const std::int32_t* row = p.map + static_cast<std::int64_t>(g) * p.s;
    m[0] = lane < p.s ? __ldg(row + lane) : 0;
    m[1] = lane + 32 < p.s ? __ldg(row + lane + 32) : 0;
  };
  int s = p.endst[p.nseg];
  const int top = p.nseg - 1;
#pragma unroll
  for (int d = 0; d < kDepth; ++d) fetch(top - d, ring[d]);
  for (int g0 = top; g0 >= 0; g0 -= kDepth) {
#pragma unroll
    for (int d = 0; d < kDepth; ++d) {
      const int g = g0 - d;
      if (g >= 0) {
        if (lane == 0) p.endst[g] = s;
        const std::int32_t a = __shfl_sync(kFull, ring[d][0], s & 31), b = __shfl_sync(kFull, ring[d][1], s & 31);
        s = (s >> 5) ? b : a;
        fetch(g - kDepth, ring[d]);  // refill this slot for the next round
      }
    }
  }
}

// one warp per segment: the segment's decision words are staged into shared
// memory in chunks (coalesced), lane 0 walks them with 8 stages of words in
// registers (no load on the state chain) and writes whole output words.
constexpr int kEmitChunk = 1024;
template <int NPL>
__global__ void __launch_bounds__(128) segment_emit_kernel(const SerialParams p) {
  __shared__ std::uint32_t tb_all[4][kEmitChunk * NPL];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = blockIdx.x * 4 + w;
  if (g >= p.nseg) return;
  std::uint32_t* tb = tb_all[w];
  const std::uint32_t lmask = static_cast<std::uint32_t>(p.s / 2 - 1);
  const int ksh = p.k - 2;
  const std::int64_t t0 = static_cast<std::int64_t>(g) * p.seg_len;
  const std::int64_t t1 = t0 + p.seg_len < p.len ? t0 + p.seg_len : p.len;
  std::uint32_t state = static_cast<std::uint32_t>(p.endst[g]);
  std::uint32_t acc = 0;
  std::int64_t cur = -1;
  auto step = [&](std::int64_t t, std::uint32_t word) {
    if (t >= p.emit_lo && t < p.emit_hi) {
      const std::int64_t bit = p.out_bit0 + t;
      const std::int64_t wd = bit >> 5;
      if (wd != cur) {
        if (cur >= 0 && acc) atomicOr(p.out + cur, acc);
        cur = wd;
        acc = 0;
      }
      acc |= (state >> ksh) << (bit & 31);
    }
    state = ((state & lmask) << 1) | ((word >> (state & 31)) & 1u);
  };
  for (std::int64_t chi = t1 - 1; chi >= t0; chi -= kEmitChunk) {
    const std::int64_t clo = chi - kEmitChunk + 1 > t0 ? chi - kEmitChunk + 1 : t0;
    const int cnt = static_cast<int>(chi - clo + 1) * NPL;
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) tb[i] = __ldg(p.dec + clo * NPL + i);
    __syncwarp();
    if (lane == 0) {
      std::int64_t t = chi;
      for (; t - 7 >= clo; t -= 8) {
        std::uint32_t wv[8][NPL];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
          for (int r = 0; r < NPL; ++r) wv[u][r] = tb[(t - u - clo) * NPL + r];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          std::uint32_t word = wv[u][0];
#pragma unroll
          for (int r = 1; r < NPL; ++r) word = (state >> 5) == static_cast<std::uint32_t>(r) ? wv[u][r] : word;
          step(t - u, word);
        }
      }
      for (; t >= clo; --t) step(t, tb[(t - clo) * NPL + (NPL > 1 ? (state >> 5) : 0)]);
    }
  }
  if (lane == 0 && cur >= 0 && acc) atomicOr(p.out + cur, acc);
}

using SK7a = SCode<7, 2, 0171, 0133>;
using SK7b = SCode<7, 2, 0133, 0171>;
using SK7c = SCode<7, 3, 0133, 0171, 0165>;
using SK5a = SCode<5, 2, 023, 035>;
using SK6a = SCode<6, 2, 053, 075>;
using SK3a = SCode<3, 2, 07, 05>;

// register-column kernel A for the compile-time codes; false -> caller uses the generic one
bool launch_cols(const SerialParams& p, cudaStream_t s) {
  if (!VD_SERIAL_COLS) return false;
  const std::int64_t cols = static_cast<std::int64_t>(p.nseg) * p.s;
  const unsigned grid = static_cast<unsigned>((cols + 63) / 64);
#define VD_TRY_COLS(C)                                                   \
  if (C::matches(p.k, p.b, p.polys)) {                                   \
    segment_matrix_cols_kernel<C><<<grid, 64, 0, s>>>(p);                \
    return true;                                                         \
  }
  VD_TRY_COLS(SK7a)
  VD_TRY_COLS(SK7b)
  VD_TRY_COLS(SK7c)
  VD_TRY_COLS(SK5a)
  VD_TRY_COLS(SK6a)
  VD_TRY_COLS(SK3a)
#undef VD_TRY_COLS
  return false;
}

template <int NPL, int BT>
cudaError_t run(SerialParams p, cudaStream_t s) {
  const std::size_t S = static_cast<std::size_t>(p.s);
  const std::size_t bytes = sizeof(std::int32_t) * p.nseg * S * S + sizeof(std::int64_t) * (p.nseg + 1) * S +
                            sizeof(std::uint32_t) * p.len * NPL + sizeof(std::int32_t) * (p.nseg * S + p.nseg + 1) + 64;
  unsigned char* buf = nullptr;
  if (cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, s); e != cudaSuccess) return e;
  unsigned char* q = buf;
  p.mat = reinterpret_cast<std::int32_t*>(q);
  q += sizeof(std::int32_t) * p.nseg * S * S;
  p.sig0 = reinterpret_cast<std::int64_t*>(q);
  q += sizeof(std::int64_t) * (p.nseg + 1) * S;
  p.dec = reinterpret_cast<std::uint32_t*>(q);
  q += sizeof(std::uint32_t) * p.len * NPL;
  p.map = reinterpret_cast<std::int32_t*>(q);
  q += sizeof(std::int32_t) * p.nseg * S;
  p.endst = reinterpret_cast<std::int32_t*>(q);
  const std::int64_t warpsA = static_cast<std::int64_t>(p.nseg) * p.s;
  if (!launch_cols(p, s)) segment_matrix_kernel<NPL, BT><<<static_cast<unsigned>((warpsA + 3) / 4), 128, 0, s>>>(p);
  note_launch();
  // B: two-level max-plus scan of the segment matrices. Group products (in
  // parallel), a sequential chain over the groups, then every group's own
  // chain from its start metrics (in parallel).
  const int ngroups = (p.nseg + kGroup - 1) / kGroup;
  std::int32_t* prod = nullptr;
  std::int64_t* gsig = nullptr;
  if (cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&prod),
                                      sizeof(std::int32_t) * S * S * ngroups + sizeof(std::int64_t) * S * (ngroups + 1), s);
      e != cudaSuccess) {
    cudaFreeAsync(buf, s);
    return e;
  }
  gsig = reinterpret_cast<std::int64_t*>(prod + S * S * ngroups);
  group_product_kernel<<<ngroups, 256, 0, s>>>(p, prod);
  ChainArgs top{prod, 0, nullptr, gsig, 0, ngroups, ngroups, p.s};
  chain_matvec_kernel<<<1, 256, 0, s>>>(top);
  ChainArgs per{p.mat, kGroup, gsig, p.sig0, kGroup, p.nseg, kGroup, p.s};
  chain_matvec_kernel<<<ngroups, 256, 0, s>>>(per);
  segment_forward_kernel<NPL, BT><<<static_cast<unsigned>((p.nseg + 3) / 4), 128, 0, s>>>(p);
  segment_map_kernel<NPL><<<static_cast<unsigned>((p.nseg + 3) / 4), 128, 0, s>>>(p);
  chain_kernel<<<1, 32, 0, s>>>(p);
  segment_emit_kernel<NPL><<<static_cast<unsigned>((p.nseg + 3) / 4), 128, 0, s>>>(p);
  note_launch(7);  // group products, 2 chains, forward, map, chain, emit
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(prod, s);
  const cudaError_t ef = cudaFreeAsync(buf, s);
  return e != cudaSuccess ? e : ef;
}

}  // namespace

bool serial_parallel_supported(const DecodeLaunch& p) {
  if (p.s < 4 || p.s > 64 || (p.b != 2 && p.b != 3)) return false;
  if (p.frame_end - p.frame_begin != 1 || p.nblocks > 0 || p.frame_list || p.sigma) return false;
  if (p.f0 > 0 && p.f0 < p.f) return false;  // one traceback per frame
  const FrameGeom g(p.frame_begin, p.n, p.f, p.v1, p.v2, p.f0);
  return g.len() >= 8192;
}

cudaError_t launch_serial_parallel_i8(const DecodeLaunch& p, cudaStream_t stream) {
  const FrameGeom g(p.frame_begin, p.n, p.f, p.v1, p.v2, p.f0);
  SerialParams sp{};
  sp.llr = static_cast<const std::int8_t*>(p.llr) + (g.beg - p.llr_stage0) * p.b;
  sp.k = p.k;
  sp.b = p.b;
  sp.s = p.s;
  sp.len = g.len();
  // segments: enough of them to fill the GPU in kernel A, short enough for
  // the sequential kernels B and D2
  std::int64_t seg = 512;
  while (seg < 16384 && (sp.len + seg - 1) / seg > 1024) seg *= 2;
  sp.seg_len = static_cast<int>(seg);
  sp.nseg = static_cast<int>((sp.len + seg - 1) / seg);
  sp.in_out = p.in_out;
  for (int i = 0; i < 4 && i < p.b; ++i) sp.polys[i] = p.polys[i];
  sp.out = p.out;
  sp.out_bit0 = g.beg - p.out_stage0;
  sp.emit_lo = g.out_lo - g.beg;
  sp.emit_hi = g.out_hi - g.beg;
  const int npl = p.s > 32 ? 2 : 1;
  if (npl == 2) return p.b == 2 ? run<2, 2>(sp, stream) : run<2, 3>(sp, stream);
  return p.b == 2 ? run<1, 2>(sp, stream) : run<1, 3>(sp, stream);
}

}  // namespace vd
