// Large-constraint-length path (K = 13 .. 16, 4096 .. 32768 states): one CTA
// (1024 threads) per frame. The reference accepts K <= 16 (trellis.cpp:44);
// the register / warp-per-frame kernels stop at K = 12 (their per-warp state
// vectors no longer fit on chip), so these codes are decoded here.
//
// Per frame (reference decode_frame, decoder.cpp:170-237):
//   forward pass over the clipped window: per stage the 2^B branch metrics
//   (decoder.cpp:22-51, the reference's add order, complement half by exact
//   negation) go to shared memory; thread j then owns states j, j + 1024, ...
//   and does the reference ACS (decoder.cpp:53-76: strict '>', ties -> the
//   second predecessor) on path metrics double-buffered in a per-CTA global
//   scratch (2 x S metrics, <= 512 KiB, L2-resident for a full grid); the
//   decisions are warp ballots (32 states per word) into a per-CTA global
//   decision array; a CTA barrier separates stages;
//   stored-max argmax at every subframe start stage (decoder.cpp:80-90,
//   205-211: lowest index on ties) as a block reduction;
//   traceback: subframe s walked by thread s (decoder.cpp:214-236), output
//   bits OR-ed into the packed words.
// int8 LLRs use int32 metrics (renormalised every 4096 stages, differences
// exact); double LLRs use double metrics in the reference's operation order.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "vd_common.cuh"
#include "vd_internal.h"

namespace vd {
namespace {

constexpr int kThreads = 1024;
constexpr int kStageBuf = 256;  // LLR staging depth (stages)
constexpr unsigned kFull = 0xffffffffu;

struct BigKParams {
  DecodeLaunch p;
  int words;          // decision words per stage = S / 32
  int len_max;        // max processed stages of a launched frame
  int nsub_max;
  void* metrics;      // [grid][2][S] of M
  std::uint32_t* dec; // [grid][len_max][words]
};

template <typename M>
__device__ __forceinline__ bool better(M v, int i, M bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

template <typename In, typename M>
__global__ void __launch_bounds__(kThreads, 1) bigk_kernel(const BigKParams bp) {
  const DecodeLaunch& p = bp.p;
  __shared__ M table[256];
  __shared__ In stage_buf[kStageBuf * 8];
  __shared__ M red_v[kThreads / 32];
  __shared__ int red_i[kThreads / 32];
  __shared__ int start_state_s[64];
  __shared__ M ref_s;
  extern __shared__ int start_state_dyn[];
  int* start_state = bp.nsub_max <= 64 ? start_state_s : start_state_dyn;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int S = p.s;
  const int words = bp.words;
  const std::uint32_t low_mask = static_cast<std::uint32_t>(S / 2 - 1);
  const int b = p.b;
  const std::uint32_t half = 1u << (b - 1), tmask = (1u << b) - 1u;
  M* const mbase = static_cast<M*>(bp.metrics) + static_cast<std::size_t>(blockIdx.x) * 2 * S;
  std::uint32_t* const dec = bp.dec + static_cast<std::size_t>(blockIdx.x) * bp.len_max * words;
  const In* llr = static_cast<const In*>(p.llr);

  for (std::int64_t mi = p.frame_begin + blockIdx.x; mi < p.frame_end; mi += gridDim.x) {
    const FrameRef fr = resolve_frame(p, mi);
    const std::int64_t m = fr.m;
    const FrameGeom g(m, fr.n, p.f, p.v1, p.v2, p.f0);
    const int len = static_cast<int>(g.len());
    M* sp = mbase;
    M* sc = mbase + S;
    for (int j = tid; j < S; j += kThreads) sp[j] = M(0);  // sigma_0 = 0 (decoder.cpp:195)
    std::int64_t offset = 0;
    int next_record = 0;
    int next_start = static_cast<int>(g.start_stage(0, p.v2));
    const In* src = llr + (fr.base + g.beg - p.llr_stage0) * b;
    __syncthreads();

    for (int t = 0; t < len; ++t) {
      if ((t & (kStageBuf - 1)) == 0) {
        const int cnt = (kStageBuf < len - t ? kStageBuf : len - t) * b;
        for (int i = tid; i < cnt; i += kThreads) stage_buf[i] = src[static_cast<std::int64_t>(t) * b + i];
        __syncthreads();
      }
      if (tid <= static_cast<int>(tmask)) {
        // stage table (decoder.cpp:41-51): direct entries in the reference's
        // add order (0 + (+/-l0) + (+/-l1) ...), the complements by negation
        const In* lt = stage_buf + (t & (kStageBuf - 1)) * b;
        const std::uint32_t bo = static_cast<std::uint32_t>(tid);
        const std::uint32_t x = bo < half ? bo : (bo ^ tmask);
        M acc = M(0);
        for (int i = 0; i < b; ++i) {
          const M v = static_cast<M>(lt[i]);
          acc += ((x >> (b - 1 - i)) & 1u) ? -v : v;
        }
        table[bo] = bo < half ? acc : -acc;
      }
      __syncthreads();
      // ACS (decoder.cpp:53-76); S is a multiple of 32, every warp owns whole words
      for (int j = tid; j < S; j += kThreads) {
        const std::uint32_t i1 = (static_cast<std::uint32_t>(j) & low_mask) << 1;
        const M s1 = sp[i1] + table[__ldg(p.in_out + 2 * j)];
        const M s2 = sp[i1 | 1] + table[__ldg(p.in_out + 2 * j + 1)];
        const bool d = !(s1 > s2);
        sc[j] = d ? s2 : s1;
        const std::uint32_t w = __ballot_sync(kFull, d);
        if (lane == 0) dec[static_cast<std::size_t>(t) * words + (j >> 5)] = w;
      }
      __syncthreads();
      M* tmp = sp;
      sp = sc;
      sc = tmp;
      if constexpr (std::is_integral<M>::value) {
        if ((t & 4095) == 4095) {  // keep int32 metrics bounded (differences exact)
          if (tid == 0) ref_s = sp[0];
          __syncthreads();
          const M ref = ref_s;
          for (int j = tid; j < S; j += kThreads) sp[j] -= ref;
          offset += ref;
          __syncthreads();
        }
      }
      // stored-max start states (decoder.cpp:205-211), lowest index on ties
      while (next_record < g.num_sub && next_start == t) {
        M bv = sp[tid];
        int bi = tid;
        for (int j = tid + kThreads; j < S; j += kThreads) {
          if (sp[j] > bv) {
            bv = sp[j];
            bi = j;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const M ov = __shfl_xor_sync(kFull, bv, o);
          const int oi = __shfl_xor_sync(kFull, bi, o);
          if (better(ov, oi, bv, bi)) {
            bv = ov;
            bi = oi;
          }
        }
        if (lane == 0) {
          red_v[warp] = bv;
          red_i[warp] = bi;
        }
        __syncthreads();
        if (warp == 0) {
          bv = red_v[lane];
          bi = red_i[lane];
          for (int o = 16; o > 0; o >>= 1) {
            const M ov = __shfl_xor_sync(kFull, bv, o);
            const int oi = __shfl_xor_sync(kFull, bi, o);
            if (better(ov, oi, bv, bi)) {
              bv = ov;
              bi = oi;
            }
          }
          if (lane == 0) start_state[next_record] = bi;
        }
        __syncthreads();
        ++next_record;
        if (next_record < g.num_sub) next_start = static_cast<int>(g.start_stage(next_record, p.v2));
      }
    }

    if (p.sigma) {
      for (int j = tid; j < S; j += kThreads) {
        if constexpr (std::is_integral<M>::value) {
          static_cast<std::int64_t*>(p.sigma)[(mi - p.frame_begin) * S + j] = static_cast<std::int64_t>(sp[j]) + offset;
        } else {
          static_cast<double*>(p.sigma)[(mi - p.frame_begin) * S + j] = sp[j];
        }
      }
    }
    __syncthreads();

    // parallel traceback (decoder.cpp:214-236): thread s walks subframe s
    for (std::int64_t s = tid; s < g.num_sub; s += kThreads) {
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
        const std::uint32_t d = (dec[static_cast<std::size_t>(t) * words + (state >> 5)] >> (state & 31)) & 1u;
        state = ((state & low_mask) << 1) | d;
      }
      if (cur >= 0 && acc) atomicOr(p.out + cur, acc);
    }
    __syncthreads();
  }
}

template <typename In, typename M>
cudaError_t launch_bigk(const DecodeLaunch& p, cudaStream_t stream) {
  const std::int64_t frames = p.frame_end - p.frame_begin;
  if (frames <= 0) return cudaSuccess;
  if (p.s < 64 || p.b > 8) return cudaErrorInvalidValue;
  BigKParams bp;
  bp.p = p;
  bp.words = p.s / 32;
  const std::int64_t len_max = imin(static_cast<std::int64_t>(p.f) + p.v1 + p.v2, p.n);
  const std::int64_t nsub_max = p.f0 > 0 ? (static_cast<std::int64_t>(p.f) + p.f0 - 1) / p.f0 : 1;
  if (len_max > 0x7fffffffLL) return cudaErrorInvalidValue;
  bp.len_max = static_cast<int>(len_max);
  bp.nsub_max = static_cast<int>(nsub_max);
  const std::size_t dyn = nsub_max > 64 ? sizeof(int) * static_cast<std::size_t>(nsub_max) : 0;
  if (dyn > 96 * 1024) return cudaErrorInvalidValue;
  // grid: one CTA per frame, at most one per SM, and at most what the
  // per-CTA decision arrays allow in 16 GiB of scratch
  const std::size_t dec_bytes = sizeof(std::uint32_t) * static_cast<std::size_t>(len_max) * bp.words;
  const std::size_t met_bytes = sizeof(M) * 2 * static_cast<std::size_t>(p.s);
  std::int64_t grid = frames < sm_count() ? frames : sm_count();
  const std::int64_t cap = static_cast<std::int64_t>((std::size_t{16} << 30) / (dec_bytes + met_bytes));
  if (cap < 1) return cudaErrorInvalidValue;
  if (grid > cap) grid = cap;
  if (cudaError_t e = retain_async_pool(); e != cudaSuccess) return e;
  unsigned char* scratch = nullptr;
  if (cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), (dec_bytes + met_bytes) * grid, stream);
      e != cudaSuccess)
    return e;
  bp.metrics = scratch;
  bp.dec = reinterpret_cast<std::uint32_t*>(scratch + met_bytes * grid);
  auto kern = bigk_kernel<In, M>;
  cudaError_t e = cudaSuccess;
  if (dyn > 0) e = allow_max_smem(reinterpret_cast<const void*>(kern));
  if (e == cudaSuccess) {
    kern<<<static_cast<unsigned>(grid), kThreads, dyn, stream>>>(bp);
    note_launch();
    e = cudaGetLastError();
  }
  const cudaError_t ef = cudaFreeAsync(scratch, stream);
  return e != cudaSuccess ? e : ef;
}

}  // namespace

cudaError_t launch_bigk_i8(const DecodeLaunch& p, cudaStream_t stream) {
  return launch_bigk<std::int8_t, std::int32_t>(p, stream);
}

cudaError_t launch_bigk_f64(const DecodeLaunch& p, cudaStream_t stream) {
  return launch_bigk<double, double>(p, stream);
}

}  // namespace vd
