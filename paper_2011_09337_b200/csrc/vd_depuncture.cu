// Device depuncture: punctured int8 stream -> stage-major int8 LLR block with
// 0 at the punctured positions (reference decoder.cpp:131-163, `depuncture`,
// which the BER harness and CLI call right before framed_decode:
// berlab.cpp:79-80, vitdec_cli.cpp:172-173).
//
// HBM-bound byte work (read kept/period bytes, write B bytes per stage), run
// as its own streaming pass on the decode stream right before the decode
// kernels (DESIGN.md §3.4 gives the measured cost and why it is not folded
// into the ALU-bound decoder's LLR staging).
//
// Units are U whole puncture periods aligned to global period boundaries,
// with U * period * B and U * kept multiples of 16 / 4 bytes, so every unit
// has the same input and output byte alignment. That makes the byte mapping
// unit-invariant: a per-CTA table gives, for each aligned 32-bit output word
// slot of a unit, the shared-memory input word it starts in, a PRMT selector
// over that word and the next, and a zero mask for punctured bytes. A tile
// (~32 KiB of output, TU units) is staged per iteration: coalesced 32-bit
// loads of its punctured bytes into shared memory, then one LDS.64 (table) +
// 2 LDS + PRMT + LOP + coalesced STG.32 per output word. CTAs are persistent
// (grid-stride over tiles).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>

#include "vd_internal.h"

namespace vd {
namespace {

__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t s) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}

// kept index, relative to the input of the unit holding unit-relative output
// byte j (j may be negative: the tail of the previous unit), or INT_MIN if
// the byte is punctured.
__device__ __forceinline__ int src_of(const DepunctureLaunch& p, int j) {
  const int pb = p.period * p.b;
  int shift = 0;
  if (j < 0) {
    j += p.unit_bytes;
    shift = p.unit_in;
  }
  const int q = j % pb;
  return p.rank[q] < 0 ? INT_MIN : (j / pb) * p.kept + p.rank[q] - shift;
}

__global__ void __launch_bounds__(256) depuncture_kernel(DepunctureLaunch p) {
  extern __shared__ __align__(16) std::uint32_t smem[];
  const int uw = p.unit_bytes / 4;   // output word slots per unit
  const int uin = p.unit_in / 4;     // input words per unit
  const int tile_bytes = p.tu * p.unit_bytes;
  const int in_words = p.tu * uin + 4;  // + front pad word + alignment / PRMT spill
  uint2* lut = reinterpret_cast<uint2*>(smem);
  std::uint32_t* s_in = smem + 2 * uw;

  const std::int64_t out_bytes = p.n * p.b;
  // byte alignment of unit starts (identical for all units of the launch)
  const int a_out = static_cast<int>(static_cast<std::uint64_t>(-(p.t0 * p.b)) & 3u);
  const int a_in = static_cast<int>((reinterpret_cast<std::uintptr_t>(p.in) - static_cast<std::uint64_t>(p.in0)) & 3u);
  // Slot s of a unit covers unit-relative output bytes [4s - a_out, 4s - a_out + 4);
  // s_in word 1 + x holds the unit's input bytes 4x - a_in .. (word 0 = front pad).
  for (int s = threadIdx.x; s < uw; s += blockDim.x) {
    int r[4];
    int first = INT_MIN;
    for (int i = 0; i < 4; ++i) {
      r[i] = src_of(p, 4 * s - a_out + i);
      if (r[i] != INT_MIN && first == INT_MIN) first = r[i];
    }
    const int base = first == INT_MIN ? 0 : ((first + a_in + 4) >> 2);  // s_in word (front pad folded in)
    std::uint32_t sel = 0, mask = 0;
    for (int i = 0; i < 4; ++i) {
      if (r[i] != INT_MIN) {
        sel |= static_cast<std::uint32_t>(r[i] + a_in + 4 - 4 * base) << (4 * i);
        mask |= 0xffu << (8 * i);
      }
    }
    lut[s] = make_uint2(static_cast<std::uint32_t>(base) | (sel << 16), mask);
  }

  const std::int64_t unit_stages = static_cast<std::int64_t>(p.unit_periods) * p.period;
  const std::int64_t tile_stages = unit_stages * p.tu;
  const std::int64_t g_first = p.t0 / tile_stages;
  const std::int64_t g_last = (p.t0 + p.n - 1) / tile_stages;
  const std::int64_t in_len = p.in_len;
  for (std::int64_t g = g_first + blockIdx.x; g <= g_last; g += gridDim.x) {
    const std::int64_t tile_o = (g * tile_stages - p.t0) * p.b;                          // out index of byte 0
    const std::int64_t in_rel = g * p.tu * static_cast<std::int64_t>(p.unit_in) - p.in0;  // in index of byte 0
    __syncthreads();  // previous tile's readers are done with s_in (first pass: table built)
    // ---- stage the tile's punctured bytes: s_in word w = input bytes in_rel - a_in + 4 (w - 1) ...
    const std::int64_t b00 = in_rel - a_in - 4;  // input index of s_in word 0 (4-byte aligned address)
    const std::uint32_t* wbase = reinterpret_cast<const std::uint32_t*>(p.in + b00);
    if (b00 >= 0 && b00 + 4 * in_words <= in_len) {
      // interior: batches of 8 independent loads per thread, then the stores
      constexpr int kBatch = 8;
      for (int w0 = 0; w0 < in_words; w0 += kBatch * 256) {
        std::uint32_t v[kBatch];
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
          const int w = w0 + i * 256 + static_cast<int>(threadIdx.x);
          v[i] = w < in_words ? __ldg(wbase + w) : 0u;
        }
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
          const int w = w0 + i * 256 + static_cast<int>(threadIdx.x);
          if (w < in_words) s_in[w] = v[i];
        }
      }
    } else {
      for (int w = threadIdx.x; w < in_words; w += blockDim.x) {
        const std::int64_t b0 = b00 + 4 * w;
        std::uint32_t v = 0;
        for (int i = 0; i < 4; ++i) {
          const std::int64_t bi = b0 + i;
          if (bi >= 0 && bi < in_len) v |= static_cast<std::uint32_t>(static_cast<std::uint8_t>(p.in[bi])) << (8 * i);
        }
        s_in[w] = v;
      }
    }
    __syncthreads();
    // ---- output: tile slot k = u * uw + s covers global word slot0 + k
    const std::int64_t slot0 = (tile_o - a_out) >> 2;  // 4-aligned by construction
    std::uint32_t* out32 = reinterpret_cast<std::uint32_t*>(p.out) + slot0;
    const std::int64_t lo = tile_o > 0 ? tile_o : 0;
    const std::int64_t hi = (tile_o + tile_bytes < out_bytes) ? tile_o + tile_bytes : out_bytes;
    auto word_at = [&](int k) {
      const int u = k / uw;
      const uint2 e = lut[k - u * uw];
      const std::uint32_t base = (e.x & 0xffffu) + static_cast<std::uint32_t>(u * uin);
      return prmt(s_in[base], s_in[base + 1], e.x >> 16) & e.y;
    };
    auto store_bytes = [&](int k, std::uint32_t v) {  // own bytes of a word shared with a neighbour / range end
      const std::int64_t o0 = (slot0 + k) << 2;
      for (int i = 0; i < 4; ++i) {
        const std::int64_t o = o0 + i;
        if (o >= lo && o < hi) p.out[o] = static_cast<std::int8_t>((v >> (8 * i)) & 0xffu);
      }
    };
    if (tile_o >= 0 && tile_o + tile_bytes <= out_bytes) {
      // interior tile: every slot but k = 0 (when a_out != 0) is a whole word of this tile
      for (int s = threadIdx.x; s < uw; s += blockDim.x) {
        const uint2 e = lut[s];
        const std::uint32_t b0 = e.x & 0xffffu, sel = e.x >> 16;
#pragma unroll 4
        for (int u = 0; u < p.tu; ++u) {
          const int k = u * uw + s;
          const std::uint32_t base = b0 + static_cast<std::uint32_t>(u * uin);
          const std::uint32_t v = prmt(s_in[base], s_in[base + 1], sel) & e.y;
          if (k != 0 || a_out == 0) out32[k] = v;
        }
      }
      if (a_out != 0 && threadIdx.x < 2) {
        const int k = threadIdx.x == 0 ? 0 : p.tu * uw;
        store_bytes(k, word_at(k));
      }
    } else {
      // first / last tile of the launch: guarded per word
      const std::int64_t w_lo = (lo >> 2) - slot0, w_hi = ((hi + 3) >> 2) - slot0;
      for (std::int64_t k = w_lo + threadIdx.x; k < w_hi; k += blockDim.x) {
        const std::uint32_t v = word_at(static_cast<int>(k));
        const std::int64_t o0 = (slot0 + k) << 2;
        if (o0 >= lo && o0 + 4 <= hi) {
          out32[k] = v;
        } else {
          store_bytes(static_cast<int>(k), v);
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_depuncture_i8(const DepunctureLaunch& p, cudaStream_t stream) {
  if (p.n <= 0) return cudaSuccess;
  if ((reinterpret_cast<std::uintptr_t>(p.out) & 3u) != 0) return cudaErrorMisalignedAddress;
  const std::size_t smem = sizeof(uint2) * (p.unit_bytes / 4) + sizeof(std::uint32_t) * (p.tu * p.unit_in / 4 + 4);
  cudaError_t e =
      allow_max_smem(reinterpret_cast<const void*>(depuncture_kernel));
  if (e != cudaSuccess) return e;
  const std::int64_t tile_stages = static_cast<std::int64_t>(p.unit_periods) * p.period * p.tu;
  const std::int64_t tiles = (p.t0 + p.n - 1) / tile_stages - p.t0 / tile_stages + 1;
  const std::int64_t cap = static_cast<std::int64_t>(sm_count()) * 4;
  const unsigned grid = static_cast<unsigned>(tiles < cap ? tiles : cap);
  depuncture_kernel<<<grid, 256, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

namespace {
struct RankTable {
  std::int16_t r[kMaxPunctureCells];
};

__global__ void depuncture_f64_kernel(const double* __restrict__ in, std::int64_t count, int b, int period, int kept,
                                      RankTable rt, double* __restrict__ out) {
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t t = e / b;
    const int row = static_cast<int>(e - t * b);
    const int cell = static_cast<int>(t % period) * b + row;
    const int r = rt.r[cell];
    out[e] = r < 0 ? 0.0 : in[(t / period) * kept + r];
  }
}
}  // namespace

cudaError_t launch_depuncture_f64(const double* in, std::int64_t n_stages, int b, int period, int kept,
                                  const std::int16_t* rank, double* out, cudaStream_t stream) {
  RankTable rt{};
  for (int i = 0; i < period * b && i < kMaxPunctureCells; ++i) rt.r[i] = rank[i];
  const std::int64_t count = n_stages * b;
  const std::int64_t blocks = std::min<std::int64_t>((count + 255) / 256, static_cast<std::int64_t>(sm_count()) * 8);
  depuncture_f64_kernel<<<static_cast<unsigned>(blocks > 0 ? blocks : 1), 256, 0, stream>>>(in, count, b, period, kept,
                                                                                         rt, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace vd
