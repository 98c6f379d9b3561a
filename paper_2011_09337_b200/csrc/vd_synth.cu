// Device-side synthetic input for benchmarks and large-N streaming tests:
// random message -> convolutional encoder -> BPSK -> AWGN -> int8 quantiser.
//
// This is NOT the reference's data chain (mt19937_64 + Marsaglia polar,
// reference channel.cpp:22-83, which is inherently sequential); parity
// tests use the host oracle's restatement of that chain instead. Here every
// value is a pure function of (seed, index) via the splitmix64 finaliser, so
// gigabit-scale inputs are generated in HBM in milliseconds and are
// reproducible for any sharding.
#include <cuda_runtime.h>

#include <cstdint>

#include "vd_common.cuh"
#include "vd_internal.h"

namespace vd {
namespace {

__device__ __forceinline__ std::uint32_t msg_word(std::uint64_t seed, std::int64_t w) {
  return static_cast<std::uint32_t>(mix_seed(seed, static_cast<std::uint64_t>(w)));
}

__device__ __forceinline__ std::uint32_t msg_bit(std::uint64_t seed, std::int64_t t) {
  return t < 0 ? 0u : (msg_word(seed, t >> 5) >> (t & 31)) & 1u;
}

constexpr int kStagesPerThread = 8;

__global__ void synth_kernel(int k, int b, std::uint32_t p0, std::uint32_t p1, std::uint32_t p2, std::uint32_t p3,
                             std::int64_t tb, std::int64_t n, float sigma, float scale, std::uint64_t seed,
                             std::int8_t* __restrict__ llr, std::uint32_t* __restrict__ bits) {
  const std::uint32_t polys[4] = {p0, p1, p2, p3};
  const std::uint64_t noise_seed = mix_seed(seed, 0xA5A5A5A5ull);
  // stream stages [tb, tb + n); local index = t - tb
  const std::int64_t l0 = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kStagesPerThread;
  if (l0 >= n) return;
  const std::int64_t t0 = tb + l0;
  // Encoder register before stage t0: bits t0-1 ... t0-K+1 (newest at the MSB).
  std::uint32_t state = 0;
  for (int i = k - 1; i >= 1; --i) state = (state >> 1) | (msg_bit(seed, t0 - i) << (k - 2));
  for (int j = 0; j < kStagesPerThread; ++j) {
    const std::int64_t t = t0 + j;
    if (t - tb >= n) break;
    const std::uint32_t u = msg_bit(seed, t);
    const std::uint32_t reg = (u << (k - 1)) | state;
    for (int i = 0; i < b; ++i) {
      const std::uint32_t c = __popc(polys[i] & reg) & 1u;
      const std::uint64_t h = mix_seed(noise_seed, static_cast<std::uint64_t>(t * b + i));
      // Box-Muller on two 24-bit uniforms (u1 in (0, 1]).
      const float u1 = (static_cast<float>(h >> 40) + 1.0f) * (1.0f / 16777216.0f);
      const float u2 = static_cast<float>((h >> 16) & 0xffffffu) * (1.0f / 16777216.0f);
      const float z = sqrtf(-2.0f * __logf(u1)) * __cosf(6.2831853f * u2);
      const float y = (c ? -1.0f : 1.0f) + sigma * z;
      float q = rintf(scale * y);
      q = fminf(fmaxf(q, -127.0f), 127.0f);
      if (llr) llr[(t - tb) * b + i] = static_cast<std::int8_t>(q);
    }
    state = (u << (k - 2)) | (state >> 1);
  }
  if (bits && (l0 & 31) == 0) {
    // the thread whose first stage starts a 32-stage word writes that word
    // (tb % 32 == 0: local and stream words coincide up to the offset)
    std::uint32_t v = msg_word(seed, t0 >> 5);
    const std::int64_t rem = n - l0;
    if (rem < 32) v &= (1u << rem) - 1u;
    bits[l0 >> 5] = v;
  }
}

__global__ void count_errors_kernel(const std::uint32_t* __restrict__ a, const std::uint32_t* __restrict__ b,
                                    std::int64_t n_bits, unsigned long long* count) {
  const std::int64_t words = (n_bits + 31) / 32;
  unsigned long long local = 0;
  for (std::int64_t w = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < words;
       w += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    std::uint32_t x = a[w] ^ b[w];
    const std::int64_t rem = n_bits - w * 32;
    if (rem < 32) x &= (1u << rem) - 1u;
    local += __popc(x);
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

}  // namespace

cudaError_t launch_synth_i8(int k, int b, const std::uint32_t* polys, std::int64_t t_begin, std::int64_t n,
                            double sigma, double scale, std::uint64_t seed, std::int8_t* llr, std::uint32_t* bits,
                            cudaStream_t stream) {
  if (b > 4) return cudaErrorNotSupported;
  std::uint32_t p[4] = {0, 0, 0, 0};
  for (int i = 0; i < b; ++i) p[i] = polys[i];
  const std::int64_t threads = (n + kStagesPerThread - 1) / kStagesPerThread;
  const std::int64_t blocks = (threads + 255) / 256;
  synth_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(k, b, p[0], p[1], p[2], p[3], t_begin, n,
                                                                  static_cast<float>(sigma), static_cast<float>(scale),
                                                                  seed, llr, bits);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_count_bit_errors(const std::uint32_t* a, const std::uint32_t* b, std::int64_t n_bits,
                                    unsigned long long* count, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  count_errors_kernel<<<sm_count() * 4, 256, 0, stream>>>(a, b, n_bits, count);
  note_launch();
  return cudaGetLastError();
}

}  // namespace vd
