// 4-bit LLR wire format: two signed 4-bit LLRs per byte,
// element i of the stage-major stream in nibble i (low nibble first), values
// in [-8, 7]. Streaming decodes over PCIe move 1 B per r1/2 stage instead of
// 2 B; each chunk is widened to int8 on the device right before its decode
// (the decode kernels then run unchanged and are exact for those integers).
//
// unpack_i4_kernel: HBM-bound, 8 LLRs per thread — one aligned 32-bit load
// (+ one more when the chunk starts on an odd nibble), two PRMTs to
// interleave the nibbles into bytes, sign extension as
// ((x ^ 8) + 0x78) ^ 0x80 per byte (no inter-byte carries), two 32-bit stores.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "vd_internal.h"

namespace vd {
namespace {

__device__ __forceinline__ std::uint32_t prmt(std::uint32_t a, std::uint32_t b, std::uint32_t s) {
  std::uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}

__device__ __forceinline__ std::uint32_t sext4x4(std::uint32_t x) {  // 4 nibble values (one per byte) -> int8
  return ((x ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
}

__global__ void unpack_i4_kernel(const std::uint32_t* __restrict__ in, std::int64_t nbytes, int nib_off,
                                 std::int64_t count, std::int8_t* __restrict__ out) {
  const std::int64_t groups = (count + 7) / 8;
  for (std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < groups;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t b0 = 4 * t;  // first byte of this group's 8 nibbles (+ 1 nibble when nib_off)
    std::uint32_t w0, w1 = 0;
    if (b0 + 4 <= nbytes) {
      w0 = __ldg(in + t);
    } else {
      const std::uint8_t* p = reinterpret_cast<const std::uint8_t*>(in);
      w0 = 0;
      for (int i = 0; i < 4 && b0 + i < nbytes; ++i) w0 |= static_cast<std::uint32_t>(p[b0 + i]) << (8 * i);
    }
    if (nib_off) {
      if (b0 + 8 <= nbytes) {
        w1 = __ldg(in + t + 1);
      } else if (b0 + 4 < nbytes) {
        w1 = reinterpret_cast<const std::uint8_t*>(in)[b0 + 4];
      }
      w0 = static_cast<std::uint32_t>(((static_cast<std::uint64_t>(w1) << 32) | w0) >> 4);
    }
    const std::uint32_t lo = w0 & 0x0F0F0F0Fu, hi = (w0 >> 4) & 0x0F0F0F0Fu;
    const std::uint32_t o0 = sext4x4(prmt(lo, hi, 0x5140u)), o1 = sext4x4(prmt(lo, hi, 0x7362u));
    const std::int64_t e0 = 8 * t;
    if (e0 + 8 <= count) {
      reinterpret_cast<uint2*>(out)[t] = make_uint2(o0, o1);
    } else {
      for (int i = 0; i < 8 && e0 + i < count; ++i) {
        out[e0 + i] = static_cast<std::int8_t>(((i < 4 ? o0 : o1) >> (8 * (i & 3))) & 0xffu);
      }
    }
  }
}

}  // namespace

cudaError_t launch_unpack_i4(const std::uint8_t* in, int nib_off, std::int64_t count, std::int8_t* out,
                             cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  if ((reinterpret_cast<std::uintptr_t>(in) & 3u) || (reinterpret_cast<std::uintptr_t>(out) & 7u)) {
    return cudaErrorMisalignedAddress;
  }
  const std::int64_t nbytes = (nib_off + count + 1) / 2;
  const std::int64_t groups = (count + 7) / 8;
  const std::int64_t cap = static_cast<std::int64_t>(sm_count()) * 8;
  const std::int64_t grid = std::min<std::int64_t>((groups + 255) / 256, cap);
  unpack_i4_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(reinterpret_cast<const std::uint32_t*>(in),
                                                                     nbytes, nib_off & 1, count, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace vd
