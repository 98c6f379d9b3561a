// Integer-pipe microbenchmarks for the ACS roofline denominator (bench.py,
// DESIGN.md §4). Each variant runs 8 independent dependency chains per
// thread over a full-occupancy grid and reports warp-instructions per SM
// clock (clock64 deltas on every SM) plus the achieved lane-op rate.
//
// op codes:
//   0 VIADD.16x2           (__vadd2)
//   1 VIMNMX.S16x2         (__vmaxs2)
//   2 VIADD.16x2 + VIMNMX  (the packed ACS mix: 2 adds : 1 max)
//   3 IADD3                (a - b + c)
//   4 IMAD                 (a * b + c)
//   5 PRMT                 (__byte_perm)
//   6 LOP3                 ((a & b) | c)
//   7 VIADD.16x2 + IMAD    (pipe co-issue probe)
//   8 VIMNMX + IMAD        (pipe co-issue probe)
//   9 SHFL.BFLY            (__shfl_xor_sync)
//  10 VIMNMX with predicate outputs consumed by SEL (decision extraction)
//  11 the fast kernel's packed ACS: s2 = VIADD.16x2(sO, T'), n = VIADDMNMX.S16x2(sE, T, s2)
//     (1:1 fmaheavy : alu; 3 lane-ops per instruction, 2 frames per register)
#include <cuda_runtime.h>

#include <cstdint>

namespace {

template <int OP>
__global__ void __launch_bounds__(256) mb_kernel(std::uint32_t seed, int iters, std::uint32_t* out,
                                                 unsigned long long* span) {
  std::uint32_t x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = seed * (threadIdx.x + 3 * i + 1);
    y[i] = seed ^ (i * 0x9e3779b9u + threadIdx.x);
  }
  const std::uint32_t m = seed | 1u;
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if constexpr (OP == 0) {
          x[i] = __vadd2(x[i], y[i]);
        } else if constexpr (OP == 1) {
          x[i] = __vmaxs2(x[i], y[i]);
          y[i] ^= 1u;  // keep the max from being constant-folded across iterations
        } else if constexpr (OP == 2) {
          const std::uint32_t a = __vadd2(x[i], y[i]);
          const std::uint32_t b = __vadd2(x[(i + 1) & 7], y[(i + 3) & 7]);
          x[i] = __vmaxs2(a, b);
        } else if constexpr (OP == 3) {
          x[i] = x[i] - y[i] + x[(i + 1) & 7];
        } else if constexpr (OP == 4) {
          x[i] = x[i] * m + y[i];
        } else if constexpr (OP == 5) {
          x[i] = __byte_perm(x[i], y[i], 0x5140 + u);
        } else if constexpr (OP == 6) {
          x[i] = (x[i] & y[i]) | x[(i + 1) & 7];
        } else if constexpr (OP == 7) {
          x[i] = __vadd2(x[i], y[i]);
          y[i] = y[i] * m + x[(i + 1) & 7];
        } else if constexpr (OP == 8) {
          x[i] = __vmaxs2(x[i], y[i]);
          y[i] = y[i] * m + x[(i + 1) & 7];
        } else if constexpr (OP == 9) {
          x[i] = __shfl_xor_sync(0xffffffffu, x[i], 1 + (i & 3)) + y[i];
        } else if constexpr (OP == 11) {
          const std::uint32_t s2 = __vadd2(x[(i + 1) & 7], y[i]);
          x[i] = __viaddmax_s16x2(x[i], y[(i + 3) & 7], s2);
        } else if constexpr (OP == 10) {
          bool hi, lo;
          x[i] = __vibmax_s16x2(x[i], y[i], &hi, &lo);
          y[i] += lo ? 3u : 5u;
          y[i] += hi ? 7u : 11u;
        }
      }
    }
  }
  const long long c1 = clock64();
  std::uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= x[i] + y[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  // per-SM active span: earliest start and latest end of any block on this SM
  // (clock64 is a per-SM counter; blocks of one SM need not overlap fully)
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    atomicMin(span + 2 * smid, static_cast<unsigned long long>(c0));
    atomicMax(span + 2 * smid + 1, static_cast<unsigned long long>(c1));
  }
}

__global__ void span_init(unsigned long long* span, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) span[i] = (i & 1) ? 0ull : ~0ull;
}

template <int OP>
cudaError_t run(int blocks, int threads, int iters, float* ms, double* avg_cycles) {
  std::uint32_t* out = nullptr;
  unsigned long long* cyc = nullptr;
  const int nspan = 2 * 1024;  // smid < 1024
  cudaMalloc(&out, sizeof(std::uint32_t) * blocks * threads);
  cudaMalloc(&cyc, sizeof(unsigned long long) * nspan);
  span_init<<<(nspan + 255) / 256, 256>>>(cyc, nspan);
  mb_kernel<OP><<<blocks, threads>>>(0x12345u, 16, out, cyc);  // warm-up
  span_init<<<(nspan + 255) / 256, 256>>>(cyc, nspan);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mb_kernel<OP><<<blocks, threads>>>(0x12345u, iters, out, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  static unsigned long long h[2 * 1024];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * nspan, cudaMemcpyDeviceToHost);
  double sum = 0.0;
  int used = 0;
  for (int i = 0; i < nspan / 2; ++i) {
    if (h[2 * i + 1] != 0ull) {
      sum += static_cast<double>(h[2 * i + 1] - h[2 * i]);
      ++used;
    }
  }
  *avg_cycles = used ? sum / used : 0.0;  // mean per-SM active span (cycles)
  cudaFree(out);
  cudaFree(cyc);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (err == cudaSuccess) err = cudaGetLastError();
  return err;
}

}  // namespace

extern "C" {

/// Instructions of the measured kind issued per thread per inner iteration
/// (x8 chains x4 unroll), by op code.
int vdmb_instr_per_iter(int op) {
  static const int k[] = {32, 32, 96, 32, 32, 32, 32, 64, 64, 32, 32, 64};
  return (op >= 0 && op <= 11) ? k[op] : 0;
}

/// Runs op over blocks x threads for iters iterations. Returns the elapsed
/// milliseconds and the mean per-SM active span (clock64 cycles from the
/// first block start to the last block end on that SM) of the timed loop.
int vdmb_run(int op, int blocks, int threads, int iters, float* ms, double* avg_cycles) {
  switch (op) {
    case 0: return run<0>(blocks, threads, iters, ms, avg_cycles);
    case 1: return run<1>(blocks, threads, iters, ms, avg_cycles);
    case 2: return run<2>(blocks, threads, iters, ms, avg_cycles);
    case 3: return run<3>(blocks, threads, iters, ms, avg_cycles);
    case 4: return run<4>(blocks, threads, iters, ms, avg_cycles);
    case 5: return run<5>(blocks, threads, iters, ms, avg_cycles);
    case 6: return run<6>(blocks, threads, iters, ms, avg_cycles);
    case 7: return run<7>(blocks, threads, iters, ms, avg_cycles);
    case 8: return run<8>(blocks, threads, iters, ms, avg_cycles);
    case 9: return run<9>(blocks, threads, iters, ms, avg_cycles);
    case 10: return run<10>(blocks, threads, iters, ms, avg_cycles);
    case 11: return run<11>(blocks, threads, iters, ms, avg_cycles);
    default: return -1;
  }
}

int vdmb_sm_count(void) {
  int d = 0, n = 0;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  return n;
}

}  // extern "C"
