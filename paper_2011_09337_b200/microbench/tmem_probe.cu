// TMEM round-trip probe: 4 warps allocate 512 columns, each warp stores
// (warp, lane, col) signatures with tcgen05.st.32x32b and reads them back with
// tcgen05.ld.32x32b.x4; verifies the lane/column addressing the fast decoder
// kernel relies on (TMEM as survivor-decision storage).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(384, 1) probe(unsigned* out, int* ok) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((unsigned)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s;
  const uint32_t q = warp & 3, cb = (warp >> 2) * 170;
  const uint32_t t = base + ((32u * q) << 16) + cb;
  for (int c = 0; c < 168; ++c) {
    const uint32_t v = (warp << 24) | (lane << 16) | c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(t + c), "r"(v) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  int good = 1;
  long long t0 = clock64();
  for (int c = 0; c < 168; c += 4) {
    uint32_t a, b, d, e;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(d), "=r"(e) : "r"(t + c) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const uint32_t ex = (warp << 24) | (lane << 16) | c;
    good &= (a == ex) && (b == ex + 1) && (d == ex + 2) && (e == ex + 3);
  }
  long long t1 = clock64();
  if (!good) atomicExch(ok, 0);
  if (threadIdx.x == 0) out[0] = (unsigned)((t1 - t0) / 42);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
}

int main() {
  unsigned* out; int* ok;
  cudaMalloc(&out, 4); cudaMalloc(&ok, 4);
  int one = 1; cudaMemcpy(ok, &one, 4, cudaMemcpyHostToDevice);
  probe<<<148, 384>>>(out, ok);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned cyc; int good;
  cudaMemcpy(&cyc, out, 4, cudaMemcpyDeviceToHost); cudaMemcpy(&good, ok, 4, cudaMemcpyDeviceToHost);
  printf("tmem probe: %s, err=%s, cycles per ld.x4+wait = %u\n", good ? "OK" : "MISMATCH", cudaGetErrorString(e), cyc);
  return good && e == cudaSuccess ? 0 : 1;
}
