// LDGSTS (cp.async) throughput from NW producer warps per SM: each CTA copies
// 112 rows x 448 B planes (the conv2d tile staging pattern) into shared memory,
// one cp.async.cg 16 B per lane per row, waits, repeats.  Prints GB/s.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const float* __restrict__ x, int planes_per_cta, int nw, int mode) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= nw) return;
  const unsigned s0 = (unsigned)__cvta_generic_to_shared(sm);
  for (int it = 0; it < planes_per_cta; ++it) {
    const float* src = x + ((size_t)(blockIdx.x * planes_per_cta + it) % 2048) * 112 * 112;
    for (int i = warp; i < 112; i += nw) {
      if (lane < 28) {
        const unsigned d = s0 + (unsigned)(i * 116 + 4 * lane) * 4u;
        if (mode == 0)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + i * 112 + 4 * lane) : "memory");
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + i * 112 + 4 * lane) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
}
int main() {
  float* x;
  cudaMalloc(&x, (size_t)2048 * 112 * 112 * 4);
  cudaMemset(x, 0, (size_t)2048 * 112 * 112 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode)
    for (int nw : {1, 2, 4, 8, 16}) {
      const int ppc = 14;
      k<<<148, 512, 116 * 112 * 4>>>(x, ppc, nw, mode);
      cudaEventRecord(a);
      k<<<148, 512, 116 * 112 * 4>>>(x, ppc, nw, mode);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("mode %s warps %2d: %.1f us, %.0f GB/s\n", mode ? "ca" : "cg", nw, ms * 1e3,
             148.0 * ppc * 112 * 112 * 4 / (ms * 1e-3) / 1e9);
    }
  return 0;
}
