// Microbenchmarks used to pick kernel designs (not part of the product):
//  1. FFMA throughput with a constant-bank operand vs FFMA2 (fma.rn.f32x2, sm_100a)
//  2. streaming copy bandwidth with 128-bit LDG/STG
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Taps { float f[64]; };

template <int NACC>
__global__ void ffma_cbank(float* out, Taps t, int iters) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float x = blockIdx.x * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) acc[i] = fmaf(t.f[j], acc[i], x);
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

template <int NACC>
__global__ void ffma2_kernel(float* out, Taps t, int iters) {
  // NACC float accumulators as NACC/2 pairs
  unsigned long long acc[NACC / 2];
#pragma unroll
  for (int i = 0; i < NACC / 2; ++i) {
    float a = threadIdx.x * 1e-3f + i, b = a + 0.5f;
    acc[i] = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
  }
  float x = blockIdx.x * 1e-4f;
  unsigned long long xx = ((unsigned long long)__float_as_uint(x) << 32) | __float_as_uint(x);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      unsigned long long ff = ((unsigned long long)__float_as_uint(t.f[j]) << 32) | __float_as_uint(t.f[j]);
#pragma unroll
      for (int i = 0; i < NACC / 2; ++i)
        asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(acc[i]) : "l"(ff), "l"(xx));
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC / 2; ++i) s += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32));
  if (s == 12345.f) out[0] = s;
}

__global__ void copy128(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n4; i += stride) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d l2 %d MB smem/blk optin %zu clock %d kHz\n", p.name, p.multiProcessorCount,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, clk);
  float* out; cudaMalloc(&out, 4);
  Taps t; for (int i = 0; i < 64; ++i) t.f[i] = 0.999f + i * 1e-6f;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  for (int blocksPerSM : {2, 4, 8}) {
    int grid = p.multiProcessorCount * blocksPerSM, block = 256;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      ffma_cbank<16><<<grid, block>>>(out, t, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas = (double)grid * block * iters * 32 * 16;
      if (rep) printf("FFMA  cbank  blocks/SM %d : %.2f TFMA/s (%.3f ms)\n", blocksPerSM, fmas / ms / 1e9, ms);
      cudaEventRecord(e0);
      ffma2_kernel<16><<<grid, block>>>(out, t, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("FFMA2        blocks/SM %d : %.2f TFMA/s (%.3f ms)\n", blocksPerSM, fmas / ms / 1e9, ms);
    }
  }
  size_t n = (size_t)1 << 30;  // 1 Gi floats = 4 GiB each
  float *a, *b; cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4);
  cudaMemset(a, 0, n * 4);
  for (int bps : {2, 4, 8}) {
    int grid = p.multiProcessorCount * bps;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      copy128<<<grid, 512>>>((const float4*)a, (float4*)b, n / 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("copy128 grid %d x 512: %.1f GB/s\n", grid, 2.0 * n * 4 / ms / 1e6);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
