// FFMA2 issue rate probe: 8 warps per SMSP-group, N independent accumulator
// pairs per thread, operand shapes (a) 3 register pairs, (b) pair x scalar
// broadcast, (c) pair x constant-bank pair.  Prints FMA/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
__constant__ float2 kc[64];
template <int MODE>
__global__ void probe(float* out, int iters, long long* cyc) {
  float2 acc[16], a[16], b[16];
  for (int i = 0; i < 16; ++i) { acc[i] = make_float2(threadIdx.x, i); a[i] = make_float2(1.0001f * i + threadIdx.x, 0.999f * threadIdx.x); b[i] = make_float2(0.5f + i * threadIdx.x, 0.25f + threadIdx.x); }
  float s = threadIdx.x * 0.001f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (MODE == 3) { acc[i].x = __fmaf_rn(a[(i + j) & 15].x, kc[j].x, acc[i].x); acc[i].y = __fmaf_rn(a[(i + j) & 15].y, kc[j].x, acc[i].y); }
        else if (MODE == 4) { acc[i].x = __fmaf_rn(a[(i + j) & 15].x, b[j].x, acc[i].x); acc[i].y = __fmaf_rn(a[(i + j) & 15].y, b[j].y, acc[i].y); }
        else if (MODE == 0) acc[i] = __ffma2_rn(a[(i + j) & 15], b[j], acc[i]);
        else if (MODE == 1) acc[i] = __ffma2_rn(a[(i + j) & 15], make_float2(s + j, s + j), acc[i]);
        else acc[i] = __ffma2_rn(a[(i + j) & 15], kc[j], acc[i]);
      }
  }
  long long t1 = clock64();
  float r = 0;
  for (int i = 0; i < 16; ++i) r += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4 * 4); cudaMalloc(&cyc, 8);
  float2 h[64]; for (int i = 0; i < 64; ++i) h[i] = make_float2(0.1f * i, 0.2f); cudaMemcpyToSymbol(kc, h, sizeof h);
  const int iters = 2000;
  for (int mode = 0; mode < 5; ++mode)
    for (int threads : {256, 512}) {
      auto k = mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2> : mode == 3 ? probe<3> : probe<4>;
      k<<<148, threads>>>(out, 10, cyc);
      cudaDeviceSynchronize();
      k<<<148, threads>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double fma = 2.0 * 256 * iters * threads;  // per SM (one CTA per SM)
      const char* names[] = {"FFMA2 3 reg pairs", "FFMA2 pair x scalar", "FFMA2 pair x c-bank pair", "FFMA scalar x c-bank", "FFMA 3 regs"};
      printf("%-26s threads %4d: %.1f FMA/clk/SM\n", names[mode], threads, fma / c);
    }
  return 0;
}
