// FFMA2 throughput in the conv kernel's operand pattern: acc_pair += x_pair * f_scalar,
// with NACC independent accumulator pairs and NX distinct input pairs.
#include <cstdio>
#include <cuda_runtime.h>
struct Taps { float f[64]; };
template <int NACC, int NX>
__global__ void __launch_bounds__(512, 1) k_ffma2(float* out, Taps t, int iters) {
  float2 acc[NACC], x[NX];
  for (int i = 0; i < NACC; ++i) acc[i] = make_float2(0.f, 0.f);
  for (int i = 0; i < NX; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float2 f2 = make_float2(t.f[j], t.f[j]);
#pragma unroll
      for (int i = 0; i < NACC; ++i) acc[i] = __ffma2_rn(x[(i + j) % NX], f2, acc[i]);
    }
  }
  float s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i].x + acc[i].y;
  if (s == 1234.5f) out[0] = s;
}
template <int NACC, int NX>
__global__ void __launch_bounds__(512, 1) k_ffma(float* out, Taps t, int iters) {
  float acc[2 * NACC], x[2 * NX];
  for (int i = 0; i < 2 * NACC; ++i) acc[i] = 0.f;
  for (int i = 0; i < 2 * NX; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float f = t.f[j];
#pragma unroll
      for (int i = 0; i < 2 * NACC; ++i) acc[i] = __fmaf_rn(x[(i + j) % (2 * NX)], f, acc[i]);
    }
  }
  float s = 0;
  for (int i = 0; i < 2 * NACC; ++i) s += acc[i];
  if (s == 1234.5f) out[0] = s;
}
template <class F>
void run(const char* name, F kern, int threads, double fma_per_thread_iter) {
  float* out; cudaMalloc(&out, 4);
  Taps t; for (int i = 0; i < 64; ++i) t.f[i] = 0.999f;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 400;
  kern<<<148, threads>>>(out, t, iters);
  cudaEventRecord(a);
  kern<<<148, threads>>>(out, t, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fmas = 148.0 * threads * iters * fma_per_thread_iter;
  printf("%-40s threads %d: %.2f TFMA/s\n", name, threads, fmas / ms / 1e9);
}
int main() {
  run("ffma2 acc8 x24 (conv-like)", k_ffma2<8, 24>, 512, 32 * 16);
  run("ffma2 acc9 x24", k_ffma2<9, 24>, 512, 32 * 18);
  run("ffma2 acc16 x24", k_ffma2<16, 24>, 512, 32 * 32);
  run("ffma2 acc8 x24 256thr", k_ffma2<8, 24>, 256, 32 * 16);
  run("ffma  acc16 x48", k_ffma<8, 24>, 512, 32 * 16);
  run("ffma  acc32 x48", k_ffma<16, 24>, 512, 32 * 32);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
