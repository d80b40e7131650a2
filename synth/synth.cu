// synth.cu -- device twin of synth/__init__.py: the counter-based splitmix64
// input generator.  Holds none of the method's arithmetic.
// Element i of a stream depends only on (seed, i), so any shard / slice can be
// produced independently and matches the host generator bit for bit.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sm64(uint64_t seed, uint64_t c) {
  uint64_t z = seed + (c + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_uniform(float* out, int64_t n, uint64_t seed, int64_t start, int pm1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t z = sm64(seed, (uint64_t)(start + i));
    const float u = __fmul_rn((float)(uint32_t)(z >> 40), 5.9604644775390625e-08f);  // 2^-24
    out[i] = pm1 ? __fsub_rn(__fmul_rn(2.0f, u), 1.0f) : u;
  }
}

// uniform on [lo, lo+span): fl(lo + fl(span * u01)), the host twin's order.
__global__ void k_uab(float* out, int64_t n, uint64_t seed, float lo, float span, int64_t start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t z = sm64(seed, (uint64_t)(start + i));
    const float u = __fmul_rn((float)(uint32_t)(z >> 40), 5.9604644775390625e-08f);  // 2^-24
    out[i] = __fadd_rn(lo, __fmul_rn(span, u));
  }
}

__global__ void k_randint(int32_t* out, int64_t n, uint64_t seed, int64_t lo, uint64_t span, int64_t start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t z = sm64(seed, (uint64_t)(start + i));
    const uint64_t r = ((z >> 32) * span) >> 32;
    out[i] = (int32_t)((int64_t)r + lo);
  }
}

__global__ void k_normal(float* out, int64_t n, uint64_t seed, double sigma, int64_t start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t base = (uint64_t)(start + i) * 3ull;
    int64_t S = 0;
#pragma unroll
    for (int part = 0; part < 3; ++part) {
      const uint64_t z = sm64(seed, base + part);
#pragma unroll
      for (int lane = 0; lane < 4; ++lane) S += (int64_t)((z >> (16 * lane)) & 0xFFFFull);
    }
    const double v = __dmul_rn((double)(S - 6 * 65536), 1.52587890625e-05);  // 2^-16, exact
    out[i] = __double2float_rn(__dmul_rn(v, sigma));
  }
}

static unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (unsigned)(g > 148 * 32 ? 148 * 32 : (g < 1 ? 1 : g));
}

extern "C" {
int synth_uniform01(float* out, int64_t n, uint64_t seed, int64_t start, void* stream) {
  k_uniform<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, n, seed, start, 0);
  return (int)cudaGetLastError();
}
int synth_uniform_pm1(float* out, int64_t n, uint64_t seed, int64_t start, void* stream) {
  k_uniform<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, n, seed, start, 1);
  return (int)cudaGetLastError();
}
int synth_uab(float* out, int64_t n, uint64_t seed, float lo, float span, int64_t start, void* stream) {
  k_uab<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, n, seed, lo, span, start);
  return (int)cudaGetLastError();
}
int synth_randint(int32_t* out, int64_t n, uint64_t seed, int64_t lo, int64_t hi, int64_t start, void* stream) {
  k_randint<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, n, seed, lo, (uint64_t)(hi - lo + 1), start);
  return (int)cudaGetLastError();
}
int synth_normal(float* out, int64_t n, uint64_t seed, double sigma, int64_t start, void* stream) {
  k_normal<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, n, seed, sigma, start);
  return (int)cudaGetLastError();
}
}
