// tc_lbo_probe.cu -- MN-major B whose MN atoms are the same rows shifted by one K row (LBO = 128 B); tcgen05.mma kind::f16 (bf16) with A in tensor memory (16-bit
// K pairs packed per 32-bit column, low half first) and an MN-major SWIZZLE_128B B
// operand (N contiguous, 64 bf16 per 128-B atom row), plus a B start shifted by two
// K rows (256 B): the layout a mixed-precision (TF32 + bf16 correction) filter
// gradient would use for its cross terms.  Small integers: exact, compared bit for bit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tc_lbo_probe.cu -o tc_lbo_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16_bmn(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr int kK = 24;  // three 8-row K atoms
constexpr int kN = 128;
constexpr uint32_t kLBO = (kK / 8) * 1024;  // MN atom (64 bf16) stride
__host__ __device__ inline float aval(int m, int k) { return (float)((m * 3 + k * 5) % 7 - 3); }
__host__ __device__ inline float bval(int k, int n) { return (float)((k * 7 + n * 3) % 11 - 5); }
__device__ inline uint16_t bf(float f) { return (uint16_t)(__float_as_uint(f) >> 16); }

__global__ void probe(float* out) {
  __shared__ __align__(1024) uint8_t bsm[(kN / 64) * kLBO];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < kK * 64; e += blockDim.x) {
    const int k = e / 64, c = e % 64;
    const int g = k / 8, r = k % 8, cc = c / 8;
    const uint32_t off = g * 1024 + r * 128 + ((cc ^ r) << 4) + (c % 8) * 2;
    *reinterpret_cast<uint16_t*>(bsm + off) = bf(bval(k, c));  // row k of the single-atom tile
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t a_t = tmem, d1 = tmem + 32, d2 = tmem + 32 + 128;
  {  // A[m][k], k < 16: column c = k pair (2c low, 2c + 1 high)
    const int m = threadIdx.x;
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) v[c] = (uint32_t)bf(aval(m, 2 * c)) | ((uint32_t)bf(aval(m, 2 * c + 1)) << 16);
    const uint32_t lanebits = (uint32_t)(32 * warp) << 16;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a_t + lanebits),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint64_t b1 = desc(smem_u32(bsm), 128, 1024), b2 = desc(smem_u32(bsm) + 256, 128, 1024);
    constexpr uint32_t i1 = idesc_bf16_bmn(128, 128), i2 = idesc_bf16_bmn(128, 64);
    asm volatile(
        "{\n\t.reg .pred e, z;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 z, %8, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, z;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%4], [%1], %5, %6, z;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}" ::"r"(d1),
        "r"(a_t), "l"(b1), "r"(i1), "r"(d2), "l"(b2), "r"(i2), "r"(smem_u32(&bar)), "r"(0));
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int m = threadIdx.x;
    const uint32_t lanebits = (uint32_t)(32 * warp) << 16;
    for (int c0 = 0; c0 < 192; c0 += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(d1 + lanebits + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int t = 0; t < 8; ++t) out[m * 192 + c0 + t] = __uint_as_float(v[t]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 192 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  static float h[128 * 192];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int bad1 = 0, bad2 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 192; ++n) {
      double ref = 0;
      if (n < 128) { for (int k = 0; k < 16; ++k) ref += aval(m, k) * bval(k + n / 64, n % 64); bad1 += h[m * 192 + n] != ref; }
      else { for (int k = 0; k < 16; ++k) ref += aval(m, k) * bval(k + 2, n - 128); bad2 += h[m * 192 + n] != ref; }
    }
  printf("LBO = 128 B (atom a = K rows shifted by a): N=128 mismatches %d / %d; control N=64 mismatches %d / %d\n",
         bad1, 128 * 128, bad2, 128 * 64);
  return (bad1 || bad2) ? 2 : 0;
}
