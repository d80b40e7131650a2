// tc_mn_probe.cu -- does tcgen05.mma kind::tf32 accept an MN-major SWIZZLE_128B B
// operand (N contiguous in shared memory), with A in tensor memory, and does a
// B start address shifted by one K row (128 B, inside a 1024-B swizzle atom)
// read K rows 1..8?  Integer-valued operands: the products are exact, so D is
// compared with a host reference bit for bit.  (Needed by a tensor-core filter
// gradient: B = x viewed as [chunk u][s] rows of 128, A = dy chunks.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tc_mn_probe.cu -o tc_mn_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MN-major SWIZZLE_128B descriptor: LBO = stride between 128-B MN atoms, SBO = stride between 8-row K atoms
__device__ __forceinline__ uint64_t mn_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

constexpr int kK = 16;  // two K atoms
constexpr int kN = 128;
constexpr uint32_t kLBO = (kK / 4) * 512;  // MN atom stride (SWIZZLE_128B_BASE32B: 4-row K atoms of 512 B)

__host__ __device__ inline float aval(int m, int k) { return (float)((m * 3 + k * 5) % 7 - 3); }
__host__ __device__ inline float bval(int k, int n) { return (float)((k * 7 + n * 3) % 11 - 5); }

__global__ void probe(float* out, int mode) {
  __shared__ __align__(1024) uint8_t bsm[16384];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < kK * kN; e += blockDim.x) {
    const int k = e / kN, n = e % kN;
    if (mode == 1) {  // MN-major 128B_BASE32B: 32-B chunk (n % 32) / 8 XOR (row % 4)
      const int a = n / 32, g = k / 4, r = k % 4, c = (n % 32) / 8;
      const uint32_t off = a * kLBO + g * 512 + r * 128 + ((c ^ r) << 5) + (n % 8) * 4;
      *reinterpret_cast<float*>(bsm + off) = bval(k, n);
    } else if (k < 8) {  // K-major control: row n (128 B), K index k at 16-B chunk k/4 ^ (n % 8)
      const uint32_t off = (n / 8) * 1024 + (n % 8) * 128 + (((k / 4) ^ (n % 8)) << 4) + (k % 4) * 4;
      *reinterpret_cast<float*>(bsm + off) = bval(k, n);
    }
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
  {  // A[m][k] in TMEM: lane m, column k (32-bit)
    const int m = threadIdx.x;
    uint32_t v[8];
    for (int k = 0; k < 8; ++k) v[k] = __float_as_uint(aval(m, k));
    const uint32_t lanebits = (uint32_t)(32 * warp) << 16;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a_t + lanebits),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint64_t b1 = mode ? mn_desc(smem_u32(bsm), kLBO, 512, 1) : mn_desc(smem_u32(bsm), 16, 1024);
    const uint64_t b2 = mn_desc(smem_u32(bsm) + 128, kLBO, 512, 1);  // K rows 1..8
    const uint32_t i1 = idesc_tf32(128, 128, mode), i2 = idesc_tf32(128, 64, 1);
    asm volatile(
        "{\n\t.reg .pred e, z;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 z, %8, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, z;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%4], [%1], %5, %6, z;\n\t"
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

int main(int argc, char** argv) {
  float* d;
  cudaMalloc(&d, 128 * 192 * 4);
  const int mode = argc > 1 ? atoi(argv[1]) : 1;
  printf("mode %d (%s)\n", mode, mode ? "MN-major B" : "K-major control");
  probe<<<1, 128>>>(d, mode);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  static float h[128 * 192];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int bad1 = 0, bad2 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 192; ++n) {
      double ref = 0;
      if (n < 128) { for (int k = 0; k < 8; ++k) ref += aval(m, k) * bval(k, n); if (h[m * 192 + n] != ref) ++bad1; }
      else { for (int k = 0; k < 8; ++k) ref += aval(m, k) * bval(k + 1, n - 128); if (h[m * 192 + n] != ref) ++bad2; }
    }
  printf("MN-major tf32 B: N=128 mismatches %d / %d, K-row-shifted N=64 mismatches %d / %d\n", bad1, 128 * 128, bad2,
         128 * 64);
  for (int n = 0; n < 12; ++n) { double r = 0; for (int k = 0; k < 8; ++k) r += aval(5, k) * bval(k, n); printf("D[5][%d]=%g ref %g\n", n, h[5*192+n], r); }
  { int nz = 0; for (int i = 0; i < 128 * 192; ++i) nz += h[i] != 0; printf("nonzero %d\n", nz); }
  printf("sample D[5][7] = %g (ref %g)\n", h[5 * 192 + 7], [] { double r = 0; for (int k = 0; k < 8; ++k) r += aval(5, k) * bval(k, 7); return r; }());
  return (bad1 || bad2) ? 2 : 0;
}
