// tc_mn_rate.cu -- clk per back-to-back kind::f16 (bf16) tcgen05.mma with both operands in shared
// memory, MN-major (the filter-gradient layout, mc_fgrad.cu) vs K-major, by M, N and the B operand's
// MN-atom stride (LBO = 128 B: atoms overlap, one row apart -- the tap trick; 2048 B: disjoint).
// Operand values are zeros; only timing is reported.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tc_mn_rate.cu -o tc_mn_rate
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
__host__ __device__ constexpr uint32_t idesc(int M, int N, int mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)mn << 15) | ((uint32_t)mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void probe(long long* out, int M, int N, int mn, uint32_t blbo, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
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
  if (warp == 0) {
    const uint32_t id = idesc(M, N, mn);
    // MN-major: A atoms (64 M each) 16 KB apart, K step 2 KB (16 rows); B atoms blbo apart.
    // K-major: 8-row groups SBO 1024, K step 32 B.
    const uint32_t a0 = smem_u32(s), b0 = smem_u32(s + 49152);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t ks = (uint32_t)(r & 7);
      const uint64_t ad = mn ? desc(a0 + 2048u * ks, 16384u, 1024u) : desc(a0 + 32u * (ks & 3), 16u, 1024u);
      const uint64_t bd = mn ? desc(b0 + 2048u * ks, blbo, 1024u) : desc(b0 + 32u * (ks & 3), 16u, 1024u);
      asm volatile(
          "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(id), "r"(r > 0 ? 1 : 0)
          : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)));
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  struct C { int M, N, mn; uint32_t lbo; const char* what; } cs[] = {
      {64, 192, 1, 128, "MN M64 N192 B atoms overlap (mc_fgrad k=3)"},
      {64, 192, 1, 16384, "MN M64 N192 B atoms disjoint"},
      {64, 64, 1, 16384, "MN M64 N64"},
      {64, 128, 1, 16384, "MN M64 N128"},
      {64, 256, 1, 128, "MN M64 N256 overlap (k=4)"},
      {128, 64, 1, 16384, "MN M128 N64"},
      {128, 128, 1, 128, "MN M128 N128 overlap (cout=128, k=2)"},
      {128, 192, 1, 16384, "MN M128 N192"},
      {64, 192, 0, 0, "K-major M64 N192"},
      {128, 192, 0, 0, "K-major M128 N192"},
      {128, 64, 0, 0, "K-major M128 N64"},
  };
  const int reps = 4096;
  for (auto& c : cs) {
    probe<<<148, 128, 110 * 1024>>>(d, c.M, c.N, c.mn, c.lbo, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: error %s\n", c.what, cudaGetErrorString(e)); return 1; }
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += h[i];
    printf("%-45s %7.1f clk/MMA (all 148 SMs)\n", c.what, s / 148 / reps);
  }
  return 0;
}
