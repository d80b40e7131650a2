// tc_mma_rate.cu -- issue-to-completion time of back-to-back tcgen05.mma on one
// SM: kind::tf32 (K = 8) vs kind::f16 bf16 (K = 16), A from TMEM vs SMEM,
// N = 64 / 128, one accumulator vs two alternating.  Operand values are
// irrelevant (zeros); only timing is reported (clk per MMA).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int fmt, int M, int N) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int KIND, bool A_TMEM, int N, int NACC, int M = 128, int AROW = 0>
__global__ void probe(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
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
    constexpr uint32_t id = idesc(KIND == 0 ? 2 : 1, M, N);
    const uint64_t bdesc = sw128_desc(smem_u32(s));
    const uint64_t adesc = sw128_desc(smem_u32(s + 32768 + 128 * AROW));  // AROW: start AROW rows into a SW128 atom
    const uint32_t a_t = tmem, d0 = tmem + 256;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = d0 + (uint32_t)((r % NACC) * N);
      const uint32_t kb = (uint32_t)(r & 7);
      if (KIND == 2) {  // alternate kind::f16 and kind::tf32 into the same accumulator
        if (r & 1)
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
                       "r"(a_t + 8 * kb), "l"(bdesc + 2 * (kb & 3)), "r"(idesc(2, 128, N)) : "memory");
        else
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
                       "r"(a_t + 64 + 8 * kb), "l"(bdesc + 2 * (kb & 3)), "r"(idesc(1, 128, N)) : "memory");
      } else if (A_TMEM) {
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
                       "r"(a_t + 8 * kb), "l"(bdesc + 2 * (kb & 3)), "r"(id) : "memory");
        else
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
                       "r"(a_t + 8 * kb), "l"(bdesc + 2 * (kb & 3)), "r"(id) : "memory");
      } else {
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
                       "l"(adesc + 2 * (kb & 3)), "l"(bdesc + 2 * (kb & 3)), "r"(id) : "memory");
        else
          asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(d),
                       "l"(adesc + 2 * (kb & 3)), "l"(bdesc + 2 * (kb & 3)), "r"(id) : "memory");
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                     smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
        smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, bool A_TMEM, int N, int NACC, int M = 128, int AROW = 0>
void run(const char* name, long long* d) {
  auto k = probe<KIND, A_TMEM, N, NACC, M, AROW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int reps = 4096;
  k<<<148, 128, 80 * 1024>>>(d, 64);
  k<<<148, 128, 80 * 1024>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) printf("%-40s error %s\n", name, cudaGetErrorString(e));
  else printf("%-40s %6.1f clk/MMA (all 148 SMs busy)\n", name, (double)c / reps);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<0, true, 64, 1>("tf32 K=8  A=TMEM N=64  1 acc", d);
  run<1, true, 64, 1>("bf16 K=16 A=TMEM N=64  1 acc", d);
  run<0, false, 64, 1>("tf32 K=8  A=SMEM N=64  1 acc", d);
  run<1, false, 64, 1>("bf16 K=16 A=SMEM N=64  1 acc", d);
  run<0, true, 64, 2>("tf32 K=8  A=TMEM N=64  2 acc", d);
  run<1, true, 64, 2>("bf16 K=16 A=TMEM N=64  2 acc", d);
  run<0, true, 128, 1>("tf32 K=8  A=TMEM N=128 1 acc", d);
  run<1, true, 128, 1>("bf16 K=16 A=TMEM N=128 1 acc", d);
  run<1, false, 128, 1>("bf16 K=16 A=SMEM N=128 1 acc", d);
  run<0, true, 32, 1>("tf32 K=8  A=TMEM N=32  1 acc", d);
  run<2, true, 64, 1>("alternating f16/tf32 A=TMEM N=64 1 acc", d);
  run<2, true, 64, 2>("alternating f16/tf32 A=TMEM N=64 2 acc", d);
  run<0, true, 64, 1, 64>("M=64 tf32 K=8  A=TMEM N=64  1 acc", d);
  run<1, true, 64, 1, 64>("M=64 bf16 K=16 A=TMEM N=64  1 acc", d);
  run<0, false, 64, 1, 64>("M=64 tf32 K=8  A=SMEM N=64  1 acc", d);
  run<0, true, 128, 1, 64>("M=64 tf32 K=8  A=TMEM N=128 1 acc", d);
  run<1, false, 64, 1, 128, 1>("bf16 A=SMEM start +1 row (SW128) N=64", d);
  run<1, false, 64, 1, 128, 3>("bf16 A=SMEM start +3 rows (SW128) N=64", d);
  run<1, false, 64, 1, 128, 8>("bf16 A=SMEM start +8 rows (SW128) N=64", d);
  run<1, false, 128, 1, 128, 1>("bf16 A=SMEM start +1 row (SW128) N=128", d);
  return 0;
}
