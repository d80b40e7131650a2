// tc_bf16_tmem_probe.cu -- layout of a 16-bit A operand held in tensor memory
// for tcgen05.mma kind::f16 (bf16), needed by the mixed-precision conv_tc
// correction term.  A[r][k] is written with tcgen05.st (32-bit columns, two
// bf16 per column); B is a K-major SWIZZLE_128B selector, B[n][k] = (k == n),
// so D[r][n] = A[r][n] reveals which (column, half) holds K index n.
// Also checks that a kind::tf32 and a kind::f16 MMA accumulate into the same
// fp32 accumulator.
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
__device__ __forceinline__ uint16_t bf16_bits(float f) {  // exact for the small integers used here
  return (uint16_t)(__float_as_uint(f) >> 16);
}

__global__ void probe(float* out, int mode) {
  __shared__ __align__(1024) uint8_t bsm[16 * 1024];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (int)sizeof(bsm) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0;
  __syncthreads();
  constexpr int N = 32;
  if (threadIdx.x < 16) {
    // bf16 selector: row n (< 16), K index k = n -> 1.0
    const int n = threadIdx.x, k = n;
    const int unit = (k * 2) >> 4, byte = (k * 2) & 15;
    const int phys = unit ^ (n & 7);
    uint8_t* row = bsm + (n >> 3) * 1024 + (n & 7) * 128;
    *reinterpret_cast<uint16_t*>(row + phys * 16 + byte) = bf16_bits(1.0f);
  }
  if (threadIdx.x >= 32 && threadIdx.x < 32 + 8) {
    // tf32 selector at bsm + 8 KB: row n (< 8), K index n -> 1.0 (fp32)
    const int n = threadIdx.x - 32, k = n;
    const int unit = (k * 4) >> 4, byte = (k * 4) & 15;
    const int phys = unit ^ (n & 7);
    uint8_t* row = bsm + 8192 + (n & 7) * 128;
    *reinterpret_cast<float*>(row + phys * 16 + byte) = 1.0f;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t a_bf = tmem, a_tf = tmem + 8, d = tmem + 32;
  // A bf16: 8 columns, column c = {lo: 10 c + 1, hi: 10 c + 2} (+ 100 r for row r)
  // A tf32: 8 columns (K = 8), column c = 1000 + c
  {
    const int r = threadIdx.x;  // 128 threads: lane r of quarter r / 32
    uint32_t v[8], t[8];
    for (int c = 0; c < 8; ++c) {
      const float lo = 10.0f * c + 1.0f + (r & 1) * 100.0f, hi = 10.0f * c + 2.0f + (r & 1) * 100.0f;
      v[c] = (uint32_t)bf16_bits(lo) | ((uint32_t)bf16_bits(hi) << 16);
      t[c] = __float_as_uint(1000.0f + c);
    }
    const uint32_t lanebits = (uint32_t)(32 * warp) << 16;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a_bf + lanebits),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a_tf + lanebits),
                 "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint32_t idesc_bf = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc_tf = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bdesc = sw128_desc(smem_u32(bsm)), tdesc = sw128_desc(smem_u32(bsm + 8192));
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 0;\n\t}" ::"r"(d),
        "r"(a_bf), "l"(bdesc), "r"(idesc_bf)
        : "memory");
    if (mode == 1)
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(d),
          "r"(a_tf), "l"(tdesc), "r"(idesc_tf)
          : "memory");
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t v[32];
    const uint32_t lanebits = (uint32_t)(32 * warp) << 16;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(d + lanebits));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 32; ++n) out[threadIdx.x * 32 + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 32 * 4);
  float h[128 * 32];
  for (int mode = 0; mode < 2; ++mode) {
    probe<<<1, 128>>>(d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %d (%s)\n", mode, mode ? "bf16 then tf32 into the same D" : "bf16 only");
    for (int r : {0, 1, 64}) {
      printf("  D[%d][0..15] =", r);
      for (int n = 0; n < 16; ++n) printf(" %g", h[r * 32 + n]);
      printf("\n");
    }
  }
  printf("hypothesis (column n/2, half n%%2): D[0][n] = 10 (n/2) + n%%2 + 1; mode 1 adds 1000 + n for n < 8\n");
  return 0;
}
