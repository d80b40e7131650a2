// tc_probe.cu -- validates the tcgen05 (kind::tf32) encodings used by the
// tensor-core conv: SW128 K-major smem descriptors (incl. start addresses
// shifted by whole 128-B rows, i.e. the "overlapping im2col rows" trick),
// the instruction descriptor, TMEM alloc/ld and commit-to-mbarrier.
//
// A (M=128 x K) is read from a swizzled "stage" of 32-element rows:
//   A[m][k] = stage_row(m + k/32)[k%32]  ->  A[m][k] = x[32*m + k]
// B (N=32 x K, K-major) holds B[n][k] = f[k - n] (Toeplitz), so
//   D[m][n] = sum_k x[32m + k] f[k - n] = y[32m + n]  (a 1-D correlation).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t swz128(uint32_t off) { return off ^ ((off >> 3) & 0x70u); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t sbo, int base_mode) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)(1) << 16;                        // LBO (unused for SW128 K-major) = 1
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;      // SBO
  d |= (uint64_t)1 << 46;                          // version = 1 (sm100)
  if (base_mode == 1) d |= (uint64_t)((saddr >> 7) & 7) << 49;  // base offset
  d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
  return d;
}

constexpr int M = 128, N = 32;
template <int KSTEPS>
__global__ void probe(const float* __restrict__ x, const float* __restrict__ f, float* __restrict__ y,
                      int row_shift, int base_mode, int nbatch) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage: (M + KSTEPS/4 + 8) rows of 128 B; B: KSTEPS/4 atoms of 32 rows x 128 B
  constexpr int KA = (KSTEPS + 3) / 4;                  // 128-B K-atoms
  constexpr int SROWS = M + KA + 8;
  uint8_t* stage = smem;
  uint8_t* bsm = smem + ((SROWS * 128 + 1023) / 1024) * 1024;
  uint64_t* bar = reinterpret_cast<uint64_t*>(bsm + KA * 4096);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // fill stage: element e of row r = x[32*(r - row_shift) + e] (rows before row_shift = 0)
  for (int i = tid; i < SROWS * 32; i += blockDim.x) {
    int r = i / 32, e = i % 32;
    int g = 32 * (r - row_shift) + e;
    float v = (g >= 0 && g < 32 * (M + KA + 4)) ? x[g] : 0.f;
    *reinterpret_cast<float*>(stage + swz128((uint32_t)(4 * i))) = v;
  }
  // fill B: atom a, row n, element e (k = 32a + e): f[k - n]
  for (int i = tid; i < KA * 32 * 32; i += blockDim.x) {
    int a = i / 1024, n = (i / 32) % 32, e = i % 32;
    int k = 32 * a + e, j = k - n;
    float v = (j >= 0 && j < 4 * KSTEPS) ? f[j] : 0.f;  // f has 4*KSTEPS entries
    *reinterpret_cast<float*>(bsm + a * 4096 + swz128((uint32_t)(4 * (n * 32 + e)))) = v;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    for (int kb = 0; kb < KSTEPS; ++kb) {
      const uint32_t a_addr = smem_u32(stage) + 128u * (row_shift + kb / 4) + 32u * (kb % 4);
      const uint32_t b_addr = smem_u32(bsm) + 4096u * (kb / 4) + 32u * (kb % 4);
      const uint64_t ad = make_desc(a_addr, 1024, base_mode);
      const uint64_t bd = make_desc(b_addr, 1024, base_mode);
      const uint32_t acc = kb > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  }
  // wait
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
          smem_u32(bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int m = 32 * warp + lane;
    for (int n = 0; n < 32; ++n) y[m * 32 + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  constexpr int KS = 12;  // K = 96
  const int NX = 32 * (M + 8 + 8);
  float *x, *f, *y;
  cudaMallocManaged(&x, NX * 4);
  cudaMallocManaged(&f, 4 * KS * 4);
  cudaMallocManaged(&y, M * N * 4);
  srand(1);
  // values exactly representable in tf32 (11 significant bits) -> exact products
  for (int i = 0; i < NX; ++i) x[i] = (float)((rand() % 2001) - 1000) / 64.f;
  for (int j = 0; j < 4 * KS; ++j) f[j] = (j < 63) ? (float)((rand() % 201) - 100) / 32.f : 0.f;
  const size_t smem = 1024 + ((M + 3 + 8) * 128 + 1023) / 1024 * 1024 + 3 * 4096 + 64;
  cudaFuncSetAttribute(probe<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int base_mode = 0; base_mode < 2; ++base_mode) {
    for (int shift : {0, 1, 3, 5}) {
      cudaMemset(y, 0, M * N * 4);
      probe<KS><<<1, 128, smem>>>(x, f, y, shift, base_mode, 1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("base_mode %d shift %d: CUDA error %s\n", base_mode, shift, cudaGetErrorString(e)); return 1; }
      double maxerr = 0; int bad = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int j = 0; j < 63; ++j) ref += (double)f[j] * x[32 * m + n + j];
          double err = fabs(ref - y[m * N + n]);
          if (err > maxerr) maxerr = err;
          if (err > 1e-3 * (1 + fabs(ref))) ++bad;
        }
      printf("base_mode %d row_shift %d: max err %.3g, bad %d of %d\n", base_mode, shift, maxerr, bad, M * N);
    }
  }
  return 0;
}
