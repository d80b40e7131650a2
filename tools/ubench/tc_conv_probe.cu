// tc_conv_probe.cu -- validates the building blocks of a tensor-core conv1d for
// large k ("small matrix multiplication"),
// in the TRANSPOSED orientation:
//   D[r][m] = sum_kk A[r][kk] * B[m][kk] = y[P0 + 128 m + r]
//   A[r][kk] = f[kk - r]        (Toeplitz, 128 x K, resident in TMEM, hi + lo)
//   B[m][kk] = x[P0 + 128 m + kk] (x chunks, K-major SW128 in smem, one 128-B
//                                 K-atom a = x rows 4m + a: overlapping TMA box)
// Checks: (1) which TMA form produces the B layout (3-D map with non-monotonic
// strides, or a 2-D map with elementStrides {1,4}); (2) MMA with A from TMEM;
// (3) whether the tensor core truncates or rounds fp32 -> tf32 (error of
// 3xTF32 with lo = x - trunc(x) vs lo = x - rna(x)); (4) MMA issue rate
// (N = 32 / 64, A from TMEM vs smem) on all SMs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts_e(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ss_e(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_e(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

constexpr int KMAX = 64;
constexpr int NC = 32;  // chunks (B rows, MMA N) per tile
struct Prm {
  CUtensorMap tm;       // B staging map
  int tma_mode;         // 0: 3-D overlapped strides; 1: 2-D elementStrides {1,4}, one load per atom
  int k, K, atoms;      // filter length, MMA K (mult of 8), K-atoms of 32
  int lo_mode;          // 0: lo = x - trunc(x); 1: lo = x - rna(x)
  int products;         // 1: hi*hi only; 3: 3xTF32
  float f[KMAX];
};

// One tile: outputs y[128 m + r], m < NC, r < 128, from x (flat, 16-B aligned).
__global__ void __launch_bounds__(128, 1) conv_tile(const __grid_constant__ Prm p, float* y) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int atom_bytes = NC * 128;
  uint8_t* bhi = sm;
  uint8_t* blo = sm + p.atoms * atom_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(blo + p.atoms * atom_bytes);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + 1)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t bytes = (uint32_t)(p.atoms * atom_bytes);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    if (p.tma_mode == 0) {
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(bhi)),
          "l"(reinterpret_cast<uint64_t>(&p.tm)), "r"(0), "r"(0), "r"(0), "r"(smem_u32(bar))
          : "memory");
    } else {
      for (int a = 0; a < p.atoms; ++a)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(bhi + a * atom_bytes)),
            "l"(reinterpret_cast<uint64_t>(&p.tm)), "r"(0), "r"(a), "r"(smem_u32(bar))
            : "memory");
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  const uint32_t a_hi = tmem, a_lo = tmem + 192, dcol = tmem + 384;
  // Toeplitz rows into TMEM: lane r = tid holds A[r][kk] = f[kk - r]
  {
    const int r = tid;
    for (int c = 0; c < p.K / 32 + ((p.K % 32) ? 1 : 0); ++c) {
      float vh[32], vl[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int t = 32 * c + j - r;
        const float f = (t >= 0 && t < p.k) ? p.f[t] : 0.f;
        vh[j] = tf32_trunc(f);
        vl[j] = tf32_trunc(f - vh[j]);
      }
      const uint32_t lanebits = (uint32_t)(32 * warp) << 16;
      tmem_st32(a_hi + lanebits + 32 * c, vh);
      tmem_st32(a_lo + lanebits + 32 * c, vl);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  wait_bar(bar, 0);
  // lo pass (elementwise: swizzle-agnostic)
  for (int i = tid; i < p.atoms * atom_bytes / 4; i += blockDim.x) {
    const float x = reinterpret_cast<const float*>(bhi)[i];
    reinterpret_cast<float*>(blo)[i] = x - (p.lo_mode == 0 ? tf32_trunc(x) : tf32_rna(x));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t id = idesc_tf32(128, NC);
    uint32_t acc = 0;
    for (int kb = 0; kb < p.K / 8; ++kb) {
      const uint32_t off = (uint32_t)((kb >> 2) * atom_bytes + 32 * (kb & 3));
      const uint64_t dh = make_desc(smem_u32(bhi) + off, 1024);
      const uint64_t dl = make_desc(smem_u32(blo) + off, 1024);
      if (p.products == 3) {
        mma_ts(dcol, a_lo + 8 * kb, dh, id, acc);
        acc = 1;
        mma_ts(dcol, a_hi + 8 * kb, dl, id, acc);
      }
      mma_ts(dcol, a_hi + 8 * kb, dh, id, acc);
      acc = 1;
    }
    commit(bar + 1);
  }
  wait_bar(bar + 1, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t v[32];
    tmem_ld32(dcol + ((uint32_t)(32 * warp) << 16), v);
    for (int m = 0; m < NC; ++m) y[128 * m + tid] = __uint_as_float(v[m]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// MMA issue-rate loop: one CTA per SM, one thread issues `iters` x KS MMAs
// (M=128, N, K=8) with A from TMEM (a_src 0) or smem (a_src 1).
template <int N>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, int a_src, int nd, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536 + 16384);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (65536 + 16384) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    const uint32_t id = idesc_tf32(128, N);
    const uint32_t bbase = __shfl_sync(0xffffffffu, smem_u32(sm + 65536), 0);
    const uint32_t abase = __shfl_sync(0xffffffffu, smem_u32(sm), 0);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const long long t0 = clock64();
    if (a_src == 0) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kb = 0; kb < 24; ++kb)
          mma_ts_e(tm + 256 + (uint32_t)((kb % nd) * N), tm + 8 * (kb & 15),
                   make_desc(bbase + 32 * (kb & 3), 1024), id, 1);
      }
    } else {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kb = 0; kb < 24; ++kb)
          mma_ss_e(tm + 256 + (uint32_t)((kb % nd) * N),
                   make_desc(abase + ((kb >> 2) & 3) * 16384 + 32 * (kb & 3), 1024),
                   make_desc(bbase + 32 * (kb & 3), 1024), id, 1);
      }
    }
    commit_e(bar);
    wait_bar(bar, 0);
    const long long t1 = clock64();
    if (tid == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fp;
  const int k = 63;
  const int K = ((127 + k) + 7) / 8 * 8;  // 192
  const int atoms = (K + 31) / 32;        // 6
  const int nx = 128 * NC + 32 * atoms + 1024;
  std::vector<float> hx(nx), hf(k);
  srand(7);
  auto rnd = [] { return (float)((double)rand() / RAND_MAX * 2.0 - 1.0); };
  for (auto& v : hx) v = rnd();
  for (auto& v : hf) v = rnd() * 0.2f;
  float *dx, *dy;
  CK(cudaMalloc(&dx, nx * 4));
  CK(cudaMalloc(&dy, 128 * NC * 4));
  CK(cudaMemcpy(dx, hx.data(), nx * 4, cudaMemcpyHostToDevice));
  const size_t smem = 1024 + 2 * atoms * NC * 128 + 64;
  CK(cudaFuncSetAttribute(conv_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int mext = (nx - 32 * atoms) / 128;  // chunks whose whole K span is inside x
  for (int tma_mode = 0; tma_mode < 2; ++tma_mode) {
    Prm p;
    memset(&p, 0, sizeof p);
    CUresult r;
    if (tma_mode == 0) {
      cuuint64_t dims[3] = {32, (cuuint64_t)mext, (cuuint64_t)atoms};
      cuuint64_t strides[2] = {512, 128};
      cuuint32_t box[3] = {32, NC, (cuuint32_t)atoms};
      cuuint32_t es[3] = {1, 1, 1};
      r = enc(&p.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[2] = {32, (cuuint64_t)(nx / 32)};
      cuuint64_t strides[1] = {128};
      cuuint32_t box[2] = {32, 4 * NC};
      cuuint32_t es[2] = {1, 4};
      r = enc(&p.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("tma_mode %d: encode %s\n", tma_mode, r == CUDA_SUCCESS ? "ok" : "FAILED");
    if (r != CUDA_SUCCESS) continue;
    p.tma_mode = tma_mode;
    p.k = k;
    p.K = K;
    p.atoms = atoms;
    for (int j = 0; j < k; ++j) p.f[j] = hf[j];
    for (int products : {1, 3})
      for (int lo_mode = 0; lo_mode < 2; ++lo_mode) {
        if (products == 1 && lo_mode == 1) continue;
        p.products = products;
        p.lo_mode = lo_mode;
        CK(cudaMemset(dy, 0, 128 * NC * 4));
        conv_tile<<<1, 128, smem>>>(p, dy);
        CK(cudaDeviceSynchronize());
        std::vector<float> hy(128 * NC);
        CK(cudaMemcpy(hy.data(), dy, hy.size() * 4, cudaMemcpyDeviceToHost));
        double worst = 0, worst_abs = 0;
        int bad = 0;
        for (int o = 0; o < 128 * NC; ++o) {
          double ref = 0, mag = 0;
          for (int j = 0; j < k; ++j) {
            ref += (double)hf[j] * hx[o + j];
            mag += fabs((double)hf[j] * hx[o + j]);
          }
          const double err = fabs(hy[o] - ref);
          worst = fmax(worst, err / mag);
          worst_abs = fmax(worst_abs, err);
          if (err > 1e-5 * mag + 1e-6) ++bad;
        }
        printf("  products %d lo_mode %d: max err/sum|xf| %.3g (abs %.3g), outside BJ bound: %d of %d\n",
               products, lo_mode, worst, worst_abs, bad, 128 * NC);
      }
  }
  // MMA issue rate
  unsigned long long* dc;
  CK(cudaMalloc(&dc, 148 * 8));
  const size_t smem2 = 1024 + 65536 + 16384 + 64;
  CK(cudaFuncSetAttribute(mma_rate<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
  CK(cudaFuncSetAttribute(mma_rate<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
  CK(cudaFuncSetAttribute(mma_rate<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
  for (int n : {32, 64, 128})
    for (int a_src = 0; a_src < 2; ++a_src)
    for (int nd : {1, 2}) {
      if (n * nd > 256) continue;
      const int iters = 2000;
      if (n == 32) mma_rate<32><<<148, 128, smem2>>>(iters, a_src, nd, dc);
      if (n == 64) mma_rate<64><<<148, 128, smem2>>>(iters, a_src, nd, dc);
      if (n == 128) mma_rate<128><<<148, 128, smem2>>>(iters, a_src, nd, dc);
      CK(cudaDeviceSynchronize());
      std::vector<unsigned long long> hc(148);
      CK(cudaMemcpy(hc.data(), dc, 148 * 8, cudaMemcpyDeviceToHost));
      unsigned long long mx = 0;
      for (auto c : hc) mx = mx > c ? mx : c;
      const double per = (double)mx / (iters * 24.0);
      printf("MMA M=128 N=%d K=8 tf32, A from %s, %d accumulators: %.1f clk/MMA -> %.0f MAC/clk/SM\n", n,
             a_src ? "smem" : "TMEM", nd, per, 128.0 * n * 8 / per);
    }
  return 0;
}
