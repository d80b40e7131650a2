// Probe: TMA tiled 3-D loads with a box larger than the tensor and negative start
// coordinates (zero fill), SWIZZLE_NONE.  Prints which start coordinates work.
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, float* out, int n) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n * 4));
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"(&m), "r"(c0), "r"(c1), "r"(c2), "r"(b) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  const int W = 148, H = 35, PL = 3, BW = argc > 1 ? atoi(argv[1]) : 164, BH = argc > 2 ? atoi(argv[2]) : 39;
  float* x; float* o;
  cudaMalloc(&x, W * H * PL * 4); cudaMalloc(&o, BW * BH * 4);
  float* hx = new float[W * H * PL];
  for (int i = 0; i < W * H * PL; ++i) hx[i] = 1.0f + i;
  cudaMemcpy(x, hx, W * H * PL * 4, cudaMemcpyHostToDevice);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[3] = {W, H, PL}; cuuint64_t st[2] = {W * 4, W * H * 4};
  cuuint32_t box[3] = {(cuuint32_t)BW, (cuuint32_t)BH, 1}; cuuint32_t es[3] = {1, 1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, st, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d (box %d x %d)\n", (int)r, BW, BH);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int starts[4][2] = {{0, 0}, {0, -2}, {-4, -2}, {-8, -6}};
  float* ho = new float[BW * BH];
  for (auto& s : starts) {
    k<<<1, 128, BW * BH * 4>>>(m, s[0], s[1], 1, o, BW * BH);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("start (%d,%d): %s\n", s[0], s[1], cudaGetErrorString(e)); return 1; }
    cudaMemcpy(ho, o, BW * BH * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < BH; ++rr) for (int cc = 0; cc < BW; ++cc) {
      int gr = rr + s[1], gc = cc + s[0];
      float want = (gr >= 0 && gr < H && gc >= 0 && gc < W) ? hx[(1 * H + gr) * W + gc] : 0.0f;
      bad += ho[rr * BW + cc] != want;
    }
    printf("start (%d,%d): %d mismatches\n", s[0], s[1], bad);
  }
  return 0;
}
