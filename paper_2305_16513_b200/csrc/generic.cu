// generic.cu -- direct-window kernels for the cases the TMA tile kernel does
// not take (stride > 1, tiny or misaligned inputs, very long windows, k > 64).
// One output per thread, window loop over the read-only path (Eq. 3 as
// written; conv as Sec. 2.5, l.86-87).  Conv uses the tile
// kernel's association (even-tap and odd-tap FMA chains, then one add), so
// both produce bitwise-identical outputs.
#include <cstdint>
#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

template <class Op>
__global__ void __launch_bounds__(256) pool_generic_kernel(const __grid_constant__ GenericParams p) {
  using T = typename Op::T;
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ y = static_cast<T*>(p.y);
  const int64_t total = p.batch * p.L;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = o / p.L, i = o - b * p.L;
    const T* xr = x + b * p.N + i * p.stride;
    T acc = __ldg(xr);
    for (int64_t j = 1; j < p.w; ++j) acc = Op::combine(acc, __ldg(xr + j));
    y[o] = acc;
  }
}

__global__ void __launch_bounds__(256) conv_generic_kernel(const __grid_constant__ GenericParams p) {
  const float* __restrict__ x = static_cast<const float*>(p.x);
  float* __restrict__ y = static_cast<float*>(p.y);
  const int64_t total = p.batch * p.L;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = o / p.L, i = o - b * p.L;
    const float* xr = x + b * p.N + i * p.stride;
    // even-tap and odd-tap partial sums, each in increasing j, then added:
    // the association of the tile kernel (slide1d.cu ConvKind)
    float s0 = 0.0f, s1 = 0.0f;
    for (int64_t j = 0; j < p.w; j += 2) s0 = __fmaf_rn(p.taps[j], __ldg(xr + j), s0);
    for (int64_t j = 1; j < p.w; j += 2) s1 = __fmaf_rn(p.taps[j], __ldg(xr + j), s1);
    y[o] = __fadd_rn(s0, s1);
  }
}

// Direct 2-D window (used when a band of rows does not fit shared memory).
template <bool kAvg>
__global__ void __launch_bounds__(256) pool2d_direct_kernel(const __grid_constant__ Pool2DParams p) {
  const int64_t total = p.planes * p.OH * p.OW;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = o % p.OW, t = o / p.OW, r = t % p.OH, pl = t / p.OH;
    const float* xp = p.x + (pl * p.H + r * p.sh) * p.W + c * p.sw;
    float acc = kAvg ? 0.0f : __ldg(xp);
    for (int64_t dr = 0; dr < p.kh; ++dr)
      for (int64_t dc = 0; dc < p.kw; ++dc) {
        const float v = __ldg(xp + dr * p.W + dc);
        acc = kAvg ? __fadd_rn(acc, v) : (v > acc ? v : acc);
      }
    p.y[o] = kAvg ? __fmul_rn(acc, p.inv_area) : acc;
  }
}

static int64_t grid_for(int64_t total, int grid_cap) {
  int64_t g = (total + 255) / 256;
  if (g > grid_cap) g = grid_cap;
  return g < 1 ? 1 : g;
}

cudaError_t launch_pool_generic(const GenericParams& p, int op, int dtype, cudaStream_t stream,
                                int grid) {
  const int64_t g = grid_for(p.batch * p.L, grid);
  if (op == kOpSum && dtype == 1) pool_generic_kernel<OpSumI32><<<(unsigned)g, 256, 0, stream>>>(p);
  else if (op == kOpSum && dtype == 0) pool_generic_kernel<OpSumF32><<<(unsigned)g, 256, 0, stream>>>(p);
  else if (op == kOpMax && dtype == 1) pool_generic_kernel<OpMaxI32><<<(unsigned)g, 256, 0, stream>>>(p);
  else if (op == kOpMax && dtype == 0) pool_generic_kernel<OpMaxF32><<<(unsigned)g, 256, 0, stream>>>(p);
  else return cudaErrorInvalidValue;
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv_generic(const GenericParams& p, cudaStream_t stream, int grid) {
  const int64_t g = grid_for(p.batch * p.L, grid);
  conv_generic_kernel<<<(unsigned)g, 256, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pool2d_direct(const Pool2DParams& p, cudaStream_t stream, int grid) {
  const int64_t g = grid_for(p.planes * p.OH * p.OW, grid);
  if (p.mode == 1) pool2d_direct_kernel<true><<<(unsigned)g, 256, 0, stream>>>(p);
  else pool2d_direct_kernel<false><<<(unsigned)g, 256, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ss
