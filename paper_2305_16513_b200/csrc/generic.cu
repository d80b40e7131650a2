// generic.cu -- direct-window kernels for the cases the TMA tile kernel does
// not take (stride > 1, tiny or misaligned inputs, very long windows, k > 64).
// Window loops over the read-only path, 4 outputs per thread (Eq. 3 as
// written; conv as Sec. 2.5, l.86-87).  Conv uses the tile
// kernel's association (even-tap and odd-tap FMA chains, then one add), so
// both produce bitwise-identical outputs.
#include <cstdint>
#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

// Grid: blockIdx.y walks batch rows, blockIdx.x chunks of kGenChunk outputs
// of a row; each thread evaluates kGenOuts outputs (ILP), consecutive threads
// consecutive outputs (coalesced stores, L1-shared window loads).
constexpr int kGenThreads = 256;
constexpr int kGenOuts = 4;
constexpr int kGenChunk = kGenThreads * kGenOuts;

template <class Op>
__global__ void __launch_bounds__(kGenThreads) pool_generic_kernel(const __grid_constant__ GenericParams p) {
  using T = typename Op::T;
  const int w = (int)p.w;
  for (int64_t b = blockIdx.y; b < p.batch; b += gridDim.y) {
    const T* __restrict__ xr = static_cast<const T*>(p.x) + b * p.N;
    T* __restrict__ yr = static_cast<T*>(p.y) + b * p.L;
    for (int64_t i0 = (int64_t)blockIdx.x * kGenChunk; i0 < p.L; i0 += (int64_t)gridDim.x * kGenChunk) {
      T acc[kGenOuts];
      const T* xs[kGenOuts];
#pragma unroll
      for (int k = 0; k < kGenOuts; ++k) {
        const int64_t i = i0 + threadIdx.x + k * kGenThreads;
        xs[k] = xr + (i < p.L ? i : p.L - 1) * p.stride;
        acc[k] = __ldg(xs[k]);
      }
      for (int j = 1; j < w; ++j) {
#pragma unroll
        for (int k = 0; k < kGenOuts; ++k) acc[k] = Op::combine(acc[k], __ldg(xs[k] + j));
      }
#pragma unroll
      for (int k = 0; k < kGenOuts; ++k) {
        const int64_t i = i0 + threadIdx.x + k * kGenThreads;
        if (i < p.L) yr[i] = acc[k];
      }
    }
  }
}

// Window spec with dilation and zero padding (NEXT #1): tap j of output i
// reads x[i*s + j*d - pl] when in range; padding adds nothing to a sum and
// never wins a max (identity).  Full mode: kGenOuts outputs per thread with
// an unchecked loop when all of their windows lie inside the row.  Skip mode
// (skip_lo < skip_hi): only outputs outside [skip_lo, skip_hi) -- the edges
// around an interior the tile kernel computed -- one per thread.
// Window taps are loaded in unrolled groups of 8 before they are combined, so a
// thread has 8 loads in flight instead of one (the edge launches are latency
// bound: ~12 us per launch with a serial load -> combine chain); the combine
// order (increasing j, skipped taps contribute nothing) is unchanged.
constexpr int kTapGroup = 8;

// x index of padded position u (u = i*s + j*d - pad_left, possibly outside [0, N)), or -1
// for zero padding (ss.h ss_pad_mode_t; the API bounds the pads so one reflection / one
// period suffices)
__device__ __forceinline__ int64_t pad_source(int64_t u, int64_t N, int mode) {
  if (u >= 0 && u < N) return u;
  if (mode == kPadReflect) return u < 0 ? -u : 2 * (N - 1) - u;
  if (mode == kPadCircular) return u < 0 ? u + N : u - N;
  if (mode == kPadReplicate) return u < 0 ? 0 : N - 1;
  return -1;
}

template <class Op>
__device__ __forceinline__ typename Op::T window_checked(const typename Op::T* __restrict__ xr,
                                                         int64_t t0, const GenericParams& p) {
  typename Op::T acc = Op::identity();
  for (int j0 = 0; j0 < (int)p.w; j0 += kTapGroup) {
    typename Op::T v[kTapGroup];
    bool ok[kTapGroup];
#pragma unroll
    for (int u = 0; u < kTapGroup; ++u) {
      const int64_t t = pad_source(t0 + (int64_t)(j0 + u) * p.dilation, p.N, p.pad_mode);
      ok[u] = j0 + u < (int)p.w && t >= 0;
      v[u] = ok[u] ? __ldg(xr + t) : Op::identity();
    }
#pragma unroll
    for (int u = 0; u < kTapGroup; ++u)
      if (ok[u]) acc = Op::combine(acc, v[u]);
  }
  return acc;
}

template <class Op>
__global__ void __launch_bounds__(kGenThreads) pool_generic_ex_kernel(const __grid_constant__ GenericParams p) {
  using T = typename Op::T;
  const int w = (int)p.w;
  const int64_t ext = (int64_t)(w - 1) * p.dilation;
  if (p.skip_lo < p.skip_hi) {
    const int64_t n_lo = p.skip_lo, n_work = n_lo + (p.L - p.skip_hi);
    for (int64_t b = blockIdx.y; b < p.batch; b += gridDim.y) {
      const T* __restrict__ xr = static_cast<const T*>(p.x) + b * p.N;
      T* __restrict__ yr = static_cast<T*>(p.y) + b * p.L;
      for (int64_t q = (int64_t)blockIdx.x * kGenThreads + threadIdx.x; q < n_work;
           q += (int64_t)gridDim.x * kGenThreads) {
        const int64_t i = q < n_lo ? q : p.skip_hi + (q - n_lo);
        yr[i] = window_checked<Op>(xr, i * p.stride - p.pad_left, p);
      }
    }
    return;
  }
  for (int64_t b = blockIdx.y; b < p.batch; b += gridDim.y) {
    const T* __restrict__ xr = static_cast<const T*>(p.x) + b * p.N;
    T* __restrict__ yr = static_cast<T*>(p.y) + b * p.L;
    for (int64_t i0 = (int64_t)blockIdx.x * kGenChunk; i0 < p.L; i0 += (int64_t)gridDim.x * kGenChunk) {
      const int64_t ia = i0 + threadIdx.x, ib = ia + (kGenOuts - 1) * kGenThreads;
      const int64_t ta = ia * p.stride - p.pad_left, tb = ib * p.stride - p.pad_left;
      if (ta >= 0 && tb + ext < p.N && ib < p.L) {  // every window of this thread is inside
        T acc[kGenOuts];
#pragma unroll
        for (int k = 0; k < kGenOuts; ++k) acc[k] = __ldg(xr + ta + (int64_t)k * kGenThreads * p.stride);
        for (int j = 1; j < w; ++j) {
#pragma unroll
          for (int k = 0; k < kGenOuts; ++k)
            acc[k] = Op::combine(acc[k], __ldg(xr + ta + (int64_t)k * kGenThreads * p.stride + (int64_t)j * p.dilation));
        }
#pragma unroll
        for (int k = 0; k < kGenOuts; ++k) yr[ia + k * kGenThreads] = acc[k];
      } else {
#pragma unroll
        for (int k = 0; k < kGenOuts; ++k) {
          const int64_t i = ia + k * kGenThreads;
          if (i < p.L) yr[i] = window_checked<Op>(xr, i * p.stride - p.pad_left, p);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kGenThreads) conv_generic_kernel(const __grid_constant__ GenericParams p) {
  const int k = (int)p.w;
  for (int64_t b = blockIdx.y; b < p.batch; b += gridDim.y) {
    const float* __restrict__ xr = static_cast<const float*>(p.x) + b * p.N;
    float* __restrict__ yr = static_cast<float*>(p.y) + b * p.L;
    for (int64_t i0 = (int64_t)blockIdx.x * kGenChunk; i0 < p.L; i0 += (int64_t)gridDim.x * kGenChunk) {
      // even-tap and odd-tap partial sums, each in increasing j, then added:
      // the association of the tile kernel (slide1d.cu ConvKind)
      float s0[kGenOuts], s1[kGenOuts];
      const float* xs[kGenOuts];
#pragma unroll
      for (int q = 0; q < kGenOuts; ++q) {
        const int64_t i = i0 + threadIdx.x + q * kGenThreads;
        xs[q] = xr + (i < p.L ? i : p.L - 1) * p.stride;
        s0[q] = 0.0f;
        s1[q] = 0.0f;
      }
      for (int j = 0; j < k; j += 2) {
        const float f = p.taps[j];
#pragma unroll
        for (int q = 0; q < kGenOuts; ++q) s0[q] = __fmaf_rn(f, __ldg(xs[q] + j), s0[q]);
      }
      for (int j = 1; j < k; j += 2) {
        const float f = p.taps[j];
#pragma unroll
        for (int q = 0; q < kGenOuts; ++q) s1[q] = __fmaf_rn(f, __ldg(xs[q] + j), s1[q]);
      }
#pragma unroll
      for (int q = 0; q < kGenOuts; ++q) {
        const int64_t i = i0 + threadIdx.x + q * kGenThreads;
        if (i < p.L) yr[i] = __fadd_rn(s0[q], s1[q]);
      }
    }
  }
}

__device__ __forceinline__ float conv_checked(const float* __restrict__ xr, int64_t t0,
                                              const GenericParams& p) {
  float s0 = 0.0f, s1 = 0.0f;  // same association as conv_generic_kernel / ConvKind
  for (int j0 = 0; j0 < (int)p.w; j0 += kTapGroup) {
    float v[kTapGroup];
    bool ok[kTapGroup];
#pragma unroll
    for (int u = 0; u < kTapGroup; ++u) {
      const int64_t t = pad_source(t0 + (int64_t)(j0 + u) * p.dilation, p.N, p.pad_mode);
      ok[u] = j0 + u < (int)p.w && t >= 0;
      v[u] = ok[u] ? __ldg(xr + t) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kTapGroup; u += 2)  // even taps (j0 is even)
      if (ok[u]) s0 = __fmaf_rn(p.taps[j0 + u], v[u], s0);
#pragma unroll
    for (int u = 1; u < kTapGroup; u += 2)
      if (ok[u]) s1 = __fmaf_rn(p.taps[j0 + u], v[u], s1);
  }
  return __fadd_rn(s0, s1);
}

__global__ void __launch_bounds__(kGenThreads) conv_generic_ex_kernel(const __grid_constant__ GenericParams p) {
  const int k = (int)p.w;
  const int64_t ext = (int64_t)(k - 1) * p.dilation;
  if (p.skip_lo < p.skip_hi) {
    const int64_t n_lo = p.skip_lo, n_work = n_lo + (p.L - p.skip_hi);
    for (int64_t b = blockIdx.y; b < p.batch; b += gridDim.y) {
      const float* __restrict__ xr = static_cast<const float*>(p.x) + b * p.N;
      float* __restrict__ yr = static_cast<float*>(p.y) + b * p.L;
      for (int64_t q = (int64_t)blockIdx.x * kGenThreads + threadIdx.x; q < n_work;
           q += (int64_t)gridDim.x * kGenThreads) {
        const int64_t i = q < n_lo ? q : p.skip_hi + (q - n_lo);
        yr[i] = conv_checked(xr, i * p.stride - p.pad_left, p);
      }
    }
    return;
  }
  for (int64_t b = blockIdx.y; b < p.batch; b += gridDim.y) {
    const float* __restrict__ xr = static_cast<const float*>(p.x) + b * p.N;
    float* __restrict__ yr = static_cast<float*>(p.y) + b * p.L;
    for (int64_t i0 = (int64_t)blockIdx.x * kGenChunk; i0 < p.L; i0 += (int64_t)gridDim.x * kGenChunk) {
      const int64_t ia = i0 + threadIdx.x, ib = ia + (kGenOuts - 1) * kGenThreads;
      const int64_t ta = ia * p.stride - p.pad_left, tb = ib * p.stride - p.pad_left;
      if (ta >= 0 && tb + ext < p.N && ib < p.L) {
        float s0[kGenOuts], s1[kGenOuts];
#pragma unroll
        for (int q = 0; q < kGenOuts; ++q) s0[q] = s1[q] = 0.0f;
        for (int j = 0; j < k; j += 2) {
          const float f = p.taps[j];
#pragma unroll
          for (int q = 0; q < kGenOuts; ++q)
            s0[q] = __fmaf_rn(f, __ldg(xr + ta + (int64_t)q * kGenThreads * p.stride + (int64_t)j * p.dilation), s0[q]);
        }
        for (int j = 1; j < k; j += 2) {
          const float f = p.taps[j];
#pragma unroll
          for (int q = 0; q < kGenOuts; ++q)
            s1[q] = __fmaf_rn(f, __ldg(xr + ta + (int64_t)q * kGenThreads * p.stride + (int64_t)j * p.dilation), s1[q]);
        }
#pragma unroll
        for (int q = 0; q < kGenOuts; ++q) yr[ia + q * kGenThreads] = __fadd_rn(s0[q], s1[q]);
      } else {
#pragma unroll
        for (int q = 0; q < kGenOuts; ++q) {
          const int64_t i = ia + q * kGenThreads;
          if (i < p.L) yr[i] = conv_checked(xr, i * p.stride - p.pad_left, p);
        }
      }
    }
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

static dim3 grid_1d(const GenericParams& p, int sms) {
  int64_t gy = p.batch < 65535 ? p.batch : 65535;
  int64_t gx = (p.L + kGenChunk - 1) / kGenChunk;
  const int64_t cap = (int64_t)sms * 16;  // enough resident blocks to cover latency
  if (gx * gy > cap) gx = cap / gy > 0 ? cap / gy : 1;
  return dim3((unsigned)(gx < 1 ? 1 : gx), (unsigned)gy, 1);
}

// skip mode (edges around a computed interior): one thread per edge output of a row
static dim3 edge_grid(const GenericParams& p) {
  const int64_t n_work = p.skip_lo + (p.L - p.skip_hi);
  const int64_t gx = (n_work + kGenThreads - 1) / kGenThreads;
  const int64_t gy = p.batch < 65535 ? p.batch : 65535;
  return dim3((unsigned)(gx < 1 ? 1 : (gx > 4096 ? 4096 : gx)), (unsigned)(gy < 1 ? 1 : gy), 1);
}

static bool is_ex(const GenericParams& p) {
  return p.dilation != 1 || p.pad_left != 0 || p.skip_lo < p.skip_hi ||
         (p.L - 1) * p.stride + p.w > p.N;  // right padding
}

cudaError_t launch_pool_generic(const GenericParams& p, int op, int dtype, cudaStream_t stream,
                                int grid) {
  const dim3 g = grid_1d(p, grid / 8 > 0 ? grid / 8 : 148);
  if (is_ex(p)) {
    const dim3 ge = p.skip_lo < p.skip_hi ? edge_grid(p) : g;
    if (op == kOpSum && dtype == 1) pool_generic_ex_kernel<OpSumI32><<<ge, kGenThreads, 0, stream>>>(p);
    else if (op == kOpSum && dtype == 0) pool_generic_ex_kernel<OpSumF32><<<ge, kGenThreads, 0, stream>>>(p);
    else if (op == kOpMax && dtype == 1) pool_generic_ex_kernel<OpMaxI32><<<ge, kGenThreads, 0, stream>>>(p);
    else if (op == kOpMax && dtype == 0) pool_generic_ex_kernel<OpMaxF32><<<ge, kGenThreads, 0, stream>>>(p);
    else if (op == kOpMin && dtype == 1) pool_generic_ex_kernel<OpMinI32><<<ge, kGenThreads, 0, stream>>>(p);
    else if (op == kOpMin && dtype == 0) pool_generic_ex_kernel<OpMinF32><<<ge, kGenThreads, 0, stream>>>(p);
    else return cudaErrorInvalidValue;
  } else {
    if (op == kOpSum && dtype == 1) pool_generic_kernel<OpSumI32><<<g, kGenThreads, 0, stream>>>(p);
    else if (op == kOpSum && dtype == 0) pool_generic_kernel<OpSumF32><<<g, kGenThreads, 0, stream>>>(p);
    else if (op == kOpMax && dtype == 1) pool_generic_kernel<OpMaxI32><<<g, kGenThreads, 0, stream>>>(p);
    else if (op == kOpMax && dtype == 0) pool_generic_kernel<OpMaxF32><<<g, kGenThreads, 0, stream>>>(p);
    else if (op == kOpMin && dtype == 1) pool_generic_kernel<OpMinI32><<<g, kGenThreads, 0, stream>>>(p);
    else if (op == kOpMin && dtype == 0) pool_generic_kernel<OpMinF32><<<g, kGenThreads, 0, stream>>>(p);
    else return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv_generic(const GenericParams& p, cudaStream_t stream, int grid) {
  const dim3 g = grid_1d(p, grid / 8 > 0 ? grid / 8 : 148);
  if (is_ex(p))
    conv_generic_ex_kernel<<<p.skip_lo < p.skip_hi ? edge_grid(p) : g, kGenThreads, 0, stream>>>(p);
  else conv_generic_kernel<<<g, kGenThreads, 0, stream>>>(p);
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
