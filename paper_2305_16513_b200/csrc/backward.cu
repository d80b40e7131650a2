// backward.cu -- backward passes of the sliding-window operators (SURVEY 8f
// NEXT #4: training, the abstract of PAPER.md l.7).  Each kernel evaluates the
// vector-Jacobian product of a forward definition (reading R16) as a
// GATHER over the windows that touch an input position, in increasing window
// order, so results are deterministic (no atomics):
//   sum   dx_t = sum_{i: is <= t < is+w} dy_i
//   conv  dx_t = sum_{i: 0 <= t-is < k} f_{t-is} dy_i
//         df_j = sum_b sum_i dy_i x_{is+j}        (two-pass reduction, fp64 partials)
//   max   dx_t = sum_{i: argmax_i = t} dy_i       (first maximum of each window)
//   2-D   avg / max analogues on [planes][H][W]
// Stride-1 sum and conv input gradients are the forward kernels on the
// zero-padded dy (api.cu); the kernels here serve strides > 1, max, the
// filter gradient and 2-D pooling.
#include <cstdint>
#include <type_traits>

#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kBwThreads = 256;

// first window containing position t: ceil((t - w + 1) / s), clamped at 0
__device__ __forceinline__ int64_t first_window(int64_t t, int64_t w, int64_t s) {
  const int64_t a = t - w + 1;
  return a <= 0 ? 0 : (a + s - 1) / s;
}

}  // namespace

// ---------------------------------------------------------------- strided sum / conv input
template <class T, bool kConv>
__global__ void __launch_bounds__(kBwThreads) transpose_window_kernel(const __grid_constant__ BackwardParams p) {
  const T* __restrict__ dy = static_cast<const T*>(p.dy);
  T* __restrict__ dx = static_cast<T*>(p.dx);
  const int64_t total = p.batch * p.N;
  for (int64_t e = blockIdx.x * (int64_t)kBwThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kBwThreads) {
    const int64_t b = e / p.N, t = e - b * p.N;
    const int64_t i0 = first_window(t, p.w, p.stride);
    int64_t i1 = t / p.stride;
    if (i1 > p.L - 1) i1 = p.L - 1;
    const T* __restrict__ g = dy + b * p.L;
    if constexpr (kConv) {
      float acc = 0.0f;
      for (int64_t i = i0; i <= i1; ++i) acc = __fmaf_rn(p.taps[t - i * p.stride], __ldg(g + i), acc);
      dx[e] = acc;
    } else {
      T acc = 0;
      for (int64_t i = i0; i <= i1; ++i) {
        if constexpr (std::is_same<T, int32_t>::value) acc = (T)((uint32_t)acc + (uint32_t)__ldg(g + i));  // wraps
        else acc = __fadd_rn(acc, __ldg(g + i));
      }
      dx[e] = acc;
    }
  }
}

// ---------------------------------------------------------------- max pooling
// CTA tile: kMaxTile input positions of one row.  The windows that can route a
// gradient into the tile form a contiguous range; they are processed in
// chunks of kMaxChunk: argmax (first maximum) of each window into shared
// memory, then every position gathers the dy of the chunk's windows whose
// argmax it is, in increasing window order.
constexpr int kMaxTile = 1024;
constexpr int kMaxChunk = 1024;

__global__ void __launch_bounds__(kBwThreads) pool_max_backward_kernel(const __grid_constant__ BackwardParams p) {
  __shared__ int64_t s_arg[kMaxChunk];
  __shared__ float s_g[kMaxChunk];
  const float* __restrict__ x = static_cast<const float*>(p.x);
  const float* __restrict__ dy = static_cast<const float*>(p.dy);
  float* __restrict__ dx = static_cast<float*>(p.dx);
  const int64_t tiles_per_row = (p.N + kMaxTile - 1) / kMaxTile;
  const int64_t ntiles = p.batch * tiles_per_row;
  constexpr int kPer = kMaxTile / kBwThreads;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b = tile / tiles_per_row;
    const int64_t t0 = (tile - b * tiles_per_row) * kMaxTile;
    const int64_t t1 = (t0 + kMaxTile < p.N ? t0 + kMaxTile : p.N) - 1;
    const float* __restrict__ xr = x + b * p.N;
    const float* __restrict__ gr = dy + b * p.L;
    const int64_t wlo = first_window(t0, p.w, p.stride);
    int64_t whi = t1 / p.stride;
    if (whi > p.L - 1) whi = p.L - 1;
    float acc[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) acc[q] = 0.0f;
    for (int64_t c0 = wlo; c0 <= whi; c0 += kMaxChunk) {
      const int64_t c1 = c0 + kMaxChunk - 1 < whi ? c0 + kMaxChunk - 1 : whi;
      __syncthreads();
      for (int64_t i = c0 + threadIdx.x; i <= c1; i += kBwThreads) {
        const float* xw = xr + i * p.stride;
        float m = __ldg(xw);
        int64_t a = 0;
        for (int64_t j = 1; j < p.w; ++j) {
          const float v = __ldg(xw + j);
          if (v > m) { m = v; a = j; }
        }
        s_arg[i - c0] = i * p.stride + a;
        s_g[i - c0] = __ldg(gr + i);
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int64_t t = t0 + threadIdx.x + q * kBwThreads;
        if (t > t1) continue;
        int64_t i0 = first_window(t, p.w, p.stride), i1 = t / p.stride;
        if (i0 < c0) i0 = c0;
        if (i1 > c1) i1 = c1;
        for (int64_t i = i0; i <= i1; ++i)
          if (s_arg[i - c0] == t) acc[q] = __fadd_rn(acc[q], s_g[i - c0]);
      }
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int64_t t = t0 + threadIdx.x + q * kBwThreads;
      if (t <= t1) dx[b * p.N + t] = acc[q];
    }
  }
}

// ---------------------------------------------------------------- conv filter gradient
// Pass 1: grid (ctas, tap blocks of 64).  Tile = kFgTile consecutive outputs i
// of one row; the CTA's 256 threads are 4 tap groups (16 taps) x 64 run slots
// (16 outputs).  Per tile a thread adds dy_i x_{is+j} over its 16 x 16 block
// in fp32 (stride 1: the 31 inputs it needs sit in registers), then folds the
// 16 partial sums into fp64 accumulators; at the end the 64 run slots of each
// tap group are reduced in fixed order and the CTA writes 64 fp64 partials.
// Pass 2 sums the CTA partials in fixed order.  Shared-memory x / dy are padded
// by 4 floats per 16 so the LDS.128 of 8 consecutive run slots hit distinct
// bank groups.
constexpr int kFgTaps = 64;
constexpr int kFgRun = 16;
constexpr int kFgSlots = 64;
constexpr int kFgTile = kFgRun * kFgSlots;  // 1024 outputs
__device__ __forceinline__ int fg_pad(int e) { return e + 4 * (e >> 4); }

template <bool kUnitStride>
__global__ void __launch_bounds__(kBwThreads) conv_filter_grad_kernel(const __grid_constant__ BackwardParams p,
                                                                      double* __restrict__ partials) {
  extern __shared__ __align__(16) float fg_smem[];
  const int xspan = kUnitStride ? kFgTile + kFgTaps : (int)((kFgTile - 1) * p.stride + kFgTaps);
  float* xs = fg_smem;                      // fg_pad(xspan) floats
  float* gs = fg_smem + ((fg_pad(xspan) + 16) & ~3);  // fg_pad(kFgTile) floats, 16-B aligned
  double* red = reinterpret_cast<double*>(fg_smem);  // reused for the final reduction
  const float* __restrict__ x = static_cast<const float*>(p.x);
  const float* __restrict__ dy = static_cast<const float*>(p.dy);
  const int64_t j0 = (int64_t)blockIdx.y * kFgTaps;
  const int q = threadIdx.x & 3, r = threadIdx.x >> 2;  // tap group, run slot
  const int64_t tiles_per_row = (p.L + kFgTile - 1) / kFgTile;
  const int64_t ntiles = p.batch * tiles_per_row;
  double acc64[16];
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) acc64[jj] = 0.0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b = tile / tiles_per_row;
    const int64_t i0 = (tile - b * tiles_per_row) * kFgTile;
    const int64_t nout = p.L - i0 < kFgTile ? p.L - i0 : kFgTile;
    const float* __restrict__ xr = x + b * p.N;
    const int64_t xbase = i0 * p.stride + j0;
    __syncthreads();
    for (int e = threadIdx.x; e < xspan; e += kBwThreads) {
      const int64_t t = xbase + e;
      xs[fg_pad(e)] = t < p.N ? __ldg(xr + t) : 0.0f;
    }
    for (int e = threadIdx.x; e < kFgTile; e += kBwThreads)
      gs[fg_pad(e)] = e < nout ? __ldg(dy + b * p.L + i0 + e) : 0.0f;
    __syncthreads();
    const int m0 = kFgRun * r;
    if (m0 >= nout) continue;
    float g[kFgRun];
#pragma unroll
    for (int m = 0; m < kFgRun; m += 4) {
      const float4 v = *reinterpret_cast<const float4*>(gs + fg_pad(m0 + m));
      g[m] = v.x; g[m + 1] = v.y; g[m + 2] = v.z; g[m + 3] = v.w;
    }
    float acc[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) acc[jj] = 0.0f;
    if constexpr (kUnitStride) {
      // x_{i+j} for i = i0+m0+m, j = j0+16q+jj: window xs[m0 + 16q + (m + jj)], 31 values
      float xw[32];
      const int base = m0 + 16 * q;
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 v = *reinterpret_cast<const float4*>(xs + fg_pad(base + c));
        xw[c] = v.x; xw[c + 1] = v.y; xw[c + 2] = v.z; xw[c + 3] = v.w;
      }
#pragma unroll
      for (int m = 0; m < kFgRun; ++m)
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) acc[jj] = __fmaf_rn(g[m], xw[m + jj], acc[jj]);
    } else {
#pragma unroll
      for (int m = 0; m < kFgRun; ++m) {
        const int base = (int)((m0 + m) * p.stride) + 16 * q;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) acc[jj] = __fmaf_rn(g[m], xs[fg_pad(base + jj)], acc[jj]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) acc64[jj] += (double)acc[jj];
  }
  // reduce the 64 run slots of each tap group, fixed order
  __syncthreads();
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) red[(16 * q + jj) * kFgSlots + r] = acc64[jj];
  __syncthreads();
  if (threadIdx.x < kFgTaps) {
    double s = 0.0;
    for (int rr = 0; rr < kFgSlots; ++rr) s += red[threadIdx.x * kFgSlots + rr];
    partials[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kFgTaps + threadIdx.x] = s;
  }
}

__global__ void conv_filter_grad_finish(const double* __restrict__ partials, int ctas, int64_t k,
                                        float* __restrict__ df) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= k) return;
  const int64_t blk = j / kFgTaps, jj = j - blk * kFgTaps;
  double s = 0.0;
  for (int c = 0; c < ctas; ++c) s += partials[(blk * ctas + c) * kFgTaps + jj];
  df[j] = (float)s;
}

size_t conv_filter_grad_workspace(int64_t k, int ctas) {
  return (size_t)((k + kFgTaps - 1) / kFgTaps) * ctas * kFgTaps * sizeof(double);
}

cudaError_t launch_conv_filter_grad(const BackwardParams& p, float* df, void* workspace, int ctas,
                                    cudaStream_t stream) {
  const int tap_blocks = (int)((p.w + kFgTaps - 1) / kFgTaps);
  const int xspan = p.stride == 1 ? kFgTile + kFgTaps : (int)((kFgTile - 1) * p.stride + kFgTaps);
  size_t smem = (size_t)(((xspan + 4 * (xspan >> 4) + 16) & ~3) + kFgTile + 4 * (kFgTile >> 4)) * sizeof(float);
  const size_t red = (size_t)kFgTaps * kFgSlots * sizeof(double);
  if (smem < red) smem = red;
  if (smem > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  double* part = static_cast<double*>(workspace);
  const dim3 grid((unsigned)ctas, (unsigned)tap_blocks);
  if (p.stride == 1) {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(conv_filter_grad_kernel<true>));
    if (e != cudaSuccess) return e;
    conv_filter_grad_kernel<true><<<grid, kBwThreads, smem, stream>>>(p, part);
  } else {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(conv_filter_grad_kernel<false>));
    if (e != cudaSuccess) return e;
    conv_filter_grad_kernel<false><<<grid, kBwThreads, smem, stream>>>(p, part);
  }
  note_launch();
  conv_filter_grad_finish<<<(unsigned)((p.w + 127) / 128), 128, 0, stream>>>(part, ctas, p.w, df);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- 2-D pooling
// Gather per input position over the windows containing it (row-major window
// order); max recomputes each candidate window's first maximum (row-major).
template <bool kAvg>
__global__ void __launch_bounds__(kBwThreads) pool2d_backward_kernel(const __grid_constant__ Pool2DBackwardParams p) {
  const int64_t total = p.planes * p.H * p.W;
  for (int64_t e = blockIdx.x * (int64_t)kBwThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kBwThreads) {
    const int64_t c = e % p.W, rest = e / p.W, h = rest % p.H, pl = rest / p.H;
    const int64_t r0 = first_window(h, p.kh, p.sh), c0 = first_window(c, p.kw, p.sw);
    int64_t r1 = h / p.sh, c1 = c / p.sw;
    if (r1 > p.OH - 1) r1 = p.OH - 1;
    if (c1 > p.OW - 1) c1 = p.OW - 1;
    const float* __restrict__ g = p.dy + pl * p.OH * p.OW;
    float acc = 0.0f;
    for (int64_t r = r0; r <= r1; ++r)
      for (int64_t cc = c0; cc <= c1; ++cc) {
        const float gv = __ldg(g + r * p.OW + cc);
        if constexpr (kAvg) {
          acc = __fadd_rn(acc, gv);
        } else {
          const float* xw = p.x + (pl * p.H + r * p.sh) * p.W + cc * p.sw;
          float m = __ldg(xw);
          int64_t am = 0, an = 0;
          for (int64_t a = 0; a < p.kh; ++a)
            for (int64_t bb = 0; bb < p.kw; ++bb) {
              const float v = __ldg(xw + a * p.W + bb);
              if (v > m) { m = v; am = a; an = bb; }
            }
          if (r * p.sh + am == h && cc * p.sw + an == c) acc = __fadd_rn(acc, gv);
        }
      }
    p.dx[e] = kAvg ? __fmul_rn(acc, p.inv_area) : acc;
  }
}

// ---------------------------------------------------------------- launches
static unsigned grid_elems(int64_t total, int sms) {
  int64_t g = (total + kBwThreads - 1) / kBwThreads;
  const int64_t cap = (int64_t)sms * 16;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

cudaError_t launch_transpose_window(const BackwardParams& p, int op, int dtype, cudaStream_t stream, int sms) {
  const unsigned g = grid_elems(p.batch * p.N, sms);
  if (op == kOpConv) transpose_window_kernel<float, true><<<g, kBwThreads, 0, stream>>>(p);
  else if (dtype == 1) transpose_window_kernel<int32_t, false><<<g, kBwThreads, 0, stream>>>(p);
  else transpose_window_kernel<float, false><<<g, kBwThreads, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pool_max_backward(const BackwardParams& p, cudaStream_t stream, int sms) {
  const int64_t tiles = p.batch * ((p.N + kMaxTile - 1) / kMaxTile);
  const int64_t cap = (int64_t)sms * 8;
  const unsigned g = (unsigned)(tiles < cap ? tiles : cap);
  pool_max_backward_kernel<<<g < 1 ? 1 : g, kBwThreads, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pool2d_backward(const Pool2DBackwardParams& p, cudaStream_t stream, int sms) {
  const unsigned g = grid_elems(p.planes * p.H * p.W, sms);
  if (p.mode == 1) pool2d_backward_kernel<true><<<g, kBwThreads, 0, stream>>>(p);
  else pool2d_backward_kernel<false><<<g, kBwThreads, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ss
