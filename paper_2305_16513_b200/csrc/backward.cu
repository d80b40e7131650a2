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
// Tile kernel (w <= kMaxTileW, stride <= kMaxTileS): kMaxTile positions of one
// row.  (1) Stage the x span of every window touching the tile.  (2) First
// maximum of every such window in O(1) from block-wise prefix / suffix
// argmax scans (blocks of w aligned at the span start; Alg. 2's prefix/suffix
// split, on (value, index) pairs: the earlier index wins ties, so
// suffix scans replace on >=, prefix scans on >).  (3) The window argmax a_i
// is non-decreasing in i (an element dropped from a window was not after its
// first maximum), so the windows routed to a position form one contiguous
// run: the thread of each run's first window sums its dy in increasing order
// into the staged dx tile (zero elsewhere), which is then stored coalesced.
constexpr int kMaxTile = 1024;
constexpr int kMaxTileW = 1024;
constexpr int kMaxTileS = 64;
constexpr int kMaxSpan = kMaxTile + 2 * kMaxTileW + kMaxTileS;  // x elements staged per tile (bound)
constexpr int kMaxWin = kMaxTile + kMaxTileW + 2;               // windows per tile (bound)
// shared arrays indexed by the padded position of span element e: block e / w
// at pitch w | 1 (odd), so the lanes of a warp scanning consecutive blocks hit
// distinct banks
constexpr int kMaxSpanPad = kMaxSpan + kMaxSpan / 2 + 2;
constexpr size_t kMaxTileSmem = (size_t)kMaxSpanPad * (4 + 4 + 4) + (size_t)kMaxWin * (4 + 4) + kMaxTile * 4;

__global__ void __launch_bounds__(kBwThreads) pool_max_backward_tile_kernel(const __grid_constant__ BackwardParams p) {
  extern __shared__ __align__(16) float mb_smem[];
  float* xs = mb_smem;                                        // [kMaxSpanPad], padded positions
  int* S = reinterpret_cast<int*>(xs + kMaxSpanPad);          // suffix argmax (span-relative, unpadded)
  int* P = S + kMaxSpanPad;                                   // prefix argmax
  int* A = P + kMaxSpan;                                      // window argmax [kMaxWin]
  float* gs = reinterpret_cast<float*>(A + kMaxWin);          // dy of the tile's windows
  float* dxs = gs + kMaxWin;                                  // dx tile [kMaxTile]
  const float* __restrict__ x = static_cast<const float*>(p.x);
  const float* __restrict__ dy = static_cast<const float*>(p.dy);
  float* __restrict__ dx = static_cast<float*>(p.dx);
  const int w = (int)p.w, s = (int)p.stride;
  const int pitch = w | 1;
  auto pad = [&](int e) { const int q = e / w; return q * pitch + (e - q * w); };
  const int64_t tiles_per_row = (p.N + kMaxTile - 1) / kMaxTile;
  const int64_t ntiles = p.batch * tiles_per_row;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b = tile / tiles_per_row;
    const int64_t t0 = (tile - b * tiles_per_row) * kMaxTile;
    const int nt = (int)(t0 + kMaxTile < p.N ? kMaxTile : p.N - t0);
    const int64_t wlo = first_window(t0, p.w, p.stride);
    int64_t whi = (t0 + nt - 1) / p.stride;
    if (whi > p.L - 1) whi = p.L - 1;
    const int nwin = whi >= wlo ? (int)(whi - wlo + 1) : 0;
    const int64_t xa = wlo * p.stride;
    const int span = nwin ? (int)((whi - wlo) * s + w) : 0;
    const float* __restrict__ xr = x + b * p.N;
    const float* __restrict__ gr = dy + b * p.L;
    __syncthreads();  // previous tile's readers are done
    for (int e = threadIdx.x; e < span; e += kBwThreads) xs[pad(e)] = __ldg(xr + xa + e);
    for (int e = threadIdx.x; e < nwin; e += kBwThreads) gs[e] = __ldg(gr + wlo + e);
    for (int e = threadIdx.x; e < nt; e += kBwThreads) dxs[e] = 0.0f;
    __syncthreads();
    // (2a) block-wise prefix / suffix argmax, one block of w per thread
    const int nb = (span + w - 1) / w;
    for (int blk = threadIdx.x; blk < nb; blk += kBwThreads) {
      const int lo = blk * w, n = min(lo + w, span) - lo, base = blk * pitch;
      int best = 0;
      float bv = xs[base];
      P[base] = lo;
      for (int u = 1; u < n; ++u) {
        const float v = xs[base + u];
        if (v > bv) { bv = v; best = u; }
        P[base + u] = lo + best;
      }
      best = n - 1;
      bv = xs[base + n - 1];
      S[base + n - 1] = lo + n - 1;
      for (int u = n - 2; u >= 0; --u) {
        const float v = xs[base + u];
        if (v >= bv) { bv = v; best = u; }
        S[base + u] = lo + best;
      }
    }
    __syncthreads();
    // (2b) first maximum of each window [u, u + w - 1], u = (i - wlo) s
    for (int j = threadIdx.x; j < nwin; j += kBwThreads) {
      const int u = j * s;
      int a = S[pad(u)];
      if (u % w) {
        const int a2 = P[pad(u + w - 1)];
        if (xs[pad(a2)] > xs[pad(a)]) a = a2;
      }
      A[j] = a;
    }
    __syncthreads();
    // (3) run sums, written by each run's first window
    for (int j = threadIdx.x; j < nwin; j += kBwThreads) {
      const int a = A[j];
      const int64_t t = xa + a;
      if (t < t0 || t >= t0 + nt || (j > 0 && A[j - 1] == a)) continue;
      float acc = 0.0f;
      for (int jj = j; jj < nwin && A[jj] == a; ++jj) acc = __fadd_rn(acc, gs[jj]);
      dxs[t - t0] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nt; e += kBwThreads) dx[b * p.N + t0 + e] = dxs[e];
  }
}

// Short windows (w <= kMaxDirectW): the same tile, SIMD-uniform work -- each
// window's first maximum by a direct scan of its w staged inputs, then every
// position gathers the <= ceil(w/s) windows that contain it (increasing
// window order), comparing their argmax with itself.
constexpr int kMaxDirectW = 64;

__global__ void __launch_bounds__(kBwThreads) pool_max_backward_direct_kernel(const __grid_constant__ BackwardParams p) {
  extern __shared__ __align__(16) float md_smem[];
  float* xs = md_smem;                                   // [kMaxTile + 2 kMaxDirectW + kMaxTileS]
  float* gs = xs + kMaxTile + 2 * kMaxDirectW + kMaxTileS;  // [kMaxTile + kMaxDirectW + 2]
  int* A = reinterpret_cast<int*>(gs + kMaxTile + kMaxDirectW + 2);
  const float* __restrict__ x = static_cast<const float*>(p.x);
  const float* __restrict__ dy = static_cast<const float*>(p.dy);
  float* __restrict__ dx = static_cast<float*>(p.dx);
  const int w = (int)p.w, s = (int)p.stride;
  const int64_t tiles_per_row = (p.N + kMaxTile - 1) / kMaxTile;
  const int64_t ntiles = p.batch * tiles_per_row;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t b = tile / tiles_per_row;
    const int64_t t0 = (tile - b * tiles_per_row) * kMaxTile;
    const int nt = (int)(t0 + kMaxTile < p.N ? kMaxTile : p.N - t0);
    const int64_t wlo = first_window(t0, p.w, p.stride);
    int64_t whi = (t0 + nt - 1) / p.stride;
    if (whi > p.L - 1) whi = p.L - 1;
    const int nwin = whi >= wlo ? (int)(whi - wlo + 1) : 0;
    const int64_t xa = wlo * p.stride;
    const int span = nwin ? (nwin - 1) * s + w : 0;
    const float* __restrict__ xr = x + b * p.N + xa;
    const float* __restrict__ gr = dy + b * p.L + wlo;
    __syncthreads();  // previous tile's readers are done
    for (int e = threadIdx.x; e < span; e += kBwThreads) xs[e] = __ldg(xr + e);
    for (int e = threadIdx.x; e < nwin; e += kBwThreads) gs[e] = __ldg(gr + e);
    __syncthreads();
    for (int j = threadIdx.x; j < nwin; j += kBwThreads) {
      const int u = j * s;
      float m = xs[u];
      int a = u;
      for (int q = 1; q < w; ++q) {
        const float v = xs[u + q];
        if (v > m) { m = v; a = u + q; }
      }
      A[j] = a;
    }
    __syncthreads();
    const int rel0 = (int)(t0 - xa);  // span-relative position of t0
    for (int e = threadIdx.x; e < nt; e += kBwThreads) {
      const int rel = rel0 + e;       // t = t0 + e
      const int64_t t = t0 + e;
      int64_t i0 = first_window(t, p.w, p.stride), i1 = t / p.stride;
      if (i1 > whi) i1 = whi;
      float acc = 0.0f;
      for (int j = (int)(i0 - wlo); j <= (int)(i1 - wlo); ++j)
        if (A[j] == rel) acc = __fadd_rn(acc, gs[j]);
      dx[b * p.N + t] = acc;
    }
  }
}

// Fallback for w > kMaxTileW: windows in chunks, argmax of each recomputed from
// global memory, then each position gathers the chunk's windows routed to it.
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
// Unit stride (the common case): grid (ctas, tap blocks of 64).  Tile =
// kFgTile consecutive outputs i of one row; the CTA's 256 threads are 4 tap
// groups (16 taps) x 64 run slots (16 outputs).  Per tile a thread adds
// dy_i x_{i+j} over its 16 x 16 block in fp32 with the 31 inputs it needs in
// registers, then folds the 16 partial sums into fp64 accumulators; at the end
// the 64 run slots of each tap group are reduced in fixed order and the CTA
// writes 64 fp64 partials.  Tiles stream through a kFgStages-deep ring of
// shared-memory stages filled with 4-B cp.async (rows have any alignment),
// padded by 4 floats per 16 so the LDS.128 of 8 consecutive run slots hit
// distinct bank groups.
// Strided: grid (ctas, k); each CTA sums dy_i x_{is+j} for one tap over a
// grid-strided share of the outputs (fp32 runs of 16, then fp64).
// Finish: sums the CTA partials of each tap in fixed order.
constexpr int kFgTaps = 64;
constexpr int kFgRun = 16;
constexpr int kFgSlots = 64;
constexpr int kFgTile = kFgRun * kFgSlots;  // 1024 outputs
constexpr int kFgStages = 4;
constexpr int kFgFold = 4;  // tiles accumulated in fp32 (64 terms per partial) before folding into fp64
constexpr int kFgXSpan = kFgTile + kFgTaps;  // inputs one tile needs (unit stride)
__host__ __device__ constexpr int fg_pad(int e) { return e + 4 * (e >> 4); }
// stages hold x / dy from the 16-B-aligned-down address of the tile's first
// element on (up to 3 leading elements), in the padded layout
constexpr int kFgXStride = (fg_pad(kFgXSpan + 4) + 16) & ~3;      // padded x floats per stage
constexpr int kFgStageFloats = kFgXStride + fg_pad(kFgTile + 8) + 8;
constexpr size_t kFgSmem = (size_t)kFgStages * kFgStageFloats * sizeof(float);

// (row, tile-in-row) of a grid-strided tile sequence, advanced without divisions
struct TileCursor {
  int64_t b, tr, tpr, step;
  __device__ void init(int64_t tile, int64_t tiles_per_row, int64_t stride) {
    tpr = tiles_per_row;
    step = stride;
    b = tile / tpr;
    tr = tile - b * tpr;
  }
  __device__ void advance() {
    tr += step;
    while (tr >= tpr) { tr -= tpr; ++b; }
  }
};

// stage `n` elements from src (any alignment) at padded local indices mis .. mis+n-1,
// mis = src's element offset in its 16-B granule; elements of the leading granule
// before src are filled too (never read) when they lie inside [lo_ok, src)
__device__ __forceinline__ void fg_stage(float* sdst, const float* __restrict__ src, int n, int64_t avail,
                                         bool aligned_ok, int mis) {
  if (aligned_ok) {
    const float* base = src - mis;
    const int lim = (int)(avail < n ? avail : n) + mis;  // valid elements from base (32-bit)
    for (int e = 4 * threadIdx.x; e < n + mis; e += 4 * kBwThreads) {
      const int left = lim - e;
      const uint32_t nb = left >= 4 ? 16u : (left > 0 ? 4u * (uint32_t)left : 0u);
      cp_async16(smem_u32(sdst + fg_pad(e)), nb ? base + e : src, nb);
    }
  } else {
    for (int e = threadIdx.x; e < n; e += kBwThreads)
      cp_async4(smem_u32(sdst + fg_pad(e + mis)), e < avail ? src + e : src, e < avail ? 4u : 0u);
  }
}

// Unit-stride filter gradient.  Inner product per thread and tile: 16 outputs
// m x 16 taps jj, acc[jj] += dy_m x_{m+jj}, as FFMA2 over tap pairs
// (acc[jj], acc[jj+1]) += dy_m * (x_{m+jj}, x_{m+jj+1}); the input window is
// kept twice (pairs starting at even and at odd offsets) so every pair is an
// aligned register pair.  x and dy stream with 16-B cp.async from their
// aligned-down addresses; the tile-uniform misalignment of x selects one of
// four compile-time realignments (MX), dy is read with 32-bit loads.
template <int MX, int MG>
__device__ __forceinline__ void fg_tile(const float* xs, const float* gs, int base, int m0, float2 (&acc)[8]) {
  // x window [base, base + 32) sits at local indices base + MX + (0..31): 9 aligned float4;
  // dy run [m0, m0 + 16) at local m0 + MG + (0..15): 5 aligned float4
  float w[36], gv[20];
#pragma unroll
  for (int c = 0; c < 36; c += 4) {
    const float4 v = *reinterpret_cast<const float4*>(xs + fg_pad(base + c));
    w[c] = v.x; w[c + 1] = v.y; w[c + 2] = v.z; w[c + 3] = v.w;
  }
#pragma unroll
  for (int c = 0; c < 20; c += 4) {
    const float4 v = *reinterpret_cast<const float4*>(gs + fg_pad(m0 + c));
    gv[c] = v.x; gv[c + 1] = v.y; gv[c + 2] = v.z; gv[c + 3] = v.w;
  }
  float2 E[16], O[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) E[i] = make_float2(w[MX + 2 * i], w[MX + 2 * i + 1]);
#pragma unroll
  for (int i = 0; i < 16; ++i) O[i] = make_float2(w[MX + 2 * i + 1], w[MX + 2 * i + 2]);
#pragma unroll
  for (int mt = 0; mt < kFgRun; ++mt) {
    const float2 g2 = make_float2(gv[MG + mt], gv[MG + mt]);
#pragma unroll
    for (int i = 0; i < 8; ++i)  // taps 2i, 2i+1: inputs x_{mt+2i}, x_{mt+2i+1}
      acc[i] = __ffma2_rn((mt & 1) ? O[(mt >> 1) + i] : E[(mt >> 1) + i], g2, acc[i]);
  }
}

template <int MX>
__device__ __forceinline__ void fg_tile_g(const float* xs, const float* gs, int misg, int base, int m0,
                                          float2 (&acc)[8]) {
  switch (misg) {  // tile-uniform
    case 0: fg_tile<MX, 0>(xs, gs, base, m0, acc); break;
    case 1: fg_tile<MX, 1>(xs, gs, base, m0, acc); break;
    case 2: fg_tile<MX, 2>(xs, gs, base, m0, acc); break;
    default: fg_tile<MX, 3>(xs, gs, base, m0, acc); break;
  }
}

__global__ void __launch_bounds__(kBwThreads, 2) conv_filter_grad_kernel(const __grid_constant__ BackwardParams p,
                                                                         double* __restrict__ partials) {
  extern __shared__ __align__(16) float fg_smem[];
  double* red = reinterpret_cast<double*>(fg_smem);  // reused for the final reduction
  const float* __restrict__ x = static_cast<const float*>(p.x);
  const float* __restrict__ dy = static_cast<const float*>(p.dy);
  const int64_t j0 = (int64_t)blockIdx.y * kFgTaps;
  const int q = threadIdx.x & 3, r = threadIdx.x >> 2;  // tap group, run slot
  const int64_t tiles_per_row = (p.L + kFgTile - 1) / kFgTile;
  const int64_t ntiles = p.batch * tiles_per_row;
  TileCursor ic, cc;  // issue cursor (kFgStages-1 tiles ahead) and compute cursor
  ic.init(blockIdx.x, tiles_per_row, gridDim.x);
  cc = ic;
  int64_t itile = blockIdx.x;
  auto issue = [&](int st) {
    if (itile < ntiles) {
      float* xs = fg_smem + st * kFgStageFloats;
      float* gs = xs + kFgXStride;
      const int64_t i0 = ic.tr * kFgTile;
      const int64_t nout = p.L - i0 < kFgTile ? p.L - i0 : kFgTile;
      const int64_t xg = ic.b * p.N + i0 + j0, gg = ic.b * p.L + i0;  // element offsets from x / dy
      const int misx = (int)((reinterpret_cast<uintptr_t>(x + xg) >> 2) & 3);
      const int misg = (int)((reinterpret_cast<uintptr_t>(dy + gg) >> 2) & 3);
      fg_stage(xs, x + xg, kFgXSpan, p.N - i0 - j0, xg >= misx, misx);
      fg_stage(gs, dy + gg, kFgTile, nout, gg >= misg, misg);
      ic.advance();
      itile += gridDim.x;
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int st = 0; st < kFgStages - 1; ++st) issue(st);
  double acc64[16];
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) acc64[jj] = 0.0;
  float2 acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.0f, 0.0f);
  int st = 0, nfold = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    issue((st + kFgStages - 1) % kFgStages);
    cp_async_wait<kFgStages - 1>();  // this tile's group has landed (for this thread)
    __syncthreads();                 // ... and for every thread
    const float* xs = fg_smem + st * kFgStageFloats;
    const float* gs = xs + kFgXStride;
    const int64_t i0 = cc.tr * kFgTile;
    const int misx = (int)((reinterpret_cast<uintptr_t>(x + cc.b * p.N + i0 + j0) >> 2) & 3);
    const int misg = (int)((reinterpret_cast<uintptr_t>(dy + cc.b * p.L + i0) >> 2) & 3);
    cc.advance();
    const int m0 = kFgRun * r;
    const int base = m0 + 16 * q;
    switch (misx) {  // tile-uniform
      case 0: fg_tile_g<0>(xs, gs, misg, base, m0, acc); break;
      case 1: fg_tile_g<1>(xs, gs, misg, base, m0, acc); break;
      case 2: fg_tile_g<2>(xs, gs, misg, base, m0, acc); break;
      default: fg_tile_g<3>(xs, gs, misg, base, m0, acc); break;
    }
    if (++nfold == kFgFold) {
      nfold = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc64[2 * i] += (double)acc[i].x;
        acc64[2 * i + 1] += (double)acc[i].y;
        acc[i] = make_float2(0.0f, 0.0f);
      }
    }
    __syncthreads();  // stage st is refilled by the next iteration's issue
    st = st + 1 == kFgStages ? 0 : st + 1;
  }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc64[2 * i] += (double)acc[i].x;
    acc64[2 * i + 1] += (double)acc[i].y;
  }
  // reduce the 64 run slots of each tap group, fixed order
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) red[(16 * q + jj) * kFgSlots + r] = acc64[jj];
  __syncthreads();
  if (threadIdx.x < kFgTaps) {
    double s = 0.0;
    for (int rr = 0; rr < kFgSlots; ++rr) s += red[threadIdx.x * kFgSlots + rr];
    partials[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kFgTaps + threadIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kBwThreads) conv_filter_grad_strided_kernel(const __grid_constant__ BackwardParams p,
                                                                              double* __restrict__ partials) {
  __shared__ double red[kBwThreads];
  const float* __restrict__ x = static_cast<const float*>(p.x);
  const float* __restrict__ dy = static_cast<const float*>(p.dy);
  const int64_t j = blockIdx.y;
  const int64_t total = p.batch * p.L;
  const int64_t step = (int64_t)gridDim.x * kBwThreads;
  double acc64 = 0.0;
  int64_t e = blockIdx.x * (int64_t)kBwThreads + threadIdx.x;
  while (e < total) {
    float acc = 0.0f;
    for (int n = 0; n < 16 && e < total; ++n, e += step) {
      const int64_t b = e / p.L, i = e - b * p.L;
      acc = __fmaf_rn(__ldg(dy + e), __ldg(x + b * p.N + i * p.stride + j), acc);
    }
    acc64 += (double)acc;
  }
  red[threadIdx.x] = acc64;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < kBwThreads; ++t) s += red[t];
    partials[j * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void conv_filter_grad_finish(const double* __restrict__ partials, int ctas, int64_t k, int strided,
                                        float* __restrict__ df) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= k) return;
  const int64_t blk = j / kFgTaps, jj = j - blk * kFgTaps;
  double s = 0.0;
  for (int c = 0; c < ctas; ++c)
    s += strided ? partials[j * ctas + c] : partials[(blk * ctas + c) * kFgTaps + jj];
  df[j] = (float)s;
}

int conv_filter_grad_ctas(int sms) { return 2 * sms; }

size_t conv_filter_grad_workspace(int64_t k, int ctas) {
  return (size_t)((k + kFgTaps - 1) / kFgTaps) * ctas * kFgTaps * sizeof(double);
}

cudaError_t launch_conv_filter_grad(const BackwardParams& p, float* df, void* workspace, int ctas,
                                    cudaStream_t stream) {
  double* part = static_cast<double*>(workspace);
  const bool strided = p.stride != 1;
  if (!strided) {
    static_assert(kFgSmem >= (size_t)kFgTaps * kFgSlots * sizeof(double), "reduction fits the stages");
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(conv_filter_grad_kernel));
    if (e != cudaSuccess) return e;
    const int tap_blocks = (int)((p.w + kFgTaps - 1) / kFgTaps);
    conv_filter_grad_kernel<<<dim3((unsigned)ctas, (unsigned)tap_blocks), kBwThreads, kFgSmem, stream>>>(p, part);
  } else {
    conv_filter_grad_strided_kernel<<<dim3((unsigned)ctas, (unsigned)p.w), kBwThreads, 0, stream>>>(p, part);
  }
  note_launch();
  conv_filter_grad_finish<<<(unsigned)((p.w + 127) / 128), 128, 0, stream>>>(part, ctas, p.w, strided ? 1 : 0, df);
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

// Plane kernel (32-bit index math; max: each window's first maximum computed
// once into shared memory, then every position gathers the windows routed to
// it).  One CTA per plane (grid-strided), used when a plane's window table
// fits shared memory.
__device__ __forceinline__ int div_small(int a, int d) { return d == 1 ? a : (d == 2 ? a >> 1 : a / d); }

template <bool kAvg, int KH = 0, int KW = 0>
__global__ void __launch_bounds__(512) pool2d_backward_plane_kernel(const __grid_constant__ Pool2DBackwardParams p) {
  extern __shared__ __align__(16) float s_plane[];
  const int H = (int)p.H, W = (int)p.W, OH = (int)p.OH, OW = (int)p.OW;
  const int kh = KH ? KH : (int)p.kh, kw = KW ? KW : (int)p.kw, sh = (int)p.sh, sw = (int)p.sw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  float* g = s_plane;                                  // dy plane [OH][OW]
  int* s_arg2 = reinterpret_cast<int*>(s_plane + OH * OW);  // max: window argmax [OH][OW]
  for (int64_t pl = blockIdx.x; pl < p.planes; pl += gridDim.x) {
    const float* __restrict__ xp = p.x + pl * H * W;
    const float* __restrict__ gp = p.dy + pl * OH * OW;
    float* __restrict__ d = p.dx + pl * H * W;
    __syncthreads();  // previous plane's readers are done
    for (int e = threadIdx.x; e < OH * OW; e += blockDim.x) g[e] = __ldg(gp + e);
    if constexpr (kAvg) {
      __syncthreads();
    } else {
      for (int r = warp; r < OH; r += nwarps)
        for (int c = lane; c < OW; c += 32) {
          const float* xw = xp + r * sh * W + c * sw;
          float m = __ldg(xw);
          int best = r * sh * W + c * sw;
#pragma unroll
          for (int a = 0; a < (KH ? KH : 64); ++a) {
            if (!KH && a >= kh) break;
#pragma unroll
            for (int bb = 0; bb < (KW ? KW : 64); ++bb) {
              if (!KW && bb >= kw) break;
              const float v = __ldg(xw + a * W + bb);
              if (v > m) { m = v; best = (r * sh + a) * W + c * sw + bb; }
            }
          }
          s_arg2[r * OW + c] = best;
        }
      __syncthreads();
    }
    for (int h = warp; h < H; h += nwarps) {
      const int r0 = h - kh + 1 <= 0 ? 0 : div_small(h - kh + sh, sh), r1 = min(div_small(h, sh), OH - 1);
      for (int c = lane; c < W; c += 32) {
        const int c0 = c - kw + 1 <= 0 ? 0 : div_small(c - kw + sw, sw), c1 = min(div_small(c, sw), OW - 1);
        const int e = h * W + c;
        float acc = 0.0f;
        for (int r = r0; r <= r1; ++r)
          for (int cc = c0; cc <= c1; ++cc) {
            if constexpr (kAvg) acc = __fadd_rn(acc, g[r * OW + cc]);
            else if (s_arg2[r * OW + cc] == e) acc = __fadd_rn(acc, g[r * OW + cc]);
          }
        d[e] = kAvg ? __fmul_rn(acc, p.inv_area) : acc;
      }
    }
  }
}

// Fixed-shape plane kernel (3x3/1 and 2x2/2, the DNN pooling shapes): 256
// threads, two CTAs per SM.  avg is separable: a transposed row pass
// R[r][c] = sum of dy[r][cc] over the <= ceil(KW/SW) windows cc covering c
// (shared memory), then a transposed column pass dx[h][c] = inv * sum of
// R[r][c] over the <= ceil(KH/SH) windows r covering h.  max builds the
// window-argmax table, then gathers the <= ceil(KH/SH) x ceil(KW/SW)
// candidate windows per position (row-major window order, as the direct path).
template <bool kAvg, int KH, int KW, int SH, int SW>
__global__ void __launch_bounds__(256, 2) pool2d_backward_fixed_kernel(const __grid_constant__ Pool2DBackwardParams p) {
  extern __shared__ __align__(16) float s_fx[];
  constexpr int NR = (KH + SH - 1) / SH, NCW = (KW + SW - 1) / SW;  // candidate windows per dimension
  const int H = (int)p.H, W = (int)p.W, OH = (int)p.OH, OW = (int)p.OW;
  float* g = s_fx;                          // dy plane [OH][OW]
  float* aux = s_fx + OH * OW;              // avg: R [OH][W]; max: argmax table [OH][OW] (int)
  int* tab = reinterpret_cast<int*>(aux);
  for (int64_t pl = blockIdx.x; pl < p.planes; pl += gridDim.x) {
    const float* __restrict__ gp = p.dy + pl * OH * OW;
    float* __restrict__ d = p.dx + pl * H * W;
    __syncthreads();
    for (int e = threadIdx.x; e < OH * OW; e += 256) g[e] = __ldg(gp + e);
    if constexpr (!kAvg && SH == 1) {
      // overlapping window rows: each thread walks one window column down a band
      // of rows with a ring of the last KH row results (first max of the row's KW
      // inputs, value + column); the window's first row-major maximum is the
      // first strictly greater row result in row order
      const float* __restrict__ xp = p.x + pl * H * W;
      const int bands = 256 / OW > 0 ? 256 / OW : 1;
      const int band_rows = (OH + bands - 1) / bands;
      for (int u = threadIdx.x; u < OW * bands; u += 256) {
        const int c = u % OW, band = u / OW;
        const int ra = band * band_rows, rb = min(ra + band_rows, OH);
        if (ra >= rb) continue;
        float rv[KH];
        int rc[KH];
        auto row_first_max = [&](int h, float& v, int& col) {
          const float* xr = xp + h * W + c * SW;
          v = __ldg(xr);
          col = c * SW;
#pragma unroll
          for (int b = 1; b < KW; ++b) {
            const float t = __ldg(xr + b);
            if (t > v) { v = t; col = c * SW + b; }
          }
        };
#pragma unroll
        for (int a = 0; a < KH - 1; ++a) row_first_max(ra + a, rv[a + 1], rc[a + 1]);
        for (int r = ra; r < rb; ++r) {
#pragma unroll
          for (int a = 0; a < KH - 1; ++a) { rv[a] = rv[a + 1]; rc[a] = rc[a + 1]; }
          row_first_max(r + KH - 1, rv[KH - 1], rc[KH - 1]);
          float m = rv[0];
          int best = r * W + rc[0];
#pragma unroll
          for (int a = 1; a < KH; ++a)
            if (rv[a] > m) { m = rv[a]; best = (r + a) * W + rc[a]; }
          tab[r * OW + c] = best;
        }
      }
    } else if constexpr (!kAvg) {
      const float* __restrict__ xp = p.x + pl * H * W;
      for (int e = threadIdx.x; e < OH * OW; e += 256) {
        const int r = e / OW, c = e - r * OW;
        const float* xw = xp + r * SH * W + c * SW;
        float m = __ldg(xw);
        int best = 0;
#pragma unroll
        for (int a = 0; a < KH; ++a)
#pragma unroll
          for (int b = 0; b < KW; ++b) {
            const float v = __ldg(xw + a * W + b);
            if (v > m) { m = v; best = a * W + b; }
          }
        tab[e] = (r * SH) * W + c * SW + best;
      }
    }
    __syncthreads();
    if constexpr (kAvg) {
      for (int e = threadIdx.x; e < OH * W; e += 256) {  // row pass
        const int r = e / W, c = e - r * W;
        const int c0 = c - KW + 1 <= 0 ? 0 : (c - KW + SW) / SW;
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < NCW; ++q) {
          const int cc = c0 + q;
          if (cc * SW <= c && cc < OW) acc = __fadd_rn(acc, g[r * OW + cc]);
        }
        aux[e] = acc;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < H * W; e += 256) {  // column pass
        const int h = e / W, c = e - h * W;
        const int r0 = h - KH + 1 <= 0 ? 0 : (h - KH + SH) / SH;
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int r = r0 + q;
          if (r * SH <= h && r < OH) acc = __fadd_rn(acc, aux[r * W + c]);
        }
        d[e] = __fmul_rn(acc, p.inv_area);
      }
    } else {
      for (int e = threadIdx.x; e < H * W; e += 256) {
        const int h = e / W, c = e - h * W;
        const int r0 = h - KH + 1 <= 0 ? 0 : (h - KH + SH) / SH;
        const int c0 = c - KW + 1 <= 0 ? 0 : (c - KW + SW) / SW;
        float acc = 0.0f;
#pragma unroll
        for (int qr = 0; qr < NR; ++qr)
#pragma unroll
          for (int qc = 0; qc < NCW; ++qc) {
            const int r = r0 + qr, cc = c0 + qc;
            if (r * SH <= h && r < OH && cc * SW <= c && cc < OW && tab[r * OW + cc] == e)
              acc = __fadd_rn(acc, g[r * OW + cc]);
          }
        d[e] = acc;
      }
    }
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
  if (p.w <= kMaxDirectW && p.stride <= kMaxTileS) {
    const size_t smem = sizeof(float) * (size_t)(2 * kMaxTile + 3 * kMaxDirectW + kMaxTileS + 2) +
                        sizeof(int) * (size_t)(kMaxTile + kMaxDirectW + 2);
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(pool_max_backward_direct_kernel));
    if (e != cudaSuccess) return e;
    pool_max_backward_direct_kernel<<<g < 1 ? 1 : g, kBwThreads, smem, stream>>>(p);
  } else if (p.w <= kMaxTileW && p.stride <= kMaxTileS) {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(pool_max_backward_tile_kernel));
    if (e != cudaSuccess) return e;
    pool_max_backward_tile_kernel<<<g < 1 ? 1 : g, kBwThreads, kMaxTileSmem, stream>>>(p);
  } else {
    pool_max_backward_kernel<<<g < 1 ? 1 : g, kBwThreads, 0, stream>>>(p);
  }
  note_launch();
  return cudaGetLastError();
}

template <int KH, int KW, int SH, int SW>
static cudaError_t launch_pool2d_bwd_fixed(const Pool2DBackwardParams& p, cudaStream_t stream, int sms) {
  const size_t smem = (size_t)(p.OH * p.OW + (p.mode == 1 ? p.OH * p.W : p.OH * p.OW)) * sizeof(float);
  if (smem > (size_t)kSmemBudget / 2 || p.H * p.W >= (int64_t(1) << 30)) return cudaErrorInvalidConfiguration;
  const int64_t g = p.planes < (int64_t)sms * 2 ? p.planes : (int64_t)sms * 2;
  auto kfn = p.mode == 1 ? pool2d_backward_fixed_kernel<true, KH, KW, SH, SW>
                         : pool2d_backward_fixed_kernel<false, KH, KW, SH, SW>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  kfn<<<(unsigned)g, 256, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pool2d_backward(const Pool2DBackwardParams& p, cudaStream_t stream, int sms) {
  {
    cudaError_t e = cudaErrorInvalidConfiguration;
    if (p.kh == 3 && p.kw == 3 && p.sh == 1 && p.sw == 1) e = launch_pool2d_bwd_fixed<3, 3, 1, 1>(p, stream, sms);
    else if (p.kh == 2 && p.kw == 2 && p.sh == 2 && p.sw == 2) e = launch_pool2d_bwd_fixed<2, 2, 2, 2>(p, stream, sms);
    if (e != cudaErrorInvalidConfiguration) return e;
  }
  const size_t table = (size_t)p.OH * p.OW * sizeof(float) * (p.mode == 1 ? 1 : 2);  // dy (+ argmax)
  if (p.H * p.W < (int64_t(1) << 30) && table <= (size_t)kSmemBudget) {
    const int64_t gp = p.planes < (int64_t)sms * 4 ? p.planes : (int64_t)sms * 4;
    if (p.mode == 1) {
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(pool2d_backward_plane_kernel<true>));
      if (e != cudaSuccess) return e;
      pool2d_backward_plane_kernel<true><<<(unsigned)gp, 512, table, stream>>>(p);
    } else {
      auto kfn = pool2d_backward_plane_kernel<false>;
      if (p.kh == 3 && p.kw == 3) kfn = pool2d_backward_plane_kernel<false, 3, 3>;
      else if (p.kh == 2 && p.kw == 2) kfn = pool2d_backward_plane_kernel<false, 2, 2>;
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
      if (e != cudaSuccess) return e;
      kfn<<<(unsigned)gp, 512, table, stream>>>(p);
    }
    note_launch();
    return cudaGetLastError();
  }
  const unsigned g = grid_elems(p.planes * p.H * p.W, sms);
  if (p.mode == 1) pool2d_backward_kernel<true><<<g, kBwThreads, 0, stream>>>(p);
  else pool2d_backward_kernel<false><<<g, kBwThreads, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ss
