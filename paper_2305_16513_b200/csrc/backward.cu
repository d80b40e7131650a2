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

// Unit stride, w <= 8R: O(1) work per element in registers.  A tile is
// kRunTile(R) = 256 R - 8 R positions [t0, t0 + T); its 256 R windows start at
// t0 - (w - 1) (the ones outside [0, L) get sentinel keys), R consecutive per
// thread.  (1) The thread's R window argmaxes by the pivot split of Alg. 2
// at its block end: suffix first-argmax over its own R inputs
// (right to left, ties to the earlier index), one running prefix argmax over
// the next w - 1 inputs (left to right, strictly greater), combined per window
// with the suffix side winning ties; w <= R scans each window directly.
// (2) The keys a_i are non-decreasing (see the tile kernel), so dx is a
// reduce-by-key of dy over sorted keys: each thread sums its runs left to
// right, a run that continues into the following threads is completed by the
// thread where it starts from their published head partials (in order), and
// the run owner writes dx_t into the zeroed smem tile.  x and dy are staged
// with 4-B cp.async into a layout padded by one word per R, so the stride-R
// reads of a warp hit distinct banks.
template <int R>
struct RunTile {
  static constexpr int kWindows = kBwThreads * R;
  static constexpr int kMaxW = 8 * R;
  static constexpr int kPositions = kWindows - kMaxW;
  static constexpr int kXSpan = kWindows + kMaxW;
  __host__ __device__ static constexpr int pad(int e) { return e + e / R; }
  static constexpr int kXFloats = (kXSpan + kXSpan / R + 4) & ~3;
  static constexpr int kGFloats = (kWindows + kWindows / R + 4) & ~3;
  static constexpr int kStageFloats = kXFloats + kGFloats;
  static constexpr size_t kSmem =
      sizeof(float) * (size_t)(2 * kStageFloats + kPositions + kPositions / R + 4) + 4 * sizeof(int) * kBwThreads;
};

template <int R>
__global__ void __launch_bounds__(kBwThreads) pool_max_backward_run_kernel(const __grid_constant__ BackwardParams p) {
  using RT = RunTile<R>;
  extern __shared__ __align__(16) float mr_smem[];
  // two stages of {x[t0 - (w-1) + e] at pad(e), dy[t0 - (w-1) + j] at pad(j)}: tile n+1 streams in
  // while tile n is evaluated
  float* dxs = mr_smem + 2 * RT::kStageFloats;  // dx tile at pad(t - t0): run owners write stride-R keys
  float* Hs = dxs + RT::kPositions + RT::kPositions / R + 4;  // head-run partial of each thread
  int* Ks = reinterpret_cast<int*>(Hs + kBwThreads);  // first key of each thread
  int* Ls = Ks + kBwThreads;                    // last key
  int* Fs = Ls + kBwThreads;                    // 1: the thread is one run
  const float* __restrict__ x = static_cast<const float*>(p.x);
  const float* __restrict__ dy = static_cast<const float*>(p.dy);
  float* __restrict__ dx = static_cast<float*>(p.dx);
  const int w = (int)p.w;
  constexpr int T = RT::kPositions;
  const int64_t tiles_per_row = (p.N + T - 1) / T;
  const int64_t ntiles = p.batch * tiles_per_row;
  const int tid = threadIdx.x, j0 = tid * R;
  constexpr int kLow = INT32_MIN / 2, kHigh = INT32_MAX / 2;  // sentinel keys outside any tile
  // (row, tile-in-row) cursors: issue runs one tile ahead of compute; advanced without divisions
  const int64_t step_b = gridDim.x / tiles_per_row, step_t = gridDim.x - step_b * tiles_per_row;
  int64_t ib = blockIdx.x / tiles_per_row, it = blockIdx.x - ib * tiles_per_row;
  int64_t cb = ib, ct = it;
  auto advance = [&](int64_t& b, int64_t& t) {
    b += step_b;
    t += step_t;
    if (t >= tiles_per_row) { t -= tiles_per_row; ++b; }
  };
  // valid staged ranges [lo, hi) of a tile: x index ws + e in [0, N), window ws + j in [0, L)
  struct Range { int xlo, xhi, glo, ghi; };
  auto ranges = [&](int64_t t) {
    const int64_t ws = t * T - (w - 1);
    Range r;
    r.xlo = ws < 0 ? (int)-ws : 0;
    r.glo = r.xlo;
    const int64_t xh = p.N - ws, gh = p.L - ws;
    r.xhi = xh < RT::kXSpan ? (int)xh : RT::kXSpan;
    r.ghi = gh < RT::kWindows ? (gh < 0 ? 0 : (int)gh) : RT::kWindows;
    return r;
  };
  auto issue = [&](int st) {
    if (ib < p.batch) {
      const Range rg = ranges(it);
      const int64_t ws = it * T - (w - 1);
      const float* xr = x + ib * p.N + ws;   // may point before the row: only valid e are read
      const float* gr = dy + ib * p.L + ws;
      float* xs = mr_smem + st * RT::kStageFloats;
      const uint32_t xd = smem_u32(xs + RT::pad(tid)), gd = smem_u32(xs + RT::kXFloats + RT::pad(tid));
      const int xspan = RT::kWindows + w - 1;
      // pad(e + 256 u) = pad(e) + (256 + 256 / R) u
#pragma unroll
      for (int u = 0; u < (RT::kXSpan + kBwThreads - 1) / kBwThreads; ++u) {
        const int e = tid + u * kBwThreads;
        if (e < xspan) {
          const bool ok = e >= rg.xlo && e < rg.xhi;
          cp_async4(xd + 4u * (kBwThreads + kBwThreads / R) * u, ok ? xr + e : x, ok ? 4u : 0u);
        }
      }
#pragma unroll
      for (int u = 0; u < RT::kWindows / kBwThreads; ++u) {
        const int e = tid + u * kBwThreads;
        const bool ok = e >= rg.glo && e < rg.ghi;
        cp_async4(gd + 4u * (kBwThreads + kBwThreads / R) * u, ok ? gr + e : dy, ok ? 4u : 0u);
      }
      advance(ib, it);
    }
    cp_async_commit();
  };
  issue(0);
  int st = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t t0 = ct * T;
    const int nt = (int)(t0 + T < p.N ? T : p.N - t0);
    const Range rg = ranges(ct);
    float* __restrict__ dxr = dx + cb * p.N + t0;
    advance(cb, ct);
    for (int e = tid; e < nt; e += kBwThreads) dxs[RT::pad(e)] = 0.0f;  // own store-loop slots: already read
    issue(st ^ 1);
    cp_async_wait<1>();
    __syncthreads();
    const float* xs = mr_smem + st * RT::kStageFloats;
    const float* gs = xs + RT::kXFloats;
    // (1) first maximum of windows j0 .. j0 + R - 1, as positions relative to t0
    int key[R];
    if (w > R) {
      float sv[R];
      int si[R];
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        const float v = xs[RT::pad(j0 + r)];
        if (r == R - 1 || v >= sv[r + 1 < R ? r + 1 : r]) { sv[r] = v; si[r] = j0 + r; }
        else { sv[r] = sv[r + 1 < R ? r + 1 : r]; si[r] = si[r + 1 < R ? r + 1 : r]; }
      }
      float pv = -INFINITY;
      int pi = 0;
      for (int m = R; m < w - 1; ++m) {
        const float v = xs[RT::pad(j0 + m)];
        if (v > pv) { pv = v; pi = j0 + m; }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float v = xs[RT::pad(j0 + w - 1 + r)];
        if (v > pv) { pv = v; pi = j0 + w - 1 + r; }
        key[r] = (pv > sv[r] ? pi : si[r]) - (w - 1);
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float m = xs[RT::pad(j0 + r)];
        int a = j0 + r;
        for (int q = 1; q < w; ++q) {
          const float v = xs[RT::pad(j0 + r + q)];
          if (v > m) { m = v; a = j0 + r + q; }
        }
        key[r] = a - (w - 1);
      }
    }
    float g[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (j0 + r < rg.glo) key[r] = kLow;
      else if (j0 + r >= rg.ghi) key[r] = kHigh;
      g[r] = gs[RT::pad(j0 + r)];
    }
    // (2) runs: head partial, interior runs written here, last run carried
    auto put = [&](int k, float v) {
      if (k >= 0 && k < nt) dxs[RT::pad(k)] = v;
    };
    int cur = key[0];
    float acc = g[0], head = 0.0f;
    bool single = true;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      if (key[r] != cur) {
        if (single) head = acc;
        else put(cur, acc);
        single = false;
        cur = key[r];
        acc = g[r];
      } else {
        acc = __fadd_rn(acc, g[r]);
      }
    }
    if (single) head = acc;
    Hs[tid] = head;
    Ks[tid] = key[0];
    Ls[tid] = key[R - 1];
    Fs[tid] = single ? 1 : 0;
    __syncthreads();
    auto chain = [&](int k, float total) {
      for (int u = tid + 1; u < kBwThreads && Ks[u] == k; ++u) {
        total = __fadd_rn(total, Hs[u]);
        if (!Fs[u]) break;
      }
      return total;
    };
    if (tid == 0 || Ls[tid - 1] != key[0]) put(key[0], single ? chain(key[0], head) : head);
    if (!single) put(cur, chain(cur, acc));
    __syncthreads();  // dx tile complete; stage st and Hs / Ks / Ls / Fs are free again
    for (int e = tid; e < nt; e += kBwThreads) dxr[e] = dxs[RT::pad(e)];
    st ^= 1;
  }
  cp_async_wait<0>();
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
// Unit stride (the common case): grid (ctas, tap blocks of 64), tile-pair
// kernel below.  Strided: grid (ctas, k); each CTA sums dy_i x_{is+j} for one
// tap over a grid-strided share of the outputs (fp32 runs of 16, then fp64).
// Finish: sums the CTA partials of each tap in fixed order.
constexpr int kFgTaps = 64;   // taps per tap block (partials layout)
constexpr int kFgRun = 16;    // outputs per thread and tile
constexpr int kFgFold = 4;    // tile pairs accumulated in fp32 (16 terms each) before folding into fp64

// Tile-pair kernel (unit stride).  Two tiles A, B are staged INTERLEAVED
// (pair e = (v_A[e], v_B[e]) for x and dy), so every FFMA2 operand is an
// aligned register pair straight from an LDS.128 -- (acc_A, acc_B)[j] +=
// (x_A, x_B)[m+j] * (dy_A, dy_B)[m] -- with no register shuffling (the
// per-tile tap-pair form needs odd-aligned x pairs: ~0.8 MOV per FFMA2).
// Q tap groups of 16 taps (Q = 1, 2, 4 by k) x 256/Q run slots of 16
// outputs; pair index e sits at float offset 2e + 4 (e >> 4), so the 16-pair
// blocks of neighbouring run slots start in different bank groups.  Stages
// are filled with 4-B cp.async (rows have any alignment; the interleave is
// element-granular).  A thread accumulates its 16 x 16 block in fp32 and
// folds into fp64 every kFgFold tile pairs; at the end the run slots of each
// tap are reduced in fixed order and the CTA writes its fp64 partials.
template <int Q>
struct FgPair {
  static constexpr int kSlots = kBwThreads / Q;
  static constexpr int kTile = kFgRun * kSlots;  // outputs per tile
  static constexpr int kTaps = 16 * Q;
  static constexpr int kXSpan = kTile + kTaps;   // inputs per tile
  static constexpr int kStages = Q == 4 ? 3 : 2;
  __host__ __device__ static constexpr int pad2(int e) { return 2 * e + 4 * (e >> 4); }
  static constexpr int kXFloats = pad2(kXSpan) + 8;
  static constexpr int kStageFloats = kXFloats + pad2(kTile) + 8;
  static constexpr size_t kSmem = (size_t)kStages * kStageFloats * sizeof(float);
};

template <int Q>
__global__ void __launch_bounds__(kBwThreads) conv_filter_grad_pair_kernel(const __grid_constant__ BackwardParams p,
                                                                           double* __restrict__ partials) {
  using F = FgPair<Q>;
  constexpr int S = F::kStages;
  extern __shared__ __align__(16) float fp_smem[];
  double* red = reinterpret_cast<double*>(fp_smem);  // reused for the final reduction
  const float* __restrict__ x = static_cast<const float*>(p.x);
  const float* __restrict__ dy = static_cast<const float*>(p.dy);
  const int64_t j0 = (int64_t)blockIdx.y * kFgTaps;
  const int q = threadIdx.x % Q, r = threadIdx.x / Q;  // tap group, run slot
  const int64_t tiles_per_row = (p.L + F::kTile - 1) / F::kTile;
  const int64_t ntiles = p.batch * tiles_per_row;
  const int64_t npairs = (ntiles + 1) / 2;
  int64_t ipair = blockIdx.x;
  // (row, tile-in-row) of tile A = 2 ipair, advanced by 2 gridDim.x tiles per issue without divisions
  const int64_t step = 2 * (int64_t)gridDim.x, step_b = step / tiles_per_row, step_t = step - step_b * tiles_per_row;
  int64_t cb = 2 * (int64_t)blockIdx.x / tiles_per_row, ct = 2 * (int64_t)blockIdx.x - cb * tiles_per_row;
  // one tile into lane 0 (A) or 1 (B) of the interleaved stage; 4-B cp.async (rows have any
  // alignment), compile-time trip counts, pad2(e + 256 u) = pad2(e) + 576 u
  auto stage_tile = [&](float* xs, float* gs, int64_t b, int64_t t, int lane) {
    const float* xsrc = x;
    const float* gsrc = dy;
    int xav = 0, gav = 0;
    if (b < p.batch) {
      const int64_t i0 = t * F::kTile;
      xsrc = x + b * p.N + i0 + j0;
      gsrc = dy + b * p.L + i0;
      const int64_t xa = p.N - i0 - j0, ga = p.L - i0;
      xav = xa < 0 ? 0 : (xa < F::kXSpan ? (int)xa : F::kXSpan);
      gav = ga < F::kTile ? (int)ga : F::kTile;
    }
    static_assert(F::pad2(kBwThreads) == 576 && F::kTile % kBwThreads == 0, "stage stride");
    const int tid = threadIdx.x;
    const uint32_t xd = smem_u32(xs + F::pad2(tid) + lane), gd = smem_u32(gs + F::pad2(tid) + lane);
#pragma unroll
    for (int u = 0; u < (F::kXSpan + kBwThreads - 1) / kBwThreads; ++u) {
      const int e = tid + u * kBwThreads;
      if ((u + 1) * kBwThreads <= F::kXSpan || e < F::kXSpan) {
        const bool ok = e < xav;
        cp_async4(xd + 2304u * u, ok ? xsrc + e : x, ok ? 4u : 0u);
      }
    }
#pragma unroll
    for (int u = 0; u < F::kTile / kBwThreads; ++u) {
      const int e = tid + u * kBwThreads;
      const bool ok = e < gav;
      cp_async4(gd + 2304u * u, ok ? gsrc + e : dy, ok ? 4u : 0u);
    }
  };
  auto issue = [&](int st) {
    if (ipair < npairs) {
      float* xs = fp_smem + st * F::kStageFloats;
      float* gs = xs + F::kXFloats;
      stage_tile(xs, gs, cb, ct, 0);
      if (ct + 1 < tiles_per_row) stage_tile(xs, gs, cb, ct + 1, 1);
      else stage_tile(xs, gs, cb + 1, 0, 1);
      ipair += gridDim.x;
      cb += step_b;
      ct += step_t;
      if (ct >= tiles_per_row) { ct -= tiles_per_row; ++cb; }
    }
    cp_async_commit();
  };
#pragma unroll 1
  for (int st = 0; st < S - 1; ++st) issue(st);
  double acc64[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc64[i] = 0.0;
  float2 acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = make_float2(0.0f, 0.0f);
  const int xb = F::pad2(16 * (r + q)), gb = F::pad2(16 * r);  // 16-pair blocks: offsets are block-uniform
  int st = 0, nfold = 0;
  for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    issue((st + S - 1) % S);
    cp_async_wait<S - 1>();
    __syncthreads();
    const float* xs = fp_smem + st * F::kStageFloats;
    const float* gs = xs + F::kXFloats;
    float2 X[32], G[16];
#pragma unroll
    for (int c = 0; c < 32; c += 2) {  // pairs c, c+1 of the x window; block boundary at c = 16
      const float4 v = *reinterpret_cast<const float4*>(xs + xb + 2 * c + (c >= 16 ? 4 : 0));
      X[c] = make_float2(v.x, v.y);
      X[c + 1] = make_float2(v.z, v.w);
    }
#pragma unroll
    for (int c = 0; c < 16; c += 2) {
      const float4 v = *reinterpret_cast<const float4*>(gs + gb + 2 * c);
      G[c] = make_float2(v.x, v.y);
      G[c + 1] = make_float2(v.z, v.w);
    }
#pragma unroll
    for (int mt = 0; mt < kFgRun; ++mt)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = __ffma2_rn(X[mt + i], G[mt], acc[i]);
    if (++nfold == kFgFold) {
      nfold = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        acc64[i] += (double)acc[i].x;
        acc64[i] += (double)acc[i].y;
        acc[i] = make_float2(0.0f, 0.0f);
      }
    }
    __syncthreads();  // stage st is refilled by the next iteration's issue
    st = st + 1 == S ? 0 : st + 1;
  }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    acc64[i] += (double)acc[i].x;
    acc64[i] += (double)acc[i].y;
  }
  static_assert(F::kSmem >= (size_t)F::kTaps * F::kSlots * sizeof(double), "reduction fits the stages");
#pragma unroll
  for (int i = 0; i < 16; ++i) red[(16 * q + i) * F::kSlots + r] = acc64[i];
  __syncthreads();
  if (threadIdx.x < F::kTaps) {
    double s = 0.0;
    for (int rr = 0; rr < F::kSlots; ++rr) s += red[threadIdx.x * F::kSlots + rr];
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

// One warp per tap: lane l sums partials l, l+32, ... in order, then a fixed
// butterfly -- parallel (the serial one-thread-per-tap sum was latency-bound at
// ~0.1 us per partial) and still deterministic.
__global__ void conv_filter_grad_finish(const double* __restrict__ partials, int ctas, int64_t k, int strided,
                                        float* __restrict__ df) {
  const int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= k) return;
  const int64_t blk = j / kFgTaps, jj = j - blk * kFgTaps;
  double s = 0.0;
  for (int c = lane; c < ctas; c += 32)
    s += strided ? partials[j * ctas + c] : partials[(blk * ctas + c) * kFgTaps + jj];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) df[j] = (float)s;
}

cudaError_t launch_conv_filter_grad_finish(const double* part, int ctas, int64_t k, float* df, cudaStream_t stream) {
  conv_filter_grad_finish<<<(unsigned)((k + 3) / 4), 128, 0, stream>>>(part, ctas, k, 0, df);
  note_launch();
  return cudaGetLastError();
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
    const int tap_blocks = (int)((p.w + kFgTaps - 1) / kFgTaps);
    const dim3 grid((unsigned)ctas, (unsigned)tap_blocks);
    auto launch = [&](auto kfn, size_t smem) {
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
      if (e == cudaSuccess) kfn<<<grid, kBwThreads, smem, stream>>>(p, part);
      return e;
    };
    // Q tap groups of 16: k <= 16 -> 1, k <= 32 -> 2, else 4 per 64-tap block
    cudaError_t e = p.w <= 16   ? launch(conv_filter_grad_pair_kernel<1>, FgPair<1>::kSmem)
                    : p.w <= 32 ? launch(conv_filter_grad_pair_kernel<2>, FgPair<2>::kSmem)
                                : launch(conv_filter_grad_pair_kernel<4>, FgPair<4>::kSmem);
    if (e != cudaSuccess) return e;
  } else {
    conv_filter_grad_strided_kernel<<<dim3((unsigned)ctas, (unsigned)p.w), kBwThreads, 0, stream>>>(p, part);
  }
  note_launch();
  conv_filter_grad_finish<<<(unsigned)((p.w + 3) / 4), 128, 0, stream>>>(part, ctas, p.w, strided ? 1 : 0, df);
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
  const int H = (int)p.H, W = (int)p.W, OH = (int)p.OH, OW = (int)p.OW;
  // shared: dy plane [OH][OW] (g); max: then the x plane [H][W] and the window-relative
  // first-argmax table [OH][OW] (uint8, a * KW + b)
  const int gsz = (OH * OW + 3) & ~3;
  float* g = s_fx;
  float* xs = s_fx + gsz;
  uint8_t* tab = reinterpret_cast<uint8_t*>(xs + ((H * W + 3) & ~3));
  // 16-B cp.async when the planes' starts are 16-B aligned, else 4-B
  auto stage = [&](float* dst, const float* __restrict__ src, int n) {
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (n & 3) == 0) {
      for (int e = 4 * threadIdx.x; e < n; e += 4 * 256) cp_async16(smem_u32(dst + e), src + e, 16u);
    } else {
      for (int e = threadIdx.x; e < n; e += 256) cp_async4(smem_u32(dst + e), src + e, 4u);
    }
  };
  for (int64_t pl = blockIdx.x; pl < p.planes; pl += gridDim.x) {
    const float* __restrict__ gp = p.dy + pl * OH * OW;
    float* __restrict__ d = p.dx + pl * H * W;
    __syncthreads();  // the previous plane's readers are done
    stage(g, gp, OH * OW);
    if constexpr (!kAvg) stage(xs, p.x + pl * H * W, H * W);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if constexpr (!kAvg && SH == 1) {
      // overlapping window rows: each task walks one window column down a band of
      // rows with a ring of the last KH row results (first max of the row's KW
      // inputs, value + offset); the window's first row-major maximum is the
      // first strictly greater row result in row order
      const int bands = 512 / OW > 0 ? 512 / OW : 1;
      const int band_rows = (OH + bands - 1) / bands;
      for (int u = threadIdx.x; u < OW * bands; u += 256) {
        const int c = u % OW, band = u / OW;
        const int ra = band * band_rows, rb = min(ra + band_rows, OH);
        if (ra >= rb) continue;
        float rv[KH];
        int rc[KH];
        auto row_first_max = [&](int h, float& v, int& off) {
          const float* xr = xs + h * W + c * SW;
          v = xr[0];
          off = 0;
#pragma unroll
          for (int b2 = 1; b2 < KW; ++b2) {
            const float t = xr[b2];
            if (t > v) { v = t; off = b2; }
          }
        };
#pragma unroll
        for (int a2 = 0; a2 < KH - 1; ++a2) row_first_max(ra + a2, rv[a2 + 1], rc[a2 + 1]);
        for (int r = ra; r < rb; ++r) {
#pragma unroll
          for (int a2 = 0; a2 < KH - 1; ++a2) { rv[a2] = rv[a2 + 1]; rc[a2] = rc[a2 + 1]; }
          row_first_max(r + KH - 1, rv[KH - 1], rc[KH - 1]);
          float m = rv[0];
          int best = rc[0];
#pragma unroll
          for (int a2 = 1; a2 < KH; ++a2)
            if (rv[a2] > m) { m = rv[a2]; best = a2 * KW + rc[a2]; }
          tab[r * OW + c] = (uint8_t)best;
        }
      }
    } else if constexpr (!kAvg) {
      for (int e = threadIdx.x; e < OH * OW; e += 256) {
        const int r = e / OW, c = e - r * OW;
        const float* xw = xs + r * SH * W + c * SW;
        float m = xw[0];
        int best = 0;
#pragma unroll
        for (int a2 = 0; a2 < KH; ++a2)
#pragma unroll
          for (int b2 = 0; b2 < KW; ++b2) {
            const float v = xw[a2 * W + b2];
            if (v > m) { m = v; best = a2 * KW + b2; }
          }
        tab[e] = (uint8_t)best;
      }
    }
    __syncthreads();
    if constexpr (SH > 1) {
      // strided shapes: flat position loop over the <= ceil(k/s)^2 candidate windows
      constexpr int NR = (KH + SH - 1) / SH, NCW = (KW + SW - 1) / SW;
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
            if (r * SH <= h && r < OH && cc * SW <= c && cc < OW) {
              const int q = r * OW + cc;
              if constexpr (kAvg) {
                acc = __fadd_rn(acc, g[q]);
              } else {
                const int t = tab[q];
                if (r * SH + t / KW == h && cc * SW + t % KW == c) acc = __fadd_rn(acc, g[q]);
              }
            }
          }
        d[e] = kAvg ? __fmul_rn(acc, p.inv_area) : acc;
      }
    } else if constexpr (kAvg) {
      // dx[h][c] = (sum over windows (h - a, c - b)) / (KH KW): tasks walk one column down a
      // band of rows with a ring of the KH window-row sums R[r] = sum_b dy[r][c - b] (windows
      // in increasing column order), summed in increasing row order -- the separable form
      const int bands = 512 / W > 0 ? 512 / W : 1;
      const int band_rows = (H + bands - 1) / bands;
      for (int u = threadIdx.x; u < W * bands; u += 256) {
        const int c = u % W, band = u / W;
        const int ha = band * band_rows, hb = min(ha + band_rows, H);
        if (ha >= hb) continue;
        float R[KH];
        auto row_sum = [&](int r) {
          float acc = 0.0f;
          if (r >= 0 && r < OH) {
#pragma unroll
            for (int b2 = KW - 1; b2 >= 0; --b2) {
              const int cc = c - b2;
              if (cc >= 0 && cc < OW) acc = __fadd_rn(acc, g[r * OW + cc]);
            }
          }
          return acc;
        };
#pragma unroll
        for (int a2 = 0; a2 < KH - 1; ++a2) R[a2] = row_sum(ha - 1 - a2);  // state at h = ha - 1
        for (int h = ha; h < hb; ++h) {
#pragma unroll
          for (int a2 = KH - 1; a2 > 0; --a2) R[a2] = R[a2 - 1];
          R[0] = row_sum(h);
          float acc = 0.0f;
#pragma unroll
          for (int a2 = KH - 1; a2 >= 0; --a2)
            if (h - a2 >= 0 && h - a2 < OH) acc = __fadd_rn(acc, R[a2]);
          d[h * W + c] = __fmul_rn(acc, p.inv_area);
        }
      }
    } else {
      // window (r, cc) routes its dy to (r + a, cc + b) with a KW + b = its table entry.
      // Tasks walk one column c down a band of rows and keep the table entries and dy of
      // the KH window rows r = h - a (columns cc = c - b) in a register ring: each step
      // loads one new window row (KW entries) instead of all KH x KW candidates.
      const int bands = 512 / W > 0 ? 512 / W : 1;
      const int band_rows = (H + bands - 1) / bands;
      for (int u = threadIdx.x; u < W * bands; u += 256) {
        const int c = u % W, band = u / W;
        const int ha = band * band_rows, hb = min(ha + band_rows, H);
        if (ha >= hb) continue;
        int T[KH][KW];
        float G[KH][KW];
        auto load_row = [&](int r, int (&t)[KW], float (&gv)[KW]) {
#pragma unroll
          for (int b2 = 0; b2 < KW; ++b2) {
            const int cc = c - b2;
            const bool ok = r >= 0 && r < OH && cc >= 0 && cc < OW;
            t[b2] = ok ? (int)tab[r * OW + cc] : -1;
            gv[b2] = ok ? g[r * OW + cc] : 0.0f;
          }
        };
        // state before the first step (h = ha - 1): slot a2 holds window row ha - 1 - a2
#pragma unroll
        for (int a2 = 0; a2 < KH - 1; ++a2) load_row(ha - 1 - a2, T[a2], G[a2]);
        for (int h = ha; h < hb; ++h) {
#pragma unroll
          for (int a2 = KH - 1; a2 > 0; --a2)
#pragma unroll
            for (int b2 = 0; b2 < KW; ++b2) { T[a2][b2] = T[a2 - 1][b2]; G[a2][b2] = G[a2 - 1][b2]; }
          load_row(h, T[0], G[0]);
          float acc = 0.0f;
#pragma unroll
          for (int a2 = KH - 1; a2 >= 0; --a2)  // windows in increasing row-major order
#pragma unroll
            for (int b2 = KW - 1; b2 >= 0; --b2)
              if (T[a2][b2] == a2 * KW + b2) acc = __fadd_rn(acc, G[a2][b2]);
          d[h * W + c] = acc;
        }
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
  if (p.stride == 1 && p.w <= RunTile<16>::kMaxW) {
    auto launch = [&](auto kfn, int positions, size_t smem) {
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
      if (e != cudaSuccess) return e;
      const int64_t t = p.batch * ((p.N + positions - 1) / positions);
      int per_sm = 0;  // resident CTAs: one wave of the grid-strided tile loop
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kBwThreads, smem);
      if (e != cudaSuccess) return e;
      const int64_t c = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
      const unsigned gr = (unsigned)(t < c ? (t < 1 ? 1 : t) : c);
      kfn<<<gr, kBwThreads, smem, stream>>>(p);
      note_launch();
      return cudaGetLastError();
    };
    if (p.w <= RunTile<8>::kMaxW)
      return launch(pool_max_backward_run_kernel<8>, RunTile<8>::kPositions, RunTile<8>::kSmem);
    return launch(pool_max_backward_run_kernel<16>, RunTile<16>::kPositions, RunTile<16>::kSmem);
  }
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
  // dy plane + (avg) row sums or (max) x plane and a byte table, all 16-B padded
  const size_t r4 = [](int64_t n) { return (size_t)((n + 3) & ~int64_t(3)); }(p.OH * p.OW);
  const size_t smem = p.mode == 1 ? r4 * sizeof(float)
                                  : (r4 + (size_t)((p.H * p.W + 3) & ~int64_t(3))) * sizeof(float) +
                                        (size_t)p.OH * p.OW;
  if (smem > (size_t)kSmemBudget / 2 || p.H * p.W >= (int64_t(1) << 30)) return cudaErrorInvalidConfiguration;
  auto kfn = p.mode == 1 ? pool2d_backward_fixed_kernel<true, KH, KW, SH, SW>
                         : pool2d_backward_fixed_kernel<false, KH, KW, SH, SW>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  int per_sm = 0;  // resident CTAs: one wave of the plane loop
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 256, smem);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
  const int64_t g = p.planes < cap ? p.planes : cap;
  kfn<<<(unsigned)g, 256, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

// 2x2 windows at stride 2 (disjoint, covering the plane; H even, W % 4 == 0):
// a thread owns two neighbouring windows = a 2 x 4 block of dx.  avg spreads
// dy / 4; max sends dy to the window's first maximum in row-major order (ties
// to the earlier element, reading R16) and writes 0 elsewhere.  Every x / dx
// access is one 16-B vector (rows are 16-B aligned), dy one 8-B vector: a pure
// stream, read x (max) + dy, write dx.
template <bool kAvg>
__global__ void __launch_bounds__(256) pool2d_bwd_2x2s2_kernel(const __grid_constant__ Pool2DBackwardParams p) {
  const int64_t qpr = p.W / 4;                 // window pairs per row of windows
  const int64_t total = p.planes * p.OH * qpr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e % qpr, rr = e / qpr;   // rr = plane * OH + r
    const int64_t row0 = 2 * rr;                // first input row (plane-major flat: plane * H + 2 r)
    const float2 g = *reinterpret_cast<const float2*>(p.dy + rr * p.OW + 2 * q);
    float4* d0 = reinterpret_cast<float4*>(p.dx + row0 * p.W + 4 * q);
    float4* d1 = reinterpret_cast<float4*>(p.dx + (row0 + 1) * p.W + 4 * q);
    if (kAvg) {
      const float a = g.x * p.inv_area, b = g.y * p.inv_area;
      *d0 = make_float4(a, a, b, b);
      *d1 = make_float4(a, a, b, b);
    } else {
      const float4 u = *reinterpret_cast<const float4*>(p.x + row0 * p.W + 4 * q);
      const float4 v = *reinterpret_cast<const float4*>(p.x + (row0 + 1) * p.W + 4 * q);
      // window 0: u.x u.y / v.x v.y ; window 1: u.z u.w / v.z v.w -- first maximum, row-major
      int i0 = 0;
      float m0 = u.x;
      if (u.y > m0) { m0 = u.y; i0 = 1; }
      if (v.x > m0) { m0 = v.x; i0 = 2; }
      if (v.y > m0) { m0 = v.y; i0 = 3; }
      int i1 = 0;
      float m1 = u.z;
      if (u.w > m1) { m1 = u.w; i1 = 1; }
      if (v.z > m1) { m1 = v.z; i1 = 2; }
      if (v.w > m1) { m1 = v.w; i1 = 3; }
      *d0 = make_float4(i0 == 0 ? g.x : 0.f, i0 == 1 ? g.x : 0.f, i1 == 0 ? g.y : 0.f, i1 == 1 ? g.y : 0.f);
      *d1 = make_float4(i0 == 2 ? g.x : 0.f, i0 == 3 ? g.x : 0.f, i1 == 2 ? g.y : 0.f, i1 == 3 ? g.y : 0.f);
    }
  }
}

cudaError_t launch_pool2d_backward(const Pool2DBackwardParams& p, cudaStream_t stream, int sms) {
  if (p.kh == 2 && p.kw == 2 && p.sh == 2 && p.sw == 2 && p.H % 2 == 0 && p.W % 4 == 0 &&
      ((reinterpret_cast<uintptr_t>(p.dx) | reinterpret_cast<uintptr_t>(p.x)) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(p.dy) & 7) == 0) {
    const int64_t total = p.planes * p.OH * (p.W / 4);
    int64_t g = (total + 255) / 256;
    if (g > (int64_t)sms * 16) g = (int64_t)sms * 16;
    if (p.mode == 1) pool2d_bwd_2x2s2_kernel<true><<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
    else pool2d_bwd_2x2s2_kernel<false><<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
    note_launch();
    return cudaGetLastError();
  }
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
