// conv2d_backward.cu -- gradients of the 2-D sliding dot product (SURVEY 8f
// NEXT #4 "2-D convolution and backward passes"; reading R21), the
// vector-Jacobian products of y[p][r][c] = sum_a sum_b f[a][b] x[p][r sh+a][c sw+b]:
//
//   dx[p][h][w] = sum over (r, c, a, b) with r sh + a = h, c sw + b = w of f[a][b] dy[p][r][c]
//   df[a][b]    = sum_p sum_r sum_c dy[p][r][c] x[p][r sh+a][c sw+b]
//
// Input gradient (gather form, no atomics): a CTA owns an 8 x 128 dx tile; the
// dy region every window over that tile reads is staged in shared memory with
// zeros outside [0, OH) x [0, OW) (so uncovered dx elements come out 0 and the
// inner loops carry no bounds checks), lane t owns columns t, t+32, t+64, t+96
// (conflict-free LDS), taps in shared memory (warp-broadcast).
//
// Filter gradient: a CTA walks (plane, 16-row, 128-column) dy tiles; it stages
// the dy tile and the x region under it.  kh, kw <= 4: every thread keeps all
// taps' sums for its columns in registers (one LDS of x per FMA, dy read once
// per tap set), fp32 runs of one tile flushed into fp64 registers; larger
// filters: a warp per tap (fp32 run per tile, fp64 accumulator in shared
// memory).  Per-CTA fp64 partials go to the caller's workspace and a finishing
// kernel sums them in CTA order (deterministic).  Regions too large for
// shared memory take direct kernels reading global memory.
#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kC2bThreads = 256;
constexpr int kDxTileH = 32, kDxTileW = 128;
constexpr int kDfTileR = 16, kDfTileC = 128;
constexpr size_t kC2bSmemMax = 96 * 1024;

__device__ __forceinline__ void cp_async8(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes) : "memory");
}

// Stage one row: smem words [0, n) <- global gr[c0 + j] where 0 <= c0 + j < nvalid (else 0).
// G-element cp.async granules (G = 4 / 2 / 1) when the caller guarantees that gr + c0 is
// 4G-byte aligned and c0 % G == 0 (so a granule never straddles column 0); a granule
// straddling nvalid copies its valid prefix and zero-fills the rest.
template <int G>
__device__ __forceinline__ void stage_row(uint32_t srow, const float* gr, const float* any, int c0, int n, int nvalid,
                                          bool row_ok, int lane) {
  for (int j = G * lane; j < n; j += 32 * G) {
    const int c = c0 + j;
    int nv = nvalid - c;
    nv = (!row_ok || c < 0) ? 0 : (nv < 0 ? 0 : (nv > G ? G : nv));
    const void* src = nv > 0 ? (const void*)(gr + c) : any;
    if (G == 4) cp_async16(srow + 4u * (uint32_t)j, src, 4u * (uint32_t)nv);
    else if (G == 2) cp_async8(srow + 4u * (uint32_t)j, src, 4u * (uint32_t)nv);
    else cp_async4(srow + 4u * (uint32_t)j, src, 4u * (uint32_t)nv);
  }
}

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
__device__ __forceinline__ int64_t ceildiv(int64_t a, int64_t b) { return -floordiv(-a, b); }

// ------------------------------------------------------------ input gradient
// kS1: stride 1 (KH, KW > 0: that exact filter size, loops unrolled; 0: runtime).
template <bool kS1, int KH, int KW>
__global__ void __launch_bounds__(kC2bThreads) conv2d_bwd_input_tile_kernel(const __grid_constant__ Conv2DBwdParams p) {
  extern __shared__ __align__(16) float c2b_smem[];
  const int nt = (int)(p.kh * p.kw);
  float* fs = c2b_smem;
  float* ds = c2b_smem + ((nt + 3) & ~3);
  for (int t = threadIdx.x; t < nt; t += kC2bThreads) fs[t] = p.taps[t];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kh = KH > 0 ? KH : (int)p.kh, kw = KW > 0 ? KW : (int)p.kw;
  const int64_t tiles_h = (p.H + kDxTileH - 1) / kDxTileH, tiles_w = (p.W + kDxTileW - 1) / kDxTileW;
  const int64_t ntiles = p.planes * tiles_h * tiles_w;
  const int C = p.dx_c, buf_elems = p.dx_r * p.dx_c;
  // stage tile `tl`'s dy region into buffer `bf` with cp.async (zero-filled outside dy)
  auto stage = [&](int64_t tl, int bf) {
    const int64_t tw = tl % tiles_w, rest = tl / tiles_w, th = rest % tiles_h, pl = rest / tiles_h;
    const int64_t h0 = th * kDxTileH, w0 = tw * kDxTileW;
    const int64_t r_lo = ceildiv(h0 - kh + 1, p.sh), r_hi = floordiv(h0 + kDxTileH - 1, p.sh);
    const int64_t c_lo = ceildiv(w0 - kw + 1, p.sw), c_hi = floordiv(w0 + kDxTileW - 1, p.sw);
    const int R = (int)(r_hi - r_lo + 1), Cn = (int)(c_hi - c_lo + 1);
    const float* __restrict__ g = p.dy + pl * p.OH * p.OW;
    const uint32_t sb = smem_u32(ds + bf * buf_elems);
    const int c0 = (int)c_lo, ow = (int)p.OW;
    const bool g2 = (ow & 1) == 0 && (c0 & 1) == 0 && (reinterpret_cast<uintptr_t>(g) & 7) == 0;
    for (int rr = warp; rr < R; rr += kC2bThreads / 32) {
      const int64_t r = r_lo + rr;
      const bool row_ok = r >= 0 && r < p.OH;
      const float* __restrict__ gr = g + (row_ok ? r : 0) * p.OW;
      const uint32_t srow = sb + 4u * (uint32_t)(rr * C);
      if (g2) stage_row<2>(srow, gr, g, c0, Cn, ow, row_ok, lane);
      else stage_row<1>(srow, gr, g, c0, Cn, ow, row_ok, lane);
    }
  };
  if ((int64_t)blockIdx.x < ntiles) stage(blockIdx.x, 0);
  cp_async_commit();
  int buf = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (tile + gridDim.x < ntiles) stage(tile + gridDim.x, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();  // tile's region (and, first time, the taps) visible to every warp
    const int64_t tw = tile % tiles_w, rest = tile / tiles_w, th = rest % tiles_h, pl = rest / tiles_h;
    const int64_t h0 = th * kDxTileH, w0 = tw * kDxTileW;
    const int64_t r_lo = ceildiv(h0 - kh + 1, p.sh), c_lo = ceildiv(w0 - kw + 1, p.sw);
    const float* dsb = ds + buf * buf_elems;
    for (int hh = warp; hh < kDxTileH; hh += kC2bThreads / 32) {
      const int64_t h = h0 + hh;
      if (h >= p.H) break;
      if (kS1 && KH > 0 && KW > 0) {
        // exact size, stride 1: lane owns 4 consecutive columns w0 + 4 lane + q; per filter row
        // the ceil((KW + 3) / 4) LDS.128 it needs cover all KW taps of its 4 outputs (register
        // reuse across taps); taps are constant-bank operands
        constexpr int NV = (KW + 3 + 3) / 4;
        float acc4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int a = 0; a < (KH > 0 ? KH : 1); ++a) {
          const float4* row4 = reinterpret_cast<const float4*>(dsb + (hh + KH - 1 - a) * C) + lane;
          float v[4 * NV];
#pragma unroll
          for (int u = 0; u < NV; ++u) {
            const float4 t4 = row4[u];
            v[4 * u] = t4.x; v[4 * u + 1] = t4.y; v[4 * u + 2] = t4.z; v[4 * u + 3] = t4.w;
          }
#pragma unroll
          for (int b = 0; b < (KW > 0 ? KW : 1); ++b)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc4[q] = __fmaf_rn(p.taps[a * KW + b], v[q + KW - 1 - b], acc4[q]);
        }
        float* __restrict__ out = p.dx + (pl * p.H + h) * p.W;
        const int64_t w = w0 + 4 * lane;
        if (w + 3 < p.W && (reinterpret_cast<uintptr_t>(out + w) & 15) == 0) {
          *reinterpret_cast<float4*>(out + w) = make_float4(acc4[0], acc4[1], acc4[2], acc4[3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (w + q < p.W) out[w + q] = acc4[q];
        }
        continue;
      }
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      if (kS1) {
        // r = h - a, c = w - b; smem column of output q, tap b: (lane + 32 q) + kw - 1 - b
#pragma unroll
        for (int a = 0; a < (KH > 0 ? KH : 1); ++a) {
          for (int a2 = (KH > 0 ? a : 0); a2 < (KH > 0 ? a + 1 : kh); ++a2) {
            const float* row = dsb + (hh + kh - 1 - a2) * C + lane + kw - 1;
            const float* fa = fs + a2 * kw;
#pragma unroll
            for (int b = 0; b < (KW > 0 ? KW : 1); ++b) {
              for (int b2 = (KW > 0 ? b : 0); b2 < (KW > 0 ? b + 1 : kw); ++b2) {
                const float fv = fa[b2];
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = __fmaf_rn(fv, row[32 * q - b2], acc[q]);
              }
            }
          }
        }
      } else {
        const int64_t rmin = ceildiv(h - kh + 1, p.sh), rmax = floordiv(h, p.sh);
        for (int64_t r = rmin; r <= rmax; ++r) {
          const int a = (int)(h - r * p.sh);
          const float* row = dsb + (int)(r - r_lo) * C;
          const float* fa = fs + a * kw;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int64_t w = w0 + lane + 32 * q;
            const int64_t cmin = ceildiv(w - kw + 1, p.sw), cmax = floordiv(w, p.sw);
            float s = acc[q];
            for (int64_t c = cmin; c <= cmax; ++c) s = __fmaf_rn(fa[w - c * p.sw], row[c - c_lo], s);
            acc[q] = s;
          }
        }
      }
      float* __restrict__ out = p.dx + (pl * p.H + h) * p.W;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t w = w0 + lane + 32 * q;
        if (w < p.W) out[w] = acc[q];
      }
    }
    __syncthreads();  // every warp is done with buf before it is restaged
    buf ^= 1;
  }
}

// Direct gather (any size): one dx element per thread, dy through the read-only path.
__global__ void __launch_bounds__(kC2bThreads) conv2d_bwd_input_direct_kernel(const __grid_constant__ Conv2DBwdParams p) {
  const int64_t total = p.planes * p.H * p.W;
  for (int64_t e = blockIdx.x * (int64_t)kC2bThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kC2bThreads) {
    const int64_t w = e % p.W, rest = e / p.W, h = rest % p.H, pl = rest / p.H;
    const float* __restrict__ g = p.dy + pl * p.OH * p.OW;
    int64_t rmin = ceildiv(h - p.kh + 1, p.sh), rmax = floordiv(h, p.sh);
    int64_t cmin = ceildiv(w - p.kw + 1, p.sw), cmax = floordiv(w, p.sw);
    if (rmin < 0) rmin = 0;
    if (cmin < 0) cmin = 0;
    if (rmax > p.OH - 1) rmax = p.OH - 1;
    if (cmax > p.OW - 1) cmax = p.OW - 1;
    float s = 0.0f;
    for (int64_t r = rmin; r <= rmax; ++r) {
      const int64_t a = h - r * p.sh;
      for (int64_t c = cmin; c <= cmax; ++c) s = __fmaf_rn(p.taps[a * p.kw + (w - c * p.sw)], __ldg(g + r * p.OW + c), s);
    }
    p.dx[e] = s;
  }
}

// ----------------------------------------------------------- filter gradient
struct DfTile {
  int64_t pl, r0, c0;
  int nr, nc;
};

__device__ __forceinline__ DfTile df_tile(const Conv2DBwdParams& p, int64_t tile) {
  const int64_t tiles_r = (p.OH + kDfTileR - 1) / kDfTileR, tiles_c = (p.OW + kDfTileC - 1) / kDfTileC;
  DfTile t;
  const int64_t tc = tile % tiles_c, rest = tile / tiles_c, tr = rest % tiles_r;
  t.pl = rest / tiles_r;
  t.r0 = tr * kDfTileR;
  t.c0 = tc * kDfTileC;
  t.nr = (int)min((int64_t)kDfTileR, p.OH - t.r0);
  t.nc = (int)min((int64_t)kDfTileC, p.OW - t.c0);
  return t;
}

// Stage dy[tile] into dys[kDfTileR][kDfTileC] and the x region under it into xs[XR][XC]
// (zeros outside the tile, so padded lanes contribute 0 * 0).
__device__ __forceinline__ void df_stage(const Conv2DBwdParams& p, const DfTile& t, float* dys, float* xs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* __restrict__ g = p.dy + (t.pl * p.OH + t.r0) * p.OW + t.c0;
  const uint32_t sd = smem_u32(dys), sx = smem_u32(xs);
  const bool g2 = (p.OW & 1) == 0 && (reinterpret_cast<uintptr_t>(p.dy) & 7) == 0;  // c0 % 128 == 0
  for (int rr = warp; rr < kDfTileR; rr += kC2bThreads / 32) {
    const bool row_ok = rr < t.nr;
    const float* __restrict__ gr = g + (row_ok ? rr : 0) * p.OW;
    if (g2) stage_row<2>(sd + 4u * (uint32_t)(rr * kDfTileC), gr, g, 0, kDfTileC, t.nc, row_ok, lane);
    else stage_row<1>(sd + 4u * (uint32_t)(rr * kDfTileC), gr, g, 0, kDfTileC, t.nc, row_ok, lane);
  }
  const int xr = (t.nr - 1) * (int)p.sh + (int)p.kh, xc = (t.nc - 1) * (int)p.sw + (int)p.kw;
  const float* __restrict__ xg = p.x + (t.pl * p.H + t.r0 * p.sh) * p.W + t.c0 * p.sw;
  const bool g4 = (p.W & 3) == 0 && (reinterpret_cast<uintptr_t>(p.x) & 15) == 0;  // c0 sw % 4 == 0
  for (int rr = warp; rr < p.df_xr; rr += kC2bThreads / 32) {
    const bool row_ok = rr < xr;
    const float* __restrict__ xr_g = xg + (row_ok ? rr : 0) * p.W;
    const uint32_t srow = sx + 4u * (uint32_t)(rr * p.df_xc);
    if (g4) stage_row<4>(srow, xr_g, xg, 0, p.df_xc, xc, row_ok, lane);
    else stage_row<1>(srow, xr_g, xg, 0, p.df_xc, xc, row_ok, lane);
  }
}

// kh == KH, kw == KW (3x3, 5x5, 7x7) or kh, kw <= 4 (KH = KW = 4, guarded): every
// thread keeps all taps' sums for its columns in fp32 registers over a run of
// kDfRun tiles (<= 8 kDfRun products per tap per thread), then the warp reduces
// them (fp32 butterfly) into its own fp64 accumulators in shared memory.
constexpr int kDfRun = 16;

template <int KH, int KW, bool kExact>
__global__ void __launch_bounds__(kC2bThreads) conv2d_bwd_filter_reg_kernel(const __grid_constant__ Conv2DBwdParams p,
                                                                            double* __restrict__ part) {
  constexpr int T = KH * KW;
  extern __shared__ __align__(16) float c2b_smem[];
  double(*accw)[T] = reinterpret_cast<double(*)[T]>(c2b_smem);  // [warp][tap], warp-owned
  float* dys = c2b_smem + 2 * (kC2bThreads / 32) * T;
  float* xs = dys + kDfTileR * kDfTileC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kh = kExact ? KH : (int)p.kh, kw = kExact ? KW : (int)p.kw;
  const int sh = (int)p.sh, sw = (int)p.sw, XC = p.df_xc;
  for (int i = threadIdx.x; i < (kC2bThreads / 32) * T; i += kC2bThreads) (&accw[0][0])[i] = 0.0;
  float d[T];
#pragma unroll
  for (int i = 0; i < T; ++i) d[i] = 0.0f;
  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < T; ++i) {
      float v = d[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) accw[warp][i] += (double)v;
      d[i] = 0.0f;
    }
  };
  const int64_t ntiles = p.planes * ((p.OH + kDfTileR - 1) / kDfTileR) * ((p.OW + kDfTileC - 1) / kDfTileC);
  int run = 0;
  const int buf_elems = kDfTileR * kDfTileC + p.df_xr * p.df_xc;
  if ((int64_t)blockIdx.x < ntiles) df_stage(p, df_tile(p, blockIdx.x), dys, xs);
  cp_async_commit();
  int buf = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    const DfTile t = df_tile(p, tile);
    if (tile + gridDim.x < ntiles)
      df_stage(p, df_tile(p, tile + gridDim.x), dys + (buf ^ 1) * buf_elems, xs + (buf ^ 1) * buf_elems);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const float* dyb = dys + buf * buf_elems;
    const float* xsb = xs + buf * buf_elems;
    if (sw == 1) {
      // lane owns 4 consecutive dy columns 4 lane + q: one LDS.128 of dy and ceil((KW + 3) / 4)
      // LDS.128 of x per filter row cover all KW taps (register reuse across taps)
      constexpr int NV = (KW + 3 + 3) / 4;
      for (int rr = warp; rr < t.nr; rr += kC2bThreads / 32) {
        const float4 d4 = reinterpret_cast<const float4*>(dyb + rr * kDfTileC)[lane];
        const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int a = 0; a < KH; ++a) {
          if (kExact || a < kh) {
            const float4* x4 = reinterpret_cast<const float4*>(xsb + (rr * sh + a) * XC) + lane;
            float v[4 * NV];
#pragma unroll
            for (int u = 0; u < NV; ++u) {
              const float4 t4 = x4[u];
              v[4 * u] = t4.x; v[4 * u + 1] = t4.y; v[4 * u + 2] = t4.z; v[4 * u + 3] = t4.w;
            }
#pragma unroll
            for (int b = 0; b < KW; ++b)
              if (kExact || b < kw) {
#pragma unroll
                for (int q = 0; q < 4; ++q) d[a * KW + b] = __fmaf_rn(dv[q], v[q + b], d[a * KW + b]);
              }
          }
        }
      }
    } else
    for (int rr = warp; rr < t.nr; rr += kC2bThreads / 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = lane + 32 * q;
        const float dyv = dyb[rr * kDfTileC + c];
        const float* xb = xsb + rr * sh * XC + c * sw;
#pragma unroll
        for (int a = 0; a < KH; ++a) {
          if (kExact || a < kh) {
#pragma unroll
            for (int b = 0; b < KW; ++b)
              if (kExact || b < kw) d[a * KW + b] = __fmaf_rn(dyv, xb[a * XC + b], d[a * KW + b]);
          }
        }
      }
    }
    if (++run == kDfRun) {
      flush();
      run = 0;
    }
    __syncthreads();  // every warp is done with buf before it is restaged
  }
  flush();
  __syncthreads();
  for (int i = threadIdx.x; i < T; i += kC2bThreads) {
    const int a = i / KW, b = i - a * KW;
    if (a < kh && b < kw) {
      double v = 0.0;
      for (int w = 0; w < kC2bThreads / 32; ++w) v += accw[w][i];
      part[(int64_t)(a * kw + b) * gridDim.x + blockIdx.x] = v;
    }
  }
}

// Any filter whose tile region fits: a warp per tap, fp64 accumulator per tap in shared memory.
__global__ void __launch_bounds__(kC2bThreads) conv2d_bwd_filter_tap_kernel(const __grid_constant__ Conv2DBwdParams p,
                                                                            double* __restrict__ part) {
  extern __shared__ __align__(16) float c2b_smem[];
  const int nt = (int)(p.kh * p.kw);
  double* acc = reinterpret_cast<double*>(c2b_smem);
  float* dys = c2b_smem + 2 * ((nt + 3) & ~3);
  float* xs = dys + kDfTileR * kDfTileC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kw = (int)p.kw, sh = (int)p.sh, sw = (int)p.sw, XC = p.df_xc;
  for (int t = threadIdx.x; t < nt; t += kC2bThreads) acc[t] = 0.0;
  const int64_t ntiles = p.planes * ((p.OH + kDfTileR - 1) / kDfTileR) * ((p.OW + kDfTileC - 1) / kDfTileC);
  const int buf_elems = kDfTileR * kDfTileC + p.df_xr * p.df_xc;
  if ((int64_t)blockIdx.x < ntiles) df_stage(p, df_tile(p, blockIdx.x), dys, xs);
  cp_async_commit();
  int buf = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    const DfTile t = df_tile(p, tile);
    if (tile + gridDim.x < ntiles)
      df_stage(p, df_tile(p, tile + gridDim.x), dys + (buf ^ 1) * buf_elems, xs + (buf ^ 1) * buf_elems);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const float* dyb = dys + buf * buf_elems;
    const float* xsb = xs + buf * buf_elems;
    for (int tap = warp; tap < nt; tap += kC2bThreads / 32) {
      const int a = tap / kw, b = tap - a * kw;
      float s = 0.0f;
      for (int rr = 0; rr < t.nr; ++rr) {
        const float* xb = xsb + (rr * sh + a) * XC + b;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = lane + 32 * q;
          s = __fmaf_rn(dyb[rr * kDfTileC + c], xb[c * sw], s);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) acc[tap] += (double)s;  // this warp alone owns tap
    }
    __syncthreads();  // every warp is done with buf before it is restaged
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nt; t += kC2bThreads) part[(int64_t)t * gridDim.x + blockIdx.x] = acc[t];
}

// Direct (any size): blockIdx.y = tap, grid-stride over dy elements, fp32 runs of 16 into fp64.
__global__ void __launch_bounds__(kC2bThreads) conv2d_bwd_filter_direct_kernel(const __grid_constant__ Conv2DBwdParams p,
                                                                               double* __restrict__ part) {
  __shared__ double red[kC2bThreads];
  const int64_t tap = blockIdx.y, a = tap / p.kw, b = tap - a * p.kw;
  const int64_t total = p.planes * p.OH * p.OW, step = (int64_t)gridDim.x * kC2bThreads;
  double acc64 = 0.0;
  int64_t e = blockIdx.x * (int64_t)kC2bThreads + threadIdx.x;
  while (e < total) {
    float s = 0.0f;
    for (int n = 0; n < 16 && e < total; ++n, e += step) {
      const int64_t c = e % p.OW, rest = e / p.OW, r = rest % p.OH, pl = rest / p.OH;
      s = __fmaf_rn(__ldg(p.dy + e), __ldg(p.x + (pl * p.H + r * p.sh + a) * p.W + c * p.sw + b), s);
    }
    acc64 += (double)s;
  }
  red[threadIdx.x] = acc64;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int t = 0; t < kC2bThreads; ++t) v += red[t];
    part[tap * gridDim.x + blockIdx.x] = v;
  }
}

// One warp per tap, lane-strided partial sums then a fixed butterfly (deterministic).
__global__ void conv2d_bwd_filter_finish(const double* __restrict__ part, int ctas, int64_t nt, float* __restrict__ df) {
  const int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= nt) return;
  double v = 0.0;
  for (int c = lane; c < ctas; c += 32) v += part[t * ctas + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) df[t] = (float)v;
}

size_t dx_smem(Conv2DBwdParams& p) {
  p.dx_r = (int)((kDxTileH - 1 + p.kh - 1) / p.sh + 2);
  p.dx_c = (int)((((kDxTileW - 1 + p.kw - 1) / p.sw + 2) + 3) / 4 * 4 + 4);  // LDS.128 rows + over-read
  return (size_t)(((p.kh * p.kw + 3) & ~3) + 2 * (int64_t)p.dx_r * p.dx_c) * sizeof(float);
}

}  // namespace

int conv2d_backward_filter_ctas(int sms) { return 4 * sms; }

size_t conv2d_backward_filter_workspace(int64_t taps, int ctas) { return (size_t)taps * ctas * sizeof(double); }

cudaError_t launch_conv2d_backward_input(Conv2DBwdParams& p, cudaStream_t stream, int sms) {
  const size_t smem = dx_smem(p);
  const int64_t ntiles = p.planes * ((p.H + kDxTileH - 1) / kDxTileH) * ((p.W + kDxTileW - 1) / kDxTileW);
  if (smem <= kC2bSmemMax) {
    const bool s1 = p.sh == 1 && p.sw == 1;
    auto kfn = !s1                         ? conv2d_bwd_input_tile_kernel<false, 0, 0>
               : (p.kh == 3 && p.kw == 3) ? conv2d_bwd_input_tile_kernel<true, 3, 3>
               : (p.kh == 5 && p.kw == 5) ? conv2d_bwd_input_tile_kernel<true, 5, 5>
               : (p.kh == 7 && p.kw == 7) ? conv2d_bwd_input_tile_kernel<true, 7, 7>
                                          : conv2d_bwd_input_tile_kernel<true, 0, 0>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kC2bThreads, smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = min(ntiles, (int64_t)sms * (per_sm > 0 ? per_sm : 1));
    kfn<<<(unsigned)grid, kC2bThreads, smem, stream>>>(p);
  } else {
    const int64_t total = p.planes * p.H * p.W;
    const int64_t grid = min((total + kC2bThreads - 1) / kC2bThreads, (int64_t)sms * 8);
    conv2d_bwd_input_direct_kernel<<<(unsigned)grid, kC2bThreads, 0, stream>>>(p);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv2d_backward_filter(Conv2DBwdParams& p, float* df, void* workspace, int ctas,
                                          cudaStream_t stream) {
  double* part = static_cast<double*>(workspace);
  const int64_t nt = p.kh * p.kw;
  if (p.sh == 1 && p.sw == 1 && conv2d_df_tile_supported((int)p.kh, (int)p.kw, p.H, p.W, p.OH, p.OW, p.x, p.dy)) {
    // stride-1 3x3 / 5x5 / 7x7 with TMA-able x rows: the tile kernel (conv2d_tile.cu)
    Conv2DTileParams t;
    memset(&t, 0, sizeof t);
    t.x = p.x; t.planes = p.planes;
    t.IH = (int)p.H; t.IW = (int)p.W; t.OH = (int)p.OH; t.OW = (int)p.OW; t.KH = (int)p.kh; t.KW = (int)p.kw;
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    sms = num_sms(dev);
    const int g = sms <= ctas ? launch_conv2d_df_tile(t, p.dy, part, sms, stream) : -1;
    if (g > 0) {
      conv2d_bwd_filter_finish<<<(unsigned)((nt + 3) / 4), 128, 0, stream>>>(part, g, nt, df);
      note_launch();
      return cudaGetLastError();
    }
  }
  p.df_xr = (int)((kDfTileR - 1) * p.sh + p.kh);
  p.df_xc = (int)(((kDfTileC - 1) * p.sw + p.kw + 3) / 4 * 4 + 4);  // LDS.128 rows + over-read
  const size_t tile_bytes = 2 * ((size_t)kDfTileR * kDfTileC + (size_t)p.df_xr * p.df_xc) * sizeof(float);
  const int64_t ntiles = p.planes * ((p.OH + kDfTileR - 1) / kDfTileR) * ((p.OW + kDfTileC - 1) / kDfTileC);
  const int grid = (int)min((int64_t)ctas, ntiles);
  cudaError_t e = cudaSuccess;
  auto reg = [&](auto kfn, int T) {
    const size_t smem = tile_bytes + (size_t)(kC2bThreads / 32) * T * sizeof(double);
    cudaError_t err = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
    if (err == cudaSuccess) kfn<<<(unsigned)grid, kC2bThreads, smem, stream>>>(p, part);
    return err;
  };
  const bool fits = tile_bytes + 8 * 64 * sizeof(double) <= kC2bSmemMax;
  if (fits && p.kh == 3 && p.kw == 3) {
    e = reg(conv2d_bwd_filter_reg_kernel<3, 3, true>, 9);
  } else if (fits && p.kh == 5 && p.kw == 5) {
    e = reg(conv2d_bwd_filter_reg_kernel<5, 5, true>, 25);
  } else if (fits && p.kh == 7 && p.kw == 7) {
    e = reg(conv2d_bwd_filter_reg_kernel<7, 7, true>, 49);
  } else if (fits && p.kh <= 4 && p.kw <= 4) {
    e = reg(conv2d_bwd_filter_reg_kernel<4, 4, false>, 16);
  } else if (tile_bytes + (size_t)((nt + 3) & ~3) * sizeof(double) <= kC2bSmemMax) {
    const size_t smem = tile_bytes + (size_t)((nt + 3) & ~3) * sizeof(double);
    e = ensure_smem_attr(reinterpret_cast<const void*>(conv2d_bwd_filter_tap_kernel));
    if (e == cudaSuccess) conv2d_bwd_filter_tap_kernel<<<(unsigned)grid, kC2bThreads, smem, stream>>>(p, part);
  } else {
    conv2d_bwd_filter_direct_kernel<<<dim3((unsigned)grid, (unsigned)nt), kC2bThreads, 0, stream>>>(p, part);
  }
  if (e != cudaSuccess) return e;
  note_launch();
  conv2d_bwd_filter_finish<<<(unsigned)((nt + 3) / 4), 128, 0, stream>>>(part, grid, nt, df);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ss
