// conv2d_tile.cu -- stride-1 2-D sliding dot product on FFMA2 (SURVEY 8f NEXT #4:
// the Conclusion's multi-dimensional extension, of the Sec. 2.5
// dot product; readings R17, R21):
//
//     y[p][r][c] = sum_{a<KH} sum_{b<KW} f[a][b] * xp[p][r + a][c + b]
//
// where xp is the input plane with `pad_t` / `pad_l` zero rows / columns in
// front (and as many behind as the output needs).  pad = 0 is ss_conv2d's
// valid correlation; pad = (KH-1, KW-1) with the flipped filter is the input
// gradient dx of ss_conv2d_backward_input (the full correlation of dy).
//
// * Staging, TMA mode (16-B row pitch): one TMA tensor copy per plane lands a
//   zero-bordered tile of row pitch P = 4 mod 8 floats (the 8 lanes of an
//   LDS.128 phase -- 8 consecutive rows -- hit 8 distinct bank groups; the
//   box's first column must be 16-B aligned, so the left padding is rounded
//   up to 4 and the output shifts by the difference).  Dense mode (other even
//   row widths, e.g. dy of 106 / 110 columns): one bulk copy of the dense
//   plane; a lane then reads its rows with LDS.64 (row pitch = 8 x odd bytes:
//   16 consecutive rows hit 16 distinct 8-B slots) and masks the padding
//   itself.  (A relayout of dense planes into padded tiles by two warps, and
//   per-row cp.async by one warp, were built and measured slower: staging
//   latency, not bandwidth, bound them.)  Planes are claimed by cluster launch
//   control.
// * Work unit: 16 consecutive output rows x 16 consecutive columns; a half
//   warp per unit, lane = output row.  Units are dealt round robin to the 15
//   consumer warps across plane boundaries (two per warp at a time), so no
//   warp idles at the end of a plane.
// * Arithmetic: per filter row a the lane gets the 24 input columns it needs
//   (12 register pairs E) and applies every tap with FFMA2 on output pairs:
//   even taps b act on pairs (2i, 2i+1) -> E[i + b/2], odd taps on pairs
//   (2i-1, 2i) -> E[i + (b-1)/2]; both operands are aligned register pairs.
//   y = fl(S_even + S_odd): S_even sums the even-b taps, S_odd the odd-b taps,
//   each in row-major tap order, so every output's association depends on
//   (a, b) only (tiling independent, deterministic).
// * Store: the lane's 16 outputs are one 64-B row segment (STG.128 where the
//   row is 16-B aligned, else STG.64 + STG.128 x 3 + STG.64).
#include <cstdint>

#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kTWarps = 15;                    // consumer warps
constexpr int kTThreads = (kTWarps + 1) * 32;  // + the producer warp
constexpr int kUnit = 16;                      // unit = 16 rows x 16 columns

__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

}  // namespace

template <int KH, int KW, bool TMA>
__global__ void __launch_bounds__(kTThreads, 1) conv2d_tile_kernel(const __grid_constant__ Conv2DTileParams p) {
  static_assert(KW <= 8 && KH <= 8, "a lane's fragment is 24 columns");
  constexpr int NE = (kUnit + KW + 3) / 4 * 2;  // register pairs per fragment
  constexpr int NL = NE / 2;                    // LDS.128 per fragment (TMA mode)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int ST = p.tile_stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)ST * p.tile_bytes);
  uint64_t* empty = full + ST;
  int64_t* pid = reinterpret_cast<int64_t*>(empty + ST);  // plane of each stage (-1: no more)
  __shared__ ClcSmem clc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTWarps);
    }
    clc_init(&clc);
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t smem_s = smem_u32(smem);
  const int P = p.P;

  if (warp == kTWarps) {
    // ---------------- producer lane: one TMA tensor copy (padded tile) or one bulk copy
    // (dense plane) per plane
    if (lane == 0) {
      if (TMA) prefetch_tmap(&p.tm_x);
      int64_t u = blockIdx.x;
      uint32_t cph = 0;
      if (p.clc && u < p.planes) clc_request(&clc);
      const uint32_t dense_bytes = (uint32_t)((int64_t)p.IH * p.IW * 4);
      for (int it = 0;; ++it) {
        const int st = it % ST;
        mbar_wait_poll(&empty[st], ((uint32_t)(it / ST) & 1u) ^ 1u);
        if (u < 0 || u >= p.planes) {
          pid[st] = -1;
          mbar_arrive(&full[st]);
          break;
        }
        pid[st] = u;
        if (TMA) {
          mbar_arrive_expect_tx(&full[st], p.tile_tx);
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_s + (uint32_t)st * p.tile_bytes),
              "l"(reinterpret_cast<uint64_t>(&p.tm_x)), "r"(-p.pad_c), "r"(-p.pad_t), "r"((int32_t)u),
              "r"(smem_u32(&full[st]))
              : "memory");
        } else {
          mbar_arrive_expect_tx(&full[st], dense_bytes);
          bulk_load_1d(smem + (size_t)st * p.tile_bytes, p.x + u * (int64_t)p.IH * p.IW, dense_bytes, &full[st]);
        }
        if (p.clc) {
          u = clc_wait(&clc, cph);  // requested one plane ahead
          if (u >= 0) clc_request(&clc);
        } else {
          u += gridDim.x;
        }
      }
    }
    return;
  }

  // ---------------- consumers
  const int OH = p.OH, OW = p.OW, IH = p.IH, IW = p.IW;
  const int units = p.units;            // per plane
  const int pairs = (units + 1) >> 1;   // warp units per plane
  const int half = lane >> 4, row16 = lane & 15;
  int cur = -1;                         // plane iteration whose stage this warp holds
  int64_t plane = 0;
  bool done = false;
  for (int64_t g = warp; !done; g += kTWarps) {
    const int64_t it = g / pairs;
    const int q = (int)(g - it * pairs);
    while (cur < it) {
      if (cur >= 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cur % ST]);
      }
      ++cur;
      mbar_wait_poll(&full[cur % ST], (uint32_t)(cur / ST) & 1u);
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(plane) : "r"(smem_u32(pid + cur % ST)) : "memory");
      if (plane < 0) {
        done = true;
        break;
      }
    }
    if (done) break;
    const int un = 2 * q + half;
    if (un >= units) continue;
    const int rg = un / p.col_blocks, cb = un - rg * p.col_blocks;
    const int r = rg * kUnit + row16;
    if (r >= OH) continue;
    const uint32_t stage_s = smem_s + (uint32_t)(cur % ST) * p.tile_bytes;
    // dense mode: fragment columns = input columns c_in .. c_in + 2 NE; interior blocks skip the masks
    const int c_in = cb * kUnit - p.pad_l;
    const bool interior = c_in >= 0 && c_in + 2 * NE <= IW;
    float2 A0[kUnit / 2], A1[kUnit / 2 + 1];  // A0[i]: outputs (2i, 2i+1); A1[i]: (2i-1, 2i)
#pragma unroll
    for (int i = 0; i < kUnit / 2; ++i) A0[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i <= kUnit / 2; ++i) A1[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int a = 0; a < KH; ++a) {
      float2 E[NE];
      if (TMA) {
        const uint32_t base = stage_s + (uint32_t)((r + a) * P + cb * kUnit) * 4u;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const float4 v = lds128(base + 16u * l);
          E[2 * l] = make_float2(v.x, v.y);
          E[2 * l + 1] = make_float2(v.z, v.w);
        }
      } else {
        const int i = r + a - p.pad_t;  // input row
        const bool rv = (unsigned)i < (unsigned)IH;
        const uint32_t base = stage_s + (uint32_t)(i * IW + c_in) * 4u;
        if (interior) {
#pragma unroll
          for (int m = 0; m < NE; ++m) E[m] = rv ? lds64(base + 8u * m) : make_float2(0.f, 0.f);
        } else {
#pragma unroll
          for (int m = 0; m < NE; ++m) {
            const int c = c_in + 2 * m;  // pairs (c, c+1) lie wholly inside or outside the row (c, IW even)
            E[m] = (rv && c >= 0 && c < IW) ? lds64(base + 8u * m) : make_float2(0.f, 0.f);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < KW; b += 2) {
        const float f = p.taps[a * KW + b];
#pragma unroll
        for (int i = 0; i < kUnit / 2; ++i) A0[i] = __ffma2_rn(E[i + b / 2], make_float2(f, f), A0[i]);
      }
#pragma unroll
      for (int b = 1; b < KW; b += 2) {
        const float f = p.taps[a * KW + b];
#pragma unroll
        for (int i = 0; i <= kUnit / 2; ++i) A1[i] = __ffma2_rn(E[i + (b - 1) / 2], make_float2(f, f), A1[i]);
      }
    }
    float out[kUnit];
#pragma unroll
    for (int o = 0; o < kUnit; ++o) {
      const float se = (o & 1) ? A0[o >> 1].y : A0[o >> 1].x;
      const float so = (o & 1) ? A1[(o + 1) >> 1].x : A1[o >> 1].y;
      out[o] = __fadd_rn(se, so);
    }
    // tile column t holds output column t - shift (TMA mode's rounded-up left padding)
    const int c0 = cb * kUnit - p.shift;
    float* yrow = p.y + (plane * OH + r) * (int64_t)OW;
    if (c0 < 0) {
#pragma unroll
      for (int o = 0; o < kUnit; ++o)
        if (c0 + o >= 0 && c0 + o < OW) yrow[c0 + o] = out[o];
      continue;
    }
    const int nvalid = OW - c0;
    float* yr = yrow + c0;
    const uintptr_t ya = reinterpret_cast<uintptr_t>(yr);
    if (nvalid >= kUnit && (ya & 15) == 0) {
#pragma unroll
      for (int o = 0; o < kUnit; o += 4)
        asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(yr + o), "f"(out[o]), "f"(out[o + 1]),
                     "f"(out[o + 2]), "f"(out[o + 3])
                     : "memory");
    } else if (nvalid >= kUnit && (ya & 7) == 0) {
      asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(yr), "f"(out[0]), "f"(out[1]) : "memory");
#pragma unroll
      for (int o = 2; o < kUnit - 2; o += 4)
        asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(yr + o), "f"(out[o]), "f"(out[o + 1]),
                     "f"(out[o + 2]), "f"(out[o + 3])
                     : "memory");
      asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(yr + kUnit - 2), "f"(out[kUnit - 2]),
                   "f"(out[kUnit - 1])
                   : "memory");
    } else {
#pragma unroll
      for (int o = 0; o < kUnit; ++o)
        if (o < nvalid) yr[o] = out[o];
    }
  }
}

// Smallest pitch >= need with pitch = 4 (mod 8) floats: 8 consecutive rows of
// an LDS.128 phase start in 8 distinct 16-B bank groups.
static int tile_pitch(int need) {
  int P = (need + 3) / 4 * 4;
  if (P % 8 == 0) P += 4;
  return P;
}

bool conv2d_tile_supported(int kh, int kw, int64_t oh, int64_t ow) {
  if (!((kh == 3 && kw == 3) || (kh == 5 && kw == 5) || (kh == 7 && kw == 7))) return false;
  return oh >= 1 && ow >= 1 && oh <= 4096 && ow <= 4096;
}

cudaError_t launch_conv2d_tile(Conv2DTileParams& p, cudaStream_t stream, int sms) {
  if (!conv2d_tile_supported(p.KH, p.KW, p.OH, p.OW)) return cudaErrorInvalidConfiguration;
  const int TH = p.OH + p.KH - 1;  // rows the outputs read (pad_t + IH + bottom zeros)
  if (TH < p.pad_t + p.IH) return cudaErrorInvalidConfiguration;
  const size_t fixed = 128 + 512;
  size_t smem = 0;
  // TMA mode (16-B row pitch): the box's first column must be 16-B aligned, so the tile's left
  // padding is rounded up to 4 columns and tile column t holds output column t - shift
  if ((p.IW * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(p.x) & 15) == 0) {
    p.pad_c = (p.pad_l + 3) / 4 * 4;
    p.shift = p.pad_c - p.pad_l;
    p.col_blocks = (p.OW + p.shift + kUnit - 1) / kUnit;
    const int need_cols = p.col_blocks * kUnit + (p.KW + 3) / 4 * 4;  // last block reads 16 + KW (+ pad)
    p.P = tile_pitch(need_cols > p.IW + p.pad_c ? need_cols : p.IW + p.pad_c);
    if (p.P <= 256 && TH <= 256 && encode_plane_map(&p.tm_x, p.x, p.IW, p.IH, p.planes, p.P, TH)) {
      p.tma = 1;
      p.tile_tx = (uint32_t)((size_t)TH * p.P * 4);
      p.tile_bytes = (uint32_t)(((size_t)TH * p.P * 4 + 127) / 128 * 128);
    }
  }
  if (!p.tma) {
    // dense mode: the plane as it lies in memory (one bulk copy), padding masked by the lanes; needs
    // 8-B aligned pairs (even row width and left padding) and a 16-B multiple plane
    const int64_t plane_bytes = (int64_t)p.IH * p.IW * 4;
    if (p.IW % 2 || p.pad_l % 2 || (plane_bytes & 15) || (reinterpret_cast<uintptr_t>(p.x) & 15))
      return cudaErrorInvalidConfiguration;
    p.pad_c = p.pad_l;
    p.shift = 0;
    p.col_blocks = (p.OW + kUnit - 1) / kUnit;
    p.P = p.IW;
    p.tile_bytes = (uint32_t)((plane_bytes + 127) / 128 * 128);
  }
  p.units = ((p.OH + kUnit - 1) / kUnit) * p.col_blocks;
  p.tile_stages = 4;
  while (p.tile_stages > 2 && (size_t)p.tile_stages * p.tile_bytes + fixed > (size_t)kSmemBudget) --p.tile_stages;
  smem = (size_t)p.tile_stages * p.tile_bytes + fixed;
  if (smem > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  auto kfn = p.tma ? (p.KH == 3 ? conv2d_tile_kernel<3, 3, true> : p.KH == 5 ? conv2d_tile_kernel<5, 5, true>
                                                                      : conv2d_tile_kernel<7, 7, true>)
                   : (p.KH == 3 ? conv2d_tile_kernel<3, 3, false> : p.KH == 5 ? conv2d_tile_kernel<5, 5, false>
                                                                       : conv2d_tile_kernel<7, 7, false>);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  const int64_t g = launch_grid(p.planes, sms, p.clc);
  kfn<<<(unsigned)g, kTThreads, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Filter gradient of the stride-1 2-D correlation (reading R21):
//     df[a][b] = sum_p sum_r sum_c dy[p][r][c] * x[p][r + a][c + b]
// Same staging and units as above: per plane the x tile arrives by one TMA
// tensor copy (pitch P = 4 mod 8) and the dense dy plane by one bulk copy
// (LDS.64 rows: the dy row pitch is 8 x an odd number of bytes for the
// config-4 shapes, so 16 rows hit 16 distinct 8-B slots).  A lane (dy row r,
// 16 columns) keeps all KH*KW tap sums in fp32 registers (scalar FFMA: the
// FP32 pipe, not issue, bounds it) for 8 units at most (<= 128 products per
// sum), then the warp sums each tap with a butterfly and one lane adds it to
// the warp's fp64 accumulator in shared memory.  Planes are dealt statically
// (CTA b: planes b, b + grid, ...) so the fp64 partials, the fixed-order CTA
// reduction and the finishing kernel's fixed-order sum over CTAs make df
// bitwise deterministic.
namespace {
constexpr int kDfFlush = 8;  // units per lane between fp32 -> fp64 flushes
}

template <int KH, int KW>
__global__ void __launch_bounds__(kTWarps * 32 + 32, 1)
conv2d_df_tile_kernel(const __grid_constant__ Conv2DTileParams p, const float* __restrict__ dy,
                      double* __restrict__ part) {
  constexpr int NT = KH * KW;
  constexpr int NL = (kUnit + KW + 3) / 4;  // LDS.128 per x fragment
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);  // shared-space pointer arithmetic
  const int S = p.tile_stages;
  const uint32_t stage = p.tile_bytes + p.raw_bytes;  // x tile, then the dense dy plane
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage);
  uint64_t* empty = full + S;
  int64_t* pid = reinterpret_cast<int64_t*>(empty + S);
  double* wacc = reinterpret_cast<double*>(pid + S);  // [kTWarps][NT]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kTWarps * NT; i += blockDim.x) wacc[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t smem_s = smem_u32(smem);
  const int OH = p.OH, OW = p.OW, P = p.P;
  const uint32_t dy_bytes = (uint32_t)((int64_t)OH * OW * 4);

  if (warp == kTWarps) {  // producer lane: static plane schedule
    if (lane == 0) {
      prefetch_tmap(&p.tm_x);
      int64_t u = blockIdx.x;
      for (int it = 0;; ++it, u += gridDim.x) {
        const int s = it % S;
        mbar_wait_poll(&empty[s], ((uint32_t)(it / S) & 1u) ^ 1u);
        if (u >= p.planes) {
          pid[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        pid[s] = u;
        mbar_arrive_expect_tx(&full[s], p.tile_tx + dy_bytes);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_s + (uint32_t)s * stage),
            "l"(reinterpret_cast<uint64_t>(&p.tm_x)), "r"(0), "r"(0), "r"((int32_t)u), "r"(smem_u32(&full[s]))
            : "memory");
        bulk_load_1d(smem + (size_t)s * stage + p.tile_bytes, dy + u * (int64_t)OH * OW, dy_bytes, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers
  const int units = p.units, pairs = (units + 1) >> 1;
  const int half = lane >> 4, row16 = lane & 15;
  float acc[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t] = 0.0f;
  auto flush = [&]() {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      float v = acc[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == (t & 31)) wacc[warp * NT + t] += (double)v;
      acc[t] = 0.0f;
    }
  };
  int cur = -1, since = 0;
  bool done = false;
  for (int64_t g = warp; !done; g += kTWarps) {
    const int64_t it = g / pairs;
    const int q = (int)(g - it * pairs);
    while (cur < it) {
      if (cur >= 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cur % S]);
      }
      ++cur;
      mbar_wait_poll(&full[cur % S], (uint32_t)(cur / S) & 1u);
      int64_t plane;
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(plane) : "r"(smem_u32(pid + cur % S)) : "memory");
      if (plane < 0) {
        done = true;
        break;
      }
    }
    if (done) break;
    const int un = 2 * q + half;
    const int rg = un / p.col_blocks, cb = un - rg * p.col_blocks;
    const int r = rg * kUnit + row16;
    if (un < units && r < OH) {
      const uint32_t xs = smem_s + (uint32_t)(cur % S) * stage + (uint32_t)(r * P + cb * kUnit) * 4u;
      const uint32_t ds = smem_s + (uint32_t)(cur % S) * stage + p.tile_bytes + (uint32_t)(r * OW + cb * kUnit) * 4u;
      const int nv = OW - cb * kUnit;  // valid dy columns of this block
      float d[kUnit];
#pragma unroll
      for (int j = 0; j < kUnit; j += 2) {
        float d0 = 0.f, d1 = 0.f;
        if (j < nv) asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(d0), "=f"(d1) : "r"(ds + 4u * j));
        d[j] = d0;
        d[j + 1] = j + 1 < nv ? d1 : 0.f;
      }
#pragma unroll
      for (int a = 0; a < KH; ++a) {
        float xv[4 * NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const float4 v = lds128(xs + (uint32_t)(a * P) * 4u + 16u * l);
          xv[4 * l] = v.x; xv[4 * l + 1] = v.y; xv[4 * l + 2] = v.z; xv[4 * l + 3] = v.w;
        }
#pragma unroll
        for (int b = 0; b < KW; ++b)
#pragma unroll
          for (int j = 0; j < kUnit; ++j) acc[a * KW + b] = __fmaf_rn(d[j], xv[j + b], acc[a * KW + b]);
      }
    }
    if (++since == kDfFlush) {
      flush();
      since = 0;
    }
  }
  flush();
  // fixed-order CTA reduction of the warps' fp64 sums -> this CTA's partial
  asm volatile("bar.sync 1, %0;" ::"r"(kTWarps * 32) : "memory");
  for (int t = threadIdx.x; t < NT; t += kTWarps * 32) {
    double v = 0.0;
    for (int w = 0; w < kTWarps; ++w) v += wacc[w * NT + t];
    part[(int64_t)t * gridDim.x + blockIdx.x] = v;
  }
}

bool conv2d_df_tile_supported(int kh, int kw, int64_t H, int64_t W, int64_t OH, int64_t OW, const void* x,
                              const void* dy) {
  if (!conv2d_tile_supported(kh, kw, OH, OW)) return false;
  return (W * 4) % 16 == 0 && ((OH * OW * 4) % 16) == 0 && (OW % 2) == 0 &&
         (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0 && H <= 256;
}

// Grid (CTAs whose fp64 partials the finishing kernel sums) or -1 if not applicable.
int launch_conv2d_df_tile(Conv2DTileParams& p, const float* dy, double* part, int sms, cudaStream_t stream) {
  p.col_blocks = (p.OW + kUnit - 1) / kUnit;
  p.units = ((p.OH + kUnit - 1) / kUnit) * p.col_blocks;
  const int need_cols = p.col_blocks * kUnit + (p.KW + 3) / 4 * 4;
  p.P = tile_pitch(need_cols > p.IW ? need_cols : p.IW);
  const int TH = p.IH;
  if (p.P > 256 || TH > 256) return -1;
  if (!encode_plane_map(&p.tm_x, p.x, p.IW, p.IH, p.planes, p.P, TH)) return -1;
  p.tile_tx = (uint32_t)((size_t)TH * p.P * 4);
  p.tile_bytes = (uint32_t)(((size_t)TH * p.P * 4 + 127) / 128 * 128);
  p.raw_bytes = (uint32_t)(((size_t)p.OH * p.OW * 4 + 127) / 128 * 128);
  const size_t fixed = 128 + 256 + (size_t)kTWarps * p.KH * p.KW * 8;
  p.tile_stages = 2;
  const size_t smem = (size_t)2 * (p.tile_bytes + p.raw_bytes) + fixed;
  if (smem > (size_t)kSmemBudget) return -1;
  auto kfn = p.KH == 3 ? conv2d_df_tile_kernel<3, 3>
           : p.KH == 5 ? conv2d_df_tile_kernel<5, 5>
                       : conv2d_df_tile_kernel<7, 7>;
  if (ensure_smem_attr(reinterpret_cast<const void*>(kfn)) != cudaSuccess) return -1;
  const int grid = (int)(p.planes < sms ? p.planes : sms);
  kfn<<<(unsigned)grid, kTWarps * 32 + 32, smem, stream>>>(p, dy, part);
  note_launch();
  return grid;
}

}  // namespace ss
