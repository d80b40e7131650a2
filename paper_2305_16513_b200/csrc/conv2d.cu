// conv2d.cu -- the multi-dimensional extension of the
// sliding dot product (Sec. 2.5) to single-channel 2-D filters (SURVEY 8f
// NEXT #4 "2-D convolution"): y[p][r][c] = sum_a sum_b f[a][b] x[p][r sh+a][c sw+b]
// (cross-correlation, valid padding; reading R17).
//
// Vector kernel (3x3, 5x5, 7x7, 1x3, 3x1; SH, SW in {1, 2}; plane <= 100 KB,
// 16-B aligned rows): the pool2d_vec skeleton -- warp-specialised, one
// cp.async.bulk per plane into a 3-stage ring, 15 consumer warps each owning a
// band of output rows; lane t owns VO = 4/SW consecutive output columns of a
// 128-column strip and keeps the last KH input-row fragments (4 + KW - SW
// floats each, LDS.128 loads) in a register ring, so every input element is
// read from shared memory once per row it feeds (stride-2 rows reload the ring
// per output row).  Taps sit in the parameter
// constant bank (uniform FMA operands); each output's KH*KW products are
// accumulated in row-major tap order.  Everything else: a direct kernel (one
// output per thread, same tap order).
#include <cstdint>

#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kC2Warps = 15;
constexpr int kC2Threads = (kC2Warps + 1) * 32;

__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

}  // namespace

template <int KH, int KW, int SH, int SW>
__global__ void __launch_bounds__(kC2Threads, 1) conv2d_vec_kernel(const __grid_constant__ Conv2DParams p) {
  constexpr int VO = 4 / SW;        // output columns per lane
  constexpr int NF = 4 + KW - SW;   // input columns per lane fragment
  constexpr int NL = (NF + 3) / 4;  // LDS.128 per fragment
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
  uint64_t* empty = full + S;
  int64_t* pid = reinterpret_cast<int64_t*>(empty + S);  // plane of each stage (-1: no more)
  __shared__ ClcSmem clc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kC2Warps);
    }
    clc_init(&clc);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t plane_elems = p.H * p.W;
  const uint32_t plane_bytes = (uint32_t)(plane_elems * 4);
  if (warp == kC2Warps) {  // producer
    if (lane == 0) plane_producer(p.planes, p.clc, &clc, S, full, empty, pid, [&](int64_t pl, int s) {
      mbar_arrive_expect_tx(&full[s], plane_bytes);
      bulk_load_1d(smem + (size_t)s * p.stage_bytes, p.x + pl * plane_elems, plane_bytes, &full[s]);
    });
    return;
  }
  const int OH = (int)p.OH, OW = (int)p.OW;
  const int rows_per = (OH + kC2Warps - 1) / kC2Warps;
  const int ra = warp * rows_per, rb = min(ra + rows_per, OH);
  const uint32_t W4 = (uint32_t)p.W * 4u;
  const uint32_t smem_s = smem_u32(smem);
  for (int it = 0;; ++it) {
    const int s = it % S;
    mbar_wait(&full[s], (uint32_t)(it / S) & 1u);
    const int64_t pl = *reinterpret_cast<volatile int64_t*>(pid + s);
    if (pl < 0) break;
    const uint32_t xs = smem_s + (uint32_t)s * p.stage_bytes;
    float* yp = p.y + pl * (int64_t)OH * OW;
    for (int c0 = VO * lane; c0 < OW; c0 += 32 * VO) {
      const uint32_t colb = (uint32_t)(c0 * SW) * 4u;
      auto frag = [&](uint32_t a, float (&f)[NF]) {
#pragma unroll
        for (int l = 0; l < NL; ++l) {
          const float4 v = lds4(a + 16u * l);
          if (4 * l + 0 < NF) f[4 * l + 0] = v.x;
          if (4 * l + 1 < NF) f[4 * l + 1] = v.y;
          if (4 * l + 2 < NF) f[4 * l + 2] = v.z;
          if (4 * l + 3 < NF) f[4 * l + 3] = v.w;
        }
      };
      float ring[KH][NF];
      const bool vec_ok = c0 + VO <= OW && ((reinterpret_cast<uintptr_t>(yp + c0) & 7) == 0) && ((OW & 1) == 0);
      auto emit = [&](int r, int ph) {  // output row r from ring rows ph, ph+1, ... (mod KH)
        float out[VO];
#pragma unroll
        for (int o = 0; o < VO; ++o) {
          float acc = 0.0f;
#pragma unroll
          for (int a = 0; a < KH; ++a)
#pragma unroll
            for (int b = 0; b < KW; ++b) acc = __fmaf_rn(p.taps[a * KW + b], ring[(ph + a) % KH][o * SW + b], acc);
          out[o] = acc;
        }
        float* yr = yp + (int64_t)r * OW + c0;
        if (vec_ok) {
#pragma unroll
          for (int o = 0; o < VO; o += 2)
            asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(yr + o), "f"(out[o]), "f"(out[o + 1]) : "memory");
        } else {
#pragma unroll
          for (int o = 0; o < VO; ++o)
            if (c0 + o < OW) yr[o] = out[o];
        }
      };
      int r = ra;
      if (r >= rb) continue;
      const uint32_t abase = xs + colb;
      if constexpr (SH == 1) {
        // ring shifted by one row per output row (a KH-fold unrolled, move-free
        // rotation measured no faster and spills at 7x7)
        uint32_t arow = abase + (uint32_t)r * W4;
        float* yr = yp + (int64_t)r * OW + c0;
#pragma unroll
        for (int i = 0; i < KH - 1; ++i) frag(arow + (uint32_t)i * W4, ring[i + 1]);
        for (; r < rb; ++r, arow += W4, yr += OW) {
#pragma unroll
          for (int i = 0; i < KH - 1; ++i)
#pragma unroll
            for (int j = 0; j < NF; ++j) ring[i][j] = ring[i + 1][j];
          frag(arow + (uint32_t)(KH - 1) * W4, ring[KH - 1]);
          float out[VO];
#pragma unroll
          for (int o = 0; o < VO; ++o) {
            float acc = 0.0f;
#pragma unroll
            for (int a = 0; a < KH; ++a)
#pragma unroll
              for (int b = 0; b < KW; ++b) acc = __fmaf_rn(p.taps[a * KW + b], ring[a][o * SW + b], acc);
            out[o] = acc;
          }
          if (vec_ok) {
#pragma unroll
            for (int o = 0; o < VO; o += 2)
              asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(yr + o), "f"(out[o]), "f"(out[o + 1]) : "memory");
          } else {
#pragma unroll
            for (int o = 0; o < VO; ++o)
              if (c0 + o < OW) yr[o] = out[o];
          }
        }
      } else {
        // stride SH > 1: refill the whole ring per output row (KH rows)
        for (; r < rb; ++r) {
#pragma unroll
          for (int i = 0; i < KH; ++i) frag(abase + (uint32_t)(r * SH + i) * W4, ring[i]);
          emit(r, 0);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

__global__ void __launch_bounds__(256) conv2d_direct_kernel(const __grid_constant__ Conv2DParams p) {
  const int64_t total = p.planes * p.OH * p.OW;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = o % p.OW, t = o / p.OW, r = t % p.OH, pl = t / p.OH;
    const float* xp = p.x + (pl * p.H + r * p.sh) * p.W + c * p.sw;
    float acc = 0.0f;
    for (int64_t a = 0; a < p.kh; ++a)
      for (int64_t b = 0; b < p.kw; ++b) acc = __fmaf_rn(p.taps[a * p.kw + b], __ldg(xp + a * p.W + b), acc);
    p.y[o] = acc;
  }
}

template <int KH, int KW, int SH, int SW>
static cudaError_t launch_vec(Conv2DParams& p, cudaStream_t stream, int grid) {
  p.stage_bytes = (uint32_t)((p.H * p.W * 4 + 32 + 127) / 128 * 128);  // +32: last-lane over-read
  int S = 3;
  while (S > 2 && (size_t)S * p.stage_bytes + 256 > (size_t)kSmemBudget) --S;
  if ((size_t)S * p.stage_bytes + 256 > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  p.stages = S;
  const size_t smem = (size_t)S * p.stage_bytes + 256;
  auto kfn = conv2d_vec_kernel<KH, KW, SH, SW>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  const int64_t g = launch_grid(p.planes, grid, p.clc);
  kfn<<<(unsigned)g, kC2Threads, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv2d(Conv2DParams& p, cudaStream_t stream, int grid) {
  const bool vec = (p.sh == 1 || p.sh == 2) && (p.sw == 1 || p.sw == 2) &&
                   ((reinterpret_cast<uintptr_t>(p.x) & 15) == 0) && (p.W % 4) == 0 &&
                   p.H * p.W * 4 + 32 <= 100 * 1024;
  if (vec) {
    cudaError_t e = cudaErrorInvalidValue;
#define SS_C2(KH_, KW_)                                                                       \
  if (p.kh == KH_ && p.kw == KW_)                                                             \
    e = p.sh == 1 ? (p.sw == 1 ? launch_vec<KH_, KW_, 1, 1>(p, stream, grid)                   \
                               : launch_vec<KH_, KW_, 1, 2>(p, stream, grid))                  \
                  : (p.sw == 1 ? launch_vec<KH_, KW_, 2, 1>(p, stream, grid)                   \
                               : launch_vec<KH_, KW_, 2, 2>(p, stream, grid));
    SS_C2(3, 3) else SS_C2(5, 5) else SS_C2(7, 7) else SS_C2(1, 3) else SS_C2(3, 1)
#undef SS_C2
    if (e != cudaErrorInvalidValue) return e;
  }
  const int64_t total = p.planes * p.OH * p.OW;
  int64_t g = (total + 255) / 256;
  if (g > (int64_t)grid * 16) g = (int64_t)grid * 16;
  conv2d_direct_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ss
