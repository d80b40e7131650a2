// pool2d.cu -- separable 2-D pooling (PAPER.md l.53 operators, l.226
// multi-dimensional extension): a row sliding (+) over kw at stride sw, then a
// column sliding (+) over kh at stride sh, fused on chip (the row results of a
// column never leave registers).
//
// Skeleton: persistent CTAs walk tiles = (plane, band of output rows).  The
// band's input rows are one contiguous byte range of the NCHW tensor, staged
// HBM -> smem with one cp.async.bulk (1-D TMA) per tile into a ring of stages
// (mbarrier completion).  Threads own output columns; each thread walks its
// rows down the band keeping the last KH row results in a register ring
// (stride-1 columns) so each input element is read from smem once per window
// column it belongs to.  Outputs are written with coalesced stores.
#include <cstdint>
#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

constexpr int kP2Threads = 256;

struct AvgOp {  // window sum, scaled at the end
  using T = float;
  static __device__ __forceinline__ float identity() { return 0.0f; }
  static __device__ __forceinline__ float combine(float a, float b) { return __fadd_rn(a, b); }
};

template <class Op, int KW>
__device__ __forceinline__ float row_result(const float* __restrict__ xs, int64_t c0, int kw) {
  if constexpr (KW > 0) {
    float r = xs[c0];
#pragma unroll
    for (int dc = 1; dc < KW; ++dc) r = Op::combine(r, xs[c0 + dc]);
    return r;
  } else {
    float r = xs[c0];
    for (int dc = 1; dc < kw; ++dc) r = Op::combine(r, xs[c0 + dc]);
    return r;
  }
}

template <class Op, int KH, int KW>
__global__ void __launch_bounds__(kP2Threads)
pool2d_kernel(const __grid_constant__ Pool2DParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int kh = KH > 0 ? KH : (int)p.kh;
  const int kw = KW > 0 ? KW : (int)p.kw;
  const int64_t W = p.W, OW = p.OW;
  // thread -> (column lane, row group)
  const int ncol = OW >= kP2Threads ? kP2Threads : (int)((OW + 31) / 32) * 32;
  const int groups = kP2Threads / ncol;
  const int col_lane = tid % ncol, grp = tid / ncol;

  auto tile_rows = [&](int64_t tau, int64_t& plane, int64_t& r0, int64_t& r1, int64_t& in0,
                       int64_t& nin) {
    plane = tau / p.bands;
    const int64_t band = tau - plane * p.bands;
    r0 = band * p.band_rows;
    r1 = r0 + p.band_rows < p.OH ? r0 + p.band_rows : p.OH;
    in0 = r0 * p.sh;
    nin = (r1 - 1) * p.sh + kh - in0;
  };
  auto issue = [&](int64_t tau, int s) {
    int64_t plane, r0, r1, in0, nin;
    tile_rows(tau, plane, r0, r1, in0, nin);
    const float* src = p.x + (plane * p.H + in0) * W;
    const uint32_t bytes = (uint32_t)(nin * W * 4);
    mbar_arrive_expect_tx(&full[s], bytes);
    bulk_load_1d(smem + (size_t)s * p.stage_bytes, src, bytes, &full[s]);
  };

  // prologue
  if (p.bulk && tid == 0) {
    int k = 0;
    for (int64_t tau = blockIdx.x; tau < p.ntiles && k < S - 1; tau += gridDim.x, ++k) issue(tau, k);
  }
  int it = 0;
  for (int64_t tau = blockIdx.x; tau < p.ntiles; tau += gridDim.x, ++it) {
    const int s = it % S;
    float* xs = reinterpret_cast<float*>(smem + (size_t)s * p.stage_bytes);
    int64_t plane, r0, r1, in0, nin;
    tile_rows(tau, plane, r0, r1, in0, nin);
    if (p.bulk) {
      if (tid == 0) {  // keep S-1 tiles in flight: refill the stage freed last iteration
        const int64_t nxt = tau + (int64_t)(S - 1) * gridDim.x;
        if (nxt < p.ntiles) issue(nxt, (it + S - 1) % S);
      }
      mbar_wait(&full[s], (uint32_t)(it / S) & 1u);
    } else {
      const float* src = p.x + (plane * p.H + in0) * W;
      for (int64_t e = tid; e < nin * W; e += kP2Threads) xs[e] = __ldg(src + e);
      __syncthreads();
    }
    // rows of this band handled by my group
    const int64_t nr = r1 - r0;
    const int64_t per = (nr + groups - 1) / groups;
    const int64_t ra = r0 + grp * per;
    const int64_t rb = ra + per < r1 ? ra + per : r1;
    float* yp = p.y + plane * p.OH * OW;
    for (int64_t c = col_lane; c < OW; c += ncol) {
      const int64_t xc = c * p.sw;
      bool done = false;
      if constexpr (KH > 0) {
        if (p.sh == 1) {  // overlapping row windows: register ring of row results
          float ring[KH];
          int64_t r = ra;
          if (r < rb) {
#pragma unroll
            for (int i = 0; i < KH - 1; ++i) ring[i] = row_result<Op, KW>(xs + (r + i - in0) * W, xc, kw);
          }
          for (; r < rb; ++r) {
            ring[KH - 1] = row_result<Op, KW>(xs + (r + KH - 1 - in0) * W, xc, kw);
            float acc = ring[0];
#pragma unroll
            for (int i = 1; i < KH; ++i) acc = Op::combine(acc, ring[i]);
            if (p.mode == 1) acc = __fmul_rn(acc, p.inv_area);
            yp[r * OW + c] = acc;
#pragma unroll
            for (int i = 0; i < KH - 1; ++i) ring[i] = ring[i + 1];
          }
          done = true;
        }
      }
      if (!done) {
        for (int64_t r = ra; r < rb; ++r) {
          const float* xr = xs + (r * p.sh - in0) * W;
          float acc = row_result<Op, KW>(xr, xc, kw);
          for (int dr = 1; dr < kh; ++dr) acc = Op::combine(acc, row_result<Op, KW>(xr + dr * W, xc, kw));
          if (p.mode == 1) acc = __fmul_rn(acc, p.inv_area);
          yp[r * OW + c] = acc;
        }
      }
    }
    __syncthreads();  // stage s is free for the refill issued next iteration
  }
}

// ---------------------------------------------------------------------------
// Vectorised separable kernel for small compile-time windows (KH x KW, stride
// SH x SW with SW in {1,2,4} and KW - SW <= 4; BASELINE config 4 uses 3x3/1
// and 2x2/2).  Warp-specialised: warp kP2VWarps issues one cp.async.bulk per
// plane into a 3-stage ring (full/empty mbarriers); each consumer warp owns a
// band of output rows of the plane; lane t owns VO = 4/SW consecutive output
// columns [VO*t, VO*t+VO) of a 128-column strip, reads the 4 + (KW-SW) input
// columns it needs with one LDS.128 (+ one LDS.64), forms the VO row results,
// and keeps the last KH row results per column in a register ring: the
// column pass costs KH-1 (+) per output and nothing goes back to HBM but y.
constexpr int kP2VWarps = 15;
constexpr int kP2VThreads = (kP2VWarps + 1) * 32;

template <class Op, int KH, int KW, int SH, int SW>
__global__ void __launch_bounds__(kP2VThreads, 1)
pool2d_vec_kernel(const __grid_constant__ Pool2DParams p) {
  constexpr int VO = 4 / SW;        // output columns per lane
  constexpr int XE = KW - SW;       // extra input columns past the lane's 4
  static_assert(XE >= 0 && XE <= 4, "window shape");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) &
                                             ~uintptr_t(127));
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
  uint64_t* empty = full + S;
  int64_t* pid = reinterpret_cast<int64_t*>(empty + S);  // plane of each stage (-1: no more)
  __shared__ ClcSmem clc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kP2VWarps);
    }
    clc_init(&clc);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t W = p.W, OW = p.OW, OH = p.OH, plane_elems = p.H * p.W;
  const uint32_t plane_bytes = (uint32_t)(plane_elems * 4);

  if (warp == kP2VWarps) {  // producer
    if (lane == 0) plane_producer(p.planes, p.clc, &clc, S, full, empty, pid, [&](int64_t pl, int s) {
      mbar_arrive_expect_tx(&full[s], plane_bytes);
      bulk_load_1d(smem + (size_t)s * p.stage_bytes, p.x + pl * plane_elems, plane_bytes, &full[s]);
    });
    return;
  }

  // consumers: warp -> band of output rows
  const int64_t rows_per = (OH + kP2VWarps - 1) / kP2VWarps;
  const int64_t ra = warp * rows_per;
  const int64_t rb = ra + rows_per < OH ? ra + rows_per : OH;
  const uint32_t smem_s = smem_u32(smem);
  for (int it = 0;; ++it) {
    const int s = it % S;
    mbar_wait(&full[s], (uint32_t)(it / S) & 1u);
    const int64_t pl = *reinterpret_cast<volatile int64_t*>(pid + s);
    if (pl < 0) break;
    const uint32_t xs = smem_s + (uint32_t)s * p.stage_bytes;
    float* yp = p.y + pl * OH * OW;
    const uint32_t W4 = (uint32_t)W * 4u;  // smem row pitch (plane <= 100 KB: 32-bit offsets)
    const int OWi = (int)OW;
    for (int c0 = VO * lane; c0 < OWi; c0 += 32 * VO) {  // 128-input-column strips
      const uint32_t colb = (uint32_t)(c0 * SW) * 4u;  // byte offset of the lane's first input column
      auto row_res = [&](uint32_t a, float (&rr)[VO]) {  // a: smem address of the row's 1st input
        float x[4 + XE];
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]) : "r"(a));
        if constexpr (XE > 0) {
          float e[4];
          if constexpr (XE <= 2) {
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(e[0]), "=f"(e[1]) : "r"(a + 16));
          } else {
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(e[0]), "=f"(e[1]), "=f"(e[2]), "=f"(e[3]) : "r"(a + 16));
          }
#pragma unroll
          for (int i = 0; i < XE; ++i) x[4 + i] = e[i];
        }
#pragma unroll
        for (int o = 0; o < VO; ++o) {
          float r = x[o * SW];
#pragma unroll
          for (int d = 1; d < KW; ++d) r = Op::combine(r, x[o * SW + d]);
          rr[o] = r;
        }
      };
      float ring[KH][VO];
      int r = (int)ra;
      uint32_t arow = xs + (uint32_t)(r * SH) * W4 + colb;  // input row r*SH, my columns
      float* yr = yp + (int64_t)r * OW + c0;
      const bool vec_ok = c0 + VO <= OWi && ((reinterpret_cast<uintptr_t>(yp + c0) & 7) == 0) &&
                          ((OW & 1) == 0);
      if (r < (int)rb) {
#pragma unroll
        for (int i = 0; i < KH - SH; ++i) row_res(arow + (uint32_t)i * W4, ring[i + SH]);
      }
      for (; r < (int)rb; ++r, arow += SH * W4, yr += OW) {
#pragma unroll
        for (int i = 0; i < KH - SH; ++i)  // slide the ring by SH rows
#pragma unroll
          for (int o = 0; o < VO; ++o) ring[i][o] = ring[i + SH][o];
#pragma unroll
        for (int i = (KH - SH > 0 ? KH - SH : 0); i < KH; ++i) row_res(arow + (uint32_t)i * W4, ring[i]);
        float out[VO];
#pragma unroll
        for (int o = 0; o < VO; ++o) {
          float acc = ring[0][o];
#pragma unroll
          for (int i = 1; i < KH; ++i) acc = Op::combine(acc, ring[i][o]);
          out[o] = p.mode == 1 ? __fmul_rn(acc, p.inv_area) : acc;
        }
        if (vec_ok) {
#pragma unroll
          for (int o = 0; o < VO; o += 2)
            asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(yr + o), "f"(out[o]), "f"(out[o + 1])
                         : "memory");
        } else {
#pragma unroll
          for (int o = 0; o < VO; ++o)
            if (c0 + o < OWi) yr[o] = out[o];
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

template <class Op>
static cudaError_t launch_op(Pool2DParams& p, cudaStream_t stream, int grid, size_t smem) {
  auto go = [&](auto kfn) -> cudaError_t {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
    if (e != cudaSuccess) return e;
    int64_t g = p.ntiles < grid ? p.ntiles : grid;
    kfn<<<(unsigned)(g < 1 ? 1 : g), kP2Threads, smem, stream>>>(p);
    note_launch();
    return cudaGetLastError();
  };
  if (p.kh == 3 && p.kw == 3) return go(pool2d_kernel<Op, 3, 3>);
  if (p.kh == 2 && p.kw == 2) return go(pool2d_kernel<Op, 2, 2>);
  return go(pool2d_kernel<Op, 0, 0>);
}

template <class Op, int KH, int KW, int SH, int SW>
static cudaError_t launch_vec(Pool2DParams& p, cudaStream_t stream, int grid) {
  p.stage_bytes = (uint32_t)((p.H * p.W * 4 + 16 + 127) / 128 * 128);  // +16: last-lane over-read
  int S = 3;
  while (S > 2 && (size_t)S * p.stage_bytes + 256 > (size_t)kSmemBudget) --S;
  if ((size_t)S * p.stage_bytes + 256 > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  p.stages = S;
  const size_t smem = (size_t)S * p.stage_bytes + 256;
  auto kfn = pool2d_vec_kernel<Op, KH, KW, SH, SW>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  const int64_t g = launch_grid(p.planes, grid, p.clc);
  kfn<<<(unsigned)g, kP2VThreads, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pool2d(Pool2DParams& p, cudaStream_t stream, int grid) {
  // fast vectorised path: whole plane per stage, 16-B aligned rows, known window
  if (p.bulk && (p.H * p.W * 4) % 16 == 0 && p.H * p.W * 4 + 16 <= 100 * 1024) {
    cudaError_t e = cudaErrorInvalidValue;
    const bool avg = p.mode == 1;
    if (p.kh == 3 && p.kw == 3 && p.sh == 1 && p.sw == 1)
      e = avg ? launch_vec<AvgOp, 3, 3, 1, 1>(p, stream, grid) : launch_vec<OpMaxF32, 3, 3, 1, 1>(p, stream, grid);
    else if (p.kh == 2 && p.kw == 2 && p.sh == 2 && p.sw == 2)
      e = avg ? launch_vec<AvgOp, 2, 2, 2, 2>(p, stream, grid) : launch_vec<OpMaxF32, 2, 2, 2, 2>(p, stream, grid);
    if (e != cudaErrorInvalidValue) return e;
  }
  // band size: keep a stage <= 64 KB
  const int64_t row_bytes = p.W * 4;
  int64_t max_in_rows = (64 * 1024) / row_bytes;
  if (max_in_rows < p.kh) max_in_rows = p.kh;
  int64_t band_rows = (max_in_rows - p.kh) / p.sh + 1;
  if (band_rows > p.OH) band_rows = p.OH;
  if (band_rows < 1) band_rows = 1;
  p.band_rows = band_rows;
  p.bands = (p.OH + band_rows - 1) / band_rows;
  p.ntiles = p.planes * p.bands;
  const int64_t in_rows = (band_rows - 1) * p.sh + p.kh;
  p.stage_bytes = (uint32_t)(((in_rows * row_bytes) + 127) / 128 * 128);
  int S = 4;
  while (S > 1 && (size_t)S * p.stage_bytes + 256 > (size_t)kSmemBudget) --S;
  if ((size_t)S * p.stage_bytes + 256 > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  if (!p.bulk) S = 1;
  p.stages = S;
  const size_t smem = (size_t)S * p.stage_bytes + 256;
  if (p.mode == 0) return launch_op<OpMaxF32>(p, stream, grid, smem);
  return launch_op<AvgOp>(p, stream, grid, smem);
}

}  // namespace ss
