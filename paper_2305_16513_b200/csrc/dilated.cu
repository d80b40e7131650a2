// dilated.cu -- stride-1 windows with dilation d > 1 (the
// dilated kernels of PAPER.md Fig. 2, l.205): output i covers x[i + j d],
// j < w (Eq. 3's window with gaps; conv: Sec. 2.5's dot product).
//
// Phase decomposition: outputs i = rho (mod d) read only inputs = rho (mod d),
// i.e. phase rho is an ordinary (undilated) sliding window over the sequence
// x_rho[t] = x[rho + t d].  A CTA tile is a contiguous run of kDilR * d *
// floor(256/d) outputs of one row; its input span (tile + (w-1) d) is staged
// in shared memory with cp.async, and thread (rho, tb) evaluates kDilR
// consecutive outputs of phase rho, holding the kDilR + KB - 1 inputs they
// need in registers (one LDS each), so every input is read once per thread
// instead of once per window.  kDilR = 17 (odd) makes the 32 lanes of a warp
// hit 32 distinct banks for every d | 32.  Conv uses the same association as
// the direct kernels (even-tap / odd-tap FMA chains, then one add; zero taps
// past k add exact zeros), so both paths agree bit for bit (up to the sign
// of an exact zero).
#include <cstdint>
#include <type_traits>

#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kDilThreads = 256;
constexpr int kDilR = 17;

struct ConvAcc {};  // marker: sliding dot product

template <class Op, int KB>
__device__ __forceinline__ void eval_run(const float (&xr)[kDilR + KB - 1], const DilatedParams& p,
                                         float (&out)[kDilR]) {
  if constexpr (std::is_same<Op, ConvAcc>::value) {
#pragma unroll
    for (int m = 0; m < kDilR; ++m) {
      float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
      for (int j = 0; j < KB; j += 2) s0 = __fmaf_rn(p.taps[j], xr[m + j], s0);
#pragma unroll
      for (int j = 1; j < KB; j += 2) s1 = __fmaf_rn(p.taps[j], xr[m + j], s1);
      out[m] = __fadd_rn(s0, s1);
    }
  } else {
    // sum / max: windows of exactly w terms (w <= KB), left to right
#pragma unroll
    for (int m = 0; m < kDilR; ++m) {
      float a = xr[m];
#pragma unroll
      for (int j = 1; j < KB; ++j)
        if (j < p.w) a = Op::combine(a, xr[m + j]);
      out[m] = a;
    }
  }
}

}  // namespace

template <class Op, int KB>
__global__ void __launch_bounds__(kDilThreads) dilated_tile_kernel(const __grid_constant__ DilatedParams p) {
  extern __shared__ __align__(16) float dil_smem[];
  const int d = (int)p.d;
  const int tbc = kDilThreads / d;                 // threads (run blocks) per phase
  const int64_t T = (int64_t)kDilR * d * tbc;      // outputs per tile
  const int span = (int)(T + (KB - 1) * d);        // inputs staged per tile (every register read valid)
  const int64_t tiles_per_row = (p.L_int + T - 1) / T;
  const int64_t ntiles = p.batch * tiles_per_row;
  const float* __restrict__ x = static_cast<const float*>(p.x);
  float* __restrict__ y = static_cast<float*>(p.y);
  const int rho = threadIdx.x % d, tb = threadIdx.x / d;
  const bool active = tb < tbc;
  // (row, tile-in-row) cursors advanced by gridDim.x without divisions: ic one tile ahead (issue), cc (compute)
  const int64_t step_b = gridDim.x / tiles_per_row, step_t = gridDim.x - step_b * tiles_per_row;
  int64_t ib = blockIdx.x / tiles_per_row, it = blockIdx.x - ib * tiles_per_row;
  int64_t cb = ib, ct = it;
  auto advance = [&](int64_t& b, int64_t& t) {
    b += step_b;
    t += step_t;
    if (t >= tiles_per_row) { t -= tiles_per_row; ++b; }
  };
  // two stages: tile it+1 streams in while tile it computes
  auto issue = [&](int64_t tile, int st) {
    if (tile < ntiles) {
      const int64_t b = ib;
      const int64_t i0 = it * T;
      advance(ib, it);
      const float* __restrict__ xr = x + b * p.N + i0;
      const int64_t lim = p.N - i0;
      float* s = dil_smem + st * p.stage_floats;
      if ((reinterpret_cast<uintptr_t>(xr) & 15) == 0) {  // 16-B granules (stage_floats % 4 == 0)
        for (int e = 4 * threadIdx.x; e < span; e += 4 * kDilThreads) {
          const int64_t left = lim - e;
          const uint32_t nb = left >= 4 ? 16u : (left > 0 ? 4u * (uint32_t)left : 0u);
          cp_async16(smem_u32(s + e), nb ? xr + e : x, nb);
        }
      } else {
        for (int e = threadIdx.x; e < span; e += kDilThreads)
          cp_async4(smem_u32(s + e), e < lim ? xr + e : x, e < lim ? 4u : 0u);
      }
    }
    cp_async_commit();
  };
  int64_t tile = blockIdx.x;
  issue(tile, 0);
  int st = 0;
  for (; tile < ntiles; tile += gridDim.x) {
    issue(tile + gridDim.x, st ^ 1);
    cp_async_wait<1>();
    __syncthreads();
    float* os = dil_smem + 2 * p.stage_floats;  // output tile staging (coalesced stores)
    const int64_t bq = cb;
    const int64_t iq0 = ct * T;
    advance(cb, ct);
    const int64_t nout = p.L_int - iq0 < T ? p.L_int - iq0 : T;
    if (active) {
      const float* s = dil_smem + st * p.stage_floats;
      const int base = rho + d * kDilR * tb;  // first input of this thread's run
      float xr[kDilR + KB - 1];
      // reads stay below T + (KB - 1) d = span: staged x (or zero past the row end); taps
      // past w are zero (conv) or not combined (sum / max)
      const float* sb = s + base;
#pragma unroll
      for (int q = 0; q < kDilR + KB - 1; ++q) xr[q] = sb[q * d];
      float out[kDilR];
      eval_run<Op, KB>(xr, p, out);
#pragma unroll
      for (int m = 0; m < kDilR; ++m) os[rho + d * (kDilR * tb + m)] = out[m];  // lanes hit distinct banks
    }
    __syncthreads();  // stage st is refilled by the next iteration's issue; os complete
    {
      float* __restrict__ yr = y + bq * p.y_pitch + p.y_off + iq0;
      if ((reinterpret_cast<uintptr_t>(yr) & 15) == 0 && nout == T && (T & 3) == 0) {
        for (int o = 4 * threadIdx.x; o < nout; o += 4 * kDilThreads)
          *reinterpret_cast<float4*>(yr + o) = *reinterpret_cast<const float4*>(os + o);
      } else {
        for (int o = threadIdx.x; o < nout; o += kDilThreads) yr[o] = os[o];
      }
    }
    st ^= 1;
  }
  cp_async_wait<0>();
}

template <class Op>
static cudaError_t launch_op(DilatedParams& p, cudaStream_t stream, int sms) {
  const int kb = p.w <= 8 ? 8 : (p.w <= 16 ? 16 : 32);
  const int tbc = kDilThreads / (int)p.d;
  const int64_t T = (int64_t)kDilR * p.d * tbc;
  p.stage_floats = (int)((T + (kb - 1) * p.d + 3) & ~int64_t(3));
  const size_t smem = (2 * (size_t)p.stage_floats + (size_t)T) * sizeof(float);
  if (smem > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  const int64_t tiles = p.batch * ((p.L_int + T - 1) / T);
  const int64_t cap = (int64_t)sms * 4;
  const unsigned g = (unsigned)(tiles < cap ? (tiles < 1 ? 1 : tiles) : cap);
  auto kfn = kb == 8 ? dilated_tile_kernel<Op, 8> : (kb == 16 ? dilated_tile_kernel<Op, 16>
                                                               : dilated_tile_kernel<Op, 32>);
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  kfn<<<g, kDilThreads, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_dilated(DilatedParams& p, int op, cudaStream_t stream, int sms) {
  if (p.d < 2 || p.d > kDilThreads || p.w < 1 || p.w > 32 || p.L_int < 1) return cudaErrorInvalidConfiguration;
  if (op == kOpConv) {
    for (int64_t j = p.w; j < 32; ++j) p.taps[j] = 0.0f;
    return launch_op<ConvAcc>(p, stream, sms);
  }
  if (op == kOpSum) return launch_op<OpSumF32>(p, stream, sms);
  if (op == kOpMin) return launch_op<OpMinF32>(p, stream, sms);
  return launch_op<OpMaxF32>(p, stream, sms);
}

}  // namespace ss
