// maxbwd.cu -- stride-1 max-pooling input gradient, TMA-staged tile kernel
// (reading R16):
//   dx_t = sum of dy_i over the windows i whose FIRST maximum (left to right,
//          replaced on strictly greater) is x_t,  windows [i, i+w) of Eq. 3.
//
// A tile is 4096 consecutive windows of one row, i in [iw0, iw0 + 4096), and
// stores dx for the T = 4096 - w - 2 positions [t0, t0 + T) whose windows all
// lie in it (t0 - iw0 >= w - 1).  x and dy arrive by 1-D TMA boxes over the
// flat arrays (OOB zero fill at both ends; iw0 is chosen so x's box start is
// 16-B aligned), two tiles in flight per CTA, two CTAs per SM.  Each thread
// evaluates the first argmax of 16 consecutive windows from registers (Alg. 2's
// pivot split: a suffix scan over its own 16 inputs, one running
// prefix scan over the next w - 1), so a window costs ~2-3 compares.  The
// argmaxes are non-decreasing in i, so dx is a reduce-by-key of dy over sorted
// keys: each thread sums its runs left to right (increasing window order), a
// run that continues into the following threads is completed by the thread
// where it starts from their published head partials, and the owner writes the
// run total into the zeroed dx tile, which leaves by coalesced stores.  No
// atomics: bitwise deterministic.
#include <cstdint>

#include <cuda.h>
#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kMbThreads = 256;                  // compute threads; one more warp issues the TMA loads
constexpr int kMbR = 16;                         // windows per thread
constexpr int kMbWin = kMbThreads * kMbR;        // windows per tile
constexpr int kMbBox = 256;                      // floats per TMA box
constexpr int kMbBoxes = kMbWin / kMbBox + 1;    // boxes per staged array (>= 4096 + 64 + 4 floats)
constexpr int kMbSpan = kMbBoxes * kMbBox;
constexpr int kMbStages = 2;
constexpr int kMbDX = kMbWin + 8;                // dx tile (window-relative positions < 4096)
constexpr size_t kMbSmem = 128 + (size_t)kMbStages * 2 * kMbSpan * 4 + 2 * (size_t)kMbDX * 4 +
                           (size_t)kMbThreads * 16 + 64;

// barrier 1 among the compute warps only (the producer warp never joins)
__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kMbThreads) : "memory"); }

__device__ __forceinline__ void tma_load_1d(void* smem_dst, const CUtensorMap* map, int32_t c0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2}], [%3];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int64_t floor4(int64_t v) { return v >= 0 ? (v & ~int64_t(3)) : -((-v + 3) & ~int64_t(3)); }

}  // namespace

template <int W>
__global__ void __launch_bounds__(kMbThreads + 32, 2) pool_max_backward_s1_kernel(const __grid_constant__ MaxBwdS1Params p) {
  constexpr int R = kMbR;
  extern __shared__ __align__(16) uint8_t mb_raw[];
  // 128-B aligned by pointer arithmetic on the shared array (keeps the shared address space visible
  // to the compiler: plain LDS / STS instead of generic accesses)
  float* ring = reinterpret_cast<float*>(mb_raw + ((128u - (smem_u32(mb_raw) & 127u)) & 127u));
  float* dxs = ring + kMbStages * 2 * kMbSpan;               // [2][kMbDX] (double-buffered)
  int* hk = reinterpret_cast<int*>(dxs + 2 * kMbDX);          // head key of each thread
  float* hs = reinterpret_cast<float*>(hk + kMbThreads);      // head-run partial
  int* tk = reinterpret_cast<int*>(hs + kMbThreads);          // tail key
  int* sg = tk + kMbThreads;                                  // 1: the thread is one run
  uint64_t* full = reinterpret_cast<uint64_t*>(sg + kMbThreads);  // [stages]
  uint64_t* empty = full + kMbStages;                              // [stages]: one arrive per compute warp
  const int tid = threadIdx.x, j0 = tid * R;
  const int64_t N = p.N, L = p.L, tpr = p.tiles_per_row, ntiles = p.ntiles;
  const int T = p.T;
  constexpr int kLow = -(1 << 30), kHigh = 1 << 30;  // sentinel keys of windows outside the row

  if (tid == 0) {
    for (int s = 0; s < kMbStages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, kMbThreads / 32); }
    fence_mbar_init();
    prefetch_tmap(&p.tm_x);
    prefetch_tmap(&p.tm_dy);
  }
  __syncthreads();

  // tile cursor (row b, tile-in-row c): advanced by gridDim.x tiles without divisions
  const int64_t step = gridDim.x, step_b = step / tpr, step_c = step - step_b * tpr;
  auto advance = [&](int64_t& b, int64_t& c) {
    b += step_b;
    c += step_c;
    if (c >= tpr) { c -= tpr; ++b; }
  };
  // window base: b N + iw0 = 0 mod 4 and t0 - iw0 in [w - 1, w + 2]
  auto base = [&](int64_t b, int64_t t0) { return floor4(b * N + t0 - (W - 1)) - b * N; };
  int64_t ib = blockIdx.x / tpr, ic = blockIdx.x - ib * tpr;  // issue cursor (thread 0)
  auto issue = [&](int st) {
    const int64_t t0 = ic * T, iw0 = base(ib, t0);
    const int32_t xa = (int32_t)(ib * N + iw0);
    const int32_t ga = (int32_t)floor4(ib * L + iw0);
    float* xs = ring + st * 2 * kMbSpan;
    float* gs = xs + kMbSpan;
    mbar_arrive_expect_tx(full + st, 2u * kMbSpan * 4u);
#pragma unroll 1
    for (int k = 0; k < kMbBoxes; ++k) {
      tma_load_1d(xs + k * kMbBox, &p.tm_x, xa + k * kMbBox, full + st);
      tma_load_1d(gs + k * kMbBox, &p.tm_dy, ga + k * kMbBox, full + st);
    }
    advance(ib, ic);
  };
  if (tid >= kMbThreads) {  // producer warp: lane 0 refills each stage once the compute warps release it
    if (tid == kMbThreads) {
      for (int k = 0; ib < p.batch; ++k) {
        const int st = k % kMbStages;
        mbar_wait(empty + st, ((uint32_t)(k / kMbStages) & 1u) ^ 1u);
        issue(st);
      }
    }
    return;
  }

  int64_t cb = blockIdx.x / tpr, cc = blockIdx.x - cb * tpr;  // compute cursor
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += step, ++it) {
    const int st = it % kMbStages;
    const int64_t t0 = cc * T, iw0 = base(cb, t0);
    const int64_t b = cb;
    advance(cb, cc);
    const int wpad = (int)(t0 - iw0);  // in [w - 1, w + 2]
    const int nt = (int)(t0 + T <= N ? T : N - t0);
    float* dx_t = dxs + (it & 1) * kMbDX;
#pragma unroll
    for (int m = 0; m < kMbWin / (4 * kMbThreads); ++m)  // the tile starts at zero (16-B stores)
      *reinterpret_cast<float4*>(dx_t + 4 * (tid + m * kMbThreads)) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);

    mbar_wait(full + st, (uint32_t)(it / kMbStages) & 1u);
    const float* xs = ring + st * 2 * kMbSpan;
    const float* gs = xs + kMbSpan;
    const int oy = (int)((b * L + iw0) & 3);

    // (1) first maximum of windows j0 .. j0 + R - 1 (window-relative indices)
    constexpr int NX = (R + W - 1 + 3) & ~3;
    float xv[NX];
#pragma unroll
    for (int q = 0; q < NX / 4; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(xs + j0 + 4 * q);
      xv[4 * q] = v.x; xv[4 * q + 1] = v.y; xv[4 * q + 2] = v.z; xv[4 * q + 3] = v.w;
    }
    int key[R];
    if constexpr (W <= 4) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float m = xv[r];
        int a = r;
#pragma unroll
        for (int q = 1; q < W; ++q) {
          const bool gt = xv[r + q] > m;
          m = gt ? xv[r + q] : m;
          a = gt ? r + q : a;
        }
        key[r] = j0 + a;
      }
    } else {
      // windows r = [r, r + W - 1]: suffix [r, B) of the thread's first block B = min(R, W - 1)... the
      // pivot split with the block of R inputs when W - 1 >= R, else per block of W - 1
      constexpr int B = (W - 1) < R ? (W - 1) : R;  // block length (pivot spacing)
#pragma unroll
      for (int b0 = 0; b0 < R; b0 += B) {
        // windows b0 .. b0 + B - 1: suffix over [r, b0 + B), prefix over [b0 + B, r + W)
        float sv[B];
        int si[B];
        sv[B - 1] = xv[b0 + B - 1];
        si[B - 1] = b0 + B - 1;
#pragma unroll
        for (int r = B - 2; r >= 0; --r) {
          const bool ge = xv[b0 + r] >= sv[r + 1];  // ties: the earlier index
          sv[r] = ge ? xv[b0 + r] : sv[r + 1];
          si[r] = ge ? b0 + r : si[r + 1];
        }
        float pv = -__int_as_float(0x7f800000);
        int pi = b0 + B;
#pragma unroll
        for (int m = b0 + B; m < b0 + W - 1; ++m) {
          const bool gt = xv[m] > pv;
          pv = gt ? xv[m] : pv;
          pi = gt ? m : pi;
        }
#pragma unroll
        for (int r = 0; r < B; ++r) {
          if (b0 + r < R) {
            const int m = b0 + r + W - 1;
            const bool gt = xv[m] > pv;
            pv = gt ? xv[m] : pv;
            pi = gt ? m : pi;
            key[b0 + r] = j0 + (pv > sv[r] ? pi : si[r]);
          }
        }
      }
    }
    // dy of the 16 windows (gs is offset by oy in 0..3 from a 16-B boundary)
    float gv[R];
    {
      float a[R + 4];
#pragma unroll
      for (int q = 0; q < (R + 4) / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(gs + j0 + 4 * q);
        a[4 * q] = v.x; a[4 * q + 1] = v.y; a[4 * q + 2] = v.z; a[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        gv[r] = oy == 0 ? a[r] : oy == 1 ? a[r + 1] : oy == 2 ? a[r + 2] : a[r + 3];
    }
    // windows outside the row (only in a row's first / last tile): sentinel keys, never written
    if (iw0 + j0 < 0 || iw0 + j0 + R > L) {
      const int64_t i0 = iw0 + j0;
#pragma unroll
      for (int r = 0; r < R; ++r) key[r] = i0 + r < 0 ? kLow : (i0 + r >= L ? kHigh : key[r]);
    }
    // (2) runs: head partial, tail (branch-free)
    int cur = key[0];
    float acc = gv[0], head = 0.0f;
    bool single = true;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const bool nb = key[r] != cur;
      head = nb && single ? acc : head;
      single = single && !nb;
      const float sum = __fadd_rn(acc, gv[r]);
      acc = nb ? gv[r] : sum;
      cur = key[r];
    }
    head = single ? acc : head;
    hk[tid] = key[0];
    hs[tid] = head;
    tk[tid] = cur;
    sg[tid] = single ? 1 : 0;
    compute_sync();  // (A) zeroed dx tile, published heads; the stage is consumed
    if ((tid & 31) == 0) {
      fence_proxy_async_smem();  // this warp's generic reads of the stage precede the async refill
      mbar_arrive(empty + st);
    }
    auto put = [&](int k, float v) {
      if ((unsigned)(k - wpad) < (unsigned)nt) dx_t[k] = v;
    };
    auto chain = [&](int k, float total) {
      for (int u = tid + 1; u < kMbThreads && hk[u] == k; ++u) {
        total = __fadd_rn(total, hs[u]);
        if (!sg[u]) break;
      }
      return total;
    };
    // interior runs (complete here), then the head run (if it starts here) and the tail run
    if (!single) {
      int c2 = key[0];
      float a2 = gv[0];
      bool first_run = true;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const bool nb = key[r] != c2;
        if (nb && !first_run && (unsigned)(c2 - wpad) < (unsigned)nt) dx_t[c2] = a2;
        first_run = first_run && !nb;
        const float sum = __fadd_rn(a2, gv[r]);
        a2 = nb ? gv[r] : sum;
        c2 = key[r];
      }
    }
    if (tid == 0 || tk[tid - 1] != key[0]) put(key[0], single ? chain(key[0], head) : head);
    if (!single) put(cur, chain(cur, acc));
    compute_sync();  // (B) dx tile complete
    float* __restrict__ dxr = p.dx + b * N + t0 + tid;
    const float* dsrc = dx_t + wpad + tid;
#pragma unroll
    for (int m = 0; m < kMbWin / kMbThreads; ++m)
      if (tid + m * kMbThreads < nt) dxr[m * kMbThreads] = dsrc[m * kMbThreads];
  }
}

bool pool_max_backward_s1_supported(int64_t w) {
  switch (w) {
    case 2: case 3: case 4: case 5: case 7: case 8: case 9: case 16: case 17: case 32: case 33: case 64: return true;
    default: return false;
  }
}

cudaError_t launch_pool_max_backward_s1(MaxBwdS1Params& p, cudaStream_t stream, int sms) {
  const int w = (int)p.w;
  p.T = kMbWin - w - 2;
  p.tiles_per_row = (p.N + p.T - 1) / p.T;
  p.ntiles = p.batch * p.tiles_per_row;
  const void* kfn = nullptr;
  switch (w) {
    case 2: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<2>); break;
    case 3: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<3>); break;
    case 4: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<4>); break;
    case 5: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<5>); break;
    case 7: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<7>); break;
    case 8: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<8>); break;
    case 9: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<9>); break;
    case 16: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<16>); break;
    case 17: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<17>); break;
    case 32: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<32>); break;
    case 33: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<33>); break;
    case 64: kfn = reinterpret_cast<const void*>(pool_max_backward_s1_kernel<64>); break;
    default: return cudaErrorInvalidConfiguration;
  }
  cudaError_t e = ensure_smem_attr(kfn);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kMbThreads + 32, kMbSmem);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
  const int64_t g = p.ntiles < cap ? p.ntiles : cap;
  void* args[] = {&p};
  e = cudaLaunchKernel(kfn, dim3((unsigned)(g < 1 ? 1 : g)), dim3(kMbThreads + 32), args, kMbSmem, stream);
  note_launch();
  return e;
}

}  // namespace ss
