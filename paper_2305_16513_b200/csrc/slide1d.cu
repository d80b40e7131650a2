// slide1d.cu -- sm_100a kernels for the 1-D sliding window sum (Eq. 3,
// PAPER.md l.41-44) with (+) in {+, max} (Sec. 2.3, l.53) and the sliding dot
// product / 1-D convolution (Sec. 2.5, l.86-87).
//
// Tile skeleton:
//   * Both x and y are viewed as 2-D arrays of 128-byte rows (32 elements).
//   * A persistent CTA (one per SM) walks CTA tiles of 256 output rows
//     (8192 outputs) of one batch row.  A producer warp stages the tile's
//     input rows plus the (w-1)-element halo rows HBM -> smem with TMA
//     (cp.async.bulk.tensor.2d, SWIZZLE_128B) into a ring of stages guarded
//     by full/empty mbarriers.
//   * 8 consumer warps; lane t of warp i owns the 32 consecutive outputs of
//     output row 32*i + t.  It reads its input run from the swizzled stage with
//     conflict-free 128-bit LDS, evaluates its 32 windows in registers, and
//     writes the row into a swizzled staging buffer that one lane stores with
//     a TMA tensor store (rows crossing a batch-row edge use masked stores).
//   * Window evaluation (the "P-block pivot" form of Alg. 2's prefix/suffix
//     split): the 32 outputs are cut into blocks of
//     P = 2^floor(log2 min(w,32)) outputs; for the block [g, g+P) every window
//     contains the block's last element, so
//         y_{g+r} = suffix_{g+r..g+P-1} (+) middle_{g+P..g+w-1} (+) prefix_{g+w..g+w+r-1}
//     costing ~3 (+) per output whatever w is (order-preserving, so only
//     associativity is used).
//   * Conv: each thread keeps its 32+k-1 inputs in registers and runs
//     32*k FMAs with the taps in the kernel-parameter constant bank, in the
//     fixed tap order j = 0..k-1 (bitwise independent of tiling/sharding).
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

constexpr int kWarps = 8;                    // consumer warps per CTA
constexpr int kThreads = (kWarps + 1) * 32;  // + 1 producer warp
constexpr int kTileRows = kWarps * 32;       // 256 output rows = 8192 outputs
constexpr int kHaloBoxRows = 8;
constexpr int kStageAlign = 1024;

struct TileGeom {
  int64_t b;        // batch row
  int64_t yrow0;    // first y-view row of the CTA tile
  int64_t e_y;      // y-view element index of output 0 of batch row b
  int64_t L;        // outputs per batch row
  int64_t xrow0;    // first x-view row loaded (may be -1)
  int m;            // element offset of the tile's first input inside row xrow0
  int halo_boxes;   // 8-row halo boxes loaded after the 256 main rows
  bool empty;
};

__device__ __forceinline__ int64_t floor_div32(int64_t a) { return a >= 0 ? a / 32 : -((31 - a) / 32); }

__device__ __forceinline__ TileGeom tile_geom(const Slide1DParams& p, int64_t tau) {
  TileGeom g;
  g.b = tau / p.tiles_per_row;
  int64_t j = tau - g.b * p.tiles_per_row;
  g.L = p.L;
  g.e_y = p.shift_y + g.b * p.L;
  g.yrow0 = g.e_y / 32 + (int64_t)kTileRows * j;
  g.empty = 32 * g.yrow0 >= g.e_y + p.L;
  int64_t ix0 = p.shift_x + g.b * p.N + (32 * g.yrow0 - g.e_y);
  g.xrow0 = floor_div32(ix0);
  g.m = (int)(ix0 - 32 * g.xrow0);
  int64_t last_local = 32 * (kTileRows - 1) + g.m + 31 + p.span;
  int nrows = (int)(last_local / 32) + 1;
  int halo = nrows - kTileRows;
  g.halo_boxes = halo > 0 ? (halo + kHaloBoxRows - 1) / kHaloBoxRows : 0;
  return g;
}

// ------------------------------------------------------------- input loading
// Element e of a stage lives at byte swz128(4e) from the stage base.
template <typename T>
struct StageReader {
  const uint8_t* stage;   // generic pointer to the stage (1024-B aligned)
  bool slow;              // tile touches x-view elements past the TMA-covered rows
  int64_t gbase;          // x-view element index of stage element 0
  int64_t full_elems;     // x-view elements covered by the tensor map
  int64_t total_elems;    // x-view elements that exist
  const T* xg;            // x-view element 0 in global memory

  __device__ __forceinline__ T elem(int e) const {
    if (!slow) return *reinterpret_cast<const T*>(stage + swz128(4u * (uint32_t)e));
    int64_t g = gbase + e;
    if (g >= 0 && g < full_elems) return *reinterpret_cast<const T*>(stage + swz128(4u * (uint32_t)e));
    if (g >= full_elems && g < total_elems) return __ldg(xg + g);
    return T(0);
  }
  // 4 elements of chunk c (elements 4c..4c+3)
  __device__ __forceinline__ void chunk(int c, T (&q)[4]) const {
    int64_t g = gbase + 4 * (int64_t)c;
    if (!slow || (g >= 0 && g + 3 < full_elems)) {
      const uint4 v = *reinterpret_cast<const uint4*>(stage + swz128(16u * (uint32_t)c));
      q[0] = bitcast<T>(v.x); q[1] = bitcast<T>(v.y); q[2] = bitcast<T>(v.z); q[3] = bitcast<T>(v.w);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) q[e] = elem(4 * c + e);
    }
  }
  // v[i] = element (p0 + i), i < NV; 128-bit loads plus a 2-stage select
  // network for the runtime misalignment p0 & 3.
  template <int NV>
  __device__ __forceinline__ void run(int p0, T (&v)[NV]) const {
    constexpr int NC = (NV + 3 + 3) / 4;
    T raw[4 * NC];
    const int c0 = p0 >> 2;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      T q[4];
      chunk(c0 + c, q);
      raw[4 * c + 0] = q[0]; raw[4 * c + 1] = q[1]; raw[4 * c + 2] = q[2]; raw[4 * c + 3] = q[3];
    }
    const int sh = p0 & 3;
    if (sh & 1) {
#pragma unroll
      for (int i = 0; i < 4 * NC - 1; ++i) raw[i] = raw[i + 1];
    }
    if (sh & 2) {
#pragma unroll
      for (int i = 0; i < 4 * NC - 3; ++i) raw[i] = raw[i + 2];
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = raw[i];
  }
};

// ------------------------------------------------------------- the kinds
// Conv: y_r = sum_{j<KT} taps[j] * x_{p0+r+j}; taps beyond k are zero.
template <int KT>
struct ConvKind {
  using T = float;
  static constexpr int kSpan = (32 + KT - 1) - 26;  // max elements read past the own 32 (see StageReader::run)
  template <class R>
  static __device__ __forceinline__ void compute(const Slide1DParams& p, const R& rd, int p0,
                                                 float (&y)[32]) {
    constexpr int NV = 32 + KT - 1;
    float v[NV];
    rd.template run<NV>(p0, v);
#pragma unroll
    for (int r = 0; r < 32; ++r) y[r] = 0.0f;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      const float f = p.taps[j];
#pragma unroll
      for (int r = 0; r < 32; ++r) y[r] = __fmaf_rn(f, v[r + j], y[r]);
    }
  }
};

// Pool with P-block pivots, P <= w < 2P (P < 32), all in registers.
template <class Op, int P>
struct PoolKind {
  using T = typename Op::T;
  static constexpr int kSpan = (32 + 2 * P - 2) - 26;
  template <class R>
  static __device__ __forceinline__ void compute(const Slide1DParams& p, const R& rd, int p0,
                                                 T (&y)[32]) {
    constexpr int NV = 32 + 2 * P - 2;
    T v[NV];
    rd.template run<NV>(p0, v);
    const int w = (int)p.w;
    const int s = w - P;  // in [0, P)
    // u[i] = v[i + s] for i in [P, 32 + P - 1): barrel shift by s
    T u[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) u[i] = v[i];
#pragma unroll
    for (int k = 1; k < P; k <<= 1) {
      if (s & k) {
#pragma unroll
        for (int i = 0; i + k < NV; ++i) u[i] = u[i + k];
      }
    }
#pragma unroll
    for (int g = 0; g < 32; g += P) {
      T a[P];
      a[P - 1] = v[g + P - 1];
#pragma unroll
      for (int i = P - 2; i >= 0; --i) a[i] = Op::combine(v[g + i], a[i + 1]);
      T m = Op::identity();
#pragma unroll
      for (int i = 0; i < P - 1; ++i)
        if (i < s) m = Op::combine(m, v[g + P + i]);
      y[g] = Op::combine(a[0], m);
      T pre = m;
#pragma unroll
      for (int r = 1; r < P; ++r) {
        pre = Op::combine(pre, u[g + P + r - 1]);
        y[g + r] = Op::combine(a[r], pre);
      }
    }
  }
};

// Pool with one pivot per thread (P = 32, w >= 32): the middle is streamed.
template <class Op>
struct PoolKind<Op, 32> {
  using T = typename Op::T;
  static constexpr int kSpan = -1;  // runtime: w + 5
  template <class R>
  static __device__ __forceinline__ void compute(const Slide1DParams& p, const R& rd, int p0,
                                                 T (&y)[32]) {
    const int w = (int)p.w;
    T a[32];
    rd.template run<32>(p0, a);
#pragma unroll
    for (int i = 30; i >= 0; --i) a[i] = Op::combine(a[i], a[i + 1]);
    // middle: elements [p0+32, p0+w)
    T m0 = Op::identity(), m1 = Op::identity(), m2 = Op::identity(), m3 = Op::identity();
    const int s0 = p0 + 32, e0 = p0 + w;
    if (e0 > s0) {
      const int cs = s0 >> 2, ce = (e0 - 1) >> 2;
      {  // first chunk (partial)
        T q[4];
        rd.chunk(cs, q);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int idx = 4 * cs + e;
          if (idx >= s0 && idx < e0) m0 = Op::combine(m0, q[e]);
        }
      }
      int c = cs + 1;
      for (; c + 1 < ce; c += 2) {  // full chunks
        T q[4], q2[4];
        rd.chunk(c, q);
        rd.chunk(c + 1, q2);
        m0 = Op::combine(m0, Op::combine(q[0], q2[0]));
        m1 = Op::combine(m1, Op::combine(q[1], q2[1]));
        m2 = Op::combine(m2, Op::combine(q[2], q2[2]));
        m3 = Op::combine(m3, Op::combine(q[3], q2[3]));
      }
      for (; c <= ce; ++c) {  // remaining (last may be partial)
        T q[4];
        rd.chunk(c, q);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int idx = 4 * c + e;
          if (idx < e0) {
            if (e == 0) m0 = Op::combine(m0, q[e]);
            if (e == 1) m1 = Op::combine(m1, q[e]);
            if (e == 2) m2 = Op::combine(m2, q[e]);
            if (e == 3) m3 = Op::combine(m3, q[e]);
          }
        }
      }
    }
    const T m = Op::combine(Op::combine(m0, m1), Op::combine(m2, m3));
    T b[31];
    rd.template run<31>(p0 + w, b);
    y[0] = Op::combine(a[0], m);
    T pre = m;
#pragma unroll
    for (int r = 1; r < 32; ++r) {
      pre = Op::combine(pre, b[r - 1]);
      y[r] = Op::combine(a[r], pre);
    }
  }
};

// ------------------------------------------------------------- the kernel
template <class Kind>
__global__ void __launch_bounds__(kThreads, 1)
slide1d_tma_kernel(const __grid_constant__ Slide1DParams p) {
  using T = typename Kind::T;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + kStageAlign - 1) & ~uintptr_t(kStageAlign - 1));
  const int S = p.stages;
  const uint32_t stage_bytes = p.stage_bytes;
  uint8_t* staging = smem + (size_t)S * stage_bytes;                  // kWarps * 2 * 4 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(staging + kWarps * 2 * 4096);
  uint64_t* empty = full + S;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
  }
  if (warp == kWarps && lane == 0) {
    prefetch_tmap(&p.tm_x_main);
    prefetch_tmap(&p.tm_x_halo);
    if (p.has_y_map) prefetch_tmap(&p.tm_y);
  }
  __syncthreads();

  if (warp == kWarps) {
    // ---------------- producer: one elected lane issues the TMA loads
    if (lane == 0) {
      int it = 0;
      for (int64_t tau = blockIdx.x; tau < p.ntiles; tau += gridDim.x) {
        const TileGeom g = tile_geom(p, tau);
        if (g.empty) continue;
        const int s = it % S;
        const uint32_t ph = (uint32_t)(it / S) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* dst = smem + (size_t)s * stage_bytes;
        const uint32_t bytes = (uint32_t)(kTileRows + kHaloBoxRows * g.halo_boxes) * 128u;
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_load_2d(dst, &p.tm_x_main, 0, (int32_t)g.xrow0, &full[s]);
        for (int h = 0; h < g.halo_boxes; ++h)
          tma_load_2d(dst + (size_t)(kTileRows + kHaloBoxRows * h) * 128, &p.tm_x_halo, 0,
                      (int32_t)(g.xrow0 + kTileRows + kHaloBoxRows * h), &full[s]);
        ++it;
      }
    }
    return;
  }

  // ---------------- consumers
  int it = 0;
  uint8_t* my_staging = staging + warp * 2 * 4096;
  const uint32_t my_staging_s = smem_u32(my_staging);
  for (int64_t tau = blockIdx.x; tau < p.ntiles; tau += gridDim.x) {
    const TileGeom g = tile_geom(p, tau);
    if (g.empty) continue;
    const int s = it % S;
    const uint32_t ph = (uint32_t)(it / S) & 1u;
    const uint8_t* st = smem + (size_t)s * stage_bytes;

    const int64_t wrow0 = g.yrow0 + 32 * warp;  // first y-view row of this warp
    const int64_t o_first = 32 * wrow0, o_end = 32 * (wrow0 + 32);
    const bool warp_active = o_first < g.e_y + g.L && o_end > g.e_y;
    const bool warp_full = o_first >= g.e_y && o_end <= g.e_y + g.L;

    mbar_wait(&full[s], ph);
    T y[32];
    if (warp_active) {
      StageReader<T> rd;
      rd.stage = st;
      rd.gbase = 32 * g.xrow0;
      rd.full_elems = p.x_full_elems;
      rd.total_elems = p.x_total_elems;
      rd.xg = reinterpret_cast<const T*>(p.x_view);
      const int64_t last_read = rd.gbase + 32 * (kTileRows - 1) + g.m + 31 + p.span;
      rd.slow = (rd.gbase < 0) || (last_read >= p.x_full_elems);
      const int p0 = 32 * (32 * warp + lane) + g.m;
      Kind::compute(p, rd, p0, y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (warp_active) {
      if (warp_full && p.has_y_map) {
        const int buf = it & 1;
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        const uint32_t base = my_staging_s + buf * 4096;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t off = swz128((uint32_t)lane * 128u + 16u * c);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + off),
                       "r"(bitcast<uint32_t>(y[4 * c + 0])), "r"(bitcast<uint32_t>(y[4 * c + 1])),
                       "r"(bitcast<uint32_t>(y[4 * c + 2])), "r"(bitcast<uint32_t>(y[4 * c + 3]))
                       : "memory");
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&p.tm_y, 0, (int32_t)wrow0, my_staging + buf * 4096);
          bulk_commit();
        }
      } else {
        T* yv = reinterpret_cast<T*>(p.y_view);
        const int64_t orow = 32 * (wrow0 + lane);
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const int64_t o = orow + r;
          if (o >= g.e_y && o < g.e_y + g.L) yv[o] = y[r];
        }
      }
    }
    ++it;
  }
  if (lane == 0) bulk_wait_all();
}

// ------------------------------------------------------------- host launch
template <class Kind>
static cudaError_t launch_kind(Slide1DParams& p, cudaStream_t stream, int grid) {
  int span = Kind::kSpan >= 0 ? Kind::kSpan : (int)p.w + 5;
  p.span = span;
  const int max_halo_rows = (int)((32 * (kTileRows - 1) + 31 + 31 + span) / 32) + 1 - kTileRows;
  const int halo_cap = ((max_halo_rows + kHaloBoxRows - 1) / kHaloBoxRows) * kHaloBoxRows;
  p.stage_bytes = (uint32_t)(kTileRows + (halo_cap > 0 ? halo_cap : 0)) * 128u;
  const size_t fixed = kWarps * 2 * 4096 + kStageAlign + 256;
  int S = 4;
  while (S > 2 && (size_t)S * p.stage_bytes + fixed > (size_t)kSmemBudget) --S;
  if ((size_t)S * p.stage_bytes + fixed > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  p.stages = S;
  const size_t smem = (size_t)S * p.stage_bytes + fixed;
  auto kfn = slide1d_tma_kernel<Kind>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t g = p.ntiles < grid ? p.ntiles : grid;
  if (g < 1) g = 1;
  kfn<<<(unsigned)g, kThreads, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv_tma(Slide1DParams& p, int KT, cudaStream_t stream, int grid) {
  switch (KT) {
    case 1: return launch_kind<ConvKind<1>>(p, stream, grid);
    case 2: return launch_kind<ConvKind<2>>(p, stream, grid);
    case 3: return launch_kind<ConvKind<3>>(p, stream, grid);
    case 4: return launch_kind<ConvKind<4>>(p, stream, grid);
    case 5: return launch_kind<ConvKind<5>>(p, stream, grid);
    case 7: return launch_kind<ConvKind<7>>(p, stream, grid);
    case 8: return launch_kind<ConvKind<8>>(p, stream, grid);
    case 15: return launch_kind<ConvKind<15>>(p, stream, grid);
    case 16: return launch_kind<ConvKind<16>>(p, stream, grid);
    case 24: return launch_kind<ConvKind<24>>(p, stream, grid);
    case 31: return launch_kind<ConvKind<31>>(p, stream, grid);
    case 32: return launch_kind<ConvKind<32>>(p, stream, grid);
    case 48: return launch_kind<ConvKind<48>>(p, stream, grid);
    case 63: return launch_kind<ConvKind<63>>(p, stream, grid);
    case 64: return launch_kind<ConvKind<64>>(p, stream, grid);
    default: return cudaErrorInvalidValue;
  }
}

template <class Op>
static cudaError_t launch_pool_op(Slide1DParams& p, int P, cudaStream_t stream, int grid) {
  switch (P) {
    case 1: return launch_kind<PoolKind<Op, 1>>(p, stream, grid);
    case 2: return launch_kind<PoolKind<Op, 2>>(p, stream, grid);
    case 4: return launch_kind<PoolKind<Op, 4>>(p, stream, grid);
    case 8: return launch_kind<PoolKind<Op, 8>>(p, stream, grid);
    case 16: return launch_kind<PoolKind<Op, 16>>(p, stream, grid);
    case 32: return launch_kind<PoolKind<Op, 32>>(p, stream, grid);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pool_tma(Slide1DParams& p, int op, int dtype, int P, cudaStream_t stream,
                            int grid) {
  if (op == kOpSum && dtype == 1) return launch_pool_op<OpSumI32>(p, P, stream, grid);
  if (op == kOpSum && dtype == 0) return launch_pool_op<OpSumF32>(p, P, stream, grid);
  if (op == kOpMax && dtype == 1) return launch_pool_op<OpMaxI32>(p, P, stream, grid);
  if (op == kOpMax && dtype == 0) return launch_pool_op<OpMaxF32>(p, P, stream, grid);
  return cudaErrorInvalidValue;
}

}  // namespace ss
