// slide1d.cu -- sm_100a kernels for the 1-D sliding window sum (Eq. 3,
// PAPER.md l.41-44) with (+) in {+, max} (Sec. 2.3, l.53) and the sliding dot
// product / 1-D convolution (Sec. 2.5, l.86-87).
//
// Tile skeleton:
//   * x and y are viewed as 2-D arrays of 128-byte rows (32 elements).
//   * A persistent CTA (one per SM) walks CTA tiles of 240 output rows
//     (7680 outputs) of one batch row.  A producer warp stages the tile's
//     input rows plus the (w-1)-element halo rows HBM -> smem with TMA
//     (cp.async.bulk.tensor.2d, SWIZZLE_128B) into a ring of stages guarded
//     by full/empty mbarriers.
//   * 15 consumer warps (+1 producer = 4 warps per SM sub-partition); lane t
//     of warp i owns the 16 consecutive outputs [16*(t>>4), +16) of output row
//     16*i + (t&15).  It reads its input run from the swizzled stage with
//     128-bit ld.shared (the swizzle makes the 8 lanes of every LDS.128 phase
//     hit 8 distinct bank groups), evaluates its 16 windows in registers and
//     writes them into a swizzled staging buffer that one lane stores with a
//     TMA tensor store (warps straddling a batch-row edge use masked stores).
//   * The tile's misalignment SH = (first input element) mod 4 is uniform per
//     tile, so each kind is instantiated for SH = 0..3 and the realignment of
//     the input run is pure register renaming.
//   * Pool (+, max): the "P-block pivot" form of Alg. 2's prefix/suffix split
//     (PAPER.md l.113-134): the 16 outputs are cut into blocks of
//     P = 2^floor(log2 min(w,16)) outputs; every window starting in the block
//     [g, g+P) contains the block's last element, so
//        y_{g+r} = suffix_{g+r..g+P-1} (+) middle_{g+P..g+w-1} (+) prefix_{g+w..g+w+r-1}
//     ~3 (+) per output whatever w is; order-preserving (associativity only).
//   * Conv: output pairs accumulated with FFMA2 (fma.rn.f32x2, two IEEE fp32
//     FMAs per instruction): an even-tap and an odd-tap partial sum per
//     output, each in increasing tap order from 0, added at the end -- an
//     association fixed by the tap index alone, so outputs are bitwise
//     independent of tiling and identical to the generic kernel.  Taps are
//     processed in passes of 32 to bound register use.
//   * Tiles that read past the last full 128-B row of x (the very end of the
//     array) take a compact direct-window path from global memory.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

constexpr int kWarps = kSlideWarps;          // consumer warps per CTA
constexpr int kThreads = (kWarps + 1) * 32;  // + 1 producer warp
constexpr int kR = 16;                       // outputs per thread of the pool kinds
constexpr int kMainBoxRows = kSlideTileRows; // rows per main TMA box (240)
constexpr int kHaloBoxRows = 8;
constexpr int kStageAlign = 1024;
constexpr int kStagingBufs = 1;                 // output staging buffers per warp
constexpr int kMaxStages = 5;
constexpr int kBSWarpBytes = 4 * (32 + 64 + 8);  // per-warp block totals (+64 following, +8 over-read)
constexpr int kBSBytes = kSlideWarps * kBSWarpBytes / 2;  // (2 * kBSBytes reserved in smem)

// ------------------------------------------------------------- smem access
__device__ __forceinline__ uint32_t chunk_addr(uint32_t st_s, int c) {
  return st_s + swz128(16u * (uint32_t)c);
}
__device__ __forceinline__ void lds_v4(uint32_t a, uint32_t& x0, uint32_t& x1, uint32_t& x2,
                                       uint32_t& x3) {
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
               : "r"(a));
}
__device__ __forceinline__ void lds_v2x64(uint32_t a, uint64_t& lo, uint64_t& hi) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(a));
}
__device__ __forceinline__ uint64_t pack2(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(uint64_t v, uint32_t& lo, uint32_t& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
}
// two IEEE fp32 FMAs: d.{lo,hi} = a.{lo,hi} * b.{lo,hi} + c.{lo,hi}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// v[i] = stage element (4*c0 + SH + i), i < NV  (SH compile-time: no shuffling)
template <typename T, int SH, int NV>
__device__ __forceinline__ void load_run(uint32_t st_s, int c0, T (&v)[NV]) {
  constexpr int NC = (SH + NV + 3) / 4;
  uint32_t raw[4 * NC];
#pragma unroll
  for (int c = 0; c < NC; ++c)
    lds_v4(chunk_addr(st_s, c0 + c), raw[4 * c], raw[4 * c + 1], raw[4 * c + 2], raw[4 * c + 3]);
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = bitcast<T>(raw[SH + i]);
}

// v[i] = stage element (e0 + i), i < NV, with a runtime misalignment e0 & 3
// (2-stage select network).
template <typename T, int NV>
__device__ __forceinline__ void load_run_rt(uint32_t st_s, int e0, T (&v)[NV]) {
  constexpr int NC = (NV + 3 + 3) / 4;
  uint32_t raw[4 * NC];
  const int c0 = e0 >> 2;
#pragma unroll
  for (int c = 0; c < NC; ++c)
    lds_v4(chunk_addr(st_s, c0 + c), raw[4 * c], raw[4 * c + 1], raw[4 * c + 2], raw[4 * c + 3]);
  const int sh = e0 & 3;
#pragma unroll
  for (int i = 0; i < 4 * NC - 1; ++i) raw[i] = (sh & 1) ? raw[i + 1] : raw[i];
#pragma unroll
  for (int i = 0; i < 4 * NC - 3; ++i) raw[i] = (sh & 2) ? raw[i + 2] : raw[i];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = bitcast<T>(raw[i]);
}

// ------------------------------------------------------------- the kinds
// Conv: y_r = sum_{j<KT} taps[j] * x_{p0+r+j} (taps beyond k are zero),
// evaluated as two partial sums, over the even taps and over the odd taps,
// each accumulated with fp32 FMA in increasing j from 0, then added:
//     y_r = fl( S_even(r) + S_odd(r) ).
// The association depends only on the tap index, so every output is bitwise
// independent of tiling/sharding and equal to the generic kernel's.  It lets
// FFMA2 (two FMAs per instruction) read every input pair as an aligned
// register pair: for tap parity c the output pairs start at r0 with
// (SH + r0 + c) even, so x_{p0+r0+j}, x_{p0+r0+j+1} is (raw[2m], raw[2m+1]).
template <int KT, int R>
struct ConvKind {
  using T = float;
  static constexpr bool kTwoPhase = false;
  static constexpr int kRt = R;  // outputs per thread (16: half a 128-B row; 32: a full row)
  // elements read past the thread's first input (max over SH): chunks cover
  // [0, SH + R + KT) rounded up to a chunk
  static constexpr int kSpan = 4 * ((3 + R + KT + 3) / 4) - R;
#ifndef SS_CONV_PREFETCH
#define SS_CONV_PREFETCH 3
#endif
  static constexpr int kPrefetch = SS_CONV_PREFETCH;  // chunks loaded ahead of the tap that first needs them

  template <int SH>
  static __device__ __forceinline__ void compute(const Slide1DParams& p, uint32_t st_s, int c0,
                                                 float (&y)[R]) {
    constexpr int PI0 = SH & 1;        // pairs of even taps start at outputs -PI0 (mod 2)
    constexpr int PI1 = (SH + 1) & 1;  // ... of odd taps
    constexpr int N0 = R / 2 + PI0, N1 = R / 2 + PI1;
    constexpr int NC = (SH + R + KT + 3) / 4;  // chunks of the whole run
    float2 A0[N0], A1[N1];  // A_c[i]: outputs (2i - PI_c, 2i - PI_c + 1)
#pragma unroll
    for (int i = 0; i < N0; ++i) A0[i] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < N1; ++i) A1[i] = make_float2(0.0f, 0.0f);
    float2 E[2 * NC];  // E[m] = (raw[2m], raw[2m+1]); chunk c fills E[2c], E[2c+1]
    auto load = [&](int c) {
      uint32_t a0, a1, a2, a3;
      lds_v4(chunk_addr(st_s, c0 + c), a0, a1, a2, a3);
      E[2 * c] = make_float2(__uint_as_float(a0), __uint_as_float(a1));
      E[2 * c + 1] = make_float2(__uint_as_float(a2), __uint_as_float(a3));
    };
    // Diagonal order: walk the input pairs E[m] in increasing m and apply every
    // (output pair, tap) that uses E[m] back to back, so the pair stays in the
    // operand-reuse cache.  For a fixed accumulator the taps still arrive in
    // increasing order (jj = 2m + const - 2i grows with m), so each output's
    // association is unchanged.
    constexpr int M_END = (SH + R + KT + 1) / 2 + 1;  // pairs touched by any tap
    constexpr int C_FIRST = kPrefetch + 1;
#pragma unroll
    for (int c = 0; c < (C_FIRST < NC ? C_FIRST : NC); ++c) load(c);
#pragma unroll
    for (int mm = 0; mm < M_END; ++mm) {
      if ((mm & 1) == 0) {  // entering chunk mm/2: prefetch chunk mm/2 + C_FIRST
        const int c = mm / 2 + C_FIRST;
        if (c < NC) load(c);
      }
#pragma unroll
      for (int i = 0; i < N0; ++i) {
        const int jj = 2 * mm - SH + PI0 - 2 * i;  // even tap using E[mm] for pair i
        if (jj >= 0 && jj < KT) {
          const float f = p.taps[jj];
          A0[i] = __ffma2_rn(E[mm], make_float2(f, f), A0[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        const int jj = 2 * mm - SH + PI1 - 2 * i;  // odd tap
        if (jj >= 0 && jj < KT) {
          const float f = p.taps[jj];
          A1[i] = __ffma2_rn(E[mm], make_float2(f, f), A1[i]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i0 = (r + PI0) >> 1, i1 = (r + PI1) >> 1;
      const float s0 = ((r + PI0) & 1) ? A0[i0].y : A0[i0].x;
      const float s1 = ((r + PI1) & 1) ? A1[i1].y : A1[i1].x;
      y[r] = __fadd_rn(s0, s1);
    }
  }
};

// Pool with P-block pivots.  P < 16: P <= w < 2P, own run and middle in
// registers.  P = 16: w >= 16, the middle x[p0+16, p0+w) is streamed.
template <class Op, int P>
struct PoolKind {
  using T = typename Op::T;
  static constexpr bool kTwoPhase = false;
  static constexpr int kRt = kR;
  static constexpr int kOwn = P < 16 ? kR + P - 1 : kR;  // own run length
  static constexpr int kSpan = -1;                        // runtime: w + 20

  template <int SH>
  static __device__ __forceinline__ void compute(const Slide1DParams& p, uint32_t st_s, int c0,
                                                 T (&y)[kR]) {
    const int w = (int)p.w;
    T v[kOwn];
    load_run<T, SH, kOwn>(st_s, c0, v);
    // tail run: tl[i] = x[p0 + w + i], i < 15 (runtime misalignment)
    T tl[kR - 1];
    load_run_rt<T, kR - 1>(st_s, 4 * c0 + SH + w, tl);
    if constexpr (P < 16) {
      const int s = w - P;  // middle length per block, in [0, P)
#pragma unroll
      for (int g = 0; g < kR; g += P) {
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
          pre = Op::combine(pre, tl[g + r - 1]);
          y[g + r] = Op::combine(a[r], pre);
        }
      }
    } else {
      T a[kR];
      a[kR - 1] = v[kR - 1];
#pragma unroll
      for (int i = kR - 2; i >= 0; --i) a[i] = Op::combine(v[i], a[i + 1]);
      // middle: stage elements [p0 + 16, p0 + w) with p0 = 4*c0 + SH
      T m0 = Op::identity(), m1 = Op::identity(), m2 = Op::identity(), m3 = Op::identity();
      const int e0 = 4 * c0 + SH + w;  // one past the middle
      if (w > kR) {
        const int cs = c0 + 4, ce = (e0 - 1) >> 2;  // chunk cs starts at element p0 + 16 - SH
        {
          uint32_t q0, q1, q2, q3;
          lds_v4(chunk_addr(st_s, cs), q0, q1, q2, q3);
          const int n = e0 - 4 * cs;  // elements of this chunk before e0
          if (SH <= 0 && 0 < n) m0 = Op::combine(m0, bitcast<T>(q0));
          if (SH <= 1 && 1 < n) m1 = Op::combine(m1, bitcast<T>(q1));
          if (SH <= 2 && 2 < n) m2 = Op::combine(m2, bitcast<T>(q2));
          if (3 < n) m3 = Op::combine(m3, bitcast<T>(q3));
        }
        int c = cs + 1;
#pragma unroll 2
        for (; c < ce; ++c) {
          uint32_t q0, q1, q2, q3;
          lds_v4(chunk_addr(st_s, c), q0, q1, q2, q3);
          m0 = Op::combine(m0, bitcast<T>(q0));
          m1 = Op::combine(m1, bitcast<T>(q1));
          m2 = Op::combine(m2, bitcast<T>(q2));
          m3 = Op::combine(m3, bitcast<T>(q3));
        }
        if (c == ce) {
          uint32_t q0, q1, q2, q3;
          lds_v4(chunk_addr(st_s, c), q0, q1, q2, q3);
          const int n = e0 - 4 * c;
          m0 = Op::combine(m0, bitcast<T>(q0));
          if (1 < n) m1 = Op::combine(m1, bitcast<T>(q1));
          if (2 < n) m2 = Op::combine(m2, bitcast<T>(q2));
          if (3 < n) m3 = Op::combine(m3, bitcast<T>(q3));
        }
      }
      const T m = Op::combine(Op::combine(m0, m1), Op::combine(m2, m3));
      y[0] = Op::combine(a[0], m);
      T pre = m;
#pragma unroll
      for (int r = 1; r < kR; ++r) {
        pre = Op::combine(pre, tl[r - 1]);
        y[r] = Op::combine(a[r], pre);
      }
    }
  }
};

// Pool for long windows (w >= 48): the middle x[p0+16, p0+w) is assembled
// from 16-element block totals instead of being re-read element by element.
// Within a warp the 32 threads own 32 consecutive blocks (block beta =
// 2*row + half); each publishes B[beta] = its suffix a[0] to a per-warp
// shared array, and lanes 0..q-1 also total the q blocks that follow the
// warp's range.  After __syncwarp:
//   middle = B[beta+1] (+) ... (+) B[beta+q] (+) head(block beta+q+1, rr elements),
//   q = (w-16) div 16, rr = (w-16) mod 16.
template <class Op>
struct PoolBlockKind {
  using T = typename Op::T;
  static constexpr bool kTwoPhase = true;
  static constexpr int kRt = kR;
  static constexpr int kSpan = -1;  // runtime: w + 20

  template <int SH>
  static __device__ __forceinline__ T block_total(uint32_t st_s, int c0) {
    T v[kR];
    load_run<T, SH, kR>(st_s, c0, v);
#pragma unroll
    for (int s = 1; s < kR; s <<= 1)
#pragma unroll
      for (int i = 0; i + s < kR; i += 2 * s) v[i] = Op::combine(v[i], v[i + s]);
    return v[0];
  }

  // Called by every lane of an active warp.  bs_s: this warp's block-total
  // array; lb: my block index within the warp (0..31).
  template <int SH>
  static __device__ __forceinline__ void run(const Slide1DParams& p, uint32_t st_s, int c0,
                                             uint32_t bs_s, int lb, int lane, T (&y)[kR]) {
    const int w = (int)p.w;
    const int q = (w - kR) >> 4, rr = (w - kR) & 15;
    T a[kR];
    load_run<T, SH, kR>(st_s, c0, a);
#pragma unroll
    for (int i = kR - 2; i >= 0; --i) a[i] = Op::combine(a[i], a[i + 1]);
    __syncwarp();  // previous tile's readers of bs are done
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(bs_s + 4u * lb), "r"(bitcast<uint32_t>(a[0]))
                 : "memory");
    // blocks 32..31+q of the warp's block sequence: the 16 rows after the warp
    // (block 32 + e starts 16*(32 + e - lb) elements after my block)
    for (int e = lane; e < q; e += 32) {
      const T t = block_total<SH>(st_s, c0 + 4 * (32 + e - lb));
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(bs_s + 4u * (32 + e)), "r"(bitcast<uint32_t>(t))
                   : "memory");
    }
    __syncwarp();
    // fold B[lb+1 .. lb+q]: loads issued 8 at a time ahead of their folds
    T m0 = Op::identity(), m1 = Op::identity();
    for (int i = 1; i <= q; i += 8) {
      uint32_t b[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b[k]) : "r"(bs_s + 4u * (lb + i + k)));
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        if (i + k <= q) m0 = Op::combine(m0, bitcast<T>(b[k]));
        if (i + k + 1 <= q) m1 = Op::combine(m1, bitcast<T>(b[k + 1]));
      }
    }
    T m = Op::combine(m0, m1);
    if (rr > 0) {  // head: first rr elements of block lb+q+1
      T hb[kR - 1];
      load_run<T, SH, kR - 1>(st_s, c0 + 4 * (q + 1), hb);
      T h = hb[0];
#pragma unroll
      for (int k = 1; k < kR - 1; ++k)
        if (k < rr) h = Op::combine(h, hb[k]);
      m = Op::combine(m, h);
    }
    T tl[kR - 1];
    load_run_rt<T, kR - 1>(st_s, 4 * c0 + SH + w, tl);
    y[0] = Op::combine(a[0], m);
    T pre = m;
#pragma unroll
    for (int r = 1; r < kR; ++r) {
      pre = Op::combine(pre, tl[r - 1]);
      y[r] = Op::combine(a[r], pre);
    }
  }
};

template <class Kind>
struct SlowPath;  // direct windows from global memory (array-end tiles)

template <int KT, int R>
struct SlowPath<ConvKind<KT, R>> {
  static __device__ __forceinline__ float eval(const Slide1DParams& p, const float* x) {
    float s0 = 0.0f, s1 = 0.0f;  // even taps, odd taps (same association as compute())
    for (int j = 0; j < (int)p.w; j += 2) s0 = __fmaf_rn(p.taps[j], __ldg(x + j), s0);
    for (int j = 1; j < (int)p.w; j += 2) s1 = __fmaf_rn(p.taps[j], __ldg(x + j), s1);
    return __fadd_rn(s0, s1);
  }
};
template <class Op, int P>
struct SlowPath<PoolKind<Op, P>> {
  static __device__ __forceinline__ typename Op::T eval(const Slide1DParams& p,
                                                        const typename Op::T* x) {
    typename Op::T acc = __ldg(x);
    for (int j = 1; j < (int)p.w; ++j) acc = Op::combine(acc, __ldg(x + j));
    return acc;
  }
};

template <class Op>
struct SlowPath<PoolBlockKind<Op>> : SlowPath<PoolKind<Op, 16>> {};

// ------------------------------------------------------------- tile walk
struct TileCursor {
  int64_t b, j;  // batch row, tile within the row
  __device__ __forceinline__ void init(int64_t tau, int64_t tpr) {
    b = tau / tpr;
    j = tau - b * tpr;
  }
  __device__ __forceinline__ void advance(int64_t step, int64_t tpr) {
    j += step;
    while (j >= tpr) {
      j -= tpr;
      ++b;
    }
  }
};

struct TileGeom {
  int64_t yrow0;  // first y-view row of the CTA tile
  int64_t e_y;    // y-view element index of output 0 of batch row b
  int64_t xrow0;  // first x-view row loaded (may be -1: TMA zero-fills)
  int m;          // element offset of the tile's first input inside row xrow0
  int halo_boxes; // 8-row halo boxes loaded after the main rows
  bool empty;
  bool slow;      // reads past the TMA-covered part of x
};

__device__ __forceinline__ int64_t floor_div32(int64_t a) {
  return a >= 0 ? (a >> 5) : -((31 - a) >> 5);
}

template <int kTileRows>
__device__ __forceinline__ TileGeom tile_geom(const Slide1DParams& p, const TileCursor& tc) {
  TileGeom g;
  g.e_y = p.shift_y + tc.b * p.y_pitch + p.y_off;
  g.yrow0 = (g.e_y >> 5) + (int64_t)kTileRows * tc.j;
  g.empty = 32 * g.yrow0 >= g.e_y + p.L;
  const int64_t ix0 = p.shift_x + tc.b * p.N + (32 * g.yrow0 - g.e_y);
  g.xrow0 = floor_div32(ix0);
  g.m = (int)(ix0 - 32 * g.xrow0);
  const int last_local = 32 * (kTileRows - 1) + g.m + 31 + p.span;
  const int halo = (last_local >> 5) + 1 - kTileRows;
  g.halo_boxes = halo > 0 ? (halo + kHaloBoxRows - 1) / kHaloBoxRows : 0;
  // Rows past the tensor map read as zeros and only feed masked outputs; a
  // tile is "slow" only if a window of a valid output needs an element of
  // x's partial last 128-B row (not covered by the tensor map).
  if (p.x_total_elems > p.x_full_elems) {
    const int64_t o_end = min(32 * (g.yrow0 + kTileRows), g.e_y + p.L);  // one past last valid output
    const int64_t x_last = (o_end - 1 - g.e_y) + p.shift_x + tc.b * p.N + p.w - 1;
    g.slow = x_last >= p.x_full_elems;
  } else {
    g.slow = false;
  }
  return g;
}

// ------------------------------------------------------------- the kernel
// Per-stage tile header written by the producer before it arms the stage's
// full barrier (release) and read by the consumers after their wait
// (acquire): consumers never redo the 64-bit tile arithmetic.
struct TileHdr {
  int64_t yrow0;  // first y-view row of the tile
  int64_t y_lo;   // valid outputs of the batch row: [y_lo, y_hi) in y-view elements
  int64_t y_hi;
  int64_t dxy;    // x-view index of output o's first input = o + dxy
  int32_t m;      // tile misalignment (element offset of the first input in its row)
  int32_t flags;  // bit 0: slow (direct path), bit 1: done (no more tiles)
  int64_t pad;
};

template <class Kind>
__global__ void __launch_bounds__(kThreads, 1)
slide1d_tma_kernel(const __grid_constant__ Slide1DParams p) {
  using T = typename Kind::T;
  constexpr int KR = Kind::kRt;                       // outputs per thread
  constexpr int kWarpRows = KR == 32 ? 32 : 16;       // output rows per warp
  constexpr int kTileRows = kWarps * kWarpRows;       // 240 or 480
  constexpr int kStagingBytes = kWarpRows * 128;      // per warp buffer
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((kStageAlign - (smem_u32(smem_raw) & (kStageAlign - 1u))) &
                              (kStageAlign - 1u));  // shared-space pointer arithmetic
  const int S = p.stages;
  const uint32_t stage_bytes = p.stage_bytes;
  uint8_t* staging = smem + (size_t)S * stage_bytes;  // kWarps * kStagingBufs * 2 KB
  uint8_t* bsbuf = staging + kWarps * kStagingBufs * kStagingBytes;  // block totals
  uint64_t* full = reinterpret_cast<uint64_t*>(bsbuf + 2 * kBSBytes);
  uint64_t* empty = full + S;
  TileHdr* hdr = reinterpret_cast<TileHdr*>(empty + S);
  const uint32_t smem_s = smem_u32(smem);

  __shared__ ClcSmem clc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    clc_init(&clc);
    fence_mbar_init();
  }
  if (warp == kWarps && lane == 0) {
    prefetch_tmap(&p.tm_x_main);
    prefetch_tmap(&p.tm_x_halo);
    if (p.has_y_map) prefetch_tmap(&p.tm_y);
  }
  __syncthreads();

  if (warp == kWarps) {
    // ---------------- producer: one lane walks the tiles, publishes headers, issues TMA
    if (lane == 0) {
      // CTA b starts with tile b, then claims tiles by cluster launch control
      // (dynamic: SMs that stream faster take more tiles) or strides by gridDim.x
      const int64_t tpr = p.tiles_per_row;
      int it = 0;
      uint32_t cph = 0;
      TileCursor tc;
      tc.init(blockIdx.x, tpr);
      if (p.clc && (int64_t)blockIdx.x < p.ntiles) clc_request(&clc);
      for (int64_t tau = blockIdx.x; tau >= 0 && tau < p.ntiles;) {
        const TileGeom g = tile_geom<kTileRows>(p, tc);
        const int64_t b_cur = tc.b;
        if (!g.empty) {
          const int s = it % S;
          mbar_wait(&empty[s], ((uint32_t)(it / S) & 1u) ^ 1u);
          TileHdr& h = hdr[s];
          h.yrow0 = g.yrow0;
          h.y_lo = g.e_y;
          h.y_hi = g.e_y + p.L;
          h.dxy = p.shift_x + b_cur * p.N - g.e_y;
          h.m = g.m;
          h.flags = g.slow ? 1 : 0;
          uint8_t* dst = smem + (size_t)s * stage_bytes;
          if (g.slow) {  // consumers read global memory directly for this tile
            mbar_arrive(&full[s]);
          } else {
            const uint32_t bytes = (uint32_t)(kTileRows + kHaloBoxRows * g.halo_boxes) * 128u;
            mbar_arrive_expect_tx(&full[s], bytes);
#pragma unroll
            for (int mb = 0; mb < kTileRows / kMainBoxRows; ++mb)
              tma_load_2d(dst + (size_t)mb * kMainBoxRows * 128, &p.tm_x_main, 0,
                          (int32_t)(g.xrow0 + mb * kMainBoxRows), &full[s]);
            for (int h2 = 0; h2 < g.halo_boxes; ++h2)
              tma_load_2d(dst + (size_t)(kTileRows + kHaloBoxRows * h2) * 128, &p.tm_x_halo, 0,
                          (int32_t)(g.xrow0 + kTileRows + kHaloBoxRows * h2), &full[s]);
          }
          ++it;
        }
        if (p.clc) {
          // the claim was requested one tile ahead: its round trip overlapped the slot wait and the TMA issue
          tau = clc_wait(&clc, cph);
          if (tau >= 0) {
            clc_request(&clc);
            tc.init(tau, tpr);
          }
        } else {
          tc.advance(gridDim.x, tpr);
          tau += gridDim.x;
        }
      }
      const int s = it % S;  // end marker
      mbar_wait(&empty[s], ((uint32_t)(it / S) & 1u) ^ 1u);
      hdr[s].flags = 2;
      mbar_arrive(&full[s]);
    }
    return;
  }

  // ---------------- consumers
  const int row_in_warp = KR == 32 ? lane : (lane & 15);
  const int half = KR == 32 ? 0 : (lane >> 4);
  const int row = kWarpRows * warp + row_in_warp;  // output row within the tile
  uint8_t* my_staging = staging + warp * kStagingBufs * kStagingBytes;
  const uint32_t my_staging_s = smem_u32(my_staging);
  for (int it = 0;; ++it) {
    const int s = it % S;
    mbar_wait(&full[s], (uint32_t)(it / S) & 1u);
    const TileHdr& h = hdr[s];
    const int flags = h.flags;
    if (flags & 2) break;
    const int64_t yrow0 = h.yrow0, y_lo = h.y_lo, y_hi = h.y_hi;
    const int m = h.m;
    const bool slow = flags & 1;
    const uint32_t st_s = smem_s + (uint32_t)s * stage_bytes;

    const int64_t wrow0 = yrow0 + kWarpRows * warp;  // first y-view row of this warp
    const bool warp_active = 32 * wrow0 < y_hi && 32 * (wrow0 + kWarpRows) > y_lo;
    const bool warp_full = 32 * wrow0 >= y_lo && 32 * (wrow0 + kWarpRows) <= y_hi;
    const int64_t o0 = 32 * (wrow0 + row_in_warp) + KR * half;  // my first output (y view)

    T y[KR];
    if constexpr (Kind::kTwoPhase) {
      if (warp_active && !slow) {
        const int p0 = 32 * row + KR * half + m;
        const int c0 = p0 >> 2;
        // block order inside the warp: lb = 2*row_in_warp + half (consecutive blocks)
        const int lb = 2 * row_in_warp + half;
        const uint32_t bs_s = smem_u32(bsbuf) + (uint32_t)warp * kBSWarpBytes;
        switch (m & 3) {
          case 0: Kind::template run<0>(p, st_s, c0, bs_s, lb, lane, y); break;
          case 1: Kind::template run<1>(p, st_s, c0, bs_s, lb, lane, y); break;
          case 2: Kind::template run<2>(p, st_s, c0, bs_s, lb, lane, y); break;
          default: Kind::template run<3>(p, st_s, c0, bs_s, lb, lane, y); break;
        }
      }
    } else if (warp_active && !slow) {
      const int p0 = 32 * row + KR * half + m;  // stage element of my first input
      const int c0 = p0 >> 2;
      switch (m & 3) {
        case 0: Kind::template compute<0>(p, st_s, c0, y); break;
        case 1: Kind::template compute<1>(p, st_s, c0, y); break;
        case 2: Kind::template compute<2>(p, st_s, c0, y); break;
        default: Kind::template compute<3>(p, st_s, c0, y); break;
      }
    }
    const int64_t dxy = h.dxy;  // read before releasing the stage (header reuse)
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (warp_active) {
      if (slow) {
        // array-end tile: direct windows from global memory (valid outputs only)
        const T* xg = reinterpret_cast<const T*>(p.x_view);
        T* yv = reinterpret_cast<T*>(p.y_view);
        for (int r = 0; r < KR; ++r) {
          const int64_t o = o0 + r;
          if (o >= y_lo && o < y_hi) yv[o] = SlowPath<Kind>::eval(p, xg + o + dxy);
        }
      } else if (warp_full && p.has_y_map) {
        const int buf = kStagingBufs == 1 ? 0 : (it & 1);
        if (lane == 0) bulk_wait_read<kStagingBufs - 1>();
        __syncwarp();
        const uint32_t base = my_staging_s + buf * kStagingBytes;
#pragma unroll
        for (int c = 0; c < KR / 4; ++c) {
          const uint32_t off = swz128((uint32_t)row_in_warp * 128u + 64u * half + 16u * c);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + off),
                       "r"(bitcast<uint32_t>(y[4 * c + 0])), "r"(bitcast<uint32_t>(y[4 * c + 1])),
                       "r"(bitcast<uint32_t>(y[4 * c + 2])), "r"(bitcast<uint32_t>(y[4 * c + 3]))
                       : "memory");
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&p.tm_y, 0, (int32_t)wrow0, my_staging + buf * kStagingBytes);
          bulk_commit();
        }
      } else {
        T* yv = reinterpret_cast<T*>(p.y_view);
#pragma unroll
        for (int r = 0; r < KR; ++r) {
          const int64_t o = o0 + r;
          if (o >= y_lo && o < y_hi) yv[o] = y[r];
        }
      }
    }
  }
  if (lane == 0) bulk_wait_all();
}

// ------------------------------------------------------------- host launch
template <class Kind>
static cudaError_t launch_kind(Slide1DParams& p, cudaStream_t stream, int grid) {
  constexpr int KR = Kind::kRt;
  constexpr int kWarpRows = KR == 32 ? 32 : 16;
  constexpr int kTileRows = kWarps * kWarpRows;
  constexpr int kStagingBytes = kWarpRows * 128;
  const int span = Kind::kSpan >= 0 ? Kind::kSpan : (int)p.w + 20;
  p.span = span;
  p.tiles_per_row = (p.L / 32 + 2 + kTileRows - 1) / kTileRows;
  p.ntiles = p.batch * p.tiles_per_row;
  if (p.has_y_map && kWarpRows != 16 && !encode_rows_map(&p.tm_y, p.y_view, p.y_rows, kWarpRows))
    p.has_y_map = 0;
  const int max_halo_rows = (32 * (kTileRows - 1) + 31 + 31 + span) / 32 + 1 - kTileRows;
  const int halo_cap =
      max_halo_rows > 0 ? ((max_halo_rows + kHaloBoxRows - 1) / kHaloBoxRows) * kHaloBoxRows : 0;
  p.stage_bytes = (uint32_t)(kTileRows + halo_cap) * 128u;
  const size_t fixed = (size_t)kWarps * kStagingBufs * kStagingBytes + 2 * kBSBytes + kStageAlign +
                       16 * kMaxStages + sizeof(TileHdr) * kMaxStages + 256;
  int S = kMaxStages;
  while (S > 2 && (size_t)S * p.stage_bytes + fixed > (size_t)kSmemBudget) --S;
  if ((size_t)S * p.stage_bytes + fixed > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  p.stages = S;
  const size_t smem = (size_t)S * p.stage_bytes + fixed;
  auto kfn = slide1d_tma_kernel<Kind>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  const int64_t g = launch_grid(p.ntiles, grid, p.clc);
  kfn<<<(unsigned)g, kThreads, smem, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv_tma(Slide1DParams& p, int KT, cudaStream_t stream, int grid) {
  switch (KT) {
    case 1: return launch_kind<ConvKind<1, 16>>(p, stream, grid);
    case 2: return launch_kind<ConvKind<2, 16>>(p, stream, grid);
    case 3: return launch_kind<ConvKind<3, 16>>(p, stream, grid);
    case 4: return launch_kind<ConvKind<4, 16>>(p, stream, grid);
    case 5: return launch_kind<ConvKind<5, 16>>(p, stream, grid);
    case 7: return launch_kind<ConvKind<7, 16>>(p, stream, grid);
    case 8: return launch_kind<ConvKind<8, 16>>(p, stream, grid);
    case 15: return launch_kind<ConvKind<15, 16>>(p, stream, grid);
    case 16: return launch_kind<ConvKind<16, 16>>(p, stream, grid);
    case 24: return launch_kind<ConvKind<24, 32>>(p, stream, grid);
    case 31: return launch_kind<ConvKind<31, 32>>(p, stream, grid);
    case 32: return launch_kind<ConvKind<32, 32>>(p, stream, grid);
    case 48: return launch_kind<ConvKind<48, 32>>(p, stream, grid);
    case 63: return launch_kind<ConvKind<63, 32>>(p, stream, grid);
    case 64: return launch_kind<ConvKind<64, 32>>(p, stream, grid);
    default: return cudaErrorInvalidValue;
  }
}

template <class Op>
static cudaError_t launch_pool_op(Slide1DParams& p, int P, cudaStream_t stream, int grid) {
  if (p.w >= 48 && p.w <= 16 + 16 * 64) return launch_kind<PoolBlockKind<Op>>(p, stream, grid);
  switch (P) {
    case 1: return launch_kind<PoolKind<Op, 1>>(p, stream, grid);
    case 2: return launch_kind<PoolKind<Op, 2>>(p, stream, grid);
    case 4: return launch_kind<PoolKind<Op, 4>>(p, stream, grid);
    case 8: return launch_kind<PoolKind<Op, 8>>(p, stream, grid);
    case 16: return launch_kind<PoolKind<Op, 16>>(p, stream, grid);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pool_tma(Slide1DParams& p, int op, int dtype, int P, cudaStream_t stream,
                            int grid) {
  if (P > 16) P = 16;
  if (op == kOpSum && dtype == 1) return launch_pool_op<OpSumI32>(p, P, stream, grid);
  if (op == kOpSum && dtype == 0) return launch_pool_op<OpSumF32>(p, P, stream, grid);
  if (op == kOpMax && dtype == 1) return launch_pool_op<OpMaxI32>(p, P, stream, grid);
  if (op == kOpMax && dtype == 0) return launch_pool_op<OpMaxF32>(p, P, stream, grid);
  if (op == kOpMin && dtype == 1) return launch_pool_op<OpMinI32>(p, P, stream, grid);
  if (op == kOpMin && dtype == 0) return launch_pool_op<OpMinF32>(p, P, stream, grid);
  return cudaErrorInvalidValue;
}

}  // namespace ss
