// conv_tc.cu -- conv1d on the 5th-generation tensor cores (SURVEY 8f NEXT #2:
// the Conclusion's "small matrix multiplication" reformulation, PAPER.md
// l.228), for filters long enough that the FP32 FMA pipe, not HBM, bounds the
// FFMA2 tile kernel (k = 63 runs at ~0.65 of the FP32 peak there).
//
// Formulation.  The sliding dot product (Sec. 2.5, l.86-87) over a block of
// 128 consecutive outputs is a matrix product with a Toeplitz matrix:
//     D[r][m] = sum_kk A[r][kk] * B[m][kk] = y(P0 + 128 m + r)
//     A[r][kk] = f[kk - r]                (128 x K, K = 127 + k rounded to 8)
//     B[m][kk] = x(P0 + 128 m + kk)        (NC chunks of the input, K-major)
// A (the filter, fixed) lives in tensor memory for the whole kernel; B is the
// input itself, staged by TMA straight from HBM -- K-atom a of chunk m is the
// 128-B input row 4m + a, so a 3-D tensor map with strides {512 B, 128 B}
// lays the overlapping rows out as the canonical SWIZZLE_128B K-major operand
// (no im2col copy in HBM; the 1.5x overlap is re-read from L2 only).
//
// fp32 accuracy with TF32 MMAs (kind::tf32, fp32 accumulation in TMEM):
// the tensor core truncates fp32 operands to TF32 (measured:
// tools/ubench/tc_conv_probe.cu); with x = xh + xl, xh = trunc(x), xl = x - xh
// (exact), and likewise f = fh + fl:
//   mixed (default): per K-step of 8 kk, ONE kind::f16 MMA of K = 16 computes
//     the correction [bf16(xh) | bf16(xl)] . [bf16(fl) | bf16(fh)], then
//     D += xh fh (kind::tf32): two MMAs instead of three.  Per-product error
//     <= ~2^-18 |x f| (bf16 rounding of the two 2^-10-sized correction terms,
//     plus the dropped xl fl), inside BASELINE.json's 1e-5 sum|x f| + 1e-6
//     (measured worst err / bound 0.27 over tools/tc_conv_check.py parity).
//     The 16-bit A operand layout in TMEM (column c = K indices 2c, 2c + 1) is
//     measured by tools/ubench/tc_bf16_tmem_probe.cu.
//   3xTF32 (SS_CONV_TC_MIXED=0): D += xh fl + xl fh + xh fh, ~3 * 2^-22 (worst
//     err / bound 0.08).
// The Toeplitz rows of fh and of the correction (fl, or bf16 {fl | fh}) are
// written to TMEM once; the split warps build the per-tile correction operand
// (xl, or bf16 {xh | xl}) in a second smem ring.
//
// Warp roles (persistent CTA per SM, 576 threads):
//   warp 0      TMA producer (one lane): 3-D box {32, NC, 3} per K-atom group;
//               starts streaming while the other roles set up TMEM; claims
//               tiles from the launch's dynamic counter slot (ss_internal.h),
//               so SMs that run faster take more tiles
//   warp 1      MMA issuer (one elected lane, warp-uniform operands)
//   warps 2-9   split: correction operand of each staged group
//   warps 10-17 epilogue: TMEM -> registers (tcgen05.ld 32x32b) -> one
//               coalesced 128-B store per warp per chunk column (a tile
//               inside one batch row stores with immediate offsets; tiles
//               crossing a row edge mask outputs whose window leaves the row)
// Pipelines: hi stages (TMA -> split/MMA), lo buffers (split -> MMA), two
// TMEM accumulators (MMA -> epilogue), a ring of tile ids (producer -> all).
// A transposed formulation (x as the A operand from one contiguous TMA tile
// by row shifts, the filter Toeplitz as an N = 32 B operand; K = 96) was
// built and measured slower (160 us vs 117 us at k = 63): with A from shared
// memory every N = 32 MMA re-reads a 4 KB A slice.
#include <cstdint>

#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"


namespace ss {

namespace {

constexpr int kTcWarpProducer = 0;
constexpr int kTcWarpMma = 1;
constexpr int kTcWarpSplit0 = 2;
constexpr int kTcSplitWarps = 8;
constexpr int kTcWarpEpi0 = kTcWarpSplit0 + kTcSplitWarps;
constexpr int kTcEpiWarps = 8;  // two per TMEM lane quarter, each half of the chunk columns
constexpr int kTcThreads = 32 * (kTcWarpEpi0 + kTcEpiWarps);
// Tile ids travel producer -> consumers through a smem ring: the split warps
// read slot it % kTcTileRing after their `full` wait for the tile's first group
// and the MMA warp after its `lofull` wait (the existing acquire chain), the
// epilogue warps through their own tfull / tempty barriers.  The producer
// cannot run kTcTileRing tiles ahead of the MMA warp (its hi ring holds fewer).
constexpr int kTcTileRing = 16;
constexpr int kTcTileReaders = kTcEpiWarps;  // warps that release a ring slot

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);  // start address
  d |= (uint64_t)1 << 16;                  // LBO (ignored for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, K-major both, N, M.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// kind::f16 instruction descriptor with bf16 A and B (format code 1).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// {lo, hi} -> one 32-bit word of two bf16 (round to nearest even); lo = lower K index
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// D[tmem] (+)= A[tmem] * B[smem desc]; issued by one elected lane of the
// calling (converged) warp.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on `bar` when every tcgen05 op issued so far by this thread is done.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mbarrier wait without a suspend-time hint: a warp parked on a hinted
// try_wait is not woken promptly by tcgen05.commit arrivals (measured: 10 us
// per tile), so these pipelines poll.
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace

// Debug trace (SS_CONV_TC_TRACE): CTA 0 records clock64() per tile and role
// event into p.trace[tile_iter * 8 + event].
#define TC_TRACE(it, ev)                                                                 \
  do {                                                                                   \
    if (p.trace && blockIdx.x == 0 && (it) < 63) p.trace[(it) * 8 + (ev)] = clock64(); \
  } while (0)
// row 63: {globaltimer, clock64} at kernel entry, after setup, and at exit (thread 0 of CTA 0)
// entries [512 + 2 b] / [512 + 2 b + 1]: globaltimer at entry / exit of CTA b (b < 256)
__device__ __forceinline__ void tc_trace_stamp(unsigned long long* tr, int slot) {
  if (tr && threadIdx.x == (slot == 2 ? 32 * kTcWarpMma : 0)) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    if (blockIdx.x == 0) {
      tr[63 * 8 + 2 * slot] = g;
      tr[63 * 8 + 2 * slot + 1] = clock64();
    }
    if (slot != 1 && blockIdx.x < 256) tr[512 + 2 * blockIdx.x + (slot == 2 ? 1 : 0)] = g;
  }
}

// Fixed MMA depth: K = 192 (6 K-atoms of 32, 24 K-steps of 8) serves every
// k <= 65 (the Toeplitz is zero beyond k); the pipelines move whole tiles (one
// TMA box of 4 K-atom blocks, one split pass, 24 K-steps of MMAs per sync).
constexpr int kTcK = 192;
// accumulator buffers per chunk count: NC = 64 keeps two TMEM
// accumulators (epilogue of tile i overlaps the MMAs of tile i+1); NC = 128
// (N = 128 MMAs: half the issue count) has room for one, drained by the
// epilogue into registers before the next tile's first MMA.
template <int NC> struct TcShape {
  static constexpr int kBlockRows = NC + 8;  // chunks per staged K-atom block (one extra, 1024-B aligned)
  static constexpr int kDBufs = NC == 128 ? 1 : 2;
};

// KA = MMA K-atoms: 6 (K = 192) for k <= 65, 5 (K = 160) for k <= 33
template <int NC, bool kMixed, int KA>
__global__ void __launch_bounds__(kTcThreads, 1) conv_tc_kernel(const __grid_constant__ ConvTCParams p) {
  static_assert(KA == 5 || KA == 6, "K-atoms 4 and 5 are read from blocks 0 and 1");
  constexpr int kK = 32 * KA;
  static_assert(NC % 32 == 0 && NC <= 128, "NC/2 columns per epilogue warp, loaded 16 at a time");
  constexpr int kBlockRows = TcShape<NC>::kBlockRows, ND = TcShape<NC>::kDBufs;
  extern __shared__ __align__(16) uint8_t smem_raw[];  // aligned to 1024 by hand (slack in conv_tc_smem_bytes)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // shared-space pointer arithmetic
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Rings of tile stages: 4 K-atom blocks of kBlockRows chunks x 128 B.  K-atoms 4 and 5 of
  // chunk m are atoms 0 and 1 of chunk m + 1, i.e. blocks 0 and 1 read one row further down
  // (a whole-row shift of the operand start stays a canonical SWIZZLE_128B operand).
  const int SH = p.hi_stages, SL = p.lo_bufs;
  constexpr uint32_t kAtomBytes = kBlockRows * 128u;
  constexpr uint32_t kSlot = 4 * kAtomBytes;
  static_assert(kAtomBytes % 1024 == 0, "blocks stay 1024-B aligned");
  uint8_t* hi = smem;
  uint8_t* lo = smem + (size_t)SH * kSlot;
  uint64_t* bars = reinterpret_cast<uint64_t*>(lo + (size_t)SL * kSlot);
  uint64_t* full = bars;                // [SH] TMA -> split, MMA
  uint64_t* empty = full + SH;          // [SH] MMA commit -> producer
  uint64_t* lofull = empty + SH;        // [SL] split -> MMA
  uint64_t* loempty = lofull + SL;      // [SL] MMA commit -> split
  uint64_t* dfull = loempty + SL;       // [ND] MMA commit -> epilogue
  uint64_t* dempty = dfull + 2;         // [ND] epilogue -> MMA
  uint64_t* tfull = dempty + 2;         // [kTcTileRing] producer -> epilogue: tile id published
  uint64_t* tempty = tfull + kTcTileRing;  // [kTcTileRing] the epilogue warps have read it
  int64_t* tring = reinterpret_cast<int64_t*>(tempty + kTcTileRing);  // tile ids (-1: no more tiles)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tring + kTcTileRing);
  float* fsm = reinterpret_cast<float*>(tslot + 4);  // [2][kConvTcMaxK + 256] zero-padded hi/lo taps

  __shared__ ClcSmem clc;
  // ---- setup: barriers, TMEM, taps -----------------------------------------
  tc_trace_stamp(p.trace, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < SH; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    for (int i = 0; i < SL; ++i) { mbar_init(lofull + i, kTcSplitWarps); mbar_init(loempty + i, 1); }
    for (int i = 0; i < ND; ++i) { mbar_init(dfull + i, 1); mbar_init(dempty + i, kTcEpiWarps); }
    for (int i = 0; i < kTcTileRing; ++i) { mbar_init(tfull + i, 1); mbar_init(tempty + i, kTcTileReaders); }
    clc_init(&clc);
    fence_mbar_init();
    prefetch_tmap(&p.tm_b);
  }
  // fsm[0][128 + t] = hi(f_t), fsm[1][128 + t] = lo(f_t); zeros around, so the
  // Toeplitz row r reads fsm[.][128 + kk - r] without bounds checks.
  constexpr int kFPad = kConvTcMaxK + 256;
  static_assert(128 + kTcK <= kFPad, "Toeplitz reads stay inside fsm");  // (kK <= kTcK)
  for (int i = threadIdx.x; i < kFPad; i += kTcThreads) {
    const int t = i - 128;
    const float f = (t >= 0 && t < p.k) ? p.taps[t] : 0.0f;
    const float fh = tf32_trunc(f);
    fsm[i] = fh;
    fsm[kFPad + i] = tf32_trunc(f - fh);
  }
  if (warp == kTcWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // the producer starts streaming now; the other roles wait (named barrier 1)
  // until the Toeplitz operands are in TMEM
  if (warp == kTcWarpProducer) {
    tc_trace_stamp(p.trace, 1);
    if (lane == 0) {
      // tiles: CTA b starts with tile b, then claims tiles by cluster launch
      // control (dynamic: SMs that run faster take more tiles) or strides by gridDim.x
      int s = 0;
      uint32_t ph = 0, cph = 0;
      int64_t t = blockIdx.x;
      if (p.clc && t < p.ntiles) clc_request(&clc);
      for (int it = 0;; ++it) {
        const int ts = it % kTcTileRing;
        bar_wait(tempty + ts, ((uint32_t)(it / kTcTileRing) & 1u) ^ 1u);
        if (t < 0) t = p.ntiles;
        tring[ts] = t < p.ntiles ? t : -1;
        mbar_arrive(tfull + ts);
        if (t >= p.ntiles) {
          // end marker for the split warps (and, through them, the MMA warp): complete
          // the next `full` phase with no data
          bar_wait(empty + s, ph ^ 1);
          mbar_arrive(full + s);
          break;
        }
        bar_wait(empty + s, ph ^ 1);
        mbar_arrive_expect_tx(full + s, kSlot);
        tma_load_3d(hi + (size_t)s * kSlot, &p.tm_b, 0, (int32_t)(t * NC), 0, full + s);
        if (++s == SH) { s = 0; ph ^= 1; }
        TC_TRACE(it, 0);
        if (p.clc) {
          t = clc_wait(&clc, cph);  // requested one tile ahead
          if (t >= 0) clc_request(&clc);
        } else {
          t += gridDim.x;
        }
      }
    }
    __syncwarp();
    __syncthreads();  // matches the final barrier of the other roles
    return;
  }
  const uint32_t tmem = *tslot;
  // TMEM columns: A_hi [0, 192), A_lo [192, 384), accumulators [512 - 2 NC, 512)
  const uint32_t a_hi = tmem, a_lo = tmem + (uint32_t)kTcK;
  const uint32_t d_col0 = tmem + 512u - (uint32_t)(ND * NC);
  static_assert(2 * kTcK + ND * NC <= 512, "TMEM budget");

  auto ring_tile = [&](int it) -> int64_t { return *reinterpret_cast<volatile int64_t*>(tring + it % kTcTileRing); };
  // epilogue side of the tile-id ring: read slot it % kTcTileRing after its
  // tfull phase, then (lane 0) release it
  auto next_tile = [&](int it) -> int64_t {
    const int ts = it % kTcTileRing;
    bar_wait(tfull + ts, (uint32_t)(it / kTcTileRing) & 1u);
    const int64_t t = *reinterpret_cast<volatile int64_t*>(tring + ts);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(tempty + ts);
    return t;
  };

  if (warp >= kTcWarpEpi0 && warp < kTcWarpEpi0 + 4) {
    // Toeplitz rows of fh / fl into TMEM: lane r holds A[r][kk] = f[kk - r].
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int r = 32 * q + lane;
    const uint32_t lanebits = (uint32_t)(32 * q) << 16;
#pragma unroll 1
    for (int c = 0; c < kK; c += 32) {
      float vh[32], vl[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int t = 128 + c + j - r;  // in [1, 128 + K) -> inside fsm
        vh[j] = fsm[t];
        vl[j] = fsm[kFPad + t];
      }
      tmem_st32(a_hi + lanebits + (uint32_t)c, vh);
      if constexpr (kMixed) {
        // bf16 correction operand, K-step kb = (c + 8 j8) / 8: columns 0-3 hold fl(kk - r)
        // for kk = 8 kb + 0..7 (pairs with bf16(xh)), columns 4-7 hold fh(kk - r) (pairs with
        // bf16(xl)); column c holds K indices 2c (low half) and 2c + 1 (measured:
        // tools/ubench/tc_bf16_tmem_probe.cu)
        float vc[32];
#pragma unroll
        for (int j8 = 0; j8 < 4; ++j8)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            vc[8 * j8 + u] = __uint_as_float(pack_bf16(vl[8 * j8 + 2 * u], vl[8 * j8 + 2 * u + 1]));
            vc[8 * j8 + 4 + u] = __uint_as_float(pack_bf16(vh[8 * j8 + 2 * u], vh[8 * j8 + 2 * u + 1]));
          }
        tmem_st32(a_lo + lanebits + (uint32_t)c, vc);
      } else {
        tmem_st32(a_lo + lanebits + (uint32_t)c, vl);
      }
    }
    tmem_wait_st();
  }
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"n"(kTcThreads - 32) : "memory");
  tc_fence_after();

  if (warp == kTcWarpMma) {
    constexpr uint32_t idesc = idesc_tf32(128, NC);
    constexpr uint32_t idesc_c = idesc_bf16(128, NC);
    // warp-uniform bases; descriptors advance by adding to the start-address field
    const uint64_t dhi0 = sw128_desc(__shfl_sync(0xffffffffu, smem_u32(hi), 0));
    const uint64_t dlo0 = sw128_desc(__shfl_sync(0xffffffffu, smem_u32(lo), 0));
    const uint32_t ahi = __shfl_sync(0xffffffffu, a_hi, 0), alo = __shfl_sync(0xffffffffu, a_lo, 0);
    const uint32_t dc0 = __shfl_sync(0xffffffffu, d_col0, 0);
    int s = 0, l = 0, d = 0;
    uint32_t ph = 0, lph = 0, dph = 0;
    int it = 0;
    for (;; ++it) {
      // the split warps observed `full` (TMA data landed) before arriving on
      // `lofull`, so one wait covers both operands and the tile id (acquire chain)
      bar_wait(lofull + l, lph);
      if (ring_tile(it) < 0) break;
      bar_wait(dempty + d, dph ^ 1);
      const uint32_t dcol = dc0 + (uint32_t)(d * NC);
      if (lane == 0) TC_TRACE(it, 3);
      tc_fence_after();
      const uint64_t dh = dhi0 + (uint64_t)((s * kSlot) >> 4), dl = dlo0 + (uint64_t)((l * kSlot) >> 4);
#pragma unroll
      for (int kb = 0; kb < 4 * KA; ++kb) {
        // K-step kb: K-atom a = kb / 4 -> block a (a < 4) or block a - 4 one row down; 32-B column block kb % 4
        const int a = kb >> 2;
        const uint64_t off = (uint64_t)(((uint32_t)(a & 3) * kAtomBytes + (a >= 4 ? 128u : 0u) + 32u * (kb & 3)) >> 4);
        // small terms first: xh*fl and xl*fh, then xh*fh
        if constexpr (kMixed) {
          // one bf16 MMA (K = 16: [bf16(xh) | bf16(xl)] . [fl | fh] over these 8 kk)
          mma_bf16_ts(dcol, alo + 8u * (uint32_t)kb, dl + off, idesc_c, kb > 0 ? 1u : 0u);
        } else {
          mma_tf32_ts(dcol, alo + 8u * (uint32_t)kb, dh + off, idesc, kb > 0 ? 1u : 0u);
          mma_tf32_ts(dcol, ahi + 8u * (uint32_t)kb, dl + off, idesc, 1u);
        }
        mma_tf32_ts(dcol, ahi + 8u * (uint32_t)kb, dh + off, idesc, 1u);
      }
      mma_commit(empty + s);
      mma_commit(loempty + l);
      if (++s == SH) { s = 0; ph ^= 1; }
      if (++l == SL) { l = 0; lph ^= 1; }
      mma_commit(dfull + d);
      if (lane == 0) TC_TRACE(it, 4);
      if (++d == ND) { d = 0; dph ^= 1; }
    }
  } else if (warp < kTcWarpEpi0) {
    // split warps: the correction operand of a staged tile (rows 0..NC of each of the 4 blocks;
    // the rows past NC are never read), position by position
    const int st = threadIdx.x - 32 * kTcWarpSplit0;  // 0 .. 32 kTcSplitWarps - 1
    constexpr int kRowsUsed = NC + 1;
    int s = 0, l = 0;
    uint32_t ph = 0, lph = 0;
    for (int it = 0;; ++it) {
      bar_wait(full + s, ph);
      bar_wait(loempty + l, lph ^ 1);
      if (ring_tile(it) < 0) {  // end marker: pass it on to the MMA warp
        __syncwarp();
        if (lane == 0) mbar_arrive(lofull + l);
        break;
      }
      if (st == 0) TC_TRACE(it, 2);
      const uint32_t src = smem_u32(hi + (size_t)s * kSlot), dst = smem_u32(lo + (size_t)l * kSlot);
      if constexpr (kMixed) {
        // per 32-B block (one K-step of 8 kk in one 128-B row): logical halves
        // [bf16(xh) x 8 | bf16(xl) x 8].  SWIZZLE_128B XORs the 16-B unit index
        // with the row's low 3 bits, so the two units of a 32-B block stay
        // together and swap order on odd rows: the unit that held x[kk0..kk0+3]
        // receives the bf16(xh), the other the bf16(xl).  (Block bases are
        // multiples of 1024 B, so the row parity is the in-block row's.)
        constexpr int kItems = 4 * kRowsUsed * 4;
#pragma unroll
        for (int i = st; i < kItems; i += 32 * kTcSplitWarps) {
          const int blk = i / (kRowsUsed * 4), rem = i - blk * (kRowsUsed * 4);
          const uint32_t o = (uint32_t)blk * kAtomBytes + 32u * (uint32_t)rem;  // rem = row * 4 + unit pair
          float4 a = lds128(src + o), b = lds128(src + o + 16u);
          const bool odd = (rem >> 2) & 1;
          if (odd) { const float4 t = a; a = b; b = t; }
          const float xv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float h0 = tf32_trunc(xv[2 * u]), h1 = tf32_trunc(xv[2 * u + 1]);
            hw[u] = pack_bf16(h0, h1);
            lw[u] = pack_bf16(xv[2 * u] - h0, xv[2 * u + 1] - h1);
          }
          const uint32_t dh_ = dst + o + (odd ? 16u : 0u), dl_ = dst + o + (odd ? 0u : 16u);
          sts128(dh_, __uint_as_float(hw[0]), __uint_as_float(hw[1]), __uint_as_float(hw[2]), __uint_as_float(hw[3]));
          sts128(dl_, __uint_as_float(lw[0]), __uint_as_float(lw[1]), __uint_as_float(lw[2]), __uint_as_float(lw[3]));
        }
      } else {
        constexpr int kItems = 4 * kRowsUsed * 8;  // 16-B units
#pragma unroll
        for (int i = st; i < kItems; i += 32 * kTcSplitWarps) {
          const int blk = i / (kRowsUsed * 8), rem = i - blk * (kRowsUsed * 8);
          const uint32_t o = (uint32_t)blk * kAtomBytes + 16u * (uint32_t)rem;
          const float4 v = lds128(src + o);
          sts128(dst + o, v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                 v.w - tf32_trunc(v.w));
        }
      }
      fence_proxy_async_smem();  // generic-proxy writes -> tensor core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(lofull + l);
      if (st == 0) TC_TRACE(it, 5);
      if (++s == SH) { s = 0; ph ^= 1; }
      if (++l == SL) { l = 0; lph ^= 1; }
    }
  } else {
    // epilogue: lane r of quarter q owns output row r = 32q + lane of each chunk;
    // warp half h stores chunk columns [h NC/2, (h+1) NC/2)
    constexpr int NH = NC / 2;
    const int q = warp & 3;
    const int h = (warp - kTcWarpEpi0) >> 2;
    const int r = 32 * q + lane;
    const uint32_t lanebits = (uint32_t)(32 * q) << 16;
    int d = 0;
    uint32_t dph = 0;
    int it = 0;
    bool did_last = false;  // this CTA computed the last tile: it also does the array tail
    for (;; ++it) {
      const int64_t t = next_tile(it);
      if (t < 0) break;
      did_last |= t == p.ntiles - 1;
      bar_wait(dfull + d, dph);
      if (warp == kTcWarpEpi0 && lane == 0) TC_TRACE(it, 7);
      tc_fence_after();
      uint32_t v[NH];
#pragma unroll
      for (int c = 0; c < NH; c += 16) tmem_ld16(d_col0 + lanebits + (uint32_t)(d * NC + h * NH + c), v + c);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty + d);
      // chunk c covers view positions 128 (t NC + c) + [0, 128)
      const int64_t m0 = t * NC + h * NH;
      const int64_t cmax = p.m_ext - m0 < NH ? p.m_ext - m0 : NH;  // chunks inside the map
      if (cmax <= 0) {
        // nothing (tail chunks are done below)
      } else {
        // warp-uniform fast path: every position of these columns is a valid
        // output of one batch row
        const int64_t q0 = 128 * m0 - p.shift_x, q1 = 128 * (m0 + cmax) - 1 - p.shift_x;
        const int64_t b0 = q0 >= 0 ? q0 / p.N : -1;
        const bool fast = cmax == NH && b0 >= 0 && q1 - b0 * p.N < p.L_int;
        if (fast) {
          float* __restrict__ yr = p.y + b0 * p.y_pitch + p.y_off + (q0 - b0 * p.N) + r;
#pragma unroll
          for (int c = 0; c < NH; ++c) yr[128 * c] = __uint_as_float(v[c]);
        } else {
          int64_t qq = q0 + r;
#pragma unroll
          for (int c = 0; c < NH; ++c, qq += 128) {
            if (c < cmax && qq >= 0) {
              const int64_t b = qq / p.N, i = qq - b * p.N;
              if (b < p.batch && i < p.L_int) p.y[b * p.y_pitch + p.y_off + i] = __uint_as_float(v[c]);
            }
          }
        }
      }
      if (++d == ND) { d = 0; dph ^= 1; }
    }
    // view positions beyond the tensor map (array tail, < 320): direct FMA windows on all
    // 256 epilogue threads, the window's loads issued together (a serial load->FMA chain
    // here cost ~8 us at the end of the kernel)
    if (did_last) {  // (with CLC the grid's last CTA may never run: it can be canceled)
      const float* __restrict__ xv = p.x_view;
      const int e = 32 * (warp - kTcWarpEpi0) + lane;
      for (int64_t pos = 128 * p.m_ext + e; pos < p.total_view; pos += 32 * kTcEpiWarps) {
        const int64_t qq = pos - p.shift_x;
        if (qq < 0) continue;
        const int64_t b = qq / p.N, i = qq - b * p.N;
        if (b >= p.batch || i >= p.L_int) continue;
        float xw[kConvTcMaxK];
#pragma unroll
        for (int j = 0; j < kConvTcMaxK; ++j) xw[j] = j < p.k ? __ldg(xv + pos + j) : 0.0f;
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < kConvTcMaxK; ++j)
          if (j < p.k) acc = __fmaf_rn(p.taps[j], xw[j], acc);
        p.y[b * p.y_pitch + p.y_off + i] = acc;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_trace_stamp(p.trace, 2);
  if (warp == kTcWarpMma) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

size_t conv_tc_smem_bytes(int hi_slots, int lo_slots, int nc) {
  const size_t stage = 4 * (size_t)(nc + 8) * 128;
  return 1024 + (size_t)(hi_slots + lo_slots) * stage + 8 * (2 * hi_slots + 2 * lo_slots + 4) +
         24 * kTcTileRing + 16 + 2 * sizeof(float) * (kConvTcMaxK + 256);
}

template <int NC, bool kMixed, int KA>
static cudaError_t launch_nc(ConvTCParams& p, cudaStream_t stream, int grid) {
  // lo ring: two tile stages (the split runs ahead of the MMAs); hi ring: every
  // remaining stage (TMA prefetch depth)
  if (p.lo_bufs < 1) p.lo_bufs = 2;
  int SH = kTcTileRing - 4;
  while (SH > 2 && conv_tc_smem_bytes(SH, p.lo_bufs, NC) > (size_t)kSmemBudget) --SH;
  if (conv_tc_smem_bytes(SH, p.lo_bufs, NC) > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  p.hi_stages = SH;
  p.ntiles = (p.m_ext + NC - 1) / NC;
  auto kfn = conv_tc_kernel<NC, kMixed, KA>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  const int64_t g = launch_grid(p.ntiles, grid, p.clc);
  kfn<<<(unsigned)g, kTcThreads, conv_tc_smem_bytes(SH, p.lo_bufs, NC), stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv_tc(ConvTCParams& p, int nc, cudaStream_t stream, int grid) {
  // K = 32 KA >= 127 + k: 160 covers k <= 33, 192 covers k <= 65
  const int ka = 127 + p.k <= 160 ? 5 : 6;
  const bool mixed = p.mixed != 0;
  if (nc != 64) return cudaErrorInvalidValue;
#define SS_TC_LAUNCH(NC_, M_, KA_) \
  if (nc == NC_ && mixed == M_ && ka == KA_) return launch_nc<NC_, M_, KA_>(p, stream, grid);
  SS_TC_LAUNCH(64, true, 5) SS_TC_LAUNCH(64, true, 6) SS_TC_LAUNCH(64, false, 5) SS_TC_LAUNCH(64, false, 6)
#undef SS_TC_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace ss
