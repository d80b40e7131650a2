// conv_mc.cu -- multi-channel 1-D convolution (with C_in > 1
// the sliding dot product of Sec. 2.5, becomes a real
// contraction): y[b][i][co] = sum_{j<k} sum_ci w[co][ci][j] x[b][i+j][ci],
// channels-last bf16 activations and weights, fp32 accumulation and output
// (reading R18).
//
// Tensor-core formulation (kind::f16, BF16 x BF16 -> F32 in TMEM): a tile is
// 128 consecutive positions (M = 128, TMEM lanes) x all C_out channels
// (N = C_out).  For tap j the A operand is the staged input tile shifted by j
// positions -- channels-last, one position's C_in channels are one 128-B
// K-atom row (per 64 channels), so the shift is a start-address offset of j
// rows in the canonical SWIZZLE_128B K-major layout (no im2col) -- and the B
// operand is w[:, :, j] (C_out x C_in, K-major), staged once per CTA.  The k
// taps x C_in/16 K-steps accumulate into one TMEM accumulator:
//     D[m][co] += sum_ci X[p0 + m + j][ci] W_j[co][ci]
// Products of bf16 values are exact in fp32; accumulation is fp32.
//
// Warps (persistent CTA per SM, 320 threads): 0 TMA producer (3-D box over
// [flat position][atom][64] of x per tile into a 3-stage ring), 1 MMA issuer
// (one elected lane), 2-9 epilogue (tcgen05.ld 16x256b: four lanes hold 32
// contiguous bytes of an output row, so stores are whole sectors; channels
// split over two warps per lane quarter; positions whose window leaves their
// batch row are masked).  Two TMEM accumulators.
#include <cstdint>
#include <cstdlib>

#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kMcThreads = 320;
constexpr int kMcWarpMma = 1;
constexpr int kMcWarpEpi0 = 2;
constexpr int kMcEpiWarps = 8;
constexpr int kMcStages = 3;
constexpr int kMcRing = 8;    // tile-id ring entries

__device__ __forceinline__ uint64_t sw128_desc_mc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// kind::f16 instruction descriptor: D f32, A bf16, B bf16, both K-major, N, M.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mc_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mc_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ __attribute__((unused)) void mc_tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
// 16 TMEM lanes x 256 bits: thread t gets columns 2(t%4), 2(t%4)+1 of lanes
// t/4 (v0, v1) and t/4 + 8 (v2, v3) -> four threads hold 32 contiguous bytes
// of a row, so a warp's stores are whole 32-B sectors.
__device__ __forceinline__ void mc_tmem_ld_16x256(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
}
// .x4 / .x8: the same pattern repeated over 4 / 8 consecutive 8-column blocks (registers 4 r .. 4 r + 3
// hold block r) -- one instruction per 16 lanes instead of one per 8 columns.
__device__ __forceinline__ void mc_tmem_ld_16x256_x4(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(taddr)
               : "memory");
}
template <int NB>
__device__ __forceinline__ void mc_tmem_ld_row_blocks(uint32_t taddr, uint32_t (*v)[4]) {
#pragma unroll
  for (int c = 0; c < NB; c += 4) mc_tmem_ld_16x256_x4(taddr + 8u * c, &v[c][0]);
}
__device__ __forceinline__ void tma_load_3d_mc(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                               int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d_mc(void* smem_dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                               int32_t c2, int32_t c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_5d_mc(void* smem_dst, const CUtensorMap* map, int32_t c1, int32_t c2,
                                               int32_t c3, int32_t c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace

template <int CIN, int COUT>
__global__ void __launch_bounds__(kMcThreads, 1) conv_mc_kernel(const __grid_constant__ ConvMcParams p) {
  constexpr int AT = CIN / 64;                        // K-atoms (64 bf16 = 128 B) per position
  const uint32_t kAtomBytes = (uint32_t)p.rows * 128u;  // one atom of a staged tile
  const uint32_t kStage = AT * kAtomBytes;
  constexpr uint32_t kWTap = AT * COUT * 128u;        // one tap of the weights
  constexpr int NH = COUT / 2;                        // epilogue columns per warp
  constexpr int kAccMax = 4;                          // TMEM accumulators: p.nacc <= 4, nacc * mblk * COUT <= 512
  const int kAcc = p.nacc, MB = p.mblk, TP = 128 * p.mblk;  // tile positions
  extern __shared__ __align__(16) uint8_t mc_raw[];  // aligned to 1024 by hand (slack in conv_mc_smem_bytes)
  uint8_t* smem = mc_raw + ((1024u - (smem_u32(mc_raw) & 1023u)) & 1023u);  // shared-space pointer arithmetic
  const int k = (int)p.k;
  const int kMcStages = p.stages;
  uint8_t* xs = smem;                                  // [stages][AT][rows][128 B]
  uint8_t* ws = smem + kMcStages * kStage;             // [k][AT][COUT][128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ws + (size_t)k * kWTap);
  uint64_t* full = bars;                               // [stages]
  uint64_t* empty = full + kMcStages;                  // [stages]
  uint64_t* dfull = empty + kMcStages;                 // [kAcc]
  uint64_t* dempty = dfull + kAccMax;                  // [kAcc]
  // tile ids, producer -> MMA (read after its `full` wait) and epilogue (own barrier pair);
  // the producer is at most kMcStages + kAcc tiles ahead of the epilogue
  uint64_t* tfull = dempty + kAccMax;                  // [kMcRing]
  uint64_t* tempty = tfull + kMcRing;                  // [kMcRing]
  int64_t* tring = reinterpret_cast<int64_t*>(tempty + kMcRing);  // [kMcRing][3]: tile, b0, i0
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tring + 3 * kMcRing);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ ClcSmem clc;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kMcStages; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
    for (int i = 0; i < kAcc; ++i) { mbar_init(dfull + i, 1); mbar_init(dempty + i, kMcEpiWarps); }
    for (int i = 0; i < kMcRing; ++i) { mbar_init(tfull + i, 1); mbar_init(tempty + i, kMcEpiWarps); }
    clc_init(&clc);
    fence_mbar_init();
    prefetch_tmap(&p.tm_x);
  }
  // weights: w[co][ci][j] (bf16) -> tap j, atom ci/64, row co, 16-B chunk (ci%64)/8 ^ (co%8);
  // input gradient: the staged w'[co][ci][j] is w[ci][co][k-1-j] (transposed and flipped).
  // The source is read in chunks of R1 outer rows with coalesced 16-B loads into the (still
  // unused) x ring, then each thread assembles whole 16-B destination units from 8 shared
  // loads: per-element index math with 8 warps cost ~6 us per CTA.
  {
    const uint16_t* __restrict__ w = static_cast<const uint16_t*>(p.w);
    const int D1 = p.bwd_in ? CIN : COUT, D2 = p.bwd_in ? COUT : CIN;  // outer / middle source dims
    const int row_elems = D2 * k;                                       // one outer row
    const int RS = row_elems * 2 + 4;  // padded scratch row (bytes): odd word stride, conflict-free gathers
    int R1 = D1;
    while (R1 > 8 && (size_t)R1 * RS > (size_t)kMcStages * kStage) R1 >>= 1;
    const bool chunked = (reinterpret_cast<uintptr_t>(w) & 15) == 0 && (size_t)R1 * RS <= (size_t)kMcStages * kStage;
    const uint32_t ws_s = smem_u32(ws), sc_s = smem_u32(xs);
    if (chunked) {
      const int q16 = row_elems / 8;  // 16-B pieces per source row
      for (int c0 = 0; c0 < D1; c0 += R1) {
        const uint4* __restrict__ src = reinterpret_cast<const uint4*>(w + (size_t)c0 * row_elems);
        const int n16 = R1 * q16;
        for (int base = 0; base < n16; base += 16 * kMcThreads) {
          uint4 v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int i = base + u * kMcThreads + (int)threadIdx.x;
            if (i < n16) v[u] = __ldg(src + i);
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int i = base + u * kMcThreads + (int)threadIdx.x;
            if (i < n16) {
              const int row = i / q16;
              const uint32_t a0 = sc_s + (uint32_t)(row * RS) + 16u * (uint32_t)(i - row * q16);
              asm volatile("st.shared.b32 [%0], %1;\n\tst.shared.b32 [%0+4], %2;\n\t"
                           "st.shared.b32 [%0+8], %3;\n\tst.shared.b32 [%0+12], %4;" ::"r"(a0),
                           "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                           : "memory");
            }
          }
        }
        __syncthreads();
        // destination units of this chunk, tap by tap: (co, 8 consecutive ci); fwd: ci-group fastest,
        // bwd: co fastest (both power-of-two extents: shifts only)
        const int gi = p.bwd_in ? R1 / 8 : CIN / 8;  // ci groups
        const int nco = p.bwd_in ? COUT : R1;        // co rows
        const int lg_fast = 31 - __clz(p.bwd_in ? nco : gi);
        const int lg_tap = 31 - __clz(nco * gi);
        const int units = k << lg_tap;
        {
#pragma unroll 4
          for (int e0 = threadIdx.x; e0 < units; e0 += kMcThreads) {
            const int j = e0 >> lg_tap, e = e0 & ((1 << lg_tap) - 1);
            const int fast = e & ((1 << lg_fast) - 1), slow = e >> lg_fast;
            int co, ci0;
            uint32_t s0, step;  // scratch address of element t = 0, stride between t
            if (p.bwd_in) {     // source (ci = c0 + 8 g + t, co, k-1-j)
              co = fast; ci0 = c0 + 8 * slow;
              s0 = sc_s + (uint32_t)(8 * slow * RS) + 2u * (uint32_t)(co * k + (k - 1 - j));
              step = (uint32_t)RS;
            } else {            // source (co = c0 + col, ci = 8 g + t, j)
              co = c0 + slow; ci0 = 8 * fast;
              s0 = sc_s + (uint32_t)(slow * RS) + 2u * (uint32_t)(ci0 * k + j);
              step = 2u * (uint32_t)k;
            }
            uint32_t h[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              uint16_t q;
              asm volatile("ld.shared.u16 %0, [%1];" : "=h"(q) : "r"(s0 + step * t) : "memory");
              h[t] = q;
            }
            const uint32_t off = (uint32_t)j * kWTap + (uint32_t)(ci0 >> 6) * (COUT * 128u) + (uint32_t)co * 128u +
                                 ((((uint32_t)(ci0 & 63) >> 3) ^ ((uint32_t)co & 7u)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ws_s + off), "r"(h[0] | (h[1] << 16)),
                         "r"(h[2] | (h[3] << 16)), "r"(h[4] | (h[5] << 16)), "r"(h[6] | (h[7] << 16))
                         : "memory");
          }
        }
        __syncthreads();  // scratch reused by the next chunk / the x ring
      }
    } else {  // unaligned weights: element by element
      const int total = COUT * CIN * k;
      for (int e = threadIdx.x; e < total; e += kMcThreads) {
        const int r = e / k, c1 = r / D2, c2 = r % D2, jj = e - r * k;
        const int co = p.bwd_in ? c2 : c1, ci = p.bwd_in ? c1 : c2, j = p.bwd_in ? k - 1 - jj : jj;
        const uint32_t off = (uint32_t)j * kWTap + (uint32_t)(ci >> 6) * (COUT * 128u) + (uint32_t)co * 128u +
                             ((((uint32_t)(ci & 63) >> 3) ^ ((uint32_t)co & 7u)) << 4) + 2u * (uint32_t)(ci & 7);
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(ws_s + off), "h"(__ldg(w + e)) : "memory");
      }
    }
  }
  fence_proxy_async_smem();  // generic-proxy weight writes -> tensor core reads
  if (warp == kMcWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const int64_t ntiles = p.ntiles;

  if (warp == 0) {
    if (lane == 0) {  // producer: tile b, then claims by cluster launch control (or + gridDim.x)
      int s = 0;
      uint32_t ph = 0, cph = 0;
      int64_t t = blockIdx.x;
      if (p.clc && t < ntiles) clc_request(&clc);
      for (int it = 0;; ++it) {
        const int ts = it % kMcRing;
        mbar_wait(tempty + ts, ((uint32_t)(it / kMcRing) & 1u) ^ 1u);
        tring[3 * ts] = t < ntiles ? t : -1;
        if (t < ntiles && p.pad2d) {  // dx rows r0.., columns c0..: global row b H + r0, packed c0 / valid extents
          const int64_t per = p.pd_nrt * p.pd_nct, b = t / per, rem = t - b * per, rt = rem / p.pd_nct;
          const int64_t r0 = rt * p.pd_R, c0 = (rem - rt * p.pd_nct) * p.pd_Cw;
          const int64_t nr = p.H - r0 < p.pd_R ? p.H - r0 : p.pd_R, nc = p.W - c0 < p.pd_Cw ? p.W - c0 : p.pd_Cw;
          tring[3 * ts + 1] = b * p.H + r0;
          tring[3 * ts + 2] = (c0 << 18) | (nr << 9) | nc;
        } else if (t < ntiles) {  // the tile's first position (row b0, position i0 in it): divisions here, off the epilogue
          const int64_t b0 = p.batched ? t / p.tiles_per_row : (t * TP) / p.N;
          tring[3 * ts + 1] = b0;
          tring[3 * ts + 2] = p.batched ? (t - b0 * p.tiles_per_row) * TP : t * TP - b0 * p.N;
        }
        mbar_arrive(tfull + ts);
        mbar_wait(empty + s, ph ^ 1);
        if (t >= ntiles) {  // end marker for the MMA warp: the next `full` phase without data
          mbar_arrive(full + s);
          break;
        }
        mbar_arrive_expect_tx(full + s, p.pad2d ? (uint32_t)p.pd_tx : kStage);
        if (p.pad2d) {  // one box per atom: (R + kh - 1) dy rows x P positions, kh-1 rows / kw-1 columns early
          const int64_t per = p.pd_nrt * p.pd_nct, b = t / per, rem = t - b * per, rt = rem / p.pd_nct;
          const int32_t r0 = (int32_t)(rt * p.pd_R), c0 = (int32_t)((rem - rt * p.pd_nct) * p.pd_Cw);
          for (int a = 0; a < AT; ++a)
            tma_load_5d_mc(xs + (size_t)s * kStage + (size_t)a * kAtomBytes, &p.tm_x, c0 - (p.pd_kw - 1),
                           r0 - (p.pd_kh - 1), a, (int32_t)b, full + s);
        } else if (p.batched) {  // tile = 128 positions of one row, staged from `pad` positions earlier
          const int64_t b = t / p.tiles_per_row;
          const int32_t t0 = (int32_t)((t - b * p.tiles_per_row) * TP) - p.pad;
          for (int a = 0; a < AT; ++a)
            for (int bx = 0; bx < p.nbox; ++bx)
              tma_load_4d_mc(xs + (size_t)s * kStage + (size_t)a * kAtomBytes + (size_t)bx * p.box_rows * 128,
                             &p.tm_x, 0, t0 + bx * p.box_rows, a, (int32_t)b, full + s);
        } else {
          for (int a = 0; a < AT; ++a)  // one SW128 block per K-atom, nbox boxes of box_rows positions
            for (int bx = 0; bx < p.nbox; ++bx)
              tma_load_3d_mc(xs + (size_t)s * kStage + (size_t)a * kAtomBytes + (size_t)bx * p.box_rows * 128,
                             &p.tm_x, 0, (int32_t)(t * TP + bx * p.box_rows), a, full + s);
        }
        if (++s == kMcStages) { s = 0; ph ^= 1; }
        if (p.clc) {
          t = clc_wait(&clc, cph);  // requested one tile ahead
          if (t < 0) t = ntiles;
          else clc_request(&clc);
        } else {
          t += gridDim.x;
        }
      }
    }
  } else if (warp == kMcWarpMma) {
    constexpr uint32_t idesc = idesc_bf16(128, COUT);
    const uint64_t dx0 = sw128_desc_mc(__shfl_sync(0xffffffffu, smem_u32(xs), 0));
    const uint64_t dw0 = sw128_desc_mc(__shfl_sync(0xffffffffu, smem_u32(ws), 0));
    const uint32_t dc0 = __shfl_sync(0xffffffffu, tmem, 0);
    int s = 0, d = 0;
    uint32_t ph = 0, dph = 0;
    for (int it = 0;; ++it) {
      mc_wait(full + s, ph);
      if (*reinterpret_cast<volatile int64_t*>(tring + 3 * (it % kMcRing)) < 0) break;
      mc_wait(dempty + d, dph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int mb = 0; mb < MB; ++mb) {  // M-block mb: positions 128 mb .. 128 mb + 127 of the tile
        const uint32_t dcol = dc0 + (uint32_t)((d * MB + mb) * COUT);
        const uint64_t dxs = dx0 + (uint64_t)((s * kStage + (uint32_t)mb * 128u * 128u) >> 4);
        uint32_t acc = 0;
#pragma unroll 1
        for (int j = 0; j < k; ++j) {
#pragma unroll
          for (int a = 0; a < AT; ++a)
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // K-steps of 16 channels (32 B) inside the atom
              const uint64_t da = dxs + (uint64_t)((a * kAtomBytes + (uint32_t)p.tap_off[j] * 128u + 32u * q) >> 4);
              const uint64_t db = dw0 + (uint64_t)(((uint32_t)j * kWTap + a * (COUT * 128u) + 32u * q) >> 4);
              mma_bf16_ss(dcol, da, db, idesc, acc);
              acc = 1;
            }
        }
      }
      mc_commit(empty + s);
      mc_commit(dfull + d);
      if (++s == kMcStages) { s = 0; ph ^= 1; }
      if (++d == kAcc) { d = 0; dph ^= 1; }
    }
  } else {
    // epilogue: quarter q's lanes (positions p0 + 32 q + [0, 32)) are read as two
    // 16-lane halves; warp half h stores channels [h NH, (h+1) NH)
    const int q = warp & 3, h = (warp - kMcWarpEpi0) >> 2;
    int d = 0;
    uint32_t dph = 0;
    for (int it = 0;; ++it) {
      const int ts = it % kMcRing;
      mc_wait(tfull + ts, (uint32_t)(it / kMcRing) & 1u);
      const int64_t t = *reinterpret_cast<volatile int64_t*>(tring + 3 * ts);
      const int64_t b0 = *reinterpret_cast<volatile int64_t*>(tring + 3 * ts + 1);
      const int64_t i0 = *reinterpret_cast<volatile int64_t*>(tring + 3 * ts + 2);
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + ts);
      if (t < 0) break;
      mc_wait(dfull + d, dph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int mb = 0; mb < MB; ++mb) {  // M-block by M-block (registers); the accumulator is freed after the last
        uint32_t v[2][NH / 8][4];          // [16-lane half][8-column block][4]
#pragma unroll
        for (int lh = 0; lh < 2; ++lh)
          mc_tmem_ld_row_blocks<NH / 8>(
              tmem + ((uint32_t)(32 * q + 16 * lh) << 16) + (uint32_t)((d * MB + mb) * COUT + h * NH), v[lh]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (mb == MB - 1) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(dempty + d);
        }
        // rows of this thread: output index of flat position i0 + m of row / image b0 (-1: not an output);
        // all four first, then the stores (independent chains, no per-row division)
        int64_t orow[2][2];
#pragma unroll
        for (int lh = 0; lh < 2; ++lh)
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int m = 128 * mb + 32 * q + 16 * lh + (lane >> 2) + 8 * rr;
            int64_t b = b0, i = i0 + m;
            int64_t o = -1;
            if (p.pad2d) {  // m = row P + col of the tile's staged grid
              const uint32_t mu = (uint32_t)m;
              const uint32_t r = (uint32_t)(((uint64_t)__umulhi(mu, p.w_magic) + mu) >> p.w_shift);
              const uint32_t c = mu - r * (uint32_t)p.pd_P;
              if (r < (uint32_t)((i0 >> 9) & 511) && c < (uint32_t)(i0 & 511)) o = (b0 + r) * p.W + (i0 >> 18) + c;
            } else if (p.batched) {
              if (i < p.n_out) o = b * p.n_out + i;
            } else {
              while (i >= p.N) { i -= p.N; ++b; }
              if (!p.two_d) {
                if (b < p.batch && i < p.L) o = b * p.L + i;
              } else {
                const uint32_t iu = (uint32_t)i;
                const uint32_t r = (uint32_t)(((uint64_t)__umulhi(iu, p.w_magic) + iu) >> p.w_shift);
                const uint32_t c = iu - r * (uint32_t)p.W;
                if (b < p.batch && r < (uint32_t)p.OH && c < (uint32_t)p.OW) o = (b * p.OH + r) * p.OW + c;
              }
            }
            orow[lh][rr] = o;
          }
#pragma unroll
        for (int lh = 0; lh < 2; ++lh)
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {  // rows lane/4 and lane/4 + 8 of this 16-lane half
            const int64_t o = orow[lh][rr];
            if (o >= 0) {
              float* __restrict__ yr = p.y + o * COUT + h * NH + 2 * (lane & 3);
#pragma unroll
              for (int cb = 0; cb < NH / 8; ++cb)
                *reinterpret_cast<float2*>(yr + 8 * cb) =
                    make_float2(__uint_as_float(v[lh][cb][2 * rr]), __uint_as_float(v[lh][cb][2 * rr + 1]));
            }
          }
      }
      if (++d == kAcc) { d = 0; dph ^= 1; }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kMcWarpMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Direct kernel (any shape / alignment): one (position, channel) per thread,
// fp32 accumulation of the exact bf16 products in (j, ci) order.
__global__ void __launch_bounds__(256) conv2d_mc_direct_kernel(const __grid_constant__ ConvMcParams p) {
  const uint16_t* __restrict__ x = static_cast<const uint16_t*>(p.x);
  const uint16_t* __restrict__ w = static_cast<const uint16_t*>(p.w);
  const int64_t kw = p.k / (p.H - p.OH + 1);
  const int64_t kh = p.k / kw;
  const int64_t total = p.batch * p.OH * p.OW * p.cout;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t co = o % p.cout, pix = o / p.cout, c = pix % p.OW, rb = pix / p.OW, r = rb % p.OH, b = rb / p.OH;
    float acc = 0.0f;
    for (int64_t a = 0; a < kh; ++a)
      for (int64_t e = 0; e < kw; ++e)
        for (int64_t ci = 0; ci < p.cin; ++ci) {
          const float xv = __uint_as_float((uint32_t)__ldg(x + ((b * p.H + r + a) * p.W + c + e) * p.cin + ci) << 16);
          const float wv = __uint_as_float((uint32_t)__ldg(w + ((co * p.cin + ci) * kh + a) * kw + e) << 16);
          acc = __fmaf_rn(wv, xv, acc);
        }
    p.y[o] = acc;
  }
}

__global__ void __launch_bounds__(256) conv_mc_direct_kernel(const __grid_constant__ ConvMcParams p) {
  const uint16_t* __restrict__ x = static_cast<const uint16_t*>(p.x);
  const uint16_t* __restrict__ w = static_cast<const uint16_t*>(p.w);
  const int64_t total = p.batch * p.L * p.cout;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t co = o % p.cout, r = o / p.cout, i = r % p.L, b = r / p.L;
    float acc = 0.0f;
    for (int64_t j = 0; j < p.k; ++j)
      for (int64_t ci = 0; ci < p.cin; ++ci) {
        const float xv = __uint_as_float((uint32_t)__ldg(x + (b * p.N + i + j) * p.cin + ci) << 16);
        const float wv = __uint_as_float((uint32_t)__ldg(w + (co * p.cin + ci) * p.k + j) << 16);
        acc = __fmaf_rn(wv, xv, acc);
      }
    p.y[o] = acc;
  }
}

// Input gradient, direct: dx[b][t][ci] = sum_j sum_co w[co][ci][k-1-j] dy[b][t-(k-1)+j][co] (dy rows of
// p.N = N-k+1 positions, p.cin = C_out dy channels, p.cout = C_in dx channels, p.n_out = N).
__global__ void __launch_bounds__(256) conv_mc_bwd_direct_kernel(const __grid_constant__ ConvMcParams p) {
  const uint16_t* __restrict__ dy = static_cast<const uint16_t*>(p.x);
  const uint16_t* __restrict__ w = static_cast<const uint16_t*>(p.w);
  const int64_t total = p.batch * p.n_out * p.cout;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ci = o % p.cout, r = o / p.cout, t = r % p.n_out, b = r / p.n_out;
    float acc = 0.0f;
    for (int64_t j = 0; j < p.k; ++j) {
      const int64_t s = t - (p.k - 1) + j;
      if (s < 0 || s >= p.N) continue;
      for (int64_t co = 0; co < p.cin; ++co) {
        const float gv = __uint_as_float((uint32_t)__ldg(dy + (b * p.N + s) * p.cin + co) << 16);
        const float wv = __uint_as_float((uint32_t)__ldg(w + (co * p.cout + ci) * p.k + (p.k - 1 - j)) << 16);
        acc = __fmaf_rn(wv, gv, acc);
      }
    }
    p.y[o] = acc;
  }
}

// 2-D input gradient, direct: dx[b][r][c][ci] = sum_{a,e,co} w[co][ci][a][e] dy[b][r-a][c-e][co] (p.cin = C_out
// dy channels, p.cout = C_in dx channels; H x W = dx, OH x OW = dy), fp32 accumulation in (a, e, co) order.
__global__ void __launch_bounds__(256) conv2d_mc_bwd_direct_kernel(const __grid_constant__ ConvMcParams p) {
  const uint16_t* __restrict__ dy = static_cast<const uint16_t*>(p.x);
  const uint16_t* __restrict__ w = static_cast<const uint16_t*>(p.w);
  const int64_t kh = p.H - p.OH + 1, kw = p.W - p.OW + 1;
  const int64_t total = p.batch * p.H * p.W * p.cout;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ci = o % p.cout, pix = o / p.cout, c = pix % p.W, rb = pix / p.W, r = rb % p.H, b = rb / p.H;
    float acc = 0.0f;
    for (int64_t a = 0; a < kh; ++a) {
      const int64_t rr = r - a;
      if (rr < 0 || rr >= p.OH) continue;
      for (int64_t e = 0; e < kw; ++e) {
        const int64_t cc = c - e;
        if (cc < 0 || cc >= p.OW) continue;
        for (int64_t co = 0; co < p.cin; ++co) {
          const float gv = __uint_as_float((uint32_t)__ldg(dy + ((b * p.OH + rr) * p.OW + cc) * p.cin + co) << 16);
          const float wv = __uint_as_float((uint32_t)__ldg(w + ((co * p.cout + ci) * kh + a) * kw + e) << 16);
          acc = __fmaf_rn(wv, gv, acc);
        }
      }
    }
    p.y[o] = acc;
  }
}

size_t conv_mc_smem_bytes(int64_t cin, int64_t cout, int64_t k, int rows, int stages) {
  const size_t stage = (size_t)(cin / 64) * rows * 128;
  return 1024 + stages * stage + (size_t)k * (cin / 64) * cout * 128 + 8 * (2 * stages + 8) + 40 * kMcRing + 16;
}

int conv_mc_choose_mblk(int64_t cin, int64_t cout, int64_t k, int rows1, bool prefer_one) {
  static const int forced = [] {
    const char* e = getenv("SS_MC_MBLK");
    return e ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2) return forced;
  if (prefer_one) return 1;
  return conv_mc_smem_bytes(cin, cout, k, mc_round_rows(rows1 + 128), kMcStages) <= (size_t)kSmemBudget ? 2 : 1;
}

// pad2d tiling: over pitches P = Cw + kw - 1 <= 256 and M-blocks (2 preferred when it fits three
// stages, as conv_mc_choose_mblk), R = min(128 mblk / P, H, 257 - kh) dx rows per tile; fewest tiles
// wins (the MMA work), then the fewest staged rows.  Staged rows cover the box and every row a tap of
// a masked output reads (positions past the box are never stored).
bool conv_mc_plan_pad2d(ConvMcParams& p) {
  static const int forced = [] {
    const char* e = getenv("SS_MC_MBLK");
    return e ? atoi(e) : 0;
  }();
  const int64_t kh = p.pd_kh, kw = p.pd_kw;
  if (kh * kw > kMcMaxTaps || kh > 256) return false;
  for (int mb = 2; mb >= 1; --mb) {
    if (forced && forced != mb) continue;
    const int64_t TP = 128 * mb;
    int64_t best = -1, best_rows = 0;
    int bP = 0, bR = 0, bC = 0;
    for (int64_t Cw = 1; Cw <= p.W && Cw + kw - 1 <= 256; ++Cw) {
      const int64_t P = Cw + kw - 1;
      int64_t R = TP / P;
      if (R > p.H) R = p.H;
      if (R > 257 - kh) R = 257 - kh;
      if (R < 1) continue;
      const int64_t box = (R + kh - 1) * P, reach = TP + (kh - 1) * P + kw - 1;
      const int64_t rows = ((box > reach ? box : reach) + 7) / 8 * 8;
      if (rows > 2048) continue;
      const int64_t nt = ((p.H + R - 1) / R) * ((p.W + Cw - 1) / Cw);
      if (best < 0 || nt < best || (nt == best && rows < best_rows)) {
        best = nt; best_rows = rows; bP = (int)P; bR = (int)R; bC = (int)Cw;
      }
    }
    if (best < 0) continue;
    const int stages_needed = mb == 2 && !forced ? kMcStages : 2;
    if (conv_mc_smem_bytes(p.cin, p.cout, kh * kw, (int)best_rows, stages_needed) > (size_t)kSmemBudget) continue;
    p.mblk = mb; p.rows = (int)best_rows; p.nbox = 1; p.box_rows = 0;
    p.pd_P = bP; p.pd_R = bR; p.pd_Cw = bC;
    p.pd_nrt = (p.H + bR - 1) / bR; p.pd_nct = (p.W + bC - 1) / bC;
    p.pd_tx = (int)((p.cin / 64) * (bR + kh - 1) * bP * 128);
    for (int64_t a = 0; a < kh; ++a)
      for (int64_t e = 0; e < kw; ++e) p.tap_off[a * kw + e] = (int)(a * bP + e);
    return true;
  }
  return false;
}

template <int CIN, int COUT>
static cudaError_t launch_mc(ConvMcParams& p, cudaStream_t stream, int sms) {
  p.nacc = 512 / (p.mblk * COUT) < 4 ? 512 / (p.mblk * COUT) : 4;
  p.stages = kMcStages;  // ring depth: 3, or 2 when the staged rows and the weights need the room
  while (p.stages > 2 && conv_mc_smem_bytes(CIN, COUT, p.k, p.rows, p.stages) > (size_t)kSmemBudget) --p.stages;
  const size_t smem = conv_mc_smem_bytes(CIN, COUT, p.k, p.rows, p.stages);
  if (smem > (size_t)kSmemBudget) return cudaErrorInvalidConfiguration;
  auto kfn = conv_mc_kernel<CIN, COUT>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kfn));
  if (e != cudaSuccess) return e;
  // one CTA per SM (each allocates TMEM): pad the request past half the budget
  const size_t smem_req = smem > (size_t)kSmemBudget / 2 ? smem : (size_t)kSmemBudget / 2 + 1024;
  const int64_t g = launch_grid(p.ntiles, sms, p.clc);
  kfn<<<(unsigned)g, kMcThreads, smem_req, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv_mc(ConvMcParams& p, bool tensor_path, cudaStream_t stream, int sms) {
  if (p.two_d || (p.pad2d && tensor_path)) {  // exact unsigned division by W (pad2d: P) for 31-bit numerators
    const uint64_t dv = p.pad2d ? (uint64_t)p.pd_P : (uint64_t)p.W;
    int sft = 0;
    while ((1ull << sft) < dv) ++sft;
    p.w_shift = sft;
    p.w_magic = (uint32_t)(((1ull << 32) * ((1ull << sft) - dv)) / dv + 1);
  }
  if (tensor_path) {
    if (p.mblk < 1) p.mblk = 1;
    const int64_t tp = 128 * p.mblk;
    if (p.batched) p.tiles_per_row = (p.n_out + tp - 1) / tp;
    p.ntiles = p.pad2d ? p.batch * p.pd_nrt * p.pd_nct
                       : p.batched ? p.batch * p.tiles_per_row : (p.batch * p.N + tp - 1) / tp;
    cudaError_t e = cudaErrorInvalidConfiguration;
    if (p.cin == 64 && p.cout == 64) e = launch_mc<64, 64>(p, stream, sms);
    else if (p.cin == 64 && p.cout == 128) e = launch_mc<64, 128>(p, stream, sms);
    else if (p.cin == 128 && p.cout == 64) e = launch_mc<128, 64>(p, stream, sms);
    else if (p.cin == 128 && p.cout == 128) e = launch_mc<128, 128>(p, stream, sms);
    if (e != cudaErrorInvalidConfiguration) return e;
  }
  const int64_t total = p.pad2d  ? p.batch * p.H * p.W * p.cout
                      : p.two_d ? p.batch * p.OH * p.OW * p.cout
                                : p.bwd_in ? p.batch * p.n_out * p.cout : p.batch * p.L * p.cout;
  int64_t g = (total + 255) / 256;
  if (g > (int64_t)sms * 16) g = (int64_t)sms * 16;
  if (p.pad2d) conv2d_mc_bwd_direct_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
  else if (p.bwd_in) conv_mc_bwd_direct_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
  else if (p.two_d) conv2d_mc_direct_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
  else conv_mc_direct_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ss
