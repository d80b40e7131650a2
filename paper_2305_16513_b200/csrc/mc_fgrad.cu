// mc_fgrad.cu -- filter gradient of the multi-channel 1-D convolution (SURVEY 8f
// NEXT #4, training; reading R25):
//   dw[co][ci][j] = sum_b sum_{i < N-k+1} dy[b][i][co] * x[b][i+j][ci]
// dy [batch][N-k+1][cout] and x [batch][N][cin] bfloat16 (channels-last), dw
// [cout][cin][k] fp32.
//
// As a matrix product per tile of 128 positions of one row:
//   D[co][(j, ci)] += sum_{p < 128} dy[p][co] * x[p + j][ci]
// M = cout, N = k x 64 (cin = 64), K = positions.  Both operands are the
// activations as they lie in memory, read MN-major (channels contiguous):
// A = the dy tile (K row p = dy[p][0..cout)), B for tap j = the x tile read j K
// rows further down (descriptor start + 128 j bytes; the same row-shift trick as
// the forward), so no im2col and no transposes.  bf16 products are exact; the
// tensor memory accumulates one tile (128 positions, fp32), the epilogue adds the
// tile into an fp32 run accumulator in registers (32 tiles per run), and each run
// goes straight from registers into this CTA's fp64 slice of the caller's workspace
// (slice [64 k][cout]: a warp's rows are contiguous; the first run is stored, later
// ones are added by fire-and-forget reductions, in program order per slot); a
// finish kernel sums the slices in a fixed order.  |error| <= (128 + 32)
// fp32 roundings of partial sums bounded by sum |terms| (~9.5e-6 of it) -- inside
// the 1e-5 bound.
//
// Roles (320 threads, one CTA per SM): warp 0 TMA producer (dy tile + x tile of
// 136 rows per stage, as many stages as shared memory holds: 6 at cout = 64), warp 1 MMA issuer (8 K-steps, one N = 64 k MMA each:
// tap j is B's MN atom j = the x tile j rows down, an atom stride of 128 B), warps
// 2-9 epilogue (two per TMEM lane quarter, half the columns each; for cout = 64 the M = 64 accumulator
// occupies lanes 0-15 of each quarter: tools/ubench/tc_m64_probe.cu).
#include <cstdint>

#include <cuda.h>
#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kMfThreads = 320;
constexpr int kMfMaxStages = 8;                   // ring depth: as many one-tile stages as shared memory holds
constexpr int kMfTileP = 128;                      // positions per tile
constexpr int kMfXRows = 136;                      // x rows per tile (128 + k - 1 <= 131, 17 atoms)
constexpr uint32_t kMfXBytes = kMfXRows * 128u;
constexpr int kMfRunTiles = 32;                    // tiles per fp32 run

__device__ __forceinline__ uint64_t mf_desc(uint32_t saddr, uint32_t lbo) {  // MN-major bf16, SWIZZLE_128B
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((1024u >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t mf_idesc(int M, int N) {  // bf16 x bf16 -> f32, A and B MN-major
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mf_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mf_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mf_wait(uint64_t* bar, uint32_t parity) {  // polls (commit-driven phases)
  asm volatile(
      "{\n\t.reg .pred p;\nMF_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra MF_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mf_tma_4d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                          int32_t c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mf_tma_5d(void* dst, const CUtensorMap* map, int32_t c1, int32_t c2, int32_t c3,
                                          int32_t c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mf_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ __attribute__((unused)) void mf_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

constexpr size_t mf_stage_bytes(int dyreg, int dyrow_cap, int xrows) {
  return (size_t)dyreg * dyrow_cap * 128u + (size_t)xrows * 128u;
}
constexpr size_t mf_smem(size_t stage, int stages) { return 1024 + (size_t)stages * stage + 256; }

}  // namespace

template <int COUT, int KT>
__global__ void __launch_bounds__(kMfThreads, 1) mc_filter_grad_tc_kernel(const __grid_constant__ McFgradParams p) {
  constexpr int AT = COUT / 64;  // dy atoms (64 channels each)
  const uint32_t kRegBytes = (uint32_t)p.dyrow_cap * 128u;  // one dy region
  const uint32_t kDyBytes = (uint32_t)p.dyreg * kRegBytes;
  const uint32_t kStage = kDyBytes + (uint32_t)p.xrows * 128u;
  extern __shared__ __align__(16) uint8_t mf_raw[];
  uint8_t* smem = mf_raw + ((1024u - (smem_u32(mf_raw) & 1023u)) & 1023u);
  constexpr int NC = 64 * KT, NH = NC / 2;  // accumulator columns (tap j at 64 j); per epilogue warp
  const int kMfStages = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kMfStages * kStage);
  uint64_t* empty = full + kMfMaxStages;
  uint64_t* dfull = empty + kMfMaxStages;
  uint64_t* dempty = dfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = p.ntiles, tpr = p.tiles_per_row;
  // units: tiles t0, t0 + tstep, ...; 2-D: CTA c is in group c % groups, which serves tap row ta (and,
  // paired, ta - 1 through a second dy region one image row down: an M = 128 accumulator)
  const int grp = p.two_d ? (int)(blockIdx.x % (unsigned)p.groups) : 0;
  const bool paired = p.pair && 2 * grp + 1 <= p.kh - 1;
  const int ta = p.pair ? (2 * grp + 1 < p.kh - 1 ? 2 * grp + 1 : p.kh - 1) : grp;
  const int64_t t0 = p.two_d ? blockIdx.x / (unsigned)p.groups : blockIdx.x;
  const int64_t tstep = p.two_d ? gridDim.x / (unsigned)p.groups : gridDim.x;
  const bool m128 = COUT == 128 || paired;  // accumulator rows: all 128 lanes, else lanes 0-15 per quarter
  const int nreg = paired ? p.dyreg : AT;   // dy regions this CTA loads

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMfStages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(dfull + s, 1); mbar_init(dempty + s, 8); }
    fence_mbar_init();
    prefetch_tmap(&p.tm_dy);
    prefetch_tmap(&p.tm_x);
  }
  // staged rows no box writes (2-D: dy rows past R W, x rows past (R + 1) W) meet zero dy or are never
  // multiplied, but must be finite: zero them once
  if (p.dy_fill < p.dyrow_cap || p.x_rows < p.xrows) {
    for (int s = 0; s < kMfStages; ++s) {
      uint8_t* st = smem + (size_t)s * kStage;
      for (int a = 0; a < p.dyreg; ++a)
        for (int i = p.dy_fill * 32 + (int)threadIdx.x; i < p.dyrow_cap * 32; i += kMfThreads)
          reinterpret_cast<uint32_t*>(st + a * kRegBytes)[i] = 0u;
      for (int i = p.x_rows * 32 + (int)threadIdx.x; i < p.xrows * 32; i += kMfThreads)
        reinterpret_cast<uint32_t*>(st + kDyBytes)[i] = 0u;
    }
    fence_proxy_async_smem();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      for (int64_t tile = t0; tile < ntiles; tile += tstep, ++it) {
        const int s = it % kMfStages;
        mf_wait(empty + s, ((uint32_t)(it / kMfStages) & 1u) ^ 1u);  // commit-driven: poll
        uint8_t* st = smem + (size_t)s * kStage;
        mbar_arrive_expect_tx(full + s, (uint32_t)nreg * p.tx_dy + p.tx_x);
        if (p.two_d) {  // dy rows r0 .. r0 + R - 1 (pitch W; paired: and r0 + 1 ..), x rows r0 + ta .. r0 + ta + R
          const int64_t b = tile / p.nrt;
          const int32_t r0 = (int32_t)((tile - b * p.nrt) * p.R) - p.shift;
          for (int a = 0; a < nreg; ++a)
            mf_tma_5d(st + a * kRegBytes, &p.tm_dy, 0, r0 + (paired ? a : 0), paired ? 0 : a, (int32_t)b, full + s);
          mf_tma_5d(st + kDyBytes, &p.tm_x, 0, r0 + ta, 0, (int32_t)b, full + s);
        } else {
          const int64_t b = tile / tpr;
          const int32_t p0 = (int32_t)((tile - b * tpr) * kMfTileP);
#pragma unroll
          for (int a = 0; a < AT; ++a) mf_tma_4d(st + a * 16384u, &p.tm_dy, 0, p0, a, (int32_t)b, full + s);
          mf_tma_4d(st + kDyBytes, &p.tm_x, 0, p0, 0, (int32_t)b, full + s);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // one MMA per K-step covers every tap: B's MN atom j is the x tile j K rows further down, i.e. an
    // atom stride (LBO) of one 128-B row (tools/ubench/tc_lbo_probe.cu), N = 64 k
    const uint32_t idesc = mf_idesc(m128 ? 128 : 64, NC);
    const uint32_t s0 = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
    int it = 0, d = 0;
    uint32_t dph = 0;
    for (int64_t tile = t0; tile < ntiles; tile += tstep, ++it) {
      const int s = it % kMfStages;
      mf_wait(full + s, (uint32_t)(it / kMfStages) & 1u);
      mf_wait(dempty + d, dph ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dyT = s0 + (uint32_t)s * kStage, xT = dyT + kDyBytes;
      const uint32_t dcol = tmem + (uint32_t)(d * NC);
#pragma unroll 1
      for (int ks = 0; ks < p.ks; ++ks) {
        mf_mma(dcol, mf_desc(dyT + 2048u * ks, p.alo), mf_desc(xT + 128u * (16 * ks), 128u), idesc, ks > 0 ? 1u : 0u);
      }
      mf_commit(empty + s);
      mf_commit(dfull + d);
      if (++d == 2) { d = 0; dph ^= 1u; }
    }
  } else {
    // ------------------------------------------------------------ epilogue: tile -> fp32 run -> fp64 slice
    const int q = warp & 3, hh = (warp - 2) >> 2;  // lane quarter; half of the columns (two warps per quarter)
    const int co = m128 ? 32 * q + lane : 16 * q + lane;  // accumulator row (M = 64: lanes 0-15 of a quarter)
    const int cb = hh * NH;
    const uint32_t lanebits = (uint32_t)(32 * q) << 16;
    // this CTA's fp64 slice [NC][mr] (row fastest: a warp's 16 / 32 rows are contiguous, so a run
    // flushes straight from registers, coalesced); each thread owns (row co, [cb, cb + NH))
    constexpr int MR = 128;  // slice rows (M = 64 accumulators fill rows 0-63)
    double* W = p.ws + (size_t)blockIdx.x * MR * NC + (size_t)cb * MR + co;
    const bool owner = m128 || lane < 16;
    if (owner && t0 >= ntiles)  // no tiles: the slice is zero
      for (int i = 0; i < NH; ++i) W[(size_t)i * MR] = 0.0;
    bool first = true;  // the first run is stored, later runs are added (fire-and-forget reductions)
    // the fp32 run lives in registers: row co, columns [cb, cb + NH) (tcgen05.ld 32x32b: lane = row)
    float acc[NH];
#pragma unroll
    for (int i = 0; i < NH; ++i) acc[i] = 0.0f;
    int d = 0, nt = 0;
    uint32_t dph = 0;
    for (int64_t tile = t0; tile < ntiles; tile += tstep) {
      mf_wait(dfull + d, dph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c0 = 0; c0 < NH; c0 += 16) {  // x16: acc + v stay under the 10-warp CTA's 168-register cap
        uint32_t v[16];
        mf_ld16(tmem + lanebits + (uint32_t)(d * NC + cb + c0), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[c0 + i] += __uint_as_float(v[i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty + d);
      if (++nt == kMfRunTiles || tile + tstep >= ntiles) {  // end of a run: into the fp64 slice
        nt = 0;
        if (owner) {
          // one thread owns each slot and issues its writes in program order, so the additions land in
          // a fixed order (per-location coherence): deterministic; a reduction needs no round trip
          if (first) {
#pragma unroll
            for (int i = 0; i < NH; ++i) W[(size_t)i * MR] = (double)acc[i];
          } else {
#pragma unroll
            for (int i = 0; i < NH; ++i) atomicAdd(W + (size_t)i * MR, (double)acc[i]);
          }
#pragma unroll
          for (int i = 0; i < NH; ++i) acc[i] = 0.0f;
        }
        first = false;
      }
      if (++d == 2) { d = 0; dph ^= 1u; }
    }
    // CTAs past the last tile leave their slice at zero (written above)
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// dw[co][ci][a][e] = sum over the slices c of tap row a's group (c = grp, grp + groups, ...) of
// ws[c][64 e + ci][m] (1-D: one group, kh = 1, e = j; m = co, or 64 + co for the upper half of a paired
// group, which holds tap row a = 2 grp).  Block (column 64 e + ci, a), thread (co, g), G = 1024 / cout:
// slices grp + groups (g + G i) in increasing i (cout threads read cout contiguous doubles per slice),
// then the G partial sums in g order: a fixed order, deterministic.
__global__ void __launch_bounds__(1024) mc_filter_grad_finish(const double* __restrict__ ws, int ctas, int cout,
                                                              int kh, int kw, int groups, int pair, int mr,
                                                              float* __restrict__ dw) {
  __shared__ double part[1024];
  const int G = 1024 / cout, co = threadIdx.x % cout, g = threadIdx.x / cout;
  const int nc = 64 * kw, col = blockIdx.x % nc, a = blockIdx.x / nc;
  const int grp = pair ? a / 2 : a;
  const int m = (pair && a % 2 == 0 && a + 1 <= kh - 1) ? 64 + co : co;
  const int per = ctas / groups;  // slices of the group
  const double* __restrict__ src = ws + (size_t)col * mr + m;
  const size_t cstride = (size_t)nc * mr;
  double s = 0.0;
#pragma unroll 4
  for (int i = g; i < per; i += G) s += src[(size_t)(grp + groups * i) * cstride];
  part[threadIdx.x] = s;
  __syncthreads();
  if (g == 0) {
    for (int h = 1; h < G; ++h) s += part[h * cout + co];
    const int e = col / 64, ci = col % 64;
    dw[(((int64_t)co * 64 + ci) * kh + a) * kw + e] = (float)s;
  }
}

// Direct kernel (any shape): one block per output element, positions strided over the threads,
// products and sums in double, fixed-order block reduction.
__global__ void __launch_bounds__(256) mc_filter_grad_direct_kernel(const __grid_constant__ McFgradParams p) {
  __shared__ double red[256];
  const uint16_t* __restrict__ dy = p.dy;
  const uint16_t* __restrict__ x = p.x;
  const int64_t total = p.cout * p.cin * p.k, npos = p.batch * p.L;
  for (int64_t o = blockIdx.x; o < total; o += gridDim.x) {
    const int64_t j = o % p.k, ci = (o / p.k) % p.cin, co = o / (p.k * p.cin);
    double s = 0.0;
    for (int64_t e = threadIdx.x; e < npos; e += blockDim.x) {
      const int64_t b = e / p.L, i = e - b * p.L;
      const float g = __uint_as_float((uint32_t)__ldg(dy + e * p.cout + co) << 16);
      const float xv = __uint_as_float((uint32_t)__ldg(x + (b * p.N + i + j) * p.cin + ci) << 16);
      s += (double)g * (double)xv;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) p.dw[o] = (float)red[0];
    __syncthreads();
  }
}

// 2-D direct kernel: as above over the positions (b, r, c) of dy, tap (a, e).
__global__ void __launch_bounds__(256) mc_filter_grad2d_direct_kernel(const __grid_constant__ McFgradParams p) {
  __shared__ double red[256];
  const uint16_t* __restrict__ dy = p.dy;
  const uint16_t* __restrict__ x = p.x;
  const int64_t kw = p.k, kh = p.H - p.OH + 1, taps = kh * kw;
  const int64_t total = p.cout * p.cin * taps, npos = p.batch * p.OH * p.OW;
  for (int64_t o = blockIdx.x; o < total; o += gridDim.x) {
    const int64_t e = o % kw, a = (o / kw) % kh, ci = (o / taps) % p.cin, co = o / (taps * p.cin);
    double s = 0.0;
    for (int64_t q = threadIdx.x; q < npos; q += blockDim.x) {
      const int64_t c = q % p.OW, rb = q / p.OW, r = rb % p.OH, b = rb / p.OH;
      const float g = __uint_as_float((uint32_t)__ldg(dy + q * p.cout + co) << 16);
      const float xv = __uint_as_float((uint32_t)__ldg(x + ((b * p.H + r + a) * p.W + c + e) * p.cin + ci) << 16);
      s += (double)g * (double)xv;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) p.dw[o] = (float)red[0];
    __syncthreads();
  }
}

bool mc_filter_grad_tc_supported(int64_t cin, int64_t cout, int64_t k) {
  return cin == 64 && ((cout == 64 && k <= 4) || (cout == 128 && k <= 2)) && k >= 1;
}

size_t mc_filter_grad_workspace(int64_t cin, int64_t cout, int64_t k, int sms, bool two_d) {
  if (!mc_filter_grad_tc_supported(cin, cout, k)) return 0;
  (void)two_d;
  return (size_t)sms * 128 * 64 * k * sizeof(double);  // slices [64 k][128]
}

// 2-D tiling: R = the most dy rows of pitch W that fit 128 positions, balanced over the image's rows
bool mc_filter_grad_2d_plan(McFgradParams& p) {
  if (!mc_filter_grad_tc_supported(p.cin, p.cout, p.k) || p.W > 128 || p.kh < 1 || p.kh > 64) return false;
  // cout = 64 pairs tap rows (a, a - 1) into M = 128 MMAs: ceil(kh / 2) groups; tiles start one row
  // early so both halves see every dy row once (row -1 and rows past OH are the TMA's zero fill)
  p.pair = p.cout == 64 && p.kh >= 2;
  p.shift = p.pair ? 1 : 0;
  p.groups = p.pair ? (p.kh + 1) / 2 : p.kh;
  p.mr = 128;
  p.dyreg = p.pair ? 2 : (int)(p.cout / 64);
  const int64_t rows = p.OH + p.shift;  // dy rows the tiles cover (from -shift)
  const int64_t rmax = 128 / p.W, nt = (rows + rmax - 1) / rmax;
  p.R = (int)((rows + nt - 1) / nt);
  bool shifted = false;  // paired, R W % 16 == 0: one region of R + 1 rows, the upper half W rows down
  if (p.pair)
    for (int64_t r = rmax; r >= 1 && !shifted; --r)
      if ((r * p.W) % 16 == 0) { p.R = (int)r; shifted = true; }
  p.nrt = (rows + p.R - 1) / p.R;
  p.dy_rows = (int)(p.R * p.W);
  p.ks = (p.dy_rows + 15) / 16;  // K-steps: the tile's R W positions (zero rows past them)
  if (shifted) {
    p.dyreg = 1;
    p.dy_fill = (int)((p.R + 1) * p.W);
    p.dyrow_cap = (p.dy_fill + 7) / 8 * 8;
    p.alo = (uint32_t)(p.W * 128);
  } else {
    p.dy_fill = p.dy_rows;
    p.dyrow_cap = 128;
    p.alo = 16384u;
  }
  p.x_rows = (int)((p.R + 1) * p.W);
  const int reach = 16 * p.ks + (int)p.k - 1;
  p.xrows = ((p.x_rows > reach ? p.x_rows : reach) + 7) / 8 * 8;
  p.tx_dy = (uint32_t)(p.dy_fill * 128);
  p.tx_x = (uint32_t)(p.x_rows * 128);
  return p.xrows <= 256 && p.dyrow_cap <= 256;
}

cudaError_t launch_mc_filter_grad(McFgradParams& p, bool tc, cudaStream_t stream, int sms) {
  if (tc) {
    int ctas = sms;
    if (p.two_d) {  // planned by mc_filter_grad_2d_plan; kh CTA groups
      p.ntiles = p.batch * p.nrt;
      ctas = sms / p.groups * p.groups;
    } else {
      p.tiles_per_row = (p.L + kMfTileP - 1) / kMfTileP;
      p.ntiles = p.batch * p.tiles_per_row;
      p.kh = 1; p.xrows = kMfXRows; p.dy_rows = 128; p.x_rows = kMfXRows;
      p.groups = 1; p.pair = 0; p.shift = 0; p.mr = 128; p.dyreg = (int)(p.cout / 64);
      p.dyrow_cap = 128; p.dy_fill = 128; p.ks = kMfTileP / 16; p.alo = 16384u;
      p.tx_dy = 16384u; p.tx_x = kMfXRows * 128u;
    }
    const void* kfn = nullptr;
    const int k = (int)p.k;
    if (p.cout == 128) kfn = k == 1 ? reinterpret_cast<const void*>(mc_filter_grad_tc_kernel<128, 1>)
                                    : reinterpret_cast<const void*>(mc_filter_grad_tc_kernel<128, 2>);
    else kfn = k == 1   ? reinterpret_cast<const void*>(mc_filter_grad_tc_kernel<64, 1>)
               : k == 2 ? reinterpret_cast<const void*>(mc_filter_grad_tc_kernel<64, 2>)
               : k == 3 ? reinterpret_cast<const void*>(mc_filter_grad_tc_kernel<64, 3>)
                        : reinterpret_cast<const void*>(mc_filter_grad_tc_kernel<64, 4>);
    const size_t stage = mf_stage_bytes(p.dyreg, p.dyrow_cap, p.xrows);
    p.stages = (int)((kSmemBudget - 1024 - 256) / stage);
    if (p.stages > kMfMaxStages) p.stages = kMfMaxStages;
    const size_t smem = mf_smem(stage, p.stages);
    if (p.stages < 2 || smem > (size_t)kSmemBudget || ctas < p.groups) return cudaErrorInvalidConfiguration;
    cudaError_t e = ensure_smem_attr(kfn);
    if (e != cudaSuccess) return e;
    void* args[] = {&p};
    e = cudaLaunchKernel(kfn, dim3((unsigned)ctas), dim3(kMfThreads), args, smem, stream);
    note_launch();
    if (e != cudaSuccess) return e;
    mc_filter_grad_finish<<<(unsigned)(64 * p.k * p.kh), 1024, 0, stream>>>(p.ws, ctas, (int)p.cout, p.kh, (int)p.k,
                                                                         p.groups, p.pair, p.mr, p.dw);
    note_launch();
    return cudaGetLastError();
  }
  const int64_t total = p.cout * p.cin * p.k * (p.two_d ? p.H - p.OH + 1 : 1);
  const int64_t g = total < (int64_t)sms * 32 ? total : (int64_t)sms * 32;
  if (p.two_d) mc_filter_grad2d_direct_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
  else mc_filter_grad_direct_kernel<<<(unsigned)(g < 1 ? 1 : g), 256, 0, stream>>>(p);
  note_launch();
  return cudaGetLastError();
}

}  // namespace ss
