// fgrad_tc.cu -- filter gradient of the sliding dot product on the tensor cores
// (readings R16 / R24):
//   df_j = sum_b sum_{i < L} dy[b][i] x[b][i + j],   j < k <= 64, stride 1.
//
// Chunked-correlation form: cut each dy row into chunks of 128 (chunk u covers
// i = 128 u + v, v < 128) and let
//   C[v][s] = sum over chunks (b, u) of dy[b][128 u + v] * x[b][128 u + s],  s < 192,
// a matrix product with M = v (128), N = s (192) and K = the chunk index;
// then df_j = sum_v C[v][v + j] (a diagonal sum of the 128 x 192 result).  The
// 63 taps x 128 outputs of a chunk become 128 x 192 MACs (3x the direct count)
// on tensor cores instead of FP32 FMAs, and no operand needs an im2col: B is
// x itself viewed as rows of 128 (row u = x[128 u ..]); its columns 128..191
// are columns 0..63 of row u + 1, i.e. the same shared-memory tile read one
// K row further down (an N = 64 MMA whose descriptor start is shifted 128 B).
//
// Numerics: 3xTF32 (A_hi B_hi + A_hi B_lo + A_lo B_hi, hi = the TF32 truncation,
// lo = the exact remainder; ~2^-21 relative per product), fp32 accumulation in
// tensor memory over a unit of 128 chunks (<= 128 fp32 roundings of a sum bounded
// by the sum of |terms|: ~7.6e-6 of it, inside the 1e-5 bound), then fp64: the
// diagonal sums (8-term fp32 partials) and all cross-unit / cross-CTA sums are in
// double (two-pass: per-CTA partials in the caller's workspace,
// conv_filter_grad_finish sums them in CTA order).  Deterministic.
//
// Roles (704 threads, one CTA per SM; x rows need N % 128 == 0):
//   warp 21      TMA producer: x rows u0 .. u0 + 32 of each stage (32 chunks) as one
//                2-D box of x viewed as [batch N / 128][128], into a 6-deep raw ring;
//   warps 0-15   two loader groups of 8 warps taking alternate stages (slot = group):
//                thread v issues the stage's dy loads into registers, then, once the
//                MMA has drained the group's previous stage, splits dy[.., 128 u + v]
//                into hi / lo for tensor memory (A operand: lane v, one column per
//                chunk; warps w and w + 4 of a group share lane quarter w) and the raw
//                x rows into the MN-major SWIZZLE_128B_BASE32B B tiles (the only
//                MN-major layout TF32 accepts; tools/ubench/tc_mn_probe.cu);
//   warp 16      MMA issuer: per stage 4 K-groups x 3 products x {N = 128, N = 64 one
//                K row down} = 24 MMAs into one of two 192-column accumulators;
//   warps 17-20  drain an accumulator per unit: lane v reads the 96 columns its
//                diagonal can touch, a padded shared-memory transpose turns rows into
//                diagonals, and each thread sums 64 diagonal terms.
// Measured (64 x 2^20, 1 x B200): k = 63 at 120 us vs 250 us for the FFMA2 kernel; the
// tensor pipe is ~77% busy (ncu), so the 3 products are the limit.
#include <cstdint>
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

namespace {

constexpr int kFtStageChunks = 32;                 // K rows per stage (4 K-groups of 8)
// Mixed precision (the forward tensor-core conv's scheme): D += A_hi B_hi in kind::tf32 plus ONE
// kind::f16 MMA of K = 16 for both cross terms, [bf16(A_hi) | bf16(A_lo)] . [bf16(B_lo) ; bf16(B_hi)]
// (K pairs packed per TMEM column against interleaved B rows) -- two MMA-times per K-group
// instead of three.  Per-product error ~2^-18, so units shrink to 64 chunks to keep the fp32
// accumulation inside the bound.
constexpr bool kFtMixed = false;  // measured: 123.6 us (tensor pipe 45% busy) vs 120 us for 3xTF32 -- the
                                   // MMAs are not the limit once the loaders run two stages ahead
constexpr int kFtUnitStages = kFtMixed ? 2 : 4;    // stages per accumulation unit (64 / 128 chunks)
constexpr int kFtUnitChunks = kFtStageChunks * kFtUnitStages;
constexpr int kFtStages = 2;                       // slots: loader group g owns slot g (stages it = g mod 2)
constexpr int kFtRows = 36;                        // B rows per stage (33 used), 9 BASE32B atoms of 4
constexpr uint32_t kFtLBO = kFtRows * 128u;        // MN-atom stride (bytes)
constexpr uint32_t kFtB = 4u * kFtLBO;             // one B operand (hi or lo) of a stage
constexpr uint32_t kFtLBO16 = 9u * 1024u;          // mixed: bf16 pair tile, MN atom (64 bf16) stride, 72 rows
static_assert(2 * kFtLBO16 <= kFtB, "the bf16 pair tile reuses the lo tile's space");
constexpr int kFtPitch = 97;                       // transpose scratch row pitch (floats)
constexpr int kFtThreads = 22 * 32;
constexpr int kFtWarpMma = 16;                     // warps 0-15: loaders (two groups of 8)
constexpr int kFtEpi0 = 17;                        // first epilogue warp (17-20)
constexpr int kFtWarpTma = 21;                     // raw x rows of each stage by TMA, kFtRaw stages ahead
constexpr int kFtRaw = 6;                          // raw x ring
constexpr uint32_t kFtRawBytes = 34u * 512u;        // one raw stage: 33 rows of 128 floats (+1 row pad)
constexpr size_t kFtSmem = 1024 + (size_t)kFtStages * 2 * kFtB + (size_t)kFtRaw * kFtRawBytes +
                           (size_t)128 * kFtPitch * 4 + 128 * 8 + 256;

__device__ __forceinline__ uint64_t mn32_desc(uint32_t saddr) {  // MN-major, SWIZZLE_128B_BASE32B
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((kFtLBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((512u >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}
__device__ __forceinline__ uint64_t mn16_desc(uint32_t saddr) {  // MN-major bf16, SWIZZLE_128B
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((kFtLBO16 >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((1024u >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16_bmn(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t bf16_pack(float lo, float hi) {  // low half = lo (round to nearest)
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
}
__host__ __device__ constexpr uint32_t idesc_tf32_bmn(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void ft_mma(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void ft_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void ft_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\nFT_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra FT_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
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
__device__ __forceinline__ uint32_t tf32_hi(uint32_t b) { return b & 0xffffe000u; }

}  // namespace

__global__ void __launch_bounds__(kFtThreads, 1) conv_filter_grad_tc_kernel(const __grid_constant__ FgradTcParams p) {
  extern __shared__ __align__(16) uint8_t ft_raw[];
  uint8_t* smem = ft_raw + ((1024u - (smem_u32(ft_raw) & 1023u)) & 1023u);
  uint8_t* bsm = smem;                                            // [stage][hi, lo][4 atoms][36 rows][128 B]
  float* raw = reinterpret_cast<float*>(bsm + kFtStages * 2 * kFtB);  // [kFtRaw][33 x 128 (+pad)] raw x rows
  float* cs = raw + kFtRaw * (kFtRawBytes / 4);                         // [128][97] transpose scratch
  double* red = reinterpret_cast<double*>(cs + 128 * kFtPitch);      // [128]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 128);           // [stages]
  uint64_t* empty = full + kFtStages;                                // [stages]
  uint64_t* dfull = empty + kFtStages;                               // [2]
  uint64_t* dempty = dfull + 2;                                      // [2]
  uint64_t* rfull = dempty + 2;                                      // [kFtRaw] TMA landed
  uint64_t* rempty = rfull + kFtRaw;                                 // [kFtRaw] loader group consumed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rempty + kFtRaw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t N = p.N, L = p.L, U = p.U, UR = p.units_per_row, nunits = p.nunits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kFtStages; ++s) { mbar_init(full + s, 256); mbar_init(empty + s, 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(dfull + s, 1); mbar_init(dempty + s, 4); }
    for (int s = 0; s < kFtRaw; ++s) { mbar_init(rfull + s, 1); mbar_init(rempty + s, 256); }
    prefetch_tmap(&p.tm_x);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  // TMEM columns: D[2] at 0 / 192, A at 384 + 64 slot (hi: +0..31, lo: +32..63)
  constexpr uint32_t kAcol = 384;

  if (warp < kFtWarpMma) {
    // ------------------------------------------------------------ loaders: two groups of 8 warps; in a
    // group, warps w and w + 4 share TMEM lane quarter w (lane v) and take chunks [0, 16) / [16, 32)
    const int grp = warp >> 3, wg = warp & 7, v = 32 * (wg & 3) + lane, ch0 = 16 * (wg >> 2);
    const int t = threadIdx.x & 255;  // thread in the group: x items t + 256 m
    const uint32_t lanebits = (uint32_t)(32 * (wg & 3)) << 16;
    const float* __restrict__ dyp = p.dy;
    // x item m of this thread: row r = (t >> 5) + 8 m of the stage (K atom 2 m + (t >> 7), row (t >> 5) & 3
    // inside it), 16-B piece t & 31 of the row; rows >= 33 are not loaded
    const int xrow = t >> 5, s4 = 4 * (t & 31), xa = s4 >> 5, xc = (s4 & 31) >> 3, xh = (s4 & 7) >> 2;
    const uint32_t xoff0 = (uint32_t)xa * kFtLBO + (uint32_t)(xrow >> 2) * 512u + (uint32_t)(xrow & 3) * 128u +
                           ((uint32_t)(xc ^ (xrow & 3)) << 5) + (uint32_t)xh * 16u;
    // mixed: bf16 pair tile rows kr = 2 r + e (e = 0 lo, 1 hi); row r = xrow + 8 m -> K atom (2 xrow + e) / 8
    // + 2 m, row (2 xrow + e) % 8; 64-bf16 MN atom s4 / 64, 16-B chunk (s4 % 64) / 8, byte (s4 % 8) * 2
    auto poff = [&](int e2) {
      const int kr = 2 * xrow + e2, a16 = s4 >> 6, c16 = (s4 & 63) >> 3, rr16 = kr & 7;
      return (uint32_t)a16 * kFtLBO16 + (uint32_t)(kr >> 3) * 1024u + (uint32_t)rr16 * 128u +
             ((uint32_t)(c16 ^ rr16) << 4) + (uint32_t)(s4 & 7) * 2u;
    };
    const uint32_t xoffp0 = poff(0), xoffp1 = poff(1);
    int it = 0;
    for (int64_t unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
      const int64_t b = unit / UR, q = unit - b * UR;
      for (int s2 = 0; s2 < kFtUnitStages; ++s2, ++it) {
        if ((it & 1) != grp) continue;  // this group's stages: it = grp mod 2 (slot grp)
        const int st = it % kFtStages;
        const int64_t u0 = q * kFtUnitChunks + s2 * kFtStageChunks;
        // all of this thread's loads of the stage first; in-range stages (all but a row's last) take
        // unpredicated loads at immediate offsets
        const float* __restrict__ dyr = dyp + b * L + 128 * (u0 + ch0) + v;  // chunk ch0 + c: dyr[128 c]
        float dv[16];
        float4 xq[5];
        if (128 * (u0 + kFtStageChunks) <= L) {
#pragma unroll
          for (int c = 0; c < 16; ++c) dv[c] = __ldg(dyr + 128 * c);
        } else {
          const int64_t rem = L - 128 * (u0 + ch0) - v;  // chunk ch0 + c is valid iff 128 c < rem
#pragma unroll
          for (int c = 0; c < 16; ++c) dv[c] = 128 * c < rem ? __ldg(dyr + 128 * c) : 0.0f;
        }
        // x rows of the stage from the raw TMA ring (x past the row end is the next row's data or the
        // TMA's zero fill past the array: finite, and only ever multiplied by the zero dy of i >= L)
        {
          const int rs = it % kFtRaw;
          ft_wait(rfull + rs, (uint32_t)(it / kFtRaw) & 1u);
          const float* xr = raw + rs * (kFtRawBytes / 4) + 128 * xrow + s4;  // item m: xr[1024 m]
#pragma unroll
          for (int m = 0; m < 5; ++m)
            xq[m] = (m < 4 || xrow == 0) ? *reinterpret_cast<const float4*>(xr + 1024 * m)
                                         : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          mbar_arrive(rempty + rs);
        }
        // the loads are in flight while the MMA drains this group's previous stage (same slot)
        mbar_wait(empty + st, ((uint32_t)(it / kFtStages) & 1u) ^ 1u);  // sleeping wait: 16 spinning warps
        // would take issue slots from the MMA warp
        // A: dy chunk values of lane v, split into TF32 hi and the exact remainder
        {
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const uint32_t h = tf32_hi(__float_as_uint(dv[c]));
            hi[c] = h;
            const float l = dv[c] - __uint_as_float(h);
            lo[c] = kFtMixed ? bf16_pack(__uint_as_float(h), l) : __float_as_uint(l);  // mixed: (hi, lo) K pair
          }
          tmem_st16(tmem + lanebits + kAcol + 64u * st + (uint32_t)ch0, hi);
          tmem_st16(tmem + lanebits + kAcol + 64u * st + 32u + (uint32_t)ch0, lo);
        }
        // B: x rows u0 .. u0 + 32 (row r = x[b][128 (u0 + r) + s]), hi and lo, MN-major BASE32B swizzle
        {
          const uint32_t bh = smem_u32(bsm + (size_t)st * 2 * kFtB) + xoff0, bl = bh + kFtB;
          const uint32_t bp = smem_u32(bsm + (size_t)st * 2 * kFtB + kFtB);
          const uint32_t bp0 = bp + xoffp0, bp1 = bp + xoffp1;
#pragma unroll
          for (int m = 0; m < 5; ++m) {
            if (m < 4 || xrow == 0) {
              const float4 xv = xq[m];
              const uint32_t h0 = tf32_hi(__float_as_uint(xv.x)), h1 = tf32_hi(__float_as_uint(xv.y));
              const uint32_t h2 = tf32_hi(__float_as_uint(xv.z)), h3 = tf32_hi(__float_as_uint(xv.w));
              const float l0 = xv.x - __uint_as_float(h0), l1 = xv.y - __uint_as_float(h1);
              const float l2 = xv.z - __uint_as_float(h2), l3 = xv.w - __uint_as_float(h3);
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bh + 1024u * m), "r"(h0), "r"(h1), "r"(h2),
                           "r"(h3)
                           : "memory");
              if (kFtMixed) {  // rows 2 r (lo) and 2 r + 1 (hi) of the bf16 pair tile
                asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(bp0 + 2048u * m), "r"(bf16_pack(l0, l1)),
                             "r"(bf16_pack(l2, l3))
                             : "memory");
                asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(bp1 + 2048u * m),
                             "r"(bf16_pack(__uint_as_float(h0), __uint_as_float(h1))),
                             "r"(bf16_pack(__uint_as_float(h2), __uint_as_float(h3)))
                             : "memory");
              } else {
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(bl + 1024u * m), "f"(l0), "f"(l1), "f"(l2),
                             "f"(l3)
                             : "memory");
              }
            }
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_proxy_async_smem();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(full + st);
      }
    }
  } else if (warp == kFtWarpTma) {
    // ------------------------------------------------------------ raw x rows of each stage by TMA
    if (lane == 0) {
      int it = 0;
      for (int64_t unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
        const int64_t b = unit / UR, q = unit - b * UR;
        for (int s2 = 0; s2 < kFtUnitStages; ++s2, ++it) {
          const int rs = it % kFtRaw;
          mbar_wait(rempty + rs, ((uint32_t)(it / kFtRaw) & 1u) ^ 1u);
          // one box of 33 rows of 128 (x viewed as [batch N / 128][128]; N % 128 == 0)
          const int32_t row0 = (int32_t)((b * N) / 128 + q * kFtUnitChunks + s2 * kFtStageChunks);
          float* dst = raw + rs * (kFtRawBytes / 4);
          mbar_arrive_expect_tx(rfull + rs, 33u * 512u);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
              "l"(reinterpret_cast<uint64_t>(&p.tm_x)), "r"(0), "r"(row0), "r"(smem_u32(rfull + rs))
              : "memory");
        }
      }
    }
  } else if (warp == kFtWarpMma) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t i128 = idesc_tf32_bmn(128, 128), i64 = idesc_tf32_bmn(128, 64);
    constexpr uint32_t j128 = idesc_bf16_bmn(128, 128), j64 = idesc_bf16_bmn(128, 64);
    const uint32_t b0 = __shfl_sync(0xffffffffu, smem_u32(bsm), 0);
    int it = 0, d = 0;
    uint32_t dph = 0;
    for (int64_t unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
      ft_wait(dempty + d, dph ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dcol = tmem + 192u * d;
      for (int s2 = 0; s2 < kFtUnitStages; ++s2, ++it) {
        const int st = it % kFtStages;
        ft_wait(full + st, (uint32_t)(it / kFtStages) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t bh = b0 + (uint32_t)st * 2u * kFtB, bl = bh + kFtB;
        const uint32_t ah = tmem + kAcol + 64u * st, al = ah + 32u;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (kFtMixed) {
            const uint32_t acc = (s2 == 0 && g == 0) ? 0u : 1u;
            ft_mma(dcol, ah + 8u * g, mn32_desc(bh + 1024u * g), i128, acc);          // hi * hi, TF32
            ft_mma(dcol + 128u, ah + 8u * g, mn32_desc(bh + 1024u * g + 128u), i64, acc);
            ft_mma(dcol, al + 8u * g, mn16_desc(bl + 2048u * g), j128, 1u);           // both cross terms, bf16
            ft_mma(dcol + 128u, al + 8u * g, mn16_desc(bl + 2048u * g + 256u), j64, 1u);
          } else {
#pragma unroll
            for (int pr = 0; pr < 3; ++pr) {  // hi*hi, hi*lo, lo*hi
              const uint32_t a = (pr == 2 ? al : ah) + 8u * g;
              const uint32_t bb = (pr == 1 ? bl : bh) + 1024u * g;
              const uint32_t acc = (s2 == 0 && g == 0 && pr == 0) ? 0u : 1u;
              ft_mma(dcol, a, mn32_desc(bb), i128, acc);
              ft_mma(dcol + 128u, a, mn32_desc(bb + 128u), i64, acc);
            }
          }
        }
        ft_commit(empty + st);
      }
      ft_commit(dfull + d);
      if (++d == 2) { d = 0; dph ^= 1u; }
    }
  } else {
    // ------------------------------------------------------------ epilogue: diagonal sums
    const int qd = warp & 3, v = 32 * qd + lane, e = threadIdx.x - 32 * kFtEpi0;  // e in [0, 128)
    const uint32_t lanebits = (uint32_t)(32 * qd) << 16;
    const int j = e & 63, h = e >> 6;
    double acc = 0.0;
    int d = 0;
    uint32_t dph = 0;
    for (int64_t unit = blockIdx.x; unit < nunits; unit += gridDim.x) {
      ft_wait(dfull + d, dph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // row v of C, columns 32 qd + [0, 96)  ->  cs[v][0, 96), 32 columns at a time (registers)
#pragma unroll 1
      for (int t = 0; t < 3; ++t) {
        uint32_t c[32];
        tmem_ld32(tmem + lanebits + (uint32_t)(192 * d + 32 * qd + 32 * t), c);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (t == 2) {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(dempty + d);
        }
#pragma unroll
        for (int i2 = 0; i2 < 32; ++i2) cs[v * kFtPitch + 32 * t + i2] = __uint_as_float(c[i2]);
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      // thread (j, h): sum over v' in [64 h, 64 h + 64) of C[v'][v' + j] = cs[v'][v' % 32 + j]
      {
        // 8 fp32 partial sums of 8 terms each (|error| <= 8 ulp of the partial), then double
        float f[8];
#pragma unroll
        for (int g2 = 0; g2 < 8; ++g2) {
          float t2 = 0.0f;
#pragma unroll
          for (int w2 = 0; w2 < 8; ++w2) {
            const int vv = 64 * h + 8 * g2 + w2;
            t2 += cs[vv * kFtPitch + (vv & 31) + j];
          }
          f[g2] = t2;
        }
        double s = 0.0;
#pragma unroll
        for (int g2 = 0; g2 < 8; ++g2) s += (double)f[g2];
        acc += s;
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (++d == 2) { d = 0; dph ^= 1u; }
    }
    red[e] = acc;
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (e < 64) {
      double* part = p.part;
      part[(size_t)blockIdx.x * 64 + e] = red[e] + red[64 + e];
      for (int64_t c2 = blockIdx.x + gridDim.x; c2 < p.ctas; c2 += gridDim.x) part[(size_t)c2 * 64 + e] = 0.0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

bool conv_filter_grad_tc_supported(int64_t N, int64_t k, int64_t stride, const void* x) {
  return stride == 1 && k >= 1 && k <= 64 && N % 128 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
         tc_filter_grad_enabled();  // (and batch N < 2^31 for the TMA map: checked by the caller's encode)
}

cudaError_t launch_conv_filter_grad_tc(FgradTcParams& p, float* df, int ctas, int sms, cudaStream_t stream) {
  p.U = (p.L + 127) / 128;
  p.units_per_row = (p.U + kFtUnitChunks - 1) / kFtUnitChunks;
  p.nunits = p.batch * p.units_per_row;
  p.ctas = ctas;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(conv_filter_grad_tc_kernel));
  if (e != cudaSuccess) return e;
  int64_t g = sms < ctas ? sms : ctas;
  if (g > p.nunits) g = p.nunits < 1 ? 1 : p.nunits;
  conv_filter_grad_tc_kernel<<<(unsigned)g, kFtThreads, kFtSmem, stream>>>(p);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_conv_filter_grad_finish(p.part, ctas, p.k, df, stream);
}

}  // namespace ss
