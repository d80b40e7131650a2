// affine.cu -- sliding window of gamma pairs.
//
// The paper's pair operator (Eq. 8)
//     gamma_i (+) gamma_j = (u_i u_j, u_j v_i + v_j)
// is associative but not commutative.  Sliding it over a
// sequence with window w (Eq. 3) gives, per output i,
//     (U_i, V_i) = gamma_i (+) gamma_{i+1} (+) ... (+) gamma_{i+w-1},
// i.e. the linear recurrence s_t = u_t s_{t-1} + v_t run over each window from
// s = 0 (V_i) together with its gain (U_i).  No inverse exists in general
// (u may be 0), so the evaluation uses only (+) in left-to-right order.
//
// Kernel design (stride 1, w >= 9): the P-block pivot of Eq. 3 (Alg. 2's
// prefix/suffix decomposition) with P = 8 outputs per thread, order-preserving:
//   y_{8t+r} = S_t[r] (+) M_t (+) H_t[0 .. r+rho]
// where S_t[r] is the suffix of the thread's own 8-element block, M_t is the
// fold of the m = q-1 whole blocks in between (q = (w-1)/8, rho = (w-1)%8), and
// H_t the first elements of block t+q.  M_t is itself a sliding window of
// length m over the block totals; it is evaluated with one more level of the
// same decomposition (segments of length m; per-segment prefix and suffix
// scans in shared memory, one thread or one warp per segment), so the cost per
// output is O(1) in w: ~4 (+) from registers plus ~1 for the block totals.
// w <= 8 folds each window directly (<= 7 (+) per output); stride > 1 folds
// each window directly from global memory (O(w) per output).
//
// Data movement (w <= 2049): persistent CTAs, the next tile's input span
// copied with cp.async into a double buffer while the current tile computes,
// outputs staged in shared memory and written with 1-D bulk copies.
#include <cstdint>

#include <cuda_runtime.h>

#include "ss_device.cuh"
#include "ss_internal.h"

namespace ss {

struct Gp {
  float u, v;
};

// Eq. 8, a on the left: (a.u * b.u, b.u * a.v + b.v), one rounding each.
__device__ __forceinline__ Gp gcomb(Gp a, Gp b) { return Gp{a.u * b.u, fmaf(b.u, a.v, b.v)}; }
__device__ __forceinline__ Gp gid() { return Gp{1.f, 0.f}; }

constexpr int kAffThreads = 256;
constexpr int kAffR = 8;
constexpr int kAffTile = kAffThreads * kAffR;
constexpr int kAffStagedMaxQ = 256;  // w <= 2049 runs the pipelined kernel

// 8 consecutive pairs of one row starting at row element e (>= 0); elements at
// or beyond N read as the identity (1, 0).
__device__ __forceinline__ void load8(const float* __restrict__ ur, const float* __restrict__ vr,
                                      int64_t e, int64_t N, Gp* g) {
  const float* pu = ur + e;
  const float* pv = vr + e;
  if (e + 8 <= N && ((reinterpret_cast<uintptr_t>(pu) | reinterpret_cast<uintptr_t>(pv)) & 15) == 0) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(pu));
    const float4 b = __ldg(reinterpret_cast<const float4*>(pu) + 1);
    const float4 c = __ldg(reinterpret_cast<const float4*>(pv));
    const float4 d = __ldg(reinterpret_cast<const float4*>(pv) + 1);
    g[0] = Gp{a.x, c.x}; g[1] = Gp{a.y, c.y}; g[2] = Gp{a.z, c.z}; g[3] = Gp{a.w, c.w};
    g[4] = Gp{b.x, d.x}; g[5] = Gp{b.y, d.y}; g[6] = Gp{b.z, d.z}; g[7] = Gp{b.w, d.w};
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = (e + j < N) ? Gp{__ldg(pu + j), __ldg(pv + j)} : gid();
  }
}

// Store up to 8 outputs (n = how many are valid); U may be null.
__device__ __forceinline__ void store8(float* __restrict__ U, float* __restrict__ V, int64_t o,
                                       int64_t n, const Gp* y) {
  float* pv = V + o;
  float* pu = U ? U + o : nullptr;
  if (n >= 8 && ((reinterpret_cast<uintptr_t>(pv) | reinterpret_cast<uintptr_t>(pu)) & 15) == 0) {
    reinterpret_cast<float4*>(pv)[0] = make_float4(y[0].v, y[1].v, y[2].v, y[3].v);
    reinterpret_cast<float4*>(pv)[1] = make_float4(y[4].v, y[5].v, y[6].v, y[7].v);
    if (pu) {
      reinterpret_cast<float4*>(pu)[0] = make_float4(y[0].u, y[1].u, y[2].u, y[3].u);
      reinterpret_cast<float4*>(pu)[1] = make_float4(y[4].u, y[5].u, y[6].u, y[7].u);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < n) {
        pv[j] = y[j].v;
        if (pu) pu[j] = y[j].u;
      }
  }
}

// ---- sources of 8-pair runs at tile-local offsets (multiples of 8) ----------
struct GlobalSrc {
  const float* ur;
  const float* vr;
  int64_t i0, N;
  __device__ __forceinline__ void load8(int le, Gp* g) const { ss::load8(ur, vr, i0 + le, N, g); }
};

// Staged span layout: u and v in separate float arrays; 16-B chunk j of a
// 128-B row r sits at chunk ((j + (r & 1)) & 7) of that row (odd rows rotated
// by one chunk).  Eight lanes reading the same half of 8 consecutive 8-float
// runs from ANY 8-aligned start then hit 8 distinct 16-B bank groups: runs at
// the same offset mod 4 lie in adjacent rows of opposite parity.
__device__ __forceinline__ int swz_chunk(int j) { return (j & ~7) | (((j & 7) + ((j >> 3) & 1)) & 7); }

struct SmemSrc {
  const float* su;
  const float* sv;
  __device__ __forceinline__ void load8(int le, Gp* g) const {
    const int j0 = swz_chunk(le >> 2) << 2, j1 = swz_chunk((le >> 2) + 1) << 2;
    const float4 a = *reinterpret_cast<const float4*>(su + j0);
    const float4 b = *reinterpret_cast<const float4*>(su + j1);
    const float4 c = *reinterpret_cast<const float4*>(sv + j0);
    const float4 d = *reinterpret_cast<const float4*>(sv + j1);
    g[0] = Gp{a.x, c.x}; g[1] = Gp{a.y, c.y}; g[2] = Gp{a.z, c.z}; g[3] = Gp{a.w, c.w};
    g[4] = Gp{b.x, d.x}; g[5] = Gp{b.y, d.y}; g[6] = Gp{b.z, d.z}; g[7] = Gp{b.w, d.w};
  }
};

// Input span of a tile: [i0, i0 + span), covering every run a thread reads
// (own block, block totals up to block 256+q, the H blocks).
__host__ __device__ constexpr int affine_span(int q) { return (kAffTile + 8 * q + 16 + 31) & ~31; }

// Issue the asynchronous copy of one array's span of a row into the swizzled
// layout at s (16-B cp.async when the row is 16-B aligned, 4-B otherwise);
// positions at or beyond N are zero-filled, never read (they only feed
// outputs >= L, which are not stored).
__device__ __forceinline__ void issue_span(const float* __restrict__ row, int64_t i0, int64_t N,
                                           int span, float* s) {
  const int t = threadIdx.x;
  const uint32_t sb = smem_u32(s);
  if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
    for (int k = t; k < (span >> 2); k += kAffThreads) {
      const int64_t e = i0 + 4 * (int64_t)k;
      const int64_t rem = N - e;
      const uint32_t nb = rem >= 4 ? 16u : (rem > 0 ? (uint32_t)rem * 4u : 0u);
      cp_async16(sb + 16u * (uint32_t)swz_chunk(k), nb ? row + e : row, nb);
    }
  } else {
    for (int k = t; k < span; k += kAffThreads) {
      const int64_t e = i0 + k;
      cp_async4(sb + 4u * (uint32_t)((swz_chunk(k >> 2) << 2) | (k & 3)), e < N ? row + e : row,
                e < N ? 4u : 0u);
    }
  }
}

// w <= 8: direct left fold of each window.
template <int W>
__device__ __forceinline__ void affine_small_body(const Gp* g, Gp* y) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    Gp a = g[r];
#pragma unroll
    for (int j = 1; j < W; ++j) a = gcomb(a, g[r + j]);
    y[r] = a;
  }
}

// w >= 9, stride 1; RHO = (w-1) % 8.  Computes the 8 outputs of thread t of
// the tile into y (all threads take part in the block-total scans).
template <int RHO, class Src>
__device__ __forceinline__ void affine_pivot_body(const AffineParams& p, const Src& src, Gp* Bt, Gp* y) {
  Gp* Pre = Bt + p.nB;
  Gp* Suf = Pre + p.nB;
  const int t = threadIdx.x;
  const int q = p.q, m = p.q - 1;

  // (1) own block + totals of blocks 1 .. nB (tile-local block index)
  Gp own[8];
  src.load8(8 * t, own);
  // M_t = blocks t+1 .. t+m = Bt[t] (+) ... (+) Bt[t+m-1], by doubling: level k holds the
  // folds of 2^k consecutive block totals (built from level k-1 by all threads, ping-pong
  // between Pre and Suf); the set bits of m, smallest first, select the pieces of M_t from
  // left to right, so the (+) order is kept.  ~log2(m) barriers, no serial scans.
  Gp M = gid();
  if (m > 0) {
    for (int k = t; k < p.nB; k += kAffThreads) {
      Gp g[8];
      src.load8(8 * (k + 1), g);
      Gp a = g[0];
#pragma unroll
      for (int j = 1; j < 8; ++j) a = gcomb(a, g[j]);
      Bt[k] = a;
    }
    __syncthreads();
    const Gp* cur = Bt;
    int off = 0;
    for (int span = 1, lvl = 0;; span <<= 1, ++lvl) {
      if (m & span) {
        M = gcomb(M, cur[t + off]);
        off += span;
      }
      if (2 * span > m) break;
      Gp* nxt = (lvl & 1) ? Suf : Pre;
      const int nn = p.nB - 2 * span + 1;  // entries i with i + 2 span <= nB
      for (int i = t; i < nn; i += kAffThreads) nxt[i] = gcomb(cur[i], cur[i + span]);
      __syncthreads();
      cur = nxt;
    }
  }
  // S_t[r]: suffixes of the own block
  Gp S[8];
  S[7] = own[7];
#pragma unroll
  for (int r = 6; r >= 0; --r) S[r] = gcomb(own[r], S[r + 1]);
  // H: block t+q (and t+q+1 when RHO > 0)
  Gp h[16];
  src.load8(8 * (t + q), h);
  if (RHO > 0) src.load8(8 * (t + q + 1), h + 8);
  Gp E = M;
#pragma unroll
  for (int j = 0; j < RHO; ++j) E = gcomb(E, h[j]);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    E = gcomb(E, h[r + RHO]);  // E = M (+) h[0 .. r+RHO]
    y[r] = gcomb(S[r], E);
  }
}

struct TileIdx {
  int64_t b, i0;
};

// Long windows (q > kAffStagedMaxQ): one tile per CTA straight from global.
template <int RHO>
__global__ void __launch_bounds__(kAffThreads) affine_pivot_global_kernel(const AffineParams p) {
  extern __shared__ __align__(16) float smem_f[];
  const TileIdx ti{(int64_t)blockIdx.x / p.tiles_per_row, ((int64_t)blockIdx.x % p.tiles_per_row) * kAffTile};
  const float* ur = p.u + ti.b * p.N;
  const float* vr = p.v + ti.b * p.N;
  Gp y[8];
  affine_pivot_body<RHO>(p, GlobalSrc{ur, vr, ti.i0, p.N}, reinterpret_cast<Gp*>(smem_f), y);
  const int64_t i = ti.i0 + (int64_t)threadIdx.x * 8;
  if (i < p.L) store8(p.U, p.V, ti.b * p.L + i, p.L - i, y);
}

// Production path (stride 1, w <= 2049): persistent CTAs walk the tiles
// blockIdx.x, +gridDim.x, ...; tile n+1's input span is copied (cp.async,
// double-buffered) while tile n is computed; the tile's outputs are staged in
// shared memory and leave with one bulk copy per array (coalesced stores when
// the output row is not 16-B aligned).  SMALL_W > 0: w = SMALL_W <= 8, direct
// folds; SMALL_W == 0: the pivot with RHO.
template <int SMALL_W, int RHO>
__global__ void __launch_bounds__(kAffThreads) affine_pipe_kernel(const AffineParams p) {
  extern __shared__ __align__(16) float smem_f[];
  const int span = affine_span(SMALL_W ? 0 : p.q);
  float* outV = smem_f;  // [kAffTile] linear
  float* outU = outV + kAffTile;
  float* buf0 = outU + kAffTile;
  Gp* Bt = reinterpret_cast<Gp*>(buf0 + 4 * span);
  const int t = threadIdx.x;
  const int64_t ntiles = p.tiles_per_row * p.batch;
  int64_t tile = blockIdx.x;
  if (tile >= ntiles) return;
  auto issue = [&](int64_t tl, float* dst) {
    const int64_t b = tl / p.tiles_per_row, i0 = (tl % p.tiles_per_row) * kAffTile;
    issue_span(p.u + b * p.N, i0, p.N, span, dst);
    issue_span(p.v + b * p.N, i0, p.N, span, dst + span);
  };
  issue(tile, buf0);
  cp_async_commit();
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) issue(next, buf0 + 2 * span * ((it + 1) & 1));
    cp_async_commit();
    cp_async_wait<1>();  // this thread's copies of the current tile have landed
    __syncthreads();     // ... and everyone else's
    const float* cur = buf0 + 2 * span * (it & 1);
    const SmemSrc src{cur, cur + span};
    Gp y[8];
    if (SMALL_W > 0) {
      Gp g[16];
      src.load8(8 * t, g);
      if (SMALL_W > 1) src.load8(8 * t + 8, g + 8);
      affine_small_body<SMALL_W>(g, y);
    } else {
      affine_pivot_body<RHO>(p, src, Bt, y);
    }
    // the previous tile's bulk stores must have finished reading outV / outU
    if (t == 0) bulk_wait_read<0>();
    __syncthreads();
    *reinterpret_cast<float4*>(outV + 8 * t) = make_float4(y[0].v, y[1].v, y[2].v, y[3].v);
    *reinterpret_cast<float4*>(outV + 8 * t + 4) = make_float4(y[4].v, y[5].v, y[6].v, y[7].v);
    if (p.U) {
      *reinterpret_cast<float4*>(outU + 8 * t) = make_float4(y[0].u, y[1].u, y[2].u, y[3].u);
      *reinterpret_cast<float4*>(outU + 8 * t + 4) = make_float4(y[4].u, y[5].u, y[6].u, y[7].u);
    }
    const int64_t b = tile / p.tiles_per_row, i0 = (tile % p.tiles_per_row) * kAffTile;
    const int nv = (int)min((int64_t)kAffTile, p.L - i0);
    float* gV = p.V + b * p.L + i0;
    float* gU = p.U ? p.U + b * p.L + i0 : nullptr;
    const bool bulk =
        ((reinterpret_cast<uintptr_t>(gV) | reinterpret_cast<uintptr_t>(gU)) & 15) == 0 && (nv & 3) == 0;
    if (bulk) fence_proxy_async_smem();
    __syncthreads();
    if (bulk) {
      if (t == 0) {
        bulk_store_1d(gV, outV, 4u * (uint32_t)nv);
        if (gU) bulk_store_1d(gU, outU, 4u * (uint32_t)nv);
        bulk_commit();
      }
    } else {
      for (int k = t; k < nv; k += kAffThreads) {
        gV[k] = outV[k];
        if (gU) gU[k] = outU[k];
      }
    }
  }
  if (t == 0) bulk_wait_all();
}

// stride > 1: one output per thread, direct left fold from global memory.
__global__ void affine_strided_kernel(const AffineParams p) {
  const int64_t total = p.batch * p.L;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = o / p.L, i = o % p.L;
    const float* ur = p.u + b * p.N + i * p.stride;
    const float* vr = p.v + b * p.N + i * p.stride;
    Gp a = Gp{__ldg(ur), __ldg(vr)};
    for (int64_t j = 1; j < p.w; ++j) a = gcomb(a, Gp{__ldg(ur + j), __ldg(vr + j)});
    p.V[o] = a.v;
    if (p.U) p.U[o] = a.u;
  }
}

static bool affine_staged(int64_t w) { return (w - 1) / 8 <= kAffStagedMaxQ; }

size_t affine_smem_bytes(int64_t w) {
  const int64_t q = (w - 1) / 8;
  const size_t bt = w <= 8 ? 0 : 3 * sizeof(Gp) * (size_t)(kAffThreads + q);
  if (!affine_staged(w)) return bt;
  return 2 * sizeof(float) * kAffTile + 4 * sizeof(float) * (size_t)affine_span(w <= 8 ? 0 : (int)q) + bt;
}

static cudaError_t launch_with_smem(const void* kfn, dim3 grid, AffineParams& p, size_t smem,
                                    cudaStream_t stream) {
  void* args[] = {&p};
  const cudaError_t e = cudaLaunchKernel(kfn, grid, dim3(kAffThreads), args, smem, stream);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_affine(AffineParams& p, cudaStream_t stream, int num_sms) {
  if (p.stride != 1) {
    const int64_t total = p.batch * p.L;
    const int64_t blocks = (total + 255) / 256, cap = (int64_t)num_sms * 8;
    affine_strided_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, stream>>>(p);
    note_launch();
    return cudaGetLastError();
  }
  p.tiles_per_row = (p.L + kAffTile - 1) / kAffTile;
  const int64_t tiles = p.tiles_per_row * p.batch;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  p.q = (int)((p.w - 1) / 8);
  p.nB = kAffThreads + p.q;  // blocks 1 .. 256+q-1 (+1 spare) of the tile
  const size_t smem = affine_smem_bytes(p.w);
  const int rho = (int)((p.w - 1) % 8);
  const void* kfn = nullptr;
  if (!affine_staged(p.w)) {
    switch (rho) {
#define SS_AFF_GLB(R) \
  case R: kfn = reinterpret_cast<const void*>(&affine_pivot_global_kernel<R>); break;
      SS_AFF_GLB(0) SS_AFF_GLB(1) SS_AFF_GLB(2) SS_AFF_GLB(3)
      SS_AFF_GLB(4) SS_AFF_GLB(5) SS_AFF_GLB(6) SS_AFF_GLB(7)
#undef SS_AFF_GLB
    }
  } else if (p.w <= 8) {
    switch (p.w) {
#define SS_AFF_SMALL(W) \
  case W: kfn = reinterpret_cast<const void*>(&affine_pipe_kernel<W, 0>); break;
      SS_AFF_SMALL(1) SS_AFF_SMALL(2) SS_AFF_SMALL(3) SS_AFF_SMALL(4)
      SS_AFF_SMALL(5) SS_AFF_SMALL(6) SS_AFF_SMALL(7) SS_AFF_SMALL(8)
#undef SS_AFF_SMALL
    }
  } else {
    switch (rho) {
#define SS_AFF_PIV(R) \
  case R: kfn = reinterpret_cast<const void*>(&affine_pipe_kernel<0, R>); break;
      SS_AFF_PIV(0) SS_AFF_PIV(1) SS_AFF_PIV(2) SS_AFF_PIV(3)
      SS_AFF_PIV(4) SS_AFF_PIV(5) SS_AFF_PIV(6) SS_AFF_PIV(7)
#undef SS_AFF_PIV
    }
  }
  if (smem > 48 * 1024) {
    const cudaError_t e = ensure_smem_attr(kfn);
    if (e != cudaSuccess) return e;
  }
  if (!affine_staged(p.w)) return launch_with_smem(kfn, dim3((unsigned)tiles), p, smem, stream);
  int per_sm = 0;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kAffThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int64_t g = (int64_t)per_sm * num_sms;
  return launch_with_smem(kfn, dim3((unsigned)(tiles < g ? tiles : g)), p, smem, stream);
}

}  // namespace ss
