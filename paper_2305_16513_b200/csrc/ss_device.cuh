// ss_device.cuh -- device-side building blocks for the sm_100a kernels:
// mbarrier / TMA (cp.async.bulk.tensor) PTX wrappers, the 128-byte swizzle,
// and the associative operators (+) of Eq. 3.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstring>

namespace ss {

// ---------------------------------------------------------------- operators
// Eq. 3's (+): the identity is the element neutral for (+) (reading R6: the
// "0" lanes of Alg. 1/2 are the identity of the operator).
struct OpSumI32 {
  using T = int32_t;
  static __device__ __forceinline__ T identity() { return 0; }
  // wrapping addition modulo 2^32 (computed in uint32: no UB)
  static __device__ __forceinline__ T combine(T a, T b) {
    return (T)((uint32_t)a + (uint32_t)b);
  }
};
struct OpSumF32 {
  using T = float;
  static __device__ __forceinline__ T identity() { return 0.0f; }
  static __device__ __forceinline__ T combine(T a, T b) { return __fadd_rn(a, b); }
};
struct OpMaxI32 {
  using T = int32_t;
  static __device__ __forceinline__ T identity() { return INT32_MIN; }
  static __device__ __forceinline__ T combine(T a, T b) { return a > b ? a : b; }
};
struct OpMaxF32 {
  using T = float;
  static __device__ __forceinline__ T identity() { return -INFINITY; }
  // FMNMX: equals `a > b ? a : b` for finite inputs (ss.h: NaN unsupported,
  // the sign of a zero maximum unspecified)
  static __device__ __forceinline__ T combine(T a, T b) { return fmaxf(a, b); }
};
// Sliding min (Sec. 2.3's other extremum; "min is associative").
struct OpMinI32 {
  using T = int32_t;
  static __device__ __forceinline__ T identity() { return INT32_MAX; }
  static __device__ __forceinline__ T combine(T a, T b) { return a < b ? a : b; }
};
struct OpMinF32 {
  using T = float;
  static __device__ __forceinline__ T identity() { return INFINITY; }
  static __device__ __forceinline__ T combine(T a, T b) { return fminf(a, b); }
};

// ---------------------------------------------------------------- smem / PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// CU_TENSOR_MAP_SWIZZLE_128B: inside each 1024-B block the 16-B chunk index
// (address bits 4..6) is XORed with the 128-B row index (bits 7..9).
__device__ __forceinline__ uint32_t swz128(uint32_t byte_off) {
  return byte_off ^ ((byte_off >> 3) & 0x70u);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  // try_wait with a suspend-time hint: the warp sleeps in hardware until the
  // phase completes (or ~1 ms passes) instead of spinning on issue slots.
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// try_wait without a suspend hint (polling).  Needed where the phase is
// completed by cp.async.mbarrier.arrive: ncu showed the hinted wait sleeping
// out its NANOSLEEP there instead of waking on the arrival.
__device__ __forceinline__ void mbar_wait_poll(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA 2-D tile load global -> shared, completion on an mbarrier (tx bytes).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map,
                                            int32_t c0, int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy global -> shared (16-B aligned addresses, size % 16 == 0).
__device__ __forceinline__ void bulk_load_1d(void* smem_dst, const void* gsrc, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA 2-D tile store shared -> global (bulk async-group completion).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int32_t c0, int32_t c1,
                                             const void* smem_src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(smem_src))
      : "memory");
}
// 1-D bulk copy shared -> global (bulk async-group completion; 16-B aligned
// addresses, size % 16 == 0).
__device__ __forceinline__ void bulk_store_1d(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<uint64_t>(gdst)),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
// Ampere-style asynchronous copies global -> shared (LDGSTS); bytes past
// src_bytes are zero-filled and not read.
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Generic-proxy smem writes -> visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

template <typename To, typename From>
__device__ __forceinline__ To bitcast(From v) {
  static_assert(sizeof(To) == sizeof(From), "bitcast size");
  To r;
  memcpy(&r, &v, sizeof(To));
  return r;
}


// ---------------------------------------------------------------- work claims
// Dynamic work distribution by cluster launch control (sm_100 CLC): the grid
// has one CTA per work unit (tile / plane); a running CTA cancels the launch of
// a CTA that has not started yet and processes that CTA's unit itself, so the
// SMs that stream faster take more units and the kernel ends on its slowest
// unit, not its slowest SM.  The claim lives in the hardware scheduler: no
// global memory, nothing shared between launches or graph replays (ss.h
// ownership contract).  With clc == 0 the kernels stride statically by
// gridDim.x over a persistent grid instead (SS_DYNAMIC_TILES=0, A/B only).
struct alignas(16) ClcSmem {
  uint4 resp;    // 16-B try_cancel response
  uint64_t bar;  // its mbarrier (arrival count 1, tx 16 B)
};

__device__ __forceinline__ void clc_init(ClcSmem* c) { mbar_init(&c->bar, 1); }

// One thread: request the cancellation of a not-yet-launched CTA.  At most one
// request may be outstanding; none may follow a failed response.
__device__ __forceinline__ void clc_request(ClcSmem* c) {
  fence_proxy_async_smem();  // the previous response was read by the generic proxy
  mbar_arrive_expect_tx(&c->bar, 16);
  asm volatile(
      "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
          smem_u32(&c->resp)),
      "r"(smem_u32(&c->bar))
      : "memory");
}

// Wait for the outstanding request (phase bit `ph`, flipped here); returns the
// x index of the canceled CTA -- the claimed unit -- or -1 if none was left.
__device__ __forceinline__ int64_t clc_wait(ClcSmem* c, uint32_t& ph) {
  mbar_wait(&c->bar, ph);
  ph ^= 1u;
  uint32_t ok, id;
  uint64_t lo, hi;
  asm volatile(
      "{\n\t.reg .b128 r;\n\t.reg .pred p;\n\t"
      "ld.shared.v2.b64 {%2, %3}, [%4];\n\t"
      "mov.b128 r, {%2, %3};\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t"
      "mov.u32 %1, 0;\n\t"
      "@p clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, r;\n\t"
      "}"
      : "=r"(ok), "=r"(id), "=l"(lo), "=l"(hi)
      : "r"(smem_u32(&c->resp))
      : "memory");
  (void)lo;
  (void)hi;
  return ok ? (int64_t)id : -1;
}

// Producer side of a plane (or tile) ring: CTA b starts with unit b, then claims
// units by CLC (clc != 0) or strides by gridDim.x.  For each unit it waits for
// the stage, publishes the unit id in pid[stage] and calls load(unit, stage),
// which must arm full[stage] (release: consumers read pid after their full
// wait); the end marker is pid = -1 with a plain arrive.
template <class Load>
__device__ __forceinline__ void plane_producer(int64_t units, int clc, ClcSmem* cs, int S, uint64_t* full,
                                               uint64_t* empty, int64_t* pid, Load load) {
  int64_t u = blockIdx.x;
  uint32_t cph = 0;
  if (clc && u < units) clc_request(cs);
  for (int it = 0;; ++it) {
    const int s = it % S;
    mbar_wait(&empty[s], ((uint32_t)(it / S) & 1u) ^ 1u);
    if (u < 0 || u >= units) {
      pid[s] = -1;
      mbar_arrive(&full[s]);
      break;
    }
    pid[s] = u;
    load(u, s);
    if (clc) {
      u = clc_wait(cs, cph);  // the claim's round trip overlapped the stage wait and the load issue
      if (u >= 0) clc_request(cs);
    } else {
      u += gridDim.x;
    }
  }
}

}  // namespace ss
