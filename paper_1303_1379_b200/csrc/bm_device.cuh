// bm_device.cuh — device-side primitives for the B200 matching engine.
//
// Memory contract. The reference runs its kernels on emulated threads whose
// shared accesses are relaxed, indivisible 32-bit loads/stores with
// last-writer-wins semantics (kernel_grid.hpp:17-36). On sm_100a that is a
// plain 32-bit global access; the only extra care a *persistent* kernel
// needs is that L1 is not coherent across SMs inside one launch, so every
// read of state another CTA may have written goes to L2 (ld.relaxed.gpu /
// ld.global.cg), and read-only graph data goes through the non-coherent
// path (ld.global.nc).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bm {

constexpr unsigned kFull = 0xffffffffu;

// ---- loads / stores -------------------------------------------------------
__device__ __forceinline__ int ld_rlx(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// L2-coherent (bypass L1) loads for data written earlier in the same launch.
__device__ __forceinline__ int ld_cg(const int* p) {
  int v;
  asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ld_cg(const int4* p) {
  int4 v;
  asm volatile("ld.global.cg.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ int2 ld_cg(const int2* p) {
  int2 v;
  asm volatile("ld.global.cg.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_cg_u(const int4* p) {  // .w field only
  unsigned v;
  asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(v) : "l"(reinterpret_cast<const char*>(p) + 12));
  return v;
}
// L1-cacheable load for heuristic reads where a value up to one grid barrier
// old is acceptable (WR root marks).
__device__ __forceinline__ int ld_ca(const int* p) {
  int v;
  asm volatile("ld.global.ca.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// Read-only graph data (never written inside a launch).
__device__ __forceinline__ int ld_ro(const int* p) {
  int v;
  asm("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_ro(const unsigned* p) {
  unsigned v;
  asm("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ld_ro2(const unsigned* p) {  // p 8-byte aligned
  uint2 v;
  asm("ld.global.nc.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_rlx(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rlx(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_plain(int* p, int v) {
  asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_plain(int2* p, int2 v) {
  asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void st_plain(int4* p, int4 v) {
  asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// ---- L2 eviction policy for streamed data ---------------------------------
// Adjacency rows, frontier entries and predecessor stores are touched once
// per level; marking them evict_first keeps the randomly gathered state
// (rmatch, the visited bitmap, offsets, root marks) resident in L2.
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Coherent (L2) load with an L2 eviction-priority hint.
__device__ __forceinline__ int ld_rlx_hint(const int* p, unsigned long long pol) {
  int v;
  asm volatile("ld.relaxed.gpu.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx_hint(const unsigned* p, unsigned long long pol) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_ro_hint(const unsigned* p, unsigned long long pol) {
  unsigned v;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_stream(const int* p, unsigned long long pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int4 ld_cg_stream(const int4* p, unsigned long long pol) {
  int4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream(int* p, int v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream(int2* p, int2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1,%2}, %3;" ::"l"(p), "r"(v.x), "r"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_stream(int4* p, int4 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2n(const void* p) {  // normal eviction priority (streamed data)
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---- warp helpers ----------------------------------------------------------
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned warp_incl_scan(unsigned v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned t = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

}  // namespace bm
