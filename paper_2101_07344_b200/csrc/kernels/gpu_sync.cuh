// Inter-CTA arrival counters without full fences.
//
// Pattern (one thread per CTA publishes, the block barrier before it orders
// the whole CTA's prior global writes - fence cumulativity):
//   <all threads write>; __syncthreads(); if (t == 0) old = atom_add_acq_rel(ctr, 1);
//   __syncthreads(); <all threads read other CTAs' data with ld.cg>
// __threadfence() in every thread compiles to MEMBAR.SC.GPU + L1 invalidate
// per thread; executed per tile by 256 epilogue threads it cost the fused
// lookup conv ~3x its runtime (ncu, profiles/r02c_*).
#pragma once

namespace lcb {

// atom.add with acquire + release semantics at GPU scope: publishes the
// CTA's writes (after a block barrier) and acquires the other arrivals'.
__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

}  // namespace lcb
