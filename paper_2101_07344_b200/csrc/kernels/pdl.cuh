// Programmatic dependent launch: every serve-path kernel is launched with
// programmatic stream serialization, so kernel N+1's CTAs are scheduled while
// kernel N drains and run their data-independent prologue (mbarrier init,
// TMEM allocation, tensor-map prefetch) before griddepcontrol.wait. The wait
// returns once the previous grid has completed and its writes are visible;
// every kernel executes it before touching data produced upstream (counts,
// survivor ids, activations), which keeps the dependency chain transitive.
// LCB_NO_PDL=1 launches plainly (A/B measurement).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace lcb {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LCB_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace lcb

// Per-device one-time setup (cudaFuncSetAttribute applies to the current
// device only): true the first time it is called on each device.
#include <atomic>
inline bool first_on_device(std::atomic<unsigned long long>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const unsigned long long bit = 1ull << dev;
  return (done.fetch_or(bit) & bit) == 0;
}

