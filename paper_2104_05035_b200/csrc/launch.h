// launch.h — kernel launches with Programmatic Dependent Launch (PDL).
// Every kernel of the step starts with griddepcontrol.wait (pdl_wait(): no
// reads of predecessor output before it) and then lets its successor begin
// launching (pdl_trigger()), so a dependent kernel's launch latency and
// prologue (barrier init, TMEM allocation, tensor-map prefetch) overlap the
// tail of the previous one — in plain streams and in the captured CUDA graphs.
// Memory visibility is unchanged: griddepcontrol.wait returns only after the
// whole predecessor grid has completed and flushed (transitively for chains).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>

#include "error.h"

namespace rn {

bool pdl_enabled();

// true if this call site already ran on the current device (bit per device
// ordinal in *mask), else marks it: function attributes such as the dynamic-smem
// limit are per device, so a process that drives a second GPU sets them again
inline bool once_on_device(uint64_t &mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (mask & bit) return true;
  mask |= bit;
  return false;
}

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx", __FILE__, __LINE__);
}

}  // namespace rn
