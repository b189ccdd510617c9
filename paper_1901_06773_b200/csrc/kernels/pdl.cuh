// Programmatic dependent launch (PDL) for every kernel of the step.
//
// Each kernel is launched with cudaLaunchAttributeProgrammaticStreamSerialization,
// so inside a stream (or a CUDA graph captured from it) the next kernel's CTAs
// may be dispatched while the previous kernel drains.  Every kernel therefore
// calls pdl_wait() before its first global-memory access (read or write:
// the predecessor may still be reading what this kernel overwrites) and
// pdl_trigger() to let its own successor be scheduled.  Prologue work that
// touches no global memory (mbarrier init, TMEM allocation, tensor-map
// prefetch from the parameter space) runs before the wait and overlaps the
// predecessor's tail.  In a launch without the attribute both are no-ops.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace accudnn {

extern int g_pdl;  // process-wide switch (accudnn_set_pdl), default off

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace accudnn
