// launch_util.cuh — programmatic dependent launch (PDL) for the decode step.
//
// While the engine records the decode CUDA graph it turns PDL on
// (rlhf_set_pdl): every decode kernel is then launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, may be scheduled while
// its predecessor drains, and blocks in griddepcontrol.wait (pdl_entry) before
// touching anything the predecessor produced.  Outside PDL launches the wait is
// a no-op, so the same kernels serve the non-decode stages unchanged.
#pragma once

#include <cuda_runtime.h>

namespace rlhf {

inline thread_local int g_pdl = 0;

__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Trigger first, then wait: for kernels whose successor's pre-wait work only touches
// data that is final before this kernel's predecessor ran (decode LayerNorm -> GEMM
// weight prefetch).  The step's embed kernel keeps pdl_entry() so that every later
// kernel of a decode step may assume the previous step has completed.
__device__ __forceinline__ void pdl_entry_early() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline int launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...) == cudaSuccess ? 0 : 5;
}

}  // namespace rlhf
