// Persistent kernel of the parity mode (parity.cuh), compiled as its own
// translation unit so the fast solver (capi.cu) and the checker-order solver
// build in parallel.  Launched by capi.cu's launch() when cfg.parity is set.
#include <cuda_runtime.h>

#include "kernel_setup.cuh"
#include "parity.cuh"

namespace hallar {

__global__ void __launch_bounds__(kThreads, 1)
    hallar_parity_kernel(const __grid_constant__ Params P, SolveOut* so) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ctx c;
  setup_ctx(c, P, smem_raw);
  c.Pp = &P;  // debug hooks of the job phases (parity.cuh)
  p_dispatch(c, P, so);
}

const void* hallar_parity_kernel_fn() { return (const void*)hallar_parity_kernel; }

int hallar_parity_prepare() {
  if (cudaFuncSetAttribute(hallar_parity_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(kSmemBytes)) != cudaSuccess)
    return 0;
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, hallar_parity_kernel, kThreads,
                                                    kSmemBytes) != cudaSuccess)
    return 0;
  return per;
}

}  // namespace hallar
