// coop.cuh — grid-wide barrier and redundant fixed-order reductions for the
// persistent cooperative kernels (persist.cu, bicgstab.cu).  Co-residency of all
// blocks is the launcher's job (cudaLaunchCooperativeKernel, grid <= resident
// blocks x SMs).
#pragma once
#include "common.cuh"

namespace pcgb {

struct GridBar {
  unsigned int count;
  unsigned int gen;
};

__device__ __forceinline__ void grid_sync(GridBar *b) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int *vgen = &b->gen;
    const unsigned int g = *vgen;
    __threadfence();
    if (atomicAdd(&b->count, 1u) == gridDim.x - 1) {
      b->count = 0;
      __threadfence();
      atomicAdd(&b->gen, 1u);
    } else {
      while (*vgen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// fixed-order sum of NV x gridDim.x partials, identical in every block; result in all threads
template <int NV>
__device__ __forceinline__ void all_blocks_sum(const double *part, double (&out)[NV], double (*sm)[WARPS],
                                               double *s_tot) {
  double v[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) {
    double s = 0.0;
    for (unsigned int b = threadIdx.x; b < gridDim.x; b += BLOCK) s += __ldcg(part + (size_t)i * gridDim.x + b);
    v[i] = s;
  }
  block_sum<NV>(v, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int i = 0; i < NV; i++) s_tot[i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; i++) out[i] = s_tot[i];
  __syncthreads();
}

}  // namespace pcgb
