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

// Sense-counter barrier: arrival is an acq_rel atomic (gpu scope) and the waiters
// spin on an acquire load of the generation, which orders every block's prior
// writes before any block's later reads.  (Against the volatile-spin version with
// two __threadfence()s: C1 1.11 -> 1.01 ms, C2 0.163 -> 0.159 s, C3 0.926 -> 0.905 s.)
__device__ __forceinline__ void grid_sync(GridBar *b) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int g, old;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&b->gen) : "memory");
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&b->count) : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(&b->count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&b->gen) : "memory");
    } else {
      unsigned int cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&b->gen) : "memory");
      } while (cur == g);
    }
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
