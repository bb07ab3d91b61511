// dar.cu — device-initiated allreduce of the distributed solvers' scalars over NVLink
// peer memory (SURVEY §8(f) N3 "device-initiated reductions").  Opt-in at
// pcg_comm_init with the environment PCG_DEVICE_ALLREDUCE=1 (NCCL communicators).
//
// Each distributed PCG iteration reduces two tiny vectors (sigma; rho', gamma) — the
// paper's VecDot, the operation it finds does not scale.  Through NCCL
// each is a collective launch; here it is one single-thread kernel on the solver's
// stream (so it is captured in the iteration graph like any kernel):
//   * every rank owns a mailbox in its own GPU memory, mapped into every peer by CUDA
//     IPC at communicator setup: slot[parity][rank][v] and flag[parity][rank];
//   * round r (a per-communicator counter kept on the device, the same sequence on
//     every rank): rank g stores its values into slot[r & 1][g] of EVERY mailbox,
//     fences at system scope, then release-stores flag[r & 1][g] = r into every
//     mailbox; it then acquire-spins on its own mailbox until all flags of parity
//     r & 1 read r, and sums slot[r & 1][0..G-1] in rank order — the same order on
//     every rank, so all ranks get bitwise the same result (the recurrence stays in
//     lockstep) and the result does not depend on arrival order (deterministic);
//   * two parities suffice: a rank enters round r + 2 only after every peer has
//     written round r + 1, i.e. after every peer has finished reading round r;
//   * a spin that sees no progress for ~8 s sets an error word in mapped host memory;
//     comm_wait (dist.cu) reads it and aborts the communicator (PCG_ERR_NCCL).
// The protocol is validated on one GPU by pcg_dar_emulate: G "ranks" as G blocks of
// one cooperative kernel, each with its own mailbox (the same device function).
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "matrix.cuh"

namespace pcgb {

constexpr int DAR_MAXG = 8;  // ranks of one node
constexpr int DAR_NV = 4;    // values per reduction (the solvers reduce at most 3)

struct DarMail {
  double slot[2][DAR_MAXG][DAR_NV];
  unsigned long long flag[2][DAR_MAXG];
};

struct DarView {
  DarMail *peer[DAR_MAXG];  // every rank's mailbox as seen from this rank (own included)
  unsigned long long *round;
  int *err;                 // mapped host memory (may be null in the emulation)
  int rank, size;
};

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double *p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// one thread: out[0..nv) = sum over ranks (in rank order) of every rank's in[0..nv)
__device__ void dar_exchange(const DarView &V, const double *in, double *out, int nv, unsigned long long r) {
  const int par = (int)(r & 1);
  double mine[DAR_NV];
  for (int v = 0; v < nv; v++) mine[v] = in[v];
  for (int p = 0; p < V.size; p++)
    for (int v = 0; v < nv; v++) V.peer[p]->slot[par][V.rank][v] = mine[v];
  __threadfence_system();
  for (int p = 0; p < V.size; p++) st_release_sys(&V.peer[p]->flag[par][V.rank], r);
  DarMail *me = V.peer[V.rank];
  const long long t0 = clock64();
  for (int q = 0; q < V.size; q++) {
    while (ld_acquire_sys(&me->flag[par][q]) < r) {
      if (clock64() - t0 > (1ll << 34)) {  // ~8.7 s at 1.97 GHz: a peer is gone
        if (V.err) *(volatile int *)V.err = 1;
        for (int v = 0; v < nv; v++) out[v] = __longlong_as_double(0x7ff8000000000000ll);  // NaN
        return;
      }
    }
  }
  for (int v = 0; v < nv; v++) {
    double s = 0.0;
    for (int q = 0; q < V.size; q++) s += ld_relaxed_sys(&me->slot[par][q][v]);
    out[v] = s;
  }
}

__global__ void dar_kernel(DarView V, double *buf, int nv) {
  const unsigned long long r = ++*V.round;  // the same sequence of rounds on every rank
  dar_exchange(V, buf, buf, nv, r);
}

// protocol self-test: block g plays rank g of G (cooperative launch: co-resident)
__global__ void dar_emulate_kernel(DarMail *mails, int G, int rounds, int nv, const double *in, double *out) {
  if (threadIdx.x != 0) return;
  DarView V;
  for (int p = 0; p < DAR_MAXG; p++) V.peer[p] = p < G ? mails + p : nullptr;
  V.round = nullptr;
  V.err = nullptr;
  V.rank = blockIdx.x;
  V.size = G;
  for (int r = 0; r < rounds; r++) {
    const size_t o = ((size_t)r * G + blockIdx.x) * nv;
    dar_exchange(V, in + o, out + o, nv, (unsigned long long)r + 1);
  }
}

struct DarState {
  DarMail *mail = nullptr;               // own mailbox
  DarMail *peers[DAR_MAXG] = {nullptr};  // opened IPC mappings (own: null)
  unsigned long long *round = nullptr;
  int *err_host = nullptr, *err_dev = nullptr;
  DarView view{};
};

void dar_free(void *p) {
  DarState *S = (DarState *)p;
  if (!S) return;
  for (DarMail *m : S->peers)
    if (m) cudaIpcCloseMemHandle(m);
  if (S->mail) cudaFree(S->mail);
  if (S->round) cudaFree(S->round);
  if (S->err_host) cudaFreeHost(S->err_host);
  delete S;
}

bool dar_failed(const void *p) { return p && *(volatile int *)((const DarState *)p)->err_host != 0; }

pcg_status dar_allreduce(void *p, double *buf, int count, cudaStream_t st) {
  DarState *S = (DarState *)p;
  for (int o = 0; o < count; o += DAR_NV) {
    dar_kernel<<<1, 1, 0, st>>>(S->view, buf + o, count - o < DAR_NV ? count - o : DAR_NV);
    count_launch();
  }
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

// Collective over the NCCL communicator: every rank maps every other rank's mailbox.
// Returns PCG_OK with *out = null (NCCL stays in use) if any rank cannot map its peers.
pcg_status dar_setup(ncclComm_t nccl, int rank, int size, void **out) {
  *out = nullptr;
  if (size > DAR_MAXG) return PCG_OK;
  DarState *S = new DarState();
  int ok = 1;
  cudaStream_t st;
  PCG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  if (cudaMalloc(&S->mail, sizeof(DarMail)) != cudaSuccess || cudaMalloc(&S->round, sizeof(unsigned long long)) != cudaSuccess ||
      cudaHostAlloc(&S->err_host, sizeof(int), cudaHostAllocMapped) != cudaSuccess)
    ok = 0;
  if (ok) {
    cudaMemset(S->mail, 0, sizeof(DarMail));
    cudaMemset(S->round, 0, sizeof(unsigned long long));
    *S->err_host = 0;
    cudaHostGetDevicePointer((void **)&S->err_dev, S->err_host, 0);
  }
  // exchange IPC handles (64 bytes each)
  cudaIpcMemHandle_t mine{};
  if (ok && cudaIpcGetMemHandle(&mine, S->mail) != cudaSuccess) ok = 0;
  cudaGetLastError();
  char *d_h = nullptr;
  int *d_ok = nullptr;
  std::vector<cudaIpcMemHandle_t> all(size);
  PCG_CUDA(cudaMalloc(&d_h, sizeof(cudaIpcMemHandle_t) * size));
  PCG_CUDA(cudaMalloc(&d_ok, sizeof(int)));
  PCG_CUDA(cudaMemcpyAsync(d_h + sizeof(cudaIpcMemHandle_t) * rank, &mine, sizeof(mine), cudaMemcpyHostToDevice, st));
  ncclResult_t nr = ncclAllGather(d_h + sizeof(cudaIpcMemHandle_t) * rank, d_h, sizeof(cudaIpcMemHandle_t), ncclChar,
                                  nccl, st);
  if (nr != ncclSuccess) ok = 0;
  PCG_CUDA(cudaMemcpyAsync(all.data(), d_h, sizeof(cudaIpcMemHandle_t) * size, cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  for (int p = 0; p < size && ok; p++) {
    if (p == rank) continue;
    void *m = nullptr;
    if (cudaIpcOpenMemHandle(&m, all[p], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
    } else {
      S->peers[p] = (DarMail *)m;
    }
  }
  // every rank must be able to map every peer, else all keep NCCL
  PCG_CUDA(cudaMemcpyAsync(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice, st));
  if (ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, nccl, st) != ncclSuccess) ok = 0;
  int all_ok = 0;
  PCG_CUDA(cudaMemcpyAsync(&all_ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_h);
  cudaFree(d_ok);
  cudaStreamDestroy(st);
  if (!ok || !all_ok) {
    dar_free(S);
    return PCG_OK;
  }
  for (int p = 0; p < DAR_MAXG; p++) S->view.peer[p] = p == rank ? S->mail : (p < size ? S->peers[p] : nullptr);
  S->view.round = S->round;
  S->view.err = S->err_dev;
  S->view.rank = rank;
  S->view.size = size;
  *out = S;
  return PCG_OK;
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status pcg_dar_emulate(int32_t G, int32_t rounds, int32_t nv, const double *in, double *out) {
  if (G < 1 || G > DAR_MAXG || rounds < 1 || nv < 1 || nv > DAR_NV || !in || !out)
    return fail(PCG_ERR_INVALID_ARG, "pcg_dar_emulate: bad argument");
  const size_t n = (size_t)rounds * G * nv;
  DarMail *mails;
  double *din, *dout;
  PCG_CUDA(cudaMalloc(&mails, sizeof(DarMail) * G));
  PCG_CUDA(cudaMemset(mails, 0, sizeof(DarMail) * G));
  PCG_CUDA(cudaMalloc(&din, sizeof(double) * n));
  PCG_CUDA(cudaMalloc(&dout, sizeof(double) * n));
  PCG_CUDA(cudaMemcpy(din, in, sizeof(double) * n, cudaMemcpyHostToDevice));
  void *args[] = {&mails, &G, &rounds, &nv, &din, &dout};
  PCG_CUDA(cudaLaunchCooperativeKernel((const void *)dar_emulate_kernel, dim3(G), dim3(32), args, 0, 0));
  count_launch();
  PCG_CUDA(cudaMemcpy(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost));
  cudaFree(mails);
  cudaFree(din);
  cudaFree(dout);
  return PCG_OK;
}
