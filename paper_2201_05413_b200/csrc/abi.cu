// abi.cu — error reporting and diagnostics of the C ABI (include/pcg.h).
#include <atomic>
#include <string>

#include "common.cuh"

namespace pcgb {

static thread_local std::string t_last_error;
std::atomic<int64_t> g_host_launches{0};

void set_error(const std::string &msg) { t_last_error = msg; }

pcg_status fail(pcg_status s, const std::string &msg) {
  t_last_error = msg;
  return s;
}

}  // namespace pcgb

extern "C" const char *pcg_last_error(void) { return pcgb::t_last_error.c_str(); }

extern "C" const char *pcg_status_string(pcg_status s) {
  switch (s) {
    case PCG_OK: return "PCG_OK";
    case PCG_NOT_CONVERGED: return "PCG_NOT_CONVERGED";
    case PCG_ERR_INVALID_ARG: return "PCG_ERR_INVALID_ARG";
    case PCG_ERR_INDEX_OUT_OF_RANGE: return "PCG_ERR_INDEX_OUT_OF_RANGE";
    case PCG_ERR_UNSORTED_OR_DUPLICATE: return "PCG_ERR_UNSORTED_OR_DUPLICATE";
    case PCG_ERR_DIMENSION_MISMATCH: return "PCG_ERR_DIMENSION_MISMATCH";
    case PCG_ERR_ZERO_DIAGONAL: return "PCG_ERR_ZERO_DIAGONAL";
    case PCG_ERR_NOT_SPD: return "PCG_ERR_NOT_SPD";
    case PCG_ERR_NONFINITE: return "PCG_ERR_NONFINITE";
    case PCG_ERR_OOM: return "PCG_ERR_OOM";
    case PCG_ERR_CUDA: return "PCG_ERR_CUDA";
    case PCG_ERR_NCCL: return "PCG_ERR_NCCL";
    case PCG_ERR_BREAKDOWN: return "PCG_ERR_BREAKDOWN";
  }
  return "PCG_UNKNOWN";
}

extern "C" int64_t pcg_kernel_launches(void) { return pcgb::g_host_launches.load(); }
