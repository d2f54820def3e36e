// ggnn_capi_util.cuh -- error plumbing shared by the C-ABI translation units.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>
#include "ggnn_b200.h"

namespace ggnn {

void set_error(const char* fmt, ...);

#define GGNN_CHECK_ARG(cond, ...)          \
  do {                                     \
    if (!(cond)) {                         \
      ::ggnn::set_error(__VA_ARGS__);      \
      return GGNN_E_INVALID;               \
    }                                      \
  } while (0)

#define GGNN_CUDA_TRY(expr)                                                                  \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      ::ggnn::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return GGNN_E_CUDA;                                                                    \
    }                                                                                        \
  } while (0)

#define GGNN_LAUNCH_CHECK() GGNN_CUDA_TRY(cudaGetLastError())

// process-wide count of the kernels this library launched (ggnn_kernel_launches)
void count_launch(int n = 1);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

struct DevInfo {
  int sm_count;
  int smem_optin;
  int smem_per_sm;  // shared memory per multiprocessor (bytes, incl. the 1 KB per CTA the runtime reserves)
};
DevInfo dev_info();

}  // namespace ggnn
