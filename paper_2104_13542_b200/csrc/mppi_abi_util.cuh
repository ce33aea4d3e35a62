// mppi_abi_util.cuh — error plumbing and scratch buffers shared by the C-ABI
// translation units (mppi_abi.cu: plans and steps; mppi_seam.cu: the
// stateless operator-seam and cost-term functions).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "mppi_b200.h"

extern "C" int mppi_internal_fail(int code, const char* msg);  // mppi_abi.cu: sets mppi_last_error

namespace mppi {

inline int fail(int code, const std::string& msg) { return mppi_internal_fail(code, msg.c_str()); }

inline unsigned grid_for(long long n, int threads, int cap = 148 * 16) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

}  // namespace mppi

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return ::mppi::fail(MPPI_E_CUDA, std::string(#call " failed: ") + cudaGetErrorString(_e) + \
                                           " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define CKR(expr)                   \
  do {                              \
    int _rc = (expr);               \
    if (_rc != MPPI_OK) return _rc; \
  } while (0)

namespace mppi {

// Device buffers of one stateless call, on a private non-blocking stream;
// freed (after the caller synchronised) when the call returns.
struct Scratch {
  std::vector<void*> ptrs;
  cudaStream_t st = nullptr;
  ~Scratch() {
    for (void* q : ptrs) cudaFree(q);
    if (st) cudaStreamDestroy(st);
  }
  template <typename T>
  T* dev(size_t n, const T* host = nullptr) {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(1, n) * sizeof(T)) != cudaSuccess) return nullptr;
    ptrs.push_back(q);
    if (host && n) cudaMemcpyAsync(q, host, n * sizeof(T), cudaMemcpyHostToDevice, st);
    return (T*)q;
  }
  int init() {
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    return MPPI_OK;
  }
};

}  // namespace mppi

#define SCRATCH_OR_FAIL(S) \
  ::mppi::Scratch S;       \
  CKR(S.init())
#define DEVPTR(S, T, name, n, host)                \
  T* name = S.dev<T>((n), (host));                 \
  if (!name) return ::mppi::fail(MPPI_E_CUDA, "cudaMalloc failed (" #name ")")
