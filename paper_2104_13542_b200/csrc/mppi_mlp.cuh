// mppi_mlp.cuh — learned self-collision distance (surrogate.py:42-52):
// x = [sin q, cos q] (14) -> 256 -> 128 -> 64 -> 1, ReLU between layers.
//
// This first version is a CUDA-core FP32 kernel (one thread per row, weights
// broadcast from L1/L2). It is the correctness baseline the tcgen05 kernel is
// developed against.
#pragma once

#include <cuda_runtime.h>

#include <vector>

namespace mppi {

constexpr int kMlpH0 = 256, kMlpH1 = 128, kMlpH2 = 64, kMlpIn = 16;

struct MlpWeights {
  int in_dim = 0;
  float* w = nullptr;  // packed fp32: W0 (16x256, rows >= in_dim zero) | b0 | W1 | b1 | W2 | b2 | W3 | b3
};

inline size_t mlp_padded_rows(size_t rows) { return (rows + 127) / 128 * 128; }

constexpr size_t kOffW0 = 0;
constexpr size_t kOffB0 = kOffW0 + kMlpIn * kMlpH0;
constexpr size_t kOffW1 = kOffB0 + kMlpH0;
constexpr size_t kOffB1 = kOffW1 + kMlpH0 * kMlpH1;
constexpr size_t kOffW2 = kOffB1 + kMlpH1;
constexpr size_t kOffB2 = kOffW2 + kMlpH1 * kMlpH2;
constexpr size_t kOffW3 = kOffB2 + kMlpH2;
constexpr size_t kOffB3 = kOffW3 + kMlpH2;
constexpr size_t kMlpParams = kOffB3 + 1;

__global__ void __launch_bounds__(128) mlp_simt_kernel(const float* __restrict__ x, long long rows,
                                                       const float* __restrict__ w,
                                                       float* __restrict__ out) {
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  float in[kMlpIn];
#pragma unroll
  for (int k = 0; k < kMlpIn; ++k) in[k] = x[r * kMlpIn + k];
  float h2[kMlpH1];
#pragma unroll
  for (int j = 0; j < kMlpH1; ++j) h2[j] = w[kOffB1 + j];
  for (int i = 0; i < kMlpH0; ++i) {
    float a = w[kOffB0 + i];
#pragma unroll
    for (int k = 0; k < kMlpIn; ++k) a += in[k] * w[kOffW0 + k * kMlpH0 + i];
    a = a > 0.f ? a : 0.f;
#pragma unroll
    for (int j = 0; j < kMlpH1; ++j) h2[j] += a * w[kOffW1 + i * kMlpH1 + j];
  }
  float h3[kMlpH2];
#pragma unroll
  for (int j = 0; j < kMlpH2; ++j) h3[j] = w[kOffB2 + j];
#pragma unroll
  for (int i = 0; i < kMlpH1; ++i) {
    const float a = h2[i] > 0.f ? h2[i] : 0.f;
#pragma unroll
    for (int j = 0; j < kMlpH2; ++j) h3[j] += a * w[kOffW2 + i * kMlpH2 + j];
  }
  float o = w[kOffB3];
#pragma unroll
  for (int i = 0; i < kMlpH2; ++i) o += (h3[i] > 0.f ? h3[i] : 0.f) * w[kOffW3 + i];
  out[r] = o;
}

inline cudaError_t mlp_upload(MlpWeights& m, int in_dim, const double* W0, const double* b0,
                              const double* W1, const double* b1, const double* W2,
                              const double* b2, const double* W3, const double* b3,
                              cudaStream_t st) {
  std::vector<float> h(kMlpParams, 0.f);
  for (int k = 0; k < in_dim; ++k)
    for (int i = 0; i < kMlpH0; ++i) h[kOffW0 + k * kMlpH0 + i] = (float)W0[k * kMlpH0 + i];
  for (int i = 0; i < kMlpH0; ++i) h[kOffB0 + i] = (float)b0[i];
  for (int i = 0; i < kMlpH0 * kMlpH1; ++i) h[kOffW1 + i] = (float)W1[i];
  for (int i = 0; i < kMlpH1; ++i) h[kOffB1 + i] = (float)b1[i];
  for (int i = 0; i < kMlpH1 * kMlpH2; ++i) h[kOffW2 + i] = (float)W2[i];
  for (int i = 0; i < kMlpH2; ++i) h[kOffB2 + i] = (float)b2[i];
  for (int i = 0; i < kMlpH2; ++i) h[kOffW3 + i] = (float)W3[i];
  h[kOffB3] = (float)b3[0];
  cudaError_t e = cudaSuccess;
  if (!m.w) e = cudaMalloc(&m.w, kMlpParams * sizeof(float));
  if (e != cudaSuccess) return e;
  m.in_dim = in_dim;
  e = cudaMemcpyAsync(m.w, h.data(), kMlpParams * sizeof(float), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(st);
}

inline cudaError_t mlp_forward(const MlpWeights& m, const float* x, long long rows, float* out,
                               cudaStream_t st) {
  const long long blocks = (rows + 127) / 128;
  mlp_simt_kernel<<<(unsigned)blocks, 128, 0, st>>>(x, rows, m.w, out);
  return cudaGetLastError();
}

inline void mlp_release(MlpWeights& m) {
  if (m.w) cudaFree(m.w);
  m.w = nullptr;
}

}  // namespace mppi
