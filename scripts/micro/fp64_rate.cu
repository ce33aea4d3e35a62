// FP64 FMA throughput and latency per SM on the B200 (sm_100a):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/fp64_rate scripts/micro/fp64_rate.cu
#include <cstdio>
template <int CH>
__global__ void dfma(int iters, double* out, long long* cyc) {
  double a[CH];
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double m = 0.999999, c = 1e-7;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = fma(a[i], m, c);
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 8);
  const int iters = 4096;
  for (int threads : {32, 128, 256, 512, 1024}) {
    dfma<1><<<148, threads>>>(iters, o, c);
    dfma<1><<<148, threads>>>(iters, o, c);
    long long h;
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("1 chain  %4d threads/SM: %.1f DFMA/clk/SM, %.1f clk per dependent DFMA\n", threads,
           (double)threads * iters / h, (double)h / iters);
    dfma<8><<<148, threads>>>(iters, o, c);
    dfma<8><<<148, threads>>>(iters, o, c);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("8 chains %4d threads/SM: %.1f DFMA/clk/SM\n", threads, (double)threads * iters * 8 / h);
  }
  return 0;
}
