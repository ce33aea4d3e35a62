// Microbenchmark: host wait for a tiny stream step's result —
// cudaStreamSynchronize vs spinning on a flag the last kernel writes to mapped
// pinned memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 graph_poll.cu -o graph_poll
#include <cstdio>
#include <vector>
#include <algorithm>
#include <chrono>
#include <cuda_runtime.h>

__global__ void work(const double* s, double* out, volatile unsigned* flag, unsigned seq) {
  if (threadIdx.x < 15) out[threadIdx.x] = s[threadIdx.x] * 2.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *flag = seq;
  }
}

int main() {
  cudaSetDeviceFlags(cudaDeviceMapHost | cudaDeviceScheduleSpin);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  double *h, *d, *ho, *hom;
  unsigned *flag, *flagm;
  cudaHostAlloc(&h, 128, cudaHostAllocMapped);
  cudaHostAlloc(&ho, 128, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&hom, ho, 0);
  cudaHostAlloc(&flag, 64, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&flagm, flag, 0);
  cudaMalloc(&d, 128);
  *flag = 0;
  for (int variant = 0; variant < 2; ++variant) {
    std::vector<double> wall;
    for (int i = 1; i <= 3000; ++i) {
      auto t0 = std::chrono::high_resolution_clock::now();
      cudaMemcpyAsync(d, h, 120, cudaMemcpyHostToDevice, st);
      const unsigned want = (unsigned)i + variant * 100000u;
      work<<<1, 32, 0, st>>>(d, hom, flagm, want);
      if (variant == 0) {
        cudaStreamSynchronize(st);
      } else {
        while (*(volatile unsigned*)flag != want) {
        }
      }
      auto t1 = std::chrono::high_resolution_clock::now();
      if (i > 200) wall.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    cudaStreamSynchronize(st);
    std::sort(wall.begin(), wall.end());
    printf("%-28s wall median %.2f us  p90 %.2f us\n", variant ? "spin on mapped flag" : "cudaStreamSynchronize",
           wall[wall.size() / 2], wall[wall.size() * 9 / 10]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
