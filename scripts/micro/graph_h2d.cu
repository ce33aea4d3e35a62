// Microbenchmark: cost of getting a 120-byte state block to the device inside
// a CUDA graph: memcpy node from pinned memory vs a kernel reading mapped
// memory, each followed by a dependent kernel. Graph launched + synchronised
// per step (the control-step pattern).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 graph_h2d.cu -o graph_h2d
#include <cstdio>
#include <vector>
#include <algorithm>
#include <chrono>
#include <cuda_runtime.h>

__global__ void consume(const double* s, double* out) {
  if (threadIdx.x < 15) out[threadIdx.x] = s[threadIdx.x] * 2.0;
}
__global__ void fetch(const double* mapped, double* dev) {
  if (threadIdx.x < 15) dev[threadIdx.x] = mapped[threadIdx.x];
}
__global__ void consume_mapped(const double* mapped, double* out) {
  __shared__ double s[16];
  if (threadIdx.x < 15) s[threadIdx.x] = mapped[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < 15) out[threadIdx.x] = s[threadIdx.x] * 2.0;
}

int main() {
  cudaSetDeviceFlags(cudaDeviceMapHost);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  double *h, *hm, *d, *o;
  cudaHostAlloc(&h, 128, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&hm, h, 0);
  cudaMalloc(&d, 128);
  cudaMalloc(&o, 128);
  for (int i = 0; i < 16; ++i) h[i] = i;
  auto capture = [&](int mode) {
    cudaGraph_t g;
    cudaGraphExec_t e;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (mode == 0) {
      cudaMemcpyAsync(d, h, 120, cudaMemcpyHostToDevice, st);
      consume<<<1, 32, 0, st>>>(d, o);
    } else if (mode == 1) {
      consume<<<1, 32, 0, st>>>(d, o);
    } else if (mode == 2) {
      fetch<<<1, 32, 0, st>>>(hm, d);
      consume<<<1, 32, 0, st>>>(d, o);
    } else if (mode == 3) {
      consume_mapped<<<125, 128, 0, st>>>(hm, o);
    } else {
      consume<<<1, 32, 0, st>>>(d, o);
      consume<<<1, 32, 0, st>>>(d, o);
      consume<<<1, 32, 0, st>>>(d, o);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&e, g, 0);
    return e;
  };
  const char* names[] = {"memcpy node + kernel", "kernel only", "fetch kernel + kernel",
                         "125 CTAs read mapped", "3 dependent kernels"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 5; ++mode) {
    cudaGraphExec_t g = capture(mode);
    std::vector<float> dev;
    std::vector<double> wall;
    for (int i = 0; i < 2000; ++i) {
      auto t0 = std::chrono::high_resolution_clock::now();
      cudaEventRecord(e0, st);
      cudaGraphLaunch(g, st);
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      auto t1 = std::chrono::high_resolution_clock::now();
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 100) {
        dev.push_back(ms * 1e3f);
        wall.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
      }
    }
    std::sort(dev.begin(), dev.end());
    std::sort(wall.begin(), wall.end());
    printf("%-26s device %.2f us  wall %.2f us (medians)\n", names[mode], dev[dev.size() / 2],
           wall[wall.size() / 2]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
