// Cold-load latency after an L2 flush: K dependent loads spread over K
// different 2 MB pages vs K loads inside one 2 MB page (each line distinct).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/tlb_cold scripts/micro/tlb_cold.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chase(const long long* __restrict__ base, const long long* offs, int k, long long* out) {
  long long idx = 0, t0 = clock64();
  for (int i = 0; i < k; ++i) idx = base[offs[i] + (idx & 1)];  // dependent chain
  out[0] = (clock64() - t0) / k;
  out[1] = idx;
}

int main() {
  const size_t span = 512ull << 20;  // 512 MB arena
  long long *base, *offs, *out;
  cudaMalloc(&base, span);
  cudaMemset(base, 0, span);
  cudaMalloc(&offs, 64 * sizeof(long long));
  cudaMalloc(&out, 16);
  char* flush;
  cudaMalloc(&flush, 256ull << 20);
  long long h[64];
  const int k = 32;
  for (int mode = 0; mode < 3; ++mode) {
    for (int i = 0; i < k; ++i) {
      if (mode == 0) h[i] = (long long)i * (2ll << 20) / 8;          // one line in each of 32 pages (2 MB apart)
      else if (mode == 1) h[i] = (long long)i * 4096 / 8;            // 32 lines, one 128 KB window of one page
      else h[i] = (long long)i * (16ll << 20) / 8;                   // 16 MB apart
    }
    cudaMemcpy(offs, h, k * sizeof(long long), cudaMemcpyHostToDevice);
    double acc = 0;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(flush, rep, 256ull << 20);
      chase<<<1, 1>>>(base, offs, k, out);
      long long r[2];
      cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
      if (rep) acc += r[0];
    }
    const char* names[] = {"32 pages, 2 MB apart", "one page, 4 KB apart", "32 pages, 16 MB apart"};
    printf("%-24s: %.0f cycles per cold dependent load (L2 flushed)\n", names[mode], acc / 4);
  }
  // warm reference
  chase<<<1, 1>>>(base, offs, k, out);
  long long r[2];
  cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
  printf("%-24s: %lld cycles per warm dependent load\n", "warm (last layout)", r[0]);
  return 0;
}
