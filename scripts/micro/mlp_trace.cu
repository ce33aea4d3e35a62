// Per-tile event timeline of the MLP kernel (CTA 0) at a config-4-sized batch:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -DMPPI_MLP_TRACE -Iinclude -o scripts/micro/mlp_trace scripts/micro/mlp_trace.cu
//   ./scripts/micro/mlp_trace [tiles_per_cta]
// Prints the kernel time per tile and, for tiles 4..11 of CTA 0, the clock of
// each event relative to the tile's layer-2-done (epilogue view).
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../paper_2104_13542_b200/csrc/mppi_mlp.cuh"

using namespace mppi;

int main(int argc, char** argv) {
  const int tpc = argc > 1 ? atoi(argv[1]) : 24;
  const long long rows = 148LL * 128 * tpc;
  std::mt19937_64 g(0);
  std::normal_distribution<double> nd(0.0, 1.0);
  auto he = [&](int in, int out) {
    std::vector<double> w((size_t)in * out);
    for (auto& v : w) v = nd(g) * std::sqrt(2.0 / in);
    return w;
  };
  auto W0 = he(14, 256), W1 = he(256, 128), W2 = he(128, 64), W3 = he(64, 1);
  std::vector<double> b0(256, 0.01), b1(128, 0.01), b2(64, 0.01), b3(1, 0.0);
  MlpWeights m;
  if (mlp_upload(m, 14, W0.data(), b0.data(), W1.data(), b1.data(), W2.data(), b2.data(), W3.data(), b3.data(),
                 0) != cudaSuccess) {
    printf("upload failed\n");
    return 1;
  }
  std::vector<float> hx((size_t)rows * 8);
  std::uniform_real_distribution<float> ud(-2.5f, 2.5f);
  for (long long r = 0; r < rows; ++r)
    for (int j = 0; j < 8; ++j) hx[r * 8 + j] = j < 7 ? ud(g) : 0.f;
  float *x, *out;
  cudaMalloc(&x, hx.size() * 4);
  cudaMalloc(&out, rows * 4);
  cudaMemcpy(x, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) mlp_forward(m, x, rows, out, 0, 1);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) mlp_forward(m, x, rows, out, 0, 1);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return 1;
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("rows %lld (%d tiles per CTA): %.3f ms, %.1f ns per tile per SM, %.2f Mrows/ms\n", rows, tpc, ms,
         ms * 1e6 / tpc, rows / ms / 1e6);
  long long tr[32 * 32];
  cudaMemcpyFromSymbol(tr, mlp_trace, sizeof(tr));
  const char* names[32] = {"E L2done",   "E L2epi end", "E L1epi(t) start", "E L1epi(t) end", "E L3done",
                           "E out end",  "I L3done(k-1)", "",                 "I A1[0]",        "I A1[last]",
                           "I L2 issued", "I L2done",   "I A2[0]",          "I A2[last]",        "I L3 issued",
                           "",           "I X ready",   "I L1 issued",      "",               "",
                           "E A2[0] arr", "E A2[1] arr", "E A2[2] arr",     "E A2[3] arr",    "E A1[0] arr",
                           "E A1[1] arr", "E A1[2] arr", "E A1[3] arr",     "E A1[4] arr",    "E A1[5] arr",
                           "E A1[6] arr", "E A1[7] arr"};
  printf("%-18s", "event \\ tile");
  for (int k = 4; k < 12 && k < tpc; ++k) printf("%8d", k);
  printf("\n");
  for (int e = 0; e < 32; ++e) {
    if (!names[e][0]) continue;
    printf("%-18s", names[e]);
    for (int k = 4; k < 12 && k < tpc; ++k) printf("%8lld", tr[k * 32 + e] - tr[k * 32 + 0]);
    printf("\n");
  }
  printf("period (E L2done k -> k+1):");
  for (int k = 4; k < 12 && k + 1 < tpc; ++k) printf(" %lld", tr[(k + 1) * 32] - tr[k * 32]);
  printf("\n");
  return 0;
}
