// mppi_train.cu — surrogate training on the device.
//
// train_collision_surrogate (surrogate.py:146-206): the 2d -> 256 -> 128 -> 64
// -> 1 ReLU MLP fitted to oracle distances by mini-batch MSE + Adam (beta1 0.9,
// beta2 0.999, eps 1e-8; surrogate.py:83-101), step size halved at epochs 50
// and 75, then the holdout MAE and sign agreement. Everything the reference
// computes in float64 is computed here in float64 (B200 FP64 pipe); the data,
// the He initialisation and the per-epoch permutations come from the caller
// (the reference's own numpy generator draws them, so the training inputs are
// the reference's bit for bit).
//
// One optimisation step = one replay of a CUDA graph of small kernels:
//   forward  L0..L3 (gather the batch rows by the permutation, bias, ReLU)
//   loss     err = out - y, loss = mean(err^2), dout = 2 err / B
//   backward per layer: dW = a_in^T delta, db = sum delta, delta_prev = (delta W^T) * (a_in > 0)
//   (every product through one shared-memory tiled float64 GEMM kernel)
//   adam     every parameter, bias corrections from the device step counter
// The step counter, the batch offset and the learning rate live in device
// memory, so the same graph replays for every step of every epoch.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mppi_b200.h"

namespace {

constexpr int kLayers = 4;
constexpr int kHidden[3] = {256, 128, 64};
constexpr int kMaxBatch = 1024;

struct TrainState {      // device
  long long step;        // Adam t (1-based after the increment)
  long long batch;       // batch index within the epoch
  int epoch;
  int diverged;          // first non-finite loss seen
  double last_finite;    // last finite loss
};

struct Net {             // device pointers, W_i (in, out) row-major as the reference stores them
  double* W[kLayers];
  double* b[kLayers];
  double* mW[kLayers];
  double* vW[kLayers];
  double* mb[kLayers];
  double* vb[kLayers];
  double* gW[kLayers];
  double* gb[kLayers];
  int dims[kLayers + 1];
};

struct Batch {
  const double* x;          // (n, in) train encodings
  const double* y;          // (n)
  const long long* order;   // (epochs, n) permutation per epoch
  int n, in_dim, bs, batches, epochs;
  const double* lr;         // (epochs) step size per epoch
  double* act[kLayers + 1]; // act[0] = gathered input (bs, in); act[i] = post-ReLU (bs, dims[i]); act[4] = out
  double* delta[kLayers];   // delta[i] (bs, dims[i+1])
  double* err;              // (bs)
  double* losses;           // (epochs * batches)
  TrainState* st;
};

__device__ __forceinline__ int cur_rows(const Batch& B) {
  const long long lo = B.st->batch * (long long)B.bs;
  const long long hi = lo + B.bs < B.n ? lo + B.bs : B.n;
  return (int)(hi - lo);
}

// act[0] = x[order[epoch][batch*bs + r]]
__global__ void gather_kernel(Batch B) {
  const int rows = cur_rows(B);
  const long long base = (long long)B.st->epoch * B.n + B.st->batch * (long long)B.bs;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < rows * B.in_dim; t += gridDim.x * blockDim.x) {
    const int r = t / B.in_dim, i = t - r * B.in_dim;
    const long long src = B.order[base + r];
    B.act[0][(size_t)r * B.in_dim + i] = B.x[(size_t)src * B.in_dim + i];
  }
}

// ---- shared-memory tiled float64 products ---------------------------------
// C (M, N) = sum_p X(m, p) Y(p, n), X(m, p) = X[m * xm + p * xp], Y(p, n) =
// Y[p * yp + n * yn]; 32 x 32 output tile per 256-thread block (each thread 4
// rows of one column), K tiles of 32 staged in shared memory. Epilogues:
//   EPI_FWD   C = relu?(acc + bias[n])            forward layer
//   EPI_PLAIN C = acc                             weight gradient a_in^T delta
//   EPI_MASK  C = mask(m, n) > 0 ? acc : 0        delta_prev = (delta W^T) * (a_in > 0)
enum { EPI_FWD = 0, EPI_PLAIN = 1, EPI_MASK = 2 };
constexpr int kT = 32;

struct Gemm {
  const double* X;
  long long xm, xp;
  const double* Y;
  long long yp, yn;
  double* C;      // (M, N) row-major
  int M, N, K;    // M or K = -1: the current batch's row count
  int epi, relu;
  const double* bias;
  const double* mask;  // (M, N) row-major
  // weight gradients: blockIdx.z takes K rows [32z, 32z + 32) and writes its
  // partial product to C + z * split_stride (the Adam kernel sums the splits
  // in order); row `ones_row` of X is all ones, so that row of C is the bias
  // gradient (column sums of delta)
  long long split_stride;
  int ones_row;
};

__global__ void __launch_bounds__(256) gemm_kernel(Batch B, Gemm g) {
  __shared__ double xs[kT][kT + 1];
  __shared__ double ys[kT][kT + 1];
  const int rows = cur_rows(B);
  const int M = g.M < 0 ? rows : g.M, K = g.K < 0 ? rows : g.K, N = g.N;
  const int m0 = blockIdx.y * kT, n0 = blockIdx.x * kT;
  if (m0 >= M) return;
  const bool split = g.split_stride != 0;
  const int pbeg = split ? blockIdx.z * kT : 0, pend = split ? min(K, pbeg + kT) : K;
  if (pbeg >= pend && split) return;  // past this batch's rows: the Adam kernel does not read it
  double* C = g.C + (split ? blockIdx.z * g.split_stride : 0);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int p0 = pbeg; p0 < pend; p0 += kT) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = ty + 8 * u;  // tile row
      const int m = m0 + r, pp = p0 + tx;
      xs[r][tx] = (m < M && pp < pend) ? (m == g.ones_row ? 1.0 : g.X[(long long)m * g.xm + (long long)pp * g.xp])
                                       : 0.0;
      const int pq = p0 + r, n = n0 + tx;
      ys[r][tx] = (pq < pend && n < N) ? g.Y[(long long)pq * g.yp + (long long)n * g.yn] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int q = 0; q < kT; ++q) {
      const double yv = ys[q][tx];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fma(xs[ty + 8 * u][q], yv, acc[u]);
    }
    __syncthreads();
  }
  const int n = n0 + tx;
  if (n >= N) return;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int m = m0 + ty + 8 * u;
    if (m >= M) continue;
    double v = acc[u];
    if (g.epi == EPI_FWD) {
      v += g.bias[n];
      if (g.relu) v = fmax(v, 0.0);
    } else if (g.epi == EPI_MASK) {
      v = g.mask[(long long)m * N + n] > 0.0 ? v : 0.0;
    }
    C[(long long)m * N + n] = v;
  }
}

// err = out - y; loss = mean(err^2); delta3 = 2 err / rows (one block)
__global__ void loss_kernel(Batch B, double* __restrict__ dlast) {
  __shared__ double red[32];
  const int rows = cur_rows(B);
  const long long base = (long long)B.st->epoch * B.n + B.st->batch * (long long)B.bs;
  double s = 0.0;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) {
    const double e = B.act[kLayers][r] - B.y[B.order[base + r]];
    B.err[r] = e;
    dlast[r] = (2.0 / rows) * e;
    s += e * e;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    const double loss = tot / rows;
    B.losses[B.st->epoch * (long long)B.batches + B.st->batch] = loss;
    if (isfinite(loss)) {
      if (!B.st->diverged) B.st->last_finite = loss;
    } else if (!B.st->diverged) {
      B.st->diverged = 1 + B.st->epoch;  // epoch + 1 of the first non-finite loss
    }
  }
}

struct AdamSeg {
  double* p[2 * kLayers];
  const double* g[2 * kLayers];   // split 0 of the gradient; split s at g + s * gs
  long long gs[2 * kLayers];
  double* m[2 * kLayers];
  double* v[2 * kLayers];
  int n[2 * kLayers];
  int off[2 * kLayers + 1];
};

// Adam.step (surrogate.py:88-101) over every parameter, with numpy's operation
// order and no contraction (m *= b1; m += (1-b1) g; v *= b2; v += (1-b2) g g;
// p -= lr (m / b1c) / (sqrt(v / b2c) + eps)); the bias corrections
// 1 - beta^t come from the host (Python's float power).
__global__ void adam_kernel(Batch B, AdamSeg s, const double* __restrict__ bc1, const double* __restrict__ bc2) {
  const long long t = B.st->step;  // 0-based step index
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  const double b1c = bc1[t], b2c = bc2[t];
  const double lr = B.lr[B.st->epoch];
  const int total = s.off[2 * kLayers];
  const int nsplit = (cur_rows(B) + kT - 1) / kT;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < total; q += gridDim.x * blockDim.x) {
    int seg = 0;
    while (q >= s.off[seg + 1]) ++seg;
    const int i = q - s.off[seg];
    double g = 0.0;  // the weight-gradient GEMM's K splits, summed in order
    for (int z = 0; z < nsplit; ++z) g += s.g[seg][(long long)z * s.gs[seg] + i];
    double m = s.m[seg][i], v = s.v[seg][i];
    m = __dadd_rn(__dmul_rn(m, b1), __dmul_rn(1.0 - b1, g));
    v = __dadd_rn(__dmul_rn(v, b2), __dmul_rn(__dmul_rn(1.0 - b2, g), g));
    s.m[seg][i] = m;
    s.v[seg][i] = v;
    s.p[seg][i] = __dsub_rn(s.p[seg][i], __dmul_rn(lr, m / b1c) / __dadd_rn(sqrt(v / b2c), eps));
  }
}

__global__ void advance_kernel(Batch B) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    B.st->step += 1;
    if (++B.st->batch == B.batches) {
      B.st->batch = 0;
      B.st->epoch += 1;
    }
  }
}

// holdout: pred = net(x_hold); mae, sign agreement (surrogate.py:200-203)
__global__ void holdout_kernel(const Net net, const double* __restrict__ x, const double* __restrict__ y, int n,
                               int in_dim, double* __restrict__ abs_err, int* __restrict__ agree) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double h0[256], h1[128], h2[64];
    for (int j = 0; j < 256; ++j) {
      double a = 0.0;
      for (int k = 0; k < in_dim; ++k) a = fma(x[(size_t)r * in_dim + k], net.W[0][(size_t)k * 256 + j], a);
      h0[j] = fmax(a + net.b[0][j], 0.0);
    }
    for (int j = 0; j < 128; ++j) {
      double a = 0.0;
      for (int k = 0; k < 256; ++k) a = fma(h0[k], net.W[1][(size_t)k * 128 + j], a);
      h1[j] = fmax(a + net.b[1][j], 0.0);
    }
    for (int j = 0; j < 64; ++j) {
      double a = 0.0;
      for (int k = 0; k < 128; ++k) a = fma(h1[k], net.W[2][(size_t)k * 64 + j], a);
      h2[j] = fmax(a + net.b[2][j], 0.0);
    }
    double o = 0.0;
    for (int k = 0; k < 64; ++k) o = fma(h2[k], net.W[3][k], o);
    o += net.b[3][0];
    abs_err[r] = fabs(o - y[r]);
    agree[r] = (o > 0.0) == (y[r] > 0.0);
  }
}

}  // namespace

extern "C" int mppi_internal_fail(int code, const char* msg);  // mppi_abi.cu: sets mppi_last_error

namespace {

int fail(int code, const std::string& msg) { return mppi_internal_fail(code, msg.c_str()); }

#define TCK(x)                                                                                   \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return fail(MPPI_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct Arena {
  std::vector<void*> ptrs;
  ~Arena() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

unsigned blocks_for(long long n, int t = 256) {
  long long b = (n + t - 1) / t;
  return (unsigned)(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

}  // namespace

extern "C" {

int mppi_train_mlp(const mppi_train_desc* d, double* const* weights, double* const* biases, mppi_train_result* res) {
  if (!d || !weights || !biases || !res) return fail(MPPI_E_BAD_ARGUMENT, "null argument");
  if (d->in_dim < 1 || d->in_dim > 64) return fail(MPPI_E_BAD_ARGUMENT, "input width out of range");
  if (d->n_train < 1 || d->batch_size < 1 || d->batch_size > kMaxBatch || d->epochs < 0)
    return fail(MPPI_E_BAD_ARGUMENT, "bad training sizes");
  if (!d->x_train || !d->y_train || !d->order || !d->lr || (d->n_hold > 0 && (!d->x_hold || !d->y_hold)))
    return fail(MPPI_E_BAD_ARGUMENT, "null training array");
  for (int l = 0; l < kLayers; ++l)
    if (!weights[l] || !biases[l]) return fail(MPPI_E_BAD_ARGUMENT, "null weight array");
  cudaStream_t st;
  TCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  Arena A;
  const int in = d->in_dim, n = d->n_train, bs = d->batch_size, E = d->epochs;
  const int batches = (n + bs - 1) / bs;
  const int dims[kLayers + 1] = {in, kHidden[0], kHidden[1], kHidden[2], 1};
  Net net{};
  for (int l = 0; l <= kLayers; ++l) net.dims[l] = dims[l];
  AdamSeg seg{};
  int off = 0;
  for (int l = 0; l < kLayers; ++l) {
    const size_t nw = (size_t)dims[l] * dims[l + 1], nb = dims[l + 1];
    net.W[l] = A.alloc<double>(nw);
    net.b[l] = A.alloc<double>(nb);
    net.mW[l] = A.alloc<double>(nw);
    net.vW[l] = A.alloc<double>(nw);
    net.mb[l] = A.alloc<double>(nb);
    net.vb[l] = A.alloc<double>(nb);
    // weight + bias gradient partials: one (dims[l] + 1, dims[l+1]) slab per K split
    net.gW[l] = A.alloc<double>((size_t)((bs + kT - 1) / kT) * (nw + nb));
    net.gb[l] = net.gW[l] ? net.gW[l] + nw : nullptr;
    if (!net.W[l] || !net.b[l] || !net.mW[l] || !net.vW[l] || !net.mb[l] || !net.vb[l] || !net.gW[l] || !net.gb[l])
      return fail(MPPI_E_CUDA, "out of device memory");
    TCK(cudaMemcpyAsync(net.W[l], weights[l], nw * sizeof(double), cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(net.b[l], biases[l], nb * sizeof(double), cudaMemcpyHostToDevice, st));
    for (double* z : {net.mW[l], net.vW[l]}) TCK(cudaMemsetAsync(z, 0, nw * sizeof(double), st));
    for (double* z : {net.mb[l], net.vb[l]}) TCK(cudaMemsetAsync(z, 0, nb * sizeof(double), st));
    // Adam's parameter order: all weights, then all biases (surrogate.py:178-179, 197)
    seg.p[l] = net.W[l], seg.g[l] = net.gW[l], seg.m[l] = net.mW[l], seg.v[l] = net.vW[l], seg.n[l] = (int)nw;
    seg.p[kLayers + l] = net.b[l], seg.g[kLayers + l] = net.gb[l], seg.m[kLayers + l] = net.mb[l],
    seg.v[kLayers + l] = net.vb[l], seg.n[kLayers + l] = (int)nb;
    seg.gs[l] = seg.gs[kLayers + l] = (long long)(nw + nb);
  }
  for (int q = 0; q < 2 * kLayers; ++q) {
    seg.off[q] = off;
    off += seg.n[q];
  }
  seg.off[2 * kLayers] = off;
  Batch B{};
  B.n = n, B.in_dim = in, B.bs = bs, B.batches = batches, B.epochs = E;
  double* x = A.alloc<double>((size_t)n * in);
  double* y = A.alloc<double>(n);
  long long* order = A.alloc<long long>((size_t)std::max(E, 1) * n);
  double* lr = A.alloc<double>(std::max(E, 1));
  const long long nsteps = (long long)E * batches;
  double* bc = A.alloc<double>((size_t)2 * std::max(nsteps, 1LL));
  double* losses = A.alloc<double>((size_t)std::max(E, 1) * batches);
  TrainState* ts = A.alloc<TrainState>(1);
  if (!x || !y || !order || !lr || !losses || !ts || !bc) return fail(MPPI_E_CUDA, "out of device memory");
  if (nsteps > 0) {
    if (!d->bias_corr1 || !d->bias_corr2) return fail(MPPI_E_BAD_ARGUMENT, "bias corrections missing");
    TCK(cudaMemcpyAsync(bc, d->bias_corr1, sizeof(double) * nsteps, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(bc + nsteps, d->bias_corr2, sizeof(double) * nsteps, cudaMemcpyHostToDevice, st));
  }
  TCK(cudaMemcpyAsync(x, d->x_train, sizeof(double) * n * in, cudaMemcpyHostToDevice, st));
  TCK(cudaMemcpyAsync(y, d->y_train, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  if (E > 0) {
    TCK(cudaMemcpyAsync(order, d->order, sizeof(long long) * E * n, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(lr, d->lr, sizeof(double) * E, cudaMemcpyHostToDevice, st));
  }
  TrainState h0{};
  TCK(cudaMemcpyAsync(ts, &h0, sizeof(h0), cudaMemcpyHostToDevice, st));
  B.x = x, B.y = y, B.order = order, B.lr = lr, B.losses = losses, B.st = ts;
  for (int l = 0; l <= kLayers; ++l) {
    B.act[l] = A.alloc<double>((size_t)bs * dims[l]);
    if (!B.act[l]) return fail(MPPI_E_CUDA, "out of device memory");
  }
  for (int l = 0; l < kLayers; ++l) {
    B.delta[l] = A.alloc<double>((size_t)bs * dims[l + 1]);
    if (!B.delta[l]) return fail(MPPI_E_CUDA, "out of device memory");
  }
  B.err = A.alloc<double>(bs);
  if (!B.err) return fail(MPPI_E_CUDA, "out of device memory");

  float ms = 0.f;
  if (E > 0) {
    // ---- one optimisation step as a graph
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    TCK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    gather_kernel<<<blocks_for((long long)bs * in), 256, 0, st>>>(B);
    auto gemm = [&](const Gemm& gm) {
      const int mt = (gm.M < 0 ? bs : gm.M);
      const int splits = gm.split_stride ? (bs + kT - 1) / kT : 1;
      gemm_kernel<<<dim3((gm.N + kT - 1) / kT, (mt + kT - 1) / kT, splits), 256, 0, st>>>(B, gm);
    };
    for (int l = 0; l < kLayers; ++l) {  // act[l+1] = relu?(act[l] @ W[l] + b[l])
      Gemm gm{};
      gm.ones_row = -1;
      gm.X = B.act[l], gm.xm = dims[l], gm.xp = 1;
      gm.Y = net.W[l], gm.yp = dims[l + 1], gm.yn = 1;
      gm.C = B.act[l + 1], gm.M = -1, gm.N = dims[l + 1], gm.K = dims[l];
      gm.epi = EPI_FWD, gm.relu = l < kLayers - 1, gm.bias = net.b[l];
      gemm(gm);
    }
    loss_kernel<<<1, 256, 0, st>>>(B, B.delta[kLayers - 1]);
    for (int l = kLayers - 1; l >= 0; --l) {
      Gemm gw{};  // [gW[l]; gb[l]] (dims[l] + 1, dims[l+1]) = [act[l] | 1]^T delta[l], per K split
      gw.X = B.act[l], gw.xm = 1, gw.xp = dims[l];
      gw.Y = B.delta[l], gw.yp = dims[l + 1], gw.yn = 1;
      gw.C = net.gW[l], gw.M = dims[l] + 1, gw.N = dims[l + 1], gw.K = -1, gw.epi = EPI_PLAIN;
      gw.ones_row = dims[l];
      gw.split_stride = (long long)(dims[l] + 1) * dims[l + 1];
      gemm(gw);
      if (l > 0) {  // delta[l-1] (rows, dims[l]) = (delta[l] W[l]^T) * (act[l] > 0)
        Gemm gb{};
        gb.ones_row = -1;
        gb.X = B.delta[l], gb.xm = dims[l + 1], gb.xp = 1;
        gb.Y = net.W[l], gb.yp = 1, gb.yn = dims[l + 1];
        gb.C = B.delta[l - 1], gb.M = -1, gb.N = dims[l], gb.K = dims[l + 1];
        gb.epi = EPI_MASK, gb.mask = B.act[l];
        gemm(gb);
      }
    }
    adam_kernel<<<blocks_for(off), 256, 0, st>>>(B, seg, bc, bc + nsteps);
    advance_kernel<<<1, 32, 0, st>>>(B);
    cudaError_t ce = cudaStreamEndCapture(st, &g);
    if (ce != cudaSuccess) return fail(MPPI_E_CUDA, std::string("train capture: ") + cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(MPPI_E_CUDA, std::string("train instantiate: ") + cudaGetErrorString(ce));
    struct ExecGuard {
      cudaGraphExec_t e;
      ~ExecGuard() { cudaGraphExecDestroy(e); }
    } eg{ge};
    cudaEvent_t e0, e1;
    TCK(cudaEventCreate(&e0));
    TCK(cudaEventCreate(&e1));
    TCK(cudaEventRecord(e0, st));
    const long long steps = (long long)E * batches;
    for (long long s = 0; s < steps; ++s) TCK(cudaGraphLaunch(ge, st));
    TCK(cudaEventRecord(e1, st));
    TCK(cudaStreamSynchronize(st));
    TCK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  TrainState hs{};
  TCK(cudaMemcpy(&hs, ts, sizeof(hs), cudaMemcpyDeviceToHost));
  res->steps = hs.step;
  res->device_ms = ms;
  res->last_finite_loss = E > 0 ? hs.last_finite : NAN;
  res->diverged_epoch = hs.diverged - 1;  // -1: every loss finite
  for (int l = 0; l < kLayers; ++l) {
    TCK(cudaMemcpy(weights[l], net.W[l], sizeof(double) * dims[l] * dims[l + 1], cudaMemcpyDeviceToHost));
    TCK(cudaMemcpy(biases[l], net.b[l], sizeof(double) * dims[l + 1], cudaMemcpyDeviceToHost));
  }
  if (res->losses && E > 0)
    TCK(cudaMemcpy(res->losses, losses, sizeof(double) * E * batches, cudaMemcpyDeviceToHost));
  // ---- holdout metrics
  res->holdout_mae = NAN;
  res->sign_agreement = NAN;
  if (d->n_hold > 0) {
    const int nh = d->n_hold;
    double* xh = A.alloc<double>((size_t)nh * in);
    double* yh = A.alloc<double>(nh);
    double* ae = A.alloc<double>(nh);
    int* ag = A.alloc<int>(nh);
    if (!xh || !yh || !ae || !ag) return fail(MPPI_E_CUDA, "out of device memory");
    TCK(cudaMemcpyAsync(xh, d->x_hold, sizeof(double) * nh * in, cudaMemcpyHostToDevice, st));
    TCK(cudaMemcpyAsync(yh, d->y_hold, sizeof(double) * nh, cudaMemcpyHostToDevice, st));
    holdout_kernel<<<blocks_for(nh, 128), 128, 0, st>>>(net, xh, yh, nh, in, ae, ag);
    TCK(cudaGetLastError());
    std::vector<double> hae(nh);
    std::vector<int> hag(nh);
    TCK(cudaMemcpyAsync(hae.data(), ae, sizeof(double) * nh, cudaMemcpyDeviceToHost, st));
    TCK(cudaMemcpyAsync(hag.data(), ag, sizeof(int) * nh, cudaMemcpyDeviceToHost, st));
    TCK(cudaStreamSynchronize(st));
    double s = 0.0, a = 0.0;
    for (int i = 0; i < nh; ++i) {
      s += hae[i];
      a += hag[i];
    }
    res->holdout_mae = s / nh;
    res->sign_agreement = a / nh;
  }
  return MPPI_OK;
}

}  // extern "C"
