// mppi_launch.cuh — host launchers for the dof-templated kernels. Each
// precision is instantiated in its own translation unit (mppi_launch_f32.cu,
// mppi_launch_f64.cu) so the eight dof variants compile in parallel.
#pragma once

#include <cstdlib>
#include <type_traits>

#include "mppi_kernels.cuh"

namespace mppi {

template <typename R>
cudaError_t launch_rollout_any(const RolloutArgs<R>& a, int D, long long warps, cudaStream_t st);
template <typename R>
cudaError_t launch_stats_any(const StatsArgs<R>& s, int D, cudaStream_t st);
template <typename R>
cudaError_t launch_finalize(const StatsArgs<R>& s, const double* recs, int count, cudaStream_t st);
// fused rollout + learned-collision MLP (mppi_fused.cuh), float only
cudaError_t launch_rollout_mlp_any(const RolloutArgs<float>& a, int D, const unsigned char* img, float* out_d,
                                   cudaStream_t st);
size_t fused_cap_bytes_f32(const RolloutArgs<float>& a);

inline size_t stats_smem_bytes(int ppb, int nblk, int HD) {
  return sizeof(double) * (2 * (size_t)ppb + 32 + (size_t)(nblk > 8 ? nblk : 8) * (1 + kRecHead) +
                           (kRecHead + 2 * HD) + HD +
                           (kRecHead + 2 * HD) + HD + 8 * (1 + kRecHead) + 32) +  // peer-exchange scratch
         sizeof(int) * ((size_t)ppb + 2);
}

// stats_multi_kernel: G instances per block. MPPI_STATS_G in {1, 2, 4}
// (1 selects stats_kernel) and MPPI_STATS_MINBLOCKS in {0, 5} (0: the
// compiler's register count) override the default variant below.
// A/B at 4096 x 500 (update stage): 1.66 ms (G=1) -> 0.89 (G=2) / 0.98 (G=4);
// with the discount hoisted, same box: 0.79 (G=2, 72 registers, 3 blocks/SM)
// -> 0.70 (G=2 at >= 5 blocks/SM, 48 registers) / 0.96 (16 loads in flight) / 0.88 (G=4)
struct StatsMultiVariant {
  int g;           // instances per block: 1 (stats_kernel), 2 or 4
  int min_blocks;  // __launch_bounds__ minimum blocks per SM: 0 (none) or 5
};
constexpr StatsMultiVariant kStatsMultiDefault = {2, 5};
inline StatsMultiVariant stats_multi_variant() {
  StatsMultiVariant v = kStatsMultiDefault;
  if (const char* ev = getenv("MPPI_STATS_G")) {
    const int g = atoi(ev);
    if (g == 1 || g == 2 || g == 4) v.g = g;
  }
  if (const char* ev = getenv("MPPI_STATS_MINBLOCKS")) v.min_blocks = atoi(ev) == 5 ? 5 : 0;
  if (v.g == 4) v.min_blocks = 0;  // only G=2 has the occupancy build
  return v;
}
inline size_t stats_multi_smem_bytes(int G, int N, int HD) {
  return sizeof(double) * (2 * (size_t)G * N + (size_t)G * (kRecHead + 2 * HD) + HD) + sizeof(int) * (size_t)N;
}

// CTAs per SM of the many-waves rollout build (__launch_bounds__ minimum):
// 5 -> 96 registers (A/B at 4096 x 500: rollout 4.27 ms at 6 / 80 registers
// with spills, 4.02 ms at 5, 4.30 ms at 4; -DMPPI_ROLLOUT_MINB=n)
#ifndef MPPI_ROLLOUT_MINB
#define MPPI_ROLLOUT_MINB 5
#endif
constexpr int kRolloutMinBlocks = MPPI_ROLLOUT_MINB;

#ifdef MPPI_LAUNCH_IMPL
template <typename R, int D>
cudaError_t launch_rollout_d(const RolloutArgs<R>& a, long long warps, cudaStream_t st) {
  const size_t smem = rollout_needs_caps(a.cost) ? (size_t)kRolloutWarps * a.chain.n_caps * 6 * 32 * sizeof(R) : 0;
  // many waves of particles: the occupancy build (float only; see rollout_kernel)
  constexpr long long kThroughputWarps = 32768;
  const bool many = std::is_same<R, float>::value && warps >= kThroughputWarps && smem <= 24 * 1024;
  // the lean specialisation for control steps of configs 1/2 (float; the
  // float64 exact path and the evaluation modes keep the general kernel)
  const bool lean = std::is_same<R, float>::value && a.mode == 0 && !rollout_needs_caps(a.cost) &&
                    getenv("MPPI_ROLLOUT_GENERAL") == nullptr;
  // the paired build (two particles per warp, packed FP32) for many-waves
  // control steps without dumps; posenc hand-off and odd N keep the single one
  if constexpr (std::is_same<R, float>::value) {
    if (many && lean && a.N % 2 == 0 && a.out_pos == nullptr && a.out_terms == nullptr &&
        (a.mlp_x == nullptr || a.mlp_x_q) && !(getenv("MPPI_ROLLOUT_SINGLE") && atoi(getenv("MPPI_ROLLOUT_SINGLE")))) {
      const unsigned grid = (unsigned)((warps / 2 + kRolloutWarps - 1) / kRolloutWarps);
      rollout_pair_kernel<D><<<grid, kRolloutWarps * 32, 0, st>>>(a);
      return cudaGetLastError();
    }
  }
  auto kern = many ? (lean ? rollout_kernel<R, D, kRolloutMinBlocks, std::is_same<R, float>::value>
                           : rollout_kernel<R, D, kRolloutMinBlocks>)
                   : (lean ? rollout_kernel<R, D, 1, std::is_same<R, float>::value> : rollout_kernel<R, D, 1>);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const unsigned grid = (unsigned)((warps + kRolloutWarps - 1) / kRolloutWarps);
  kern<<<grid, kRolloutWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename R, int D>
cudaError_t launch_stats_cluster_d(const StatsArgs<R>& s, cudaStream_t st) {
  const size_t smem = stats_cluster_smem_bytes(s.ppb, s.H * D);
  const bool lean = s.finalize_inline && !s.dump_step && !s.dump_terms && !s.dump_weights && !s.peer_recv &&
                    getenv("MPPI_STATS_GENERAL") == nullptr;
  auto kern = lean ? stats_cluster_kernel<R, D, true> : stats_cluster_kernel<R, D, false>;
  if (s.nblk > 8) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(s.nblk, s.B, 1);
  cfg.blockDim = dim3(kStatsThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = s.nblk;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_mask() & PDL_STATS) ? 2 : 1;  // no programmatic edge unless asked for
  return cudaLaunchKernelEx(&cfg, kern, s);
}

template <typename R>
cudaError_t launch_finalize(const StatsArgs<R>& s, const double* recs, int count, cudaStream_t st);

template <typename R, int D>
cudaError_t launch_stats_d(const StatsArgs<R>& s, cudaStream_t st) {
  // one instance beyond one cluster, up to 8192 particles: clusters of 16
  // CTAs of 32 particles reduce in distributed shared memory to one record
  // each (relative to the cluster's own minimum), finalize_kernel combines the
  // records in fixed order and applies the update — one global combine level
  // instead of the block records' two (A/B, config 5: N = 4096 92.5 -> 84 us
  // per step, 8192 124.5 -> 120 us; at 32768 the block records are faster;
  // MPPI_MULTI_CLUSTER_PPB=p overrides the particles per CTA, 0 disables)
  int mc_ppb = s.N <= kClusterMax * kClusterMax * 32 ? 32 : 0;
  if (const char* e = getenv("MPPI_MULTI_CLUSTER_PPB")) mc_ppb = atoi(e) > 0 ? std::min(atoi(e), kClusterMaxPPB) : 0;
  const int mc_clusters = mc_ppb > 0 ? (s.N + kClusterMax * mc_ppb - 1) / (kClusterMax * mc_ppb) : 0;
  if (mc_ppb > 0 && !s.totals_only && s.B == 1 && s.finalize_inline && !s.peer_recv && !s.dump_step &&
      !s.dump_terms && !s.dump_weights && s.N > kClusterMax * kClusterMaxPPB &&
      mc_clusters <= stats_rec_stride(s.nblk)) {  // one record slot per cluster in the plan's buffer
    StatsArgs<R> c = s;
    c.ppb = mc_ppb;
    c.nblk = kClusterMax;
    c.finalize_inline = 0;
    c.reset_status = 0;
    c.out_record = s.records;
    const int nclu = mc_clusters;
    auto kern = stats_cluster_kernel<R, D, false>;
    const size_t smem = stats_cluster_smem_bytes(c.ppb, c.H * D);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nclu * kClusterMax, 1, 1);
    cfg.blockDim = dim3(kStatsThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kClusterMax;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, c);
    if (e != cudaSuccess) return e;
    return launch_finalize<R>(s, s.records, nclu, st);
  }
  // latency path: one cluster per instance when the particles fit 16 CTAs
  if (!s.totals_only && s.B <= 8 && s.nblk <= kClusterMax && s.ppb <= kClusterMaxPPB &&
      getenv("MPPI_NO_CLUSTER") == nullptr)
    return launch_stats_cluster_d<R, D>(s, st);
  // batched path: one block's worth of particles per instance, update applied
  // in-kernel, nothing dumped -> several instances per block share eps reads
  if (s.nblk == 1 && s.ppb == s.N && s.B >= 148 && !s.totals_only && s.finalize_inline && !s.peer_recv &&
      !s.dump_step && !s.dump_terms && !s.dump_weights && !s.dbg && s.H * D <= kStatsThreads) {
    const StatsMultiVariant v = stats_multi_variant();
    if (v.g != 1) {
      const size_t smem = stats_multi_smem_bytes(v.g, s.N, s.H * D);
      if (smem <= 200 * 1024) {
        auto kern = v.g == 4            ? stats_multi_kernel<R, D, 4>
                    : v.min_blocks == 5 ? stats_multi_kernel<R, D, 2, 8, 5>
                                        : stats_multi_kernel<R, D, 2>;
        if (smem > 48 * 1024) {
          cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          if (e != cudaSuccess) return e;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((s.B + v.g - 1) / v.g, 1, 1);
        cfg.blockDim = dim3(kStatsThreads, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = (pdl_mask() & PDL_STATS) != 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, s);
      }
    }
  }
  const size_t smem = stats_smem_bytes(s.ppb, s.nblk, s.H * D);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(stats_kernel<R, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(s.nblk, s.B, 1);
  cfg.blockDim = dim3(kStatsThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (pdl_mask() & PDL_STATS) != 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, stats_kernel<R, D>, s);
}

#define MPPI_LAUNCH_SWITCH(FN, ...)                 \
  switch (D) {                                      \
    case 1: return FN<R, 1>(__VA_ARGS__);           \
    case 2: return FN<R, 2>(__VA_ARGS__);           \
    case 3: return FN<R, 3>(__VA_ARGS__);           \
    case 4: return FN<R, 4>(__VA_ARGS__);           \
    case 5: return FN<R, 5>(__VA_ARGS__);           \
    case 6: return FN<R, 6>(__VA_ARGS__);           \
    case 7: return FN<R, 7>(__VA_ARGS__);           \
    case 8: return FN<R, 8>(__VA_ARGS__);           \
    default: return cudaErrorInvalidValue;          \
  }

template <typename R>
cudaError_t launch_rollout_any(const RolloutArgs<R>& a, int D, long long warps, cudaStream_t st) {
  MPPI_LAUNCH_SWITCH(launch_rollout_d, a, warps, st)
}
template <typename R>
cudaError_t launch_stats_any(const StatsArgs<R>& s, int D, cudaStream_t st) {
  MPPI_LAUNCH_SWITCH(launch_stats_d, s, st)
}
template <typename R>
cudaError_t launch_finalize(const StatsArgs<R>& s, const double* recs, int count, cudaStream_t st) {
  const int HD = s.H * s.D;
  const size_t smem = sizeof(double) * (32 + (size_t)(count > 8 ? count : 8) * (1 + kRecHead) + kRecHead + 2 * HD + HD);
  finalize_kernel<R><<<1, kStatsThreads, smem, st>>>(s, recs, count);
  return cudaGetLastError();
}
#endif

}  // namespace mppi
