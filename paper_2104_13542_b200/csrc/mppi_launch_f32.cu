// Explicit instantiation of the float launchers (see mppi_launch.cuh).
#define MPPI_LAUNCH_IMPL
#include "mppi_launch.cuh"
#include "mppi_fused.cuh"

namespace mppi {
template cudaError_t launch_rollout_any<float>(const RolloutArgs<float>&, int, long long, cudaStream_t);
template cudaError_t launch_stats_any<float>(const StatsArgs<float>&, int, cudaStream_t);
template cudaError_t launch_finalize<float>(const StatsArgs<float>&, const double*, int, cudaStream_t);

cudaError_t launch_rollout_mlp_any(const RolloutArgs<float>& a, int D, const unsigned char* img, float* out_d,
                                   cudaStream_t st) {
  using R = float;
  MPPI_LAUNCH_SWITCH(launch_rollout_mlp_d, a, img, out_d, st)
}
size_t fused_cap_bytes_f32(const RolloutArgs<float>& a) { return fused_cap_bytes(a); }
}  // namespace mppi
