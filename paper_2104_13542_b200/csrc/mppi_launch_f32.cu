// Explicit instantiation of the float launchers (see mppi_launch.cuh).
#define MPPI_LAUNCH_IMPL
#include "mppi_launch.cuh"

namespace mppi {
template cudaError_t launch_rollout_any<float>(const RolloutArgs<float>&, int, long long, cudaStream_t);
template cudaError_t launch_stats_any<float>(const StatsArgs<float>&, int, cudaStream_t);
template cudaError_t launch_finalize<float>(const StatsArgs<float>&, const double*, int, cudaStream_t);
}  // namespace mppi
