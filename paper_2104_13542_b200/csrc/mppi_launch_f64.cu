// Explicit instantiation of the double launchers (see mppi_launch.cuh).
#define MPPI_LAUNCH_IMPL
#include "mppi_launch.cuh"

namespace mppi {
template cudaError_t launch_rollout_any<double>(const RolloutArgs<double>&, int, long long, cudaStream_t);
template cudaError_t launch_stats_any<double>(const StatsArgs<double>&, int, cudaStream_t);
template cudaError_t launch_finalize<double>(const StatsArgs<double>&, const double*, int, cudaStream_t);
}  // namespace mppi
