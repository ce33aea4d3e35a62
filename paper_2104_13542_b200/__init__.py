"""B200-native joint-space MPPI (arXiv 2104.13542) — drop-in for jointmpc's hot path.

Public API mirrors jointmpc: Controller.control_step, evaluate_rollouts,
CostStack.evaluate, the sampling/policy free functions and the exception
classes. All arithmetic of the hot path runs in hand-written sm_100a kernels
behind the C ABI in include/mppi_b200.h (loaded lazily by ``_native``).
"""

__version__ = "0.1.0"

from .errors import ChainError, ConfigError, ContractError, DeviceError, PolicyStateError  # noqa: F401
