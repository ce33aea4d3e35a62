"""Config-4-shaped step (B instances x 500 x 30, config-2 costs) for ncu captures.

    python scripts/profile_batched.py [instances] [steps]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200 import configs  # noqa: E402
from paper_2104_13542_b200.batched import BatchedController  # noqa: E402
from paper_2104_13542_b200.kinematics import load_chain  # noqa: E402
from paper_2104_13542_b200.surrogate import load_arm7_surrogate  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
goals, th0 = configs.batched_problem(B)
kw = dict(configs.CONTROLLER_KW)
kw.pop("seed")
bc = BatchedController(load_chain("arm7.chain"), goals, weights=configs.make_weights(2),
                       self_collision=load_arm7_surrogate(), **kw)
for _ in range(steps):
    cmds, d = bc.control_step(th0, np.zeros_like(th0))
print("B", B, "device_ms", d.device_ms, d.stage_ms)
