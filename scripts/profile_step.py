"""Run N config-2 control steps (500 x 30, FP32) for ncu captures.

    python scripts/profile_step.py [steps] [particles] [config]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200 import configs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
particles = int(sys.argv[2]) if len(sys.argv) > 2 else 500
config = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c = configs.make_controller(config, particles=particles)
st = configs.start_state()
for _ in range(steps):
    cmd, d = c.control_step(st)
print("cmd", cmd, "device_ms", d.rollout_ms, d.update_ms)
