"""Run N config-2 control steps (500 x 30, FP32) for ncu captures / debug timelines.

    python scripts/profile_step.py [steps] [particles] [config] [--flush]

--flush writes a 256 MiB buffer between steps (cold L2, as bench.py times).
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200 import configs  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
flush = "--flush" in sys.argv
steps = int(args[0]) if len(args) > 0 else 5
particles = int(args[1]) if len(args) > 1 else 500
config = int(args[2]) if len(args) > 2 else 2
c = configs.make_controller(config, particles=particles)
st = configs.start_state()
buf = None
if flush:
    import torch
    buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(steps):
    if buf is not None:
        buf.fill_(1)
        torch.cuda.synchronize()
    cmd, d = c.control_step(st)
print("cmd", cmd, "device_ms", d.rollout_ms, d.update_ms)
