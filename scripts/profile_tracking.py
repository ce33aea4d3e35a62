"""Run config-3 closed-loop steps (64^3 voxel world, moving target) for ncu
captures / debug timelines, as bench.py --workload c3 does.

    python scripts/profile_tracking.py [steps] [--flush]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200 import configs  # noqa: E402
from paper_2104_13542_b200.controller import Controller  # noqa: E402
from paper_2104_13542_b200.kinematics import load_chain  # noqa: E402
from paper_2104_13542_b200.simworld import target_at  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = int(args[0]) if args else 20
script, world = configs.tracking_problem()
kw = dict(configs.CONTROLLER_KW)
c = Controller(load_chain("arm7.chain"), target_at(script, 0.0), weights=configs.make_weights(3), world=world, **kw)
buf = None
if "--flush" in sys.argv:
    import torch
    buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = configs.start_state()
for i in range(steps):
    c.set_goal(target_at(script, i * 0.05))
    if buf is not None:
        buf.fill_(1)
        torch.cuda.synchronize()
    cmd, d = c.control_step(st)
    st.theta_dot = st.theta_dot + 0.05 * cmd
    st.theta = st.theta + 0.05 * st.theta_dot
print("cmd", cmd)
