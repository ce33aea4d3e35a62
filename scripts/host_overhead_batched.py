"""Host-side cost of one config-4 step (4096 controllers): BatchedController.control_step
vs Plan.step vs the bare ctypes call (no L2 flush; medians of 30 steps)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200 import configs  # noqa: E402
from paper_2104_13542_b200.batched import BatchedController  # noqa: E402
from paper_2104_13542_b200.kinematics import load_chain  # noqa: E402
from paper_2104_13542_b200.surrogate import load_arm7_surrogate  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
goals, th0 = configs.batched_problem(B)
kw = dict(configs.CONTROLLER_KW)
kw.pop("seed")
bc = BatchedController(load_chain("arm7.chain"), goals, weights=configs.make_weights(2),
                       self_collision=load_arm7_surrogate(), **kw)
thd = np.zeros_like(th0)
for _ in range(5):
    bc.control_step(th0, thd)
p = bc.plan


def med(fn, n=30):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3


print(f"control_step   {med(lambda: bc.control_step(th0, thd)):8.3f} ms")
print(f"Plan.step      {med(lambda: p.step(th0, thd)):8.3f} ms")
print(f"ctypes step    {med(lambda: p._step_fn(p.handle, p._p_th, p._p_thd, p._p_cmd, p._info)):8.3f} ms")
cmds, infos = p.step(th0, thd)
print(f"apply_ladder   {med(lambda: bc._apply_ladder(cmds, infos)):8.3f} ms")
print(f"isfinite x2    {med(lambda: (np.isfinite(th0).all(), np.isfinite(thd).all())):8.3f} ms")
p.profile_stages(1)
for _ in range(3):
    p.step(th0, thd)
dev, wall = [], []
for _ in range(30):
    t0 = time.perf_counter()
    _, infos = p.step(th0, thd)
    wall.append((time.perf_counter() - t0) * 1e3)
    dev.append(infos[0].device_ms)
print(f"lean graph: device {np.median(dev):.3f} ms, Plan.step wall {np.median(wall):.3f} ms (level-1 events)")
