"""Host-side cost of one config-2 step: control_step vs Plan.step vs the bare
ctypes call (no L2 flush; medians of 2000 steps)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13542_b200 import configs  # noqa: E402

c = configs.make_controller(2)
st = configs.start_state()
for _ in range(50):
    c.control_step(st)


def med(fn, n=2000):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6


p = c.plan
th, thd = st.theta, st.theta_dot
print(f"control_step      {med(lambda: c.control_step(st)):7.2f} us")
print(f"Plan.step         {med(lambda: p.step(th, thd)):7.2f} us")
print(f"ctypes mppi_step  {med(lambda: p._step_fn(p.handle, p._p_th, p._p_thd, p._p_cmd, p._info)):7.2f} us")
print(f"_sync_goal        {med(lambda: c._sync_goal()):7.2f} us")
