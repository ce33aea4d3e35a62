import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2104_13542_b200 import configs
from paper_2104_13542_b200.controller import Controller
from paper_2104_13542_b200.kinematics import load_chain
from paper_2104_13542_b200.simworld import target_at
script, world = configs.tracking_problem()
kw = dict(configs.CONTROLLER_KW)
c = Controller(load_chain("arm7.chain"), target_at(script, 0.0), weights=configs.make_weights(3), world=world, **kw)
c2 = configs.make_controller(2)
st = configs.start_state()
for _ in range(50):
    c.control_step(st); c2.control_step(st)
def med(fn, n=2000):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6, np.mean(ts) * 1e6
p = c.plan
print("c3 control_step same goal  med/mean %.2f %.2f" % med(lambda: c.control_step(st)))
i = [0]
def moving():
    i[0] += 1
    c.set_goal(target_at(script, (i[0] % 200) * 0.05))
def step_after_goal():
    moving()
    t0 = time.perf_counter(); c.control_step(st); return time.perf_counter() - t0
ts = [step_after_goal() for _ in range(2000)]
print("c3 control_step moving goal med/mean %.2f %.2f" % (np.median(ts) * 1e6, np.mean(ts) * 1e6))
print("c3 set_goal               med/mean %.2f %.2f" % med(moving))
print("c2 control_step           med/mean %.2f %.2f" % med(lambda: c2.control_step(st)))
c.profile_stages(1)
ds = []
for _ in range(500):
    _, d = c.control_step(st); ds.append(c.plan._info[0].device_ms)
print("c3 device_ms (level 1, warm L2) %.2f us" % (np.median(ds) * 1e3))
