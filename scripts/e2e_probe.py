"""Where the end-to-end step time goes (bench.py's e2e loop, C5): each public call timed."""
import sys, time
sys.path.insert(0, ".")
import torch
import synth
from paper_1908_01762_b200 import Simulation
case = synth.dambreak3d()
sim = Simulation.from_case(case)
n, dim = case.n, case.dim
pin = lambda shape: torch.empty(shape, dtype=torch.float64, pin_memory=True)
hx, hu, hut, hp, outp = pin((n, dim)), pin((n, dim)), pin((n, dim)), pin((n,)), pin((n,))
for _ in range(3):
    sim.step(case.dt)
sim.get_ptr("POSITION", hx.data_ptr(), n * dim); sim.get_ptr("VELOCITY", hu.data_ptr(), n * dim)
sim.get_ptr("TRANSPORT_VELOCITY", hut.data_ptr(), n * dim); sim.get_ptr("PRESSURE", hp.data_ptr(), n)
sim.sync()
acc = {}
def tm(name, f):
    t0 = time.perf_counter(); f(); sim.sync(); acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
K = 5
for _ in range(K):
    tm("set POSITION", lambda: sim.set_ptr("POSITION", hx.data_ptr(), n * dim))
    tm("set VELOCITY", lambda: sim.set_ptr("VELOCITY", hu.data_ptr(), n * dim))
    tm("set TRANSPORT_VELOCITY", lambda: sim.set_ptr("TRANSPORT_VELOCITY", hut.data_ptr(), n * dim))
    tm("set PRESSURE", lambda: sim.set_ptr("PRESSURE", hp.data_ptr(), n))
    tm("step", lambda: sim.step(case.dt))
    tm("get PRESSURE", lambda: sim.get_ptr("PRESSURE", outp.data_ptr(), n))
for k, v in acc.items():
    print(f"{k:24s} {1e3 * v / K:8.3f} ms")
print(f"{'total':24s} {1e3 * sum(acc.values()) / K:8.3f} ms")
