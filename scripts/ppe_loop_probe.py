"""Time the PPE loop forms (graph WHILE node vs host-polled batches) on the small,
sweep-heavy configurations (BASELINE configs[0], configs[1])."""
import sys, time
sys.path.insert(0, ".")
import torch
import synth
from paper_1908_01762_b200 import Simulation

for name, case, steps in (("tgv2d (configs[0])", synth.tgv2d(), 10), ("hydrostatic (configs[1])", synth.hydrostatic(), 20)):
    for loop in (1, 2, 3):
        sim = Simulation.from_case(case, ppe_loop=loop)
        for _ in range(2):
            sim.step(case.dt)
        sim.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream()
        t0 = time.perf_counter()
        its = 0
        for _ in range(steps):
            its += sim.step(case.dt).iters
        sim.sync()
        t = time.perf_counter() - t0
        print(f"{name:26s} ppe_loop={loop} ({ {1: 'host batches', 2: 'graph WHILE', 3: 'persistent'}[loop] }): {1e3 * t / steps:8.3f} ms/step, "
              f"{its / steps:7.1f} sweeps/step, {1e6 * t / its:6.2f} us/sweep-iteration", flush=True)
        sim.close()
