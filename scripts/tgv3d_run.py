"""BASELINE configs[3] as configured (TGV-3D 128^3, fp32, tol 1e-3, 100 steps): kinetic energy
vs the early-time decay exp(-2 nu k^2 t) = exp(-6 nu t), sweeps per step."""
import sys
sys.path.insert(0, ".")
import numpy as np
import synth
from paper_1908_01762_b200 import Simulation
over = dict(a.split("=") for a in sys.argv[1:])
over = {k: float(v) if "." in v or "e" in v else int(v) for k, v in over.items()}
case = synth.tgv3d()
sim = Simulation.from_case(case, **over)
m = case.m
u0 = case.u
ke0 = 0.5 * np.sum(m[:, None] * u0 ** 2)
nu = case.params["nu"]
t, its = 0.0, []
for s in range(case.steps):
    its.append(sim.step(case.dt).iters)
    t += case.dt
    if (s + 1) % 20 == 0:
        u = sim.get("VELOCITY")
        ke = 0.5 * np.sum(m[:, None] * u ** 2)
        print(f"step {s + 1:4d} t {t:.3f} KE/KE0 {ke / ke0:.4f} (exp(-6 nu t) {np.exp(-6 * nu * t):.4f}) "
              f"max|u| {np.linalg.norm(u, axis=1).max():.3f} mean sweeps {np.mean(its[-20:]):.1f}", flush=True)
