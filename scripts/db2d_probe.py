#!/usr/bin/env python
"""2D dam break at the paper's dx = 0.01: max |u| along the run for the printed
GTVF background pressure p_ref = rho0 c^2 and for p_ref inside the sub-step stability
limit dt sqrt(p0 / rho) / h~ <= 1 (reading R22c), eq:convergence on means (R12b), eps = 1e-2.

    python scripts/db2d_probe.py > profiles/r2_db2d_probe.md
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1908_01762_b200 import Simulation  # noqa: E402

print("| p_ref | t | mean sweeps so far | max abs(u) | front x |")
print("|---|---|---|---|---|")
for label in ("rho c^2 (printed)", "R22c limit"):
    c = synth.dambreak2d(nx=100, ny=200, dx=0.01, tol=1e-2, precision=32)
    over = {"conv_mean": 1}
    if label != "rho c^2 (printed)":
        ht = 0.5 * c.h
        over["p_ref"] = c.params["rho0"] * (ht / c.dt) ** 2
    sim = Simulation.from_case(c, **over)
    its = []
    f = c.tag == 0
    for k in range(1, int(round(1.0 / c.dt)) + 1):
        its.append(sim.step(c.dt).iters)
        if k % int(round(0.125 / c.dt)) == 0:
            u = sim.get("VELOCITY")[f]
            x = sim.get("POSITION")[f]
            print(f"| {label} ({over.get('p_ref', c.params['p_ref']):.3g}) | {k * c.dt:.3f} | {np.mean(its):.2f} | "
                  f"{np.abs(u).max():.3f} | {x[:, 0].max():.3f} |", flush=True)
    sim.close()
