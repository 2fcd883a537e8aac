#!/usr/bin/env python
"""the paper's method variants on the CUDA path.

1. Tolerance sweep (a Table 1 analogue): average PPE
   sweeps per step vs epsilon on the 2D dam break (BASELINE configs[2], full
   size, fp32), the hydrostatic column (configs[1]) and the 2D Taylor-Green
   vortex (configs[0]); checks "typically 2-10 iterations".
2. EISPH vs SISPH (section 4.2): Taylor-Green at Re = 10000,
   100 x 100 particles perturbed by dx/10; one Jacobi sweep per step (EISPH)
   vs sweeps to the tolerance (SISPH); L1 velocity error against the exact
   decay exp(-8 pi^2 t / Re) (reading R28).
3. Pressure-gradient form (symm vs asymm) on the Taylor-Green
   vortex, and slip vs no-slip wall u* on the hydrostatic column.

    python scripts/variants.py [--quick] > profiles/r1_variants.md
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1908_01762_b200 import Simulation  # noqa: E402


def avg_sweeps(case, steps, **over):
    sim = Simulation.from_case(case, **over)
    its = []
    t0 = time.perf_counter()
    for _ in range(steps):
        its.append(sim.step(case.dt).iters)
    sim.sync()
    t = time.perf_counter() - t0
    sim.close()
    return float(np.mean(its)), int(np.max(its)), t


def tgv_error(sim, case, t):
    """L1 error of |u| vs the exact decaying TGV field at the particles (R28)."""
    x = sim.get("POSITION")
    u = sim.get("VELOCITY")
    nu = case.params["nu"]
    b = -8.0 * np.pi ** 2 * nu
    X, Y = x[:, 0], x[:, 1]
    ue = np.exp(b * t) * np.stack([-np.cos(2 * np.pi * X) * np.sin(2 * np.pi * Y),
                                   np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y)], 1)
    a, e = np.linalg.norm(u, axis=1), np.linalg.norm(ue, axis=1)
    return float(np.abs(a - e).sum() / e.sum()), float(a.max() / np.exp(b * t))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    q = args.quick
    out = {}
    print("# NEXT-2: method variants on the CUDA path (B200)\n")
    # ---------------------------------------------------------------- 1. tolerance sweep
    print("## 1. Average Jacobi sweeps per step vs tolerance (Table 1 analogue, PAPER.md:578-594)\n")
    print("| problem | particles | steps | tolerance | mean sweeps | max sweeps | wall s |")
    print("|---|---|---|---|---|---|---|")
    rows = []
    probs = [("dam break 2D (configs[2])", synth.dambreak2d(nx=250, ny=500, dx=0.004) if q else synth.dambreak2d(),
              100 if q else 400),
             ("hydrostatic (configs[1])", synth.hydrostatic(precision=32), 100 if q else 400),
             ("Taylor-Green 2D (configs[0])", synth.tgv2d(), 100 if q else 200)]
    for name, case, steps in probs:
        for tol in (1e-1, 5e-2, 1e-2, 5e-3, 1e-3, 5e-4):
            m, mx, t = avg_sweeps(case, steps, tol=tol)
            rows.append({"problem": name, "tol": tol, "mean": m, "max": mx})
            print(f"| {name} | {case.n_fluid} | {steps} | {tol:g} | {m:.2f} | {mx} | {t:.1f} |")
    out["tolerance_sweep"] = rows
    print("\nPaper (PAPER.md:578-594, 2D dam break at its own resolution): 5.0 sweeps at 0.001, 2.0 at 0.01.\n")
    # ---------------------------------------------------------------- 2. EISPH vs SISPH
    print("## 2. EISPH (one sweep) vs SISPH, Taylor-Green Re = 10000, 100 x 100, jitter dx/10 (P:1156-1176)\n")
    print("| scheme | steps | t | mean sweeps | L1 error of abs(u) | max abs(u) / exp(bt) |")
    print("|---|---|---|---|---|---|")
    res = []
    for label, over in (("SISPH tol 1e-2", dict(tol=1e-2)), ("SISPH tol 1e-3", dict(tol=1e-3)),
                        ("EISPH", dict(max_iter=1, min_iter=1))):
        case = synth.tgv2d(n=100, re=10000.0)
        steps = 100 if q else 400
        sim = Simulation.from_case(case, **over)
        its = [sim.step(case.dt).iters for _ in range(steps)]
        t = steps * case.dt
        err, dec = tgv_error(sim, case, t)
        res.append({"scheme": label, "t": t, "mean_sweeps": float(np.mean(its)), "l1": err, "decay": dec})
        print(f"| {label} | {steps} | {t:.2f} | {np.mean(its):.2f} | {err:.4f} | {dec:.4f} |")
        sim.close()
    out["eisph"] = res
    # ---------------------------------------------------------------- 3. forms
    print("\n## 3. Pressure-gradient form and wall u* construction\n")
    print("| case | variant | mean sweeps | metric |")
    print("|---|---|---|---|")
    forms = []
    for pg, label in ((1, "asymm (eq:mom:sph:press:pij)"), (0, "symm (eq:mom:sph:press:symm)")):
        case = synth.tgv2d()
        sim = Simulation.from_case(case, pgrad=pg)
        its = [sim.step(case.dt).iters for _ in range(case.steps)]
        err, dec = tgv_error(sim, case, case.steps * case.dt)
        forms.append({"case": "tgv2d", "variant": label, "mean": float(np.mean(its)), "l1": err})
        print(f"| TGV-2D Re 100, 10 steps | {label} | {np.mean(its):.2f} | L1 abs(u) error {err:.4f} |")
        sim.close()
    for ns, label in ((0, "slip u* (R16)"), (1, "no-slip u* (eq:vg-adami)")):
        case = synth.hydrostatic(precision=32)
        steps = 50 if q else 200
        sim = Simulation.from_case(case, ustar_noslip=ns)
        its = [sim.step(case.dt).iters for _ in range(steps)]
        p, x = sim.get("PRESSURE"), sim.get("POSITION")
        f = (case.tag == 0) & (x[:, 1] < 2.0 - 0.05)
        pex = 1000.0 * 9.81 * (2.0 - x[f, 1])
        dev = float(np.abs(p[f] - pex).mean() / (1000.0 * 9.81 * 2.0))
        forms.append({"case": "hydrostatic", "variant": label, "mean": float(np.mean(its)), "dev": dev})
        print(f"| hydrostatic, {steps} steps | {label} | {np.mean(its):.2f} | mean abs(p - rho g (H - y)) / rho g H = {dev:.4f} |")
        sim.close()
    out["forms"] = forms
    # ---------------------------------------------------------------- 4. square patch (NEXT-3)
    print("\n## 4. Square patch (NEXT-3, P:1301-1350): 100 x 100, h/dx 1.3, alpha 0.15, eps 1e-2, t = 3 s\n")
    print("| pgrad | steps | mean sweeps | angular momentum L(t)/L(0) | centre of mass | extent x | extent y |")
    print("|---|---|---|---|---|---|---|")
    sq = []
    for pg, label in ((1, "asymm"), (0, "symm")):
        case = synth.square_patch(precision=32)
        steps = int(round((0.5 if q else 3.0) / case.dt))
        sim = Simulation.from_case(case, pgrad=pg)
        m = case.m
        L0 = float(np.sum(m * (case.x[:, 0] * case.u[:, 1] - case.x[:, 1] * case.u[:, 0])))
        its = [sim.step(case.dt).iters for _ in range(steps)]
        x, u = sim.get("POSITION"), sim.get("VELOCITY")
        Lt = float(np.sum(m * (x[:, 0] * u[:, 1] - x[:, 1] * u[:, 0])))
        com = (m[:, None] * x).sum(0) / m.sum()
        sq.append({"pgrad": label, "steps": steps, "mean": float(np.mean(its)), "L_ratio": Lt / L0,
                   "com": com.tolist(), "extent": [float(np.ptp(x[:, 0])), float(np.ptp(x[:, 1]))]})
        print(f"| {label} | {steps} | {np.mean(its):.2f} | {Lt / L0:.4f} | ({com[0]:.1e}, {com[1]:.1e}) | "
              f"{np.ptp(x[:, 0]):.3f} | {np.ptp(x[:, 1]):.3f} |")
        sim.close()
    out["square_patch"] = sq
    with open(os.path.join(ROOT, "gpurun_out", "variants.json") if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
              else "/tmp/variants.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
