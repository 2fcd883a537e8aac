#!/usr/bin/env python
"""Table 1 of the paper (§3.1) at the paper's own resolutions, on the CUDA path.

Average Jacobi sweeps per step for the lid-driven cavity (100 x 100, Re = 100)
and the 2D dam break (dx = 0.01) at eps = 1e-2 and 1e-3, under both readings of
eq:convergence:
  R12   the printed sums:  sum|dp| / max(Lambda, sum|p|) < eps
  R12b  means:             mean|dp| / max(Lambda, mean|p|) < eps
The paper prints: cavity 2.0 (1e-2), 3.0 (1e-3); dam break 2.0 (1e-2), 5.0 (1e-3).

    python scripts/table1.py [--t-cavity 10] [--t-db 1.0] > profiles/r2_table1.md
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1908_01762_b200 import SisphError, Simulation  # noqa: E402

PAPER = {("cavity", 1e-2): 2.0, ("cavity", 1e-3): 3.0, ("dam break 2D", 1e-2): 2.0, ("dam break 2D", 1e-3): 5.0}


def run(case, steps, **over):
    sim = Simulation.from_case(case, **over)
    its = []
    t0 = time.perf_counter()
    status = "ok"
    for k in range(steps):
        try:
            its.append(sim.step(case.dt).iters)
        except SisphError as e:
            status = f"failed at step {k}: {str(e)[:60]}"
            break
    sim.sync()
    wall = time.perf_counter() - t0
    u = sim.get("VELOCITY")[case.tag == 0] if status == "ok" else np.array([np.nan])
    sim.close()
    its = np.array(its) if its else np.array([0])
    return dict(mean=float(its.mean()), median=float(np.median(its)), p90=float(np.percentile(its, 90)),
                max=int(its.max()), steps=len(its), wall=wall, umax=float(np.abs(u).max()), status=status)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t-cavity", type=float, default=10.0)
    ap.add_argument("--t-db", type=float, default=1.0)
    ap.add_argument("--only", choices=["cavity", "db"], default=None)
    ap.add_argument("--p-ref-limit", action="store_true",
                    help="dam break: p_ref = rho0 (h~ / dt)^2, the GTVF sub-step stability limit (R22c)")
    a = ap.parse_args()
    print("# Table 1 at the paper's resolutions (PAPER.md:575-594), CUDA path, B200\n")
    print("Average PPE sweeps per step over the whole run; R12 = eq:convergence with the printed sums, "
          "R12b = with means (DESIGN.md §5).\n")
    print("| problem | resolution | t_end | eps | reading | mean | median | p90 | max | steps | paper | max abs(u) | "
          "wall s | status |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for eps in (1e-2, 1e-3) if a.only != "db" else ():
        for cm in (0, 1):
            c = synth.cavity(n=100, t_end=a.t_cavity, tol=eps, precision=32)
            r = run(c, c.steps, conv_mean=cm)
            print(f"| cavity | 100 x 100 | {a.t_cavity:g} | {eps:g} | {'R12b' if cm else 'R12'} | {r['mean']:.2f} | "
                  f"{r['median']:.0f} | {r['p90']:.0f} | {r['max']} | {r['steps']} | {PAPER[('cavity', eps)]} | "
                  f"{r['umax']:.3f} | {r['wall']:.1f} | {r['status']} |", flush=True)
    for eps in (1e-2, 1e-3) if a.only != "cavity" else ():
        for cm in (0, 1):
            c = synth.dambreak2d(nx=100, ny=200, dx=0.01, tol=eps, precision=32)
            steps = int(round(a.t_db / c.dt))
            over = {"conv_mean": cm}
            if a.p_ref_limit:
                over["p_ref"] = c.params["rho0"] * (0.5 * c.h / c.dt) ** 2
            r = run(c, steps, **over)
            print(f"| dam break 2D | dx = 0.01, {c.n_fluid} fluid | {a.t_db:g} | {eps:g} | {'R12b' if cm else 'R12'} | "
                  f"{r['mean']:.2f} | {r['median']:.0f} | {r['p90']:.0f} | {r['max']} | {r['steps']} | "
                  f"{PAPER[('dam break 2D', eps)]} | {r['umax']:.3f} | {r['wall']:.1f} | {r['status']} |", flush=True)


if __name__ == "__main__":
    main()
