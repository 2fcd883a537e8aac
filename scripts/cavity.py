#!/usr/bin/env python
"""NEXT-4 (moving walls): the lid-driven cavity of PAPER.md:1210-1300 §4.3 on the CUDA path.

Unit square, lid at U = 1, h/dx = 1, eps = 1e-2, symm, GTVF with p_ref = 2 max p after the
first solve (R33); slip vs no-slip u* (P:863-868).  Reports the centreline profiles
u(y) at x = 0.5 and v(x) at y = 0.5 (particles within dx of the line, binned by dx),
their extrema, sweeps per step and wall time.  No reference data is used (the Ghia
tables are not in this container).

    python scripts/cavity.py [--quick] > profiles/r1_cavity.md
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


def centreline(x, u, dx, axis, comp):
    """mean of u[:, comp] over particles within dx of the line x[axis'] = 0.5, binned along axis"""
    other = 1 - axis
    sel = np.abs(x[:, other] - 0.5) < dx
    s, v = x[sel, axis], u[sel, comp]
    edges = np.arange(0.0, 1.0 + 1e-12, dx)
    idx = np.clip(np.digitize(s, edges) - 1, 0, len(edges) - 2)
    out = np.full(len(edges) - 1, np.nan)
    for b in range(len(out)):
        m = idx == b
        if m.any():
            out[b] = v[m].mean()
    return 0.5 * (edges[1:] + edges[:-1]), out


def ext(v, s, arg):
    """(extremum, position) of a binned profile; NaN if no particle lies on the line"""
    if not np.isfinite(v).any():
        return float("nan"), float("nan")
    k = arg(v)
    return float(v[k]), float(s[k])


def run(n, re, t_end, noslip, precision=64, **over):
    case = synth.cavity(n=n, re=re, t_end=t_end, ustar_noslip=noslip, precision=precision)
    case.params.update(over)
    sim = Simulation.from_case(case)
    f = case.tag == 0
    its = []
    t0 = time.perf_counter()
    status = "ok"
    done = 0
    try:
        for _ in range(case.steps):
            its.append(sim.step(case.dt).iters)
            done += 1
        sim.sync()
    except Exception as e:  # noqa: BLE001 - reported in the table
        status = f"failed at step {done}: {e}"
    wall = time.perf_counter() - t0
    x, u = sim.get("POSITION")[f], sim.get("VELOCITY")[f]
    if not np.all(np.isfinite(u)):
        status = status if status != "ok" else "non-finite velocity"
    if status != "ok":
        sim.close()
        return dict(n=n, re=re, t=done * case.dt, steps=done, ustar="no-slip" if noslip else "slip",
                    conv="means" if case.params.get("conv_mean") else "sums", tol=case.params["tol"],
                    gtvf="2 max p (R33)" if case.params.get("pref_auto") else f"p_ref {case.params['p_ref']:g}",
                    mean_sweeps=float(np.mean(its)) if its else 0.0, wall_s=wall, status=status)
    yc, uc = centreline(x, u, case.dx, 1, 0)
    xc, vc = centreline(x, u, case.dx, 0, 1)
    ke = 0.5 * float(np.sum(case.m[f] * np.sum(u * u, 1)))
    rho_min = float(sim.get("DENSITY")[f].min())
    sim.close()
    return dict(n=n, re=re, t=case.steps * case.dt, steps=case.steps, ustar="no-slip" if noslip else "slip",
                conv="means" if case.params.get("conv_mean") else "sums", tol=case.params["tol"],
                gtvf="2 max p (R33)" if case.params.get("pref_auto") else f"p_ref {case.params['p_ref']:g}",
                mean_sweeps=float(np.mean(its)), wall_s=wall, ke=ke, status=status, rho_min=rho_min,
                u_min=ext(uc, yc, np.nanargmin)[0], y_at_u_min=ext(uc, yc, np.nanargmin)[1],
                v_max=ext(vc, xc, np.nanargmax)[0], x_at_v_max=ext(vc, xc, np.nanargmax)[1],
                v_min=ext(vc, xc, np.nanargmin)[0], x_at_v_min=ext(vc, xc, np.nanargmin)[1],
                n_on_lines=[int(np.isfinite(uc).sum()), int(np.isfinite(vc).sum())],
                profile_u=[[float(a), float(b)] for a, b in zip(yc, uc)],
                profile_v=[[float(a), float(b)] for a, b in zip(xc, vc)])


def row(r):
    if r["status"] != "ok":
        return (f"| {r['n']}x{r['n']} | {r['re']:g} | {r['ustar']} | {r['conv']} | {r['tol']:g} | {r['gtvf']} | "
                f"{r['steps']} | {r['mean_sweeps']:.2f} | {r['wall_s']:.1f} | {r['status']} | | | | |")
    return (f"| {r['n']}x{r['n']} | {r['re']:g} | {r['ustar']} | {r['conv']} | {r['tol']:g} | {r['gtvf']} | "
            f"{r['steps']} | {r['mean_sweeps']:.2f} | {r['rho_min']:.3f} | "
            f"{r['wall_s']:.1f} | {r['ke']:.4f} | {r['u_min']:.4f} at {r['y_at_u_min']:.3f} | "
            f"{r['v_max']:.4f} at {r['x_at_v_max']:.3f} | {r['v_min']:.4f} at {r['x_at_v_min']:.3f} |")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    t_end = 2.0 if args.quick else 10.0
    print("# NEXT-4: lid-driven cavity on the CUDA path (B200, fp64)\n")
    print(f"PAPER.md:1210-1300 §4.3 set-up: unit square, lid U = 1, h/dx = 1, eps = 1e-2, symm, GTVF with "
          f"p_ref = 2 max p after the first solve (R33), t = {t_end:g} s.  Centreline profiles: particles within "
          f"dx of x = 0.5 (u) / y = 0.5 (v), binned by dx.\n")
    print("| N | Re | u* | eq:convergence | eps | GTVF | steps | mean sweeps | min rho/rho0 | wall s | KE | min u(x=0.5) at y | max v(y=0.5) at x | min v(y=0.5) at x |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|", flush=True)
    plan = [(50, 100.0, 0, {}), (50, 100.0, 1, {}), (50, 100.0, 0, {"conv_mean": 0}),
            (100, 100.0, 0, {}), (100, 100.0, 1, {}), (100, 100.0, 0, {"conv_mean": 0}),
            (100, 100.0, 0, {"tol": 1e-3}), (100, 100.0, 0, {"pref_auto": 0}),
            (100, 10000.0, 0, {}), (100, 10000.0, 0, {"tol": 1e-3})]
    runs = []
    for n, re, noslip, over in plan:
        runs.append(run(n, re, t_end, noslip, **over))
        print(row(runs[-1]), flush=True)
    print("\nProfiles (every 5th bin), 100 x 100, Re = 100, slip u*, means, eps = 1e-3:\n")
    r = [q for q in runs if q["n"] == 100 and q["re"] == 100.0 and q.get("tol") == 1e-3][0]
    if r["status"] != "ok":
        r = {"profile_u": [], "profile_v": []}
    print("| y | u(0.5, y) | x | v(x, 0.5) |")
    print("|---|---|---|---|")
    for (y, uu), (xx, vv) in list(zip(r["profile_u"], r["profile_v"]))[::5]:
        print(f"| {y:.3f} | {uu:.4f} | {xx:.3f} | {vv:.4f} |")
    out = os.path.join(ROOT, "gpurun_out") if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "/tmp"
    with open(os.path.join(out, "cavity.json"), "w") as fh:
        json.dump(runs, fh, indent=1)


if __name__ == "__main__":
    main()
