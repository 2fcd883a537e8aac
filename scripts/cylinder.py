#!/usr/bin/env python
"""NEXT-4's validation case on the CUDA path: flow past a circular cylinder at Re = 200
(§4.7; synth.cylinder: D = 2, dx = D/30, h/dx = 1.2, inlet 5D upstream, outlet
10D behind the centre, eps = 0.01, symm, external GTVF with p_ref = rho (10 U)^2; reading R35: a
periodic y of width 15D instead of the slip side walls).

The force on the cylinder is the paper's eq:tvf-momentum, summed over the cylinder's
wall particles i and their fluid neighbours j within 3h (host-side post-processing of the fields the
C ABI returns; not part of the hot path):
    f_i = sum_j (V_i^2 + V_j^2) [ -p~_ij gradW_ij + eta~_ij u_ij / (r^2 + eta h^2) (gradW_ij . r_ij) ]
    p~_ij = (rho_j p_i + rho_i p_j) / (rho_i + rho_j), eta~_ij = 2 eta_i eta_j / (eta_i + eta_j),
    u_ij = u_w,i - u_j (the wall's ghost velocity), eta = rho nu
c_d = 2 F_x / (rho U^2 D), c_l = 2 F_y / (rho U^2 D).  The paper reports a mean c_d = 1.609 once
shedding is established and a maximum c_l = 0.804.

    python scripts/cylinder.py [--ppd 30] [--t-end 200] > profiles/r1_cylinder.md
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1908_01762_b200 import Simulation  # noqa: E402


def dwdr(r, h):
    """quintic spline (R1) derivative, 2D: -5 sigma / h^3 [(3-q)^4 - 6(2-q)^4 + 15(1-q)^4]_+"""
    q = r / h
    s = 7.0 / (478.0 * np.pi)
    t = np.maximum(3 - q, 0) ** 4 - 6 * np.maximum(2 - q, 0) ** 4 + 15 * np.maximum(1 - q, 0) ** 4
    return -5.0 * s / h ** 3 * t


def cylinder_force(case, sim, cyl):
    """eq:tvf-momentum summed over the cylinder's wall particles (ids `cyl`)"""
    x, u, p, rho, tag = (sim.get(f) for f in ("POSITION", "VELOCITY", "PRESSURE", "DENSITY", "TAG"))
    m = case.m
    h = case.h
    nu = case.params["nu"]
    eta_reg = case.params["eta"] * h * h
    xc = np.array([case.params["x_inlet"] + 0.0, 0.0])
    fl = np.flatnonzero(tag == 0)
    cx = x[cyl].mean(0)
    near = fl[np.sum((x[fl] - cx) ** 2, 1) < (0.5 * 2.0 + 3 * h + 0.1) ** 2 * 1.5]
    F = np.zeros(2)
    for i in cyl:
        d = x[i] - x[near]                               # r_ij = r_i - r_j
        r = np.sqrt(np.sum(d * d, 1))
        k = r < 3 * h
        j = near[k]
        d, r = d[k], r[k]
        gw = (dwdr(r, h) / np.maximum(r, 1e-300))[:, None] * d
        Vi, Vj = m[i] / rho[i], m[j] / rho[j]
        pt = (rho[j] * p[i] + rho[i] * p[j]) / (rho[i] + rho[j])
        ei, ej = rho[i] * nu, rho[j] * nu
        et = 2 * ei * ej / (ei + ej)
        uij = u[i] - u[j]
        rg = np.sum(gw * d, 1)
        fi = (Vi * Vi + Vj * Vj)[:, None] * (-pt[:, None] * gw + (et * rg / (r * r + eta_reg))[:, None] * uij)
        F += fi.sum(0)
    del xc
    return F


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ppd", type=int, default=30)
    ap.add_argument("--t-end", type=float, default=200.0)
    ap.add_argument("--every", type=float, default=0.5)
    ap.add_argument("--max-wall", type=float, default=1200.0, help="stop after this many seconds")
    ap.add_argument("--set", nargs="*", default=[], help="parameter overrides key=value")
    args = ap.parse_args()
    case = synth.cylinder(ppd=args.ppd, t_end=args.t_end)
    for kv in args.set:
        k, v = kv.split("=")
        case.params[k] = float(v) if ("." in v or "e" in v) else int(v)
    sim = Simulation.from_case(case)
    cyl = np.flatnonzero(case.tag == 1)
    D, U = 2.0, 1.0
    t, hist, its = 0.0, [], []
    t0 = time.perf_counter()
    status = "ok"
    k_every = max(1, int(round(args.every / case.dt)))
    try:
        for k in range(case.steps):
            if time.perf_counter() - t0 > args.max_wall:
                status = f"stopped at the wall-clock limit ({args.max_wall:g} s)"
                break
            its.append(sim.step(case.dt).iters)
            t += case.dt
            if (k + 1) % k_every == 0:
                F = cylinder_force(case, sim, cyl)
                cd, cl = 2 * F[0] / (U * U * D), 2 * F[1] / (U * U * D)
                tags = sim.get("TAG")
                hist.append((t, cd, cl, int((tags == 0).sum()), float(np.mean(its[-k_every:]))))
                print(f"t={t:7.2f} cd={cd:8.4f} cl={cl:8.4f} fluid={hist[-1][3]} sweeps={hist[-1][4]:.1f}",
                      file=sys.stderr, flush=True)
    except Exception as e:  # noqa: BLE001
        status = f"stopped at t = {t:.2f}: {e}"
    wall = time.perf_counter() - t0
    h = np.array([r[:3] for r in hist]) if hist else np.zeros((0, 3))
    print("# Flow past a cylinder, Re = 200, on the CUDA path (B200, fp64)\n")
    print(f"D = 2, dx = D/{args.ppd}, h/dx = 1.2, {int((case.tag == 0).sum())} fluid particles at start, "
          f"dt = {case.dt:.4g}, {len(its)} steps to t = {t:.1f} s in {wall:.0f} s wall; status: {status}\n")
    late = h[h[:, 0] >= 0.5 * args.t_end] if len(h) else h
    if len(late):
        print(f"mean c_d over t >= {0.5 * args.t_end:g} s: {late[:, 1].mean():.3f} (paper: 1.609); "
              f"max |c_l|: {np.abs(late[:, 2]).max():.3f} (paper: 0.804); mean sweeps/step "
              f"{np.mean(its):.2f}\n")
    print("| t | c_d | c_l | fluid | sweeps/step |")
    print("|---|---|---|---|---|")
    for r in hist[:: max(1, len(hist) // 40)]:
        print(f"| {r[0]:.1f} | {r[1]:.4f} | {r[2]:.4f} | {r[3]} | {r[4]:.1f} |")


if __name__ == "__main__":
    main()
