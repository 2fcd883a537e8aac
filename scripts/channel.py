#!/usr/bin/env python
"""NEXT-4b (open boundaries, reading R34) on the CUDA path: plane channel with a
parabolic inlet and a do-nothing outlet, started from the developed profile.  Reports the
profile error against u = 6 U y (H - y) / H^2 in the middle third of the channel, the particle
census (fluid / inlet / outlet / dormant) and the pressure drop, over time.

    python scripts/channel.py > profiles/r1_channel.md
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1908_01762_b200 import Simulation  # noqa: E402


def run(ny, nx, re, t_out, precision=64):
    case = synth.channel(nx=nx, ny=ny, re=re, n_pool=4 * 4 * ny, precision=precision)
    sim = Simulation.from_case(case)
    H, Lf = 1.0, nx / ny
    t, its, rows = 0.0, [], []
    t0 = time.perf_counter()
    for te in t_out:
        while t < te - 1e-9:
            its.append(sim.step(case.dt).iters)
            t += case.dt
        tag, x, u, p = sim.get("TAG"), sim.get("POSITION"), sim.get("VELOCITY"), sim.get("PRESSURE")
        f = tag == 0
        sel = f & (x[:, 0] > Lf / 3) & (x[:, 0] < 2 * Lf / 3)
        err = np.abs(u[sel, 0] - synth.poiseuille_velocity(x[sel, 1], 1.0, H))
        # pressure gradient along the channel vs the Poiseuille value -12 nu U / H^2 (rho = 1)
        A = np.stack([x[sel, 0], np.ones(sel.sum())], 1)
        dpdx = np.linalg.lstsq(A, p[sel], rcond=None)[0][0]
        census = [int((tag == k).sum()) for k in (0, 2, 3, 4)]
        rows.append((te, np.mean(its[-50:]), err.mean(), err.max(), dpdx, census, time.perf_counter() - t0))
    sim.close()
    return case, rows


def main():
    print("# NEXT-4b: channel with inlet / outlet on the CUDA path (B200, fp64)\n")
    print("Developed plane channel (Re = U H / nu), parabolic inlet (tag 2), do-nothing outlet (tag 3, u and p "
          "frozen, advected with the extrapolated fluid u_x), dormant id pool (tag 4); started from the closed "
          "form.  Error of u_x against 6 U y (H - y) / H^2 over the middle third; dp/dx by least squares "
          "(Poiseuille: -12 nu U / H^2).\n")
    print("| particles across | length / H | Re | t | sweeps/step | mean err / U | max err / U | dp/dx | exact dp/dx "
          "| fluid / inlet / outlet / dormant | wall s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for ny, nx, re in ((10, 40, 10.0), (20, 80, 10.0), (40, 160, 10.0), (20, 80, 100.0)):
        case, rows = run(ny, nx, re, (1.0, 2.0, 5.0, 10.0))
        exact = -12.0 * case.params["nu"] * 1.0
        for te, sw, em, ex, g, cen, w in rows:
            print(f"| {ny} | {nx / ny:g} | {re:g} | {te:g} | {sw:.1f} | {em:.4f} | {ex:.4f} | {g:.3f} | {exact:.3f} | "
                  f"{' / '.join(map(str, cen))} | {w:.1f} |", flush=True)


if __name__ == "__main__":
    main()
