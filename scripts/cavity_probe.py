#!/usr/bin/env python
"""Lid-driven cavity stability probe (which switch keeps 100 x 100, Re = 100 alive).

    python scripts/cavity_probe.py
Prints, per variant, KE / min rho / free-surface count / mean sweeps at t = 0.5, 1, 2, 5, 10.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1908_01762_b200 import Simulation  # noqa: E402

T_OUT = (0.5, 1.0, 2.0, 5.0, 10.0)


def probe(label, n=100, re=100.0, **over):
    case = synth.cavity(n=n, re=re, t_end=10.0)
    case.params.update(over)
    sim = Simulation.from_case(case)
    f = case.tag == 0
    t, k, its, out = 0.0, 0, [], []
    try:
        for te in T_OUT:
            while t < te - 1e-9:
                its.append(sim.step(case.dt).iters)
                t += case.dt
            u = sim.get("VELOCITY")[f]
            rho = sim.get("DENSITY")[f]
            fs = int(sim.get("FREE_SURFACE")[f].sum())
            ke = 0.5 * float(np.sum(case.m[f] * np.sum(u * u, 1)))
            out.append(f"t={te:g}: KE {ke:.4f} rho_min {rho.min():.3f} fs {fs} sw {np.mean(its[-100:]):.1f}")
    except Exception as e:  # noqa: BLE001
        out.append(f"failed at t={t:.3f}: {e}")
    sim.close()
    print(f"{label:40s} | " + " | ".join(out), flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "htilde":
    probe("base (h~ = h)")
    probe("h~ = h/2", h_tilde_factor=0.5)
    probe("h~ = h/2, sums", h_tilde_factor=0.5, conv_mean=0)
    probe("h~ = h/2, tol 1e-3", h_tilde_factor=0.5, tol=1e-3)
    probe("h~ = h/2, no-slip u*", h_tilde_factor=0.5, ustar_noslip=1)
    probe("h~ = h/2, Re 10^4", re=10000.0, h_tilde_factor=0.5)
    sys.exit(0)
if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    probe("base (slip, means, GTVF 2max p)")
    probe("no GTVF (p_ref 0, no auto)", pref_auto=0, p_ref=0.0)
    probe("K = 1", K=1)
    probe("mean-free PPE", ppe_mean_free=1)
    probe("clamp wall p", clamp_wall_p=1)
    probe("wall rho summation", wall_rho_summation=1)
    probe("alpha 0.1 (c_ref 10)", alpha=0.1, c_ref=10.0)
    probe("tol 1e-3", tol=1e-3)
    probe("asymm", pgrad=1)
    probe("p_ref 1 fixed", pref_auto=0, p_ref=1.0)
    probe("p_ref 10 fixed", pref_auto=0, p_ref=10.0)
    probe("50x50 base", n=50)
