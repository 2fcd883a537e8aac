#!/usr/bin/env python
"""The fp64 C oracle timed per BASELINE config on the host's cores (SURVEY.md §8(d) "Oracle
timing"): whole SISPH steps, PPE particle-sweeps/s and s/step, next to the CUDA path's numbers
(which bench.py / profiles report).

    python scripts/oracle_timing.py > profiles/r1_oracle_timing.md
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: timing the baseline is one of its allowed uses)
import synth  # noqa: E402

CASES = [
    ("C1 tgv2d 50^2 fp64 (eps 1e-4)", lambda: synth.tgv2d(), 10),
    ("C2 hydrostatic 200x400 (eps 1e-3)", lambda: synth.hydrostatic(precision=64), 5),
    ("C3 dam break 2D 500x1000 (eps 1e-2)", lambda: synth.dambreak2d(precision=64), 2),
    ("C4 TGV-3D 128^3 (eps 1e-3)", lambda: synth.tgv3d(precision=64), 1),
    ("C5 dam break 3D per-GPU slab (eps 1e-2)", lambda: synth.dambreak3d(precision=64), 1),
]


def main():
    cores = os.cpu_count()
    print(f"# fp64 C oracle on the host ({cores} logical cores, OpenMP over destination particles)\n")
    print("| config | fluid particles | steps | sweeps/step | s per step | PPE particle-sweeps/s |")
    print("|---|---|---|---|---|---|")
    for name, mk, steps in CASES:
        case = mk()
        s = oracle.Sim(case)
        t0 = time.perf_counter()
        sw = 0
        for _ in range(steps):
            sw += s.step(case.dt)[0]
        t = time.perf_counter() - t0
        nf = case.n_fluid
        print(f"| {name} | {nf} | {steps} | {sw / steps:.1f} | {t / steps:.3f} | {sw * nf / t:.3g} |", flush=True)
        del s


if __name__ == "__main__":
    main()
