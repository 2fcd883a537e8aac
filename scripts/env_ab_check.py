"""A/B bit-identity check of an engine switch read from the environment at create:
    python scripts/env_ab_check.py SISPH_FUSED
runs each case with VAR=0 and VAR=1 for 5 steps and compares positions, velocities, pressures."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1908_01762_b200 import Simulation  # noqa: E402

var = sys.argv[1]
cases = {
    "db3d_f32": lambda: synth.dambreak3d(nfx=48, nfy=16, nfz=24, dx=1.0 / 64, tank_nx=120, wall_nz=30),
    "db3d_f64": lambda: synth.dambreak3d(nfx=24, nfy=10, nfz=12, dx=1.0 / 32, tank_nx=60, wall_nz=16, precision=64),
    "tgv2d": lambda: synth.tgv2d(),
    "db2d": lambda: synth.dambreak2d(nx=50, ny=100, dx=0.02),
    "tgv3d": lambda: synth.tgv3d(n=24),
    "cavity": lambda: synth.cavity(n=40),
    "channel": lambda: synth.channel(),
}
bad = 0
for name, mk in cases.items():
    out = {}
    for flag in ("0", "1"):
        os.environ[var] = flag
        case = mk()
        sim = Simulation.from_case(case)
        its = [sim.step(case.dt).iters for _ in range(5)]
        out[flag] = {f: sim.get(f) for f in ("POSITION", "VELOCITY", "PRESSURE", "TRANSPORT_VELOCITY")}
        out[flag]["its"] = np.array(its)
        sim.close()
    same = all(np.array_equal(out["0"][f], out["1"][f]) for f in out["0"])
    diff = max(float(np.abs(out["0"][f] - out["1"][f]).max()) for f in out["0"])
    print(f"{name:10s} bit-identical {same}  max diff {diff:.3e}", flush=True)
    bad += not same
sys.exit(1 if bad else 0)
