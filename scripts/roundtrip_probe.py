"""Does get_field/set_field of (POSITION, VELOCITY, TRANSPORT_VELOCITY, PRESSURE) capture the state a
step starts from?  From one state: (a) step; (b) round-trip the four fields through host, then step.
Prints the PPE sweep counts and the max pressure difference of the two results."""
import sys
sys.path.insert(0, ".")
import numpy as np
import synth
from paper_1908_01762_b200 import Simulation


def run(case, nwarm, f32):
    out = []
    for rt in (False, True):
        sim = Simulation.from_case(case)
        for _ in range(nwarm):
            sim.step(case.dt)
        if rt:
            st = {k: sim.get(k) for k in ("POSITION", "VELOCITY", "TRANSPORT_VELOCITY", "PRESSURE")}
            for k, v in st.items():
                sim.set(k, v)
        r = sim.step(case.dt)
        out.append((r.iters, sim.get("PRESSURE")))
        sim.close()
    (ia, pa), (ib, pb) = out
    print(f"{case.name if hasattr(case, 'name') else ''} warm {nwarm}: sweeps direct {ia}, after round trip {ib}, "
          f"max |dp| {np.abs(pa - pb).max():.3e} (max |p| {np.abs(pa).max():.3e})", flush=True)


for n in (3, 10):
    run(synth.tgv3d(n=32), n, True)
    run(synth.dambreak2d(nx=100, ny=200), n, True)
    run(synth.hydrostatic(), n, False)
