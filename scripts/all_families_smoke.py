"""A few steps of every workload family and PPE-loop form on the CUDA path, small sizes
(meant to run under compute-sanitizer where that is available; this build's GPU pool disables it).

    python scripts/all_families_smoke.py
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1908_01762_b200 import LocalGroup, Simulation, make_dist  # noqa: E402

cases = [
    ("tgv2d", synth.tgv2d(n=24), {}),
    ("tgv2d_graph", synth.tgv2d(n=24), {"ppe_loop": 2}),
    ("tgv2d_persist", synth.tgv2d(n=24), {"ppe_loop": 3}),
    ("tgv2d_meanfree", synth.tgv2d(n=24), {"ppe_mean_free": 1}),
    ("hydro", synth.hydrostatic(nx=20, ny=40, dx=0.05, precision=64), {}),
    ("db2d", synth.dambreak2d(nx=30, ny=60, dx=0.0333333, precision=32), {}),
    ("db3d", synth.dambreak3d(nfx=16, nfy=10, nfz=12, dx=1.0 / 32, tank_nx=40, wall_nz=16), {}),
    ("tgv3d", synth.tgv3d(n=14, precision=64), {"matrix_free": 1}),
    ("cavity", synth.cavity(n=20), {}),
    ("channel", synth.channel(nx=20, ny=8), {}),
    ("square", synth.square_patch(n=30), {}),
]
for name, case, over in cases:
    sim = Simulation.from_case(case, **over)
    for _ in range(3):
        sim.step(case.dt)
    sim.get("PRESSURE")
    sim.close()
    print(name, "ok", flush=True)

# two emulated slab ranks
case = synth.tgv2d(n=24)
g = LocalGroup(2)
errs = []


def work(r):
    try:
        s = Simulation.from_case(case, dist=make_dist(2, r, 0, local_group=g))
        for _ in range(3):
            s.step(case.dt)
        s.close()
    except Exception as e:  # noqa: BLE001
        errs.append(e)


th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
g.close()
print("slab ranks", "ok" if not errs else errs, flush=True)
