"""Debug: slab ranks vs single handle, stage by stage (predict, sweeps, correct)."""
import sys, threading
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import synth
from paper_1908_01762_b200 import LocalGroup, Simulation, make_dist

name = sys.argv[1] if len(sys.argv) > 1 else "tgv2d"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 2
axis = int(sys.argv[3]) if len(sys.argv) > 3 else 0
case = {"tgv2d": lambda: synth.tgv2d(),
        "db3d": lambda: synth.dambreak3d(nfx=16, nfy=10, nfz=12, dx=1.0 / 32, tank_nx=40, wall_nz=16, precision=64),
        "db2d": lambda: synth.dambreak2d(nx=30, ny=60, dx=0.0333333, precision=64)}[name]()
single = Simulation.from_case(case)
g = LocalGroup(R)
sims = [None] * R
bar = threading.Barrier(R + 1)
cmds = []
res = [None] * R

def work(r):
    s = Simulation.from_case(case, dist=make_dist(R, r, axis, local_group=g))
    sims[r] = s
    bar.wait()
    while True:
        bar.wait()
        c = cmds[-1]
        if c is None:
            return
        res[r] = c(s)
        bar.wait()

th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(R)]
for t in th: t.start()
bar.wait()

def run(c):
    cmds.append(c); bar.wait(); bar.wait()
    return list(res)

def cmp(fld, mask=None):
    a = sum(s.get(fld) for s in sims); b = single.get(fld)
    if mask is not None: a, b = a[mask], b[mask]
    d = np.abs(a - b)
    i = np.unravel_index(np.argmax(d), d.shape)
    print(f"{fld:20s} max|d| {d.max():.3e} max|ref| {np.abs(b).max():.3e} at {i} a={a[i]:.6g} b={b[i]:.6g}")

print("owned", run(lambda s: s.owned_counts()), "n_fluid", case.n_fluid)
f = case.tag == 0
cmp("POSITION"); cmp("VELOCITY"); cmp("PRESSURE")
single.predict(case.dt); run(lambda s: s.predict(case.dt))
for fld in ("DENSITY", "RSTAR", "USTAR", "DIAG", "RHS", "FREE_SURFACE"):
    cmp(fld, f if fld in ("RSTAR",) else None)
if (case.tag == 1).any():
    cmp("VELOCITY", case.tag == 1)
for k in range(1, 4):
    it1 = single.ppe_solve(0.0, k)
    # re-predict both for a fresh solve of k sweeps
    single.predict(case.dt)
print("solve 1 sweep")
single2 = Simulation.from_case(case)
single2.predict(case.dt)
print(single2.ppe_solve(0.0, 1), run(lambda s: s.ppe_solve(0.0, 1)))
a = sum(s.get("PRESSURE") for s in sims); b = single2.get("PRESSURE")
d = np.abs(a - b); print("p after 1 sweep max|d|", d.max(), "max|p|", np.abs(b).max(), "worst ids", np.argsort(-d)[:8])
print("x of worst", case.x[np.argsort(-d)[:4]])
cmds.append(None); bar.wait()
