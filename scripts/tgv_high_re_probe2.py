import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/scripts")
import synth
from paper_1908_01762_b200 import Simulation
from variants import tgv_error
def run(re, n, label, **over):
    case = synth.tgv2d(n=n, re=re)
    sim = Simulation.from_case(case, **over)
    t = 0.0; out = []
    for t_end in (0.1, 0.25, 0.5, 1.0):
        while t < t_end - 1e-9:
            sim.step(case.dt); t += case.dt
        out.append(tgv_error(sim, case, t))
    print(f"Re {re:6g} n {n} {label:34s}", " ".join(f"t={tt}: {e:.3f}/{d:.2f}" for tt, (e, d) in zip((0.1,0.25,0.5,1.0), out)), flush=True)
    sim.close()
for re in (100.0, 1000.0, 10000.0):
    run(re, 100, "pref 0 (no GTVF, no astress)", p_ref=0.0)
    run(re, 100, "pref 2maxp K10", )
    run(re, 100, "pref 2maxp K10 tol1e-4", tol=1e-4)
    run(re, 100, "pref 0.1 K10", p_ref=0.1)
run(10000.0, 100, "pref 0 EISPH", p_ref=0.0, max_iter=1, min_iter=1)
run(10000.0, 100, "pref 0 unjittered", p_ref=0.0)
