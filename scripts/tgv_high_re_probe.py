import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/scripts")
import synth
from paper_1908_01762_b200 import Simulation
from variants import tgv_error
for pref in (1.0, 10.0, 100.0):
    for label, over in (("SISPH 1e-2", dict(tol=1e-2)), ("EISPH", dict(max_iter=1, min_iter=1))):
        case = synth.tgv2d(n=100, re=10000.0)
        for K in (10, 1):
            sim = Simulation.from_case(case, p_ref=pref, K=K, **over)
            res = []
            for t_end in (0.25, 0.5, 1.0):
                while True:
                    sim.step(case.dt)
                    res_t = getattr(sim, "_t", 0.0) + case.dt
                    sim._t = res_t
                    if res_t >= t_end - 1e-9: break
                res.append(tgv_error(sim, case, sim._t))
            print(f"pref {pref:6g} K {K:2d} {label:10s}", " ".join(f"t={t:.2f}: L1 {e:.4f} dec {d:.3f}" for t, (e, d) in zip((0.25,0.5,1.0), res)), flush=True)
            sim.close()
