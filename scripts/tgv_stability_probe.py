"""TGV-2D long-run stability matrix (PAPER.md:1034-1110 settings): resolution, tolerance,
pressure-gradient form, background pressure; L1 error / max|u| over exp(bt) at several t."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import synth
from paper_1908_01762_b200 import Simulation
from variants import tgv_error
T_OUT = (0.25, 0.5, 1.0, 2.0, 5.0)
def run(n, label, re=100.0, **over):
    case = synth.tgv2d(n=n, re=re)
    sim = Simulation.from_case(case, **over)
    t, out, its = 0.0, [], 0
    for t_end in T_OUT:
        while t < t_end - 1e-9:
            its += sim.step(case.dt).iters
            t += case.dt
        out.append(tgv_error(sim, case, t))
    steps = round(t / case.dt)
    print(f"n {n:3d} Re {re:5g} {label:28s} sweeps/step {its / steps:7.1f} |",
          " ".join(f"t={tt}: {e:.3f}/{d:.2f}" for tt, (e, d) in zip(T_OUT, out)), flush=True)
    sim.close()
if __name__ != "__main__":
    pass
elif len(sys.argv) > 1 and sys.argv[1] == "re10k":
    # EISPH vs SISPH at Re = 10^4 with the stable GTVF / PPE settings (R22c, R32)
    st = dict(h_tilde_factor=0.5, ppe_mean_free=1)
    run(100, "SISPH tol 1e-2 h~=h/2 mean-free", re=10000.0, tol=1e-2, **st)
    run(100, "SISPH tol 1e-3 h~=h/2 mean-free", re=10000.0, tol=1e-3, **st)
    run(100, "EISPH (1 sweep) h~=h/2 mean-free", re=10000.0, max_iter=1, min_iter=1, **st)
    run(100, "SISPH tol 1e-2 h~=h (printed)", re=10000.0, tol=1e-2)
elif len(sys.argv) > 1 and sys.argv[1] == "htilde":
    # the GTVF kernel length: h~ = h (the paper's internal-flow choice) pairs particles on an
    # h/dx = 1 lattice; h~ = h/2 with the mean-free PPE (R32), over the paper's tolerance range
    for tol in (0.1, 0.05, 1e-2, 5e-3, 1e-3, 5e-4, 1e-4):
        run(100, f"asymm tol {tol:g} h~=h/2 mean-free", tol=tol, h_tilde_factor=0.5, ppe_mean_free=1)
    run(100, "asymm tol 0.0001 h~=h mean-free", tol=1e-4, ppe_mean_free=1)
    run(100, "asymm tol 0.0001 h~=h/2 printed", tol=1e-4, h_tilde_factor=0.5)
elif len(sys.argv) > 1 and sys.argv[1] == "meanfree":
    # reading R32: the same tolerance study with the live-row mean removed every sweep
    for tol in (1e-2, 1e-3, 1e-4):
        run(100, f"asymm tol {tol:g} as printed", tol=tol)
        run(100, f"asymm tol {tol:g} mean-free", tol=tol, ppe_mean_free=1)
elif len(sys.argv) > 1 and sys.argv[1] == "tol":
    # the paper's tolerance study: 100 x 100, asymm + GTVF
    for tol in (0.1, 0.05, 1e-2, 5e-3, 1e-3, 5e-4, 2e-4, 1e-4):
        run(100, f"asymm pref=1 tol {tol:g}", tol=tol)
else:
  for n in (50, 100):
    for tol in (1e-2, 1e-4):
        run(n, f"asymm pref=1 tol {tol:g}", tol=tol)
        run(n, f"symm  pref=1 tol {tol:g}", tol=tol, pgrad=0)
        run(n, f"symm  pref=0 tol {tol:g}", tol=tol, pgrad=0, p_ref=0.0)
        run(n, f"asymm pref=0 tol {tol:g}", tol=tol, p_ref=0.0)
if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "pref":
    for n in (50, 100):
        for pref in (1.0, 10.0, 100.0):
            for tol in (1e-2, 1e-3):
                run(n, f"asymm pref={pref:g} tol {tol:g}", tol=tol, p_ref=pref)
