"""C4 (TGV-3D 128^3) RHS at full size: fp64 handle vs oracle, and the fp32 handle's RHS error
against the cancellation A_i = sum_j |m_j/(rho_j dt) u*_ij . grad W_ij| of sampled rows."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle, synth
from parity_util import gpu_sim, oracle_from_gpu, inject_stage1

for prec in (64, 32):
    case = synth.tgv3d(precision=prec)
    sim = gpu_sim(case)
    for _ in range(2):
        sim.step(case.dt)
    o = oracle_from_gpu(case, sim)
    sim.predict(case.dt); o.predict(case.dt)
    inject_stage1(sim, o, case, prec)
    rg, ro = sim.get("RHS"), o.get("rhs")
    e = np.abs(rg - ro)
    print(prec, "rhs max|ref|", np.abs(ro).max(), "max err", e.max(), "max rel err", (e / np.maximum(np.abs(ro), 1e-30)).max())
    rng = np.random.default_rng(3)
    which = np.sort(rng.choice(case.x.shape[0], 3000, replace=False))
    off, ids = sim.neighbors_of(which)
    xs, us, rho, m = o.get("xs"), o.get("us"), o.get("rho"), o.get("m") if False else sim.get("MASS")
    L = case.hi[0] - case.lo[0]
    A = np.zeros(len(which)); R = np.zeros(len(which))
    for k, i in enumerate(which):
        j = ids[off[k]:off[k + 1]]
        d = xs[i] - xs[j]
        d = (d + 0.5 * L) % L - 0.5 * L
        r = np.linalg.norm(d, axis=1)
        g = np.array([oracle.dWdr(3, float(v), case.h) for v in r])[:, None] * d / np.where(r > 0, r, 1)[:, None]
        t = -(m[j] / (rho[j] * case.dt)) * np.sum((us[i] - us[j]) * g, axis=1)
        A[k] = np.abs(t).sum(); R[k] = t.sum()
    print(prec, "sample: recomputed-vs-oracle max", np.abs(R - ro[which]).max(), "A/|rhs| median", np.median(A / np.maximum(np.abs(ro[which]), 1e-30)),
          "max err/(eps32*A)", (e[which] / (2.0 ** -24 * A)).max(), "median", np.median(e[which] / (2.0 ** -24 * A)))
    sim.close()
