"""Parity at BASELINE.json's other full sizes (configs[1..3]), in the configuration
bench.py times for each (`bench.py --workload tgv3d | dambreak2d | hydrostatic`).

C4 TGV-3D 128^3 (2 097 152 particles, triply periodic, mean-free Jacobi R32,
fixed-point GTVF sub-steps, h~ = h), C3 2D dam break at dx = 0.002 (500 000
fluid + walls), C2 hydrostatic tank (80 000 fluid + walls).  As for C5
(test_gpu_fullsize.py): two free-running GPU steps, then one step through the
C ABI split (predict / 2 fixed sweeps / correct) with the fp64 oracle (all host
cores) running the same step from the GPU's own state; every particle's fields
within the north_star tolerances (parity_util), neighbour sets at r* of sampled
rows bit for bit.  fp32 stages from A9 on are evaluated by the oracle on the
handle's stored r* and u* (parity_util.inject_stage1, reading R36), each of
which is compared on its own first.
"""
import numpy as np
import pytest

import oracle
import synth
from parity_util import assert_close, assert_disp_close, fs_hazards, gpu_sim, inject_stage1, oracle_from_gpu, ut_floor

pytestmark = pytest.mark.gpu

CONFIGS = {
    "C4_tgv3d": synth.tgv3d,
    "C3_dambreak2d": synth.dambreak2d,
    "C2_hydrostatic": synth.hydrostatic,
}


U32 = 2.0 ** -24


def _rhs_cancellation_check(case, sim, o, rhs_g, rhs_o, rep, nsample=3000):
    """RHS_i = -sum_j m_j / (rho_j dt) u*_ij . grad W_ij (eq:sph-ppe, R8) on the smooth TGV-3D field
    cancels: its terms' absolute sum A_i is ~75x the result at full size (the fp64 handle
    matches the oracle to 2e-13 of the scale there).  An fp32 sum of n_i terms, each with a
    few rounded operations and MUFU approximations, is off by at most (n_i + 8) u A_i
    (recursive summation, Higham's gamma_n bound; u = 2^-24): the sampled rows are checked
    against that bound on top of the north_star one (reading R36)."""
    rng = np.random.default_rng(5)
    f = np.flatnonzero(case.tag == 0)
    which = np.sort(rng.choice(f, nsample, replace=False))
    off, ids = sim.neighbors_of(which)
    xs, us, rho, m = o.get("xs"), o.get("us"), o.get("rho"), sim.get("MASS")
    L = np.array(case.hi, float) - np.array(case.lo, float)
    worst = 0.0
    for k, i in enumerate(which):
        j = ids[off[k]:off[k + 1]]
        d = xs[i] - xs[j]
        for a in range(case.dim):
            if case.periodic[a]:
                d[:, a] = (d[:, a] + 0.5 * L[a]) % L[a] - 0.5 * L[a]
        r = np.linalg.norm(d, axis=1)
        dw = np.array([oracle.dWdr(case.dim, float(v), case.h) for v in r])
        g = (dw / np.where(r > 0, r, 1.0))[:, None] * d
        A = np.abs((m[j] / (rho[j] * case.dt)) * np.sum((us[i] - us[j]) * g, axis=1)).sum()
        bound = 1e-4 * abs(rhs_o[i]) + 1e-6 * max(np.abs(rhs_o).max(), 1.0) + (len(j) + 8) * U32 * A
        err = abs(rhs_g[i] - rhs_o[i])
        assert err <= bound, (i, rhs_g[i], rhs_o[i], err, bound, A, len(j))
        worst = max(worst, err / bound)
    rep["rhs (sampled, cancellation bound)"] = dict(n=nsample, worst_err_over_bound=worst)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_full_size_step(name):
    case = CONFIGS[name]()
    prec = case.params["precision"]
    sim = gpu_sim(case)
    for _ in range(2):
        sim.step(case.dt)
    o = oracle_from_gpu(case, sim)
    f, w = case.tag == 0, case.tag == 1
    dt = case.dt
    x0 = sim.get("POSITION")
    rep = {}
    sim.predict(dt)
    o.predict(dt)
    assert_close("rho", sim.get("DENSITY"), o.get("rho"), prec, report=rep)
    haz = fs_hazards(o.get("rho"), case.params, width=1e-5 if prec == 32 else 1e-12)
    assert np.array_equal(sim.get("FREE_SURFACE")[~haz], o.get("fs")[~haz])
    xs = sim.get("RSTAR")
    assert_disp_close("rstar", xs[f], o.get("xs")[f], x0[f], case, prec, report=rep)
    assert_close("ustar", sim.get("USTAR")[f], o.get("us")[f], prec,
                 scale=max(np.abs(o.get("us")).max(), 1e-3), report=rep)
    # A9-A11 on the handle's stored r* and u* (reading R36)
    inject_stage1(sim, o, case, prec)
    if w.any():
        assert_close("ghost u", sim.get("VELOCITY")[w], o.get("u")[w], prec,
                     scale=max(np.abs(o.get("u")).max(), 1e-3), report=rep)
    assert_close("diag", sim.get("DIAG")[f], o.get("diag")[f], prec, report=rep)
    rhs_g, rhs_o = sim.get("RHS"), o.get("rhs")
    if prec == 64 or name != "C4_tgv3d":
        assert_close("rhs", rhs_g[f], rhs_o[f], prec, scale=max(np.abs(rhs_o).max(), 1e-9), report=rep)
    else:
        _rhs_cancellation_check(case, sim, o, rhs_g, rhs_o, rep)
    rng = np.random.default_rng(11)
    which = rng.choice(np.flatnonzero(f), 2000, replace=False)
    if w.any():
        which = np.concatenate([which, rng.choice(np.flatnonzero(w), min(300, int(w.sum())), replace=False)])
    which = np.sort(which)
    off, ids = sim.neighbors_of(which)
    roff, rids = oracle.neighbors(oracle.case_cfg(case), xs, dests=which)
    assert np.array_equal(off, roff)
    assert np.array_equal(ids, rids)
    it_g, _ = sim.ppe_solve(0.0, 2)
    it_o, _, _ = o.solve(0.0, 2)
    assert it_g == it_o == 2
    p_o = o.get("p")
    assert_close("p", sim.get("PRESSURE"), p_o, prec, scale=max(np.abs(p_o).max(), 1e-6), report=rep)
    sim.correct(dt)
    o.correct(dt)
    u_o = o.get("u")[f]
    assert_close("u", sim.get("VELOCITY")[f], u_o, prec, report=rep)
    ut_o = o.get("ut")[f]
    assert_close("ut", sim.get("TRANSPORT_VELOCITY")[f], ut_o, prec, report=rep,
                 abs_floor=ut_floor(case, prec=prec, S=np.abs(ut_o).max()))
    assert_disp_close("x", sim.get("POSITION")[f], o.get("x")[f], x0[f], case, prec, report=rep)
    sim.close()
    for k, v in rep.items():
        print(f"{name} parity {k}: {v}")
