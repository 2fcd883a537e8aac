"""GPU (libsisph.so, sm_100a) vs the fp64 oracle, on identical seeded inputs.

Every call goes through the C ABI (ctypes binding).  Discrete results (cell
order, neighbour sets, sweep counts) must be bit-exact; fields must be within
the north_star tolerances (parity_util.TOL).
"""
import numpy as np
import pytest

import oracle
import synth
from parity_util import (assert_close, assert_disp_close, fs_hazards, gpu_sim, inject_rstar, oracle_from_gpu,
                         resync, small_cases, ut_floor, wrap_delta)

pytestmark = pytest.mark.gpu

CASES = small_cases()


def _prec(case):
    return case.params["precision"]


# ------------------------------------------------------------------ A1-A4
@pytest.mark.parametrize("name", list(CASES))
def test_cell_order_is_the_stable_sort(name):
    case = CASES[name]
    sim = gpu_sim(case)
    nf = case.n_fluid
    cfg = oracle.case_cfg(case)
    x = sim.get("POSITION")
    # walls: sorted once at create, stable in creation order
    order0 = sim.order()
    wid = np.flatnonzero(case.tag == 1)
    if wid.size:
        o, _ = oracle.cell_order(cfg, x[wid])
        assert np.array_equal(order0[nf:], wid[o])
    # move the fluid, rebuild: new order = stable sort of the CURRENT order by key
    rng = np.random.default_rng(3)
    x2 = x.copy()
    f = case.tag == 0
    x2[f] += rng.uniform(-0.7, 0.7, (nf, case.dim)) * case.h
    for a in range(case.dim):
        if case.periodic[a]:
            L = case.hi[a] - case.lo[a]
            x2[:, a] = np.where(x2[:, a] >= case.hi[a], x2[:, a] - L, x2[:, a])
            x2[:, a] = np.where(x2[:, a] < case.lo[a], x2[:, a] + L, x2[:, a])
    sim.set("POSITION", x2)
    x2 = sim.get("POSITION")            # precision-rounded
    cur = sim.order()[:nf]
    sim.build_neighbors()
    new = sim.order()
    o, keys = oracle.cell_order(cfg, x2[cur])
    assert np.array_equal(new[:nf], cur[o])
    assert np.array_equal(new[nf:], order0[nf:])


# ------------------------------------------------------------------ A5
@pytest.mark.parametrize("name", list(CASES))
def test_neighbor_sets_bit_exact(name):
    case = CASES[name]
    sim = gpu_sim(case)
    x = sim.get("POSITION")
    off, ids = sim.neighbors()
    roff, rids = oracle.neighbors(oracle.case_cfg(case), x)
    assert np.array_equal(off, roff)
    assert np.array_equal(ids, rids)


def test_neighbor_sets_with_exact_ties_fp64():
    # hydrostatic lattice: every lattice pair at exactly 3h is a tie and must be excluded
    case = synth.hydrostatic(nx=30, ny=30, dx=0.02, precision=64)
    sim = gpu_sim(case)
    off, ids = sim.neighbors()
    roff, rids = oracle.neighbors(oracle.case_cfg(case), sim.get("POSITION"))
    assert np.array_equal(off, roff) and np.array_equal(ids, rids)
    interior = np.diff(off)[(case.tag == 0)]
    assert np.median(interior) == 24


def _moving(case, frac=0.4, seed=5):
    """Transport velocities of |u~| ~ frac h / dt on the fluid: a skin of ~2 frac h."""
    rng = np.random.default_rng(seed)
    ut = np.zeros((case.n, case.dim))
    f = case.tag == 0
    ut[f] = rng.uniform(-1, 1, (f.sum(), case.dim)) * frac * case.h / case.dt / np.sqrt(case.dim)
    return ut


@pytest.mark.parametrize("name", list(CASES))
def test_rstar_sets_of_the_single_build(name):
    """A9 by the single build (R3): the r* sets filtered out of the loose r^n
    list equal the oracle's exact sets at r*, bit for bit."""
    case = CASES[name]
    sim = gpu_sim(case)
    sim.set("TRANSPORT_VELOCITY", _moving(case))
    sim.predict(case.dt)
    xs = sim.get("RSTAR")
    off, ids = sim.neighbors()
    roff, rids = oracle.neighbors(oracle.case_cfg(case), xs)
    assert np.array_equal(off, roff)
    assert np.array_equal(ids, rids)


@pytest.mark.parametrize("name", ["tgv2d_f64", "db2d_f64", "tgv3d_f64", "db3d_f64", "db3d_f32"])
def test_single_build_equals_two_builds(name):
    case = CASES[name]
    a, b = gpu_sim(case), gpu_sim(case, rebuild_mode=1)
    # db3d_f64's periodic y axis has 3.3 cells of 3h: only a thin skin keeps 3 cells
    ut = _moving(case, 0.05 if name == "db3d_f64" else 0.3)
    for s in (a, b):
        s.set("TRANSPORT_VELOCITY", ut)
    x0 = b.get("POSITION")
    ra, rb = a.step(case.dt), b.step(case.dt)
    assert ra.single_build == 1 and rb.single_build == 0
    assert ra.iters == rb.iters and ra.pairs == rb.pairs
    prec = _prec(case)
    for fld in ("PRESSURE", "VELOCITY", "TRANSPORT_VELOCITY"):
        assert_close(fld, a.get(fld), b.get(fld), prec)
    assert_disp_close("POSITION", a.get("POSITION"), b.get("POSITION"), x0, case, prec)


# ------------------------------------------------------------------ A6-A11
@pytest.mark.parametrize("name", list(CASES))
def test_predict_parity(name):
    case = CASES[name]
    prec = _prec(case)
    sim = gpu_sim(case)
    o = oracle_from_gpu(case, sim)
    f, w = case.tag == 0, case.tag == 1
    if w.any():
        assert_close("normal", sim.get("NORMAL")[w], o.get("normal")[w], prec, scale=1.0)
    x0 = sim.get("POSITION")
    sim.predict(case.dt)
    o.predict(case.dt)
    rho_o = o.get("rho")
    assert_close("rho", sim.get("DENSITY"), rho_o, prec)
    # free-surface flags: exact, except hazards within 1e-6 of the threshold (counted)
    haz = fs_hazards(rho_o, case.params)
    assert np.array_equal(sim.get("FREE_SURFACE")[~haz], o.get("fs")[~haz])
    assert_disp_close("rstar", sim.get("RSTAR")[f], o.get("xs")[f], x0[f], case, prec)
    inject_rstar(sim, o, case, prec)
    assert_close("ustar", sim.get("USTAR"), o.get("us"), prec)
    if w.any():
        assert_close("ghost u", sim.get("VELOCITY")[w], o.get("u")[w], prec,
                     scale=max(np.abs(o.get("u")).max(), 1e-3))
    assert_close("diag", sim.get("DIAG")[f], o.get("diag")[f], prec)
    assert_close("rhs", sim.get("RHS")[f], o.get("rhs")[f], prec, scale=max(np.abs(o.get("rhs")).max(), 1e-9))


# ------------------------------------------------------------------ A12
@pytest.mark.parametrize("name", [n for n in CASES if n.endswith("f64")])
def test_solve_parity_fp64_iteration_count(name):
    case = CASES[name]
    sim = gpu_sim(case)
    o = oracle_from_gpu(case, sim)
    sim.predict(case.dt)
    o.predict(case.dt)
    tol, mx = case.params["tol"], case.params["max_iter"]
    it_g, res_g = sim.ppe_solve(tol, mx)
    it_o, res_o, lam = o.solve(tol, mx)
    hazard = abs(res_o - tol) <= 1e-9 * tol
    if not hazard:
        assert it_g == it_o, (it_g, it_o, res_g, res_o)
    assert res_g == pytest.approx(res_o, rel=1e-8, abs=1e-14)
    f = case.tag == 0
    assert_close("p", sim.get("PRESSURE")[f], o.get("p")[f], 64)


@pytest.mark.parametrize("name", ["tgv2d_f64", "hydro_f64", "db3d_f64", "tgv3d_f32", "db2d_f32"])
def test_stored_coefficients_equal_matrix_free(name):
    """The sweep streaming the per-pair factor stored by A11 and the sweep
    recomputing it from the positions take the same decisions
    and agree to rounding (the factor is the same expression)."""
    case = CASES[name]
    a, b = gpu_sim(case), gpu_sim(case, matrix_free=1)
    for s in (a, b):
        s.predict(case.dt)
    tol, mx = case.params["tol"], case.params["max_iter"]
    ia, ra = a.ppe_solve(tol, mx)
    ib, rb = b.ppe_solve(tol, mx)
    assert ia == ib
    assert ra == pytest.approx(rb, rel=1e-12, abs=1e-300)
    pa, pb = a.get("PRESSURE"), b.get("PRESSURE")
    assert np.abs(pa - pb).max() <= 1e-13 * max(np.abs(pb).max(), 1e-300) * (1 if _prec(case) == 64 else 1e7)


@pytest.mark.parametrize("name", list(CASES))
def test_fixed_sweeps_parity(name):
    # tol = 0, max_iter = S: both sides do exactly S sweeps (SURVEY §8(c) fp32 contract)
    case = CASES[name]
    prec = _prec(case)
    sim = gpu_sim(case)
    o = oracle_from_gpu(case, sim)
    sim.predict(case.dt)
    o.predict(case.dt)
    inject_rstar(sim, o, case, prec)
    S = 7
    it_g, _ = sim.ppe_solve(0.0, S)
    it_o, _, _ = o.solve(0.0, S)
    assert it_g == it_o == S
    assert_close("p", sim.get("PRESSURE"), o.get("p"), prec)


# ------------------------------------------------------------------ A13-A15
@pytest.mark.parametrize("name", list(CASES))
def test_full_step_parity_resynced(name):
    """Several full Algorithm-1 steps; before each step the oracle is loaded with
    the GPU's state, so both sides step from identical inputs."""
    case = CASES[name]
    prec = _prec(case)
    sim = gpu_sim(case)
    o = oracle_from_gpu(case, sim)
    f = case.tag == 0
    steps = 3 if case.dim == 3 else 4
    over = {} if prec == 64 else {"tol": 0.0, "max_iter": 5}
    tol = over.get("tol", case.params["tol"])
    mx = over.get("max_iter", case.params["max_iter"])
    for s in range(steps):
        resync(case, sim, o)
        x0 = sim.get("POSITION")
        sim.predict(case.dt)
        o.predict(case.dt)
        inject_rstar(sim, o, case, prec)
        it_g, _ = sim.ppe_solve(tol, mx)
        it_o, res_o, _ = o.solve(tol, mx)
        if prec == 64 and abs(res_o - tol) > 1e-9 * tol:
            assert it_g == it_o, (s, it_g, it_o)
        sim.correct(case.dt)
        o.correct(case.dt)
        assert_close(f"p step {s}", sim.get("PRESSURE")[f], o.get("p")[f], prec)
        assert_close(f"u step {s}", sim.get("VELOCITY")[f], o.get("u")[f], prec)
        ut_o = o.get("ut")[f]
        assert_close(f"ut step {s}", sim.get("TRANSPORT_VELOCITY")[f], ut_o, prec,
                     abs_floor=ut_floor(case, prec=prec, S=np.abs(ut_o).max()))
        assert_disp_close(f"x step {s}", sim.get("POSITION")[f], o.get("x")[f], x0[f], case, prec)


def test_tgv2d_ten_steps_free_running():
    """C1 exactly as configured (fp64, tol 1e-4, 10 steps), both sides free
    running from the same inputs: sweep counts equal each step, fields close,
    and the decay matches exp(b t)."""
    case = synth.tgv2d()
    sim = gpu_sim(case)
    o = oracle_from_gpu(case, sim)
    for s in range(case.steps):
        rep = sim.step(case.dt)
        it_o, res_o, _ = o.step(case.dt)
        if abs(res_o - case.params["tol"]) > 1e-9 * case.params["tol"]:
            assert rep.iters == it_o, (s, rep.iters, it_o)
    f = case.tag == 0
    u = sim.get("VELOCITY")[f]
    assert np.abs(u - o.get("u")[f]).max() < 1e-8
    umax = np.linalg.norm(u, axis=1).max()
    assert umax == pytest.approx(np.exp(-8 * np.pi ** 2 / 100 * case.steps * case.dt), rel=1e-2)


# ------------------------------------------------------------------ properties
def test_step_is_deterministic():
    case = CASES["db3d_f32"]
    a, b = gpu_sim(case), gpu_sim(case)
    for _ in range(3):
        ra, rb = a.step(case.dt), b.step(case.dt)
        assert ra.iters == rb.iters and ra.residual == rb.residual
    for fld in ("POSITION", "VELOCITY", "PRESSURE"):
        assert np.array_equal(a.get(fld), b.get(fld))


def test_edge_single_fluid_particle():
    # no neighbours: D_ii = 0 -> p = 0; the step still runs
    from paper_1908_01762_b200 import Simulation, domain, params_from_dict
    x = np.array([[0.5, 0.5]])
    sim = Simulation(x, np.zeros((1, 2)), np.ones(1), np.ones(1), np.zeros(1, np.int32), 0.01,
                     domain(2, [0, 0], [1, 1], [0, 0]), params_from_dict({"precision": 64, "rho0": 1e-9}))
    sim.set("PRESSURE", np.array([3.0]))
    rep = sim.step(1e-3)
    assert rep.iters == 2
    assert sim.get("PRESSURE")[0] == 0.0


def test_edge_fluid_only_ragged_and_max_iter_cap():
    case = synth.tgv2d(n=23)   # 529 particles: ragged against 128/256-thread blocks
    sim = gpu_sim(case)
    o = oracle_from_gpu(case, sim)
    sim.predict(case.dt)
    o.predict(case.dt)
    it_g, res_g = sim.ppe_solve(1e-15, 3)     # non-convergence is not an error
    it_o, res_o, _ = o.solve(1e-15, 3)
    assert it_g == it_o == 3 and res_g >= 1e-15
    assert_close("p", sim.get("PRESSURE"), o.get("p"), 64)


def test_eisph_single_sweep():
    case = CASES["hydro_f64"]
    sim = gpu_sim(case)
    sim.predict(case.dt)
    it, _ = sim.ppe_solve(1e-2, 1)
    assert it == 1


# ------------------------------------------------------------------ NEXT-1: adaptive dt
@pytest.mark.parametrize("name", list(CASES))
def test_adaptive_dt_parity(name):
    """sisph_next_dt (device-reduced max|u|, max|f|) vs the oracle's P:675-694 rule."""
    from paper_1908_01762_b200 import SisphError
    case = CASES[name]
    prec = _prec(case)
    sim = gpu_sim(case)
    o = oracle_from_gpu(case, sim)
    with pytest.raises(SisphError):
        sim.next_dt()
    tol, mx = (case.params["tol"], case.params["max_iter"]) if prec == 64 else (0.0, 5)
    sim.predict(case.dt)
    o.predict(case.dt)
    inject_rstar(sim, o, case, prec)
    sim.ppe_solve(tol, mx)
    o.solve(tol, mx)
    sim.correct(case.dt)
    o.correct(case.dt)
    rel = 1e-9 if prec == 64 else 1e-4
    for g, r in zip(sim.next_dt(), o.next_dt()):
        if np.isinf(r):
            assert np.isinf(g)
        else:
            assert g == pytest.approx(r, rel=rel)


def test_adaptive_dt_free_fall_closed_form_gpu():
    # f^n = g exactly and u^{n+1} = U0 + dt g for a uniformly translating periodic
    # lattice under gravity (see the oracle pin): the device reductions must give
    # 0.25 h / |U0 + dt g| and 0.25 sqrt(h / |g|)
    case = synth.lattice_periodic(2, 16, dx=1.0 / 16, jitter=0.1)
    case.params.update(p_ref=0.0, g=[0.0, -9.81, 0.0], nu=0.01, alpha=0.05, c_ref=10.0, pgrad=1)
    U0 = np.array([0.3, 0.2])
    case.u[:] = U0
    sim = gpu_sim(case)
    dt = 1e-3
    sim.step(dt)
    dtn, dtc, dtf = sim.next_dt()
    assert dtc == pytest.approx(0.25 * case.h / np.linalg.norm(U0 + dt * np.array([0.0, -9.81])), rel=1e-12)
    assert dtf == pytest.approx(0.25 * np.sqrt(case.h / 9.81), rel=1e-9)
    assert dtn == min(dtc, dtf)


# ------------------------------------------------------------------ NEXT-2: method variants
@pytest.mark.parametrize("name,over", [
    ("tgv2d_f64", {"max_iter": 1, "min_iter": 1}),        # EISPH: one sweep, no minimum of two
    ("hydro_f64", {"max_iter": 1, "min_iter": 1}),
    ("hydro_f64", {"ustar_noslip": 1}),                   # no-slip wall u*
    ("db2d_f64", {"pgrad": 1}),                           # asymm pressure gradient on a free surface
    ("tgv2d_f64", {"pgrad": 0}),                          # symm on the TGV
    ("db3d_f64", {"tol": 1e-3}),                          # a tighter tolerance (Table 1)
])
def test_variant_step_parity(name, over):
    case = CASES[name]
    sim = gpu_sim(case, **over)
    o = oracle_from_gpu(case, sim, params=over)
    f = case.tag == 0
    tol = over.get("tol", case.params["tol"])
    mx = over.get("max_iter", case.params["max_iter"])
    for s in range(3):
        resync(case, sim, o)
        sim.predict(case.dt)
        o.predict(case.dt)
        it_g, _ = sim.ppe_solve(tol, mx)
        it_o, res_o, _ = o.solve(tol, mx)
        if abs(res_o - tol) > 1e-9 * tol:
            assert it_g == it_o, (s, it_g, it_o)
        sim.correct(case.dt)
        o.correct(case.dt)
        assert_close(f"p step {s}", sim.get("PRESSURE")[f], o.get("p")[f], 64)
        assert_close(f"u step {s}", sim.get("VELOCITY")[f], o.get("u")[f], 64)


# ------------------------------------------------------------------ NEXT-3: square patch
@pytest.mark.parametrize("prec", [64, 32])
def test_square_patch_parity(prec):
    """Free surface everywhere, no walls: full steps vs the oracle."""
    case = synth.square_patch(n=30, precision=prec)
    sim = gpu_sim(case)
    o = oracle_from_gpu(case, sim)
    over = {} if prec == 64 else {"tol": 0.0, "max_iter": 5}
    tol = over.get("tol", case.params["tol"])
    mx = over.get("max_iter", case.params["max_iter"])
    for s in range(3):
        resync(case, sim, o)
        sim.predict(case.dt)
        o.predict(case.dt)
        inject_rstar(sim, o, case, prec)
        haz = fs_hazards(o.get("rho"), case.params)
        assert np.array_equal(sim.get("FREE_SURFACE")[~haz], o.get("fs")[~haz])
        it_g, _ = sim.ppe_solve(tol, mx)
        it_o, res_o, _ = o.solve(tol, mx)
        if prec == 64 and abs(res_o - tol) > 1e-9 * tol:
            assert it_g == it_o
        sim.correct(case.dt)
        o.correct(case.dt)
        assert_close(f"p {s}", sim.get("PRESSURE"), o.get("p"), prec)
        assert_close(f"u {s}", sim.get("VELOCITY"), o.get("u"), prec)


# ------------------------------------------------------------------ PPE loop forms
@pytest.mark.parametrize("name", ["tgv2d_f64", "hydro_f64", "db3d_f32", "tgv3d_f64", "db2d_f64"])
def test_ppe_loop_forms_agree(name):
    """Host-polled batches (1), the CUDA-graph WHILE node (2), the persistent
    cooperative kernel (3) and the thread-block cluster (4) run the same row
    arithmetic: equal sweep counts and bitwise-equal pressures; the graph runs the
    very same kernels, so its residual is bitwise equal too (forms 3 and 4 group the
    residual sums -- and the R32 live-row mean of the periodic cases -- in another
    order: equal to rounding there)."""
    case = CASES[name]
    mf = bool(case.params.get("ppe_mean_free", 0))
    sims = {m: gpu_sim(case, ppe_loop=m) for m in (1, 2, 3, 4)}
    for _ in range(3):
        r = {m: s.step(case.dt) for m, s in sims.items()}
        assert r[1].iters == r[2].iters == r[3].iters == r[4].iters
        assert r[1].residual == r[2].residual
        assert r[3].residual == pytest.approx(r[1].residual, rel=1e-9)
        assert r[4].residual == pytest.approx(r[1].residual, rel=1e-9)
    for fld in ("PRESSURE", "VELOCITY", "POSITION"):
        ref = sims[1].get(fld)
        assert np.array_equal(sims[2].get(fld), ref)
        for m in (3, 4):
            if mf:
                assert_close(fld, sims[m].get(fld), ref, case.params["precision"])
            else:
                assert np.array_equal(sims[m].get(fld), ref), (m, fld)
    # split API with another tolerance than the parameters': read per solve
    for s in sims.values():
        s.predict(case.dt)
    its = {m: s.ppe_solve(1e-6, 50)[0] for m, s in sims.items()}
    assert its[1] == its[2] == its[3] == its[4]
    assert np.array_equal(sims[2].get("PRESSURE"), sims[1].get("PRESSURE"))
    for m in (3, 4):
        if mf:
            assert_close("p", sims[m].get("PRESSURE"), sims[1].get("PRESSURE"), case.params["precision"])
        else:
            assert np.array_equal(sims[m].get("PRESSURE"), sims[1].get("PRESSURE")), m


# ------------------------------------------------------------------ the sweep's 16-bit list
@pytest.mark.parametrize("name", ["db3d_f32", "tgv3d_f64", "hydro_f64", "tgv2d_f64"])
@pytest.mark.parametrize("loop", [1, 4])
def test_sweep_codes_bit_equal(name, loop, monkeypatch):
    """Code mode (SISPH_SWEEP_CODES=1, read at create): A11 writes each fluid row's
    list as (16-bit step code, factor) slots with two-slot long steps (z-rows, walls,
    periodic images) and the sweep decodes them -- the same entries in the same
    order, so the solve is bitwise equal to the 32-bit sweep."""
    case = CASES[name]
    sims = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("SISPH_SWEEP_CODES", flag)
        sims[flag] = gpu_sim(case, ppe_loop=loop)
    for _ in range(3):
        r = {k: s.step(case.dt) for k, s in sims.items()}
        assert r["0"].iters == r["1"].iters
        assert r["0"].residual == r["1"].residual
    for fld in ("PRESSURE", "VELOCITY", "POSITION"):
        assert np.array_equal(sims["1"].get(fld), sims["0"].get(fld)), fld


# ------------------------------------------------------------------ the persistent loop's caches
@pytest.mark.parametrize("name", ["hydro_f64", "db2d_f64", "db3d_f32", "db3d_f64"])
def test_persistent_loop_caches_bit_equal(name, monkeypatch):
    """The persistent PPE loop keeps, for the whole solve, p^k of a block's neighbour span
    in a shared-memory tile, every thread's row (tile slots + stored factors) and every
    wall lane's Shepard weights (SISPH_PERS_CACHE = cached chunks per row, read at each
    launch; 0 = the plain form, 1 = almost every row finishes from the list).  Same
    entries, same order, same fused multiply-adds: bitwise-equal solves, with walls whose
    rows fit the wall cache (2D) and walls that fall back to the list (3D)."""
    case = CASES[name]
    sims = {}
    for flag in ("0", "1", "8"):
        monkeypatch.setenv("SISPH_PERS_CACHE", flag)
        sims[flag] = gpu_sim(case, ppe_loop=3)
        its = []
        for _ in range(3):
            r = sims[flag].step(case.dt)
            its.append((r.iters, r.residual))
        sims[flag + "its"] = its
    for flag in ("1", "8"):
        assert sims[flag + "its"] == sims["0its"]
        for fld in ("PRESSURE", "VELOCITY", "POSITION"):
            assert np.array_equal(sims[flag].get(fld), sims["0"].get(fld)), (flag, fld)
    # a tight solve: many sweeps on the cached rows
    monkeypatch.setenv("SISPH_PERS_CACHE", "0")
    for s in (sims["0"], sims["8"]):
        s.predict(case.dt)
    it0 = sims["0"].ppe_solve(1e-7, 60)[0]
    monkeypatch.setenv("SISPH_PERS_CACHE", "8")
    it8 = sims["8"].ppe_solve(1e-7, 60)[0]
    assert it0 == it8
    assert np.array_equal(sims["8"].get("PRESSURE"), sims["0"].get("PRESSURE"))


# ------------------------------------------------------------------ reading R32: mean-free Jacobi
@pytest.mark.parametrize("name", ["tgv2d_f64", "tgv3d_f64", "hydro_f64", "db2d_f64", "tgv3d_f32"])
def test_mean_free_solve_parity(name):
    """ppe_mean_free = 1 (R32): every iterate has the live-row mean removed
    (k_mean_fix; fused first sweep included).  A tight tolerance runs well into
    the regime where plain Jacobi drifts on the periodic cases."""
    case = CASES[name]
    prec = _prec(case)
    over = {"ppe_mean_free": 1}
    sim = gpu_sim(case, **over)
    o = oracle_from_gpu(case, sim, params=over)
    sim.predict(case.dt)
    o.predict(case.dt)
    inject_rstar(sim, o, case, prec)
    tol, mx = (1e-7, 400) if prec == 64 else (0.0, 9)
    it_g, res_g = sim.ppe_solve(tol, mx)
    it_o, res_o, _ = o.solve(tol, mx)
    if prec == 64 and abs(res_o - tol) > 1e-9 * tol:
        assert it_g == it_o, (it_g, it_o, res_g, res_o)
        assert res_g == pytest.approx(res_o, rel=1e-6, abs=1e-14)
    assert_close("p", sim.get("PRESSURE"), o.get("p"), prec)
    f = case.tag == 0
    live = f & (sim.get("FREE_SURFACE") == 0)
    p = sim.get("PRESSURE")
    assert abs(p[live].mean()) <= 1e-9 * np.abs(p[live]).max() * (1 if prec == 64 else 1e5)


@pytest.mark.parametrize("name", ["tgv2d_f64", "db3d_f32"])
def test_mean_free_loop_forms_agree(name):
    """Host batches and the graph WHILE node (whose body ends with k_mean_fix
    setting the condition) run identical kernels: bitwise-equal results; the
    persistent form falls back to the graph for mean-free; the cluster form (4)
    reduces the live-row mean in block-rank order: equal sweep counts, fields equal
    to rounding."""
    case = CASES[name]
    sims = {m: gpu_sim(case, ppe_loop=m, ppe_mean_free=1) for m in (1, 2, 3, 4)}
    for _ in range(3):
        r = {m: s.step(case.dt) for m, s in sims.items()}
        assert r[1].iters == r[2].iters == r[3].iters == r[4].iters
        assert r[1].residual == r[2].residual == r[3].residual
        assert r[4].residual == pytest.approx(r[1].residual, rel=1e-6)
    for fld in ("PRESSURE", "VELOCITY", "POSITION"):
        ref = sims[1].get(fld)
        assert np.array_equal(sims[2].get(fld), ref)
        assert np.array_equal(sims[3].get(fld), ref)
        assert_close(fld, sims[4].get(fld), ref, case.params["precision"])


def test_mean_free_steps_parity_resynced():
    case = CASES["tgv2d_f64"]
    over = {"ppe_mean_free": 1, "tol": 1e-6}
    sim = gpu_sim(case, **over)
    o = oracle_from_gpu(case, sim, params=over)
    f = case.tag == 0
    for s in range(3):
        resync(case, sim, o)
        sim.predict(case.dt)
        o.predict(case.dt)
        it_g, _ = sim.ppe_solve(1e-6, 500)
        it_o, res_o, _ = o.solve(1e-6, 500)
        if abs(res_o - 1e-6) > 1e-9 * 1e-6:
            assert it_g == it_o, (s, it_g, it_o)
        sim.correct(case.dt)
        o.correct(case.dt)
        assert_close(f"p step {s}", sim.get("PRESSURE")[f], o.get("p")[f], 64)
        assert_close(f"u step {s}", sim.get("VELOCITY")[f], o.get("u")[f], 64)


# ------------------------------------------------------------------ NEXT-4: moving walls
def _moving_cases():
    return {
        "couette_f64": synth.couette(nx=10, ny=20, re=10.0),
        "couette_f32": synth.couette(nx=10, ny=20, re=10.0, precision=32),
        "cavity_slip_f64": synth.cavity(n=24, t_end=0.1),
        "cavity_noslip_f64": synth.cavity(n=24, t_end=0.1, ustar_noslip=1),
        "cavity_f32": synth.cavity(n=24, t_end=0.1, precision=32),
    }


@pytest.mark.parametrize("name", list(_moving_cases()))
def test_moving_wall_step_parity(name):
    """Sliding walls (eq:vg-adami with u_wall != 0, R15a) and the first-solve
    background pressure (R33, cavity): resynced full steps vs the oracle."""
    case = _moving_cases()[name]
    prec = case.params["precision"]
    sim = gpu_sim(case)
    assert np.array_equal(sim.get("WALL_VELOCITY")[case.tag == 1], case.u[case.tag == 1].astype(
        np.float32 if prec == 32 else np.float64))
    o = oracle_from_gpu(case, sim)
    uw = case.u.copy()
    uw[case.tag == 0] = 0
    o.set("uwall", uw)
    f = case.tag == 0
    over = {} if prec == 64 else {"tol": 0.0, "max_iter": 5}
    tol = over.get("tol", case.params["tol"])
    mx = over.get("max_iter", case.params["max_iter"])
    for s in range(4):
        resync(case, sim, o)
        x0 = sim.get("POSITION")
        sim.predict(case.dt)
        o.predict(case.dt)
        inject_rstar(sim, o, case, prec)
        it_g, _ = sim.ppe_solve(tol, mx)
        it_o, res_o, _ = o.solve(tol, mx)
        if prec == 64 and abs(res_o - tol) > 1e-9 * tol:
            assert it_g == it_o, (s, it_g, it_o)
        sim.correct(case.dt)
        o.correct(case.dt)
        w = case.tag == 1
        assert_close(f"wall u {s}", sim.get("VELOCITY")[w], o.get("u")[w], prec, scale=1.0)
        # Couette is a pure shear flow: p is zero up to round-off; its scale is rho0 U^2 = 1
        assert_close(f"p step {s}", sim.get("PRESSURE")[f], o.get("p")[f], prec, scale=1.0)
        assert_close(f"u step {s}", sim.get("VELOCITY")[f], o.get("u")[f], prec)
        assert_disp_close(f"x step {s}", sim.get("POSITION")[f], o.get("x")[f], x0[f], case, prec)


@pytest.mark.parametrize("prec", [64, 32])
def test_couette_start_up_closed_form_gpu(prec):
    """The CUDA path against the start-up Couette series (same bound as the oracle's pin)."""
    case = synth.couette(nx=10, ny=20, re=10.0, precision=prec)
    sim = gpu_sim(case)
    steps = int(round(4.0 / case.dt))
    for _ in range(steps):
        sim.step(case.dt)
    f = case.tag == 0
    x, u = sim.get("POSITION"), sim.get("VELOCITY")
    ue = synth.couette_velocity(x[f, 1], steps * case.dt, 1.0, 1.0, case.params["nu"])
    err = np.abs(u[f, 0] - ue)
    assert err.max() < 0.01 and err.mean() < 0.005


def test_wall_velocity_field_roundtrip():
    case = synth.cavity(n=16, t_end=0.1)
    sim = gpu_sim(case)
    uw = np.zeros_like(case.u)
    w = case.tag == 1
    uw[w, 0] = np.linspace(-1, 1, w.sum())
    sim.set("WALL_VELOCITY", uw)
    assert np.array_equal(sim.get("WALL_VELOCITY"), uw)
    # the ghost velocity of a wall far from the fluid is its own velocity (R15a)
    sim.step(case.dt)
    x = case.x
    far = w & ((x[:, 1] > 1 + 2 * case.dx) | (x[:, 1] < -2 * case.dx))
    far &= (x[:, 0] > 3 * case.dx) & (x[:, 0] < 1 - 3 * case.dx)
    assert far.sum() > 0
    assert np.abs(sim.get("VELOCITY")[far, 0] - uw[far, 0]).max() < 1e-12


@pytest.mark.parametrize("make", [lambda: synth.tgv3d(n=16), lambda: synth.dambreak2d(nx=60, ny=120),
                                  lambda: synth.hydrostatic(nx=40, ny=80)], ids=["tgv3d", "db2d", "hydro"])
def test_state_roundtrip_exact(make):
    """POSITION, VELOCITY, TRANSPORT_VELOCITY and PRESSURE are the whole state a step starts
    from (bench.py's e2e loop relies on it): a step after a host round trip of the four
    fields equals the step without it, bit for bit, with the same sweep count."""
    case = make()
    res = []
    for rt in (False, True):
        sim = gpu_sim(case)
        for _ in range(3):
            sim.step(case.dt)
        if rt:
            st = {k: sim.get(k) for k in ("POSITION", "VELOCITY", "TRANSPORT_VELOCITY", "PRESSURE")}
            for k, v in st.items():
                sim.set(k, v)
        r = sim.step(case.dt)
        res.append((r.iters, sim.get("PRESSURE"), sim.get("POSITION")))
        sim.close()
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])


@pytest.mark.parametrize("make", [lambda: synth.tgv3d(n=16), lambda: synth.dambreak2d(nx=60, ny=120)],
                         ids=["tgv3d", "db2d"])
def test_staged_upload_equals_set_field(make):
    """sisph_stage_field / sisph_commit_staged (bench.py's pipelined e2e): the staged state,
    uploaded while steps run and committed afterwards, gives the same next step, bit for bit,
    as sisph_set_field of the same buffers; a field staged twice before a commit is
    rejected; a commit with nothing staged is a no-op."""
    from paper_1908_01762_b200 import SisphError
    case = make()
    ref = gpu_sim(case)
    for _ in range(2):
        ref.step(case.dt)
    state = {k: ref.get(k, dtype=np.float32) for k in ("POSITION", "VELOCITY", "TRANSPORT_VELOCITY", "PRESSURE")}
    res = []
    for staged in (False, True):
        sim = gpu_sim(case)
        if staged:
            for k, v in state.items():
                sim.stage_ptr(k, v.ctypes.data, v.size, True)
            with pytest.raises(SisphError):
                v = state["PRESSURE"]
                sim.stage_ptr("PRESSURE", v.ctypes.data, v.size, True)
            sim.step(case.dt)              # runs on the creation state; the upload overlaps it
            sim.commit_staged()
            sim.commit_staged()            # nothing staged: no-op
        else:
            sim.step(case.dt)
            for k, v in state.items():
                sim.set(k, v)
        r = sim.step(case.dt)
        res.append((r.iters, sim.get("PRESSURE"), sim.get("POSITION"), sim.get("VELOCITY")))
        sim.close()
    ref.close()
    assert res[0][0] == res[1][0]
    for a, b in zip(res[0][1:], res[1][1:]):
        assert np.array_equal(a, b)


def test_staged_positions_with_moved_walls():
    """A staged POSITION whose wall particles moved takes set_field's re-sort path (the wall
    check ran on the upload stream): the next step equals the set_field one bit for bit."""
    case = synth.dambreak2d(nx=60, ny=120)
    x = None
    res = []
    for staged in (False, True):
        sim = gpu_sim(case)
        sim.step(case.dt)
        if x is None:
            x = sim.get("POSITION", dtype=np.float32)
            w = case.tag == 1
            x[w, 0] += np.float32(0.25 * case.dx)
        if staged:
            sim.stage_ptr("POSITION", x.ctypes.data, x.size, True)
            sim.commit_staged()
        else:
            sim.set("POSITION", x)
        r = sim.step(case.dt)
        res.append((r.iters, sim.get("PRESSURE"), sim.get("POSITION")))
        sim.close()
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])


def test_fetch_field_equals_get_field():
    """sisph_fetch_field / sisph_fetch_wait (bench.py's pipelined e2e): the value fetched right
    after a step, read while the next step runs, equals sisph_get_field's after that step; a
    second fetch before the wait is rejected; a wait with nothing pending is a no-op."""
    from paper_1908_01762_b200 import SisphError
    case = synth.dambreak2d(nx=60, ny=120)
    sim = gpu_sim(case)
    sim.step(case.dt)
    ref = sim.get("PRESSURE", dtype=np.float32)
    ref_x = sim.get("POSITION")
    out = np.zeros(ref.size, np.float32)
    sim.fetch_ptr("PRESSURE", out.ctypes.data, out.size, True)
    with pytest.raises(SisphError):
        sim.fetch_ptr("PRESSURE", out.ctypes.data, out.size, True)
    sim.step(case.dt)                  # the copy of the previous p overlaps this step
    sim.fetch_wait()
    sim.fetch_wait()
    assert np.array_equal(out, ref)
    x64 = np.zeros(ref_x.size)
    sim2 = gpu_sim(case)
    sim2.step(case.dt)
    sim2.fetch_ptr("POSITION", x64.ctypes.data, x64.size, False)
    sim2.fetch_wait()
    assert np.array_equal(x64.reshape(ref_x.shape), ref_x)
    sim.close()
    sim2.close()


@pytest.mark.parametrize("name", ["tgv2d_f64", "hydro_f64", "db2d_f64"])
def test_conv_mean_solve_parity(name):
    """Reading R12b (eq:convergence on means, scaled by the global fluid count):
    same stopping sweep and residual as the oracle, from p^0 = 0 where Lambda
    decides the first sweeps."""
    case = CASES[name]
    over = {"conv_mean": 1}
    sim = gpu_sim(case, **over)
    sim.set("PRESSURE", np.zeros(case.n))
    o = oracle_from_gpu(case, sim, params=over)
    sim.predict(case.dt)
    o.predict(case.dt)
    for tol in (1e-2, 1e-4):
        it_g, res_g = sim.ppe_solve(tol, 300)
        it_o, res_o, _ = o.solve(tol, 300)
        if abs(res_o - tol) > 1e-9 * tol:
            assert it_g == it_o, (tol, it_g, it_o, res_g, res_o)
        assert res_g == pytest.approx(res_o, rel=1e-8, abs=1e-14)
        assert_close("p", sim.get("PRESSURE")[case.tag == 0], o.get("p")[case.tag == 0], 64)


def test_fp32_host_io_matches_fp64_io():
    """sisph_{get,set}_field_f32: an fp32 handle's fields read as float32 equal the
    float64 read rounded; a step from state set through the f32 calls equals the
    step from the same values set through the f64 calls."""
    case = synth.dambreak3d(nfx=24, nfy=12, nfz=16, dx=1.0 / 32, tank_nx=60, wall_nz=24, precision=32)
    a, b = gpu_sim(case), gpu_sim(case)
    for _ in range(2):
        a.step(case.dt)
    for fld in ("POSITION", "VELOCITY", "TRANSPORT_VELOCITY", "PRESSURE", "DENSITY", "MASS"):
        g64, g32 = a.get(fld), a.get(fld, dtype=np.float32)
        assert g32.dtype == np.float32
        assert np.array_equal(g32, g64.astype(np.float32)), fld
    for fld in ("POSITION", "VELOCITY", "TRANSPORT_VELOCITY", "PRESSURE"):
        b.set(fld, a.get(fld, dtype=np.float32))
    c = gpu_sim(case)
    for fld in ("POSITION", "VELOCITY", "TRANSPORT_VELOCITY", "PRESSURE"):
        c.set(fld, a.get(fld))
    rb, rc = b.step(case.dt), c.step(case.dt)
    assert rb.iters == rc.iters
    for fld in ("POSITION", "VELOCITY", "PRESSURE"):
        assert np.array_equal(b.get(fld), c.get(fld)), fld


# ------------------------------------------------------------------ NEXT-4b: open boundaries (R34)
@pytest.mark.parametrize("dim", [2, 3])
def test_open_boundary_parity_fp64(dim):
    """Inlet / outlet / dormant conversions and the id pool (reading R34): the CUDA
    path and the oracle, free running from the same inputs, agree on every type
    change and id draw (bit-exact TAG field), on the sweep counts, and on the
    fields of the active particles (fp64 tolerance).  3D: the same channel, periodic
    in z."""
    import oracle
    case = synth.channel(nx=20, ny=8) if dim == 2 else synth.channel(nx=12, ny=8, nz=12)
    sim = gpu_sim(case)
    o = oracle.Sim(case)
    moved = 0
    for s in range(40 if dim == 2 else 25):
        x0, t0, xg0 = o.get("x"), o.tags(), sim.get("POSITION")
        rg = sim.step(case.dt)
        it_o, res_o, _ = o.step(case.dt)
        if abs(res_o - case.params["tol"]) > 1e-9 * case.params["tol"]:
            assert rg.iters == it_o, (s, rg.iters, it_o)
        tg, to = sim.get("TAG").astype(np.int32), o.tags()
        assert np.array_equal(tg, to), s
        act = (to == 0) | (to == synth.INLET) | (to == synth.OUTLET)
        same = act & (t0 != synth.DORMANT)         # not spawned this step: compare the displacement
        assert_disp_close(f"x {s}", sim.get("POSITION")[same], o.get("x")[same], xg0[same], case, 64,
                          x0_ref=x0[same])
        assert_close(f"x spawned {s}", sim.get("POSITION")[act & ~same], o.get("x")[act & ~same], 64)
        assert_close(f"u {s}", sim.get("VELOCITY")[act], o.get("u")[act], 64)
        assert_close(f"p {s}", sim.get("PRESSURE")[act], o.get("p")[act], 64)
        moved += int((to != case.tag).sum())
    assert moved > 0
    # dormant ids read zero
    dorm = o.tags() == synth.DORMANT
    assert np.all(sim.get("POSITION")[dorm] == 0)


def test_open_boundary_pool_exhaustion_is_an_error():
    from paper_1908_01762_b200 import SisphError
    case = synth.channel(nx=20, ny=8, n_pool=0)
    sim = gpu_sim(case)
    with pytest.raises(SisphError) as e:
        for _ in range(200):
            sim.step(case.dt)
    assert "dormant pool" in str(e.value)


def test_channel_keeps_the_poiseuille_profile_gpu():
    """The oracle's closed-form pin on the CUDA path (same bound)."""
    case = synth.channel()
    sim = gpu_sim(case)
    for _ in range(int(round(2.0 / case.dt))):
        sim.step(case.dt)
    tag, x, u = sim.get("TAG"), sim.get("POSITION"), sim.get("VELOCITY")
    sel = (tag == 0) & (x[:, 0] > 2.0) & (x[:, 0] < 3.0)
    err = np.abs(u[sel, 0] - synth.poiseuille_velocity(x[sel, 1], 1.0, 1.0))
    assert err.mean() < 0.025 and err.max() < 0.06


def test_cylinder_steps_parity_fp64():
    """The cylinder workload (R35: curved walls of wall-particle rings, inlet / outlet,
    external GTVF, symm, periodic y): free-running steps equal the oracle's (sweep
    counts, every type change, the fields of the active particles to fp64
    round-off).  The start's large GTVF shifts exceed the single build's skin, so the
    two-build fallback runs with open boundaries here too."""
    import oracle
    case = synth.cylinder(ppd=6, t_end=1.0)
    sim = gpu_sim(case)
    o = oracle.Sim(case)
    for s in range(6):
        x0, t0, xg0 = o.get("x"), o.tags(), sim.get("POSITION")
        rg = sim.step(case.dt)
        it_o, res_o, _ = o.step(case.dt)
        if abs(res_o - case.params["tol"]) > 1e-9 * case.params["tol"]:
            assert rg.iters == it_o, (s, rg.iters, it_o)
        to = o.tags()
        assert np.array_equal(sim.get("TAG").astype(np.int32), to), s
        act = (to == 0) | (to == synth.INLET) | (to == synth.OUTLET)
        same = act & (t0 != synth.DORMANT)
        assert_disp_close(f"x {s}", sim.get("POSITION")[same], o.get("x")[same], xg0[same], case, 64,
                          x0_ref=x0[same])
        assert_close(f"x spawned {s}", wrap_delta(sim.get("POSITION")[act & ~same] - o.get("x")[act & ~same],
                                                  case), 0.0 * o.get("x")[act & ~same], 64, scale=30.0)
        assert_close(f"u {s}", sim.get("VELOCITY")[act], o.get("u")[act], 64)
        assert_close(f"p {s}", sim.get("PRESSURE")[act], o.get("p")[act], 64)


def test_tgv_tight_tolerance_with_half_h_gtvf_and_mean_free():
    """R22c + R32 on the CUDA path: at eps = 1e-4 the 50^2 Taylor-Green vortex follows the
    exact decay exp(-8 pi^2 t / Re) to t = 1 (with h~ = h and the printed iteration it
    goes unstable there; profiles/r1_variants.md §6-8)."""
    case = synth.tgv2d()
    sim = gpu_sim(case, tol=1e-4, h_tilde_factor=0.5, ppe_mean_free=1)
    steps = int(round(1.0 / case.dt))
    for _ in range(steps):
        sim.step(case.dt)
    u = sim.get("VELOCITY")
    decay = np.abs(u).max() / np.exp(-8 * np.pi ** 2 * case.params["nu"] * steps * case.dt)
    assert abs(decay - 1.0) < 0.03, decay


# ------------------------------------------------------------------ A5 build kernels
@pytest.mark.parametrize("name", ["db3d_f32", "db3d_f64", "tgv3d_f32"])
def test_masked_loose_build_equals_fused(name, monkeypatch):
    """k_build_loose_m (test into masks, then append) writes the loose list of k_build_loose
    entry for entry, so whole steps are bit-identical (SISPH_BUILD_MASK=0 selects the fused
    kernel; the switch is read when a handle is created)."""
    case = CASES[name]
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("SISPH_BUILD_MASK", flag)
        sim = gpu_sim(case)
        sim.set("TRANSPORT_VELOCITY", _moving(case, 0.3))
        its = [sim.step(case.dt).iters for _ in range(3)]
        out[flag] = [np.array(its)] + [sim.get(f) for f in ("POSITION", "VELOCITY", "PRESSURE", "DENSITY")]
        sim.close()
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)
