"""Slab decomposition of the CUDA path, on one GPU.

R ranks run as threads of this process sharing the GPU through the
in-process transport (sisph_local_group): every exchange synchronises the
rank's stream and meets the other ranks at a host barrier, so no kernel ever
waits on another rank's kernel (B200_PROFILING.md).  The same engine code
runs over NCCL in production; only the transport differs.

Each case runs a few free SISPH steps decomposed over R slabs and on a single
handle, from the same inputs: the PPE sweep counts must be equal (the
residual sums and Lambda are allreduced) and the fields must agree to the
north_star tolerance (summation order differs across decompositions).
"""
import threading

import numpy as np
import pytest

import synth
from parity_util import assert_close, assert_disp_close, gpu_sim

pytestmark = pytest.mark.gpu


def run_ranks(case, R, axis, nsteps, **over):
    from paper_1908_01762_b200 import LocalGroup, Simulation, make_dist
    g = LocalGroup(R)
    sims, reps, errs = [None] * R, [[] for _ in range(R)], [None] * R

    def work(r):
        try:
            s = Simulation.from_case(case, dist=make_dist(R, r, axis, local_group=g), **over)
            sims[r] = s
            for _ in range(nsteps):
                reps[r].append(s.step(case.dt))
        except Exception as e:  # noqa: BLE001 - reported below
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), f"a rank hung; errors of the other ranks: {errs}"
    for e in errs:
        if e is not None:
            raise e
    return sims, reps, g


def gathered(sims, field):
    return sum(s.get(field) for s in sims)


CASES = {
    # periodic both ways, jittered: slabs along x (R = 2, 4) and y (R = 3)
    "tgv2d_f64_x2": (lambda: synth.tgv2d(), 2, 0),
    "tgv2d_f64_y3": (lambda: synth.tgv2d(), 3, 1),
    "tgv2d_f64_x4": (lambda: synth.tgv2d(), 4, 0),
    # walls, free surface, bounded slab axis (x across the tank)
    "db2d_f64_x2": (lambda: synth.dambreak2d(nx=30, ny=60, dx=0.0333333, precision=64), 2, 0),
    "hydro_f64_x3": (lambda: synth.hydrostatic(nx=40, ny=80, dx=0.025, precision=64), 3, 0),
    # the bench family: periodic spanwise y is the slab axis
    "db3d_f64_y2": (lambda: synth.dambreak3d(nfx=16, nfy=10, nfz=12, dx=1.0 / 32, tank_nx=40, wall_nz=16,
                                             precision=64), 2, 1),
    "db3d_f32_y2": (lambda: synth.dambreak3d(nfx=24, nfy=12, nfz=16, dx=1.0 / 32, tank_nx=60, wall_nz=24,
                                             precision=32), 2, 1),
    "tgv3d_f32_z3": (lambda: synth.tgv3d(n=20, precision=32), 3, 2),
}


@pytest.mark.parametrize("name", list(CASES))
def test_slab_ranks_equal_single_gpu(name):
    mk, R, axis = CASES[name]
    case = mk()
    prec = case.params["precision"]
    # fp32: one step (the two decompositions sum in different orders; over free-running fp32
    # steps the difference grows through the fp32 position rounding, reading R36)
    steps = 3 if prec == 64 else 1
    # fp32: fixed sweeps so both decompositions do identical work
    over = {} if prec == 64 else {"tol": 0.0, "max_iter": 4}
    single = gpu_sim(case, **over)
    rs = [single.step(case.dt) for _ in range(steps)]
    sims, reps, g = run_ranks(case, R, axis, steps, **over)
    for s in range(steps):
        its = {reps[r][s].iters for r in range(R)}
        assert len(its) == 1, f"ranks disagree on the sweep count at step {s}: {its}"
        assert its.pop() == rs[s].iters, (s, rs[s].iters, [reps[r][s].iters for r in range(R)])
    # every particle owned by exactly one rank
    own = sum(s.owned_counts()[0] for s in sims)
    assert own == case.n_fluid
    for fld in ("PRESSURE", "VELOCITY", "TRANSPORT_VELOCITY"):
        assert_close(fld, gathered(sims, fld), single.get(fld), prec)
    # positions through the displacement over the run (from the creation positions)
    assert_disp_close("POSITION", gathered(sims, "POSITION"), single.get("POSITION"), case.x, case, prec)
    # halos were exchanged (and ghosts were present where fluid borders fluid)
    assert sum(reps[r][-1].halo_bytes for r in range(R)) > 0
    if not name.startswith("db2d"):      # db2d: the water column lies in one slab
        assert all(reps[r][-1].n_ghost_fluid > 0 for r in range(R))
    for s in sims:
        s.close()
    g.close()


def test_migration_moves_ownership():
    """Particles pushed across a slab face change owner at the next step and
    every particle stays owned exactly once."""
    case = synth.tgv2d()
    R, axis = 2, 0
    case.u[:, 0] = 0.9          # uniform drift along the slab axis: particles cross both faces
    case.u[:, 1] = 0.0
    sims, reps, g = run_ranks(case, R, axis, 4, tol=1e-3)
    own = [s.owned_counts()[0] for s in sims]
    assert sum(own) == case.n_fluid
    ids = [np.flatnonzero(np.abs(s.get("MASS")) > 0) for s in sims]
    assert len(np.intersect1d(ids[0], ids[1])) == 0
    assert len(ids[0]) + len(ids[1]) == case.n
    x = gathered(sims, "POSITION")
    from paper_1908_01762_b200 import domain, slab_bounds
    dom = domain(case.dim, case.lo, case.hi, case.periodic)
    for r, s in enumerate(sims):
        lo, hi = slab_bounds(dom, axis, R, r)
        mine = ids[r][case.tag[ids[r]] == 0]
        # owned at the start of the last step: at most one step's motion outside the slab
        xs = x[mine, axis]
        L = case.hi[axis] - case.lo[axis]
        d = np.minimum(np.abs(((xs - lo) + 0.5 * L) % L - 0.5 * L), np.abs(((xs - hi) + 0.5 * L) % L - 0.5 * L))
        outside = ~((xs >= lo) & (xs < hi))
        assert np.all(d[outside] < 0.9 * case.dt * 2)
    for s in sims:
        s.close()
    g.close()


@pytest.mark.parametrize("transport", ["nccl", "local"])
def test_one_rank_periodic_self_halo(transport):
    """One rank with the slab path forced on a periodic axis: its halo comes
    from its own opposite face through the transport (NCCL send/recv to self,
    or the in-process copy), with the periodic image shift; the result must
    equal the single handle's minimum-image run."""
    from paper_1908_01762_b200 import LocalGroup, Simulation, default_nccl_lib, make_dist, nccl_unique_id
    case = synth.tgv2d()
    single = gpu_sim(case)
    if transport == "nccl":
        lib = default_nccl_lib()
        d = make_dist(1, 0, 0, nccl_id=nccl_unique_id(lib), nccl_lib=lib, always_slab=True)
    else:
        g = LocalGroup(1)
        d = make_dist(1, 0, 0, local_group=g, always_slab=True)
    sim = Simulation.from_case(case, dist=d)
    for _ in range(3):
        ra, rb = sim.step(case.dt), single.step(case.dt)
        assert ra.iters == rb.iters
        assert ra.n_ghost_fluid > 0 and ra.halo_bytes > 0
    for fld in ("PRESSURE", "VELOCITY"):
        a, b = sim.get(fld), single.get(fld)
        assert np.abs(a - b).max() <= 1e-10 * np.abs(b).max()
    sim.close()


def test_adaptive_dt_over_slab_ranks():
    """sisph_next_dt is collective: every rank returns the single GPU's value."""
    case = synth.tgv2d()
    single = gpu_sim(case)
    single.step(case.dt)
    ref = single.next_dt()
    from paper_1908_01762_b200 import LocalGroup, Simulation, make_dist
    R = 3
    g = LocalGroup(R)
    out, errs = [None] * R, [None] * R

    def work(r):
        try:
            s = Simulation.from_case(case, dist=make_dist(R, r, 1, local_group=g))
            s.step(case.dt)
            out[r] = s.next_dt()
            s.close()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    for e in errs:
        if e is not None:
            raise e
    for r in range(R):
        for a, b in zip(out[r], ref):
            assert a == pytest.approx(b, rel=1e-12)
    g.close()


def test_full_size_two_slabs_equal_single_gpu():
    """The bench's N = 2 weak-scaling problem at full size: BASELINE configs[4]
    with two per-GPU slabs along the periodic y (4.2M fluid particles), as two
    emulated ranks vs one handle holding the whole problem; fp32, 3 steps with
    fixed sweeps so both sides do identical work."""
    case = synth.dambreak3d(ranks=2)
    over = {"tol": 0.0, "max_iter": 3}
    single = gpu_sim(case, **over)
    rs = [single.step(case.dt) for _ in range(3)]
    sims, reps, g = run_ranks(case, 2, 1, 3, **over)
    assert all(reps[r][s].iters == rs[s].iters == 3 for r in range(2) for s in range(3))
    assert sum(s.owned_counts()[0] for s in sims) == case.n_fluid
    for fld in ("PRESSURE", "VELOCITY"):
        assert_close(fld, gathered(sims, fld), single.get(fld), 32)
    assert_disp_close("POSITION", gathered(sims, "POSITION"), single.get("POSITION"), case.x, case, 32)
    assert all(reps[r][-1].n_ghost_fluid > 0 for r in range(2))
    for s in sims:
        s.close()
    g.close()


def test_mean_free_over_slab_ranks():
    """R32 on slab ranks: the live sum and count are allreduced before the
    mean is removed, the residual sums after: same sweep counts as one handle."""
    case = synth.tgv2d()
    over = {"ppe_mean_free": 1, "tol": 1e-6}
    single = gpu_sim(case, **over)
    rs = [single.step(case.dt) for _ in range(3)]
    sims, reps, g = run_ranks(case, 3, 0, 3, **over)
    for s in range(3):
        assert {reps[r][s].iters for r in range(3)} == {rs[s].iters}
    for fld in ("PRESSURE", "VELOCITY"):
        assert_close(fld, gathered(sims, fld), single.get(fld), 64)
    for s in sims:
        s.close()
    g.close()


def test_moving_lid_over_slab_ranks():
    """The lid-driven cavity (sliding lid, R33 first-solve p_ref allreduced as a
    max) decomposed along x over 2 ranks equals one handle."""
    case = synth.cavity(n=30, t_end=0.1)
    single = gpu_sim(case)
    rs = [single.step(case.dt) for _ in range(4)]
    sims, reps, g = run_ranks(case, 2, 0, 4)
    for s in range(4):
        assert {reps[r][s].iters for r in range(2)} == {rs[s].iters}
    for fld in ("PRESSURE", "VELOCITY"):
        assert_close(fld, gathered(sims, fld), single.get(fld), 64)
    assert_disp_close("POSITION", gathered(sims, "POSITION"), single.get("POSITION"), case.x, case, 64)
    for s in sims:
        s.close()
    g.close()


@pytest.mark.parametrize("name", ["db3d_f32_y2", "tgv3d_f32_z3"])
def test_gtvf_halo_overlap_is_bit_identical(name, monkeypatch):
    """SISPH_GTVF_OVERLAP=1 steps the rows other ranks hold as ghosts first and runs their fp32
    GTVF delta halo on a second stream while the other rows are stepped: the same arithmetic on
    the same data, so every rank's fields are bit-identical to the unsplit sub-steps."""
    mk, R, axis = CASES[name]
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("SISPH_GTVF_OVERLAP", flag)
        sims, reps, _ = run_ranks(mk(), R, axis, 2)
        out[flag] = ([[r.iters for r in rr] for rr in reps],
                     [[s.get(f) for f in ("POSITION", "VELOCITY", "PRESSURE")] for s in sims])
        for s in sims:
            s.close()
    assert out["0"][0] == out["1"][0]
    for a, b in zip(out["0"][1], out["1"][1]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
