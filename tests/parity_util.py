"""Helpers for GPU-vs-oracle parity: build both sides on identical inputs and
compare fields ELEMENT BY ELEMENT with the tolerances north_star states
(BASELINE.json) and SURVEY.md §8(c) makes concrete:

* fp64 mode: |gpu_i - ref_i| <= 1e-10 * max(|ref_i|, 1e-3 * S)
  (per-particle relative 1e-10 where |ref_i| > 1e-3 S; below that the bound is
  1e-13 S, tighter than the survey's normwise 1e-10 S for those elements)
* fp32 mode: |gpu_i - ref_i| <= 1e-4 * |ref_i| + 1e-6 * max(S, 1)

S is the field's scale, max_i |ref_i| (or a physical floor the caller passes).
north_star's "1e-6 absolute" is taken literally in the field's units where the
field's scale is at most 1 (velocities in m/s, positions' displacements) and
relative to its scale where that exceeds 1 (p in Pa reaches 2e4 in the dam
breaks, where fp32 cannot represent 1e-6 Pa; DESIGN.md §5 R36).

Positions are compared through the step's displacement d = x^{n+1} - x^n
(assert_disp_close): |d_gpu,i - d_ref,i| <= the bound above on d, plus the
storage rounding of the coordinate itself (2 ulp of x_i in the handle's
precision: an fp32 handle stores r in fp32, so the oracle's fp64 x^{n+1} is
representable only to 0.5 ulp, each side rounds its own update x + dt ū by
0.5 ulp, and the oracle's ũ^{n+1} carries up to 2 ulp / dt of cancellation in
(r^K - r^0)/dt, which dt ū turns into <= 1 ulp: 4 ulp in all).

Discrete results (cell order, neighbour sets, iteration counts) are compared
exactly.  Hazards (a residual within 1e-9 of the tolerance, a free-surface
ratio within 1e-6 of 0.8) are counted and reported rather than hidden.
"""
import numpy as np

import oracle
import synth

TOL = {64: (1e-10, 0.0), 32: (1e-4, 1e-6)}


def gpu_sim(case, **over):
    from paper_1908_01762_b200 import Simulation
    return Simulation.from_case(case, **over)


def oracle_from_gpu(case, sim, params=None):
    """An oracle Sim holding exactly the GPU's (precision-rounded) state."""
    prm = dict(case.params)
    prm.update(params or {})
    cfg = oracle.make_cfg(case.dim, case.lo, case.hi, case.periodic, case.h, prm)
    x = sim.get("POSITION")
    u = sim.get("VELOCITY")
    w = case.tag == 1
    # a wall's creation velocity is its prescribed velocity (VELOCITY of a wall is its ghost velocity)
    u[w] = sim.get("WALL_VELOCITY")[w]
    m = sim.get("MASS")
    rho = sim.get("DENSITY")
    p = sim.get("PRESSURE")
    o = oracle.Sim(cfg=cfg, x=x, u=u, m=m, rho=rho, p=p, tag=case.tag)
    o.set("ut", sim.get("TRANSPORT_VELOCITY") if (case.tag == 0).any() else u)
    return o


def resync(case, sim, o):
    """Load the GPU's carried state (r, u, u~, p) into the oracle."""
    f = case.tag == 0
    x = sim.get("POSITION")
    ut = sim.get("TRANSPORT_VELOCITY")
    u = sim.get("VELOCITY")
    p = sim.get("PRESSURE")
    o.set("x", x)
    uo = o.get("u")
    uo[f] = u[f]
    o.set("u", uo)
    o.set("ut", ut)
    o.set("p", p)


def _bound(ref, prec, S):
    rel, ab = TOL[prec]
    a = np.abs(ref)
    if prec == 64:
        return rel * np.maximum(a, 1e-3 * S)
    return rel * a + ab * max(S, 1.0)


def _check(name, got, ref, bound, S):
    err = np.abs(got - ref)
    bad = err > bound
    if bad.any():
        k = np.unravel_index(np.argmax(err - bound), err.shape)
        raise AssertionError(
            f"{name}: {int(bad.sum())} of {err.size} elements out of bound; worst element {k}: "
            f"gpu {got[k]:.9e} ref {ref[k]:.9e} |diff| {err[k]:.3e} > bound {bound[k]:.3e} "
            f"(field scale {S:.3e})")
    small = int((np.abs(ref) <= 1e-3 * S).sum())
    return float((err / bound).max()), small


def assert_close(name, got, ref, prec, mask=None, scale=None, report=None, abs_floor=0.0):
    """Per-element parity (module docstring).  S = max(max|ref|, scale): `scale` is a
    physical floor of the field's scale (a field that is zero up to round-off, e.g.
    the pressure of a pure shear flow, has no scale of its own).  `abs_floor` adds
    an absolute allowance derived from the arithmetic (e.g. the oracle's own
    cancellation in (r^K - r^0)/dt).  Returns the worst ratio |diff| / bound; `report`
    (a dict) collects the element count, that ratio and the count in the absolute
    regime (|ref_i| <= 1e-3 S) under `name`."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if mask is not None:
        got, ref = got[mask], ref[mask]
    if ref.size == 0:
        return 0.0
    S = float(np.abs(ref).max())
    if scale is not None:
        S = max(S, float(scale))
    worst, small = _check(name, got, ref, _bound(ref, prec, S) + abs_floor, S)
    if report is not None:
        report[name] = dict(n=int(ref.size), small=small, worst_err_over_bound=worst)
    return worst


def wrap_delta(d, case):
    d = np.array(d, np.float64)
    for a in range(case.dim):
        if case.periodic[a]:
            L = case.hi[a] - case.lo[a]
            d[..., a] = (d[..., a] + 0.5 * L) % L - 0.5 * L
    return d


def assert_disp_close(name, got_x, ref_x, x0, case, prec, report=None, x0_ref=None):
    """Positions through the step's displacement d = x - x0 (module docstring).
    Free-running comparisons pass each side's own previous positions (x0 for the
    GPU, x0_ref for the oracle)."""
    got_x, ref_x, x0 = (np.asarray(v, np.float64) for v in (got_x, ref_x, x0))
    x0r = x0 if x0_ref is None else np.asarray(x0_ref, np.float64)
    dg = wrap_delta(got_x - x0, case)
    dr = wrap_delta(ref_x - x0r, case)
    S = float(np.abs(dr).max())
    if S == 0.0:
        S = 1.0
    ulp = np.spacing(np.abs(ref_x).astype(np.float32 if prec == 32 else np.float64)).astype(np.float64)
    bound = _bound(dr, prec, S) + 4.0 * ulp
    worst, small = _check(name, dg, dr, bound, S)
    if report is not None:
        report[name] = dict(n=int(dr.size), small=small, worst_err_over_bound=worst, disp_scale=S)
    return worst


def ut_floor(case, dt=None, prec=64, S=1.0):
    """Absolute allowance on u~^{n+1} = u^{n+1} + (r^K - r^0)/dt (eq:int:vhatnp2): the oracle
    forms r^K - r^0 as a difference of two fp64 positions, whose rounding is up to 1 ulp of
    the coordinate, divided by dt (the GPU carries the displacement explicitly).  fp32: the
    GTVF force of eq:mom:sph:gtvf sums m_j / rho_j^2 grad W over a near-lattice
    neighbourhood whose terms cancel to ~1e-3 of their absolute sum, so the fp32 shift
    carries up to ~1e-6 of the velocity scale on top of the generic bound (R36).  That shift is
    a cancelling sum over positions the handle stores in fp32 (r^{n+1} before the sub-steps),
    so its rounding moves linearly with the coordinate quantum relative to h: the allowance is
    GTVF_CANCEL * ulp32(x_max) / h of the velocity scale, GTVF_CANCEL = 1e-6 / (ulp32(3.2) * 256)
    fixed on C5 (|x| <= 3.2, h = 1/256), and never below C5's 1e-6 (C3: |x| <= 4, h = 0.002,
    about twice C5's quantum relative to h)."""
    xm = max(abs(float(np.max(case.hi))), abs(float(np.min(case.lo))), 1.0)
    fl = 2.0 * float(np.spacing(xm)) / (case.dt if dt is None else dt)
    if prec == 32:
        q = float(np.spacing(np.float32(xm))) / case.h
        fl += max(1e-6, GTVF_CANCEL * q) * max(S, 1.0)
    return fl


GTVF_CANCEL = 1e-6 / (float(np.spacing(np.float32(3.2))) * 256.0)


def inject_rstar(sim, o, case, prec, dt=None):
    """fp32 handles keep r* in fp32 (reading R36): the oracle evaluates A9-A11 (and the
    rest of the step) on the r* the handle holds, so that the comparison measures the
    arithmetic, not the storage rounding of r* (checked on its own: assert_disp_close)."""
    if prec == 32:
        o.set("xs", sim.get("RSTAR"))
        o.predict_stage2(case.dt if dt is None else dt)


def inject_stage1(sim, o, case, prec, dt=None):
    """As inject_rstar, and the fluid u* too: an fp32 handle stores u* in fp32, and the RHS of
    eq:sph-ppe is a divergence of u* that cancels on a smooth field (TGV-3D at full size: the
    terms' absolute sum is ~1e3 times the result), so the storage rounding of u*, 6e-8 of |u|,
    moves it by ~1e-4 of its scale (reading R36).  Call after u* itself was compared."""
    if prec == 32:
        f = case.tag == 0
        us = o.get("us")
        us[f] = sim.get("USTAR")[f]
        o.set("us", us)
    inject_rstar(sim, o, case, prec, dt)


def fs_hazards(rho_o, params, width=1e-6):
    """Rows whose free-surface ratio rho/rho0 lies within `width` of the threshold."""
    haz = np.abs(rho_o / params["rho0"] - params["fs_ratio"]) < width
    print(f"free-surface hazards (|rho/rho0 - {params['fs_ratio']}| < {width}): {int(haz.sum())}")
    return haz


def small_cases():
    """Small instances of every BASELINE config, spanning several tiles with ragged tails."""
    return {
        "tgv2d_f64": synth.tgv2d(),                                           # C1 as configured
        "tgv2d_f32": synth.tgv2d(n=37, precision=32),
        "hydro_f64": synth.hydrostatic(nx=40, ny=80, dx=0.025, precision=64),
        "hydro_f32": synth.hydrostatic(nx=40, ny=80, dx=0.025, precision=32),
        "db2d_f32": synth.dambreak2d(nx=50, ny=100, dx=0.02, precision=32),
        "db2d_f64": synth.dambreak2d(nx=30, ny=60, dx=0.0333333, precision=64),
        "tgv3d_f32": synth.tgv3d(n=20, precision=32),
        "tgv3d_f64": synth.tgv3d(n=14, precision=64),
        "db3d_f32": synth.dambreak3d(nfx=24, nfy=12, nfz=16, dx=1.0 / 32, tank_nx=60, wall_nz=24,
                                     precision=32),
        "db3d_f64": synth.dambreak3d(nfx=16, nfy=10, nfz=12, dx=1.0 / 32, tank_nx=40, wall_nz=16,
                                     precision=64),
    }
