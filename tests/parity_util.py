"""Helpers for GPU-vs-oracle parity: build both sides on identical inputs and
compare fields with the tolerances north_star states (BASELINE.json):

* fp64 mode: |gpu - ref| <= 1e-10 * max|ref| (normwise; p crosses zero)
* fp32 mode: |gpu - ref| <= 1e-4 * max|ref| + 1e-6

Discrete results (cell order, neighbour sets, iteration counts) are compared
exactly.  Hazards (a residual within 1e-9 of the tolerance) are counted and
reported rather than hidden.
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


def assert_close(name, got, ref, prec, mask=None, scale=None):
    rel, ab = TOL[prec]
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if mask is not None:
        got, ref = got[mask], ref[mask]
    if ref.size == 0:
        return 0.0
    s = np.abs(ref).max() if scale is None else scale
    err = np.abs(got - ref).max()
    bound = rel * s + ab
    assert err <= bound, f"{name}: max|gpu-ref| = {err:.3e} > {bound:.3e} (max|ref| = {s:.3e})"
    return err / max(s, 1e-300)


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
