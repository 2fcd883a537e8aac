"""NEXT-3 square patch (§4.4): the initial-condition series
and the oracle's free-surface dynamics, pinned without the CUDA path."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spl

import synth


def test_initial_pressure_solves_the_poisson_problem():
    # eq:sqp:p with reading R30 must be the solution of lap p = 2 rho omega^2
    # (incompressible rigid rotation: -rho div((u.grad)u) = 2 rho omega^2) with
    # p = 0 on the patch boundary.  Independent check: a 5-point finite-difference
    # solve on a 199 x 199 interior grid (O(h^2) accurate).  A wrong (m pi^2/L)^2
    # denominator, a dropped factor or a sign fails it.
    L, M = 1.0, 199
    hh = L / (M + 1)
    xs = -L / 2 + hh * np.arange(1, M + 1)
    e = np.ones(M)
    T = sp.diags([e[:-1], -2 * e, e[:-1]], [-1, 0, 1]) / hh ** 2
    A = sp.kron(sp.identity(M), T) + sp.kron(T, sp.identity(M))
    omega, rho = 1.3, 2.0
    pfd = spl.spsolve(A.tocsc(), np.full(M * M, 2.0 * rho * omega ** 2))
    X, Y = np.meshgrid(xs, xs, indexing="xy")
    ps = synth.square_patch_pressure(X.ravel(), Y.ravel(), L, omega, rho)
    assert np.abs(ps - pfd).max() < 1e-4 * np.abs(pfd).max()
    # the textbook torsion constant of a square: p(0, 0) = -0.14734 rho omega^2 L^2
    p0 = synth.square_patch_pressure(np.zeros(1), np.zeros(1), L, omega, rho)[0]
    assert p0 == pytest.approx(-0.147343 * rho * omega ** 2 * L ** 2, rel=1e-4)
    # zero on the boundary, symmetric under the square's symmetries
    b = np.linspace(-L / 2, L / 2, 11)
    assert np.abs(synth.square_patch_pressure(b, np.full(11, L / 2), L, omega, rho)).max() < 1e-12
    q = np.random.default_rng(0).uniform(-L / 2, L / 2, (50, 2))
    pa = synth.square_patch_pressure(q[:, 0], q[:, 1], L, omega, rho)
    for qq in (q[:, ::-1], -q, q * [1, -1]):
        assert np.allclose(synth.square_patch_pressure(qq[:, 0], qq[:, 1], L, omega, rho), pa, rtol=1e-12, atol=1e-14)


def _angular_momentum(x, u, m):
    return float(np.sum(m * (x[:, 0] * u[:, 1] - x[:, 1] * u[:, 0])))


def test_oracle_square_patch_symmetry_and_rotation(orc):
    # The lattice and the initial field are point-symmetric ((x, y) -> (-x, -y),
    # u -> -u), so the centre of mass stays at the origin; no external torque
    # acts, so the angular momentum changes only through the asymm pressure
    # gradient's non-conservation (small over a few steps); the free surface is
    # flagged (rho / rho0 < 0.8) on the patch edge only.
    case = synth.square_patch(n=24)
    s = orc.Sim(case)
    m = case.m
    L0 = _angular_momentum(case.x, case.u, m)
    for _ in range(5):
        s.step(case.dt)
    x, u = s.get("x"), s.get("u")
    com = (m[:, None] * x).sum(0) / m.sum()
    assert np.abs(com).max() < 1e-12
    assert _angular_momentum(x, u, m) == pytest.approx(L0, rel=2e-2)
    fs = s.get("fs").astype(bool)
    r = np.abs(case.x).max(1)
    assert fs.any() and not fs[r < 0.3].any()
    # the patch keeps rotating clockwise (omega > 0 with u = omega y, v = -omega x)
    assert _angular_momentum(x, u, m) < 0
