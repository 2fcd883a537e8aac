"""Seeded synthetic workloads shaped like the paper's test cases.

This module is shared by the oracle tests and the CUDA path.  It holds NO part of
the method's arithmetic (no kernel, no neighbour search, no pressure solve): it
only lays particles on lattices, applies the seeded jitter, evaluates the
*initial conditions* the paper prints, and records the scheme parameters each
case uses.  Everything returned is plain numpy (fp64 / int32).

Case recipes (SURVEY.md §8(d) "Synthetic inputs"):

* ``tgv2d``   — PAPER.md:931-946 §4.1 eq:tgv (BASELINE configs[0]).
* ``hydrostatic`` — BASELINE configs[1]; wall layout of PAPER.md:808-813 §3.4.
* ``dambreak2d``  — PAPER.md:1352-1371 §4.5 (BASELINE configs[2]).
* ``tgv3d``   — BASELINE configs[3] (not in the paper; standard 3D TG field).
* ``dambreak3d``  — PAPER.md:1407-1428 §4.6, per-GPU slab of BASELINE configs[4].

Lattice sites sit at (i + 1/2) dx with x fastest; jitter is
``numpy.random.default_rng(seed).uniform(-a, a, (N, dim))`` in lattice order,
then wrapped into periodic boxes.  Masses are rho0 * dx**dim for every particle
(fluid and wall); initial density is rho0.  Tags: 0 fluid, 1 wall.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

FLUID = 0
WALL = 1

# pressure-gradient forms (PAPER.md:320-339 eq:mom:sph:press:symm / :pij)
PGRAD_SYMM = 0
PGRAD_ASYMM = 1


@dataclass
class Case:
    """A synthetic workload: particles, domain, scheme parameters, timestep."""

    name: str
    dim: int
    h: float
    dx: float
    dt: float
    steps: int
    lo: list
    hi: list
    periodic: list
    x: np.ndarray          # (n, dim) fp64
    u: np.ndarray          # (n, dim) fp64
    m: np.ndarray          # (n,) fp64
    rho: np.ndarray        # (n,) fp64
    p: np.ndarray          # (n,) fp64
    tag: np.ndarray        # (n,) int32
    params: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.x.shape[0])

    @property
    def n_fluid(self) -> int:
        return int((self.tag == FLUID).sum())

    @property
    def n_wall(self) -> int:
        return int((self.tag == WALL).sum())


def default_params(**kw) -> dict:
    """Scheme parameters with the paper's defaults.

    omega=0.5, tol=1e-2, max_iter=1000 and
    min_iter=2, eta=0.01, free-surface
    ratio 0.8, K=10 GTVF sub-steps (reading R22).
    """
    p = dict(
        rho0=1.0, nu=0.0, g=[0.0, 0.0, 0.0], alpha=0.0, c_ref=0.0,
        omega=0.5, tol=1e-2, max_iter=1000, min_iter=2, K=10,
        pgrad=PGRAD_SYMM, h_tilde_factor=1.0, pref_external=0, p_ref=0.0,
        ustar_noslip=0, clamp_wall_p=0, fs_ratio=0.8, eta=0.01, precision=64,
        conv_mean=1,   # reading R12b: eq:convergence on means (reproduces Table 1)
    )
    p.update(kw)
    return p


def _lattice(counts, dx, origin):
    """Sites (i + 1/2) dx + origin, x fastest.  counts = (nx, ny[, nz])."""
    axes = [origin[a] + (np.arange(c) + 0.5) * dx for a, c in enumerate(counts)]
    grids = np.meshgrid(*axes[::-1], indexing="ij")  # slowest first
    pts = np.stack([g.ravel() for g in grids[::-1]], axis=1)
    return pts


def _jitter(x, amp, seed, lo, hi, periodic):
    if amp <= 0:
        return x
    rng = np.random.default_rng(seed)
    x = x + rng.uniform(-amp, amp, x.shape)
    for a in range(x.shape[1]):
        if periodic[a]:
            L = hi[a] - lo[a]
            x[:, a] = np.where(x[:, a] >= hi[a], x[:, a] - L, x[:, a])
            x[:, a] = np.where(x[:, a] < lo[a], x[:, a] + L, x[:, a])
    return x


def _pad3(v):
    v = list(v)
    return v + [0.0] * (3 - len(v))


# --------------------------------------------------------------------------
# C1  2D Taylor-Green vortex (§4.1, eq:tgv)
# --------------------------------------------------------------------------
def tgv2d(n: int = 50, re: float = 100.0, jitter: float = 0.1, seed: int = 101,
          steps: int = 10, tol: float = 1e-4, K: int = 10, precision: int = 64, mean_free: int = 1) -> Case:
    L, U, rho0 = 1.0, 1.0, 1.0
    dx = L / n
    h = dx  # h/dx = 1.0
    nu = U * L / re
    lo, hi, per = [0.0, 0.0], [L, L], [1, 1]
    x = _lattice((n, n), dx, lo)
    x = _jitter(x, jitter * dx, seed, lo, hi, per)
    X, Y = x[:, 0], x[:, 1]
    # eq:tgv at t = 0
    u = np.stack([-U * np.cos(2 * np.pi * X) * np.sin(2 * np.pi * Y),
                  U * np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y)], axis=1)
    p = -U * U * (np.cos(4 * np.pi * X) + np.cos(4 * np.pi * Y)) / 4.0
    npart = x.shape[0]
    # fixed dt = min(0.25 h/U, 0.25 h^2/nu)
    dt = min(0.25 * h / U, 0.25 * h * h / nu)
    # internal flow: p_ref = 2 max(p) (reading R22); max p = U^2/2
    # fully periodic: the PPE has no Dirichlet row and the printed Jacobi drifts along its
    # constant null space (reading R32): the mean-free projection is the configured default
    params = default_params(rho0=rho0, nu=nu, pgrad=PGRAD_ASYMM, h_tilde_factor=1.0,
                            pref_external=0, p_ref=2.0 * 0.5 * rho0 * U * U, tol=tol, K=K,
                            precision=precision, ppe_mean_free=mean_free)
    return Case("tgv2d", 2, h, dx, dt, steps, _pad3(lo), _pad3(hi), per + [0], x, u,
                np.full(npart, rho0 * dx * dx), np.full(npart, rho0), p,
                np.zeros(npart, np.int32), params)


# --------------------------------------------------------------------------
# walled 2D tanks (hydrostatic column, dam break)
# --------------------------------------------------------------------------
def _tank2d(nfx, nfy, tank_nx, wall_ny, layers, dx):
    """Fluid block nfx x nfy at the tank's lower-left corner; walls: floor
    (spanning the whole tank incl. corners) and both sides up to wall_ny rows."""
    fluid = _lattice((nfx, nfy), dx, (0.0, 0.0))
    walls = []
    # floor: y = -(l + 1/2) dx, x = (i + 1/2) dx for i in [-layers, tank_nx + layers)
    xs = (np.arange(-layers, tank_nx + layers) + 0.5) * dx
    for l in range(layers):
        walls.append(np.stack([xs, np.full_like(xs, -(l + 0.5) * dx)], axis=1))
    ys = (np.arange(wall_ny) + 0.5) * dx
    for l in range(layers):
        walls.append(np.stack([np.full_like(ys, -(l + 0.5) * dx), ys], axis=1))
        walls.append(np.stack([np.full_like(ys, tank_nx * dx + (l + 0.5) * dx), ys], axis=1))
    return fluid, np.concatenate(walls, axis=0)


def hydrostatic(nx: int = 200, ny: int = 400, dx: float = 0.005, layers: int = 3,
                steps: int = 500, tol: float = 1e-3, K: int = 10, precision: int = 32,
                gtvf: bool = False) -> Case:
    """BASELINE configs[1]: 1.0 x 2.0 column at dx=0.005, 3 dummy-wall layers."""
    rho0, gmag = 1000.0, 9.81
    h = dx
    H = ny * dx
    wall_ny = int(round(1.05 * H / dx))  # side walls up to 1.05 H (2.1 m for H = 2)
    fluid, wall = _tank2d(nx, ny, nx, wall_ny, layers, dx)
    x = np.concatenate([fluid, wall])
    nf, nw = fluid.shape[0], wall.shape[0]
    tag = np.concatenate([np.zeros(nf, np.int32), np.ones(nw, np.int32)])
    c_ref = 10.0 * math.sqrt(2 * gmag * H)     # c = 10 |u|max, |u|max ~ sqrt(2 g H)
    dt = 0.125 * h / math.sqrt(2 * gmag * H)   # PAPER.md:1365-1366 formula
    # BASELINE configs[1] asks for no background-pressure homogenisation: p_ref = 0
    # (p0 = min(10|p|, 0) = 0, so the GTVF shift vanishes; reading R22a)
    params = default_params(rho0=rho0, g=[0.0, -gmag, 0.0], alpha=0.05, c_ref=c_ref,
                            pgrad=PGRAD_SYMM, h_tilde_factor=0.5, pref_external=1,
                            p_ref=0.0 if not gtvf else rho0 * c_ref * c_ref, ustar_noslip=0,
                            clamp_wall_p=1, tol=tol, K=K, precision=precision)
    lo = [-(layers + 0.5) * dx, -(layers + 0.5) * dx, 0.0]
    hi = [nx * dx + (layers + 0.5) * dx, 1.1 * H + 4 * dx, 0.0]
    n = nf + nw
    return Case("hydrostatic", 2, h, dx, dt, steps, lo, hi, [0, 0, 0], x,
                np.zeros((n, 2)), np.full(n, rho0 * dx * dx), np.full(n, rho0),
                np.zeros(n), tag, params)


def dambreak2d(nx: int = 500, ny: int = 1000, dx: float = 0.002, tank: float = 4.0,
               layers: int = 4, steps: int = 1000, tol: float = 1e-2, K: int = 10,
               precision: int = 32) -> Case:
    """BASELINE configs[2] / PAPER.md:1352-1371: 1 x 2 block in a 4 x 4 tank."""
    rho0, gmag = 1000.0, 9.81
    h = 1.3 * dx                     # h/dx = 1.3
    hw = ny * dx
    tank_nx = int(round(tank / dx))
    fluid, wall = _tank2d(nx, ny, tank_nx, tank_nx, layers, dx)
    x = np.concatenate([fluid, wall])
    nf, nw = fluid.shape[0], wall.shape[0]
    tag = np.concatenate([np.zeros(nf, np.int32), np.ones(nw, np.int32)])
    p = np.concatenate([rho0 * gmag * (hw - fluid[:, 1]), np.zeros(nw)])  # reading R29
    c_ref = 10.0 * math.sqrt(2 * gmag * hw)
    dt = 0.125 * h / math.sqrt(2 * gmag * hw)
    params = default_params(rho0=rho0, g=[0.0, -gmag, 0.0], alpha=0.05, c_ref=c_ref,
                            pgrad=PGRAD_SYMM, h_tilde_factor=0.5, pref_external=1,
                            p_ref=rho0 * c_ref * c_ref, ustar_noslip=0, clamp_wall_p=1,
                            tol=tol, K=K, precision=precision)
    lo = [-(layers + 0.5) * dx, -(layers + 0.5) * dx, 0.0]
    hi = [tank_nx * dx + (layers + 0.5) * dx, tank_nx * dx + 4 * dx, 0.0]
    n = nf + nw
    return Case("dambreak2d", 2, h, dx, dt, steps, lo, hi, [0, 0, 0], x,
                np.zeros((n, 2)), np.full(n, rho0 * dx * dx), np.full(n, rho0), p, tag, params)


# --------------------------------------------------------------------------
# NEXT-4 moving walls: plane Couette flow and the lid-driven cavity
# --------------------------------------------------------------------------
def couette_velocity(y, t, U, H, nu, terms: int = 200):
    """Start-up plane Couette flow, lower plate at rest, upper plate impulsively
    moved at U (a textbook closed form; the test's reference, not part of the
    method): u(y, t) = U y/H - (2U/pi) sum_n (-1)^(n+1)/n sin(n pi y/H) exp(-n^2 pi^2 nu t/H^2)."""
    y = np.asarray(y, np.float64)
    u = U * y / H
    for k in range(1, terms + 1):
        u -= 2.0 * U / np.pi * (-1) ** (k + 1) / k * np.sin(k * np.pi * y / H) * np.exp(
            -(k * np.pi) ** 2 * nu * t / (H * H))
    return u


def couette(nx: int = 10, ny: int = 20, H: float = 1.0, U: float = 1.0, re: float = 10.0,
            layers: int = 3, steps: int = 100, tol: float = 1e-3, K: int = 10,
            precision: int = 64) -> Case:
    """Channel of height H = ny dx between two wall blocks of `layers` rows,
    periodic in x (length nx dx); the upper wall moves at +U along x (its
    creation velocity is its prescribed velocity, eq:vg-adami P:845-846), the
    lower wall is at rest; fluid at rest, p = 0, no body force.  Internal flow:
    symm gradient without GTVF (p_ref = 0: P:1244-1246 says "symm" works
    without it), no-slip u* on the walls."""
    rho0 = 1.0
    dx = H / ny
    h = dx
    nu = U * H / re
    L = nx * dx
    fluid = _lattice((nx, ny), dx, (0.0, 0.0))
    xs = (np.arange(nx) + 0.5) * dx
    low = [np.stack([xs, np.full_like(xs, -(l + 0.5) * dx)], 1) for l in range(layers)]
    top = [np.stack([xs, np.full_like(xs, H + (l + 0.5) * dx)], 1) for l in range(layers)]
    wall = np.concatenate(low + top)
    x = np.concatenate([fluid, wall])
    nf, nw = fluid.shape[0], wall.shape[0]
    tag = np.concatenate([np.zeros(nf, np.int32), np.ones(nw, np.int32)])
    u = np.zeros((nf + nw, 2))
    u[nf + nw // 2:, 0] = U                      # the upper wall block slides at U
    dt = min(0.25 * h / U, 0.25 * h * h / nu)
    params = default_params(rho0=rho0, nu=nu, pgrad=PGRAD_SYMM, h_tilde_factor=1.0, pref_external=0,
                            p_ref=0.0, ustar_noslip=1, tol=tol, K=K, precision=precision)
    lo = [0.0, -(layers + 0.5) * dx, 0.0]
    hi = [L, H + (layers + 0.5) * dx, 0.0]
    n = nf + nw
    return Case("couette", 2, h, dx, dt, steps, lo, hi, [1, 0, 0], x, u,
                np.full(n, rho0 * dx * dx), np.full(n, rho0), np.zeros(n), tag, params)


def cavity(n: int = 50, re: float = 100.0, U: float = 1.0, layers: int = 3, t_end: float = 10.0,
           tol: float = 1e-2, K: int = 10, precision: int = 64, ustar_noslip: int = 0) -> Case:
    """Lid-driven cavity (§4.3): unit square of n x n fluid
    particles, h/dx = 1, Re = U L / nu; the lid (every wall particle above the
    fluid, corners included) moves at +U along x, the other walls are at rest.
    Internal flow: symm gradient, GTVF with p_ref = 2 max(p_i) after the first
    solve (reading R33); u* slip by default; eq:convergence on
    means (reading R12b: with the printed sums the enclosed cavity at 50 x 50 runs
    tens of sweeps per step and voids at the upper corners)."""
    rho0, L = 1.0, 1.0
    dx = L / n
    h = dx
    nu = U * L / re
    fluid, wall = _tank2d(n, n, n, n, layers, dx)
    xs = (np.arange(-layers, n + layers) + 0.5) * dx
    lid = np.concatenate([np.stack([xs, np.full_like(xs, L + (l + 0.5) * dx)], 1) for l in range(layers)])
    wall = np.concatenate([wall, lid])
    x = np.concatenate([fluid, wall])
    nf, nw = fluid.shape[0], wall.shape[0]
    tag = np.concatenate([np.zeros(nf, np.int32), np.ones(nw, np.int32)])
    u = np.zeros((nf + nw, 2))
    u[nf + nw - lid.shape[0]:, 0] = U
    dt = min(0.25 * h / U, 0.25 * h * h / nu)
    params = default_params(rho0=rho0, nu=nu, pgrad=PGRAD_SYMM, h_tilde_factor=1.0, pref_external=0,
                            p_ref=0.0, pref_auto=1, conv_mean=1, ustar_noslip=ustar_noslip, tol=tol, K=K,
                            precision=precision)
    lo = [-(layers + 0.5) * dx, -(layers + 0.5) * dx, 0.0]
    hi = [L + (layers + 0.5) * dx, L + (layers + 0.5) * dx, 0.0]
    nn = nf + nw
    return Case("cavity", 2, h, dx, dt, int(round(t_end / dt)), lo, hi, [0, 0, 0], x, u,
                np.full(nn, rho0 * dx * dx), np.full(nn, rho0), np.zeros(nn), tag, params)


# --------------------------------------------------------------------------
# NEXT-4b open boundaries: channel with an inlet and an outlet
# --------------------------------------------------------------------------
INLET = 2
OUTLET = 3
DORMANT = 4


def poiseuille_velocity(y, U, H):
    """fully developed plane channel flow with mean velocity U (textbook closed form):
    u(y) = 6 U y (H - y) / H^2"""
    y = np.asarray(y, np.float64)
    return 6.0 * U * y * (H - y) / (H * H)


def channel(nx: int = 40, ny: int = 10, H: float = 1.0, U: float = 1.0, re: float = 10.0, n_in: int = 4,
            n_out: int = 4, n_pool: int | None = None, layers: int = 3, t_end: float = 10.0, tol: float = 1e-3,
            precision: int = 64, nz: int = 0) -> Case:
    """Plane channel of height H (ny particles across) between two resting walls.
    Inlet region x in [-n_in dx, 0): tag 2 with the developed (parabolic, mean U)
    profile as prescribed velocity; fluid x in [0, nx dx) and the outlet region
    [nx dx, (nx + n_out) dx) (tag 3, frozen until they leave at x_end) start
    with the same profile.  n_pool dormant particles (tag 4)
    hold the ids new inlet particles are drawn from (reading R34).  Re = U H / nu,
    asymm gradient (the frozen outlet pressures ratchet the absolute level
    upward with the flow; eq:mom:sph:press:pij is blind to it), internal-flow
    GTVF with p_ref = 2 max p after the first solve (R33: without it the liquid
    count drifts and the profile error reaches 8 % by t = 10 H / U; with it 2.5 %),
    no-slip u* on the walls.  nz > 0: a 3D channel, periodic in z
    over nz particles (the same plane flow in every z layer)."""
    rho0 = 1.0
    dx = H / ny
    h = dx
    nu = U * H / re
    Lf = nx * dx
    L_in, L_out = n_in * dx, n_out * dx
    d3 = nz > 0
    ext = (nz,) if d3 else ()
    org = (0.0,) if d3 else ()
    fluid = _lattice((nx, ny) + ext, dx, (0.0, 0.0) + org)
    inlet = _lattice((n_in, ny) + ext, dx, (-L_in, 0.0) + org)
    outlet = _lattice((n_out, ny) + ext, dx, (Lf, 0.0) + org)
    n_pool = 2 * n_in * ny * max(nz, 1) if n_pool is None else n_pool
    pool = _lattice((n_in, ny) + ext, dx, (-L_in, 0.0) + org)
    pool = np.concatenate([pool] * (n_pool // len(pool) + 1))[:n_pool]
    nwx = n_in + nx + n_out + 2 * layers
    walls = []
    for l in range(layers):
        for yl in (-(l + 0.5) * dx, H + (l + 0.5) * dx):
            w = _lattice((nwx, 1) + ext, dx, (-(n_in + layers) * dx, 0.0) + org)
            w[:, 1] = yl
            walls.append(w)
    wall = np.concatenate(walls)
    x = np.concatenate([fluid, inlet, outlet, wall, pool])
    tag = np.concatenate([np.zeros(len(fluid), np.int32), np.full(len(inlet), INLET, np.int32),
                          np.full(len(outlet), OUTLET, np.int32), np.ones(len(wall), np.int32),
                          np.full(len(pool), DORMANT, np.int32)])
    n = len(x)
    u = np.zeros((n, 3 if d3 else 2))
    # the developed profile everywhere (inlet prescribed, fluid and outlet initial): the
    # steady state is the initial state, and the open boundaries must keep it
    liq = (tag == INLET) | (tag == OUTLET) | (tag == FLUID)
    u[liq, 0] = poiseuille_velocity(x[liq, 1], U, H)
    umax = 1.5 * U
    dt = min(0.25 * h / umax, 0.25 * h * h / nu)
    params = default_params(rho0=rho0, nu=nu, pgrad=PGRAD_ASYMM, h_tilde_factor=1.0, pref_external=0, p_ref=0.0,
                            pref_auto=1, ustar_noslip=1, tol=tol, precision=precision, open_x=1, x_inlet=0.0, x_outlet=Lf,
                            x_end=Lf + L_out, inlet_length=L_in)
    lo = [-L_in - (layers + 0.5) * dx, -(layers + 0.5) * dx, 0.0]
    hi = [Lf + L_out + (layers + 0.5) * dx, H + (layers + 0.5) * dx, nz * dx if d3 else 0.0]
    dim = 3 if d3 else 2
    return Case("channel", dim, h, dx, dt, int(round(t_end / dt)), lo, hi, [0, 0, 1 if d3 else 0], x, u,
                np.full(n, rho0 * dx ** dim), np.full(n, rho0), np.zeros(n), tag, params)


def cylinder(D: float = 2.0, re: float = 200.0, U: float = 1.0, ppd: int = 30, h_ratio: float = 1.2,
             up: float = 5.0, down: float = 10.0, half_width: float = 7.5, n_in: int = 4, n_out: int = 4,
             layers: int = 4, t_end: float = 200.0, tol: float = 1e-2, precision: int = 64,
             n_pool: int | None = None, jitter: float = 0.05, seed: int = 1504,
             p_ref: float | None = None) -> Case:
    """Flow past a circular cylinder (§4.7): D = 2, Re = U D / nu = 200,
    dx = D / ppd (30: 200 k fluid particles), h / dx = 1.2, cylinder centre 5D behind
    the inlet (uniform U, tag 2), outlet (tag 3) 10D behind the centre, eps = 0.01,
    symm, no artificial viscosity, external
    GTVF with p_ref = rho c^2, c = 10 |U|max, h~ = h / 2.  The cylinder is
    `layers` rings of wall particles inside the circumference, the outer ring dx/2
    inside it, each ring evenly spaced at about dx.  Reading
    R35: the slip side walls at +-7.5D become a periodic y axis of width
    15D (no slip-wall construction for the viscous ghost velocity here); the same
    blockage ratio D / 15D.  And the fluid starts as the uniform stream U instead of
    impulsively from rest: with the fluid at rest the inlet's first pressure spike
    drives a GTVF shift (p0 = min(10|p|, rho c^2)) past the single build's skin."""
    rho0 = 1.0
    dx = D / ppd
    h = h_ratio * dx
    nu = U * D / re
    R = 0.5 * D
    xc = up * D
    L_in, L_out = n_in * dx, n_out * dx
    x_out = xc + down * D
    W = 2.0 * half_width * D
    nx = int(round(x_out / dx))
    ny = int(round(W / dx))
    fl = _lattice((nx, ny), dx, (0.0, -half_width * D))
    outside = (fl[:, 0] - xc) ** 2 + fl[:, 1] ** 2 >= (R + 0.5 * dx) ** 2 - 1e-12   # dx/2 gap to the surface
    fl = fl[outside]
    # a seeded jitter breaks the set-up's mirror symmetry about y = 0 (a perfectly symmetric,
    # deterministic start delays the shedding indefinitely)
    fl = _jitter(fl, jitter * dx, seed, [0.0, -half_width * D], [x_out, half_width * D], [0, 1])
    inlet = _lattice((n_in, ny), dx, (-L_in, -half_width * D))
    n_pool = 2 * n_in * ny if n_pool is None else n_pool
    pool = np.concatenate([inlet] * (n_pool // len(inlet) + 1))[:n_pool]
    rings = []
    for l in range(layers):
        r = R - (l + 0.5) * dx
        if r <= 0:
            break
        m = max(int(round(2 * np.pi * r / dx)), 3)
        th = 2 * np.pi * (np.arange(m) + 0.5) / m
        rings.append(np.stack([xc + r * np.cos(th), r * np.sin(th)], 1))
    wall = np.concatenate(rings)
    x = np.concatenate([fl, inlet, wall, pool])
    tag = np.concatenate([np.zeros(len(fl), np.int32), np.full(len(inlet), INLET, np.int32),
                          np.ones(len(wall), np.int32), np.full(len(pool), DORMANT, np.int32)])
    n = len(x)
    u = np.zeros((n, 2))
    u[(tag == INLET) | (tag == 0), 0] = U     # R35: a uniform stream at t = 0 (see below)
    umax = 1.5 * U
    dt = min(0.25 * h / umax, 0.25 * h * h / nu)
    c_ref = 10.0 * umax
    # p_ref: the paper's rho c^2 unless given; R22c: the GTVF sub-steps are an
    # undamped oscillator over one step and need dt sqrt(p0 / rho) / h~ <~ 1 (here p0 <~ 9)
    params = default_params(rho0=rho0, nu=nu, pgrad=PGRAD_SYMM, h_tilde_factor=0.5, pref_external=1,
                            p_ref=rho0 * c_ref * c_ref if p_ref is None else p_ref, c_ref=c_ref, ustar_noslip=0,
                            tol=tol, precision=precision,
                            open_x=1, x_inlet=0.0, x_outlet=x_out, x_end=x_out + L_out, inlet_length=L_in)
    lo = [-L_in - 4 * h, -half_width * D, 0.0]
    hi = [x_out + L_out + 4 * h, half_width * D, 0.0]
    return Case("cylinder", 2, h, dx, dt, int(round(t_end / dt)), lo, hi, [0, 1, 0], x, u,
                np.full(n, rho0 * dx * dx), np.full(n, rho0), np.zeros(n), tag, params)


# --------------------------------------------------------------------------
# C4  3D Taylor-Green vortex (BASELINE configs[3])
# --------------------------------------------------------------------------
def tgv3d(n: int = 128, re: float = 100.0, jitter: float = 0.05, seed: int = 104,
          steps: int = 100, tol: float = 1e-3, K: int = 10, precision: int = 32, mean_free: int = 1) -> Case:
    L, U, rho0 = 2.0 * np.pi, 1.0, 1.0
    dx = L / n
    h = dx
    nu = 0.01 if re == 100.0 else U * 1.0 / re
    lo, hi, per = [0.0] * 3, [L] * 3, [1, 1, 1]
    x = _lattice((n, n, n), dx, lo)
    x = _jitter(x, jitter * dx, seed, lo, hi, per)
    X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
    u = np.stack([np.sin(X) * np.cos(Y) * np.cos(Z),
                  -np.cos(X) * np.sin(Y) * np.cos(Z),
                  np.zeros_like(X)], axis=1)
    p = rho0 / 16.0 * (np.cos(2 * X) + np.cos(2 * Y)) * (np.cos(2 * Z) + 2.0)  # reading R29
    npart = x.shape[0]
    dt = min(0.25 * h / U, 0.25 * h * h / nu)
    # internal flow: p_ref = 2 max(p) (reading R22); max p = 3/16 rho U^2
    # fully periodic: mean-free Jacobi (reading R32), as tgv2d
    params = default_params(rho0=rho0, nu=nu, pgrad=PGRAD_ASYMM, h_tilde_factor=1.0,
                            pref_external=0, p_ref=2.0 * 3.0 / 16.0 * rho0 * U * U, tol=tol,
                            K=K, precision=precision, ppe_mean_free=mean_free)
    return Case("tgv3d", 3, h, dx, dt, steps, lo, hi, per, x, u,
                np.full(npart, rho0 * dx ** 3), np.full(npart, rho0), p,
                np.zeros(npart, np.int32), params)


# --------------------------------------------------------------------------
# C5  3D dam break, per-GPU slab (BASELINE configs[4])
# --------------------------------------------------------------------------
def dambreak3d(nfx: int = 256, nfy: int = 64, nfz: int = 128, dx: float = 1.0 / 256,
               tank_nx: int = 824, wall_nz: int = 154, layers: int = 3, ranks: int = 1,
               steps: int = 100, tol: float = 1e-2, K: int = 10, precision: int = 32) -> Case:
    """Water block nfx*dx x (ranks*nfy*dx) x nfz*dx at the x=0 end of a tank of
    length tank_nx*dx, open top, y periodic (spanwise; the slab axis).  Walls:
    floor under the whole tank and both x-end walls up to wall_nz rows."""
    rho0, gmag = 1000.0, 9.81
    h = dx                                   # h/dx = 1.0
    ny = nfy * ranks
    Ly = ny * dx
    hw = nfz * dx
    fluid = _lattice((nfx, ny, nfz), dx, (0.0, 0.0, 0.0))
    walls = []
    ys = (np.arange(ny) + 0.5) * dx
    xs = (np.arange(-layers, tank_nx + layers) + 0.5) * dx
    for l in range(layers):                  # floor z = -(l + 1/2) dx
        X, Y = np.meshgrid(xs, ys, indexing="xy")
        walls.append(np.stack([X.ravel(), Y.ravel(), np.full(X.size, -(l + 0.5) * dx)], 1))
    zs = (np.arange(wall_nz) + 0.5) * dx
    for l in range(layers):                  # end walls x = -(l+1/2)dx and L + (l+1/2)dx
        for xw in (-(l + 0.5) * dx, tank_nx * dx + (l + 0.5) * dx):
            Y, Z = np.meshgrid(ys, zs, indexing="xy")
            walls.append(np.stack([np.full(Y.size, xw), Y.ravel(), Z.ravel()], 1))
    wall = np.concatenate(walls)
    x = np.concatenate([fluid, wall])
    nf, nw = fluid.shape[0], wall.shape[0]
    tag = np.concatenate([np.zeros(nf, np.int32), np.ones(nw, np.int32)])
    p = np.concatenate([rho0 * gmag * (hw - fluid[:, 2]), np.zeros(nw)])  # reading R29
    v_ref = math.sqrt(2 * gmag * hw)
    c_ref = 10.0 * v_ref
    dt = h / (8.0 * v_ref)
    params = default_params(rho0=rho0, g=[0.0, 0.0, -gmag], alpha=0.25, c_ref=c_ref,
                            pgrad=PGRAD_SYMM, h_tilde_factor=0.5, pref_external=1,
                            p_ref=rho0 * c_ref * c_ref, ustar_noslip=0, clamp_wall_p=1,
                            tol=tol, K=K, precision=precision)
    lo = [-(layers + 0.5) * dx, 0.0, -(layers + 0.5) * dx]
    hi = [tank_nx * dx + (layers + 0.5) * dx, Ly, 2.0 * hw + 4 * dx]
    n = nf + nw
    return Case("dambreak3d", 3, h, dx, dt, steps, lo, hi, [0, 1, 0], x,
                np.zeros((n, 3)), np.full(n, rho0 * dx ** 3), np.full(n, rho0), p, tag, params)


# --------------------------------------------------------------------------
# NEXT-3  square patch (§4.4, eq:sqp:vel, eq:sqp:p)
# --------------------------------------------------------------------------
def square_patch_pressure(x, y, L: float = 1.0, omega: float = 1.0, rho: float = 1.0, nterms: int = 80):
    """Initial pressure of the rotating square patch, eq:sqp:p:
        p0 = rho sum_{m, n odd} -32 omega^2 / (m n pi^2 [(n pi / L)^2 + (m pi / L)^2])
                                 sin(m pi x* / L) sin(n pi y* / L),   x* = x + L/2, y* = y + L/2.
    The printed (m pi^2 / L)^2 is read as (m pi / L)^2 (reading R30: the series must solve
    lap p = 2 rho omega^2 with p = 0 on the patch boundary, which fixes the symmetric form).
    nterms odd values of m and of n (the coefficients fall as 1/(m n (m^2 + n^2)))."""
    k = 2 * np.arange(nterms) + 1.0                          # 1, 3, 5, ...
    xs, ys = np.asarray(x) + L / 2, np.asarray(y) + L / 2
    Sx = np.sin(np.pi * np.outer(xs, k) / L)                # (N, M)
    Sy = np.sin(np.pi * np.outer(ys, k) / L)
    C = -32.0 * omega ** 2 / (np.outer(k, k) * np.pi ** 2 * ((np.pi / L) ** 2 * (k[None, :] ** 2 + k[:, None] ** 2)))
    return rho * np.einsum("im,mn,in->i", Sx, C, Sy)


def square_patch(n: int = 100, L: float = 1.0, omega: float = 1.0, h_ratio: float = 1.3, alpha: float = 0.15,
                 steps: int = 100, tol: float = 1e-2, K: int = 10, precision: int = 64,
                 box: float = 4.0) -> Case:
    """An L x L patch of fluid centred at the origin rotating rigidly (eq:sqp:vel:
    u0 = omega y, v0 = -omega x) with the balancing pressure eq:sqp:p; no walls, free
    surface everywhere (100 x 100, h/dx = 1.3, alpha = 0.15,
    epsilon = 1e-2, asymm pressure gradient)."""
    rho0 = 1.0
    dx = L / n
    h = h_ratio * dx
    x = _lattice((n, n), dx, (-L / 2, -L / 2))
    u = np.stack([omega * x[:, 1], -omega * x[:, 0]], axis=1)
    p = square_patch_pressure(x[:, 0], x[:, 1], L, omega, rho0)
    umax = omega * L / math.sqrt(2.0)
    c_ref = 10.0 * umax                      # c = 10 |u|max
    dt = 0.25 * h / umax                     # CFL
    params = default_params(rho0=rho0, alpha=alpha, c_ref=c_ref, pgrad=PGRAD_ASYMM, h_tilde_factor=0.5,
                            pref_external=1, p_ref=rho0 * c_ref * c_ref, tol=tol, K=K, precision=precision)
    lo, hi = [-box * L / 2, -box * L / 2], [box * L / 2, box * L / 2]
    npart = x.shape[0]
    return Case("square_patch", 2, h, dx, dt, steps, _pad3(lo), _pad3(hi), [0, 0, 0], x, u,
                np.full(npart, rho0 * dx * dx), np.full(npart, rho0), p, np.zeros(npart, np.int32), params)


def lattice_periodic(dim: int, n: int, dx: float = 1.0, h_ratio: float = 1.0,
                     jitter: float = 0.0, seed: int = 7, rho0: float = 1.0) -> Case:
    """A resting periodic lattice (used for lattice identities and invariants)."""
    L = n * dx
    lo, hi, per = [0.0] * dim, [L] * dim, [1] * dim
    x = _lattice((n,) * dim, dx, lo)
    x = _jitter(x, jitter * dx, seed, lo, hi, per)
    npart = x.shape[0]
    params = default_params(rho0=rho0, p_ref=0.0, K=1)
    return Case(f"lattice{dim}d", dim, h_ratio * dx, dx, 1e-3, 1, _pad3(lo), _pad3(hi),
                per + [0] * (3 - dim), x, np.zeros((npart, dim)),
                np.full(npart, rho0 * dx ** dim), np.full(npart, rho0), np.zeros(npart),
                np.zeros(npart, np.int32), params)


def random_box(dim: int, n: int, L: float, h: float, seed: int, periodic) -> Case:
    """Uniform random particles in [0, L)^dim (neighbour-search fuzzing)."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, L, (n, dim))
    lo, hi = [0.0] * dim, [L] * dim
    per = list(periodic)[:dim]
    params = default_params()
    return Case("random", dim, h, L / max(n, 1) ** (1.0 / dim), 1e-3, 1, _pad3(lo), _pad3(hi),
                per + [0] * (3 - dim), x, np.zeros((n, dim)), np.ones(n), np.ones(n),
                np.zeros(n), np.zeros(n, np.int32), params)


CASES = {
    "tgv2d": tgv2d,
    "hydrostatic": hydrostatic,
    "dambreak2d": dambreak2d,
    "tgv3d": tgv3d,
    "dambreak3d": dambreak3d,
}
