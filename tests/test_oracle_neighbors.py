"""Pins of the oracle's neighbour sets and cell order (A1-A5, reading R2, R26, R27).

* The cell-list neighbour search equals an O(N^2) brute force on >= 50 random
  configurations, periodic and bounded (SURVEY.md §8(c) pins).
* Perfect-lattice counts equal the number of integer points strictly inside
  the support sphere (enumerated here independently).
* The cell order is a stable sort: keys non-decreasing, ties in input order,
  and every particle lies inside the cell its key names.
"""
import itertools

import numpy as np
import pytest

import synth


def _sets(off, nbr):
    return [tuple(nbr[off[i]:off[i + 1]]) for i in range(len(off) - 1)]


@pytest.mark.parametrize("seed", range(50))
def test_cell_list_equals_brute_force(orc, seed):
    rng = np.random.default_rng(1000 + seed)
    dim = 2 if seed % 2 == 0 else 3
    n = int(rng.integers(20, 400 if dim == 2 else 300))
    L = 1.0
    h = float(rng.uniform(L / 30, L / 9.5))  # >= 3 cells per axis (3h <= L/3)
    per = [int(b) for b in rng.integers(0, 2, dim)]
    case = synth.random_box(dim, n, L, h, seed, per)
    if seed % 5 == 0:  # put exact ties at R on a lattice-aligned subset
        case.x[: n // 2] = np.round(case.x[: n // 2] / h) * h % L
    cfg = orc.make_cfg(dim, case.lo, case.hi, case.periodic, h)
    a = orc.neighbors(cfg, case.x)
    b = orc.neighbors(cfg, case.x, brute=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # symmetric relation, no self pairs
    S = _sets(*a)
    for i, s in enumerate(S):
        assert i not in s
        for j in s:
            assert i in S[j]


@pytest.mark.parametrize("dim,h_ratio,expect", [(2, 1.0, 24), (2, 1.3, 44), (3, 1.0, 92)])
def test_perfect_lattice_counts(orc, dim, h_ratio, expect):
    # integer points v != 0 with |v|^2 < (3 h/dx)^2, counted by enumeration
    R2 = (3 * h_ratio) ** 2
    rng = range(-4, 5)
    count = sum(1 for v in itertools.product(rng, repeat=dim)
                if any(v) and sum(c * c for c in v) < R2 - 1e-9)
    assert count == expect
    n = 12 if dim == 2 else 10
    case = synth.lattice_periodic(dim, n, dx=1.0, h_ratio=h_ratio)
    cfg = orc.make_cfg(dim, case.lo, case.hi, case.periodic, case.h)
    off, nbr = orc.neighbors(cfg, case.x)
    assert (np.diff(off) == expect).all()


def test_cell_order_is_stable_sort(orc):
    for dim, per in ((2, [1, 1]), (2, [0, 0]), (3, [1, 0, 1])):
        case = synth.random_box(dim, 3000, 1.0, 0.04, 11 + dim, per)
        # also particles outside a bounded box (clamped to edge cells)
        if not per[0]:
            case.x[:10, 0] = -0.3
            case.x[10:20, 0] = 1.7
        cfg = orc.make_cfg(dim, case.lo, case.hi, case.periodic, case.h)
        order, keys = orc.cell_order(cfg, case.x)
        assert sorted(order.tolist()) == list(range(case.n))
        ks = keys[order]
        assert (np.diff(ks) >= 0).all()
        ties = np.diff(ks) == 0
        assert (np.diff(order)[ties] > 0).all()
        nc, cl = orc.cell_geometry(cfg)
        assert all(cl[a] >= 3 * case.h for a in range(dim))
        c = np.stack([keys % nc[0], (keys // nc[0]) % nc[1], keys // (nc[0] * nc[1])], 1)
        for a in range(dim):
            f = (case.x[:, a] - case.lo[a]) / cl[a]
            inside = (f >= 0) & (f < nc[a])
            assert (c[inside, a] == np.floor(f[inside])).all()
            assert (c[~inside, a] == np.clip(np.floor(f[~inside]), 0, nc[a] - 1)).all()
