"""Pins of the oracle's smoothing kernel (reading R1: M6 quintic spline).

Each value below is fixed by mathematics, not by the oracle: normalisation
(integral of W over its support is 1), W(0) = 66 sigma_d / h^d, the derivative
against a central finite difference, compact support at 3h, continuity of the
piecewise polynomial.  SPEC.md's printed 2D gradient at q = 1 (0.34644) is a
slip; the closed form is 50 * 7 / (478 pi) = 0.2330721.
"""
import math

import numpy as np
import pytest
from scipy import integrate


@pytest.mark.parametrize("dim,h", [(2, 1.0), (2, 0.013), (3, 1.0), (3, 0.02)])
def test_normalisation(orc, dim, h):
    # integral over R^d of W(|r|) = 1  (radial quadrature, breakpoints at q = 1, 2)
    area = (lambda r: 2 * math.pi * r) if dim == 2 else (lambda r: 4 * math.pi * r * r)
    tot = sum(integrate.quad(lambda r: orc.W(dim, r, h) * area(r), a * h, (a + 1) * h,
                             epsabs=0, epsrel=1e-13)[0] for a in range(3))
    assert abs(tot - 1.0) < 1e-11


def test_values_at_origin(orc):
    # W(0) = sigma (3^5 - 6*2^5 + 15) = 66 sigma
    assert orc.W(2, 0.0, 1.0) == pytest.approx(66 * 7 / (478 * math.pi), rel=1e-14)
    assert orc.W(3, 0.0, 1.0) == pytest.approx(66 / (120 * math.pi), rel=1e-14)
    assert orc.W(2, 0.0, 1.0) == pytest.approx(0.3076552, abs=1e-7)
    assert orc.W(3, 0.0, 1.0) == pytest.approx(0.1750704, abs=1e-7)
    assert orc.W(2, 0.0, 0.5) == pytest.approx(4 * orc.W(2, 0.0, 1.0), rel=1e-14)
    assert orc.W(3, 0.0, 0.5) == pytest.approx(8 * orc.W(3, 0.0, 1.0), rel=1e-14)


def test_gradient_closed_form_q1(orc):
    # dW/dq at q=1 (2D, h=1) = -5 sigma (2^4 - 6) = -50 sigma
    assert orc.dWdr(2, 1.0, 1.0) == pytest.approx(-50 * 7 / (478 * math.pi), rel=1e-14)
    assert orc.dWdr(2, 1.0, 1.0) == pytest.approx(-0.2330721, abs=1e-7)


@pytest.mark.parametrize("dim", [2, 3])
def test_gradient_matches_finite_difference(orc, dim):
    h = 0.37
    rng = np.random.default_rng(3)
    for r in rng.uniform(0.01, 2.99, 200) * h:
        e = 1e-6 * h
        fd = (orc.W(dim, r + e, h) - orc.W(dim, r - e, h)) / (2 * e)
        ref = orc.dWdr(dim, r, h)
        assert abs(fd - ref) <= 1e-7 * max(abs(ref), orc.W(dim, 0, h) / h * 1e-3)


@pytest.mark.parametrize("dim", [2, 3])
def test_compact_support_and_continuity(orc, dim):
    h = 1.0
    assert orc.W(dim, 3.0, h) == 0.0 and orc.dWdr(dim, 3.0, h) == 0.0
    assert orc.W(dim, 3.5, h) == 0.0 and orc.dWdr(dim, 7.0, h) == 0.0
    for q in (1.0, 2.0):
        e = 1e-9
        assert abs(orc.W(dim, q - e, h) - orc.W(dim, q + e, h)) < 1e-8
        assert abs(orc.dWdr(dim, q - e, h) - orc.dWdr(dim, q + e, h)) < 1e-8
    # W >= 0 and monotone decreasing on [0, 3h)
    r = np.linspace(0, 3, 301)
    w = np.array([orc.W(dim, x, h) for x in r])
    assert (w >= 0).all() and (np.diff(w) <= 1e-15).all()
