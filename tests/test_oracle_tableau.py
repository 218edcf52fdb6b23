"""Pins for the oracle's tableau (PAPER.md P:L109-116 collocation conditions,
P:L139-155 symplecticity and mu rounding, P:L165-178 nu extrapolation).

Each pin compares the oracle with something other than itself: closed forms
(s = 1, 2), an independent mpmath computation (different root finder and
different linear-algebra route), or the order / simplifying conditions the
paper states.
"""
import math

import mpmath as mp
import numpy as np
import pytest

from tests import mp_tableau

mp.mp.dps = 50


def dd(hi, lo):
    return mp.mpf(float(hi)) + mp.mpf(float(lo))


def test_s1_midpoint(orc):
    c, b, mu, nu = orc.tableau(1)
    assert c[0] == 0.5 and b[0] == 1.0 and mu[0, 0] == 0.5 and nu[0, 0] == 0.5


def test_s2_closed_form(orc):
    (ch, cl), (bh, bl), (ah, al), _ = orc.tableau_dd(2)
    r3 = mp.sqrt(3)
    c_ex = [mp.mpf(1) / 2 - r3 / 6, mp.mpf(1) / 2 + r3 / 6]
    a_ex = [[mp.mpf(1) / 4, mp.mpf(1) / 4 - r3 / 6], [mp.mpf(1) / 4 + r3 / 6, mp.mpf(1) / 4]]
    for i in range(2):
        assert abs(dd(ch[i], cl[i]) - c_ex[i]) < 1e-30
        assert abs(dd(bh[i], bl[i]) - mp.mpf(1) / 2) < 1e-30
        for j in range(2):
            assert abs(dd(ah[i, j], al[i, j]) - a_ex[i][j]) < 1e-30
    c, b, mu, nu = orc.tableau(2)
    assert mu[1, 0] == mp_tableau.rn(a_ex[1][0] / mp.mpf(0.5))  # RN(1/2 + sqrt3/3)
    assert mu[0, 1] == 1.0 - mu[1, 0]


@pytest.mark.parametrize("s", [2, 3, 4, 8])
def test_against_independent_mpmath(orc, s):
    c_mp, b_mp, a_mp, nu_mp = mp_tableau.tableau(s)
    (ch, cl), (bh, bl), (ah, al), (nh, nl) = orc.tableau_dd(s)
    for i in range(s):
        assert abs(dd(ch[i], cl[i]) - c_mp[i]) < 1e-30
        assert abs(dd(bh[i], bl[i]) - b_mp[i]) < 1e-30
        for j in range(s):
            assert abs(dd(ah[i, j], al[i, j]) - a_mp[i][j]) < 1e-29
            assert abs(dd(nh[i, j], nl[i, j]) - nu_mp[i][j]) < 1e-24 * max(1, abs(nu_mp[i][j]))
    # fp64 rounding: bitwise RN of the exact values (P:L155 for mu)
    c, b, mu, nu = orc.tableau(s)
    for i in range(s):
        assert c[i] == mp_tableau.rn(c_mp[i])
        assert b[i] == mp_tableau.rn(b_mp[i])
        for j in range(s):
            assert nu[i, j] == mp_tableau.rn(nu_mp[i][j])
            if i > j:
                assert mu[i, j] == mp_tableau.rn(a_mp[i][j] / b_mp[j])


def test_s8_printed_digits(orc):
    """20-digit values of c and b (mpmath 60 digits)."""
    (ch, cl), (bh, bl), _, _ = orc.tableau_dd(8)
    c20 = ["0.019855071751231884158", "0.10166676129318663020", "0.23723379504183550709",
           "0.40828267875217509753", "0.59171732124782490247", "0.76276620495816449291",
           "0.89833323870681336980", "0.98014492824876811584"]
    b20 = ["0.050614268145188129576", "0.11119051722668723527", "0.15685332293894364367",
           "0.18134189168918099148"]
    for i in range(8):
        assert abs(dd(ch[i], cl[i]) - mp.mpf(c20[i])) < 1e-20
    for i in range(4):
        assert abs(dd(bh[i], bl[i]) - mp.mpf(b20[i])) < 1e-20
        assert abs(dd(bh[7 - i], bl[7 - i]) - mp.mpf(b20[i])) < 1e-20


def test_order_conditions_B16_C8_D8(orc):
    """Gauss quadrature of order 2s = 16: B(16) holds, B(17) fails;
    C(8) (the collocation conditions themselves) and D(8)."""
    (ch, cl), (bh, bl), (ah, al), _ = orc.tableau_dd(8)
    c = [dd(ch[i], cl[i]) for i in range(8)]
    b = [dd(bh[i], bl[i]) for i in range(8)]
    a = [[dd(ah[i, j], al[i, j]) for j in range(8)] for i in range(8)]
    for k in range(1, 17):
        assert abs(sum(b[j] * c[j] ** (k - 1) for j in range(8)) - mp.mpf(1) / k) < 1e-29
    assert abs(sum(b[j] * c[j] ** 16 for j in range(8)) - mp.mpf(1) / 17) > 1e-12
    for i in range(8):
        for k in range(1, 9):
            assert abs(sum(a[i][j] * c[j] ** (k - 1) for j in range(8)) - c[i] ** k / k) < 1e-29
    for j in range(8):
        for k in range(1, 9):
            lhs = sum(b[i] * c[i] ** (k - 1) * a[i][j] for i in range(8))
            assert abs(lhs - b[j] * (1 - c[j] ** k) / k) < 1e-29


def test_symplectic_condition_and_mu_identity(orc):
    """Eq. (sym) P:L141 in high precision; the rounded mu~ satisfies
    mu~_ij + mu~_ji = 1 exactly and mu~_ii = 1/2."""
    _, (bh, bl), (ah, al), _ = orc.tableau_dd(8)
    b = [dd(bh[i], bl[i]) for i in range(8)]
    a = [[dd(ah[i, j], al[i, j]) for j in range(8)] for i in range(8)]
    for i in range(8):
        for j in range(8):
            assert abs(b[i] * a[i][j] + b[j] * a[j][i] - b[i] * b[j]) < 1e-30
    c, bb, mu, nu = orc.tableau(8)
    for i in range(8):
        assert mu[i, i] == 0.5
        for j in range(8):
            if i != j:
                assert mu[i, j] + mu[j, i] == 1.0
    # the lower triangle lies in [0.95, 1.09]: 1 - mu~_ji is exact (Sterbenz)
    low = mu[np.tril_indices(8, -1)]
    assert low.min() > 0.95 and low.max() < 1.09


def test_nu_extrapolation(orc):
    """nu reproduces P_{n-1}(t_{n-1} + c_i h) (Eq. Pol0): sum_j nu_ij b_j = c_i,
    and the guess is exact for polynomial trajectories of degree <= 8."""
    (ch, cl), (bh, bl), _, (nh, nl) = orc.tableau_dd(8)
    c = [dd(ch[i], cl[i]) for i in range(8)]
    b = [dd(bh[i], bl[i]) for i in range(8)]
    nu = [[dd(nh[i, j], nl[i, j]) for j in range(8)] for i in range(8)]
    for i in range(8):
        assert abs(sum(nu[i][j] * b[j] for j in range(8)) - c[i]) < 1e-24
    # y(t) = t^p, step n-1 on [-1, 0] (h = 1): L_{n-1,j} = b_j p (c_j - 1)^(p-1),
    # y_{n-1} = 0 -> guess at c_i must equal c_i^p
    for p in range(1, 9):
        for i in range(8):
            g = sum(nu[i][j] * b[j] * p * (c[j] - 1) ** (p - 1) for j in range(8))
            assert abs(g - c[i] ** p) < 1e-22
    _, _, _, nuf = orc.tableau(8)
    assert 3e4 < np.abs(nuf).max() < 4e4


def test_node_weight_symmetry(orc):
    c, b, mu, nu = orc.tableau(8)
    for i in range(8):
        assert abs(c[i] + c[7 - i] - 1.0) <= 2 * np.finfo(float).eps
        assert abs(b[i] - b[7 - i]) <= 2 * np.finfo(float).eps
    assert abs(math.fsum(b) - 1.0) <= 4 * np.finfo(float).eps
    assert np.all(np.diff(c) > 0)
