"""Pins for the oracle's Schwarzschild black-hole problem (Eq. Ham_SBH,
P:L508-533), the paper's first-order test problem (NEXT f1 of SURVEY 8(f)), and
for the canonical sin/cos it needs.  Nothing here compares the oracle with
itself: mpmath evaluates sin/cos, the Hamiltonian of the paper and its exact
derivatives, and an independent 40-digit stage solve; the rest are
invariants the method must keep (energy, time symmetry, order 16)."""
import math

import mpmath as mp
import numpy as np
import pytest

from paper_2511_03655_b200 import workloads as wl
from tests import mp_tableau

EPS = np.finfo(float).eps
SBH = 6
P = [wl.SBH_E, wl.SBH_L, wl.SBH_BETA]


def ulp(x):
    return math.ulp(abs(x)) if x != 0 else 5e-324


# ------------------------------------------------------------ canonical sin/cos
def test_canonical_sincos_within_one_ulp(orc):
    """CANON.md sin/cos (Cody-Waite by pi/2, Taylor degree 19/20) against mpmath at
    40 digits on 4,000 seeded arguments in [-20, 20] plus special points."""
    g = np.random.default_rng(11)
    xs = list(g.uniform(-20, 20, 4000)) + [0.0, -0.0, math.pi / 2, math.pi, 1e-300, 0.7853981633974483,
                                           0.7853981633974484, 1.5707963267948966 + 1e-9]
    with mp.workdps(40):
        for x in xs:
            s, c = orc.sincos(x)
            es, ec = mp.sin(mp.mpf(x)), mp.cos(mp.mpf(x))
            assert abs(s - float(es)) <= ulp(float(es)) + 1e-300, x
            assert abs(c - float(ec)) <= ulp(float(ec)) + 1e-300, x
    assert orc.sincos(0.0) == (0.0, 1.0)
    for x in xs[:200]:
        s1, c1 = orc.sincos(x)
        s2, c2 = orc.sincos(-x)
        assert s2 == -s1 and c2 == c1  # odd / even exactly (reduction and polynomials are symmetric)


# ------------------------------------------------------- Hamilton's equations
def _H_mp(y):
    """Eq. Ham_SBH written out in mpmath."""
    r, th, pr, pth = y
    E, L, beta = (mp.mpf(v) for v in P)
    f = 1 - 2 / r
    s = mp.sin(th)
    return (f * pr ** 2 / 2 - E ** 2 / (2 * f) + pth ** 2 / (2 * r ** 2)
            + (L - beta / 2 * r ** 2 * s ** 2) ** 2 / (2 * r ** 2 * s ** 2))


def test_rhs_is_hamiltons_equations(orc):
    """r' = dH/dp_r, theta' = dH/dp_theta, p_r' = -dH/dr, p_theta' = -dH/dtheta with
    the derivatives of the paper's H taken by mpmath at 40 digits (not from the
    hand-derived formulas), at 40 seeded states; relative 1e-13."""
    g = np.random.default_rng(12)
    with mp.workdps(40):
        for _ in range(40):
            y = [g.uniform(4, 60), g.uniform(0.4, 2.7), g.normal(0, 0.3), g.normal(0, 3)]
            f = orc.rhs(SBH, 4, P, y)
            Y = [mp.mpf(v) for v in y]
            grad = []
            for k in range(4):
                def Hk(x, k=k):
                    Z = list(Y)
                    Z[k] = x
                    return _H_mp(Z)
                grad.append(mp.diff(Hk, Y[k]))
            want = [grad[2], grad[3], -grad[0], -grad[1]]
            scale = max(abs(float(w)) for w in want)
            for k in range(4):
                assert abs(f[k] - float(want[k])) <= 1e-13 * scale, (k, y, f[k], want[k])


def test_energy_matches_paper_hamiltonian_and_ic(orc):
    """The canonical H equals Eq. Ham_SBH (mpmath) to a few ulp; the workload's
    initial conditions lie on the paper's energy shell H = -1/2."""
    w = wl.schwarzschild(batch=16)
    with mp.workdps(40):
        for b in range(w.batch):
            y = w.y[:, b]
            h = orc.energy(SBH, 4, P, y)
            assert abs(h - float(_H_mp([mp.mpf(v) for v in y]))) <= 8 * EPS
            assert abs(h + 0.5) <= 8 * EPS
    assert w.y[0, 0] == 11.0 and w.y[1, 0] == math.pi / 2 and w.y[2, 0] == 0.0 and w.y[3, 0] > 0


# ------------------------------------------------------- integrator behaviour
def test_single_step_vs_mpmath_stage_solve(orc):
    """One first-order step (zero history) at h = 16 vs 200 plain fixed-point
    iterations of Eq. (Yi) with the exact tableau and mpmath's f at 40
    digits: relative 1e-14."""
    w = wl.schwarzschild()
    y0 = w.y[:, 0]
    c, b, A, _ = mp_tableau.tableau(8)
    with mp.workdps(40):
        h = mp.mpf(w.h)
        E, L, beta = (mp.mpf(v) for v in P)

        def f(Y):
            r, th, pr, pth = Y
            s, co = mp.sin(th), mp.cos(th)
            fr = 1 - 2 / r
            Aa = L - beta / 2 * r ** 2 * s ** 2
            return [fr * pr, pth / r ** 2,
                    -(pr ** 2 / r ** 2 + E ** 2 / (r ** 2 * fr ** 2) - pth ** 2 / r ** 3 - beta * Aa / r
                      - Aa ** 2 / (r ** 3 * s ** 2)),
                    beta * Aa * co / s + Aa ** 2 * co / (r ** 2 * s ** 3)]

        y = [mp.mpf(float(v)) for v in y0]
        Ys = [list(y) for _ in range(8)]
        for _ in range(200):
            Fs = [f(Y) for Y in Ys]
            Ys = [[y[l] + h * sum(A[i][j] * Fs[j][l] for j in range(8)) for l in range(4)] for i in range(8)]
        Fs = [f(Y) for Y in Ys]
        y1 = [y[l] + h * sum(b[i] * Fs[i][l] for i in range(8)) for l in range(4)]
    got = orc.integrate(SBH, y0, P, w.h, 1, mode=orc.FIRST_ORDER)["y"]
    for l in range(4):
        assert abs(got[l] - float(y1[l])) <= 1e-14 * max(abs(float(y1[l])), 1.0), (l, got[l], y1[l])


def test_energy_bounded_and_time_reversible(orc):
    """Paper IC, h = 16, 20,000 steps (t = 3.2e5, several radial oscillations
    between r ~ 11 and r ~ 200): max |dH/H| <= 2e-14 with no drift; one step
    +h then -h returns within 10 ulp; the radius stays in the allowed band."""
    w = wl.schwarzschild(nsteps=20000)
    y0 = w.y[:, 0]
    r = orc.integrate(SBH, y0, P, w.h, w.nsteps, mode=orc.FIRST_ORDER, energy_every=50)
    E = r["energy"][:, 0]
    dH = np.abs((E - E[0]) / E[0])
    assert dH.max() <= 2e-14
    half = len(dH) // 2
    assert dH[half:].max() <= 2 * dH[:half].max() + 4 * EPS
    assert r["status"][0, 1] == -1 and r["status"][0, 0] == 0
    r1 = orc.integrate(SBH, y0, P, w.h, 1, mode=orc.FIRST_ORDER)
    r2 = orc.integrate(SBH, r1["y"], P, -w.h, 1, mode=orc.FIRST_ORDER)
    assert np.all(np.abs(r2["y"] - y0) <= 10 * EPS * np.maximum(np.abs(y0), 1.0))


def test_empirical_order_16(orc):
    """Global error at t = 640 against an h = 2.5 reference: halving h from 40 to
    20 divides it by ~2^16 (measured slope 15.5; gate 14.5..17.5, both errors
    above roundoff)."""
    w = wl.schwarzschild()
    y0 = w.y[:, 0]
    T = 640.0
    ref = orc.integrate(SBH, y0, P, 2.5, int(T / 2.5), mode=orc.FIRST_ORDER)["y"]
    errs = []
    for h in (40.0, 20.0):
        yh = orc.integrate(SBH, y0, P, h, int(T / h), mode=orc.FIRST_ORDER)["y"]
        errs.append(np.max(np.abs(yh - ref) / np.maximum(np.abs(ref), 1.0)))
    slope = math.log2(errs[0] / errs[1])
    assert errs[1] > 1e-14, errs
    assert 14.5 < slope < 17.5, (errs, slope)


def test_partitioned_mode_rejected(orc):
    """Eq. Ham_SBH is not separable: the partitioned iteration does not apply."""
    w = wl.schwarzschild()
    with pytest.raises(Exception):
        orc.integrate(SBH, w.y[:, 0], P, w.h, 1)
