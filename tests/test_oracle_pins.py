"""Pins for the oracle integrator against what the paper and mathematics fix
(DESIGN.md "Pins").  None of these compares the oracle with itself: each uses a
closed form (Pade / modal / Kepler equation), an independent mpmath stage
solve, an invariant the method must conserve, or a worked example from SPEC.md.
"""
import math

import mpmath as mp
import numpy as np
import pytest

from paper_2511_03655_b200 import workloads as wl
from tests import mp_tableau

EPS = np.finfo(float).eps


# --------------------------------------------------------------- stop test
def test_stop_test_spec_examples(orc):
    """Eq. (stopping) P:L243 on SPEC.md's worked examples."""
    assert not orc.stop_test([1e-3, 1e-8, 1e-16, 1e-16])
    assert orc.stop_test([1e-3, 1e-8, 1e-16, 1e-16, 1e-16])
    assert orc.stop_test([0.0])                # Delta = 0 branch
    assert not orc.stop_test([1e-3])
    assert not orc.stop_test([1e-3, 1e-5])     # min branch needs a history
    assert orc.stop_test([1e-5, 1e-3, 1e-3])   # min(1e-5) <= min(1e-3, 1e-3): stagnation
    assert not orc.stop_test([1e-3, 1e-5, 1e-3])  # min(1e-3) > min(1e-5, 1e-3)
    assert not orc.stop_test([1e-3, 1e-5, 1e-7])


# ------------------------------------------------- Pade closed form, order 16
def pade(z, s=8):
    f = mp.factorial
    P = lambda x: sum(f(2 * s - k) * f(s) / (f(2 * s) * f(k) * f(s - k)) * x ** k for k in range(s + 1))
    return P(z) / P(-z)


@pytest.mark.parametrize("div", [2, 3, 4, 128])
def test_harmonic_oscillator_pade(orc, div):
    """Henon-Heiles with lambda = xi = 0 is two harmonic oscillators; the Gauss
    collocation solution of w' = -i w is w_n = R(-ih)^n w_0 with R the (8,8) Pade
    approximant of exp (order 2s = 16).  The converged fixed-point
    iteration must reproduce it to roundoff, while the error against exp grows
    like h^16."""
    mp.mp.dps = 40
    y0 = np.array([0.3, -0.7, 0.5, 0.2])
    h = 2 * math.pi / div
    n = 100 * div
    y = orc.integrate(wl.HENON_HEILES, y0, [0.0, 0.0], h, n)["y"]
    Rn = pade(mp.mpc(0, -mp.mpf(h))) ** n
    for j in range(2):
        w = complex(Rn * mp.mpc(y0[j], y0[2 + j]))
        assert abs(w - complex(y[j], y[2 + j])) < 1e-13


def test_empirical_order_16(orc):
    """Global error vs the exact solution over 100 periods at h = 2pi/2, 2pi/3:
    slope log(e2/e3)/log(3/2) ~ 16 (north star pin (b))."""
    y0 = np.array([0.3, -0.7, 0.5, 0.2])
    errs = []
    for div in (2, 3):
        h = 2 * math.pi / div
        n = 100 * div
        y = orc.integrate(wl.HENON_HEILES, y0, [0.0, 0.0], h, n)["y"]
        t = n * h
        ex = [y0[j] * math.cos(t) + y0[2 + j] * math.sin(t) for j in range(2)]
        errs.append(max(abs(y[j] - ex[j]) for j in range(2)))
    slope = math.log(errs[0] / errs[1]) / math.log(1.5)
    assert 15.0 < slope < 17.0, (errs, slope)


# ----------------------------------------------------------------- free motion
def test_free_motion_two_sweeps(orc):
    """g = 0 (Kepler with GM = 0): positions advance linearly, velocities exact,
    and under reading R2 every step stops at k = 2 with Delta = 0."""
    y0 = np.array([[0.3, -1.0], [0.1, 2.0], [0.25, -0.5], [-0.75, 0.125]])
    r = orc.integrate(wl.KEPLER, y0, [0.0], 0.01, 100)
    assert np.all(r["iters"] == 200)
    assert np.array_equal(r["y"][2:], y0[2:])
    exact = y0[:2] + 100 * 0.01 * y0[2:]
    assert np.allclose(r["y"][:2], exact, rtol=0, atol=50 * EPS * 2)


# -------------------------------------------------- SPEC single-step, mpmath
def test_single_step_vs_mpmath_stage_solve(orc):
    """Henon-Heiles, h = 2pi/68: one step (zero history) vs 200 plain fixed-point
    iterations of Eq. (Yi) with the exact tableau at 40 digits
    (SPEC S:L267 asks 1e-14; gate 1e-15 relative)."""
    w = wl.henon_heiles()
    y0 = w.y[:, 0]
    h = mp.mpf(w.h)
    c, b, A, _ = mp_tableau.tableau(8)
    with mp.workdps(40):
        y = [mp.mpf(float(v)) for v in y0]

        def f(Y):
            q1, q2, p1, p2 = Y
            return [p1, p2, -q1 - 2 * q1 * q2, -q2 - (q1 * q1 - q2 * q2)]

        Ys = [list(y) for _ in range(8)]
        for _ in range(200):
            Fs = [f(Y) for Y in Ys]
            Ys = [[y[l] + h * sum(A[i][j] * Fs[j][l] for j in range(8)) for l in range(4)]
                  for i in range(8)]
        Fs = [f(Y) for Y in Ys]
        y1 = [y[l] + h * sum(b[i] * Fs[i][l] for i in range(8)) for l in range(4)]
    got = orc.integrate(wl.HENON_HEILES, y0, w.params, w.h, 1)["y"]
    for l in range(4):
        assert abs(got[l] - float(y1[l])) <= 1e-15 * max(abs(float(y1[l])), 1e-300) + 1e-17


# ------------------------------------------------------------- reversibility
def test_time_reversibility(orc):
    """Symmetry of Gauss methods: a step with h then one with -h (fresh
    history) returns to y0 within a few ulp; 1280 steps (10 periods) each way
    within the roundoff random walk with linear phase growth (5e-12)."""
    w = wl.kepler_single()
    y0 = w.y[:, 0]
    r1 = orc.integrate(w.problem, y0, w.params, w.h, 1)
    r2 = orc.integrate(w.problem, r1["y"], w.params, -w.h, 1)
    assert np.max(np.abs(r2["y"] - y0)) < 10 * EPS * 2
    r1 = orc.integrate(w.problem, y0, w.params, w.h, 1280)
    r2 = orc.integrate(w.problem, r1["y"], w.params, -w.h, 1280)
    assert np.max(np.abs(r2["y"] - y0)) < 5e-12


# ---------------------------------------------------------- Kepler invariants
def _kepler_LH(y):
    q1, q2, v1, v2 = y
    return q1 * v2 - q2 * v1, 0.5 * (v1 * v1 + v2 * v2) - 1.0 / np.sqrt(q1 * q1 + q2 * q2)


def test_kepler_config1_energy_bounded_no_drift(orc):
    """Config 1 over 100 periods: max |dH/H| <= 1e-13 and no drift (second-half
    max <= 2x first-half max, or LSQ slope <= 2e-16 per time unit);
    H0 = -1/2, L = sqrt(3)/2 closed forms."""
    w = wl.kepler_single()
    L0, H0 = _kepler_LH(w.y[:, 0])
    assert abs(H0 + 0.5) < 1e-15 and abs(L0 - math.sqrt(3) / 2) < 1e-15
    r = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=16)
    e = r["energy"][:, 0]
    assert abs(e[0] + 0.5) < 1e-15
    dh = (e - e[0]) / e[0]
    assert np.abs(dh).max() <= 1e-13
    half = len(dh) // 2
    t = np.arange(len(dh)) * 16 * w.h
    slope = np.polyfit(t, dh, 1)[0]
    assert np.abs(dh[half:]).max() <= 2 * np.abs(dh[:half]).max() or abs(slope) <= 2e-16
    L1, _ = _kepler_LH(r["y"][:, 0])
    assert abs(L1 - L0) / L0 < 1e-13
    assert r["status"][0, 0] == 0  # no MAX_ITERS hits


def test_kepler_angular_momentum_quadratic_invariant(orc):
    """Gauss methods conserve quadratic invariants exactly; at e = 0.9 and
    config-2 h the energy error is truncation-dominated but L drifts only by
    roundoff (catches a wrong mu rounding or a non-converged stop)."""
    a, e = 0.5, 0.9
    rp = a * (1 - e)
    vp = math.sqrt((1 + e) / rp)
    y0 = np.array([rp, 0.0, 0.0, vp])
    r = orc.integrate(wl.KEPLER, y0, [1.0], wl.KEPLER_T_MIN / 128, 10000)
    L0, H0 = _kepler_LH(y0)
    L1, H1 = _kepler_LH(r["y"])
    assert abs(H1 - H0) / abs(H0) > 1e-8          # truncation visible in energy
    assert abs(L1 - L0) / abs(L0) < 1e-13         # but L conserved to roundoff


def test_kepler_vs_kepler_equation(orc):
    """Config-1 orbit over one period vs the closed-form solution from Kepler's
    equation E - e sin E = M (Newton in mpmath)."""
    w = wl.kepler_single()
    n = 128
    y = orc.integrate(w.problem, w.y, w.params, w.h, 64)["y"][:, 0]  # half a period
    mp.mp.dps = 30
    e, a = mp.mpf("0.5"), mp.mpf(1)
    M = mp.mpf(w.h) * 64          # mean motion 1
    E = mp.findroot(lambda E: E - e * mp.sin(E) - M, M)
    x = a * (mp.cos(E) - e)
    yy = a * mp.sqrt(1 - e * e) * mp.sin(E)
    Edot = 1 / (1 - e * mp.cos(E))
    vx = -a * mp.sin(E) * Edot
    vy = a * mp.sqrt(1 - e * e) * mp.cos(E) * Edot
    ex = [float(x), float(yy), float(vx), float(vy)]
    assert n == 128
    assert np.max(np.abs(y - ex)) < 1e-13


# ------------------------------------------------------------ nu independence
def test_nu_guess_only_changes_iteration_count(orc):
    """Replacing the nu-extrapolated guess (Eq. IRK_init2) by the zero-history
    guess at every step changes only the sweep count, not the converged result
    (<= 1e-10 relative after 12,800 steps; SURVEY C-10 item 9)."""
    w = wl.kepler_single()
    ref = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps)
    y = w.y.copy()
    sweeps = 0
    for n in range(w.nsteps):
        r = orc.integrate(w.problem, y, w.params, w.h, 1, n0=n)
        y = r["y"]
        sweeps += int(r["iters"][0])
    rel = np.max(np.abs(y - ref["y"])) / np.max(np.abs(ref["y"]))
    assert rel <= 1e-10
    assert sweeps > 1.5 * ref["iters"][0]


# --------------------------------------------------------- chunk continuity
def test_chunked_run_is_bitwise_continuous(orc):
    """(y, L_{n-1}, n) is the whole state: two chunks == one run, bitwise."""
    w = wl.kepler_ensemble(batch=8, nsteps=300)
    one = orc.integrate(w.problem, w.y, w.params, w.h, 300)
    a = orc.integrate(w.problem, w.y, w.params, w.h, 120)
    b = orc.integrate(w.problem, a["y"], w.params, w.h, 180, n0=120, hist=a["hist"])
    assert np.array_equal(one["y"], b["y"])
    assert np.array_equal(one["iters"], a["iters"] + b["iters"])


# ----------------------------------------------------------- FPU beta = 0
def test_fpu_linear_modal_closed_form(orc):
    """FPU with beta = 0 is linear: mode k (DST-I) has omega_k = 2 sin(k pi/(2(N+1)))
    and the Gauss solution is w_n = R(-i h omega)^n w_0, w = omega Q + i V."""
    N = 8
    g = np.random.default_rng(11)
    y0 = np.concatenate([g.standard_normal(N), g.standard_normal(N)])
    h, n = 0.1, 1000
    y = orc.integrate(wl.FPU_BETA, y0, [0.0], h, n)["y"]
    idx = np.arange(1, N + 1)
    S = np.sqrt(2 / (N + 1)) * np.sin(np.pi * np.outer(idx, idx) / (N + 1))  # orthogonal
    mp.mp.dps = 30
    Q0, V0, Q1, V1 = S @ y0[:N], S @ y0[N:], S @ y[:N], S @ y[N:]
    for k in range(N):
        om = 2 * math.sin((k + 1) * math.pi / (2 * (N + 1)))
        w = complex(pade(mp.mpc(0, -h * om)) ** n * mp.mpc(om * Q0[k], V0[k]))
        assert abs(w - complex(om * Q1[k], V1[k])) < 1e-12


# ------------------------------------------------------------------ N-body
def test_nbody_momentum_and_angular_momentum(orc):
    """Eq. Ham2: total linear momentum and (quadratic) angular momentum
    are conserved to roundoff; energy error bounded."""
    w = wl.six_body_ensemble(batch=2, nsteps=2000)
    m = w.params[2:]
    r = orc.integrate(w.problem, w.y, w.params, w.h, 2000, energy_every=1000)
    for b in range(2):
        def PL(y):
            q = y[:18].reshape(6, 3); v = y[18:].reshape(6, 3)
            return (m[:, None] * v).sum(0), (m[:, None] * np.cross(q, v)).sum(0)
        P0, L0 = PL(w.y[:, b]); P1, L1 = PL(r["y"][:, b])
        assert np.max(np.abs(P1 - P0)) < 1e-15
        assert np.max(np.abs(L1 - L0)) < 1e-13 * np.abs(L0).max()
        e = r["energy"][:, b]
        assert abs((e[-1] - e[0]) / e[0]) < 1e-12


def test_two_body_reduces_to_kepler(orc):
    """N-body with masses (1, 1e-3, 0, ...): bodies 0-1 are a Kepler problem in
    relative coordinates with GM = G(m0+m1); compare with Kepler's equation."""
    m0, m1 = 1.0, 1e-3
    N = 3
    GM = m0 + m1
    a, e = 1.0, 0.3
    rp = a * (1 - e)
    vp = math.sqrt(GM * (1 + e) / rp)
    q = np.zeros((N, 3)); v = np.zeros((N, 3))
    q[1] = [rp, 0, 0]; v[1] = [0, vp, 0]
    q[2] = [5.0, 1.0, 0.5]; v[2] = [0.0, 0.1, 0.0]
    cm = (m0 * q[0] + m1 * q[1]) / GM; cv = (m0 * v[0] + m1 * v[1]) / GM
    q -= cm; v -= cv
    y0 = np.concatenate([q.reshape(-1), v.reshape(-1)])
    nmean = math.sqrt(GM / a ** 3)
    T = 2 * math.pi / nmean
    h = T / 256
    y = orc.integrate(wl.NBODY, y0, [1.0, 0.0, m0, m1, 0.0], h, 100)["y"]
    rel = y[3:6] - y[0:3]
    mp.mp.dps = 30
    M = mp.mpf(nmean) * mp.mpf(h) * 100
    E = mp.findroot(lambda E: E - e * mp.sin(E) - M, M)
    x = a * (mp.cos(E) - e); yy = a * mp.sqrt(1 - e * e) * mp.sin(E)
    assert abs(rel[0] - float(x)) < 1e-13 and abs(rel[1] - float(yy)) < 1e-13 and rel[2] == 0


# ------------------------------------------------ RHS = -grad U (FD of H)
@pytest.mark.parametrize("problem,dim,params", [
    (wl.KEPLER, 4, [1.3]),
    (wl.HENON_HEILES, 4, [0.7, 0.0]),
    (wl.FPU_BETA, 16, [1.0]),
    (wl.NBODY, 18, [1.0, 0.0, 1.0, 0.5, 0.25]),
    (wl.NBODY_DIRECT, 18, [1.0, 0.05, 1.0, 0.5, 0.25]),
])
def test_rhs_is_minus_grad_U(orc, problem, dim, params):
    """For H = T(v) + U(q), the accelerations g(q) = -M^-1 grad U (Eq. sHam,
    P:L258-260): central finite differences of the oracle's own H."""
    g = np.random.default_rng(5)
    d = dim // 2
    masses = np.ones(d) if problem not in (wl.NBODY, wl.NBODY_DIRECT) else np.repeat(params[2:], 3)
    for _ in range(5):
        q = g.uniform(0.5, 1.5, d) * g.choice([-1, 1], d)
        if problem in (wl.NBODY, wl.NBODY_DIRECT):
            q = g.standard_normal(d) * 2
        a = orc.accel(problem, dim, params, q)
        for l in range(d):
            hh = 1e-5
            qp, qm = q.copy(), q.copy()
            qp[l] += hh; qm[l] -= hh
            yp = np.concatenate([qp, np.zeros(d)]); ym = np.concatenate([qm, np.zeros(d)])
            grad = (orc.energy(problem, dim, params, yp) - orc.energy(problem, dim, params, ym)) / (2 * hh)
            assert abs(a[l] + grad / masses[l]) <= 1e-6 * max(1.0, abs(a[l]))


def test_direct_and_pair_nbody_agree(orc):
    """The two canonical N-body sequences (cyclic pairs, blocked direct sum)
    evaluate the same formula Eq. Ham2: agree to a few ulp of the force scale."""
    g = np.random.default_rng(9)
    N = 40
    q = g.standard_normal(3 * N)
    P = np.concatenate([[1.0, 0.01], g.uniform(0.1, 1, N)])
    a1 = orc.accel(wl.NBODY, 6 * N, P, q)
    a2 = orc.accel(wl.NBODY_DIRECT, 6 * N, P, q)
    assert np.max(np.abs(a1 - a2)) < 1e-12 * np.max(np.abs(a1))


# ---------------------------------------------------- energies, closed forms
def test_energy_closed_forms(orc):
    w = wl.kepler_single()
    assert abs(orc.energy(w.problem, 4, w.params, w.y[:, 0]) + 0.5) < 1e-15
    hh = wl.henon_heiles()
    assert abs(orc.energy(hh.problem, 4, hh.params, hh.y[:, 0]) - 1 / 12) < 1e-15
    assert abs(hh.y[2, 0] - math.sqrt(41 / 750)) < 1e-15
    # FPU: lowest mode of amplitude 1, beta = 1 -> H = sum_b (D^2/2 + D^4/4), D_b closed form
    N = 64
    n = np.arange(1, N + 1)
    y = np.concatenate([np.sin(np.pi * n / (N + 1)), np.zeros(N)])
    Db = np.diff(np.concatenate([[0], np.sin(np.pi * n / (N + 1)), [0]]))
    om1 = 2 * math.sin(math.pi / (2 * (N + 1)))
    H2 = 0.5 * om1 ** 2 * (N + 1) / 2   # sum sin^2 over n = (N+1)/2
    assert abs(math.fsum(0.5 * Db ** 2) - H2) < 1e-14
    assert abs(orc.energy(wl.FPU_BETA, 2 * N, [1.0], y) - (H2 + math.fsum(0.25 * Db ** 4))) < 1e-14
    assert abs(H2 - 0.0379) < 1e-3


def test_first_order_mode_same_fixed_point(orc):
    """Eqs. IRK_FP and IRK_FP2 solve the same stage equations (Yi2): at small h*omega
    the first-order iteration reaches the partitioned result to roundoff."""
    w = wl.henon_heiles(batch=3, h=0.05, nsteps=200)
    a = orc.integrate(w.problem, w.y, w.params, w.h, 200)
    b = orc.integrate(w.problem, w.y, w.params, w.h, 200, mode=orc.FIRST_ORDER)
    assert np.max(np.abs(a["y"] - b["y"])) < 1e-13
    assert b["iters"].sum() >= a["iters"].sum()


def test_divergence_is_flagged(orc):
    """A trajectory that blows up is frozen and flagged with its step index."""
    y0 = np.array([[1e-200, 1.0], [0.0, 0.0], [0.0, 0.0], [0.0, 1.0]])
    r = orc.integrate(wl.KEPLER, y0, [1.0], 0.1, 20)
    assert r["status"][0, 1] >= 1           # q = 1e-200 -> r^3 underflows -> inf/nan
    assert r["status"][1, 1] == -1


def test_argument_errors(orc):
    with pytest.raises(ValueError):
        orc.integrate(wl.KEPLER, np.zeros(6), [1.0], 0.1, 1)
    with pytest.raises(ValueError):
        orc.integrate(wl.KEPLER, np.zeros(4), [1.0], 0.0, 1)
    with pytest.raises(ValueError):
        orc.integrate(wl.NBODY_DIRECT, np.zeros(12), [1.0, 0.0, 1.0, 1.0], 0.1, 1)


def test_local_energy_error_pins(orc):
    """Eq. DHlocmax: for the harmonic oscillator the Gauss solution
    conserves the quadratic energy exactly, so Delta H^loc_max is roundoff
    (<= 4 ulp); for Henon-Heiles at the paper's h = 2 pi/68 it is at
    roundoff level too, while a coarse h shows the truncation error."""
    y0 = np.array([0.3, -0.7, 0.5, 0.2])
    r = orc.integrate(wl.HENON_HEILES, y0, [0.0, 0.0], 2 * math.pi / 8, 400, local_energy=True)
    assert r["dhloc"][0] <= 4 * EPS
    w = wl.henon_heiles(nsteps=2000)
    r = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, local_energy=True)
    assert r["dhloc"][0] < 5e-15
    errs = [orc.integrate(w.problem, w.y, w.params, 2 * math.pi / div, 20 * div, local_energy=True)["dhloc"][0]
            for div in (3, 4, 6)]
    assert errs[0] > 1e-9 and errs[0] > 50 * errs[1] > 2500 * errs[2]   # truncation ~ h^(2s+1) shrinking
    # the value is the max over steps of |(H_n - H_{n-1}) / H_{n-1}| (checked step by step)
    y = w.y[:, 0].copy()
    hmax = 0.0
    hist = None
    for n in range(50):
        rr = orc.integrate(w.problem, y, w.params, w.h, 1, n0=n, hist=hist)
        h0 = orc.energy(w.problem, 4, w.params, y)
        h1 = orc.energy(w.problem, 4, w.params, rr["y"])
        hmax = max(hmax, abs((h1 - h0) / h0))
        y, hist = rr["y"], rr["hist"]
    r3 = orc.integrate(w.problem, w.y, w.params, w.h, 50, local_energy=True)
    assert r3["dhloc"][0] == hmax
