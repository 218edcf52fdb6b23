"""Independent high-precision Gauss-Legendre tableau for the pins (mpmath).

Nodes by mpmath.findroot (secant/Newton) on mpmath.legendre -- not the oracle's
bisection; b, A and nu by dense LU solves of the Vandermonde systems stated in
PAPER.md P:L109-116 (collocation conditions) and the nu-system of reading R-3
(the printed P:L177 is garbled) -- not the oracle's Lagrange-basis
integration.
"""
import functools

import mpmath as mp


@functools.lru_cache(maxsize=None)
def tableau(s=8, dps=60):
    with mp.workdps(dps):
        xs = []
        for i in range(s):
            guess = -mp.cos(mp.pi * (i + 0.75) / (s + 0.5))
            dP = lambda x: s * (x * mp.legendre(s, x) - mp.legendre(s - 1, x)) / (x * x - 1)
            xs.append(mp.findroot(lambda x: mp.legendre(s, x), guess, solver="newton", df=dP,
                                  tol=mp.mpf(10) ** (-2 * dps + 10)))
        xs.sort()
        c = [(1 + x) / 2 for x in xs]
        V = mp.matrix(s, s)
        for k in range(s):
            for j in range(s):
                V[k, j] = c[j] ** k
        b = mp.lu_solve(V, mp.matrix([mp.mpf(1) / (k + 1) for k in range(s)]))
        A = []
        for i in range(s):
            row = mp.lu_solve(V, mp.matrix([c[i] ** (k + 1) / (k + 1) for k in range(s)]))
            A.append([row[j] for j in range(s)])
        W = mp.matrix(s, s)
        for k in range(s):
            for j in range(s):
                W[k, j] = (c[j] - 1) ** k
        nu = []
        for i in range(s):
            at = mp.lu_solve(W, mp.matrix([c[i] ** (k + 1) / (k + 1) for k in range(s)]))
            nu.append([at[j] / b[j] for j in range(s)])
        return c, [b[j] for j in range(s)], A, nu


def rn(x):
    """Round an mpf to the nearest fp64 (ties-to-even, via mpmath's exact rounding)."""
    with mp.workprec(53):
        return float(+x)
