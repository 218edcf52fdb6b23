"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes binding of the scalar-C IRKGL16 oracle (oracle/irk_oracle.c), written
from arXiv 2511.03655 (Sec. 2, Eqs. Yi2/yn3/IRK_init2/IRK_FP2/stopping).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It shares no code with the CUDA path.

Parity unpinned ("Pins"): the exact sweep index at which each
step stops has no external reference; its effect on the result is pinned to
roundoff by the Pade, nu-independence and single-step mpmath pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "irk_oracle.c")
LIB = os.path.join(HERE, "build", "liboracle.so")

KEPLER, NBODY, FPU_BETA, HENON_HEILES, NBODY_DIRECT, SCHWARZSCHILD = 1, 2, 3, 4, 5, 6
PARTITIONED, FIRST_ORDER = 0, 1

# -O2 without vectorisation or contraction: every op is the one written (CANON.md)
CFLAGS = ["-O2", "-fno-tree-vectorize", "-ffp-contract=off", "-fno-fast-math",
          "-fopenmp", "-fPIC", "-shared", "-Wall", "-Wextra"]

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc).  Returns its path."""
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "irk_oracle.h"))):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Cfg(ctypes.Structure):
    _fields_ = [("problem", ctypes.c_int), ("dim", ctypes.c_int), ("mode", ctypes.c_int),
                ("max_iters", ctypes.c_int), ("h", ctypes.c_double), ("t0", ctypes.c_double),
                ("nsteps", ctypes.c_int64), ("batch", ctypes.c_int64), ("n0", ctypes.c_int64),
                ("energy_every", ctypes.c_int64), ("params", ctypes.POINTER(ctypes.c_double)),
                ("nparams", ctypes.c_int), ("nthreads", ctypes.c_int),
                ("dhloc", ctypes.POINTER(ctypes.c_double))]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            l = ctypes.CDLL(build())
            dp = ctypes.POINTER(ctypes.c_double)
            ip = ctypes.POINTER(ctypes.c_int64)
            l.orc_tableau.argtypes = [ctypes.c_int, dp, dp, dp, dp]
            l.orc_tableau_dd.argtypes = [ctypes.c_int] + [dp] * 8
            l.orc_stop_test.argtypes = [dp, ctypes.c_int]
            l.orc_accel.argtypes = [ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, ctypes.c_double, dp, dp]
            l.orc_energy.argtypes = [ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, dp]
            l.orc_rhs.argtypes = [ctypes.c_int, ctypes.c_int, dp, ctypes.c_int, ctypes.c_double, dp, dp]
            l.orc_sincos.argtypes = [ctypes.c_double, dp, dp]
            l.orc_sincos.restype = None
            l.orc_energy.restype = ctypes.c_double
            l.orc_integrate.argtypes = [ctypes.POINTER(_Cfg), dp, dp, dp, ip, ip]
            _lib = l
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def tableau(s: int = 8):
    """fp64 (c, b, mu, nu) with the symplectic rounding of P:L155."""
    c, b = np.zeros(s), np.zeros(s)
    mu, nu = np.zeros((s, s)), np.zeros((s, s))
    if lib().orc_tableau(s, _dp(c), _dp(b), _dp(mu), _dp(nu)):
        raise RuntimeError("orc_tableau failed")
    return c, b, mu, nu


def tableau_dd(s: int = 8):
    """Unrounded __float128 (c, b, a, nu) as double-double (hi, lo) pairs."""
    arrs = [np.zeros(s), np.zeros(s), np.zeros(s), np.zeros(s),
            np.zeros((s, s)), np.zeros((s, s)), np.zeros((s, s)), np.zeros((s, s))]
    if lib().orc_tableau_dd(s, *[_dp(a) for a in arrs]):
        raise RuntimeError("orc_tableau_dd failed")
    c = (arrs[0], arrs[1]); b = (arrs[2], arrs[3]); a = (arrs[4], arrs[5]); nu = (arrs[6], arrs[7])
    return c, b, a, nu


def stop_test(deltas) -> bool:
    d = _f64(deltas)
    return bool(lib().orc_stop_test(_dp(d), len(d)))


def accel(problem: int, dim: int, params, q, t: float = 0.0):
    p = _f64(params); q = _f64(q); a = np.zeros(dim // 2)
    if lib().orc_accel(problem, dim, _dp(p), len(p), t, _dp(q), _dp(a)):
        raise ValueError("orc_accel: bad problem/dim/params")
    return a


def rhs(problem: int, dim: int, params, y, t: float = 0.0):
    """Full first-order f(t, y) of one state (Hamilton's equations for SCHWARZSCHILD)."""
    p = _f64(params); y = _f64(y); f = np.zeros(dim)
    if lib().orc_rhs(problem, dim, _dp(p), len(p), t, _dp(y), _dp(f)):
        raise ValueError("orc_rhs: bad problem/dim/params")
    return f


def sincos(x: float):
    """The canonical (sin x, cos x) of CANON.md."""
    s = np.zeros(1); c = np.zeros(1)
    lib().orc_sincos(float(x), _dp(s), _dp(c))
    return float(s[0]), float(c[0])


def energy(problem: int, dim: int, params, y) -> float:
    p = _f64(params); y = _f64(y)
    return float(lib().orc_energy(problem, dim, _dp(p), len(p), _dp(y)))


def integrate(problem: int, y, params, h: float, nsteps: int, *, t0: float = 0.0, n0: int = 0,
              hist=None, mode: int = PARTITIONED, max_iters: int = 100, energy_every: int = 0,
              nthreads: int = 0, local_energy: bool = False):
    """Run the oracle.  y: SoA (dim, batch) (a 1-D y is one trajectory).

    Returns dict(y, hist, energy, iters, status) -- y in the input's shape,
    hist (batch, 8, dim), energy ((nsteps//E)+1, batch) or None, iters (batch,),
    status (batch, 3) = {maxiter_hits, diverged_step (-1), last_step_sweeps},
    dhloc (batch,) = max local relative energy error (Eq. DHlocmax) if local_energy.
    """
    y = _f64(y)
    one = y.ndim == 1
    Y = np.array(y.reshape(-1, 1) if one else y, dtype=np.float64, order="C")
    dim, batch = Y.shape
    H = (np.zeros((batch, 8, dim)) if hist is None else np.array(hist, dtype=np.float64, order="C"))
    assert H.shape == (batch, 8, dim)
    p = _f64(params)
    E = np.zeros(((nsteps // energy_every) + 1, batch)) if energy_every > 0 else None
    it = np.zeros(batch, dtype=np.int64)
    st = np.zeros((batch, 3), dtype=np.int64)
    dhl = np.zeros(batch) if local_energy else None
    cfg = _Cfg(problem, dim, mode, max_iters, h, t0, nsteps, batch, n0, energy_every,
               _dp(p), len(p), nthreads, _dp(dhl) if dhl is not None else None)
    rc = lib().orc_integrate(ctypes.byref(cfg), _dp(Y), _dp(H),
                             _dp(E) if E is not None else None,
                             it.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                             st.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    if rc:
        raise ValueError("orc_integrate: argument error")
    return dict(y=Y[:, 0] if one else Y, hist=H, energy=E, iters=it, status=st, dhloc=dhl)
