"""Seeded synthetic workloads for the five BASELINE.json configs.

This module is the ONE thing the CUDA path and the oracle share: it draws
initial conditions and parameters with numpy's PCG64 and holds none of the
method's arithmetic (no tableau, no stage solve, no right-hand side).  The
recipe for each config is stated in DESIGN.md ("Input recipe"); the paper's own
workloads (outer Solar System with DE430 data) are not in the
container, so config 3 is a synthetic stand-in of the same size and structure.

Layout: y is SoA with shape (dim, batch); component
order (q_1..q_d, v_1..v_d) as in Listing 2; N-body positions are
body-major xyz (the (3,N) VecArray of P:L394).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

KEPLER, NBODY, FPU_BETA, HENON_HEILES, NBODY_DIRECT, SCHWARZSCHILD = 1, 2, 3, 4, 5, 6

SEEDS = {1: 1, 2: 2, 3: 3, 4: 4, 5: 5}


@dataclass
class Workload:
    name: str
    problem: int
    dim: int
    y: np.ndarray            # (dim, batch) float64, SoA
    params: np.ndarray       # float64
    h: float
    nsteps: int
    t0: float = 0.0
    meta: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return self.y.shape[1]


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def kepler_single() -> Workload:
    """Config 1: planar Kepler, GM=1, e=0.5, a=1, at pericentre; h=2pi/128, 12,800 steps."""
    y = np.array([[0.5], [0.0], [0.0], [math.sqrt(3.0)]])
    return Workload("kepler_single", KEPLER, 4, y, np.array([1.0]), 2 * math.pi / 128, 12800)


KEPLER_T_MIN = 2 * math.pi * 0.5 ** 1.5  # period of the smallest orbit (a = 1/2), GM = 1


def kepler_ensemble(batch: int = 65536, nsteps: int = 10000, seed: int = SEEDS[2]) -> Workload:
    """Config 2: e~U[0,0.9], a=exp(U[ln 1/2, ln 2]), omega~U[0,2pi), start at pericentre;
    h = T_min/128, T_min = 2pi (1/2)^(3/2)."""
    g = _rng(seed)
    e = g.uniform(0.0, 0.9, batch)
    a = np.exp(g.uniform(math.log(0.5), math.log(2.0), batch))
    om = g.uniform(0.0, 2 * math.pi, batch)
    rp = a * (1 - e)
    vp = np.sqrt((1 + e) / rp)
    y = np.stack([rp * np.cos(om), rp * np.sin(om), -vp * np.sin(om), vp * np.cos(om)])
    return Workload("kepler_ensemble", KEPLER, 4, y, np.array([1.0]), KEPLER_T_MIN / 128, nsteps,
                    meta=dict(e=e, a=a, omega=om))


def six_body_ensemble(batch: int = 16384, nsteps: int = 50000, seed: int = SEEDS[3]) -> Workload:
    """Config 3: central mass 1 + 5 bodies, masses log-U[1e-8,1e-3], radii log-U[5,40] (sorted),
    circular speeds, inclinations U[0,2 deg], barycentre at rest; members perturbed by
    relative 1e-8 Gaussian noise.  h = T_1/200 (innermost period).  Stand-in for the
    outer Solar System of P:L542-551 (DE430 data are not available)."""
    g = _rng(seed)
    N = 6
    m = np.empty(N)
    m[0] = 1.0
    m[1:] = np.exp(g.uniform(math.log(1e-8), math.log(1e-3), N - 1))
    r = np.sort(np.exp(g.uniform(math.log(5.0), math.log(40.0), N - 1)))
    inc = np.deg2rad(g.uniform(0.0, 2.0, N - 1))
    node = g.uniform(0.0, 2 * math.pi, N - 1)
    phase = g.uniform(0.0, 2 * math.pi, N - 1)
    pos = np.zeros((N, 3))
    vel = np.zeros((N, 3))
    for k in range(N - 1):
        vc = math.sqrt((1.0 + m[k + 1]) / r[k])
        p = np.array([r[k] * math.cos(phase[k]), r[k] * math.sin(phase[k]), 0.0])
        v = np.array([-vc * math.sin(phase[k]), vc * math.cos(phase[k]), 0.0])
        ci, si, cn, sn = math.cos(inc[k]), math.sin(inc[k]), math.cos(node[k]), math.sin(node[k])
        Rx = np.array([[1, 0, 0], [0, ci, -si], [0, si, ci]])
        Rz = np.array([[cn, -sn, 0], [sn, cn, 0], [0, 0, 1]])
        R = Rz @ Rx
        pos[k + 1] = R @ p
        vel[k + 1] = R @ v
    M = m.sum()
    pos -= (m[:, None] * pos).sum(0) / M
    vel -= (m[:, None] * vel).sum(0) / M
    base = np.concatenate([pos.reshape(-1), vel.reshape(-1)])  # (36,)
    noise = g.standard_normal((36, batch))
    y = base[:, None] * (1.0 + 1e-8 * noise)
    T1 = 2 * math.pi * math.sqrt(r[0] ** 3 / (1.0 + m[1]))
    params = np.concatenate([[1.0, 0.0], m])
    return Workload("six_body_ensemble", NBODY, 36, y, params, T1 / 200, nsteps,
                    meta=dict(masses=m, radii=r, base=base))


def fpu_ensemble(batch: int = 4096, nsteps: int = 100000, N: int = 64, beta: float = 1.0,
                 seed: int = SEEDS[4]) -> Workload:
    """Config 4: FPU-beta, N=64 unit masses, fixed ends, beta=1; q_n = sin(pi n/(N+1)) +
    1e-6 N(0,1), v_n = 1e-6 N(0,1) (lowest normal mode, amplitude 1); h = 0.1."""
    g = _rng(seed)
    n = np.arange(1, N + 1)
    mode = np.sin(math.pi * n / (N + 1))
    q = mode[:, None] + 1e-6 * g.standard_normal((N, batch))
    v = 1e-6 * g.standard_normal((N, batch))
    return Workload("fpu_ensemble", FPU_BETA, 2 * N, np.concatenate([q, v]), np.array([beta]),
                    0.1, nsteps)


def plummer(N: int = 8192, nsteps: int = 1000, eps: float = 1e-3, seed: int = SEEDS[5]) -> Workload:
    """Config 5: Plummer sphere (Aarseth-Henon-Wielen 1974 sampling), equal masses 1/N,
    G=1, Henon units, softening eps, centre of mass at rest; h = 1e-3."""
    g = _rng(seed)
    r = np.empty(N)
    i = 0
    while i < N:
        X = g.uniform(0.0, 1.0)
        if X <= 0.0:
            continue
        rr = (X ** (-2.0 / 3.0) - 1.0) ** -0.5
        if rr > 10.0:
            continue
        r[i] = rr
        i += 1

    def iso(rad):
        ct = g.uniform(-1.0, 1.0, rad.shape)
        ph = g.uniform(0.0, 2 * math.pi, rad.shape)
        st = np.sqrt(1 - ct * ct)
        return np.stack([rad * st * np.cos(ph), rad * st * np.sin(ph), rad * ct], axis=1)

    pos = iso(r)
    qv = np.empty(N)
    i = 0
    while i < N:  # von Neumann rejection on g(q) = q^2 (1-q^2)^(7/2), envelope 0.1
        x = g.uniform(0.0, 1.0)
        yv = g.uniform(0.0, 0.1)
        if yv < x * x * (1 - x * x) ** 3.5:
            qv[i] = x
            i += 1
    speed = qv * math.sqrt(2.0) * (1 + r * r) ** -0.25
    vel = iso(speed)
    pos *= 3 * math.pi / 16
    vel *= math.sqrt(16 / (3 * math.pi))
    pos -= pos.mean(0)
    vel -= vel.mean(0)
    y = np.concatenate([pos.reshape(-1), vel.reshape(-1)])[:, None]
    params = np.concatenate([[1.0, eps], np.full(N, 1.0 / N)])
    return Workload(f"plummer_{N}", NBODY_DIRECT, 6 * N, y, params, 1e-3, nsteps)


def henon_heiles(batch: int = 1, lam: float = 1.0, xi: float = 0.0, h: float = 2 * math.pi / 68,
                 nsteps: int = 1000, seed: int = 6) -> Workload:
    """Henon-Heiles (Listing 2); trajectory 0 is the paper's IC q1=0, q2=0.3,
    p2=0.2, p1>0 with H=1/12; others are seeded nearby ICs."""
    p1 = math.sqrt(2 * (1 / 12 - 0.5 * 0.2 ** 2 - 0.5 * 0.3 ** 2 + lam * 0.3 ** 3 / 3))
    base = np.array([0.0, 0.3, p1, 0.2])
    g = _rng(seed)
    y = base[:, None] * np.ones((1, batch))
    if batch > 1:
        y[:, 1:] += 1e-2 * g.standard_normal((4, batch - 1))
    return Workload("henon_heiles", HENON_HEILES, 4, y, np.array([lam, xi]), h, nsteps)


SBH_E, SBH_L, SBH_BETA = 0.995, 4.6, 8.9e-4


def schwarzschild(batch: int = 1, nsteps: int = 10000, h: float = 16.0, seed: int = 7) -> Workload:
    """Charged particle near a magnetised Schwarzschild black hole (Eq. Ham_SBH,
    P:L508-518) with the paper's parameters E = 0.995, L = 4.6, beta = 8.9e-4
    (P:L533).  y = (r, theta, p_r, p_theta).  Trajectory 0 is the paper's initial
    condition theta = pi/2, p_r = 0, r = 11 (a regular orbit), p_theta > 0 from
    H = -1/2; the others start at r = 11 (1 + 1e-3 N(0,1)), same rule.  h = 16 is
    the paper's reference step; the paper does not state the time span."""
    g = _rng(seed)
    r = np.full(batch, 11.0)
    if batch > 1:
        r[1:] *= 1.0 + 1e-3 * g.standard_normal(batch - 1)
    f = 1.0 - 2.0 / r
    A = SBH_L - 0.5 * SBH_BETA * r * r          # theta = pi/2: sin = 1
    # H = -1/2 at p_r = 0: p_theta^2/(2 r^2) = -1/2 + E^2/(2 f) - A^2/(2 r^2)
    pth = r * np.sqrt(2.0 * (-0.5 + 0.5 * SBH_E ** 2 / f - A * A / (2 * r * r)))
    y = np.stack([r, np.full(batch, math.pi / 2), np.zeros(batch), pth])
    return Workload("schwarzschild", SCHWARZSCHILD, 4, y, np.array([SBH_E, SBH_L, SBH_BETA]), h, nsteps)


def config(i: int, **kw) -> Workload:
    """BASELINE.json configs[i-1] (1-based as in SURVEY.md)."""
    return {1: kepler_single, 2: kepler_ensemble, 3: six_body_ensemble, 4: fpu_ensemble,
            5: plummer}[i](**kw)
