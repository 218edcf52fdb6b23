"""Statistical sanity of the seeded config generators (SURVEY C-10 item 11) and
the recipe constants they encode."""
import math

import numpy as np

from paper_2511_03655_b200 import workloads as wl


def test_config1_closed_form():
    w = wl.kepler_single()
    assert np.array_equal(w.y[:, 0], [0.5, 0.0, 0.0, math.sqrt(3.0)])
    assert w.nsteps == 12800 and w.h == 2 * math.pi / 128


def test_config2_moments():
    w = wl.kepler_ensemble()
    e, a, om = w.meta["e"], w.meta["a"], w.meta["omega"]
    assert w.y.shape == (4, 65536) and w.nsteps == 10000
    assert abs(e.mean() - 0.45) < 0.01 and e.min() >= 0 and e.max() <= 0.9
    assert abs(np.log(a).mean()) < 0.01 and a.min() >= 0.5 and a.max() <= 2.0
    assert abs(om.mean() - math.pi) < 0.03
    r = np.hypot(w.y[0], w.y[1])
    assert np.allclose(r, a * (1 - e))                       # pericentre start
    assert np.allclose(w.y[0] * w.y[2] + w.y[1] * w.y[3], 0, atol=1e-12)  # radial velocity 0
    assert abs(w.h - 2 * math.pi * 0.5 ** 1.5 / 128) < 1e-18


def test_config3_structure(orc):
    w = wl.six_body_ensemble(batch=64)
    m = w.meta["masses"]
    assert m[0] == 1.0 and np.all((m[1:] >= 1e-8) & (m[1:] <= 1e-3))
    base = w.meta["base"]
    q = base[:18].reshape(6, 3); v = base[18:].reshape(6, 3)
    assert np.abs((m[:, None] * v).sum(0)).max() < 1e-15   # barycentre at rest
    rel = w.y / base[:, None] - 1
    assert 0.5e-8 < rel.std() < 2e-8                      # 1e-8 relative noise
    incl = np.degrees(np.arccos(np.abs(np.cross(q[1:] - q[0], v[1:] - v[0])[:, 2]) /
                                np.linalg.norm(np.cross(q[1:] - q[0], v[1:] - v[0]), axis=1)))
    assert incl.max() < 2.1
    E = orc.energy(w.problem, w.dim, w.params, base)
    assert E < 0


def test_config4_lowest_mode():
    w = wl.fpu_ensemble(batch=256)
    n = np.arange(1, 65)
    mode = np.sin(np.pi * n / 65)
    assert np.abs(w.y[:64].mean(1) - mode).max() < 5e-7
    assert 0.5e-6 < w.y[64:].std() < 2e-6


def test_config5_plummer_virial(orc):
    w = wl.plummer(N=1024)
    N = 1024
    q = w.y[:3 * N, 0].reshape(N, 3); v = w.y[3 * N:, 0].reshape(N, 3)
    assert np.abs(q.mean(0)).max() < 1e-14 and np.abs(v.mean(0)).max() < 1e-14
    T = 0.5 * (1.0 / N) * (v ** 2).sum()
    E = orc.energy(w.problem, w.dim, w.params, w.y[:, 0])
    U = E - T
    assert 0.8 < 2 * T / abs(U) < 1.25
    assert -0.3 < E < -0.2
