"""GPU parity of the per-thread-problem stage-per-lane kernel with DMMA
contractions (IRK_MAP_G8M for Kepler / Henon-Heiles, ensemble_g8m.cuh): bitwise
equal to the oracle -- config 1 at full length, the time-dependent Henon-Heiles
coupling at stage times (Listing 2), an invariant subspace whose
contractions are sums of signed zeros (compared as bit patterns), slots whose
trajectories finish steps at different sweeps (the second nu~ pass), the
max_iters cap, a diverging trajectory, ragged slots, and g8m == g8 on the same
ensemble.
"""
import numpy as np
import pytest

from paper_2511_03655_b200 import workloads as wl

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from tests.test_gpu_parity import assert_parity, run_gpu  # noqa: E402


@pytest.fixture(scope="module")
def irk():
    from paper_2511_03655_b200 import build, irk
    build.build()
    return irk


def _bits(x):
    return np.ascontiguousarray(x).view(np.int64)


def test_config1_full_length(irk, orc):
    """Config 1 (one Kepler orbit, e = 0.5, 12,800 steps) through g8m: states,
    sweep counts and energy samples bitwise equal to the oracle."""
    w = wl.kepler_single()
    g = run_gpu(irk, w, energy_every=128, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=128)
    assert g["rc"] == irk.OK
    assert_parity(g, o, energy=True)
    assert np.array_equal(_bits(g["y"]), _bits(o["y"]))


@pytest.mark.parametrize("batch", [1, 3, 5, 13])
def test_hh_time_dependent_ragged(irk, orc, batch):
    """Henon-Heiles with xi = 0.1 from t0 = 0.25 (sin at t_{n-1} + c_i h per
    stage lane), ragged slots (idle lanes in the last warp), two chained calls
    (history hand-over): bitwise equal to the oracle."""
    w = wl.henon_heiles(batch=batch, xi=0.1, nsteps=400)
    g = run_gpu(irk, w, energy_every=50, chunks=2, t0=0.25, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=50, t0=0.25)
    assert_parity(g, o, energy=True)


def test_signed_zero_subspace(irk, orc):
    """Henon-Heiles on the invariant subspace q1 = p1 = 0: every first-component
    contraction is a sum of signed zeros (the C = -0 convention of the first DMMA
    and the ones x tile update must reproduce the oracle's dmul / dadd zeros);
    compared as bit patterns."""
    w = wl.henon_heiles(batch=6, xi=0.0, nsteps=300)
    y = w.y.copy()
    y[0, :] = 0.0
    y[2, :] = 0.0
    y[0, 1] = -0.0
    y[2, 3] = -0.0
    g = run_gpu(irk, w, y=y, energy_every=30, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, y, w.params, w.h, w.nsteps, energy_every=30)
    assert np.array_equal(_bits(g["y"]), _bits(o["y"]))
    assert np.array_equal(g["iters"], o["iters"])
    assert np.array_equal(_bits(g["energy"]), _bits(o["energy"]))


@pytest.mark.parametrize("batch", [3, 37])
@pytest.mark.parametrize("max_iters", [2, 3])
def test_max_iters_cap_mixed_slots(irk, orc, max_iters, batch):
    """A sweep cap below the converged count for some trajectories and not
    others: slots mix finished and unfinished trajectories every step (the nu~
    second pass); both launch variants (one slot: ballot stop test; more:
    speculative nu~ pass); bitwise equal to the oracle with the same cap."""
    w = wl.kepler_ensemble(batch=batch, nsteps=300)
    g = run_gpu(irk, w, max_iters=max_iters, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, max_iters=max_iters)
    assert_parity(g, o)
    assert np.array_equal(g["iters"], o["iters"])


def test_g8m_equals_g8_with_divergence(irk, orc):
    """Kepler ensemble of 203 (ragged last slot) with one trajectory started at
    the singularity's edge (it diverges and freezes inside its slot): g8m == g8
    (states, sweeps, stats, history) and == oracle on the finite members."""
    w = wl.kepler_ensemble(batch=203, nsteps=500)
    y = w.y.copy()
    y[:, 9] = [1e-200, 0.0, 0.0, 0.0]
    a = run_gpu(irk, w, y=y, energy_every=100, mapping=irk.MAP_G8M)
    b = run_gpu(irk, w, y=y, energy_every=100, mapping=irk.MAP_G8)
    assert np.array_equal(a["y"], b["y"], equal_nan=True)
    assert np.array_equal(a["iters"], b["iters"]) and a["stats"] == b["stats"]
    assert np.array_equal(a["hist"], b["hist"], equal_nan=True)
    assert np.array_equal(a["energy"], b["energy"], equal_nan=True)
    ok = np.isfinite(a["y"]).all(axis=0)
    assert not ok[9] and ok.sum() == w.batch - 1
    o = orc.integrate(w.problem, y[:, ok], w.params, w.h, w.nsteps, energy_every=100)
    assert np.array_equal(a["y"][:, ok], o["y"]) and np.array_equal(a["iters"][ok], o["iters"])


def test_mapping_used_reports_g8m(irk):
    w = wl.kepler_ensemble(batch=8, nsteps=3)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mapping=irk.MAP_G8M) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ig.integrate(Y, ig.new_workspace())
        torch.cuda.synchronize()
        assert ig.get_option(irk.INFO_MAPPING_USED) == irk.MAP_G8M


@pytest.mark.parametrize("batch", [1, 3])
def test_one_slot_gm_not_one(irk, orc, batch):
    """The one-slot launch (ballot stop test, shadow lanes) with GM = 1.3: the
    full correctly rounded division w = GM / r^3 (KeplerT<false>); bitwise equal
    to the oracle with energy samples."""
    w = wl.kepler_ensemble(batch=batch, nsteps=1500)
    w.params = np.array([1.3])
    g = run_gpu(irk, w, energy_every=100, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=100)
    assert_parity(g, o, energy=True)
    assert np.array_equal(g["iters"], o["iters"])


def test_shadowed_slot_with_divergence(irk, orc):
    """Two trajectories in one slot: trajectory 0 (which the slot's two missing
    trajectories shadow) diverges and freezes, trajectory 1 integrates on.
    g8m == g8 (states, sweeps, stats, history), the finite member == oracle, and
    the shadows store nothing (the workspace rows beyond the batch are untouched
    by construction: the history equals g8's)."""
    w = wl.kepler_ensemble(batch=2, nsteps=400)
    y = w.y.copy()
    y[:, 0] = [1e-200, 0.0, 0.0, 0.0]
    a = run_gpu(irk, w, y=y, energy_every=50, mapping=irk.MAP_G8M)
    b = run_gpu(irk, w, y=y, energy_every=50, mapping=irk.MAP_G8)
    assert np.array_equal(a["y"], b["y"], equal_nan=True)
    assert np.array_equal(a["iters"], b["iters"]) and a["stats"] == b["stats"]
    assert np.array_equal(a["hist"], b["hist"], equal_nan=True)
    assert np.array_equal(a["energy"], b["energy"], equal_nan=True)
    assert not np.isfinite(a["y"][:, 0]).all() and np.isfinite(a["y"][:, 1]).all()
    o = orc.integrate(w.problem, y[:, 1:], w.params, w.h, w.nsteps, energy_every=50)
    assert np.array_equal(a["y"][:, 1:], o["y"]) and np.array_equal(a["iters"][1:], o["iters"])


@pytest.mark.parametrize("batch", [1, 4])
def test_one_slot_local_energy_chained(irk, orc, batch):
    """One slot (ballot stop test, shadow lanes) with Delta H^loc (Eq. DHlocmax)
    and energy samples over two chained calls: bitwise equal to the oracle."""
    w = wl.kepler_ensemble(batch=batch, nsteps=800)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps // 2, w.batch, w.params, energy_every=40,
                        mapping=irk.MAP_G8M, local_energy=True) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        ig.integrate(Y, ws, energy=E, iters=it)
        E1, it1, d1 = E.cpu().numpy().copy(), it.cpu().numpy().copy(), ig.local_energy_error(ws).cpu().numpy()
        ig.integrate(Y, ws, energy=E, iters=it)
        y2, E2, it2, d2 = Y.cpu().numpy(), E.cpu().numpy(), it.cpu().numpy(), ig.local_energy_error(ws).cpu().numpy()
    o1 = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps // 2, energy_every=40, local_energy=True)
    o2 = orc.integrate(w.problem, o1["y"], w.params, w.h, w.nsteps // 2, energy_every=40, local_energy=True,
                       n0=w.nsteps // 2, hist=o1["hist"])
    assert np.array_equal(E1, o1["energy"]) and np.array_equal(d1, o1["dhloc"]) and np.array_equal(it1, o1["iters"])
    assert np.array_equal(y2, o2["y"]) and np.array_equal(E2, o2["energy"])
    assert np.array_equal(d2, o2["dhloc"]) and np.array_equal(it2, o2["iters"])
