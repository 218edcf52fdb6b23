"""GPU parity of the N-body stage-per-lane kernel with DMMA contractions
(IRK_MAP_G8M, ensemble_nbody8m.cuh): bitwise equal to the oracle and to the
other two N-body mappings -- configs with energy samples and Delta H^loc over
chained calls, every N, G != 1, exactly planar systems (signed zeros in the
contractions), ragged batches (idle slot lanes) and the config-3 batch.
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


def _chained(irk, w, mp, energy_every=40):
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps // 2, w.batch, w.params, energy_every=energy_every,
                        mapping=mp, local_energy=True) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        ig.integrate(Y, ws, energy=E, iters=it)
        E1, it1 = E.cpu().numpy().copy(), it.cpu().numpy().copy()
        ig.integrate(Y, ws, energy=E, iters=it)
        assert ig.get_option(irk.INFO_MAPPING_USED) == mp
        return (Y.cpu().numpy(), E1, E.cpu().numpy(), it1 + it.cpu().numpy(),
                ig.local_energy_error(ws).cpu().numpy(), ig.stats(ws)[1])


def test_dmma_equals_other_mappings_and_oracle(irk, orc):
    """Six-body config-3 generator, 601 trajectories (the last slot holds one),
    two chained calls of 200 steps with energy every 40 and Delta H^loc: DMMA
    mapping == shared-memory stage per lane == oracle, bit for bit."""
    w = wl.six_body_ensemble(batch=601, nsteps=400)
    o9 = _chained(irk, w, irk.MAP_G8M)
    o8 = _chained(irk, w, irk.MAP_G8)
    for a_, b_ in zip(o9[:5], o8[:5]):
        assert np.array_equal(a_, b_)
    assert o9[5] == o8[5]
    idx = np.arange(0, w.batch, 97)
    o1 = orc.integrate(w.problem, w.y[:, idx], w.params, w.h, w.nsteps // 2, energy_every=40)
    o2 = orc.integrate(w.problem, o1["y"], w.params, w.h, w.nsteps // 2, energy_every=40, local_energy=True,
                       n0=w.nsteps // 2, hist=o1["hist"])
    assert np.array_equal(o9[0][:, idx], o2["y"]) and np.array_equal(o9[2][:, idx], o2["energy"])
    assert np.array_equal(o9[3][idx], o1["iters"] + o2["iters"])
    assert np.array_equal(o9[4][idx], o2["dhloc"])


@pytest.mark.parametrize("N", [2, 3, 4, 5, 7, 8])
def test_dmma_small_n(irk, orc, N):
    """Every other N (odd 3N: a padding component in the last tile), random
    softened systems, 23 trajectories (a partly idle slot), energy samples."""
    rng = np.random.default_rng(3 + N)
    B = 23
    q = rng.standard_normal((3 * N, B))
    v = 0.3 * rng.standard_normal((3 * N, B))
    params = np.concatenate([[1.0, 0.05], rng.uniform(0.2, 1.0, N)])
    w = wl.Workload(f"nb{N}", wl.NBODY, 6 * N, np.concatenate([q, v]), params, 0.01, 300)
    g = run_gpu(irk, w, energy_every=100, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=100)
    assert_parity(g, o, energy=True)


def test_dmma_g_not_one(irk, orc):
    """G = 0.5 runs the full correctly rounded division (ens_nbody8m<NB, false>)."""
    w = wl.six_body_ensemble(batch=37, nsteps=300)
    w.params = np.asarray(w.params, dtype=np.float64).copy()
    w.params[0] = 0.5
    g = run_gpu(irk, w, energy_every=100, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=100)
    assert_parity(g, o, energy=True)


def test_dmma_planar_signed_zeros(irk, orc):
    """Exactly planar systems (z = 0, v_z = 0 for every body): the z stage
    contractions are sums of signed zeros, where the DMMA chain must reproduce
    the oracle's leading dmul (C = -0); compared bit for bit including the sign
    of zero."""
    w = wl.six_body_ensemble(batch=29, nsteps=300)
    y = np.asarray(w.y, dtype=np.float64).copy()
    y[2:18:3, :] = 0.0
    y[20:36:3, :] = 0.0
    y[20:36:3, ::2] = -0.0
    w.y = y
    g = run_gpu(irk, w, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps)
    assert_parity(g, o)
    assert np.array_equal(np.signbit(g["y"]), np.signbit(o["y"]))


def test_dmma_config3_full_batch_vs_g8(irk):
    """Config 3 at full batch (16,384), 1,000 steps: DMMA mapping == ens_nbody8,
    states and sweep counts bitwise (the oracle checks of ens_nbody8 carry over)."""
    w = wl.six_body_ensemble(nsteps=1000)
    g9 = run_gpu(irk, w, mapping=irk.MAP_G8M)
    g8 = run_gpu(irk, w, mapping=irk.MAP_G8)
    assert np.array_equal(g9["y"], g8["y"]) and np.array_equal(g9["iters"], g8["iters"])


def test_dmma_max_iters_cap_mixed_slots(irk, orc):
    """max_iters = 3 on heterogeneous systems: trajectories of a slot hit the cap or
    converge at different sweeps (the mixed mu~ / nu~ velocity pass), flagged and
    bitwise like the oracle."""
    rng = np.random.default_rng(11)
    N, B = 6, 45
    q = rng.standard_normal((3 * N, B)) * rng.uniform(0.3, 3.0, B)
    v = 0.4 * rng.standard_normal((3 * N, B))
    params = np.concatenate([[1.0, 0.02], rng.uniform(0.2, 1.0, N)])
    w = wl.Workload("nb6_hetero", wl.NBODY, 6 * N, np.concatenate([q, v]), params, 0.02, 120)
    g = run_gpu(irk, w, max_iters=3, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, max_iters=3)
    assert_parity(g, o)
    assert g["stats"]["maxiter_traj"] == int((o["status"][:, 0] > 0).sum()) > 0


def test_dmma_divergence_flag_and_freeze(irk, orc):
    """Two bodies at the same position and velocity with eps = 0 in one trajectory of a slot:
    the weight is infinite, the step non-finite; the trajectory is flagged at the
    oracle's step and frozen, its slot partners are unaffected (bitwise)."""
    w = wl.six_body_ensemble(batch=7, nsteps=40)
    w.params = np.asarray(w.params, dtype=np.float64).copy()
    w.params[1] = 0.0
    y = np.asarray(w.y, dtype=np.float64).copy()
    y[3:6, 2] = y[0:3, 2]      # body 1 on body 0 in trajectory 2,
    y[21:24, 2] = y[18:21, 2]  # with the same velocity: they coincide at every stage
    w.y = y
    g = run_gpu(irk, w, mapping=irk.MAP_G8M)
    o = orc.integrate(w.problem, y, w.params, w.h, w.nsteps)
    assert g["rc"] == irk.E_DIVERGED
    assert g["stats"]["diverged_traj"] == 1
    assert g["stats"]["first_bad_step"] == o["status"][2, 1]
    keep = [b for b in range(w.batch) if b != 2]
    np.testing.assert_array_equal(g["y"][:, keep], o["y"][:, keep])
    np.testing.assert_array_equal(g["iters"][keep], o["iters"][keep])
