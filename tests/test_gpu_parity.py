"""GPU parity: the CUDA path (through the C ABI) against the scalar-C oracle on
the same seeded inputs.

The bar: both sides execute the same IEEE operation
sequence, so states, sweep counts and energy samples must be BITWISE equal;
the north-star tolerances (max relative state error <= 1e-10, |dH_gpu - dH_orc|
<= 1e-13) are asserted as well so a failure report says by how much.
"""
import math

import numpy as np
import pytest

from paper_2511_03655_b200 import workloads as wl

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.fixture(scope="module")
def irk():
    from paper_2511_03655_b200 import build, irk
    build.build()
    return irk


def run_gpu(irk, w, y=None, nsteps=None, energy_every=0, max_iters=100, chunks=1, t0=0.0, mapping=0):
    y = w.y if y is None else y
    nsteps = w.nsteps if nsteps is None else nsteps
    assert nsteps % chunks == 0
    per = nsteps // chunks
    B = y.shape[1]
    with irk.Integrator(w.problem, w.dim, w.h, per, B, w.params, energy_every=energy_every,
                        max_iters=max_iters, mapping=mapping) as ig:
        Y = torch.tensor(y, dtype=torch.float64, device="cuda").contiguous()
        ws = ig.new_workspace()
        it_total = torch.zeros(B, dtype=torch.int64, device="cuda")
        it = torch.zeros(B, dtype=torch.int64, device="cuda")
        E = (torch.zeros((ig.n_energy(), B), dtype=torch.float64, device="cuda")
             if energy_every else None)
        Es = []
        for _ in range(chunks):
            ig.integrate(Y, ws, t0=t0, energy=E, iters=it)
            it_total += it
            if E is not None:
                Es.append(E.cpu().numpy().copy())
        torch.cuda.synchronize()
        rc, st = ig.stats(ws)
        return dict(y=Y.cpu().numpy(), iters=it_total.cpu().numpy(),
                    energy=(np.concatenate([Es[0]] + [e[1:] for e in Es[1:]]) if Es else None),
                    rc=rc, stats=st, hist=ig.hist_view(ws).cpu().numpy())


def assert_parity(g, o, energy=False):
    yg, yo = g["y"], o["y"] if o["y"].ndim == 2 else o["y"][:, None]
    scale = np.maximum(np.abs(yo).max(axis=0), 1e-300)
    rel = (np.abs(yg - yo).max(axis=0) / scale).max()
    assert rel <= 1e-10, f"max relative state error {rel:.3e}"
    if energy:
        eg, eo = g["energy"], o["energy"]
        dg = (eg - eg[0]) / eg[0]
        do = (eo - eo[0]) / eo[0]
        assert np.abs(dg - do).max() <= 1e-13
        assert np.array_equal(eg, eo), "energy samples not bitwise equal"
    nbad = int((yg != yo).any(axis=0).sum())
    assert nbad == 0, f"{nbad} trajectories not bitwise equal (max rel {rel:.3e})"
    assert np.array_equal(g["iters"], o["iters"]), "sweep counts differ"


def test_config1_kepler_single_full(irk, orc):
    """Config 1 in full: 12,800 steps, energy every 128 steps, bitwise."""
    w = wl.kepler_single()
    g = run_gpu(irk, w, energy_every=128)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=128)
    assert_parity(g, o, energy=True)
    assert g["rc"] == irk.OK


def test_config2_ragged_subset_full_length(irk, orc):
    """Config 2 generator, a ragged batch (1000 = not a multiple of the block),
    full 10,000 steps, energy samples every 500 steps, bitwise."""
    w = wl.kepler_ensemble(batch=1000)
    g = run_gpu(irk, w, energy_every=500)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=500)
    assert_parity(g, o, energy=True)


def test_config2_full_batch_sampled(irk, orc):
    """Config 2 at full size (65,536 x 10,000) in the launch configuration the
    bench times; the oracle recomputes a sample of 192 trajectories spread over
    the batch plus the 64 most eccentric (hardest) ones."""
    w = wl.kepler_ensemble()
    g = run_gpu(irk, w)
    e = w.meta["e"]
    idx = np.unique(np.concatenate([np.linspace(0, w.batch - 1, 192).astype(int),
                                    np.argsort(e)[-64:]]))
    o = orc.integrate(w.problem, w.y[:, idx], w.params, w.h, w.nsteps)
    sub = dict(y=g["y"][:, idx], iters=g["iters"][idx])
    assert_parity(sub, o)
    assert g["stats"]["diverged_traj"] == 0


def test_chunked_calls_continue_bitwise(irk, orc):
    """Workspace (history + n) carries the state: 4 chunks == one oracle run."""
    w = wl.kepler_ensemble(batch=130, nsteps=400)
    g = run_gpu(irk, w, chunks=4)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps)
    assert_parity(g, o)
    oh = o["hist"].transpose(1, 2, 0)  # (batch, 8, dim) -> (8, dim, batch)
    assert np.array_equal(g["hist"], oh)


def test_henon_heiles_parity(irk, orc):
    w = wl.henon_heiles(batch=300, nsteps=2000)
    g = run_gpu(irk, w, energy_every=100)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=100)
    assert_parity(g, o, energy=True)


@pytest.mark.parametrize("mode", [0, 1])
def test_henon_heiles_time_dependent_bitwise(irk, orc, mode):
    """xi != 0 (Listing 2's time-dependent coupling) uses the canonical sin of
    CANON.md on both sides (R-12), so the time-dependent case is
    bitwise too -- partitioned and first-order mode, t0 != 0, chained calls
    (absolute step index in t_{n-1})."""
    w = wl.henon_heiles(batch=64, nsteps=500, xi=0.1, lam=1.0, h=0.05 if mode else 2 * math.pi / 68)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps // 2, w.batch, w.params, mode=mode) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        ig.integrate(Y, ws, t0=0.25, iters=it)
        it1 = it.cpu().numpy().copy()
        ig.integrate(Y, ws, t0=0.25, iters=it)
        yg, itg = Y.cpu().numpy(), it1 + it.cpu().numpy()
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, t0=0.25, mode=mode)
    assert np.array_equal(yg, o["y"]) and np.array_equal(itg, o["iters"])


def test_max_iters_cap_flagged_like_oracle(irk, orc):
    w = wl.kepler_ensemble(batch=70, nsteps=50)
    g = run_gpu(irk, w, max_iters=3)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, max_iters=3)
    assert_parity(g, o)
    assert g["rc"] == irk.W_MAXITER
    assert g["stats"]["maxiter_traj"] == int((o["status"][:, 0] > 0).sum())


def test_negative_h_reversibility(irk, orc):
    w = wl.kepler_ensemble(batch=65, nsteps=64)
    g1 = run_gpu(irk, w)
    wb = wl.Workload(w.name, w.problem, w.dim, g1["y"], w.params, -w.h, 64)
    g2 = run_gpu(irk, wb)
    o2 = orc.integrate(w.problem, g1["y"], w.params, -w.h, 64)
    assert_parity(g2, o2)
    assert np.abs(g2["y"] - w.y).max() < 1e-12


def test_divergence_flag_and_freeze(irk, orc):
    y = np.array([[1e-200, 1.0, 0.5], [0.0, 0.0, 0.0], [0.0, 0.0, 0.0], [0.0, 1.0, 1.0]])
    w = wl.Workload("div", wl.KEPLER, 4, y, np.array([1.0]), 0.1, 20)
    g = run_gpu(irk, w)
    o = orc.integrate(w.problem, y, w.params, w.h, 20)
    assert g["rc"] == irk.E_DIVERGED
    assert g["stats"]["diverged_traj"] == 1
    assert g["stats"]["first_bad_step"] == o["status"][0, 1]
    np.testing.assert_array_equal(g["y"][:, 1:], o["y"][:, 1:])


def test_zero_steps_and_batch_one(irk):
    w = wl.kepler_single()
    g = run_gpu(irk, w, nsteps=0)
    assert np.array_equal(g["y"], w.y) and g["iters"][0] == 0


def test_energy_entry_point_matches_oracle(irk, orc):
    w = wl.kepler_ensemble(batch=257)
    with irk.Integrator(w.problem, w.dim, w.h, 1, w.batch, w.params) as ig:
        H = ig.energy(torch.tensor(w.y, device="cuda")).cpu().numpy()
    Ho = np.array([orc.energy(w.problem, 4, w.params, w.y[:, b]) for b in range(w.batch)])
    assert np.array_equal(H, Ho)


def test_integrate_host_end_to_end(irk, orc):
    w = wl.kepler_ensemble(batch=100, nsteps=200)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=50) as ig:
        y = np.ascontiguousarray(w.y.copy())
        E, it = ig.integrate_host(y)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=50)
    assert np.array_equal(y, o["y"]) and np.array_equal(it, o["iters"])
    assert np.array_equal(E, o["energy"])


def test_fast_div_sqrt_bitwise(irk):
    """The branch-free div/sqrt/reciprocal of the hot path (fp64.cuh) equal
    __ddiv_rn / __dsqrt_rn / __ddiv_rn(1, .) bit for bit: 2^26 random operands
    over many binades, plus specials (0, denormals, inf, nan, negative)."""
    g = torch.Generator(device="cuda").manual_seed(1234)
    n = 1 << 24
    for _ in range(4):
        ea = torch.randint(-60, 60, (n,), device="cuda", generator=g).double()
        eb = torch.randint(-60, 60, (n,), device="cuda", generator=g).double()
        a = (torch.rand(n, device="cuda", generator=g, dtype=torch.float64) + 0.5) * torch.exp2(ea)
        b = (torch.rand(n, device="cuda", generator=g, dtype=torch.float64) + 0.5) * torch.exp2(eb)
        a = torch.where(torch.rand(n, device="cuda", generator=g) < 0.5, -a, a)
        out = irk.probe_divsqrt(a, b)
        assert torch.equal(out[:, 0].view(torch.int64), out[:, 1].view(torch.int64))
        assert torch.equal(out[:, 2].view(torch.int64), out[:, 3].view(torch.int64))
        assert torch.equal(out[:, 4].view(torch.int64), out[:, 5].view(torch.int64))
    sp = torch.tensor([0.0, -0.0, 5e-324, 1e-310, 2.2250738585072014e-308, 1e308, 1.7976931348623157e308,
                       float("inf"), float("-inf"), float("nan"), -1.0, 1.0, 3.0, 1e-300, 4e-320],
                      dtype=torch.float64, device="cuda")
    A = sp.repeat_interleave(len(sp))
    B = sp.repeat(len(sp))
    out = irk.probe_divsqrt(A, B).cpu().numpy()
    np.testing.assert_array_equal(out[:, 0].view(np.int64), out[:, 1].view(np.int64))
    np.testing.assert_array_equal(out[:, 2].view(np.int64), out[:, 3].view(np.int64))
    np.testing.assert_array_equal(out[:, 4].view(np.int64), out[:, 5].view(np.int64))


def test_cost_balanced_schedule_is_bitwise_neutral(irk, orc):
    """Chunked, cost-sorted scheduling (IRK_OPT_BALANCE) only changes which
    thread runs which trajectory: results equal the single-launch run and the
    oracle bit for bit, including energy samples that straddle chunks."""
    w = wl.kepler_ensemble(batch=9000, nsteps=1000)
    outs = []
    for bal in (0, 230, -1):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=100,
                            balance=bal) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
            it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
            ig.integrate(Y, ws, energy=E, iters=it)
            rc, st = ig.stats(ws)
            outs.append((Y.cpu().numpy(), E.cpu().numpy(), it.cpu().numpy(), st["total_sweeps"]))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])
        assert np.array_equal(o[2], outs[0][2]) and o[3] == outs[0][3]
    idx = np.arange(0, w.batch, 97)
    orr = orc.integrate(w.problem, w.y[:, idx], w.params, w.h, w.nsteps, energy_every=100)
    assert np.array_equal(outs[1][0][:, idx], orr["y"])
    assert np.array_equal(outs[1][1][:, idx], orr["energy"])
    assert np.array_equal(outs[1][2][idx], orr["iters"])


@pytest.mark.timeout(240)
@pytest.mark.parametrize("unit", [7, 1])
def test_work_queue_schedule_bitwise(irk, orc, unit):
    """The persistent work-queue launch (IRK_OPT_SCHEDULE = 2): more trajectories
    than resident lanes, units of 7 (or 1: every step a hand-off, maximal
    parking of blocked units) steps, energy samples and Delta H^loc straddling
    units, and two trajectories that diverge mid-call.  Bitwise equal to the
    chunked launches and to the oracle on a sample that includes the diverged
    trajectories."""
    w = wl.kepler_ensemble(batch=70001, nsteps=119 if unit == 7 else 40)
    y = w.y.copy()
    y[:, 5] = [1e-200, 0.0, 0.0, 0.0]      # r = 0 -> non-finite at step 1
    y[:, 69990] = [1e-150, 0.0, 0.0, 1e-160]
    outs = []
    for sched, bal in ((1, 0), (2, unit), (0, -1)):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=10,
                            balance=bal, schedule=sched, local_energy=True) as ig:
            Y = torch.tensor(y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
            it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
            ig.integrate(Y, ws, energy=E, iters=it)
            rc, st = ig.stats(ws)
            outs.append((Y.cpu().numpy(), E.cpu().numpy(), it.cpu().numpy(), st,
                         ig.local_energy_error(ws).cpu().numpy(), rc))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0], equal_nan=True)
        assert np.array_equal(o[1], outs[0][1], equal_nan=True)
        assert np.array_equal(o[2], outs[0][2]) and o[3] == outs[0][3]
        assert np.array_equal(o[4], outs[0][4], equal_nan=True) and o[5] == outs[0][5]
    assert outs[1][5] == irk.E_DIVERGED and outs[1][3]["diverged_traj"] == 2
    idx = np.r_[5, 69990, np.arange(0, w.batch, 1009)]
    orr = orc.integrate(w.problem, y[:, idx], w.params, w.h, w.nsteps, energy_every=10, local_energy=True)
    assert np.array_equal(outs[1][0][:, idx], orr["y"], equal_nan=True)
    assert np.array_equal(outs[1][1][:, idx], orr["energy"], equal_nan=True)
    assert np.array_equal(outs[1][2][idx], orr["iters"])
    assert np.array_equal(outs[1][4][idx], orr["dhloc"], equal_nan=True)


def test_work_queue_chain_bitwise(irk, orc):
    """Warp-level work queue of the FPU chain kernel: more chains than resident
    warps, units of 9 steps, energy samples and Delta H^loc across units; equal
    to the chunked launches and to the oracle."""
    w = wl.fpu_ensemble(batch=4100, nsteps=90)
    outs = []
    for sched, bal in ((1, 0), (2, 9)):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=15,
                            balance=bal, schedule=sched, local_energy=True) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
            it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
            ig.integrate(Y, ws, energy=E, iters=it)
            rc, st = ig.stats(ws)
            outs.append((Y.cpu().numpy(), E.cpu().numpy(), it.cpu().numpy(), st,
                         ig.local_energy_error(ws).cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[0][2], outs[1][2]) and outs[0][3] == outs[1][3]
    assert np.array_equal(outs[0][4], outs[1][4])
    idx = np.arange(0, w.batch, 517)
    orr = orc.integrate(w.problem, w.y[:, idx], w.params, w.h, w.nsteps, energy_every=15, local_energy=True)
    assert np.array_equal(outs[1][0][:, idx], orr["y"]) and np.array_equal(outs[1][1][:, idx], orr["energy"])
    assert np.array_equal(outs[1][2][idx], orr["iters"]) and np.array_equal(outs[1][4][idx], orr["dhloc"])


@pytest.mark.parametrize("G", [8, 4, 2, 9])
@pytest.mark.parametrize("which", ["kepler", "hh"])
def test_g8_stage_per_lane_mapping(irk, orc, which, G):
    """IRK_OPT_MAPPING = 8 / 4 / 2 (G lanes per trajectory, 8/G stages per lane,
    shared-memory all-gather, xor-shuffle Delta reduction) and 9 (g8m: stage per
    lane, DMMA contractions): bitwise equal to the
    oracle and to g1 -- states, sweeps, energy samples, Delta H^loc, a diverging
    trajectory, and two chained calls."""
    if which == "kepler":
        w = wl.kepler_ensemble(batch=203, nsteps=600)
        y = w.y.copy()
        y[:, 7] = [1e-200, 0.0, 0.0, 0.0]
    else:
        w = wl.henon_heiles(batch=77, nsteps=600)
        y = w.y.copy()
    outs = []
    for mp in (G, 1):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps // 2, w.batch, w.params, energy_every=50,
                            mapping=mp, local_energy=True) as ig:
            Y = torch.tensor(y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
            it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
            ig.integrate(Y, ws, energy=E, iters=it)
            E1, it1, d1 = E.cpu().numpy().copy(), it.cpu().numpy().copy(), ig.local_energy_error(ws).cpu().numpy()
            ig.integrate(Y, ws, energy=E, iters=it)
            rc, st = ig.stats(ws)
            outs.append((Y.cpu().numpy(), E1, E.cpu().numpy(), it1 + it.cpu().numpy(), d1,
                         ig.local_energy_error(ws).cpu().numpy(), st))
    for a_, b_ in zip(outs[0][:6], outs[1][:6]):
        assert np.array_equal(a_, b_, equal_nan=True)
    assert outs[0][6] == outs[1][6]
    o1 = orc.integrate(w.problem, y, w.params, w.h, w.nsteps // 2, energy_every=50, local_energy=True)
    o2 = orc.integrate(w.problem, o1["y"], w.params, w.h, w.nsteps // 2, energy_every=50, local_energy=True,
                       n0=w.nsteps // 2, hist=o1["hist"])
    g = outs[0]
    assert np.array_equal(g[0], o2["y"], equal_nan=True)
    assert np.array_equal(g[1], o1["energy"], equal_nan=True) and np.array_equal(g[2], o2["energy"], equal_nan=True)
    ok = np.isfinite(o1["y"]).all(axis=0)  # the oracle has no frozen state across calls
    assert np.array_equal(g[3][ok], (o1["iters"] + o2["iters"])[ok])
    assert np.array_equal(g[4], o1["dhloc"], equal_nan=True)
    assert np.array_equal(g[5][ok], o2["dhloc"][ok], equal_nan=True)


def test_schwarzschild_first_order_parity(irk, orc):
    """Eq. Ham_SBH (the paper's first-order problem) through the first-order
    kernel: bitwise equal to the oracle (states, sweeps, energy samples, Delta
    H^loc, the H entry point) on the paper's IC plus perturbed members; the
    partitioned mode is rejected."""
    w = wl.schwarzschild(batch=45, nsteps=600)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=40,
                        local_energy=True) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        ig.integrate(Y, ws, energy=E, iters=it)
        rc, st = ig.stats(ws)
        d = ig.local_energy_error(ws).cpu().numpy()
        H = ig.energy(Y).cpu().numpy()
        yg = Y.cpu().numpy()
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, mode=orc.FIRST_ORDER, energy_every=40,
                      local_energy=True)
    assert rc == irk.OK
    assert np.array_equal(yg, o["y"]) and np.array_equal(it.cpu().numpy(), o["iters"])
    assert np.array_equal(E.cpu().numpy(), o["energy"]) and np.array_equal(d, o["dhloc"])
    assert np.array_equal(H, [orc.energy(w.problem, 4, w.params, o["y"][:, b]) for b in range(w.batch)])
    assert np.abs(o["energy"] + 0.5).max() < 1e-13
    with pytest.raises(irk.IrkError):
        irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mode=irk.PARTITIONED)


def test_work_queue_nbody_bitwise(irk, orc):
    """Warp-level work queue of the body-per-lane kernel (16,384 = 3,276 full warp
    slots + a partial one), more warp slots than resident warps, units of 13
    steps, energy samples and Delta H^loc across units; equal to the single
    launch, to the chunked cost-sorted launches (whose permutation once overran
    its buffer for this mapping), to the stage-per-lane queue kernel (the auto
    mapping at this batch) and to the oracle."""
    w = wl.six_body_ensemble(batch=16384, nsteps=130)
    outs = []
    # (1, 26): chunked + cost-sorted permutation; mapping 8: stage per lane (ens_nbody8)
    for sched, bal, mp in ((1, 0, 1), (2, 13, 1), (1, 26, 1), (2, 13, 8), (0, -1, 0)):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=26,
                            balance=bal, schedule=sched, local_energy=True, mapping=mp) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
            it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
            ig.integrate(Y, ws, energy=E, iters=it)
            rc, st = ig.stats(ws)
            outs.append((Y.cpu().numpy(), E.cpu().numpy(), it.cpu().numpy(), st,
                         ig.local_energy_error(ws).cpu().numpy()))
    for o in outs[1:]:
        assert np.array_equal(outs[0][0], o[0]) and np.array_equal(outs[0][1], o[1])
        assert np.array_equal(outs[0][2], o[2]) and outs[0][3] == o[3]
        assert np.array_equal(outs[0][4], o[4])
    idx = np.r_[np.arange(0, w.batch, 1499), w.batch - 1]
    orr = orc.integrate(w.problem, w.y[:, idx], w.params, w.h, w.nsteps, energy_every=26, local_energy=True)
    assert np.array_equal(outs[1][0][:, idx], orr["y"]) and np.array_equal(outs[1][1][:, idx], orr["energy"])
    assert np.array_equal(outs[1][2][idx], orr["iters"]) and np.array_equal(outs[1][4][idx], orr["dhloc"])


def test_nbody_stage_per_lane_mapping(irk, orc):
    """IRK_NBODY with IRK_OPT_MAPPING = 8 (stage per lane, all pair weights of a
    stage in one lane, shared-memory all-gather) equals the body-per-lane mapping
    and the oracle bit for bit, over two chained calls with energy samples and
    Delta H^loc, on a batch that leaves groups idle at the end of the queue."""
    w = wl.six_body_ensemble(batch=601, nsteps=400)
    outs = []
    for mp in (8, 1):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps // 2, w.batch, w.params, energy_every=40,
                            mapping=mp, local_energy=True) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
            it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
            ig.integrate(Y, ws, energy=E, iters=it)
            E1, it1 = E.cpu().numpy().copy(), it.cpu().numpy().copy()
            ig.integrate(Y, ws, energy=E, iters=it)
            outs.append((Y.cpu().numpy(), E1, E.cpu().numpy(), it1 + it.cpu().numpy(),
                         ig.local_energy_error(ws).cpu().numpy(), ig.stats(ws)[1]))
    for a_, b_ in zip(outs[0][:5], outs[1][:5]):
        assert np.array_equal(a_, b_)
    assert outs[0][5] == outs[1][5]
    idx = np.arange(0, w.batch, 97)
    o1 = orc.integrate(w.problem, w.y[:, idx], w.params, w.h, w.nsteps // 2, energy_every=40)
    o2 = orc.integrate(w.problem, o1["y"], w.params, w.h, w.nsteps // 2, energy_every=40, local_energy=True,
                       n0=w.nsteps // 2, hist=o1["hist"])
    assert np.array_equal(outs[0][0][:, idx], o2["y"]) and np.array_equal(outs[0][2][:, idx], o2["energy"])
    assert np.array_equal(outs[0][3][idx], o1["iters"] + o2["iters"])
    assert np.array_equal(outs[0][4][idx], o2["dhloc"])


def test_million_trajectory_batch(irk, orc):
    """2^20 Kepler trajectories (18 units of work per queue lane, 16 M-entry
    SoA rows), 60 steps with energy samples: sampled members bitwise equal to
    the oracle."""
    B, ns = 1 << 20, 60
    w = wl.kepler_ensemble(batch=B, nsteps=ns)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=20) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), B), dtype=torch.float64, device="cuda")
        it = torch.zeros(B, dtype=torch.int64, device="cuda")
        ig.integrate(Y, ws, energy=E, iters=it)
        rc, st = ig.stats(ws)
        idx = np.r_[0, np.arange(1, B, B // 61), B - 1]
        yg, Eg, itg = Y.cpu().numpy()[:, idx], E.cpu().numpy()[:, idx], it.cpu().numpy()[idx]
    o = orc.integrate(w.problem, np.ascontiguousarray(w.y[:, idx]), w.params, w.h, w.nsteps, energy_every=20)
    assert rc == irk.OK
    assert np.array_equal(yg, o["y"]) and np.array_equal(Eg, o["energy"]) and np.array_equal(itg, o["iters"])


# ------------------------------------------------------------------ config 3
def test_config3_six_body_ragged_energy(irk, orc):
    """Config-3 generator, ragged batch of 37 members, 3,000 steps, energy every
    250 steps; body-per-lane kernel vs oracle, bitwise."""
    w = wl.six_body_ensemble(batch=37, nsteps=3000)
    g = run_gpu(irk, w, energy_every=250)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=250)
    assert_parity(g, o, energy=True)


def test_config3_full_length_subset(irk, orc):
    """Config 3 at full length (50,000 steps) on 48 members, bitwise."""
    w = wl.six_body_ensemble(batch=48)
    g = run_gpu(irk, w)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps)
    assert_parity(g, o)


def test_config3_full_batch_sampled(irk, orc):
    """Config 3 at full batch (16,384 members) in the default launch (body-per-lane
    work queue), 2,000 steps; oracle on 40 sampled members."""
    w = wl.six_body_ensemble(nsteps=2000)
    g = run_gpu(irk, w)
    idx = np.linspace(0, w.batch - 1, 40).astype(int)
    o = orc.integrate(w.problem, w.y[:, idx], w.params, w.h, w.nsteps)
    assert_parity(dict(y=g["y"][:, idx], iters=g["iters"][idx]), o)


@pytest.mark.parametrize("mapping", [1, 8])
def test_nbody_small_n_variants(irk, orc, mapping):
    """Other N of both N-body mappings (N = 2, 3, 4, 5, 7, 8; body per lane and
    stage per lane): random softened systems, bitwise."""
    rng = np.random.default_rng(3)
    for N in (2, 3, 4, 5, 7, 8):
        B = 23
        q = rng.standard_normal((3 * N, B))
        v = 0.3 * rng.standard_normal((3 * N, B))
        params = np.concatenate([[1.0, 0.05], rng.uniform(0.2, 1.0, N)])
        w = wl.Workload(f"nb{N}", wl.NBODY, 6 * N, np.concatenate([q, v]), params, 0.01, 300)
        g = run_gpu(irk, w, energy_every=100, mapping=mapping)
        o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=100)
        assert_parity(g, o, energy=True)


def test_nbody_energy_entry_point(irk, orc):
    w = wl.six_body_ensemble(batch=50)
    with irk.Integrator(w.problem, w.dim, w.h, 1, w.batch, w.params) as ig:
        H = ig.energy(torch.tensor(w.y, device="cuda")).cpu().numpy()
    Ho = np.array([orc.energy(w.problem, w.dim, w.params, w.y[:, b]) for b in range(w.batch)])
    assert np.array_equal(H, Ho)


# ------------------------------------------------------------------ config 4
def test_config4_fpu_ragged_energy(irk, orc):
    """Config-4 generator (N = 64, beta = 1, h = 0.1), 19 chains, 4,000 steps,
    energy every 500; site-per-lane kernel vs oracle, bitwise."""
    w = wl.fpu_ensemble(batch=19, nsteps=4000)
    g = run_gpu(irk, w, energy_every=500)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=500)
    assert_parity(g, o, energy=True)


def test_config4_full_length_subset(irk, orc):
    """Config 4 at full length (100,000 steps) on 16 chains, bitwise."""
    w = wl.fpu_ensemble(batch=16)
    g = run_gpu(irk, w)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps)
    assert_parity(g, o)


def test_config4_full_batch_sampled(irk, orc):
    """Config 4 at full batch (4,096 chains), 3,000 steps, default launch (warp-level
    work queue); oracle on 24 sampled chains."""
    w = wl.fpu_ensemble(nsteps=3000)
    g = run_gpu(irk, w)
    idx = np.linspace(0, w.batch - 1, 24).astype(int)
    o = orc.integrate(w.problem, w.y[:, idx], w.params, w.h, w.nsteps)
    assert_parity(dict(y=g["y"][:, idx], iters=g["iters"][idx]), o)


def test_fpu_other_sizes_and_energy_entry(irk, orc):
    for N in (32, 96, 128):
        w = wl.fpu_ensemble(batch=5, nsteps=500, N=N)
        g = run_gpu(irk, w, energy_every=100)
        o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=100)
        assert_parity(g, o, energy=True)
    for N in (64, 96):
        w = wl.fpu_ensemble(batch=33, N=N)
        with irk.Integrator(w.problem, w.dim, w.h, 1, w.batch, w.params) as ig:
            H = ig.energy(torch.tensor(w.y, device="cuda")).cpu().numpy()
        Ho = np.array([orc.energy(w.problem, w.dim, w.params, w.y[:, b]) for b in range(w.batch)])
        assert np.array_equal(H, Ho)


# ------------------------------------------------------------------ config 5
def test_config5_plummer_small_full_length_energy(irk, orc):
    """Plummer N = 1,024 (one j-block), 200 steps, energy every 50: the large-N
    path (pos / blocked-force / vel kernels) vs the oracle, bitwise."""
    w = wl.plummer(N=1024, nsteps=200)
    g = run_gpu(irk, w, energy_every=50)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=50)
    assert_parity(g, o, energy=True)


@pytest.mark.parametrize("N,nsteps,chunks", [(2500, 25, 5), (1025, 6, 2), (1023, 6, 1)])
def test_config5_ragged_blocks(irk, orc, N, nsteps, chunks):
    """Ragged j-blocks: N = 2,500 (three blocks, the last partial, TMA-staged);
    N = 1,025 (a one-body last block: odd, so gathered instead of bulk-copied);
    N = 1,023 (one odd block, gathered)."""
    w = wl.plummer(N=N, nsteps=nsteps)
    g = run_gpu(irk, w, chunks=chunks)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps)
    assert_parity(g, o)


def test_config5_full_size_first_steps(irk, orc):
    """Config 5 at full size (N = 8,192) for the first 4 steps, bitwise."""
    w = wl.plummer(nsteps=4)
    g = run_gpu(irk, w, energy_every=2)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=2)
    assert_parity(g, o, energy=True)


@pytest.mark.parametrize("vshards", [1, 4])
def test_config5_device_loop_equals_host_loop(irk, orc, vshards):
    """IRK_OPT_DEVICE_LOOP: the sweeps of the large-N path as a CUDA-graph
    conditional WHILE loop (segments end at energy samples) give the host-loop
    and oracle results bit for bit, and the graph loop is what ran."""
    w = wl.plummer(N=1024, nsteps=9)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=4)
    outs = []
    for dl in (1, 0):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params, energy_every=4, vshards=vshards,
                            device_loop=dl) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            E = torch.zeros((ig.n_energy(), 1), dtype=torch.float64, device="cuda")
            it = torch.zeros(1, dtype=torch.int64, device="cuda")
            ig.integrate(Y, ws, energy=E, iters=it)
            assert ig.get_option(irk.INFO_DEVICE_LOOP_USED) == dl
            outs.append((Y.cpu().numpy(), E.cpu().numpy(), int(it.item())))
    for y, E, it in outs:
        assert np.array_equal(y, o["y"]) and np.array_equal(E, o["energy"]) and it == int(o["iters"][0])


# ---------------------------------------------------------- first-order mode
def test_first_order_mode_parity(irk, orc):
    """IRK_OPT_MODE = 1 (Eqs. IRK_init / IRK_FP, stop test over all D from k = 1)
    vs the oracle's first-order step, bitwise, Kepler and Henon-Heiles, chunked."""
    for w in (wl.kepler_ensemble(batch=200, nsteps=600), wl.henon_heiles(batch=70, nsteps=600, h=0.05)):
        with irk.Integrator(w.problem, w.dim, w.h, 200, w.batch, w.params, mode=irk.FIRST_ORDER,
                            energy_every=100) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
            E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
            tot = np.zeros(w.batch, dtype=np.int64)
            for _ in range(3):
                ig.integrate(Y, ws, energy=E, iters=it)
                tot += it.cpu().numpy()
            y = Y.cpu().numpy()
            hist = ig.hist_view(ws).cpu().numpy()
        o = orc.integrate(w.problem, w.y, w.params, w.h, 600, mode=orc.FIRST_ORDER)
        assert np.array_equal(y, o["y"]) and np.array_equal(tot, o["iters"])
        assert np.array_equal(hist, o["hist"].transpose(1, 2, 0))


def test_config5_virtual_shards_bitwise(irk, orc):
    """The body-sharded code path (slot-major gathered stage positions, global
    stop flag, per-shard force/vel) driven as P = 2, 4, 8 virtual shards on one
    GPU equals the oracle bit for bit (the j-order does not depend on P)."""
    w = wl.plummer(N=1024, nsteps=12)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=4)
    for P in (2, 4, 8):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params, energy_every=4, vshards=P) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            E = torch.zeros((ig.n_energy(), 1), dtype=torch.float64, device="cuda")
            it = torch.zeros(1, dtype=torch.int64, device="cuda")
            ig.integrate(Y, ws, energy=E, iters=it)
            assert np.array_equal(Y.cpu().numpy(), o["y"]), P
            assert np.array_equal(E.cpu().numpy(), o["energy"]), P
            assert int(it.item()) == int(o["iters"][0])


def test_config5_nccl_single_rank_path(irk, orc):
    """irk_set_comm with one rank: the NCCL exchange (in-place ncclAllGather per
    iteration, energy gathers) runs and the result is bitwise the oracle's."""
    import torch.distributed as dist
    w = wl.plummer(N=512, nsteps=6)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=3)
    try:
        uid = irk.nccl_unique_id()
    except irk.IrkError:
        pytest.skip("NCCL not loadable")
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params, energy_every=3) as ig:
        ig.set_comm(uid, 0, 1)
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), 1), dtype=torch.float64, device="cuda")
        ig.integrate(Y, ws, energy=E)
        print("NCCL path ran the device loop:", ig.get_option(irk.INFO_DEVICE_LOOP_USED))
        H = ig.energy(Y).cpu().numpy()
        assert np.array_equal(Y.cpu().numpy(), o["y"])
        assert np.array_equal(E.cpu().numpy(), o["energy"])
        assert H[0] == orc.energy(w.problem, w.dim, w.params, o["y"][:, 0])


def _direct_comm_run(irk, w, exchange, calls=1, energy_every=0, device_loop=1, y=None):
    """IRK_NBODY_DIRECT under a 1-rank communicator, `calls` chained calls of w.nsteps."""
    try:
        uid = irk.nccl_unique_id()
    except irk.IrkError:
        pytest.skip("NCCL not loadable")
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params, energy_every=energy_every,
                        device_loop=device_loop, exchange=exchange) as ig:
        ig.set_comm(uid, 0, 1)
        Y = torch.tensor(w.y if y is None else y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        E = (torch.zeros((ig.n_energy(), 1), dtype=torch.float64, device="cuda") if energy_every else None)
        it = torch.zeros(1, dtype=torch.int64, device="cuda")
        Es, its = [], 0
        for _ in range(calls):
            ig.integrate(Y, ws, energy=E, iters=it)
            its += int(it.item())
            if E is not None:
                Es.append(E.cpu().numpy().copy())
        rc, st = ig.stats(ws)
        assert ig.get_option(irk.OPT_EXCHANGE) == exchange
        return dict(y=Y.cpu().numpy(), iters=its, rc=rc, stats=st,
                    energy=(np.concatenate([Es[0]] + [e[1:] for e in Es[1:]]) if Es else None),
                    loop=ig.get_option(irk.INFO_DEVICE_LOOP_USED))


@pytest.mark.parametrize("device_loop", [1, 0])
def test_config5_fused_exchange_single_rank(irk, orc, device_loop):
    """IRK_OPT_EXCHANGE = 1 (NEXT f3): nbd_pos stores Q^[k] through the NVLink
    mapping of a symmetric NCCL window, its last CTA signals arrival, nbd_or waits
    -- double-buffered by exchange epoch.  One rank (the box has one GPU): the
    peer-pointer stores, the arrival/wait barrier and the buffer/flag parity over
    three chained calls (odd sweep counts flip the parity) give the oracle's bits."""
    w = wl.plummer(N=512, nsteps=5)
    o = orc.integrate(w.problem, w.y, w.params, w.h, 15, energy_every=5)
    g = _direct_comm_run(irk, w, 1, calls=3, energy_every=5, device_loop=device_loop)
    assert g["loop"] == device_loop
    assert np.array_equal(g["y"], o["y"])
    assert np.array_equal(g["energy"], o["energy"])
    assert g["iters"] == int(o["iters"][0]) and g["rc"] == irk.OK


def test_config5_exchange_switch_between_calls(irk, orc):
    """IRK_OPT_EXCHANGE switched 1 -> 0 -> 1 between chained calls (the window
    stays allocated while the all-gather runs): still the oracle's bits."""
    try:
        uid = irk.nccl_unique_id()
    except irk.IrkError:
        pytest.skip("NCCL not loadable")
    w = wl.plummer(N=512, nsteps=3)
    o = orc.integrate(w.problem, w.y, w.params, w.h, 9)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params, exchange=1) as ig:
        ig.set_comm(uid, 0, 1)
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        for ex in (1, 0, 1):
            ig.set_option(irk.OPT_EXCHANGE, ex)
            ig.integrate(Y, ws)
        assert np.array_equal(Y.cpu().numpy(), o["y"])


def test_config5_fused_exchange_divergence(irk):
    """A non-finite body: the divergence flag travels through the fused exchange
    (nbd_vel's store into the next buffer, the final barrier) exactly as through
    the all-gather -- same frozen state, same first bad step, same sweep count."""
    w = wl.plummer(N=256, nsteps=6)
    y = w.y.copy()
    y[3 * 256 + 7, 0] = np.inf  # a velocity component of body 2
    outs = [_direct_comm_run(irk, w, ex, calls=2, y=y) for ex in (0, 1)]
    assert outs[0]["rc"] == irk.E_DIVERGED and outs[1]["rc"] == irk.E_DIVERGED
    assert outs[0]["stats"] == outs[1]["stats"] and outs[0]["iters"] == outs[1]["iters"]
    assert np.array_equal(outs[0]["y"], outs[1]["y"], equal_nan=True)


# ------------------------------------------------- local energy error (f2)
@pytest.mark.parametrize("which", ["kepler", "hh", "hh_fo", "nbody", "fpu"])
def test_local_energy_error_parity(irk, orc, which):
    """In-kernel Delta H^loc_max (Eq. DHlocmax, IRK_OPT_LOCAL_ENERGY) equals the
    oracle's bit for bit, also across chunked calls and balance chunks."""
    mode = 0
    if which == "kepler":
        w = wl.kepler_ensemble(batch=9000, nsteps=400)
    elif which == "hh":
        w = wl.henon_heiles(batch=100, nsteps=400)
    elif which == "hh_fo":
        w = wl.henon_heiles(batch=50, nsteps=300, h=0.05)
        mode = 1
    elif which == "nbody":
        w = wl.six_body_ensemble(batch=12, nsteps=300)
    else:
        w = wl.fpu_ensemble(batch=6, nsteps=300)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps // 2, w.batch, w.params, mode=mode,
                        local_energy=True) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        ig.integrate(Y, ws)
        d1 = ig.local_energy_error(ws).cpu().numpy()
        y1 = Y.cpu().numpy()
        ig.integrate(Y, ws)
        d2 = ig.local_energy_error(ws).cpu().numpy()
    o1 = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps // 2, mode=mode, local_energy=True)
    o2 = orc.integrate(w.problem, o1["y"], w.params, w.h, w.nsteps // 2, mode=mode, local_energy=True,
                       n0=w.nsteps // 2, hist=o1["hist"])
    assert np.array_equal(y1, o1["y"])
    assert np.array_equal(d1, o1["dhloc"]) and np.array_equal(d2, o2["dhloc"])
    assert np.all(d1 > 0)
