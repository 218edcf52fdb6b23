"""GPU parity, round 2: the kernel families no round-1 test ran end to end
(G != 1 / GM != 1 instantiations), config 5 at the parity subsets of
SURVEY.md 8(d) D-5 (first 20 steps at N = 8,192; the full 1,000 steps at
N = 1,024), the resolved-mapping query and the binding's argument checks.

Bar: bitwise equality of states, sweep counts and energy samples with the
scalar-C oracle, plus the north-star tolerances.
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


def _with_params(w, params):
    w.params = np.asarray(params, dtype=np.float64)
    return w


# ------------------------------------------------------ G != 1 instantiations
@pytest.mark.parametrize("mapping", [1, 2, 4, 8, 9])
def test_kepler_gm_not_one_every_mapping(irk, orc, mapping):
    """Kepler with GM = 1.3 runs KeplerT<false> (the full correctly rounded
    division w = GM / r^3, Eq. of the Kepler functor in CANON.md) in every
    per-thread mapping; bitwise with energy samples."""
    w = _with_params(wl.kepler_ensemble(batch=300, nsteps=2000), [1.3])
    g = run_gpu(irk, w, energy_every=250, mapping=mapping)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=250)
    assert_parity(g, o, energy=True)


@pytest.mark.parametrize("mapping", [1, 8])
def test_nbody_g_half_both_mappings(irk, orc, mapping):
    """Six-body ensembles with G = 0.5 (Eq. Ham2 P:L545 carries G): the
    ens_nbody8_kernel<6, false> (stage per lane) and body-per-lane kernels."""
    w = wl.six_body_ensemble(batch=200, nsteps=2000)
    w.params = np.concatenate([[0.5], w.params[1:]])
    g = run_gpu(irk, w, energy_every=500, mapping=mapping)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=500)
    assert_parity(g, o, energy=True)


def test_nbody_direct_g_two_multi_block(irk, orc):
    """One large system with G = 2 (nbd_force_kernel<false>), three j-blocks."""
    w = wl.plummer(N=2500, nsteps=8)
    w.params = np.concatenate([[2.0], w.params[1:]])
    g = run_gpu(irk, w, energy_every=4)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=4)
    assert_parity(g, o, energy=True)


# ------------------------------------------------------ config 5, D-5 subsets
def test_config5_full_size_first_20_steps(irk, orc):
    """Config 5 (N = 8,192 Plummer) for its first 20 steps with energy samples
    every 5 steps, in the launch configuration the bench times (device loop);
    bitwise."""
    w = wl.plummer(nsteps=20)
    g = run_gpu(irk, w, energy_every=5)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=5)
    assert_parity(g, o, energy=True)


def test_config5_n1024_full_1000_steps(irk, orc):
    """The config-5 generator at N = 1,024 for the full 1,000 steps, energy every
    100 steps, bitwise."""
    w = wl.plummer(N=1024, nsteps=1000)
    g = run_gpu(irk, w, energy_every=100)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=100)
    assert_parity(g, o, energy=True)


# ------------------------------------------------------ resolved mapping
@pytest.mark.parametrize("problem,batch,expect", [
    ("kepler", 1, 9), ("kepler", 4096, 9), ("kepler", 8192, 4), ("kepler", 65536, 1),
    ("fpu", 64, 0), ("plummer", 1, 0), ("sixbody", 16384, 9), ("sixbody", 1, 9)])
def test_mapping_used_info(irk, problem, batch, expect):
    """IRK_INFO_MAPPING_USED reports what IRK_OPT_MAPPING auto resolved to."""
    if problem == "kepler":
        w = wl.kepler_ensemble(batch=batch, nsteps=3)
    elif problem == "fpu":
        w = wl.fpu_ensemble(batch=batch, nsteps=3)
    elif problem == "sixbody":
        w = wl.six_body_ensemble(batch=batch, nsteps=3)
    else:
        w = wl.plummer(N=1024, nsteps=1)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ig.integrate(Y, ig.new_workspace())
        torch.cuda.synchronize()
        assert ig.get_option(irk.INFO_MAPPING_USED) == expect


# ------------------------------------------------------ binding checks
def test_binding_rejects_bad_buffers(irk):
    """The C ABI cannot see sizes: the binding refuses wrong dtype / shape /
    device / contiguity before any pointer crosses it."""
    w = wl.kepler_ensemble(batch=64, nsteps=2)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=1) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        bad = [
            dict(y=Y.float()), dict(y=Y[:, :32]), dict(y=Y.t().contiguous().t()),
            dict(energy=E.float()), dict(energy=E[:-1]), dict(energy=None),
            dict(iters=it.int()), dict(iters=it[:10]), dict(ws=ws[:100]),
        ]
        for b in bad:
            kw = dict(y=Y, ws=ws, energy=E, iters=it)
            kw.update(b)
            with pytest.raises(ValueError):
                ig.integrate(kw["y"], kw["ws"], energy=kw["energy"], iters=kw["iters"])
        with pytest.raises(ValueError):
            ig.energy(Y, out=torch.zeros(w.batch, dtype=torch.float32, device="cuda"))
        ig.integrate(Y, ws, energy=E, iters=it)   # the good call still works
        torch.cuda.synchronize()


# ------------------------------------------------------ FPU chains, two warps per chain
@pytest.mark.parametrize("N,batch", [(64, 37), (128, 20)])
def test_fpu_two_warps_per_chain(irk, orc, N, batch):
    """Small batches run the FPU chain with two warps per chain (ens_chainw,
    IRK_CHAINW_MAX): bitwise the oracle, with energy samples, and the same bits as
    the one-warp chunked kernel (IRK_OPT_SCHEDULE = 1)."""
    w = wl.fpu_ensemble(batch=batch, nsteps=600, N=N)
    g = run_gpu(irk, w, energy_every=100)
    o = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps, energy_every=100)
    assert_parity(g, o, energy=True)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, schedule=1) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        ig.integrate(Y, ig.new_workspace())
        torch.cuda.synchronize()
        assert np.array_equal(Y.cpu().numpy(), g["y"])


def test_work_queue_int32_guard(irk):
    """Work-queue chunk indices are int32 (progress / orphan words): a call whose
    step-chunk count reaches 2^31 - 1 is refused with IRK_E_ARG before any launch
    (ADVICE r1), instead of overflowing the counters and hanging."""
    w = wl.kepler_ensemble(batch=131072, nsteps=1)
    with irk.Integrator(w.problem, w.dim, w.h, 2 ** 31 + 7, w.batch, w.params, balance=1) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        with pytest.raises(irk.IrkError) as ei:
            ig.integrate(Y, ig.new_workspace())
        assert ei.value.code == irk.E_ARG
        assert np.array_equal(Y.cpu().numpy(), w.y)
