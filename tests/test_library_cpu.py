"""Host-side checks of the C-ABI library (no GPU): the .so loads and exports
every symbol include/irk.h declares; the library's own tableau (Newton +
Bjorck-Pereyra in __float128) equals, bit for bit, the oracle's independently
computed one and the mpmath round-to-nearest values; argument errors are
reported synchronously by irk_create / irk_set_params / irk_set_option.
"""
import ctypes
import math
import os
import re

import mpmath as mp
import numpy as np
import pytest

from tests import mp_tableau

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def irk():
    from paper_2511_03655_b200 import build, irk
    build.build()
    return irk


def declared_symbols():
    names = []
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            src = open(os.path.join(ROOT, "include", f)).read()
            names += re.findall(r"^\s*(?:const\s+)?[a-zA-Z_][\w\s\*]*?\b(irk_\w+)\s*\(", src, re.M)
    return sorted(set(names))


def test_exports_every_declared_symbol(irk):
    names = declared_symbols()
    assert len(names) >= 12
    lib = ctypes.CDLL(irk.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(irk.SYMBOLS)


def test_library_tableau_bitwise_equals_oracle_and_mpmath(irk, orc):
    c, b, mu, nu = irk.tableau()
    oc, ob, omu, onu = orc.tableau(8)
    assert np.array_equal(c, oc) and np.array_equal(b, ob)
    assert np.array_equal(mu, omu) and np.array_equal(nu, onu)
    c_mp, b_mp, a_mp, nu_mp = mp_tableau.tableau(8)
    for i in range(8):
        assert c[i] == mp_tableau.rn(c_mp[i])
        for j in range(i):
            assert mu[i, j] == mp_tableau.rn(a_mp[i][j] / b_mp[j])


@pytest.mark.parametrize("args", [
    (1, 6, 0.1, 10, 4),          # Kepler needs dim 4
    (4, 4, 0.0, 10, 4),          # h = 0
    (1, 4, float("nan"), 10, 4),
    (1, 4, 0.1, -1, 4),          # nsteps < 0
    (1, 4, 0.1, 10, 0),          # batch < 1
    (1, 4, 0.1, 10, 2**31),      # batch > 2^31 - 1 (int32 trajectory indices)
    (9, 4, 0.1, 10, 4),          # unknown problem
    (2, 13, 0.1, 10, 4),         # N-body dim % 6
    (2, 54, 0.1, 10, 4),         # N-body ensembles: N = 9 unsupported (2 <= N <= 8)
    (3, 7, 0.1, 10, 4),          # FPU odd dim
    (3, 40, 0.1, 10, 4),         # FPU: N must be 32, 64, 96 or 128 (one warp per chain)
    (3, 160, 0.1, 10, 4),        # FPU: N = 80 unsupported
])
def test_create_argument_errors(irk, args):
    with pytest.raises(irk.IrkError):
        irk.Integrator(*args, params=[1.0])


def test_params_and_options_errors(irk):
    with pytest.raises(irk.IrkError):
        irk.Integrator(irk.KEPLER, 4, 0.1, 10, 4, params=[1.0, 2.0])
    with pytest.raises(irk.IrkError):
        irk.Integrator(irk.KEPLER, 4, 0.1, 10, 4, params=[float("inf")])
    with pytest.raises(irk.IrkError):
        irk.Integrator(irk.KEPLER, 4, 0.1, 10, 4, params=[1.0], max_iters=0)
    with pytest.raises(irk.IrkError):  # first-order mode is built for the per-thread problems only
        irk.Integrator(irk.FPU_BETA, 128, 0.1, 10, 4, params=[1.0], mode=irk.FIRST_ORDER)
    irk.Integrator(irk.HENON_HEILES, 4, 0.1, 10, 4, params=[1.0, 0.0], mode=irk.FIRST_ORDER).close()
    for mp in (irk.MAP_AUTO, irk.MAP_G1, irk.MAP_G2, irk.MAP_G4, irk.MAP_G8, irk.MAP_G8M):  # lanes per trajectory
        k = irk.Integrator(irk.KEPLER, 4, 0.1, 10, 4, params=[1.0], mapping=mp)
        assert k.get_option(irk.OPT_MAPPING) == mp
        k.close()
    irk.Integrator(irk.HENON_HEILES, 4, 0.1, 10, 4, params=[1.0, 0.1], mapping=irk.MAP_G8M).close()
    with pytest.raises(irk.IrkError):  # g8m: Kepler, Henon-Heiles and the N-body ensembles only
        irk.Integrator(irk.FPU_BETA, 128, 0.1, 10, 4, params=[1.0], mapping=irk.MAP_G8M)
    for mp in (3, 16):
        with pytest.raises(irk.IrkError):
            irk.Integrator(irk.KEPLER, 4, 0.1, 10, 4, params=[1.0], mapping=mp)
    with pytest.raises(irk.IrkError):  # g2 / g4 are built for the per-thread problems only
        irk.Integrator(irk.FPU_BETA, 128, 0.1, 10, 4, params=[1.0], mapping=irk.MAP_G4)
    with pytest.raises(irk.IrkError):  # the fused exchange is an IRK_NBODY_DIRECT option
        irk.Integrator(irk.KEPLER, 4, 0.1, 10, 4, params=[1.0]).set_option(irk.OPT_EXCHANGE, 1)
    with pytest.raises(irk.IrkError):
        irk.Integrator(irk.NBODY_DIRECT, 6 * 64, 0.1, 10, 1, params=[1.0, 0.01] + [1 / 64] * 64, exchange=2)
    d = irk.Integrator(irk.NBODY_DIRECT, 6 * 64, 0.1, 10, 1, params=[1.0, 0.01] + [1 / 64] * 64, exchange=1)
    assert d.get_option(irk.OPT_EXCHANGE) == 1
    d.close()
    w = irk.Integrator(irk.KEPLER, 4, -0.1, 10, 4, params=[1.0])  # negative h is allowed
    assert w.workspace_bytes == 64 + 8 * 8 * 4 * 4 + 8 * 4 * 4 + 4 * (256 + 2 * 4 + 1024)
    w.close()


def test_build_is_sm100a_only(irk):
    """The library carries sm_100a SASS (cuobjdump) and nothing for other archs."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", irk.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_nccl_unique_id_loads_nccl_at_run_time(irk):
    """irk_nccl_unique_id dlopens NCCL (no link-time dependency) and returns 128 bytes."""
    try:
        u = irk.nccl_unique_id()
    except irk.IrkError:
        pytest.skip("NCCL not loadable here")
    assert len(u) == 128 and u != bytes(128)
