"""bench.py's multi-GPU launch contract, on CPU (the reference arm needs no GPU):
`--gpus N` without a torchrun environment re-launches itself with N ranks and
rank 0 alone prints one JSON line with n_gpus = N; under torchrun a WORLD_SIZE
that differs from --gpus is refused with exit code 2."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=ROOT)


def test_world_size_mismatch_is_refused():
    p = _run(["--gpus", "1", "--impl", "reference"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode == 2
    assert "WORLD_SIZE" in p.stderr


def test_self_launch_two_ranks_one_line():
    p = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.gpu
def test_bench_own_arm_contract_keys():
    """The GPU arm at full config-2 size (one timed step, no extra configs): the keys the
    driver reads, the roofline against the FP64 peak, e2e with declared copies, and a
    non-zero count of this library's launches."""
    p = _run(["--steps", "1", "--warmup", "3", "--configs", "none", "--no-cpu-baseline"], timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["config"]["batch"] == 65536 and d["config"]["nsteps"] == 10000
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0 < r["frac"] < 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 65536 * 4 * 8 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["status"]["rc"] == 0 and d["status"]["diverged_traj"] == 0
    assert "sm_mhz" in d["clocks"]
