"""Per-config throughput of the CUDA path (configs 1-4 of BASELINE.json) with the
algorithmic-flop roofline fraction; writes one JSON object per config.

python tools/bench_all.py [--configs 1,2,3,4] [--out file.json]
Timing: CUDA events around irk_integrate on the launching stream, state reset
and L2 flush outside the timed region, best of --reps after one warm-up call.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

PEAK = 148 * 64 * 2 * 1.965e9  # FP64 FMA pipe, flop/s


def f_flops(w):
    """Canonical flops of one RHS evaluation g(q)."""
    if w.problem == wl.KEPLER:
        return 8
    if w.problem == wl.HENON_HEILES:
        return 13
    if w.problem == wl.FPU_BETA:
        N = w.dim // 2
        return 5 * (N + 1) + N
    if w.problem == wl.NBODY:
        N = w.dim // 6
        return 26 * N * (N - 1) // 2
    if w.problem == wl.NBODY_DIRECT:  # canonical direct sum incl. j = i: 19 flops per (i, j)
        N = w.dim // 6
        return 19 * N * N
    raise ValueError


def run(cfg, reps):
    w = wl.config(cfg)
    d = w.dim // 2
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params) as ig:
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(y0)
        ws = ig.new_workspace()
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        ts = []
        for r in range(reps + 1):
            Y.copy_(y0)
            ws.zero_()
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ig.integrate(Y, ws, iters=it)
            e1.record()
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1) * 1e-3)
        rc, st = ig.stats(ws)
    T = min(ts)
    sweeps = int(it.sum().item())
    steps = w.batch * w.nsteps
    fl = steps * 144 * d + sweeps * (280 * d + 8 * f_flops(w))
    out = {"config": cfg, "workload": w.name, "batch": w.batch, "nsteps": w.nsteps, "dim": w.dim,
           "seconds": T, "traj_steps_per_s": steps / T, "sweeps_per_step": sweeps / steps,
           "alg_tflops": fl / T / 1e12, "frac_fp64_peak": fl / T / PEAK, "times": ts, "rc": rc, **st}
    if w.problem == wl.NBODY_DIRECT:  # one system -> system-steps/s and pair interactions/s
        N = w.dim // 6
        out["system_steps_per_s"] = w.nsteps / T
        out["pair_interactions_per_s"] = float(N) * N * 8 * sweeps / T  # (i, j) incl. i = j (zero force), 8 stages
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = []
    for c in [int(x) for x in a.configs.split(",")]:
        r = run(c, a.reps)
        print(json.dumps(r), flush=True)
        res.append(r)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
