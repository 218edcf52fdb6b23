"""IRKGL16 work-precision sweep on the GPU: the IRKGL16 side of the paper's
Figures 1-4 on its own test problems, single trajectory and
ensemble (NEXT f2 of SURVEY 8(f)).

For each problem and step size h, one trajectory from the paper's initial
condition is integrated over a fixed time span T, and we record
  - Delta H^loc_max (Eq. DHlocmax; in-kernel, IRK_OPT_LOCAL_ENERGY),
  - Delta H^glob_max (Eq. DHglobmax; from per-step energy samples),
  - function evaluations = 8 x fixed-point sweeps (the paper's work measure),
  - GPU time of the single-trajectory call (CUDA events) and, for an ensemble of
    B perturbed copies, the throughput in trajectory-steps/s.
Problems: the Schwarzschild black hole (Eq. Ham_SBH, first-order form, paper's
IC r = 11; the paper gives no time span: T = 163,840 = 10,240 reference steps of
h = 16), Henon-Heiles (T = 2 pi 10^4, IC q = (0, 0.3), p2 = 0.2, H =
1/12), and the config-3 six-body stand-in for the outer Solar System (member 0,
T = 200 innermost periods).

python tools/work_precision.py [--out profiles/r1/work_precision.json] [--batch 4096]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402


def run(w, h, nsteps, batch_y, energy_every=1):
    B = batch_y.shape[1]
    with irk.Integrator(w.problem, w.dim, h, nsteps, B, w.params, energy_every=energy_every,
                        local_energy=True) as ig:
        y0 = torch.tensor(batch_y, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(y0)
        ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), B), dtype=torch.float64, device="cuda") if energy_every else None
        it = torch.zeros(B, dtype=torch.int64, device="cuda")
        ts = []
        for _ in range(3):
            Y.copy_(y0)
            ws.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ig.integrate(Y, ws, energy=E, iters=it)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        rc, st = ig.stats(ws)
        dloc = ig.local_energy_error(ws).cpu().numpy()
        out = dict(ms=min(ts[1:]), rc=rc, sweeps=it.cpu().numpy(), dloc=dloc)
        if E is not None:
            En = E.cpu().numpy()
            out["dglob"] = np.nanmax(np.abs((En - En[0]) / En[0]), axis=0)
        return out


def problems():
    sbh = wl.schwarzschild()
    hh = wl.henon_heiles()
    six = wl.six_body_ensemble(batch=1)
    T1 = six.h * 200.0  # innermost period (config 3 uses h = T1/200)
    return [
        ("schwarzschild", sbh, 163840.0, [64.0, 48.0, 40.0, 32.0, 24.0, 20.0, 16.0]),
        ("henon_heiles", hh, 2 * math.pi * 1e4,
         [2 * math.pi / k for k in (4, 6, 8, 12, 16, 24, 32)]),
        ("six_body_standin", six, 200 * T1, [T1 / k for k in (8, 10, 12, 15, 20, 25, 35, 50, 100, 200)]),
    ]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--batch", type=int, default=4096)
    a = ap.parse_args()
    res = []
    for name, w, T, hs in problems():
        for h in hs:
            n = int(round(T / h))
            one = run(w, h, n, w.y[:, :1])
            # ensemble throughput: B copies with relative 1e-8 perturbations (seeded)
            g = np.random.default_rng(1234)
            yb = w.y[:, :1] * (1.0 + 1e-8 * g.standard_normal((w.dim, a.batch)))
            yb[:, 0] = w.y[:, 0]
            if name == "schwarzschild":
                yb = wl.schwarzschild(batch=a.batch).y  # stay on the H = -1/2 shell
            ens = run(w, h, n, yb, energy_every=0)
            r = dict(problem=name, h=h, nsteps=n, T=n * h, fevals=int(8 * one["sweeps"][0]),
                     sweeps_per_step=float(one["sweeps"][0]) / n, dH_loc_max=float(one["dloc"][0]),
                     dH_glob_max=float(one["dglob"][0]), gpu_ms_single=one["ms"], rc=one["rc"],
                     ensemble_batch=a.batch, ensemble_ms=ens["ms"],
                     ensemble_traj_steps_per_s=a.batch * n / (ens["ms"] * 1e-3),
                     ensemble_dH_loc_max_median=float(np.median(ens["dloc"])))
            print(json.dumps(r), flush=True)
            res.append(r)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
