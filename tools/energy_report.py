"""Energy behaviour of the full-size ensembles on the GPU: relative energy error
max_n |H(y_n) - H(y_0)| / |H(y_0)| per trajectory (Eq. DHglobmax) from
in-kernel samples, and the in-kernel Delta H^loc_max (Eq. DHlocmax), summarised
over the ensemble (median / p99 / max), plus the drift between the first and
last tenth of the run.  Bounded, non-drifting energy errors are what a
symplectic 16th-order scheme at these step sizes should show.

python tools/energy_report.py [--configs 2,3,4] [--out profiles/r1/energy_report.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4")
    ap.add_argument("--samples", type=int, default=100)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = []
    for cfg in [int(x) for x in a.configs.split(",")]:
        w = wl.config(cfg)
        E = max(1, w.nsteps // a.samples)
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=E,
                            local_energy=True) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ws = ig.new_workspace()
            H = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
            ig.integrate(Y, ws, energy=H)
            rc, st = ig.stats(ws)
            dloc = ig.local_energy_error(ws).cpu().numpy()
            H = H.cpu().numpy()
        rel = np.abs((H - H[0]) / H[0])
        glob = rel.max(axis=0)
        m = H.shape[0] // 10
        drift = np.abs(rel[-m:].mean(axis=0) - rel[1:m + 1].mean(axis=0))
        q = lambda x: dict(median=float(np.median(x)), p99=float(np.quantile(x, 0.99)), max=float(x.max()))
        r = dict(config=cfg, workload=w.name, batch=w.batch, nsteps=w.nsteps, h=w.h, samples=H.shape[0],
                 dH_glob_max=q(glob), dH_loc_max=q(dloc), drift_first_vs_last_tenth=q(drift), rc=rc, stats=st)
        print(json.dumps(r), flush=True)
        res.append(r)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
