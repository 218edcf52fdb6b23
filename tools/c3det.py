"""Diagnostic: config-3 results under different schedules must be bitwise equal;
report differing trajectories and check them against the oracle."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
w = wl.six_body_ensemble(nsteps=nsteps)
variants = [(2, -1), (2, nsteps), (1, 0), (1, -1)]
res = []
for sched, bal in variants:
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, schedule=sched, balance=bal) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda"); ws = ig.new_workspace()
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        ig.integrate(Y, ws, iters=it); torch.cuda.synchronize()
        res.append((Y.cpu().numpy(), it.cpu().numpy()))
diffs = set()
for (s, b), r in zip(variants, res):
    nd = np.nonzero((r[0] != res[0][0]).any(0))[0]
    diffs |= set(nd[:4].tolist())
    print(json.dumps({"schedule": s, "balance": b, "ndiff_vs_first": int(len(nd)), "sweeps": int(r[1].sum())}))
idx = sorted(diffs)[:6]
if idx:
    from oracle import oracle
    o = oracle.integrate(w.problem, np.ascontiguousarray(w.y[:, idx]), w.params, w.h, w.nsteps)
    for (s, b), r in zip(variants, res):
        print(json.dumps({"schedule": s, "balance": b,
                          "oracle_equal": [bool(np.array_equal(r[0][:, i], o["y"][:, k])) for k, i in enumerate(idx)]}))
