"""Config 3: body-per-lane (default) vs stage-per-lane (IRK_OPT_MAPPING = 8):
time per call and bitwise agreement."""
import json
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
w = wl.six_body_ensemble(nsteps=nsteps, batch=batch)
res = []
for mp in (0, 8):
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mapping=mp, energy_every=nsteps // 5,
                        local_energy=True) as ig:
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda"); Y = torch.empty_like(y0)
        ws = ig.new_workspace(); it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        E = torch.zeros((ig.n_energy(), w.batch), dtype=torch.float64, device="cuda")
        ts = []
        for r in range(4):
            Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); ig.integrate(Y, ws, iters=it, energy=E); e1.record(); torch.cuda.synchronize()
            ts.append(round(e0.elapsed_time(e1), 2))
        rc, st = ig.stats(ws)
        res.append((Y.cpu(), it.cpu(), E.cpu(), ig.local_energy_error(ws).cpu()))
        print(json.dumps({"mapping": mp, "ms": ts, "rc": rc, "sweeps": int(it.sum())}), flush=True)
same = [bool(torch.equal(a, b)) for a, b in zip(res[0], res[1])]
nd = int((res[0][0] != res[1][0]).any(0).sum())
print(json.dumps({"bitwise_y_it_E_dloc": same, "ndiff_traj": nd}))
