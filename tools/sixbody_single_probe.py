"""Single six-body trajectory (config-3 stand-in): time vs step count for both
N-body mappings (linearity check of the stage-per-lane kernel at batch 1)."""
import json
import sys

import torch

sys.path.insert(0, '/root/repo')
from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

six = wl.six_body_ensemble(batch=1)
T1 = six.h * 200.0
for h, n in ((T1 / 100, 20000), (T1 / 200, 20000), (T1 / 50, 20000)):
    for mp in (8, 1):
        with irk.Integrator(six.problem, six.dim, h, n, 1, six.params, mapping=mp) as ig:
            y0 = torch.tensor(six.y[:, :1], dtype=torch.float64, device="cuda")
            Y = torch.empty_like(y0)
            ws = ig.new_workspace()
            it = torch.zeros(1, dtype=torch.int64, device="cuda")
            ts = []
            for _ in range(3):
                Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); ig.integrate(Y, ws, iters=it); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
        print(json.dumps(dict(h=h, nsteps=n, mapping=mp, ms=round(min(ts[1:]), 1), sweeps=int(it.item()),
                              us_per_sweep=round(1e3 * min(ts[1:]) / int(it.item()), 3))), flush=True)
