"""Throughput of the first-order kernel (Schwarzschild, Eq. Ham_SBH) vs batch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

for B in (4096, 16384, 65536):
    w = wl.schwarzschild(batch=B, nsteps=1000)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params) as ig:
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(y0)
        ws = ig.new_workspace()
        it = torch.zeros(B, dtype=torch.int64, device="cuda")
        ts = []
        for _ in range(3):
            Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ig.integrate(Y, ws, iters=it); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        sw = int(it.sum().item())
    ms = min(ts[1:])
    print(json.dumps({"batch": B, "nsteps": w.nsteps, "ms": ms, "traj_steps_per_s": B * w.nsteps / (ms * 1e-3),
                      "sweeps_per_step": sw / (B * w.nsteps), "traj_sweeps_per_s": sw / (ms * 1e-3)}), flush=True)
