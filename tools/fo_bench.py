"""First-order mode (Schwarzschild, Eq. Ham_SBH): work-queue per-thread kernel
(mapping 1) vs stage-per-lane (mapping 8) across batch sizes, bitwise check."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

for B in (1, 64, 1024, 4096, 8192, 16384, 65536):
    w = wl.schwarzschild(batch=B, nsteps=1000)
    out = {}
    for mp in (1, 8):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mapping=mp) as ig:
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
            out[mp] = (min(ts[1:]), Y.cpu(), it.cpu())
    print(json.dumps({"batch": B, "nsteps": w.nsteps, "ms_g1": out[1][0], "ms_g8": out[8][0],
                      "bitwise": bool(torch.equal(out[1][1], out[8][1]) and torch.equal(out[1][2], out[8][2])),
                      "traj_steps_per_s_best": B * w.nsteps / (min(out[1][0], out[8][0]) * 1e-3)}), flush=True)
