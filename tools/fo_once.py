"""One first-order-mode call (Schwarzschild ensemble, 65,536 x 500 steps) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

w = wl.schwarzschild(batch=65536, nsteps=500)
with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params) as ig:
    Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
    ws = ig.new_workspace()
    ig.integrate(Y, ws)
    torch.cuda.synchronize()
    print("rc", ig.stats(ws))
