import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2511_03655_b200 import irk, workloads as wl
w = wl.six_body_ensemble(nsteps=1000)
with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mapping=8) as ig:
    Y = torch.tensor(w.y, dtype=torch.float64, device="cuda"); ws = ig.new_workspace()
    ig.integrate(Y, ws); torch.cuda.synchronize(); print(ig.stats(ws))
