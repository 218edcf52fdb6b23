import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2511_03655_b200 import irk, workloads as wl
from oracle import oracle
for B, ns in ((1 << 20, 60), (300001, 200)):
    w = wl.kepler_ensemble(batch=B, nsteps=ns)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, energy_every=20) as ig:
        Y = torch.tensor(w.y, dtype=torch.float64, device="cuda"); ws = ig.new_workspace()
        E = torch.zeros((ig.n_energy(), B), dtype=torch.float64, device="cuda"); it = torch.zeros(B, dtype=torch.int64, device="cuda")
        ig.integrate(Y, ws, energy=E, iters=it); torch.cuda.synchronize()
        rc, st = ig.stats(ws)
        idx = np.r_[0, np.arange(1, B, B // 97), B - 1]
        o = oracle.integrate(w.problem, np.ascontiguousarray(w.y[:, idx]), w.params, w.h, w.nsteps, energy_every=20)
        print(B, rc, np.array_equal(Y.cpu().numpy()[:, idx], o["y"]), np.array_equal(E.cpu().numpy()[:, idx], o["energy"]),
              np.array_equal(it.cpu().numpy()[idx], o["iters"]), st["total_sweeps"])
