import sys, torch, json, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2511_03655_b200 import irk, workloads as wl
w1 = wl.six_body_ensemble(batch=1, nsteps=1000)
w16 = wl.six_body_ensemble(batch=16, nsteps=1000)
print("B=1 y:", np.array2string(w1.y[:, 0], precision=3, max_line_width=200))
def run(y, mp):
    with irk.Integrator(w1.problem, w1.dim, w1.h, 1000, y.shape[1], w1.params, mapping=mp) as ig:
        y0 = torch.tensor(y, dtype=torch.float64, device="cuda"); Y = torch.empty_like(y0); ws = ig.new_workspace()
        it = torch.zeros(y.shape[1], dtype=torch.int64, device="cuda"); ts = []
        for _ in range(3):
            Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); ig.integrate(Y, ws, iters=it); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        return min(ts[1:]), int(it.sum().item())
for name, y in (("B1", w1.y), ("B16m0", w16.y[:, :1].copy()), ("B16m5", w16.y[:, 5:6].copy()), ("B16", w16.y)):
    for mp in (8, 1):
        t, sw = run(y, mp)
        print(json.dumps(dict(case=name, mapping=mp, ms=round(t, 2), sweeps=sw)))
