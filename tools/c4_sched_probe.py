import sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_2511_03655_b200 import irk, workloads as wl
w = wl.config(4, nsteps=20000)
for B in (1024, 1536, 2048, 3072):
    y = w.y[:, :B].copy()
    for sched, bal in ((0, -1), (2, 2500), (2, 1250), (2, 312), (1, -1)):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, B, w.params, schedule=sched, balance=bal) as ig:
            y0 = torch.tensor(y, dtype=torch.float64, device="cuda"); Y = torch.empty_like(y0); ws = ig.new_workspace()
            ts = []
            for r in range(3):
                Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); ig.integrate(Y, ws); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
        print(json.dumps(dict(B=B, sched=sched, bal=bal, ms=min(ts[1:]))), flush=True)
