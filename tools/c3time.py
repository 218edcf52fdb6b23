"""Config-3 timing stability: several reps per schedule with nvidia-smi clock samples."""
import json
import subprocess
import sys
import tempfile

import torch

sys.path.insert(0, '/root/repo')
from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

w = wl.six_body_ensemble()
f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active,temperature.gpu",
                      "--format=csv,noheader,nounits", "-lms", "100"], stdout=f)
for sched, bal in ((2, -1), (2, 781), (2, 390), (2, 3125), (1, -1)):
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, schedule=sched, balance=bal) as ig:
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda"); Y = torch.empty_like(y0)
        ws = ig.new_workspace()
        ts = []
        for r in range(5):
            Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ig.integrate(Y, ws); e1.record(); torch.cuda.synchronize()
            ts.append(round(e0.elapsed_time(e1), 1))
        print(json.dumps({"schedule": sched, "balance": bal, "ms": ts}), flush=True)
p.terminate(); p.wait()
rows = [l.strip().split(",") for l in open(f.name) if l.strip()]
clk = [float(r[0]) for r in rows]; pw = [float(r[1]) for r in rows]
print("sm clock min/median/max", min(clk), sorted(clk)[len(clk) // 2], max(clk), "power max", max(pw))
print("reasons seen:", sorted(set(r[2].strip() for r in rows)), "temp max", max(float(r[3]) for r in rows))
