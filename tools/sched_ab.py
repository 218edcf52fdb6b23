"""A/B of the ensemble schedules (IRK_OPT_SCHEDULE / BALANCE) on one config:
time per call (CUDA events, best of 3 after a warm-up) and bitwise agreement of
state, sweeps and stats across all variants."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
variants = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [[1, -1], [2, -1], [2, 157], [2, 625], [2, 1250]]
w = wl.config(cfg)
ref = None
for sched, bal in variants:
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, schedule=sched, balance=bal) as ig:
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(y0)
        ws = ig.new_workspace()
        it = torch.zeros(w.batch, dtype=torch.int64, device="cuda")
        ts = []
        for r in range(4):
            Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); ig.integrate(Y, ws, iters=it); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        rc, st = ig.stats(ws)
        out = (Y.cpu(), it.cpu())
    same = None
    if ref is None:
        ref = out
    else:
        same = bool(torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1]))
    print(json.dumps({"config": cfg, "schedule": sched, "balance": bal, "ms": min(ts[1:]), "all_ms": ts,
                      "rc": rc, "stats": list(st), "bitwise_vs_first": same}), flush=True)
