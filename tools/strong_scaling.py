"""Strong scaling of the ensemble configs from single-GPU shard measurements.

The ensembles shard by trajectory with no communication,
so P GPUs take max over ranks of one GPU's time on its shard
(parallel.batch_slice).  For P = 1, 2, 4, 8 every shard of each config is timed
on one B200 with the default (auto) mapping; the projected strong-scaling
efficiency is T(B) / (P max_r T(shard_r)).  bench.py --gpus P measures the same
thing on P GPUs (max over ranks, device clocks).

python tools/strong_scaling.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, parallel, workloads as wl  # noqa: E402


def time_call(w, y):
    B = y.shape[1]
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, B, w.params) as ig:
        y0 = torch.tensor(y, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(y0)
        ws = ig.new_workspace()
        ts = []
        for _ in range(2):
            Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); ig.integrate(Y, ws); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return ts[-1], ig.get_option(irk.INFO_MAPPING_USED)


res = []
for cfg, nsteps in ((2, 10000), (3, 10000), (4, 20000)):
    w = wl.config(cfg, nsteps=nsteps)
    t1 = None
    for P in (1, 2, 4, 8):
        shard_ms, maps = [], set()
        for r in range(P):
            sl = parallel.batch_slice(w.batch, r, P)
            t, m = time_call(w, w.y[:, sl].copy())
            shard_ms.append(t)
            maps.add(m)
        t = max(shard_ms)
        t1 = t if P == 1 else t1
        r = {"config": cfg, "nsteps": nsteps, "P": P, "batch_per_gpu": w.batch // P, "ms": t,
             "shard_ms": shard_ms, "mapping_used": sorted(maps),
             "efficiency": t1 / (P * t), "traj_steps_per_s_total": w.batch * nsteps / (t * 1e-3)}
        print(json.dumps(r), flush=True)
        res.append(r)
if len(sys.argv) > 1:
    json.dump(res, open(sys.argv[1], "w"), indent=1)
