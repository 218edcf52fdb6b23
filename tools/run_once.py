"""Run one irk_integrate of a config (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--nsteps", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--host-loop", action="store_true", help="config 5: host-driven sweep loop (ncu sees each kernel)")
ap.add_argument("--comm", action="store_true", help="config 5: 1-rank NCCL communicator")
ap.add_argument("--exchange", type=int, default=0, help="config 5 with --comm: IRK_OPT_EXCHANGE")
ap.add_argument("--mapping", type=int, default=0, help="IRK_OPT_MAPPING (0 auto, 1 g1 / body per lane, 8 stage per lane)")
a = ap.parse_args()
kw = {}
if a.batch:
    kw["batch"] = a.batch
if a.nsteps:
    kw["nsteps"] = a.nsteps
w = wl.config(a.config, **kw)
kw2 = {"device_loop": 0} if (a.host_loop and w.problem == wl.NBODY_DIRECT) else {}
if a.exchange:
    kw2["exchange"] = a.exchange
if a.mapping:
    kw2["mapping"] = a.mapping
with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, **kw2) as ig:
    if a.comm:
        ig.set_comm(irk.nccl_unique_id(), 0, 1)
    y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
    for _ in range(a.reps):
        ws = ig.new_workspace()
        ig.integrate(y, ws)
    torch.cuda.synchronize()
    print("rc", ig.stats(ws))
