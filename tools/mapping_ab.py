"""Per-thread-problem mappings (IRK_OPT_MAPPING 1 / 2 / 4 / 8 / 9) across batch sizes
on the config-2 generator (batch 1 = config 1): time per call (CUDA events, best of
3 after a warm-up) and bitwise agreement of the mappings.

python tools/mapping_ab.py [--nsteps N] [--batches 1,512,...] [--maps 1,4,8,9] [--lib path ...]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--nsteps", type=int, default=2000)
ap.add_argument("--batches", default="512,2048,4096,8192,12288,16384,24576,32768,65536")
ap.add_argument("--maps", default="1,2,4,8")
ap.add_argument("--lib", nargs="*", default=[""])
args = ap.parse_args()
CODE = r"""
import json, os, sys, torch
sys.path.insert(0, {root!r})
from paper_2511_03655_b200 import irk, workloads as wl
for B in {batches}:
    w = wl.kepler_single() if B == 1 else wl.kepler_ensemble(batch=B, nsteps={nsteps})
    outs, ms = [], {{}}
    for mp in {maps}:
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mapping=mp) as ig:
            y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda"); Y = torch.empty_like(y0)
            ws = ig.new_workspace(); it = torch.zeros(B, dtype=torch.int64, device="cuda")
            ts = []
            for r in range(4):
                Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); ig.integrate(Y, ws, iters=it); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            outs.append((Y.cpu(), it.cpu())); ms["g%d_ms" % mp] = round(min(ts[1:]), 3)
    same = all(bool(torch.equal(outs[0][0], o[0]) and torch.equal(outs[0][1], o[1])) for o in outs[1:])
    print(json.dumps(dict(lib=os.environ.get("IRK_LIB_OVERRIDE", "default")[-24:], batch=B, nsteps=w.nsteps,
                          bitwise=same, **ms)), flush=True)
"""
batches = [int(x) for x in args.batches.split(",")]
maps = [int(x) for x in args.maps.split(",")]
for lib in args.lib:
    env = dict(os.environ)
    if lib:
        env["IRK_LIB_OVERRIDE"] = lib
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT, nsteps=args.nsteps, batches=batches, maps=maps)],
                       env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-800:], flush=True)
