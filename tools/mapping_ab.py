"""g1 vs g2 vs g4 vs g8 mapping (IRK_OPT_MAPPING) across batch sizes on the config-2
generator: time per call (CUDA events, best of 3 after a warm-up) and bitwise
agreement of the mappings.  python tools/mapping_ab.py [nsteps] [lib...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NSTEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
LIBS = sys.argv[2:] or [""]
CODE = r"""
import json, os, sys, torch
sys.path.insert(0, {root!r})
from paper_2511_03655_b200 import irk, workloads as wl
res = []
for B in (512, 2048, 4096, 8192, 12288, 16384, 24576, 32768, 65536):
    w = wl.kepler_ensemble(batch=B, nsteps={nsteps})
    outs, ms = [], []
    for mp in (1, 2, 4, 8):
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mapping=mp) as ig:
            y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda"); Y = torch.empty_like(y0)
            ws = ig.new_workspace(); it = torch.zeros(B, dtype=torch.int64, device="cuda")
            ts = []
            for r in range(4):
                Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); ig.integrate(Y, ws, iters=it); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            outs.append((Y.cpu(), it.cpu())); ms.append(min(ts[1:]))
    same = all(bool(torch.equal(outs[0][0], o[0]) and torch.equal(outs[0][1], o[1])) for o in outs[1:])
    print(json.dumps({{"lib": os.environ.get("IRK_LIB_OVERRIDE", "default")[-24:], "batch": B, "nsteps": {nsteps},
                      "g1_ms": ms[0], "g2_ms": ms[1], "g4_ms": ms[2], "g8_ms": ms[3], "bitwise": same}}), flush=True)
"""
for lib in LIBS:
    env = dict(os.environ)
    if lib:
        env["IRK_LIB_OVERRIDE"] = lib
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT, nsteps=NSTEPS)], env=env,
                       capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-800:], flush=True)
