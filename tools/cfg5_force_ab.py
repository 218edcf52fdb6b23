"""A/B of config-5 force-kernel build variants (lib/variants/libirk_<name>.so), interleaved,
with a bitwise digest of the final state (usage: python tools/cfg5_force_ab.py NSTEPS name...)."""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NSTEPS = int(sys.argv[1])
CODE = """
import os, sys, hashlib, torch
os.environ['IRK_LIB_OVERRIDE'] = {lib!r}
sys.path.insert(0, {root!r})
from paper_2511_03655_b200 import irk, workloads as wl
w = wl.config(5, nsteps={n})
ig = irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params)
y0 = torch.tensor(w.y, device='cuda'); Y = torch.empty_like(y0); ws = ig.new_workspace()
ts = []
for r in range(3):
    Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); ig.integrate(Y, ws); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print({name!r}, 'ms', round(min(ts[1:]), 2), [round(t, 2) for t in ts], hashlib.sha1(Y.cpu().numpy().tobytes()).hexdigest()[:16])
"""
for rep in range(2):
    for name in sys.argv[2:]:
        lib = os.path.join(ROOT, "paper_2511_03655_b200", "lib", "variants", f"libirk_{name}.so")
        r = subprocess.run([sys.executable, "-c", CODE.format(lib=lib, root=ROOT, n=NSTEPS, name=name)],
                           capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-500:], flush=True)
