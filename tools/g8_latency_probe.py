"""Config 1 (one Kepler trajectory, g8) and small g8/g4 batches for library
variants (tools/variants.py build): python tools/g8_latency_probe.py name..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r"""
import json, sys, torch
sys.path.insert(0, {root!r})
from paper_2511_03655_b200 import irk, workloads as wl
for B, steps in ((1, 12800), (2048, 2000), (12288, 2000)):
    w = wl.kepler_single() if B == 1 else wl.kepler_ensemble(batch=B, nsteps=steps)
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params) as ig:
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda"); Y = torch.empty_like(y0); ws = ig.new_workspace()
        ts = []
        for _ in range(4):
            Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); ig.integrate(Y, ws); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(json.dumps(dict(lib={name!r}, batch=B, nsteps=w.nsteps, ms=round(min(ts[1:]), 3))), flush=True)
"""
for name in sys.argv[1:]:
    env = dict(os.environ, IRK_LIB_OVERRIDE=os.path.join(ROOT, "paper_2511_03655_b200", "lib", "variants", f"libirk_{name}.so"))
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT, name=name)], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-600:], flush=True)
