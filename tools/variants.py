"""A/B timing of library build variants (-D flags) on config 2 (one call each)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

_VF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants_current.json")
VARIANTS = json.loads(os.environ.get("IRK_VARIANTS") or (open(_VF).read() if os.path.exists(_VF) else "{}"))


def build_all():
    import shutil
    from paper_2511_03655_b200 import build
    shutil.rmtree(os.path.join(ROOT, "paper_2511_03655_b200", "lib", "variants"), ignore_errors=True)
    for name, defs in VARIANTS.items():
        out = os.path.join(ROOT, "paper_2511_03655_b200", "lib", "variants", f"libirk_{name}.so")
        build.build(force=True, out=out, defines=tuple(defs))
        log = open(out + ".ptxas.log").read()
        import re
        for kern in ("ens_g1_kernelINS_6Kepler", "ens_nbody_kernelILi6", "ens_chain_kernelILi2"):
            m = re.search(r"Compiling entry function '_ZN3irk\d+" + kern + r".*?\n.*?\n(.*?)\n(.*?)\n", log, re.S)
            if m:
                print(name, kern, m.group(1).strip(), "|", m.group(2).strip()[:60])


CFG = int(os.environ.get("IRK_VARIANT_CONFIG", "2"))
NSTEPS = int(os.environ.get("IRK_VARIANT_NSTEPS", "0"))
SCHED = int(os.environ.get("IRK_VARIANT_SCHEDULE", "0"))
MAPPING = int(os.environ.get("IRK_VARIANT_MAPPING", "0"))


def time_one(name):
    lib = os.path.join(ROOT, "paper_2511_03655_b200", "lib", "variants", f"libirk_{name}.so")
    code = f"""
import os, sys, torch
os.environ['IRK_LIB_OVERRIDE'] = {lib!r}
sys.path.insert(0, {ROOT!r})
from paper_2511_03655_b200 import irk, workloads as wl
w = wl.config({CFG}, **({{'nsteps': {NSTEPS}}} if {NSTEPS} else {{}}))
ig = irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, schedule={SCHED}, mapping={MAPPING})
y0 = torch.tensor(w.y, device='cuda'); Y = torch.empty_like(y0); ws = ig.new_workspace()
ts = []
for r in range(4):
    Y.copy_(y0); ws.zero_(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); ig.integrate(Y, ws); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print({name!r}, 'sched', {SCHED}, 'ms', min(ts[1:]), ts)
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-500:])


if __name__ == "__main__":
    if sys.argv[1] == "build":
        if os.environ.get("IRK_VARIANTS"):
            open(_VF, "w").write(os.environ["IRK_VARIANTS"])
        build_all()
    else:
        for n in VARIANTS:
            time_one(n)
