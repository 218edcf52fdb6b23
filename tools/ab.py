"""A/B timing of library builds on the GPU: each build in its own process
(IRK_LIB_OVERRIDE), interleaved repetitions, one full irk_integrate call per
repetition (state reset and L2 flush outside the events), and a digest of the
final state so that every build must give the same bits.

python tools/ab.py --libs base=lib/variants/libirk_base.so,new=lib/libirk.so[@mapping] \
                   --configs 2,3:5000,5:100 [--reps 3] [--out gpurun_out/ab.json]
A config is `i`, `i:nsteps` or `i:nsteps:batch`.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, json, os, sys, torch
sys.path.insert(0, {root!r})
from paper_2511_03655_b200 import irk, workloads as wl
kw = {{}}
if {nsteps}: kw['nsteps'] = {nsteps}
if {batch}: kw['batch'] = {batch}
w = wl.config({cfg}, **kw)
ig = irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mapping=int(os.environ.get('IRK_AB_MAPPING', '0')))
y0 = torch.tensor(w.y, dtype=torch.float64, device='cuda'); Y = torch.empty_like(y0)
ws = ig.new_workspace(); it = torch.zeros(w.batch, dtype=torch.int64, device='cuda')
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
ts = []
for r in range({calls}):
    Y.copy_(y0); ws.zero_(); flush.fill_(1.0); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); ig.integrate(Y, ws, iters=it); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
dig = hashlib.sha1(Y.cpu().numpy().tobytes() + it.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps(dict(ms=ts[1:], digest=dig, sweeps=int(it.sum().item()),
                      mapping=ig.get_option(irk.INFO_MAPPING_USED))))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--configs", default="2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--calls", type=int, default=3, help="calls per process (the first is a warm-up)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    libs = dict(x.split("=", 1) for x in a.libs.split(","))
    res = {}
    for cs in a.configs.split(","):
        cfg, _, rest = cs.partition(":")
        ns, _, bt = rest.partition(":")
        key = f"config{cfg}" + (f"_n{ns}" if ns else "") + (f"_b{bt}" if bt else "")
        res[key] = {n: {"ms": []} for n in libs}
        for rep in range(a.reps):
            order = list(libs) if rep % 2 == 0 else list(libs)[::-1]
            for n in order:
                libpath, _, mp = libs[n].partition("@")   # name=path[@mapping]
                env = dict(os.environ, IRK_AB_MAPPING=mp or "0", IRK_LIB_OVERRIDE=os.path.abspath(os.path.join(ROOT, libpath)
                                                                        if not os.path.isabs(libpath) else libpath))
                code = CHILD.format(root=ROOT, cfg=int(cfg), nsteps=int(ns or 0), batch=int(bt or 0), calls=a.calls)
                p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
                if p.returncode:
                    res[key][n]["error"] = p.stderr[-400:]
                    continue
                d = json.loads(p.stdout.strip().splitlines()[-1])
                res[key][n]["ms"] += d["ms"]
                res[key][n].update(digest=d["digest"], sweeps=d["sweeps"], mapping=d["mapping"])
        for n in libs:
            if res[key][n]["ms"]:
                res[key][n]["best_ms"] = min(res[key][n]["ms"])
        digs = {res[key][n].get("digest") for n in libs}
        res[key]["bitwise_equal"] = len(digs) == 1 and None not in digs
        print(key, json.dumps({n: (res[key][n].get("best_ms"), res[key][n].get("digest")) for n in libs}),
              "equal" if res[key]["bitwise_equal"] else "DIFFER", flush=True)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
