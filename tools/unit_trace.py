"""Work-unit timeline of the persistent work-queue kernel (config 2, ens_g1q).

Builds libirk with -DIRK_TRACE into lib/variants/, runs one full config-2 call
with a device trace buffer, and summarises where lane time goes:
  * busy / waiting / idle lane-time fractions over the whole launch,
  * active lanes per 2 % time bin (the tail),
  * the critical chains: trajectories whose last unit ends last, with their
    total sweeps relative to the mean.
python tools/unit_trace.py [--build-only] [--out gpurun_out/unit_trace.json]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "paper_2511_03655_b200", "lib", "variants", "libirk_trace.so")


def build():
    from paper_2511_03655_b200 import build as b
    b.build(force=True, out=VAR, defines=("IRK_TRACE",))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build-only", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "unit_trace.json"))
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--nsteps", type=int, default=10000)
    a = ap.parse_args()
    if a.build_only or not os.path.exists(VAR):
        build()
        if a.build_only:
            return
    os.environ["IRK_LIB_OVERRIDE"] = VAR
    import numpy as np
    import torch
    from paper_2511_03655_b200 import irk, workloads as wl
    L = irk.lib()
    L.irk_trace_set.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    w = wl.kepler_ensemble(batch=a.batch, nsteps=a.nsteps)
    cap = w.batch * 64
    buf = torch.zeros(cap * 6, dtype=torch.int64, device="cuda")
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params) as ig:
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        for rep in range(2):   # warm-up call, then the traced call
            Y = y0.clone()
            ws = ig.new_workspace()
            assert L.irk_trace_set(ctypes.c_void_p(buf.data_ptr()), cap) == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ig.integrate(Y, ws)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    r = buf.view(-1, 6).cpu().numpy()
    r = r[r[:, 4] != 0]
    c = r[:, 0] >> 32
    b = r[:, 0] & 0xffffffff
    tf, ts, te, sw = r[:, 2], r[:, 3], r[:, 4], r[:, 5]
    t0 = tf.min()
    T = te.max() - t0
    lanes = int(len(np.unique(r[:, 1])))   # distinct (SM, block, thread) slots that ran units
    busy = (te - ts).sum() / (lanes * T)
    wait = (ts - tf).sum() / (lanes * T)
    bins = 50
    edges = np.linspace(0, T, bins + 1)
    act = np.zeros(bins)
    for i in range(bins):
        lo, hi = edges[i] + t0, edges[i + 1] + t0
        act[i] = (np.clip(np.minimum(te, hi) - np.maximum(ts, lo), 0, None)).sum() / (hi - lo)
    tot = np.bincount(b, weights=sw, minlength=w.batch)
    endb = np.zeros(w.batch, dtype=np.int64)
    np.maximum.at(endb, b, te - t0)
    order = np.argsort(-endb)[:20]
    unit_ns = (te - ts) / np.maximum(sw, 1)
    out = {"ms_call": ms, "trace_span_ms": T / 1e6, "units": int(len(r)), "busy_frac": float(busy),
           "wait_frac": float(wait), "idle_frac": float(1 - busy - wait),
           "active_lanes_per_bin": [float(x) for x in act], "lanes": lanes,
           "mean_sweeps_per_traj": float(tot.mean()), "max_sweeps_per_traj": float(tot.max()),
           "last_finishers": [{"b": int(x), "end_ms": float(endb[x] / 1e6), "sweeps_rel": float(tot[x] / tot.mean())}
                              for x in order],
           "ns_per_sweep_median": float(np.median(unit_ns)),
           "ns_per_sweep_p10_p90": [float(np.percentile(unit_ns, 10)), float(np.percentile(unit_ns, 90))]}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "active_lanes_per_bin"}, indent=1))
    print("active lanes per 2% bin:", " ".join(f"{x / lanes:.2f}" for x in act))


if __name__ == "__main__":
    main()
