"""Config 5 (IRK_NBODY_DIRECT) on one GPU: the exchange variants side by side.

  none       no communicator (one process owns every body; nothing to exchange)
  allgather  1-rank NCCL communicator, in-place ncclAllGather per sweep (default)
  fused      1-rank NCCL communicator, IRK_OPT_EXCHANGE = 1 (peer-pointer stores
             into a symmetric window + arrival/wait barrier, NEXT f3)

At one rank the exchange moves no data between GPUs, so this measures the fixed
per-sweep cost each variant adds (NCCL kernel launch and its proxy vs the fused
barrier), device-timed with CUDA events, and checks the three agree bit for bit.

python tools/exchange_ab.py [--N 8192] [--nsteps 100] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402


def run(w, variant, reps, device_loop):
    kw = dict(device_loop=device_loop)
    if variant == "fused":
        kw["exchange"] = 1
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params, **kw) as ig:
        if variant != "none":
            ig.set_comm(irk.nccl_unique_id(), 0, 1)
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(y0)
        it = torch.zeros(1, dtype=torch.int64, device="cuda")
        ts = []
        for _ in range(reps + 1):
            Y.copy_(y0)
            ws = ig.new_workspace()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ig.integrate(Y, ws, iters=it)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        sweeps = int(it.item())
        return dict(variant=variant, device_loop=device_loop, ms=min(ts[1:]), sweeps=sweeps,
                    us_per_sweep=1e3 * min(ts[1:]) / sweeps,
                    loop=ig.get_option(irk.INFO_DEVICE_LOOP_USED)), Y.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=8192)
    ap.add_argument("--nsteps", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    w = wl.plummer(N=a.N, nsteps=a.nsteps)
    res, ys = [], []
    for dl in (1, 0):
        for v in ("none", "allgather", "fused"):
            r, y = run(w, v, a.reps, dl)
            r["N"], r["nsteps"] = a.N, a.nsteps
            print(json.dumps(r), flush=True)
            res.append(r)
            ys.append(y)
    same = all(np.array_equal(ys[0], y) for y in ys[1:])
    print(json.dumps({"bitwise_equal": same}))
    if a.out:
        json.dump(dict(runs=res, bitwise_equal=same), open(a.out, "w"), indent=1)
    if not same:
        sys.exit(1)


if __name__ == "__main__":
    main()
