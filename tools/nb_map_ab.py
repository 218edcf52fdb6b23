"""N-body ensembles, every supported N: body-per-lane (IRK_OPT_MAPPING = 1) vs
stage-per-lane (8) vs stage-per-lane with DMMA contractions (9) -- time per call
(CUDA events, best of 3) and bitwise agreement.  N = 6 uses the config-3 generator; other N seeded random softened
systems (as tests/test_gpu_parity.py::test_nbody_small_n_variants).

python tools/nb_map_ab.py [--nsteps 1000] [--batches 2048,16384] [--ns 2,3,4,5,6,8] [--out f.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_03655_b200 import irk, workloads as wl  # noqa: E402


def system(N, B, nsteps):
    if N == 6:
        return wl.six_body_ensemble(batch=B, nsteps=nsteps)
    rng = np.random.default_rng(100 + N)
    q = rng.standard_normal((3 * N, B))
    v = 0.3 * rng.standard_normal((3 * N, B))
    params = np.concatenate([[1.0, 0.05], rng.uniform(0.2, 1.0, N)])
    return wl.Workload(f"nb{N}", wl.NBODY, 6 * N, np.concatenate([q, v]), params, 0.01, nsteps)


def run(w, mapping):
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, w.batch, w.params, mapping=mapping) as ig:
        y0 = torch.tensor(w.y, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(y0)
        ts = []
        for _ in range(4):
            Y.copy_(y0)
            ws = ig.new_workspace()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ig.integrate(Y, ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts[1:]), Y.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nsteps", type=int, default=1000)
    ap.add_argument("--batches", default="2048,16384")
    ap.add_argument("--ns", default="2,3,4,5,6,8")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = []
    for N in [int(x) for x in a.ns.split(",")]:
        for B in [int(x) for x in a.batches.split(",")]:
            w = system(N, B, a.nsteps)
            t1, y1 = run(w, irk.MAP_G1)
            t8, y8 = run(w, irk.MAP_G8)
            t9, y9 = run(w, irk.MAP_G8M)
            r = dict(N=N, batch=B, nsteps=a.nsteps, body_per_lane_ms=t1, stage_per_lane_ms=t8, dmma_ms=t9,
                     bitwise_equal=bool(np.array_equal(y1, y8, equal_nan=True)),
                     dmma_bitwise_equal=bool(np.array_equal(y1, y9, equal_nan=True)))
            print(json.dumps(r), flush=True)
            res.append(r)
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
