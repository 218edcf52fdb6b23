"""Config 5 (one Plummer system) body-sharded over P GPUs: all-gather vs fused exchange.

torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/cfg5_multi.py [--N 8192] [--nsteps 50]

Each rank integrates its N/P bodies (irk_set_comm), once with IRK_OPT_EXCHANGE = 0
(in-place ncclAllGather per sweep) and once with 1 (NVLink stores into symmetric
windows, NEXT f3).  Reports the device time (CUDA events, max over ranks) per
variant and checks that both assembled end states are bitwise equal to each
other; with --check also to a 1-process run on rank 0's GPU.  Runs at P = 1 too
(the only size this repo's round-1 box has), where it is a smoke test.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2511_03655_b200 import irk, parallel, workloads as wl  # noqa: E402


def run(w, rank, world, exchange, reps, uid):
    with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params, exchange=exchange) as ig:
        ig.set_comm(uid, rank, world)
        y0 = torch.tensor(parallel.shard_rows(w.y, rank, world), dtype=torch.float64, device="cuda")
        Y = torch.empty_like(y0)
        it = torch.zeros(1, dtype=torch.int64, device="cuda")
        best = float("inf")
        for _ in range(reps + 1):
            Y.copy_(y0)
            ws = ig.new_workspace()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ig.integrate(Y, ws, iters=it)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, parallel.max_over_ranks(e0.elapsed_time(e1), device="cuda"))
        return best, int(it.item()), Y.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=8192)
    ap.add_argument("--nsteps", type=int, default=50)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--check", action="store_true", help="also compare with a 1-process run on rank 0")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    w = wl.plummer(N=a.N, nsteps=a.nsteps)
    out = {}
    finals = []
    for ex in (0, 1):
        uid = parallel.nccl_bootstrap(rank)
        ms, sweeps, y = run(w, rank, world, ex, a.reps, uid)
        parts = [None] * world
        dist.all_gather_object(parts, y)
        finals.append(parallel.assemble_rows(parts))
        out[f"exchange{ex}"] = dict(ms=ms, sweeps=sweeps, us_per_sweep=1e3 * ms / sweeps)
    same = bool(np.array_equal(finals[0], finals[1]))
    if a.check and rank == 0:
        with irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params) as ig:
            Y = torch.tensor(w.y, dtype=torch.float64, device="cuda")
            ig.integrate(Y, ig.new_workspace())
            same = same and bool(np.array_equal(Y.cpu().numpy(), finals[0]))
    if rank == 0:
        print(json.dumps(dict(N=a.N, nsteps=a.nsteps, ranks=world, bitwise_equal=same, **out)), flush=True)
    dist.destroy_process_group()
    if not same:
        sys.exit(1)


if __name__ == "__main__":
    main()
