#!/usr/bin/env python
"""IRKGL16 fp64 benchmark (BASELINE.json metric: trajectory-steps/s).

One bench "step" = one irk_integrate call over the whole workload: config 2,
the Kepler ensemble of 65,536 trajectories x 10,000 IRKGL16 steps, all hot-path
rows (nu-init, position sweep, stop test, 8 RHS, velocity sweep, update)
inside the timed region, inputs resident in HBM.  L2 is flushed (256 MiB
write) before every timed step; state and workspace are reset from a pristine
device copy outside the timed region.

Multi-GPU: `torchrun --nproc-per-node N bench.py --gpus N`; every rank
integrates its own 65,536-trajectory ensemble (seed + rank) with no
collective on the data path (weak scaling); time = max over ranks.

--impl reference: the scalar-C oracle (oracle/) on the host cores, each step a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IRKGL16 fp64 trajectory-steps/s"
UNIT = "traj-steps/s"
SM_COUNT = 148
FP64_FMA_PER_CLK_PER_SM = 64  # B200 (sm_100a) non-tensor FP64 rate


def flops_per_traj(d: int, f_flops: int, steps: int, sweeps: int) -> int:
    """Algorithmic flops: per step 128d (nu-init) +
    16d (update); per sweep 136d (a2) + 8d (Delta) + 8 f (a3) + 136d (a4)."""
    return steps * 144 * d + sweeps * (280 * d + 8 * f_flops)


KEPLER_F_FLOPS = 8  # fma(2) + mul + sqrt + mul + div + 2 mul


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = [l.split(",") for l in open(self.f.name).read().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except ValueError:
                continue
            for n, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def probe_fp64(torch, irk, dev):
    out = torch.empty(SM_COUNT * 8 * 256, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev)
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fl = irk.probe_dfma(out, SM_COUNT * 8, 8192, s)
        e1.record(s)
        torch.cuda.synchronize(dev)
        best = max(best, fl / (e0.elapsed_time(e1) * 1e-3))
    return best


def cpu_baseline(w, target_s: float = 15.0):
    """The oracle as it stands, on all host cores, over a bounded sample of the
    workload: the first S trajectories of the config-2 batch for the full
    10,000 steps, S calibrated to ~target_s seconds."""
    from oracle import oracle
    import numpy as np
    cores = os.cpu_count() or 1
    t = time.perf_counter()
    oracle.integrate(w.problem, w.y[:, :8], w.params, w.h, 1000, nthreads=1)
    rate1 = 8 * 1000 / (time.perf_counter() - t)
    S = int(min(w.batch, max(cores, rate1 * cores * 0.8 * target_s / w.nsteps)))
    S = max(cores, (S // cores) * cores)
    t = time.perf_counter()
    oracle.integrate(w.problem, np.ascontiguousarray(w.y[:, :S]), w.params, w.h, w.nsteps, nthreads=cores)
    dt = time.perf_counter() - t
    cpu_model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu_model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": S * w.nsteps / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "value_1core": rate1, "cpu_model": cpu_model,
            "sample": f"first {S} of {w.batch} config-2 trajectories x {w.nsteps} steps "
                      f"({dt:.1f} s, OpenMP over trajectories; value_1core from 8 x 1,000 steps on one core)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2511_03655_b200 import workloads as wl
    from oracle import oracle
    import numpy as np
    w = wl.kepler_ensemble()
    cores = os.cpu_count() or 1
    S = cores * 48  # ~1 s of oracle work per step on the GPU box's host
    ysub = np.ascontiguousarray(w.y[:, :S])
    for _ in range(args.warmup):
        oracle.integrate(w.problem, ysub, w.params, w.h, 500, nthreads=cores)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle.integrate(w.problem, ysub, w.params, w.h, w.nsteps, nthreads=cores)
        times.append(time.perf_counter() - t)
    T = sum(times)
    value = S * w.nsteps * args.steps / T
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "config2_kepler_ensemble", "batch_per_gpu": w.batch, "nsteps": w.nsteps,
                       "h": w.h, "seed": wl.SEEDS[2]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"first {S} of {w.batch} config-2 trajectories x {w.nsteps} steps per step "
                                       "(the oracle as it stands, OpenMP over trajectories)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_03655_b200 import irk, workloads as wl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    w = wl.kepler_ensemble(seed=wl.SEEDS[2] + rank)
    B, D = w.batch, w.dim
    ig = irk.Integrator(w.problem, D, w.h, w.nsteps, B, w.params)
    y0 = torch.tensor(w.y, dtype=torch.float64, device=dev)
    Y = torch.empty_like(y0)
    ws = ig.new_workspace(dev)
    iters = torch.zeros(B, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream(dev)

    def step():
        Y.copy_(y0)
        ws.zero_()
        flush.fill_(1.0)  # 256 MiB write: evicts the 126 MB L2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ig.integrate(Y, ws, iters=iters, stream=s)
        e1.record(s)
        return e0, e1

    warm = max(3, args.warmup)  # the contract's minimum of 3 warm-up steps
    for _ in range(warm):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = Clocks(local)
    clk.start()
    evs = [step() for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    times = [a.elapsed_time(b) * 1e-3 for a, b in evs]
    T = sum(times)
    sweeps = int(iters.sum().item())
    rc, st = ig.stats(ws)
    if world > 1:
        t = torch.tensor([T], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        T = float(t.item())
    value = world * B * w.nsteps * args.steps / T

    # end to end through the C ABI from pinned host memory (H2D + kernel + D2H timed)
    yh_pin = torch.empty((D, B), dtype=torch.float64, pin_memory=True)
    yh = yh_pin.numpy()
    e2e_t = []
    for i in range(args.warmup + args.steps):
        yh[...] = w.y
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(1.0)
        e0.record(s)
        ig.integrate_host(yh, want_energy=False, want_iters=True, stream=s)
        e1.record(s)
        torch.cuda.synchronize(dev)
        if i >= args.warmup:
            e2e_t.append(e0.elapsed_time(e1) * 1e-3)
    assert np.array_equal(yh, Y.cpu().numpy()), "e2e result differs from the device-resident run"
    Te = sum(e2e_t)
    if world > 1:
        t = torch.tensor([Te], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        Te = float(t.item())

    # our kernels per irk_integrate call: one persistent ens_g1q launch + advance_n
    # (the two cudaMemsetAsync that reset the work queue are runtime copies, not our kernels)
    launches_per_step = 2
    line = None
    if rank == 0:
        fl = flops_per_traj(w.dim // 2, KEPLER_F_FLOPS, w.nsteps * B, sweeps)
        t_launch = T / args.steps if world == 1 else statistics.mean(times)
        achieved = fl / statistics.mean(times) / 1e12
        mp_ = measured_peaks()
        sm_max = float(mp_.get("sm_max_mhz", 1965.0))
        peak = SM_COUNT * FP64_FMA_PER_CLK_PER_SM * 2 * sm_max * 1e6 / 1e12
        probe = probe_fp64(torch, irk, dev) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get("config2_kepler_ensemble_g1q")  # bytes per launch
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": warm, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded config-2 generator, workloads.py)",
            "config": {"workload": "config2_kepler_ensemble", "batch_per_gpu": B, "nsteps": w.nsteps,
                       "h": w.h, "seed": wl.SEEDS[2], "mapping": "g1 (1 trajectory/thread)",
                       "schedule": "one persistent launch, lanes pull (trajectory, nsteps/32-step) units "
                                   "from a work queue (IRK_OPT_SCHEDULE auto)",
                       "l2": "flushed (256 MiB write) before every timed step",
                       "parallelism": f"trajectory-sharded x{world}, no collective"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per ens_g1q launch (ncu --set full, profiles/r1)",
                         "peak_note": f"FP64 pipe: {SM_COUNT} SM x {FP64_FMA_PER_CLK_PER_SM} FMA/clk x 2 x {sm_max:.0f} MHz; "
                                      f"DFMA probe measured {probe:.2f} TFLOP/s on this GPU",
                         "kernel": "ens_g1q_kernel<KeplerT<true>> (GM = 1: reciprocal form of the division)",
                         "timed": "CUDA events around irk_integrate: 1 ens_g1q launch (+2 memsets, advance_n)", "flops_per_launch": fl,
                         "sweeps_per_step": sweeps / (B * w.nsteps)},
            "e2e": {"value": world * B * w.nsteps * args.steps / Te, "unit": UNIT,
                    "h2d_bytes_per_step": D * B * 8, "d2h_bytes_per_step": D * B * 8 + B * 8},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "status": {"rc": rc, **st},
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    ig.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
