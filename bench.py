#!/usr/bin/env python
"""IRKGL16 fp64 benchmark (BASELINE.json metric: trajectory-steps/s at 1/2/4/8 B200).

One bench "step" = one irk_integrate call over the whole config-2 workload: the
Kepler ensemble of 65,536 trajectories x 10,000 IRKGL16 steps, every hot-path row
(nu-init, position sweep, stop test, 8 RHS, velocity sweep, update) inside the
timed region, inputs resident in HBM.  L2 is flushed (256 MiB write) before every
timed step; state and workspace are reset from a pristine device copy outside
the timed region.

Multi-GPU: one process per GPU.  `--gpus N` without a
torchrun environment re-launches this script under torch.distributed.run with N
ranks; under torchrun, WORLD_SIZE must equal N (else exit 2).
  * value  = STRONG scaling (default, --scaling strong): the fixed 65,536-
    trajectory batch is split into contiguous slices (parallel.batch_slice),
    each rank integrates its slice with IRK_OPT_MAPPING auto (the mapping
    follows the per-GPU batch), no data-path collective; time = max over ranks.
  * "weak": 65,536 trajectories per rank (seed + rank), reported as an extra
    field (or as `value` with --scaling weak).
  * "configs": one timed full-size call of configs 1, 3, 4 and 5 (--configs),
    sharded the same way; config 5 is ONE system sharded by body over NCCL
    (irk_set_comm, in-place all-gather of stage positions per fixed-point
    iteration), checked bitwise against a 1-GPU run of the same system, and,
    at N > 1, also run with the fused NVLink exchange (IRK_OPT_EXCHANGE = 1).

--impl reference: the scalar-C oracle (oracle/) on the host cores, each step a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import re
import socket
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
MAP_NAMES = {0: "single mapping", 1: "g1 (1 trajectory per thread / body per lane)", 2: "g2 (4 stages per lane)",
             4: "g4 (2 stages per lane)", 8: "g8 (1 stage per lane)",
             9: "g8m (1 stage per lane, DMMA stage contractions)"}


# --------------------------------------------------------------- flop model
def f_flops(problem: int, dim: int) -> int:
    """Algorithmic flops of one RHS evaluation g(q) (SURVEY.md 8(d) D-4 counts:
    + - x / sqrt = 1, fma = 2): Kepler 8, six-body 25 per symmetric pair, FPU
    5(N+1)+N, Plummer 18 per ordered pair j != i (the kernel also evaluates j = i,
    which contributes an exact zero and is not counted)."""
    from paper_2511_03655_b200 import workloads as wl
    if problem == wl.KEPLER:
        return 8
    if problem == wl.HENON_HEILES:
        return 13
    if problem == wl.FPU_BETA:
        N = dim // 2
        return 5 * (N + 1) + N
    if problem == wl.NBODY:
        N = dim // 6
        return 25 * N * (N - 1) // 2
    if problem == wl.NBODY_DIRECT:
        N = dim // 6
        return 18 * N * (N - 1)
    raise ValueError(problem)


def alg_flops(problem: int, dim: int, traj_steps: int, sweeps: int) -> int:
    """Per step 128d (nu-init) + 16d (update); per sweep 136d (a2) + 8d (Delta) +
    8 f (a3) + 136d (a4)."""
    d = dim // 2
    return traj_steps * 144 * d + sweeps * (280 * d + 8 * f_flops(problem, dim))


def fp64_peak_tflops() -> float:
    mp_ = measured_peaks()
    sm_max = float(mp_.get("sm_max_mhz", 1965.0))
    return SM_COUNT * FP64_FMA_PER_CLK_PER_SM * 2 * sm_max * 1e6 / 1e12, sm_max


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


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return ""


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
    return {"value": S * w.nsteps / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "value_1core": rate1, "cpu_model": cpu_model(),
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
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "config2_kepler_ensemble", "batch": w.batch, "nsteps": w.nsteps,
                       "h": w.h, "seed": wl.SEEDS[2]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"first {S} of {w.batch} config-2 trajectories x {w.nsteps} steps per step "
                                       "(the oracle as it stands, OpenMP over trajectories)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- our arm
class Dist:
    """torch.distributed plumbing: NCCL process group when world > 1."""

    def __init__(self, torch):
        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dev = torch.device("cuda", self.local)
        torch.cuda.set_device(self.dev)
        if self.world > 1:
            import torch.distributed as dist
            self.dist = dist
            dist.init_process_group("nccl", device_id=self.dev)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t)
        return float(t.item())

    def all_gather_obj(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out


def timed_calls(torch, ig, Y, y0, ws, iters, flush, s, n, t0=0.0):
    """n calls of irk_integrate from the pristine state, each bracketed by CUDA
    events on the launching stream; reset + L2 flush outside the events."""
    evs = []
    for _ in range(n):
        Y.copy_(y0)
        ws.zero_()
        flush.fill_(1.0)  # 256 MiB write: evicts the 126 MB L2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ig.integrate(Y, ws, t0=t0, iters=iters, stream=s)
        e1.record(s)
        evs.append((e0, e1))
    return evs


def ensemble_shard(torch, D, w, flush, s, scaling="strong"):
    """One rank's share of an ensemble config: (Integrator, y0, Y, ws, iters, batch_total)."""
    from paper_2511_03655_b200 import irk, parallel
    if scaling == "strong":
        sl = parallel.batch_slice(w.batch, D.rank, D.world)
        yl = w.y[:, sl]
        total = w.batch
    else:
        yl = w.y
        total = w.batch * D.world
    B = yl.shape[1]
    ig = irk.Integrator(w.problem, w.dim, w.h, w.nsteps, B, w.params)
    y0 = torch.tensor(yl, dtype=torch.float64, device=D.dev)
    return ig, y0, torch.empty_like(y0), ig.new_workspace(D.dev), torch.zeros(B, dtype=torch.int64, device=D.dev), total


def sub_ensemble(torch, D, cfg, flush, s):
    """One timed full-size call of ensemble config `cfg` (strong-split over ranks;
    config 1, a single trajectory, runs as replicas)."""
    from paper_2511_03655_b200 import irk, workloads as wl
    w = wl.config(cfg)
    replicas = w.batch == 1
    ig, y0, Y, ws, it, total = ensemble_shard(torch, D, w, flush, s, "weak" if replicas else "strong")
    short = irk.Integrator(w.problem, w.dim, w.h, min(w.nsteps, 200), y0.shape[1], w.params)
    Yw = y0.clone()
    short.integrate(Yw, short.new_workspace(D.dev), stream=s)   # warm-up (module load, queue)
    torch.cuda.synchronize(D.dev)
    D.barrier()
    (e0, e1), = timed_calls(torch, ig, Y, y0, ws, it, flush, s, 1)
    torch.cuda.synchronize(D.dev)
    t_local = e0.elapsed_time(e1) * 1e-3
    T = D.max(t_local)
    sweeps = D.sum(float(it.sum().item()))
    rc, st = ig.stats(ws)
    mapping = ig.get_option(irk.INFO_MAPPING_USED)
    traj_steps = total * w.nsteps
    fl = alg_flops(w.problem, w.dim, traj_steps, int(sweeps))
    peak, _ = fp64_peak_tflops()
    ig.close()
    short.close()
    return {"workload": w.name, "batch": total, "batch_per_gpu": int(y0.shape[1]), "nsteps": w.nsteps,
            "dim": w.dim, "scaling": "replicas" if replicas else "strong", "seconds": T,
            "value": traj_steps / T, "unit": UNIT, "sweeps_per_step": sweeps / traj_steps,
            "alg_tflops": fl / T / 1e12 / D.world, "frac_fp64_peak_per_gpu": fl / T / 1e12 / D.world / peak,
            "mapping": MAP_NAMES.get(mapping, str(mapping)), "rc": rc,
            "timed": "one full-size irk_integrate call per rank after a 200-step warm-up call; max over ranks"}


def nccl_comm_lines(logdir):
    """comm nRanks / NVLS facts from the NCCL_DEBUG=INFO files of this run."""
    ranks, nvls, p2p = set(), False, False
    for f in glob.glob(os.path.join(logdir, "nccl.*.log")):
        for line in open(f, errors="replace"):
            m = re.search(r"nRanks (\d+)", line)
            if m:
                ranks.add(int(m.group(1)))
            if "NVLS" in line and ("multicast support is available" in line or "enabled" in line):
                nvls = True
            if "via P2P" in line or "P2P/CUMEM" in line:
                p2p = True
    return {"comm_nranks": sorted(ranks), "nvls_seen": nvls, "p2p_seen": p2p}


def sub_plummer(torch, D, flush, s, check_steps=20):
    """Config 5: one Plummer system of 8,192 bodies, 1,000 steps, body-sharded over
    the ranks (irk_set_comm + in-place ncclAllGather of the stage positions per
    fixed-point iteration; nothing to exchange at one GPU).  A short run of the
    sharded system is compared bit for bit with a 1-GPU run on rank 0."""
    import numpy as np
    from paper_2511_03655_b200 import irk, parallel, workloads as wl
    w = wl.plummer()
    N = w.dim // 6
    out = {"workload": w.name, "N": N, "nsteps": w.nsteps, "scaling": "strong (body-sharded, one system)"}
    modes = [0, 1] if D.world > 1 else [0]
    peak, _ = fp64_peak_tflops()
    ref_short = None
    if D.rank == 0 and D.world > 1:     # 1-GPU reference of the short check run
        with irk.Integrator(w.problem, w.dim, w.h, check_steps, 1, w.params) as ig1:
            Y1 = torch.tensor(w.y, dtype=torch.float64, device=D.dev)
            ig1.integrate(Y1, ig1.new_workspace(D.dev), stream=s)
            torch.cuda.synchronize(D.dev)
            ref_short = Y1.cpu().numpy()
    for ex in modes:
        tag = "allgather" if ex == 0 else "fused"
        if ex == 1:
            os.environ["IRK_EXPERIMENTAL_FUSED_EXCHANGE"] = "1"
        res = {}
        try:
            uid = parallel.nccl_bootstrap(D.rank) if D.world > 1 else None
            yl = parallel.shard_rows(w.y, D.rank, D.world) if D.world > 1 else w.y
            y0 = torch.tensor(yl, dtype=torch.float64, device=D.dev)
            if D.world > 1:   # bitwise check of a short run against the 1-GPU result
                with irk.Integrator(w.problem, w.dim, w.h, check_steps, 1, w.params, exchange=ex) as igc:
                    igc.set_comm(uid, D.rank, D.world)
                    Yc = y0.clone()
                    igc.integrate(Yc, igc.new_workspace(D.dev), stream=s)
                    torch.cuda.synchronize(D.dev)
                    parts = D.all_gather_obj(Yc.cpu().numpy())
                ok = bool(np.array_equal(parallel.assemble_rows(parts), ref_short)) if D.rank == 0 else True
                res["bitwise_vs_1gpu"] = D.max(0.0 if ok else 1.0) == 0.0
                res["check"] = f"{check_steps} steps, {D.world} ranks vs 1 GPU"
                uid = parallel.nccl_bootstrap(D.rank)
            ig = irk.Integrator(w.problem, w.dim, w.h, w.nsteps, 1, w.params, exchange=ex)
            if D.world > 1:
                ig.set_comm(uid, D.rank, D.world)
            Y = torch.empty_like(y0)
            ws = ig.new_workspace(D.dev)
            it = torch.zeros(1, dtype=torch.int64, device=D.dev)
            if D.world == 1:   # warm-up (module load); at N > 1 the check run above is the warm-up
                with irk.Integrator(w.problem, w.dim, w.h, 3, 1, w.params) as igw:
                    Yw = y0.clone()
                    igw.integrate(Yw, igw.new_workspace(D.dev), stream=s)
                torch.cuda.synchronize(D.dev)
            D.barrier()
            (e0, e1), = timed_calls(torch, ig, Y, y0, ws, it, flush, s, 1)
            torch.cuda.synchronize(D.dev)
            T = D.max(e0.elapsed_time(e1) * 1e-3)
            sweeps = int(it.item())
            fl = alg_flops(w.problem, w.dim, w.nsteps, sweeps)
            res.update({"seconds": T, "system_steps_per_s": w.nsteps / T, "value": w.nsteps / T,
                        "unit": "system-steps/s", "sweeps_per_step": sweeps / w.nsteps,
                        "pair_interactions_per_s": float(N) * (N - 1) * 8 * sweeps / T,
                        "alg_tflops": fl / T / 1e12 / D.world,
                        "frac_fp64_peak_per_gpu": fl / T / 1e12 / D.world / peak,
                        "device_loop": bool(ig.get_option(irk.INFO_DEVICE_LOOP_USED))})
            ig.close()
        except Exception as e:  # report, do not abort the bench line
            res["error"] = str(e)[:300]
        finally:
            os.environ.pop("IRK_EXPERIMENTAL_FUSED_EXCHANGE", None)
        out[tag] = res
    return out


def run_ours(args):
    import numpy as np
    import torch

    from paper_2511_03655_b200 import irk, workloads as wl

    nccl_logdir = None
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and "NCCL_DEBUG" not in os.environ:
        # communicator facts (nRanks, NVLS) for the line; logs to files, not stdout
        nccl_logdir = os.environ.get("IRK_BENCH_NCCL_LOGDIR") or tempfile.mkdtemp(prefix="irk_nccl_")
        os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT",
                          NCCL_DEBUG_FILE=os.path.join(nccl_logdir, "nccl.%h.%p.log"))
    D = Dist(torch)
    dev, world, rank = D.dev, D.world, D.rank
    s = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    w = wl.kepler_ensemble() if args.scaling == "strong" else wl.kepler_ensemble(seed=wl.SEEDS[2] + rank)
    ig, y0, Y, ws, iters, total = ensemble_shard(torch, D, w, flush, s, args.scaling)
    B = y0.shape[1]

    warm = max(3, args.warmup)  # the contract's minimum of 3 warm-up steps
    timed_calls(torch, ig, Y, y0, ws, iters, flush, s, warm)
    torch.cuda.synchronize(dev)
    D.barrier()
    clk = Clocks(dev.index if dev.index is not None else 0)
    clk.start()
    evs = timed_calls(torch, ig, Y, y0, ws, iters, flush, s, args.steps)
    torch.cuda.synchronize(dev)
    D.barrier()
    clocks = clk.stop()
    times = [a.elapsed_time(b) * 1e-3 for a, b in evs]
    T = D.max(sum(times))
    mean_launch = D.max(statistics.mean(times))
    sweeps = D.sum(float(iters.sum().item()))
    rc, st = ig.stats(ws)
    mapping = ig.get_option(irk.INFO_MAPPING_USED)
    value = total * w.nsteps * args.steps / T

    # end to end through the C ABI from pinned host memory (H2D + kernel + D2H timed)
    yh_pin = torch.empty(tuple(y0.shape), dtype=torch.float64, pin_memory=True)
    yh = yh_pin.numpy()
    yl_host = y0.cpu().numpy()
    e2e_t = []
    for i in range(args.warmup + args.steps):
        yh[...] = yl_host
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(1.0)
        e0.record(s)
        ig.integrate_host(yh, want_energy=False, want_iters=True, stream=s)
        e1.record(s)
        torch.cuda.synchronize(dev)
        if i >= args.warmup:
            e2e_t.append(e0.elapsed_time(e1) * 1e-3)
    if not np.array_equal(yh, Y.cpu().numpy()):
        raise RuntimeError("e2e result differs from the device-resident run")
    Te = D.max(sum(e2e_t))

    # weak scaling as an extra field at N > 1 (65,536 trajectories per rank, seed + rank)
    weak = None
    if world > 1 and args.scaling == "strong":
        ww = wl.kepler_ensemble(seed=wl.SEEDS[2] + rank)
        igw, y0w, Yw, wsw, itw, totw = ensemble_shard(torch, D, ww, flush, s, "weak")
        timed_calls(torch, igw, Yw, y0w, wsw, itw, flush, s, 1)
        torch.cuda.synchronize(dev)
        D.barrier()
        evw = timed_calls(torch, igw, Yw, y0w, wsw, itw, flush, s, args.steps)
        torch.cuda.synchronize(dev)
        Tw = D.max(sum(a.elapsed_time(b) * 1e-3 for a, b in evw))
        weak = {"value": totw * ww.nsteps * args.steps / Tw, "unit": UNIT, "batch_per_gpu": ww.batch,
                "ms_per_step": 1e3 * Tw / args.steps}
        igw.close()

    subs = {}
    cfgs = [c for c in args.configs.split(",") if c.strip()] if args.configs not in ("", "none") else []
    for c in cfgs:
        c = int(c)
        try:
            subs[f"config{c}"] = sub_plummer(torch, D, flush, s) if c == 5 else sub_ensemble(torch, D, c, flush, s)
        except Exception as e:
            subs[f"config{c}"] = {"error": str(e)[:300]}

    # our kernels per irk_integrate call: one persistent ensemble launch + advance_n
    # (the cudaMemsetAsync that reset the work queue and the tableau upload are runtime copies)
    launches_per_step = 2
    line = None
    if rank == 0:
        traj_steps = total * w.nsteps
        fl = alg_flops(w.problem, w.dim, traj_steps, int(sweeps))
        achieved = fl / world / mean_launch / 1e12   # per GPU: each rank's launch does 1/world of the work
        peak, sm_max = fp64_peak_tflops()
        probe = probe_fp64(torch, irk, dev) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp) and world == 1:
            traffic = json.load(open(tp)).get("config2_kepler_ensemble_g1q")  # bytes per launch
        kname = {1: "ens_g1q_kernel<KeplerT<true>>", 2: "ens_gs_kernel<KeplerT<true>,2>",
                 4: "ens_gs_kernel<KeplerT<true>,4>", 8: "ens_gs_kernel<KeplerT<true>,8>"}.get(mapping, "?")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": warm, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded config-2 generator, workloads.py)",
            "config": {"workload": "config2_kepler_ensemble", "batch": total, "batch_per_gpu": B,
                       "nsteps": w.nsteps, "h": w.h, "seed": wl.SEEDS[2],
                       "mapping": MAP_NAMES.get(mapping, str(mapping)) + " (IRK_OPT_MAPPING auto)",
                       "schedule": "one persistent launch per call (work queue of (trajectory, step-chunk) "
                                   "units for g1; one group of lanes per trajectory for g2/g4/g8)",
                       "l2": "flushed (256 MiB write) before every timed step",
                       "parallelism": (f"trajectory-sharded x{world} (contiguous slices of the fixed batch), "
                                       "no collective") if args.scaling == "strong" else
                                      f"x{world} independent 65,536-trajectory ensembles (seed + rank)"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per ens_g1q launch (ncu --set full)",
                         "peak_note": f"FP64 pipe: {SM_COUNT} SM x {FP64_FMA_PER_CLK_PER_SM} FMA/clk x 2 x "
                                      f"{sm_max:.0f} MHz (MEASURED_PEAKS.json has no FP64 entry); "
                                      f"DFMA probe measured {probe:.2f} TFLOP/s on this GPU",
                         "kernel": kname,
                         "flop_count": "SURVEY 8(d) D-4: per traj-step 144d, per sweep 280d + 8 f_Kepler (8)",
                         "timed": "CUDA events on the launching stream around irk_integrate "
                                  "(1 ensemble launch + advance_n; tableau upload + queue memsets)",
                         "flops_per_launch": fl / world, "sweeps_per_step": sweeps / traj_steps},
            "e2e": {"value": total * w.nsteps * args.steps / Te, "unit": UNIT,
                    "h2d_bytes_per_step": int(y0.numel()) * 8 * world,
                    "d2h_bytes_per_step": (int(y0.numel()) * 8 + B * 8) * world,
                    "api": "irk_integrate_host (pinned host y in, y + iters out; copies inside the timed region)"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "status": {"rc": rc, **st},
        }
        if weak is not None:
            line["weak_scaling"] = weak
        if subs:
            line["configs"] = subs
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w)
    D.barrier()
    if nccl_logdir and rank == 0 and line is not None:
        line["nccl"] = nccl_comm_lines(nccl_logdir)
    if world > 1:
        D.dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    ig.close()
    return 0


def free_port() -> int:
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--configs", default="1,3,4,5", help="extra full-size configs to time once ('none' to skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        # self-launch: one process per GPU, rendezvous on 127.0.0.1
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
               os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if env_world is not None and int(env_world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
