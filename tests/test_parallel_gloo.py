"""World-size-2 `gloo` tests of the multi-GPU host path, on CPU.

The kernels' sharded layout is checked on the GPU (virtual shards, 1-rank NCCL);
here two processes exercise the host plumbing bench.py uses: batch slices and
their gather (ensembles), body-row sharding and reassembly plus the NCCL id
bootstrap (config 5), and the max-over-ranks timing reduction.  The device
call is stood in for by the oracle, so the reassembled results must equal a
single-process oracle run bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2511_03655_b200 import parallel, workloads as wl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    out = {}
    # ensembles: each rank integrates its slice, rank 0 gets the gathered batch
    w = wl.kepler_ensemble(batch=37, nsteps=200)
    sl = parallel.batch_slice(w.batch, rank, world)
    r = oracle.integrate(w.problem, np.ascontiguousarray(w.y[:, sl]), w.params, w.h, w.nsteps, nthreads=1)
    out["ens"] = parallel.gather_batch(r["y"])
    out["ens_it"] = parallel.gather_batch(r["iters"][None, :])[0]
    # config-5 plumbing: local rows out, reassembled rows back
    p = wl.plummer(N=64, nsteps=3)
    yl = parallel.shard_rows(p.y[:, 0], rank, world)
    full = oracle.integrate(p.problem, p.y[:, 0], p.params, p.h, p.nsteps, nthreads=1)["y"]  # device stand-in
    mine = parallel.shard_rows(full, rank, world)
    assert mine.shape == yl.shape
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    out["nbody"] = parallel.assemble_rows(parts)
    # bootstrap: every rank holds rank 0's bytes (a stand-in id when NCCL is absent)
    obj = [os.urandom(128) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    allids = [None] * world
    dist.all_gather_object(allids, obj[0])
    out["same_id"] = all(x == allids[0] for x in allids)
    out["tmax"] = parallel.max_over_ranks(float(rank + 1))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_ensemble_shards_gather_bitwise(results, orc):
    w = wl.kepler_ensemble(batch=37, nsteps=200)
    ref = orc.integrate(w.problem, w.y, w.params, w.h, w.nsteps)
    for r in (0, 1):
        assert np.array_equal(results[r]["ens"], ref["y"])
        assert np.array_equal(results[r]["ens_it"], ref["iters"])


def test_body_rows_roundtrip(results, orc):
    p = wl.plummer(N=64, nsteps=3)
    ref = orc.integrate(p.problem, p.y[:, 0], p.params, p.h, p.nsteps)["y"]
    for r in (0, 1):
        assert np.array_equal(results[r]["nbody"], ref)


def test_bootstrap_and_max_reduction(results):
    assert results[0]["same_id"] and results[1]["same_id"]
    assert results[0]["tmax"] == 2.0 and results[1]["tmax"] == 2.0


def test_batch_slice_partition():
    for B in (1, 7, 65536, 65537):
        for P in (1, 2, 3, 8):
            sl = [parallel.batch_slice(B, r, P) for r in range(P)]
            assert sl[0].start == 0 and sl[-1].stop == B
            assert all(a.stop == b.start for a, b in zip(sl, sl[1:]))
            assert max(s.stop - s.start for s in sl) - min(s.stop - s.start for s in sl) <= 1
