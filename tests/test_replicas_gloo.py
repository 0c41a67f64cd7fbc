"""N>1 path on CPU: world_size-2 gloo.

Each rank runs its own DAG replicas through libdagrt (record backend, no
GPU) with no collective on the data path; the job timing is the max over
ranks of the per-rank time and the whole-job ms per DAG divides it by the
DAGs all ranks ran -- the same helpers bench.py uses under torchrun/NCCL.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

WORLD = 2
STEPS = 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, out):
    import torch
    import torch.distributed as dist

    from golden_io import load
    from paper_2012_09646_b200 import dagrt as D
    from paper_2012_09646_b200 import replicas
    from paper_2012_09646_b200.programs import Hits

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        ids = replicas.instance_ids(rank, WORLD, STEPS)
        ctx = D.Context(backend="record", record_dag=True)
        p = Hits(ctx, mode="resident", n=300, e=900, iters=2)
        p.load_inputs(0)
        replicas.barrier(dist)
        dags = []
        for _ in ids:
            ctx.dag_clear()
            p.run()
            verts, edges = ctx.dag()
            base = min(v[0] for v in verts)  # vertex ids keep counting across runs
            dags.append({(a - base, b - base, lab) for a, b, lab in edges})
        # a deterministic per-rank "duration" so the max is checkable
        local_ms = 10.0 + 5.0 * rank
        mx = replicas.max_over_ranks(local_ms, dist)
        g = load("fig6_hits.dag")["hits"]
        ok_dag = all(d == g["edges"] for d in dags)
        allids = [None] * WORLD
        dist.all_gather_object(allids, ids)
        out[rank] = dict(mx=mx, ms=replicas.job_ms_per_dag(mx, STEPS, WORLD), ok_dag=ok_dag,
                         ids=allids)
        ctx.close()
    finally:
        dist.destroy_process_group()


def _entry(rank, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    res = {}
    _worker(rank, port, res)
    q.put((rank, res[rank]))


def test_replicas_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(WORLD):
        assert res[r]["mx"] == 15.0                      # max over ranks, seen by every rank
        assert res[r]["ms"] == pytest.approx(15.0 / (STEPS * WORLD))
        assert res[r]["ok_dag"]                          # every replica infers the golden DAG
    ids = res[0]["ids"]
    flat = sorted(i for r in ids for i in r)
    assert flat == list(range(STEPS * WORLD))            # instances partitioned, none shared
