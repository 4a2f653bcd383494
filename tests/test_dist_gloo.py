"""Multi-process (N > 1) orchestration of bench.py on CPU: world_size 2 over gloo.

The path shards into independent problem instances: every rank
gets its own data seed, there is no data-path collective, and the job value is
all ranks' units over the slowest rank's device time (MAX reduction).
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        t_rank = [0.25, 0.75][rank]
        t_max = bench.max_over_ranks(t_rank, ws, device="cpu")
        spec = bench.rank_spec(synth.scaled(synth.LARGE, 64), rank)
        ip, ix = synth.make_csr(spec)
        q.put((rank, t_max, bench.aggregate_value(ws, 1000, 3, t_max), spec.seed, int(ip[-1]), ix[:8].tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_orchestration():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, t0, v0, s0, n0, x0), (r1, t1, v1, s1, n1, x1) = out
    assert t0 == t1 == pytest.approx(0.75)               # every rank sees the slowest rank's time
    assert v0 == v1 == pytest.approx(2 * 1000 * 3 / 0.75)  # all ranks' units / max time
    assert s0 != s1 and (n0 != n1 or x0 != x1)            # independent instances: distinct data per rank


def test_single_rank_is_identity():
    assert bench.max_over_ranks(0.5, 1) == 0.5
    assert bench.aggregate_value(1, 10, 2, 0.5) == 40.0
