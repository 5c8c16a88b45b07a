"""Multi-rank host logic on CPU (gloo, world_size 2): IPC blob exchange order,
identical per-rank LB-Mini plans (every rank plans independently — no plan
broadcast on the ODC path), exact cover of the step's samples by the union of
the ranks' queues, and the max-over-ranks timing / idle-fraction reduction."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2601_19362_b200 import partition as P
        from paper_2601_19362_b200.dist import exchange_blobs, plan_digest, rank_timings

        blobs = exchange_blobs(bytes([rank]) * 64)
        assert blobs == [bytes([r]) * 64 for r in range(world)]
        lens = [max(512, x) for x in P.generate_synthetic(("lognormal", 8.0, 1.5), 256, 32768, 0)]
        plan = P.plan_flat("lb-mini", lens, world, 8, 32768, P.CostModel(1.0, 30467.0, 1))
        digests = exchange_blobs(plan_digest(plan).encode())
        assert len(set(digests)) == 1, "ranks derived different plans"
        for step in plan:
            ids = sorted(i for dev in step for mb in dev for i in mb)
            assert len(ids) == len(set(ids))
        covered = sorted(i for step in plan for dev in step for mb in dev for i in mb)
        assert covered == list(range(len(lens)))
        mx, idle, launches, rows = rank_timings(100.0 + 10 * rank, 90.0 - 20 * rank, 5)
        assert mx == 100.0 + 10 * (world - 1)
        busy = sum(90.0 - 20 * r for r in range(world))
        assert abs(idle - (1 - busy / (world * mx))) < 1e-12 and launches == 5 * world
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, traceback.format_exc()))


def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    assert res == {0: "ok", 1: "ok"}, res
