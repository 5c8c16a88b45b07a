"""Multi-GPU ODC engine parity: one process per GPU (torch.multiprocessing),
CUDA IPC-mapped peer arenas, NVLink fetch/push, device-side barrier.

Each rank pushes a DIFFERENT number of microbatches (one rank pushes none —
the LB-Mini situation the barrier must tolerate), over several minibatches,
and every rank checks its owned grad shard against the CPU oracle computed
from the same seeded inputs, then AdamW against torch fp32, then the fetch of
the updated parameters (gated on every owner's published epoch)."""
import os
import socket
import traceback

import numpy as np
import pytest

from conftest import have_gpus

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

SIZES = [7, 4099, 1_000_003]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads(epoch, client, k, n, layer):
    rng = np.random.default_rng(1000 * epoch + 100 * client + 10 * k + layer)
    return rng.standard_normal(n).astype(np.float32), np.float32(rng.random())


def _counts(world, epoch):
    # microbatch counts per rank: varying, rank (epoch % world) gets none
    return [0 if r == epoch % world else 1 + (r + epoch) % 3 for r in range(world)]


def _worker(rank, world, port, mode, q):
    try:
        import torch
        import torch.distributed as dist

        from oracle import odc_oracle as O
        from paper_2601_19362_b200.engine import OdcEngine

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        eng = OdcEngine(SIZES, rank=rank, world=world, device=rank, push_mode=mode, timeout_s=30)
        torch.manual_seed(0)
        fulls = [torch.randn(n) for n in SIZES]  # identical on every rank
        for l, f in enumerate(fulls):
            eng.set_params(l, f.to(dev))
        torch.cuda.synchronize()
        dist.barrier()
        ref = [f.clone().to(dev).requires_grad_(True) for f in fulls]
        opt = torch.optim.AdamW(ref, lr=1e-2, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.01, foreach=False)
        for l, f in enumerate(fulls):  # fetch over NVLink, bit-exact
            out = torch.empty(SIZES[l], dtype=torch.bfloat16, device=dev)
            eng.fetch(l, out)
            torch.cuda.synchronize()
            assert torch.equal(out.cpu(), f.to(torch.bfloat16)), f"fetch l={l}"
        for epoch in range(3):
            counts = _counts(world, epoch)
            for k in range(counts[rank]):
                for l, n in enumerate(SIZES):
                    g, w = _grads(epoch, rank, k, n, l)
                    eng.push(l, torch.from_numpy(g).to(dev), float(w))
            eng.minibatch_end()
            eng.check()
            for l, n in enumerate(SIZES):
                pushes = [(c, *_grads(epoch, c, k, n, l)) for c in range(world) for k in range(counts[c])]
                want_full = (O.fixed_mode_reduce(n, pushes) if mode == "fixed"
                             else O.slot_mode_reduce(world, n, pushes, np.float32))
                b, ln = eng.shard_range(l)
                got = eng.read_grad_shard(l).cpu().numpy()
                if mode in ("slot", "fixed"):
                    assert np.array_equal(got, want_full[b:b + ln]), f"slot grads e={epoch} l={l}"
                else:
                    assert np.allclose(got, want_full[b:b + ln], rtol=1e-5, atol=1e-6), f"red grads e={epoch} l={l}"
                ref[l].grad = torch.from_numpy(want_full).to(dev)
            eng.adam_step(lr=1e-2, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.01)
            opt.step()
            for l, n in enumerate(SIZES):  # fetch waits for every owner's new epoch
                m = torch.empty(n, dtype=torch.float32, device=dev)
                eng.fetch_master(l, m)
                torch.cuda.synchronize()
                assert torch.allclose(m, ref[l].detach(), rtol=1e-5, atol=1e-6), f"adam e={epoch} l={l}"
            eng.check()
        dist.barrier()
        eng.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


@pytest.mark.skipif(not have_gpus(2), reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", ["red", "slot", "fixed"])
def test_engine_multi_gpu(mode):
    import torch
    import torch.multiprocessing as mp

    world = min(4, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, msg = q.get(timeout=300)
        res[r] = msg
    for p in procs:
        p.join(timeout=60)
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad, "\n".join(f"rank {r}:\n{m}" for r, m in bad.items())


def _timeout_worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        from paper_2601_19362_b200 import errors as E
        from paper_2601_19362_b200.engine import OdcEngine

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        eng = OdcEngine([4096], rank=rank, world=world, device=rank, timeout_s=2.0)
        eng.set_params(0, torch.zeros(4096, device=dev))
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:  # rank 0 reaches the minibatch barrier; rank 1 never does
            eng.minibatch_end()
            try:
                eng.check()
                q.put((rank, "no timeout raised"))
            except E.BarrierTimeout:
                q.put((rank, "ok"))
        else:
            q.put((rank, "ok"))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        q.put((rank, traceback.format_exc()))


@pytest.mark.skipif(not have_gpus(2), reason="needs >= 2 GPUs")
def test_barrier_watchdog_turns_a_missing_peer_into_an_error():
    """SURVEY §5 failure detection: the device barrier spin is bounded by
    %globaltimer; a peer that never arrives yields BarrierTimeout on the host
    instead of a hung GPU."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_timeout_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
