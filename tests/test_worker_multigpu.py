"""ODC vs the NCCL FSDP comparison path on the same worker (2 GPUs): after
one minibatch in which the ranks run DIFFERENT numbers of microbatches (ODC,
LB-Mini style; FSDP pads with an empty microbatch that joins every
collective), every owned gradient shard must agree (fp32 sums in different
orders: rel 1e-4), and the parameters after AdamW must agree too."""
import os
import socket
import traceback

import pytest

from conftest import have_gpus

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        from paper_2601_19362_b200 import worker as W
        from paper_2601_19362_b200.engine import OdcEngine
        from paper_2601_19362_b200.shapes import Shape

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        s = Shape("tiny2", 256, 512, 2, 2, 1, 1024, True, True)
        sizes = W.unit_sizes(s)
        gen = torch.Generator(device=dev).manual_seed(0)
        units = [W.init_unit(s, u, gen, dev) for u in range(len(sizes))]
        odc = OdcEngine(sizes, rank=rank, world=world, device=rank, push_mode="slot", timeout_s=30)
        fsdp = W.FsdpComm(sizes, rank, world, dev)
        for u, t in enumerate(units):
            odc.set_params(u, t)
            fsdp.set_params(u, t)
        torch.cuda.synchronize()
        dist.barrier()
        lens = [37, 100, 63, 200, 90, 41]
        queues = {0: [[0, 1], [2]], 1: [[3, 4, 5]]}  # rank 1 has one microbatch fewer
        total = float(sum(lens))
        out = {}
        for name, comm in (("odc", W.OdcComm(odc)), ("fsdp", fsdp)):
            wk = W.Worker(s, comm, dev, ce_chunk=128)
            mine = queues[rank] + ([[]] if (name == "fsdp" and rank == 1) else [])
            for mb in mine:
                if not mb:
                    wk.empty_microbatch()
                    continue
                n = sum(lens[i] for i in mb)
                wk.microbatch(W.make_batch(lens, mb, s.vocab, dev), n / total)
            eng = odc if name == "odc" else fsdp.local
            eng.minibatch_end()
            eng.check()
            out[name] = [eng.read_grad_shard(u).clone() for u in range(len(sizes))]
        for u in range(len(sizes)):
            a, b = out["odc"][u], out["fsdp"][u]
            rel = ((a - b).norm() / b.norm().clamp_min(1e-12)).item()
            assert rel < 1e-4, (u, rel)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:
        q.put((rank, traceback.format_exc()))


@pytest.mark.skipif(not have_gpus(2), reason="needs >= 2 GPUs")
def test_odc_and_fsdp_paths_agree():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad, "\n".join(f"rank {r}:\n{m}" for r, m in bad.items())
