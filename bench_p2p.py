"""P2P fetch/push microbenchmark (BASELINE.json configs[1]; paper §5.2 /
P:247): ODC gather (fetch) and scatter-accumulate (push) vs NCCL all-gather
and reduce-scatter, per-rank shard S from 64 KB to 256 MB, N ranks.

    torchrun --nproc-per-node N bench_p2p.py [--sizes 64K,1M,...] [--reps R]

S = bytes of one rank's bf16 parameter shard. Per rank and op:
  fetch          dst[N*S] bf16  <- every owner's shard (N-1 over NVLink)
  push           owner shards fp32 += w * grad[N*S/2 elems] (N-1 over NVLink)
  all_gather     torch.distributed.all_gather_into_tensor, same bf16 bytes
  reduce_scatter torch.distributed.reduce_scatter_tensor, same fp32 bytes
  push_fixed     (--variants fixed:CTAS) deterministic int64 fixed-point push;
                 GB/s counts its int64 wire bytes ((N-1)*4S)
  fetch_ce       the fetch through the copy engines (cudaMemcpyAsync peer ->
                 local per owner, after the device gate): the driver's
                 cudaMemcpyPeerAsync path
  push_slot      SLOT-mode push as it runs in a step: the unit's first push of
                 the minibatch STORES w*g into this client's slot at every
                 owner (timed alone; the untimed minibatch_end between reps
                 releases the slots), fp32 wire bytes ((N-1)*2S)
  conc_*         fetch (TMA) and push (RED or SLOT) of the same unit at the same
                 time on two streams, as the backward overlaps them: each
                 direction's GB/s over the pair's common time (fetch = rx,
                 push = tx of this rank's NVLink ports)
  --sync         the paper's synchronous-launch protocol: every op
                 alone between barriers (torch barrier + device sync before
                 and after), time = max over ranks per op, averaged
GB/s = algorithmic NVLink bytes per rank ((N-1)*S for bf16 gathers,
(N-1)*2S for fp32 reductions) / op time, op time = max over ranks of the
CUDA-event time of R back-to-back ops divided by R (barrier + sync around).
Rank 0 prints one JSON line per (op, S) and writes a markdown table.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def size_of(s: str) -> int:
    m = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    return int(s[:-1]) * m[s[-1]] if s[-1] in m else int(s)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64K,256K,1M,4M,16M,64M,256M")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/p2p.md")
    ap.add_argument("--fetch-ctas", type=int, default=0)
    ap.add_argument("--push-ctas", type=int, default=0)
    ap.add_argument("--fetch-engine", default="tma", choices=["tma", "ldg", "ce"])
    ap.add_argument("--variants", default="", help="extra fetch variants engine:ctas,... and push:ctas,...")
    ap.add_argument("--sync", action="store_true", help="synchronous-launch protocol (barrier around every op)")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2601_19362_b200.engine import OdcEngine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    rows = []

    def timed_sync(fn, reps, after=None):
        tot = 0.0
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b)], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if after is not None:
                after()
            if _ > 0:  # the first op is a warm-up
                tot += t.item()
        return tot / reps

    def timed(fn, reps, after=None):
        if args.sync or after is not None:
            return timed_sync(fn, reps, after)
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        return t.item()

    for S in [size_of(x) for x in args.sizes.split(",")]:
        shard = S // 2
        M = shard * world
        eng = OdcEngine([M], rank=rank, world=world, device=local, push_mode="red", fetch_ctas=args.fetch_ctas,
                        push_ctas=args.push_ctas, fetch_engine=args.fetch_engine)
        eng.set_params(0, torch.randn(M, device=dev))
        torch.cuda.synchronize()
        dist.barrier()
        full = torch.empty(M, dtype=torch.bfloat16, device=dev)
        grad = torch.randn(M, device=dev)
        mine = torch.empty(shard, dtype=torch.bfloat16, device=dev)
        red_out = torch.empty(shard, dtype=torch.float32, device=dev)
        reps = max(3, min(args.reps, int(args.reps * (16 << 20) / max(S, 1 << 20))))
        ce = OdcEngine([M], rank=rank, world=world, device=local, fetch_engine="ce")
        ce.set_params(0, torch.zeros(M, device=dev))
        sl = OdcEngine([M], rank=rank, world=world, device=local, push_mode="slot", push_ctas=args.push_ctas)
        sl.set_params(0, torch.zeros(M, device=dev))
        torch.cuda.synchronize()
        dist.barrier()
        ops = {
            "odc_fetch": (lambda: eng.fetch(0, full), (world - 1) * S),
            "odc_fetch_ce": (lambda: ce.fetch(0, full), (world - 1) * S),
            "odc_push": (lambda: eng.push(0, grad, 1.0), (world - 1) * 2 * S),
            "nccl_all_gather": (lambda: dist.all_gather_into_tensor(full, mine), (world - 1) * S),
            "nccl_reduce_scatter": (lambda: dist.reduce_scatter_tensor(red_out, grad), (world - 1) * 2 * S),
        }
        extra = [ce, sl]
        for v in [x for x in args.variants.split(",") if x]:
            kind, ctas = v.split(":")
            if kind == "push":
                e2 = OdcEngine([M], rank=rank, world=world, device=local, push_mode="red", push_ctas=int(ctas))
                ops[f"odc_push[c={ctas}]"] = ((lambda e=e2: e.push(0, grad, 1.0)), (world - 1) * 2 * S)
            elif kind == "fixed":  # deterministic fixed-point push: int64 on the wire (8 B/elem)
                e2 = OdcEngine([M], rank=rank, world=world, device=local, push_mode="fixed", push_ctas=int(ctas))
                ops[f"odc_push_fixed[c={ctas}]"] = ((lambda e=e2: e.push(0, grad, 1e-3)), (world - 1) * 4 * S)
            else:
                e2 = OdcEngine([M], rank=rank, world=world, device=local, fetch_ctas=int(ctas), fetch_engine=kind)
                e2.set_params(0, torch.zeros(M, device=dev))
                ops[f"odc_fetch[{kind},c={ctas}]"] = ((lambda e=e2: e.fetch(0, full)), (world - 1) * S)
            extra.append(e2)
        torch.cuda.synchronize()
        dist.barrier()
        ops["odc_push_slot"] = ((lambda: sl.push(0, grad, 1.0)), (world - 1) * 2 * S, lambda: sl.minibatch_end())
        side = torch.cuda.Stream(device=dev)

        def concurrent(pusher):
            side.wait_stream(stream)
            eng.fetch(0, full, stream=stream)
            pusher.push(0, grad, 1.0, stream=side)
            stream.wait_stream(side)

        for tag, pusher, after in (("red", eng, None), ("slot", sl, lambda: sl.minibatch_end())):
            ops[f"conc_{tag}"] = ((lambda p=pusher: concurrent(p)), {"fetch": (world - 1) * S, "push": (world - 1) * 2 * S},
                                  after)
        for name, op in ops.items():
            fn, nbytes = op[0], op[1]
            ms = timed(fn, reps, op[2] if len(op) > 2 else None)
            parts = nbytes.items() if isinstance(nbytes, dict) else [(None, nbytes)]
            for part, nb in parts:
                row = {"op": name if part is None else f"{name}:{part}", "world": world, "shard_bytes": S,
                       "ms": round(ms, 5), "GBps": round(nb / (ms / 1e3) / 1e9, 1)}
                rows.append(row)
                if rank == 0:
                    print(json.dumps(row), flush=True)
        for e2 in [eng] + extra:
            e2.minibatch_end()
        for e2 in [eng] + extra:
            e2.check()
            e2.close()
        del full, grad
        torch.cuda.empty_cache()
    if rank == 0:
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        sizes = sorted({r["shard_bytes"] for r in rows})
        names = ["odc_fetch", "odc_fetch_ce", "nccl_all_gather", "odc_push", "odc_push_slot", "nccl_reduce_scatter",
                 "conc_red:fetch", "conc_red:push", "conc_slot:fetch", "conc_slot:push"]
        names += sorted({r["op"] for r in rows} - set(names))
        with open(args.out, "w") as f:
            f.write(f"# P2P fetch/push vs NCCL, N={world} (GB/s of algorithmic NVLink bytes per rank)"
                    f"{' — synchronous launch (barrier around every op)' if args.sync else ''}\n\n")
            f.write("| shard S | " + " | ".join(names) + " |\n|---|" + "---|" * len(names) + "\n")
            for S in sizes:
                cells = []
                for n in names:
                    r = [x for x in rows if x["op"] == n and x["shard_bytes"] == S]
                    cells.append(f"{r[0]['GBps']} ({r[0]['ms']*1e3:.1f} us)" if r else "-")
                f.write(f"| {S >> 10} KB | " + " | ".join(cells) + " |\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
