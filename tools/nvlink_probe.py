"""NVLink evidence for the fetch and push engines from ONE process driving N
GPUs (OdcEngine.local_group: direct peer access, no IPC), so that ncu — which
must never wrap a multi-rank command — can profile the real kernels with the
NVLink counters (nvlrx__bytes / nvltx__bytes):

  ncu --devices 0 --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,\
      nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum -k regex:"fetch|push_bulk" \
      python tools/nvlink_probe.py --gpus 2

Without ncu it prints the CUDA-event GB/s of each op with every rank running it
concurrently (the step's situation), max over ranks: fetch (N-1)*block*2 B of
NVLink ingress, push (RED / SLOT store) (N-1)*block*4 B of egress per rank.

usage: python tools/nvlink_probe.py --gpus N [--mb 16] [--reps 20]
"""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_19362_b200.engine import OdcEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--mb", type=int, default=16, help="per-rank shard size in MB of bf16 parameters")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    N = args.gpus
    shard = (args.mb << 20) // 2
    M = shard * N
    out = []
    for mode in ("red", "slot"):
        engs = OdcEngine.local_group([M], N, list(range(N)), push_mode=mode)
        streams, fulls, grads = [], [], []
        for e in engs:
            with torch.cuda.device(e.device):
                e.set_params(0, torch.randn(M, device=f"cuda:{e.device}"))
                streams.append(torch.cuda.Stream())
                fulls.append(torch.empty(M, dtype=torch.bfloat16, device=f"cuda:{e.device}"))
                grads.append(torch.randn(M, device=f"cuda:{e.device}"))
        for d in range(N):
            torch.cuda.synchronize(d)

        def run(op, reps, after=None):
            evs = []
            for e, s in zip(engs, streams):
                with torch.cuda.device(e.device):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s)
                    for _ in range(reps):
                        if op == "fetch":
                            e.fetch(0, fulls[e.rank], stream=s)
                        else:
                            e.push(0, grads[e.rank], 1.0, stream=s)
                    b.record(s)
                    evs.append((a, b))
            for d in range(N):
                torch.cuda.synchronize(d)
            ms = max(a.elapsed_time(b) for a, b in evs) / reps
            if after:
                for e, s in zip(engs, streams):
                    with torch.cuda.device(e.device):
                        e.minibatch_end(stream=s)
                for d in range(N):
                    torch.cuda.synchronize(d)
            return ms

        ops = [("fetch", 2)] if mode == "red" else []
        ops += [("push", 4)]
        for op, eb in ops:
            reps = args.reps if not (mode == "slot" and op == "push") else 1  # SLOT: the minibatch's first push stores
            run(op, 1, after=True)
            tot = 0.0
            for _ in range(3 if reps == 1 else 1):
                tot += run(op, reps, after=mode == "slot")
            ms = tot / (3 if reps == 1 else 1)
            nbytes = (N - 1) * shard * eb
            row = {"op": f"{op}[{mode}]" if op == "push" else op, "gpus": N, "shard_MB": args.mb, "ms": round(ms, 4),
                   "GBps_per_rank": round(nbytes / ms / 1e6, 1), "bytes_per_launch": nbytes}
            print(json.dumps(row), flush=True)
            out.append(row)
        for e in engs:
            e.check()
            e.close()


if __name__ == "__main__":
    main()
