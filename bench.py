"""bench.py — ODC hot-path benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl odc|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload "odc_minibatch_comm" (default): one ODC optimizer step (minibatch)
of the Qwen2.5-1.5B-shaped shard store (28 FSDP units x 46,797,824 elements,
bf16 params / fp32 grads, block-sharded over the N ranks) driven by the
LB-Mini plan of the BASELINE long-tail workload (generate_synthetic lognormal
mu=8 sigma=1.5, 2048 lengths, cap 32768, floored at 512; minibatch 8 per
rank; budget 32768 tokens). Per microbatch of this rank's LB-Mini queue:
fetch every unit (forward), fetch every unit again + push its fp32 gradient
(backward); then the once-per-minibatch barrier and the fused AdamW on the
owned shards. Every step of it is an sm_100a kernel of libodc.so; the model
compute between fetch and push is not part of this workload (it is the
`sft` workload's job).

value  = whole-job fetch+push bytes per second (GB/s), bytes = elements
         moved x (2 B bf16 fetch, 4 B fp32 push), summed over ranks, over the
         max-over-ranks device time of K steps (CUDA events, barrier + sync on
         both sides). Inputs are > L2 (5.2 GB of units per pass), no flush.
e2e    = the same step through the reference-facing by-value API: each
         fetched unit is copied to pinned host memory (ShardFabric::gather
         returns a host vector) and each pushed gradient comes from pinned
         host memory (scatter_accumulate takes one), copies inside the timed
         region.
--impl reference: the reference's own CPU implementation of the same path
         (ShardFabric<float> from oracle/_ref, built unmodified from
         /root/reference; the oracle port if _ref is absent) on host cores,
         one bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P2_BYTES_BF16, P4_BYTES_F32 = 2, 4
NVLINK_NOMINAL_GBS = 900.0
METRIC = "tokens/sec at 1/2/4/8 B200 on long-tail seq lengths; fetch/push GB/s vs NVLink"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="odc", choices=["odc", "reference"])
    ap.add_argument("--workload", default="sft", choices=["sft", "odc_minibatch_comm", "config0"],
                    help="config0 = BASELINE configs[0]: the small transformer at world 2 on the survey's 16 lengths")
    ap.add_argument("--no-fsdp", action="store_true", help="skip the same-box NCCL FSDP comparison arm")
    ap.add_argument("--trace", default="", help="write a Chrome trace (reference schema) of one extra ODC step")
    ap.add_argument("--cost", default="b200", choices=["b200", "flops"],
                    help="LB cost beta/alpha: FLOP ratio ('flops') or FLOP ratio x measured kernel-throughput ratio")
    ap.add_argument("--cache-params", action="store_true",
                    help="SURVEY 8(f)1: keep fetched units for the whole minibatch (one fetch per unit per step)")
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--push-mode", default="slot", choices=["red", "slot", "fixed"],
                    help="slot (default): deterministic, w*g stored into the owner-side slots; red: remote fp32 reductions; "
                         "fixed: deterministic int64 fixed point in bounded memory")
    ap.add_argument("--minibs", type=int, default=8)
    ap.add_argument("--fetch-ctas", type=int, default=0)
    ap.add_argument("--push-ctas", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cap", type=int, default=32768,
                    help="longest sample (lognormal lengths capped here) = microbatch token budget (packing ratio 1)")
    ap.add_argument("--recompute", default="auto", choices=["auto", "none", "selective", "full"],
                    help="activation recompute in the worker backward; auto = least recompute that fits HBM")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload_lengths(cap=32768):
    from paper_2601_19362_b200 import partition as P

    raw = P.generate_synthetic(("lognormal", 8.0, 1.5), 2048, cap, 0)
    return [max(512, x) for x in raw]


def log(*a):
    """Progress on stderr (ODC_BENCH_LOG=1), never on the JSON stdout line."""
    if os.environ.get("ODC_BENCH_LOG"):
        print(f"[bench {time.strftime('%H:%M:%S')} rank {os.environ.get('RANK', '0')}]", *a, file=sys.stderr, flush=True)


def act_bytes_per_token_layer(shape, mode):
    """Bytes of saved activations per token per layer (worker._keep)."""
    d, H, KV, hd, ffn = shape.d, shape.heads, shape.kv_heads, shape.head_dim, shape.ffn
    if mode == "none":  # x a q o hm bn (bf16 d) + k v + gu m + r1 r2 lse
        return 12 * d + 4 * KV * hd + 6 * ffn + 8 + 4 * H
    if mode == "selective":  # x, o, lse
        return 4 * d + 4 * H
    return 2 * d  # x


def pick_recompute(shape, budget_tokens, free_bytes):
    """Least recompute whose saved activations for the largest microbatch fit
    next to one layer's transient working set (~3x a stored layer) + 6 GB."""
    transient = 3 * act_bytes_per_token_layer(shape, "none") * budget_tokens + (6 << 30)
    for mode in ("none", "selective", "full"):
        if act_bytes_per_token_layer(shape, mode) * budget_tokens * shape.layers + transient <= free_bytes:
            return mode
    return "full"


def rank_plan(world, minibs, shape):
    """LB-Mini plan (src/partition.cpp:490-580) -> per step, per rank: list of
    microbatches (sample id lists)."""
    from paper_2601_19362_b200 import partition as P

    lens = workload_lengths()
    steps = P.plan_flat("lb-mini", lens, world, minibs, 32768, P.CostModel(1.0, shape.beta_over_alpha(), 1))
    return lens, steps


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", os.environ.get("ODC_CLOCK_MS", "100")], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][2]) if self.rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_threads(elems):
    """Host threads for the reference CPU sample: one independent FSDP unit per
    thread, bounded by the cores this process may use and by host memory (a
    ShardFabric<float> sample holds ~6 copies of the unit in fp32)."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        import psutil
        mem = psutil.virtual_memory().available
    except Exception:
        mem = 16 << 30
    per = max(1, 6 * 4 * int(elems))
    return max(1, min(cores, int(os.environ.get("ODC_CPU_THREADS", "64")), int(0.5 * mem // per)))


def cpu_reference_sample(world, elems, micro):
    """Times the reference's CPU fabric (ShardFabric<float>) on a bounded
    sample: one FSDP unit, `world` simulated ranks, each client fetching twice
    and pushing once (one microbatch of one unit), then finalize. Returns
    (seconds, bytes_equiv, kind, sample)."""
    from oracle import refbind as R

    gathers, pushes = 2, 1
    # same logical work, normalised to the B200 path's dtypes (bf16 fetch, fp32 push)
    bytes_equiv = world * (gathers * elems * P2_BYTES_BF16 + pushes * elems * P4_BYTES_F32)
    if R.available():
        thr = cpu_threads(elems)
        sec = R.fabric_seconds_f32_mt(world, elems, gathers, pushes, 1, thr) / thr
        return sec, bytes_equiv, "reference", (f"ShardFabric<float>({world}, {elems}) from oracle/_ref: "
                                                f"{world} clients x ({gathers} gather + {pushes} scatter_accumulate)"
                                                f" + finalize_minibatch, one FSDP unit of one microbatch; "
                                                f"{thr} units on {thr} host threads, per-unit time = wall/{thr}")
    import numpy as np

    from oracle import odc_oracle as O

    f = O.ShardFabric(world, elems, np.float32)
    f.set_params("u", np.zeros(elems, np.float32))
    g = np.ones(elems, np.float32)
    t = time.perf_counter()
    for c in range(world):
        for _ in range(gathers):
            f.gather(c, "u")
        f.scatter_accumulate(c, g, np.float32(1.0 / world))
    f.finalize_minibatch()
    return time.perf_counter() - t, bytes_equiv, "port", "oracle port (numpy), same sample"


def ref_lengths(cap):
    """The BASELINE workload from the REFERENCE's own generator (oracle/_ref:
    generate_synthetic, src/workload.cpp:133-145), floored at 512 — the same
    list the product's odc_generate_synthetic returns (bit-exact golden)."""
    from oracle import refbind as R

    return [max(512, x) for x in R.generate_synthetic(("lognormal", 8.0, 1.5), 2048, cap, 0)]


def ref_plan(lens, world, minibs, budget, beta):
    """LB-Mini plan from the reference's own plan() (solutions_to_json):
    per step, per device, the microbatches' token sums."""
    from oracle import refbind as R

    js = json.loads(R.plan_json("lb-mini", lens, world, minibs, budget, 1.0, beta, 1))
    return [[[mb["token_sum"] for mb in dev] for dev in st["per_device"]] for st in js["steps"]]


def sft_config(args, shape, world, beta):
    """The bench line's `config` — a function of the arguments only, so both
    arms (odc and --impl reference) print the identical dict."""
    return {"workload": "odc_sft", "model": shape.name, "plan": "lb-mini (odc) / lb-micro (fsdp)",
            "minibs_per_rank": args.minibs, "budget_tokens": args.cap,
            "lengths": f"lognormal(8,1.5) n=2048 cap={args.cap} seed=0, floor 512",
            "recompute": args.recompute, "push_mode": args.push_mode, "parallelism": f"odc-dp{world}",
            "cost_beta_over_alpha": round(beta, 1), "cost_model": args.cost, "cache_params": args.cache_params,
            "attention": "tcgen05", "l2": "inputs > L2 (GBs of activations/units), no flush"}


class RefStepTimer:
    """The reference's CPU implementation of one ODC step, measured: every
    FSDP unit at its true size (embedding + L layers) as a ShardFabric<float>
    of `world` simulated ranks from oracle/_ref; per step each client gathers
    every unit twice and scatter_accumulates it once per microbatch of its
    LB-Mini queue, then finalize_minibatch per unit. Units run in parallel on
    host threads (one fabric per thread at a time: it is not thread-safe)."""

    def __init__(self, world, unit_sizes, threads):
        from oracle import refbind as R

        self.world, self.threads = world, threads
        self.step = R.RefStep(world, unit_sizes)

    def run(self, plan_step):
        return self.step.run([len(dev) for dev in plan_step], self.threads)

    def close(self):
        self.step.close()


def ref_threads(world, unit_sizes):
    """Host threads for the reference step: every core this process may use,
    bounded by host memory (each thread's two live gather copies of the
    largest unit) and ODC_CPU_THREADS."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        import psutil
        mem = psutil.virtual_memory().available
    except Exception:
        mem = 16 << 30
    resident = 4 * sum(unit_sizes) * (2 + world)  # params + grads + ranks x slot shards, fp32
    per = 8 * max(unit_sizes)
    room = max(1, int((0.8 * mem - resident) // per))
    return max(1, min(cores, int(os.environ.get("ODC_CPU_THREADS", "256")), room))


def run_reference(args):
    """--impl reference: the reference's own CPU path of the ODC step, timed on
    host cores. Everything comes from oracle/_ref (the unmodified reference
    built by oracle/Makefile): workload lengths, the LB-Mini plan, and the
    ShardFabric<float> data path; nothing of the product is loaded."""
    from paper_2601_19362_b200.shapes import SHAPES  # pure-Python model constants

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    shape = SHAPES[args.model]
    world = args.gpus
    if args.workload == "sft":
        from oracle import refbind as R

        if not R.available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (no /root/reference at build)"}))
            return
        beta = shape.beta_over_alpha_b200() if args.cost == "b200" else shape.beta_over_alpha()
        lens = ref_lengths(args.cap)
        t_plan0 = time.perf_counter()
        plan = ref_plan(lens, world, args.minibs, args.cap, beta)
        t_plan = time.perf_counter() - t_plan0
        sizes = shape.unit_sizes()
        thr = ref_threads(world, sizes)
        timer = RefStepTimer(world, sizes, thr)
        budget_s = float(os.environ.get("ODC_REF_BUDGET_S", "300"))
        t0 = time.perf_counter()
        t_first = timer.run(plan[0])  # warm-up 1: slot allocation / first-touch page faults
        warm = 1
        while warm < args.warmup and (time.perf_counter() - t0) + (args.warmup - warm + args.steps) * t_first < budget_s:
            timer.run(plan[warm % len(plan)])
            warm += 1
        secs, toks, n = [], 0, 0
        for k in range(args.warmup, args.warmup + args.steps):
            if secs and (time.perf_counter() - t0) + sum(secs) / len(secs) > budget_s:
                break  # bounded sample: the remaining steps would exceed the time budget
            st = plan[k % len(plan)]
            secs.append(timer.run(st) + t_plan / len(plan))  # + the reference plan() share of one step
            toks += sum(sum(dev) for dev in st)
        timer.close()
        total = sum(secs)
        tps = toks / total
        sample = (f"ShardFabric<float>({world}, M) from oracle/_ref for every FSDP unit at its true size "
                  f"({len(sizes)} units: {sizes[0]:,} + {len(sizes) - 1} x {sizes[1]:,} elements); per step every "
                  f"client gathers each unit 2x and scatter_accumulates it 1x per microbatch of its LB-Mini queue "
                  f"(reference plan()), then finalize_minibatch per unit; units in parallel on {thr} host threads; "
                  f"{len(secs)} of {args.steps} steps measured (budget {budget_s:.0f} s), warmup {warm}")
        line = {"metric": METRIC, "impl": "reference", "value": round(tps, 2), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "steps_measured": len(secs), "warmup_run": warm,
                "ms_per_step": round(total / len(secs) * 1e3, 3), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": sft_config(args, shape, world, beta),
                "cpu_baseline": {"value": round(tps, 2), "unit": "tokens/s", "cores": thr, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": round(tps, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "plan_seconds": round(t_plan, 4), "tokens_timed": toks}
        print(json.dumps(line), flush=True)
        return
    for _ in range(args.warmup):
        cpu_reference_sample(world, shape.layer_elems, 1)
    secs, byts = 0.0, 0
    for _ in range(args.steps):
        s, b, kind, sample = cpu_reference_sample(world, shape.layer_elems, 1)
        secs += s
        byts += b
    gbs = byts / secs / 1e9
    line = {"metric": METRIC, "impl": "reference", "value": round(gbs, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(secs / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": args.workload, "model": shape.name, "world": world},
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s",
                             "cores": cpu_threads(shape.layer_elems) if kind == "reference" else 1,
                             "kind": kind, "sample": sample},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def analytic(lens, plan_odc, plan_fsdp, beta, steps):
    """Compute-only prediction of the reference's evaluator (src/runtime.cpp:
    52-79) on the same plans, cost alpha*s^2 + beta*s per sample: ODC total =
    max_d busy, collective total = sum over microbatch slots of max_d; bubble =
    1 - sum(busy)/(D*T) (:43). Returns (speedup, odc bubble, collective bubble)."""
    def c(mb):
        return sum(float(lens[i]) ** 2 + beta * lens[i] for i in mb)

    odc = coll = busy_o = busy_c = 0.0
    D = len(plan_odc[0])
    for k in steps:
        po = plan_odc[k % len(plan_odc)]
        odc += max(sum(c(mb) for mb in dev) for dev in po)
        busy_o += sum(c(mb) for dev in po for mb in dev)
        fs = plan_fsdp[k % len(plan_fsdp)]
        coll += sum(max(c(dev[m]) if dev[m] else 0.0 for dev in fs) for m in range(len(fs[0])))
        busy_c += sum(c(mb) for dev in fs for mb in dev if mb)
    return coll / odc, 1 - busy_o / (D * odc), 1 - busy_c / (D * coll)


def run_sft(args):
    """Workload "sft" (default): one ODC optimizer step of Qwen2.5-1.5B-shaped
    SFT on the long-tail workload per bench step (see module docstring)."""
    import torch
    import torch.distributed as dist

    from paper_2601_19362_b200 import _lib
    from paper_2601_19362_b200 import gemm as G
    from paper_2601_19362_b200 import partition as P
    from paper_2601_19362_b200 import worker as W
    from paper_2601_19362_b200.dist import rank_timings
    from paper_2601_19362_b200.engine import OdcEngine
    from paper_2601_19362_b200.shapes import SHAPES

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    shape = SHAPES[args.model]
    sizes = W.unit_sizes(shape)
    lens = workload_lengths(args.cap)
    budget = args.cap
    beta = shape.beta_over_alpha_b200() if args.cost == "b200" else shape.beta_over_alpha()
    cost = P.CostModel(1.0, beta, 1)
    plan_odc = P.plan_flat("lb-mini", lens, world, args.minibs, budget, cost)
    plan_fsdp = P.plan_flat("lb-micro", lens, world, args.minibs, budget, cost)
    do_fsdp = world > 1 and not args.no_fsdp

    def load(target):  # identical full units on every rank, each keeps its slice
        gen = torch.Generator(device=dev).manual_seed(0)
        for u in range(len(sizes)):
            full = W.init_unit(shape, u, gen, dev)
            target.set_params(u, full)
            del full
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    eng = OdcEngine(sizes, rank=rank, world=world, device=local, push_mode=args.push_mode,
                    fetch_ctas=args.fetch_ctas, push_ctas=args.push_ctas)
    load(eng)
    recompute = args.recompute
    if recompute == "auto":
        # the FSDP arm runs after the ODC engine is released; its shards + collective
        # buffers take the same HBM as the ODC arena (+ bf16/fp32 shard copies)
        free = torch.cuda.mem_get_info(dev)[0] - (eng.arena_bytes() // 3 if do_fsdp else 0)
        free -= 2 * sizes[1] * 6 + sizes[0] * 6  # the worker's unit buffers (bf16 params + fp32 grads, x2 / embedding)
        t = torch.tensor([float(free)], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
        recompute = pick_recompute(shape, budget, int(t.item()))
    log("params loaded; arena GB", eng.arena_bytes() / 1e9, "recompute", recompute)

    warm_steps = list(range(args.warmup))
    timed_steps = list(range(args.warmup, args.warmup + args.steps))

    def step_tokens(plan, k):
        return sum(lens[i] for dv in plan[k % len(plan)] for mb in dv for i in mb)

    def run_arm(comm, plan, resident: bool, record=False, clocks=None):
        worker = W.Worker(shape, comm, dev, cache_params=args.cache_params and comm.name == "odc",
                          recompute=recompute, max_positions=max(65536, args.cap))
        chk = eng.check if comm.name == "odc" else comm.local.check
        stream = torch.cuda.current_stream()

        def one(k, batches=None):
            mine = plan[k % len(plan)][rank]
            total = float(step_tokens(plan, k))
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t2 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            loss = torch.zeros((), device=dev)
            for j, mb in enumerate(mine):
                if not mb:
                    worker.empty_microbatch()
                    continue
                b = batches[j] if batches is not None else W.make_batch(lens, mb, shape.vocab, dev, heads=shape.heads, kv_heads=shape.kv_heads)
                ntok = sum(lens[i] for i in mb)
                loss += worker.microbatch(b, ntok / total) * (ntok / total)
            t1.record(stream)
            worker.minibatch_end()
            t2.record(stream)
            return t0, t1, t2, loss

        for k in warm_steps:
            one(k)
            torch.cuda.synchronize()
            log(comm.name, "warm step", k, "done")
        chk()
        pre = {}
        if resident:
            for k in timed_steps:
                pre[k] = [W.make_batch(lens, mb, shape.vocab, dev, heads=shape.heads, kv_heads=shape.kv_heads) if mb else None
                          for mb in plan[k % len(plan)][rank]]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        G.recorder = G.Recorder() if record else None
        n0 = _lib.kernel_launches()
        evs, losses = [], []
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        ctx = clocks if clocks is not None else _Null()
        with ctx:  # nvidia-smi clock/throttle sampling covers exactly the timed steps
            a.record(stream)
            for k in timed_steps:
                nvtx = os.environ.get("ODC_NVTX_STEP") and k == timed_steps[0]  # ncu --nvtx-include odc_step/
                if nvtx:
                    torch.cuda.nvtx.range_push("odc_step")
                t0, t1, t2, loss = one(k, pre.get(k))
                if nvtx:
                    torch.cuda.nvtx.range_pop()
                evs.append((t0, t1, t2))
                if not resident:
                    losses.append(loss.item())  # D2H of the step's result (e2e)
            z.record(stream)
            torch.cuda.synchronize()
        launches = _lib.kernel_launches() - n0
        chk()
        log(comm.name, "timed steps done", a.elapsed_time(z), "ms; per step",
            [round(e0.elapsed_time(e2), 2) for e0, _, e2 in evs])
        gsum = G.recorder.summary() if record else None
        G.recorder = None
        ms = a.elapsed_time(z)
        busy = sum(e0.elapsed_time(e1) for e0, e1, _ in evs)
        ms_max, idle, launches_all, _ = rank_timings(ms, busy, launches, device=dev)
        del worker
        torch.cuda.empty_cache()
        toks = sum(step_tokens(plan, k) for k in timed_steps)
        return {"ms": ms_max, "tokens": toks, "tps": toks / (ms_max / 1e3), "idle": idle,
                "launches": launches_all, "gemm": gsum,
                "loss": (sum(losses) / len(losses)) if losses else None}

    clk = ClockSampler(local)
    res = run_arm(W.OdcComm(eng), plan_odc, resident=True, record=True, clocks=clk)
    e2e = run_arm(W.OdcComm(eng), plan_odc, resident=False) if not args.no_e2e else None
    if args.trace:
        write_trace(args.trace, shape, W.OdcComm(eng), plan_odc, lens, timed_steps[0], rank, world, dev)
    comm = comm_rates(eng, sizes[1], rank, world, dev)
    fs = None
    if do_fsdp:  # release the ODC arena first (peers are idle: synchronised + barrier)
        torch.cuda.synchronize()
        dist.barrier()
        eng.check()
        eng.close()
        torch.cuda.empty_cache()
        fsdp = W.FsdpComm(sizes, rank, world, dev)
        load(fsdp)
        fs = run_arm(fsdp, plan_fsdp, resident=True)
        fsdp.local.close()

    hbm, hbm_kind = peaks()
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        tflops_peak, tkind = float(pk["bf16_tflops_sustained"]), "measured sustained"
        tflops_burst = float(pk["bf16_tflops"])
    except Exception:
        tflops_peak, tkind, tflops_burst = 1400.0, "fallback sustained", 2250.0
    roof = None
    if res["gemm"]:
        gm = res["gemm"]
        ach = gm["flops"] / (gm["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 1), "peak": tflops_peak, "unit": "TFLOP/s",
                "peak_kind": tkind, "frac": round(ach / tflops_peak, 4), "frac_vs_burst": round(ach / tflops_burst, 4),
                "kernel": "odc::gemm::gemm2_kernel (tcgen05 cta_group::2, 256x256 tile per SM pair)",
                "launches": gm["launches"], "ms_per_launch": round(gm["ms"] / gm["launches"], 4),
                "gemm_share_of_step": round(gm["ms"] / res["ms"], 4), "traffic": ncu_traffic("gemm::gemm2_kernel")[0],
                "traffic_source": f"{ncu_traffic('gemm::gemm2_kernel')[1]} (dram read+write per gemm2 launch, "
                                  "averaged over the captured launches)"}
        if gm.get("alg_bytes"):
            roof["algorithmic_bytes_per_launch"] = int(gm["alg_bytes"] / gm["launches"])
            if roof["traffic"]:
                roof["traffic_over_algorithmic"] = round(roof["traffic"] / roof["algorithmic_bytes_per_launch"], 3)
    pred = analytic(lens, plan_odc, plan_fsdp, beta, timed_steps)
    # model FLOPs utilisation of the whole step: per sequence 6*P_nonembed*s (dense)
    # + 6*L*d*s^2 (causal attention, fwd+bwd) + 6*V*d*s (LM head); recompute is not counted
    step_flops = sum(6.0 * shape.nonembed_params * lens[i] + 6.0 * shape.layers * shape.d * float(lens[i]) ** 2
                     + 6.0 * shape.vocab * shape.d * lens[i]
                     for k in timed_steps for dv in plan_odc[k % len(plan_odc)] for mb in dv for i in mb)
    model_tflops = step_flops / (res["ms"] / 1e3) / 1e12
    mfu = {"model_tflops": round(model_tflops, 1), "per_gpu_tflops": round(model_tflops / world, 1),
           "peak_per_gpu": tflops_peak, "frac": round(model_tflops / world / tflops_peak, 4),
           "frac_vs_burst": round(model_tflops / world / tflops_burst, 4),
           "flops": "6*P_nonembed*s + 6*L*d*s^2 + 6*V*d*s per sequence (SURVEY 8(d)); recompute not counted"}
    h2d = sum(16 * lens[i] + 8 + 16 * (shape.heads + shape.kv_heads) * ((lens[i] + 127) // 128)  # + attn work lists
              for k in timed_steps for mb in plan_odc[k % len(plan_odc)][rank] for i in mb)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_step_baseline(args, shape, world, beta, timed_steps)
    if rank == 0:
        line = {"metric": METRIC, "value": round(res["tps"], 1), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms"] / args.steps, 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (random-init weights, seeded random token ids of the workload lengths)",
                "config": sft_config(args, shape, world, beta),
                "recompute_resolved": recompute, "tokens_timed": res["tokens"],
                "idle_fraction": round(res["idle"], 4),
                "idle_note": "1 - sum(busy)/(N*T), busy = device time from step start to the minibatch barrier",
                "vs_fsdp": ({"fsdp_tokens_per_s": round(fs["tps"], 1), "speedup": round(res["tps"] / fs["tps"], 4),
                             "analytic_compute_only_speedup": round(pred[0], 4),
                             "analytic_bubble_odc_lbmini": round(pred[1], 4),
                             "analytic_bubble_fsdp_lbmicro": round(pred[2], 4)} if fs else None),
                "roofline": roof, "mfu": mfu, "fetch_push": comm, "clocks": clk.summary(),
                "e2e": ({"value": round(e2e["tps"], 1), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d / args.steps),
                         "d2h_bytes_per_step": 4, "loss_rank0": e2e["loss"],
                         "note": "token ids/labels/positions built on host per microbatch, staged in pinned host memory and copied H2D (async) inside the "
                                 "timed region; loss read back D2H every step (loss_rank0 = rank 0's token-weighted share of the "
                                 "step's mean loss: ~ln(V) x its token fraction)"} if e2e else None),
                "cpu_baseline": cpu, "gpu_launches": res["launches"]}
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def ncu_traffic(kernel):
    """(dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`,
    source file) from the newest committed ncu capture summary: first the
    capture of this bench's own launch mix (profiles/r02/ncu_traffic_bench.json:
    every gemm2 launch of the first bench steps), else the per-shape capture
    (profiles/r02/ncu_traffic.json), else round 1's."""
    for name in ("r02/ncu_traffic_bench.json", "r02/ncu_traffic.json", "r01/ncu_traffic.json"):
        path = os.path.join(ROOT, "profiles", name)
        try:
            with open(path) as f:
                return json.load(f)["kernels"][kernel]["dram_bytes_per_launch"], os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def comm_rates(eng, M, rank, world, dev, reps=10):
    """fetch / push GB/s of one transformer-layer unit with every rank
    fetching (then pushing) concurrently, CUDA events on the launching stream,
    max over ranks. Bytes: N>1 the NVLink share ((N-1)*block*2 B fetch,
    (N-1)*block*4 B push, per direction); N=1 the local HBM bytes."""
    import torch
    import torch.distributed as dist

    from paper_2601_19362_b200.dist import rank_timings

    out = torch.empty(M, dtype=torch.bfloat16, device=dev)
    grad = torch.full((M,), 1e-6, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    res = {}
    for name, fn in (("fetch", lambda: eng.fetch(1, out)), ("push", lambda: eng.push(1, grad, 1.0))):
        fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if name == "push" and eng.push_mode == "slot":
            # SLOT: a unit's first push of the minibatch is the store into the owners' slots; time
            # those (the untimed minibatch_end between them releases the slots)
            tot = 0.0
            for _ in range(reps):
                eng.minibatch_end()
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize()
                tot += a.elapsed_time(b)
            ms, _, _, _ = rank_timings(tot / reps, 0.0, 0, device=dev)
            eng.minibatch_end()
            torch.cuda.synchronize()
        else:
            a.record(stream)
            for _ in range(reps):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            ms, _, _, _ = rank_timings(a.elapsed_time(b) / reps, 0.0, 0, device=dev)
        block = (M + world - 1) // world
        wire = 8 if eng.push_mode == "fixed" else 4  # FIXED push moves int64 fixed-point values
        if world > 1:
            nbytes = (world - 1) * block * (2 if name == "fetch" else wire)
        else:
            nbytes = M * (4 if name == "fetch" else 4 + 2 * wire)
        res[name + "_GBps"] = round(nbytes / (ms / 1e3) / 1e9, 1)
        res[name + "_us"] = round(ms * 1e3, 1)
    peak = NVLINK_NOMINAL_GBS if world > 1 else peaks()[0]
    res.update({"bytes": ("NVLink per direction" if world > 1 else "local HBM read+write")
                + ("; push counts int64 wire bytes (FIXED mode)" if eng.push_mode == "fixed" else ""), "peak_GBps": peak,
                "fetch_frac": round(res["fetch_GBps"] / peak, 4), "push_frac": round(res["push_GBps"] / peak, 4),
                "unit_elems": M, "all_ranks_concurrent": True})
    return res


def write_trace(path, shape, comm, plan, lens, k, rank, world, dev):
    """One extra (untimed) ODC step with per-layer CUDA-event spans, gathered to
    rank 0 and written in the reference's Chrome-trace schema."""
    import torch
    import torch.distributed as dist

    from paper_2601_19362_b200 import worker as W

    worker = W.Worker(shape, comm, dev)
    worker.tracer = W.Tracer(rank)
    cur = torch.cuda.current_stream()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    worker.tracer.start(cur)
    total = float(sum(lens[i] for dv in plan[k % len(plan)] for mb in dv for i in mb))
    for mb in plan[k % len(plan)][rank]:
        ntok = sum(lens[i] for i in mb)
        worker.microbatch(W.make_batch(lens, mb, shape.vocab, dev, heads=shape.heads, kv_heads=shape.kv_heads), ntok / total)
    worker.tracer.span("barrier", 0, cur, False)
    row = worker.tracer.rows[-1]
    worker.minibatch_end()
    W.Tracer.end(row, cur)
    torch.cuda.synchronize()
    evs = worker.tracer.events()
    allv = [None] * world
    if world > 1:
        dist.all_gather_object(allv, evs)
    else:
        allv = [evs]
    if rank == 0:
        with open(path, "w") as f:
            json.dump(W.chrome_trace(allv), f)
    del worker
    torch.cuda.empty_cache()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def cpu_step_baseline(args, shape, world, beta, steps, budget_s=30.0):
    """cpu_baseline of the GPU arm (rank 0, N=1): the reference's CPU path of
    the same step (RefStepTimer: oracle/_ref ShardFabric<float> over every unit
    at its true size, for every microbatch of the reference LB-Mini plan),
    measured on host cores over a bounded sample of the timed steps (one
    untimed warm-up step, then timed steps while they fit ~budget_s)."""
    from oracle import refbind as R

    if not R.available():
        return None
    lens = ref_lengths(args.cap)
    t0 = time.perf_counter()
    plan = ref_plan(lens, world, args.minibs, args.cap, beta)
    t_plan = time.perf_counter() - t0
    sizes = shape.unit_sizes()
    thr = ref_threads(world, sizes)
    timer = RefStepTimer(world, sizes, thr)
    timer.run(plan[steps[0] % len(plan)])
    secs, toks = [], 0
    for k in steps:
        if secs and sum(secs) + sum(secs) / len(secs) > budget_s:
            break
        st = plan[k % len(plan)]
        secs.append(timer.run(st) + t_plan / len(plan))
        toks += sum(sum(dev) for dev in st)
    timer.close()
    return {"value": round(toks / sum(secs), 2), "unit": "tokens/s", "cores": thr, "kind": "reference",
            "sample": (f"{len(secs)} measured step(s) of the reference CPU path (oracle/_ref ShardFabric<float>, "
                       f"{len(sizes)} units at true size, every microbatch of the reference LB-Mini plan: 2 gathers + "
                       f"1 scatter_accumulate per unit per microbatch, finalize per unit, + plan()); {thr} host threads")}


# ----------------------------------------------------------------- configs[0]
CONFIG0_LENS = [451, 131, 1078, 28, 2048, 77, 27, 63, 76, 119, 89, 601, 435, 90, 712, 264]  # SURVEY 8(c) fixture


def config0_shape():
    """configs[0]: small transformer, d=256, 4 layers, ffn 1024, vocab 1024, tied
    (2 heads of 128: the tcgen05 attention serves head_dim 128)."""
    from paper_2601_19362_b200.shapes import Shape

    return Shape("config0", 256, 1024, 4, 2, 2, 1024, True, True)


def cpu_decoder_loss(shape, units, batch):
    """The decoder of the SFT worker in plain torch fp32 (CPU): RMSNorm, qkv
    (+bias), RoPE, causal SDPA per sequence (GQA), o-proj, SwiGLU MLP, tied LM
    head + CE. Gradients flow into `units` (leaf tensors)."""
    import torch
    import torch.nn.functional as TF

    from paper_2601_19362_b200 import worker as W

    s = shape
    E = W.views(units[0], W.embed_layout(s))
    T = batch.tokens
    h = E["emb"][batch.ids]
    cos, sin = W.rope_tables(batch.positions, s.head_dim)
    cu = batch.cu_seqlens.tolist()
    hd, H, KV = s.head_dim, s.heads, s.kv_heads

    def rms(x, w):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + W.EPS) * w

    def rope(x):
        hh = x.shape[-1] // 2
        x1, x2 = x[..., :hh], x[..., hh:]
        return torch.cat([x1 * cos[:, None] - x2 * sin[:, None], x2 * cos[:, None] + x1 * sin[:, None]], -1)

    for l in range(1, s.layers + 1):
        P = W.views(units[l], W.layer_layout(s))
        qkv = rms(h, P["ln1"]) @ P["qkv_w"].t() + (P["qkv_b"] if s.qkv_bias else 0.0)
        q = rope(qkv[:, :H * hd].view(T, H, hd))
        k = rope(qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd))
        v = qkv[:, (H + KV) * hd:].reshape(T, KV, hd)
        outs = []
        for i in range(len(cu) - 1):
            qs, ks, vs = (t[cu[i]:cu[i + 1]].transpose(0, 1) for t in (q, k, v))
            outs.append(TF.scaled_dot_product_attention(qs[None], ks.repeat_interleave(H // KV, 0)[None],
                                                        vs.repeat_interleave(H // KV, 0)[None],
                                                        is_causal=True)[0].transpose(0, 1))
        h = h + torch.cat(outs, 0).reshape(T, H * hd) @ P["o_w"].t()
        gu = rms(h, P["ln2"]) @ P["gu_w"].t()
        h = h + (TF.silu(gu[:, :s.ffn]) * gu[:, s.ffn:]) @ P["down_w"].t()
    logits = rms(h, E["norm"]) @ (E["emb"] if s.tied else E["head"]).t()
    return TF.cross_entropy(logits, batch.labels, ignore_index=-100)


def run_config0(args, reference: bool):
    """BASELINE configs[0] — the reference's CPU-runnable case: one ODC SFT
    step of the small transformer at world_size 2 on the survey's 16 fixed
    lengths (LB-Mini, minibatch 8 per rank, budget 2,048 tokens, alpha 1, beta 0:
    rank 0 [[4]], rank 1 [[2],[3,6,12,14],[0,1,...]]).
      GPU arm: both ranks in one process on cuda:0 (OdcEngine.local_group: the
        world-2 fetch / push / barrier protocol, FIXED push, AdamW), tcgen05
        worker; a step = both ranks' queues + barrier + AdamW.
      reference arm: the same step on host cores — the model in plain torch fp32
        (cpu_decoder_loss, every core) and the data path through the reference's
        ShardFabric<float> of 2 simulated ranks per unit (oracle/_ref); plan and
        lengths from the reference's plan()."""
    import torch

    from paper_2601_19362_b200 import worker as W

    s = config0_shape()
    sizes = W.unit_sizes(s)
    lens = CONFIG0_LENS
    tokens = sum(lens)
    cfg = {"workload": "config0", "model": "config0 (d256 L4 ffn1024 V1024, 2 heads x 128)", "world": 2,
           "plan": "lb-mini minibs 8 budget 2048 alpha 1 beta 0", "lengths": "SURVEY 8(c) fixture (16 samples)"}
    if reference:
        from oracle import refbind as R

        js = json.loads(R.plan_json("lb-mini", lens, 2, 8, 2048, 1.0, 0.0, 1))
        plan = [[mb["sample_ids"] for mb in dev] for dev in js["steps"][0]["per_device"]]
        torch.set_num_threads(len(os.sched_getaffinity(0)))
        gen = torch.Generator().manual_seed(0)
        units = [W.init_unit(s, u, gen, "cpu").requires_grad_(True) for u in range(len(sizes))]
        timer = RefStepTimer(2, sizes, min(len(sizes), len(os.sched_getaffinity(0))))

        def step():
            t0 = time.perf_counter()
            for dev in plan:
                for mb in dev:
                    b = W.make_batch(lens, mb, s.vocab, "cpu")
                    loss = cpu_decoder_loss(s, units, b) * (sum(lens[i] for i in mb) / tokens)
                    loss.backward()
            for u in units:
                u.grad = None
            return time.perf_counter() - t0 + timer.run(plan)

        for _ in range(args.warmup):
            step()
        secs = [step() for _ in range(args.steps)]
        timer.close()
        tps = tokens * len(secs) / sum(secs)
        line = {"metric": METRIC, "impl": "reference", "value": round(tps, 1), "unit": "tokens/s", "n_gpus": 1,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sum(secs) / len(secs) * 1e3, 3),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": cfg,
                "cpu_baseline": {"value": round(tps, 1), "unit": "tokens/s", "cores": torch.get_num_threads(),
                                 "kind": "port", "sample": "configs[0] step: torch fp32 model on CPU + reference "
                                                           "ShardFabric<float> (2 ranks) per unit, every microbatch"},
                "e2e": {"value": round(tps, 1), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    from paper_2601_19362_b200 import _lib
    from paper_2601_19362_b200 import partition as P
    from paper_2601_19362_b200.engine import OdcEngine

    dev = torch.device("cuda", 0)
    plan = P.plan_flat("lb-mini", lens, 2, 8, 2048, P.CostModel(1.0, 0.0, 1))[0]
    engs = OdcEngine.local_group(sizes, 2, [0], push_mode="fixed")
    gen = torch.Generator(device=dev).manual_seed(0)
    for u in range(len(sizes)):
        full = W.init_unit(s, u, gen, dev)
        for e in engs:
            e.set_params(u, full)
    streams = [torch.cuda.Stream(device=dev) for _ in engs]
    workers = []
    for e, st in zip(engs, streams):
        with torch.cuda.stream(st):
            workers.append(W.Worker(s, W.OdcComm(e), dev, ce_chunk=2048))
    torch.cuda.synchronize()

    def step(host_batches: bool, pre=None):
        losses = []
        for r, (wk, st) in enumerate(zip(workers, streams)):
            with torch.cuda.stream(st):
                for j, mb in enumerate(plan[r]):
                    b = pre[r][j] if pre else W.make_batch(lens, mb, s.vocab, dev, heads=s.heads, kv_heads=s.kv_heads)
                    losses.append(wk.microbatch(b, sum(lens[i] for i in mb) / tokens))
        for wk, st in zip(workers, streams):
            with torch.cuda.stream(st):
                wk.minibatch_end(lr=1e-5)
        return losses

    def timed(host_batches):
        pre = None if host_batches else [[W.make_batch(lens, mb, s.vocab, dev, heads=s.heads, kv_heads=s.kv_heads)
                                          for mb in plan[r]] for r in range(2)]
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in streams]
        for (a, _), st in zip(evs, streams):
            a.record(st)
        n0 = _lib.kernel_launches()
        for _ in range(args.steps):
            losses = step(host_batches, pre)
            if host_batches:
                float(sum(x.item() for x in losses))  # D2H of the step's loss
        for (_, b), st in zip(evs, streams):
            b.record(st)
        torch.cuda.synchronize()
        ms = max(a.elapsed_time(b) for a, b in evs)
        return ms, _lib.kernel_launches() - n0

    for _ in range(args.warmup):
        step(True)
    torch.cuda.synchronize()
    for e in engs:
        e.check()
    ms, launches = timed(False)
    ms_e2e, _ = timed(True)
    for e in engs:
        e.check()
    line = {"metric": METRIC, "value": round(tokens * args.steps / (ms / 1e3), 1), "unit": "tokens/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": cfg, "note": "two ODC ranks in one process on one GPU (world-2 protocol, FIXED push)",
            "e2e": {"value": round(tokens * args.steps / (ms_e2e / 1e3), 1), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(16 * tokens + 8 * 34), "d2h_bytes_per_step": 4 * len(plan[0] + plan[1])},
            "gpu_launches": int(launches)}
    print(json.dumps(line), flush=True)
    for e in engs:
        e.close()


def main():
    args = parse()
    if args.workload == "config0":
        return run_config0(args, reference=args.impl == "reference")
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "sft":
        return run_sft(args)

    import torch
    import torch.distributed as dist

    from paper_2601_19362_b200 import _lib
    from paper_2601_19362_b200.engine import OdcEngine
    from paper_2601_19362_b200.shapes import SHAPES

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    shape = SHAPES[args.model]
    L, M = shape.layers, shape.layer_elems
    lens, steps = rank_plan(world, args.minibs, shape)

    eng = OdcEngine([M] * L, rank=rank, world=world, device=local, push_mode=args.push_mode,
                    fetch_ctas=args.fetch_ctas, push_ctas=args.push_ctas)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    init = torch.empty(M, device=dev)
    for l in range(L):
        init.normal_(0, 0.02, generator=g)
        eng.set_params(l, init)
    del init
    bufs = [torch.empty(M, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    grad = torch.empty(M, dtype=torch.float32, device=dev).normal_(0, 1e-3, generator=g)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    stream = torch.cuda.current_stream()
    kern = {"fetch": [], "push": []}  # (start, end) event pairs on the launching stream

    def one_step(k, timed=False, host=None):
        plan = steps[k % len(steps)][rank]
        tok = [sum(lens[i] for i in mb) for mb in plan]
        total = float(sum(sum(lens[i] for i in mb) for dv in steps[k % len(steps)] for mb in dv))
        for t in tok:
            w = t / total
            for l in range(L):  # forward: fetch every unit
                if timed:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                eng.fetch(l, bufs[l % 2])
                if timed:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(stream)
                    kern["fetch"].append((e0, e1))
                if host is not None:
                    host["fetch"].copy_(bufs[l % 2], non_blocking=True)
            for l in reversed(range(L)):  # backward: re-fetch + push
                eng.fetch(l, bufs[l % 2])
                if host is not None:
                    host["fetch"].copy_(bufs[l % 2], non_blocking=True)
                    grad.copy_(host["grad"], non_blocking=True)
                if timed:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                eng.push(l, grad, w)
                if timed:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(stream)
                    kern["push"].append((e0, e1))
        eng.minibatch_end()
        eng.adam_step(lr=1e-5, weight_decay=0.0)
        return len(tok)

    def timed_region(K, host=None, record=False):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n_before = _lib.kernel_launches()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        micro = 0
        for k in range(K):
            micro += one_step(k, timed=record, host=host)
        b.record(stream)
        torch.cuda.synchronize()
        eng.check()
        ms = a.elapsed_time(b)
        launches = _lib.kernel_launches() - n_before
        if world > 1:
            dist.barrier()
        return ms, micro, launches

    for k in range(args.warmup):
        one_step(k)
    torch.cuda.synchronize()
    eng.check()

    with ClockSampler(local) as clk:
        ms, micro, launches = timed_region(args.steps, record=True)
    bytes_rank = micro * L * M * (2 * P2_BYTES_BF16 + P4_BYTES_F32)
    t = torch.tensor([ms, float(bytes_rank), float(micro), float(launches)], device=dev, dtype=torch.float64)
    if world > 1:
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, bytes_all, micro_all, launches_all = mx[0].item(), sm[1].item(), sm[2].item(), sm[3].item()
    else:
        ms_max, bytes_all, micro_all, launches_all = ms, float(bytes_rank), float(micro), float(launches)
    value = bytes_all / (ms_max / 1e3) / 1e9
    tokens_step = sum(lens[i] for s in range(args.steps) for dv in steps[s % len(steps)] for mb in dv for i in mb)

    # per-kernel durations measured live in the timed region
    def avg_ms(pairs):
        return sum(e0.elapsed_time(e1) for e0, e1 in pairs) / max(1, len(pairs))

    f_ms, p_ms = avg_ms(kern["fetch"]), avg_ms(kern["push"])
    hbm, hbm_kind = peaks()
    if world == 1:
        # local HBM copy: read + write of the whole unit
        f_bytes = M * P2_BYTES_BF16 * 2
        roof = {"bound": "hbm", "achieved": round(f_bytes / (f_ms / 1e3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                "peak_kind": hbm_kind, "kernel": "fetch_tma_kernel (odc_fetch)", "ms_per_launch": round(f_ms, 4),
                "bytes_per_launch": f_bytes, "traffic": None}
    else:
        f_bytes = (world - 1) * ((M + world - 1) // world) * P2_BYTES_BF16  # NVLink ingress per launch
        roof = {"bound": "nvlink", "achieved": round(f_bytes / (f_ms / 1e3) / 1e9, 1), "peak": NVLINK_NOMINAL_GBS,
                "unit": "GB/s", "peak_kind": "nominal per-direction", "kernel": "fetch_tma_kernel (odc_fetch)",
                "ms_per_launch": round(f_ms, 4), "bytes_per_launch": f_bytes, "traffic": None}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    # N=1: read g + read-modify-write of the local fp32 shard (12 B/elem); N>1: NVLink egress
    push_bytes = M * 12 if world == 1 else (world - 1) * ((M + world - 1) // world) * P4_BYTES_F32
    big = (M + world - 1) // world >= (1 << 20)  # engine.cu: bulk reductions from 1M-element shards
    push_kernel = {"red": "push_bulk_kernel<F32>" if big else "push_red_kernel", "fixed": "push_bulk_kernel<FIXED>",
                   "slot": "push_bulk_kernel<F32> (slot store/add at the owner)"}[args.push_mode]
    push_info = {"kernel": push_kernel,
                 "ms_per_launch": round(p_ms, 4), "GBps": round(push_bytes / (p_ms / 1e3) / 1e9, 1)}

    # e2e through host buffers (reference-facing by-value I/O)
    e2e = None
    if not args.no_e2e:
        host = {"fetch": torch.empty(M, dtype=torch.bfloat16, pin_memory=True),
                "grad": torch.empty(M, dtype=torch.float32, pin_memory=True).normal_(0, 1e-3)}
        K2 = 1
        ms2, micro2, _ = timed_region(K2, host=host)
        t2 = torch.tensor([ms2, float(micro2 * L * M * (2 * P2_BYTES_BF16 + P4_BYTES_F32))], device=dev,
                          dtype=torch.float64)
        if world > 1:
            mx2 = t2.clone()
            dist.all_reduce(mx2, op=dist.ReduceOp.MAX)
            sm2 = t2.clone()
            dist.all_reduce(sm2, op=dist.ReduceOp.SUM)
            ms2, b2 = mx2[0].item(), sm2[1].item()
        else:
            b2 = t2[1].item()
        e2e = {"value": round(b2 / (ms2 / 1e3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(micro2 * L * M * P4_BYTES_F32 / K2),
               "d2h_bytes_per_step": int(micro2 * L * M * 2 * P2_BYTES_BF16 / K2),
               "note": "fetched units copied to pinned host, pushed grads from pinned host (by-value API)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s, b, kind, sample = cpu_reference_sample(1, M, 1)
        cpu = {"value": round(b / s / 1e9, 4), "unit": "GB/s", "cores": cpu_threads(M) if kind == "reference" else 1,
               "kind": kind, "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": args.workload, "model": shape.name, "units": L, "unit_elems": M,
                           "plan": "lb-mini", "minibs_per_rank": args.minibs, "budget_tokens": 32768,
                           "lengths": "lognormal(8,1.5) n=2048 cap=32768 seed=0, floor 512",
                           "push_mode": args.push_mode, "parallelism": f"odc{world}",
                           "l2": "inputs > L2 (5.2 GB of units per pass), no flush",
                           "microbatches_all_ranks": int(micro_all), "tokens_in_timed_steps": tokens_step},
                "roofline": roof, "push": push_info, "clocks": clk.summary(), "e2e": e2e,
                "cpu_baseline": cpu, "gpu_launches": int(launches_all)}
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
