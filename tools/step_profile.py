"""Kernel-time breakdown of one SFT step at N=1 via torch.profiler (CUPTI
activity tracing, no kernel replay): share of device time per kernel family."""
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2601_19362_b200 import partition as P  # noqa: E402
from paper_2601_19362_b200 import worker as W  # noqa: E402
from paper_2601_19362_b200.engine import OdcEngine  # noqa: E402
from paper_2601_19362_b200.shapes import SHAPES  # noqa: E402

shape = SHAPES[os.environ.get("MODEL", "qwen2.5-1.5b")]
dev = torch.device("cuda", 0)
sizes = W.unit_sizes(shape)
lens = [max(512, x) for x in P.generate_synthetic(("lognormal", 8.0, 1.5), 2048, 32768, 0)]
plan = P.plan_flat("lb-mini", lens, 1, 8, 32768, P.CostModel(1.0, shape.beta_over_alpha_b200(), 1))
eng = OdcEngine(sizes)
gen = torch.Generator(device=dev).manual_seed(0)
for u in range(len(sizes)):
    eng.set_params(u, W.init_unit(shape, u, gen, dev))
wk = W.Worker(shape, W.OdcComm(eng), dev)


def step(k):
    tot = float(sum(lens[i] for dv in plan[k] for mb in dv for i in mb))
    for mb in plan[k][0]:
        wk.microbatch(W.make_batch(lens, mb, shape.vocab, dev, heads=shape.heads, kv_heads=shape.kv_heads), sum(lens[i] for i in mb) / tot)
    wk.minibatch_end()


step(0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
step(1)
b.record()
torch.cuda.synchronize()
print(f"step wall (device events) {a.elapsed_time(b):.1f} ms")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    step(1)
    torch.cuda.synchronize()
agg = defaultdict(float)
cnt = defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:80]] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name[:80]] += 1
tot = sum(agg.values())
print(f"total device time {tot / 1e3:.1f} ms; tokens {sum(lens[i] for dv in plan[1] for mb in dv for i in mb)}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:25]:
    print(f"{v / tot * 100:5.1f}%  {v / 1e3:8.2f} ms  n={cnt[k]:5d}  {k}")

# Idle gaps on the device: union of all kernel intervals (every stream) vs the
# profiled span; the largest gaps with the kernels either side of them.
iv = sorted((e.time_range.start, e.time_range.end, e.name[:60]) for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA)
if iv:
    span = iv[-1][1] - iv[0][0]
    busy, cur_s, cur_e, last = 0.0, iv[0][0], iv[0][1], iv[0][2]
    gaps = []
    for s, e, n in iv[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, last, n))
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
        if e >= cur_e:
            last = n
    busy += cur_e - cur_s
    print(f"device span {span / 1e3:.1f} ms, busy (union) {busy / 1e3:.1f} ms, idle {(span - busy) / 1e3:.1f} ms "
          f"in {len(gaps)} gaps")
    hist = defaultdict(float)
    for g, a_, b_ in gaps:
        hist[(a_[:40], b_[:40])] += g
    for (a_, b_), g in sorted(hist.items(), key=lambda x: -x[1])[:12]:
        print(f"  {g / 1e3:7.2f} ms  after {a_!r} before {b_!r}")
