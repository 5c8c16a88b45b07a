"""Generates the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run here (where /root/reference exists and oracle/_ref is built):

    make -C oracle && python tests/golden/make_golden.py

Every expected value below is produced by the unmodified reference library
(oracle/_ref/libodcref.so, built from /root/reference/proj/src by
oracle/Makefile) through oracle/ref_driver.cpp — never by our code. The
fixtures travel with the repo so the GPU box (which has no /root/reference)
can check the CUDA path against the reference's own outputs.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refbind as R  # noqa: E402

STRATS = ["local-sort", "lb-micro", "lb-mini", "verl-native", "verl-optimized"]


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print(name, os.path.getsize(os.path.join(HERE, name)), "bytes")


def bench_workload(n=2048, cap=32768, floor=512):
    """The BASELINE.md §3 workload: generate_synthetic(lognormal mu=8 sigma=1.5,
    n, cap, seed=0) then floored at 512 (harness-side transform)."""
    raw = R.generate_synthetic(("lognormal", 8.0, 1.5), n, cap, 0)
    return raw, [max(floor, x) for x in raw]


def main():
    assert R.available(), "build oracle/_ref first: make -C oracle"
    rng = np.random.default_rng(20260118)

    # --- workloads (src/workload.cpp:218-271) ---
    wl = []
    for dist in (("lognormal", 8.0, 1.5), ("lognormal", 5.0, 1.0), ("pareto", 100.0, 1.2), ("uniform", 5, 9)):
        for seed in (0, 1, 2, 77):
            for scale in (1.0, 0.0625):
                wl.append({"dist": list(dist), "n": 64, "cap": 32768, "seed": seed, "scale": scale,
                           "lens": R.generate_synthetic(dist, 64, 32768, seed, scale)})
    raw, floored = bench_workload()
    wl.append({"dist": ["lognormal", 8.0, 1.5], "n": 2048, "cap": 32768, "seed": 0, "scale": 1.0, "lens": raw})
    dump("workloads.json", wl)

    # --- plans (src/partition.cpp:490-580 -> src/experiment.cpp:215-233) ---
    plans = []
    survey = R.generate_synthetic(("lognormal", 8.0, 1.5), 16, 32768, 0, 0.0625)
    plans.append({"strategy": "lb-mini", "lens": survey, "devices": 2, "minibs": 8, "budget": 2048, "alpha": 1.0,
                  "beta": 0.0, "seed": 0, "json": R.plan_json("lb-mini", survey, 2, 8, 2048)})
    for D in (1, 2, 4, 8):  # the bench workload, both strategies, realistic beta
        for strat in ("lb-mini", "lb-micro"):
            for beta in (0.0, 30500.0):
                lens = floored[:512]
                plans.append({"strategy": strat, "lens": lens, "devices": D, "minibs": 8, "budget": 32768,
                              "alpha": 1.0, "beta": beta, "seed": 0,
                              "json": R.plan_json(strat, lens, D, 8, 32768, 1.0, beta)})
    for trial in range(240):  # random small cases over every strategy
        n = int(rng.integers(1, 70))
        D = int(rng.choice([1, 2, 3, 4, 8]))
        mb = int(rng.integers(1, 6))
        lens = rng.integers(1, 300, n).tolist()
        budget = max(lens) + int(rng.integers(0, 300))
        strat = STRATS[trial % 5]
        alpha, beta = float(rng.integers(0, 3)), float(rng.integers(1, 200))
        try:
            js = R.plan_json(strat, lens, D, mb, budget, alpha, beta, 1, trial)
            err = 0
        except R.RefError as e:
            js, err = None, e.code
        plans.append({"strategy": strat, "lens": lens, "devices": D, "minibs": mb, "budget": budget, "alpha": alpha,
                      "beta": beta, "seed": trial, "json": js, "error": err})
    dump("plans.json", plans)

    # --- KK (src/partition.cpp:84-128), incl. the reference tests' known answers ---
    kk = []
    known = [([8, 7, 6, 5, 4], 2, False), ([3, 3, 3, 3], 2, True), ([5, 5, 5, 5], 2, False), ([5, 5, 5, 5], 2, True),
             ([9, 4], 4, False), ([5], 1, False), ([64, 4, 4, 4, 4], 2, False), ([6, 5, 4, 3], 2, True)]
    for costs, k, eq in known:
        kk.append({"costs": costs, "k": k, "equal_size": eq, "ref": R.kk_partition(costs, k, eq)})
    for trial in range(200):
        k = int(rng.integers(1, 9))
        n = int(rng.integers(0, 40))
        eq = bool(trial % 3 == 0) and n % k == 0
        costs = rng.integers(1, 10000, n).astype(float).tolist()
        kk.append({"costs": costs, "k": k, "equal_size": eq, "ref": R.kk_partition(costs, k, eq)})
    dump("kk.json", kk)

    # --- fabric scripts (inc/primitives.hpp:167-207): push then finalize ---
    fab = []
    for dt in ("int64", "float64", "float32"):
        for trial in range(40):
            N = int(rng.integers(1, 9))
            M = int(rng.integers(1, 70)) if trial % 4 else int(rng.integers(1, 6))  # incl. M < N (empty shards)
            pushes = []
            for _ in range(int(rng.integers(0, 12))):
                c = int(rng.integers(0, N))
                if dt == "int64":
                    g = rng.integers(-1000, 1001, M).tolist()
                    w = int(rng.integers(0, 5))
                else:
                    g = ((rng.integers(0, 20001, M) - 10000) / 997.0).astype(dt).tolist()
                    w = float(np.asarray(rng.integers(1, 1000) / 250.0, dt))
                pushes.append([c, g, w])
            exp = R.fabric_script(N, M, [(c, np.asarray(g, dt), w) for c, g, w in pushes], np.dtype(dt))
            fab.append({"dtype": dt, "ranks": N, "elems": M, "pushes": pushes, "expected": exp.tolist()})
    dump("fabric_scripts.json", fab)

    # --- push_slice error surface (inc/primitives.hpp:105-112, tests/test_primitives.cpp:108-114) ---
    ps = []
    for N, M, c, t, off, n in [(3, 10, 0, 1, 0, 5), (3, 10, 0, 2, 1, 2), (3, 10, 0, 2, 0, 2), (3, 10, 1, 0, 0, 4),
                               (4, 5, 0, 3, 0, 1), (4, 5, 0, 3, 0, 0), (2, 7, 1, 1, 3, 1), (2, 7, 1, 1, -1, 1)]:
        ps.append({"ranks": N, "elems": M, "client": c, "target": t, "offset": off, "len": n,
                   "status": R.push_slice_status(N, M, c, t, off, n)})
    dump("push_slice.json", ps)

    # --- run_schedule interleavings (inc/primitives.hpp:242-294) ---
    sch = []
    for trial in range(60):
        N = int(rng.integers(2, 6))
        M = int(rng.integers(4, 32))
        pushes = []
        for c in range(N):
            for _ in range(int(rng.integers(0, 5))):
                pushes.append([c, rng.integers(-100, 101, M).tolist(), int(rng.integers(0, 4))])
        seed = int(rng.integers(0, 2**63))
        out, peak = R.run_schedule_i64(N, M, [(c, np.asarray(g), w) for c, g, w in pushes], seed)
        sch.append({"ranks": N, "elems": M, "pushes": pushes, "seed": seed, "expected": out.tolist(), "peak": peak})
    dump("schedules.json", sch)

    bench_plans()


def bench_plans():
    """The EXACT plans bench.py runs: the full 2,048-length workload (floored
    at 512), minibatch 8 per rank, packing ratio 1 (budget = cap), at the
    bench's cost model beta/alpha (paper_2601_19362_b200.shapes
    beta_over_alpha_b200, 26,679.8 for Qwen2.5-1.5B) for every BASELINE model
    and N = 1/2/4/8, both arms (LB-Mini for ODC, LB-Micro for FSDP). Stored as
    the sha256 of the reference's solutions_to_json bytes plus the first step
    in clear (the full dumps are ~0.1-0.3 MB each)."""
    import hashlib

    from paper_2601_19362_b200.shapes import SHAPES  # pure-Python constants (no product code runs)

    out = []
    for name, cap in (("qwen2.5-1.5b", 32768), ("llama-3-8b", 32768), ("qwen2.5-14b", 65536)):
        beta = SHAPES[name].beta_over_alpha_b200()
        _, lens = bench_workload(cap=cap)
        for D in (1, 2, 4, 8):
            for strat in ("lb-mini", "lb-micro"):
                js = R.plan_json(strat, lens, D, 8, cap, 1.0, beta)
                first = json.loads(js)["steps"][0]
                out.append({"model": name, "cap": cap, "strategy": strat, "devices": D, "minibs": 8, "budget": cap,
                            "alpha": 1.0, "beta": beta, "seed": 0, "sha256": hashlib.sha256(js.encode()).hexdigest(),
                            "bytes": len(js), "steps": len(json.loads(js)["steps"]), "first_step": first})
    dump("bench_plans.json", out)


if __name__ == "__main__":
    if sys.argv[1:] == ["bench_plans"]:
        bench_plans()
    else:
        main()
