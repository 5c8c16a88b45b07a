"""Python host mirror of the reference load balancer over libodc.so.

    plan(strategy, lens, devices, minibatch_size, budget, cost, seed)
        src/partition.cpp:490-580 (LB-Mini = "lb-mini" for ODC,
        LB-Micro = "lb-micro" for the FSDP comparison path)
    plan_json(...)      solutions_to_json (src/experiment.cpp:215-233)
    kk_partition(costs, k, equal_size)          src/partition.cpp:84-128
    generate_synthetic(dist, n, cap, seed)      src/workload.cpp:218-230
    token_budget / compute_cost                 src/cost_model.cpp:14-32

The partitioner itself runs in host C++ (csrc/lb.cpp), a bit-exact
restatement of the reference; this module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

from ._lib import check, lib

STRATEGIES = {"local-sort": 0, "lb-micro": 1, "lb-mini": 2, "verl-native": 3, "verl-optimized": 4}


@dataclass
class CostModel:
    alpha: float = 1.0
    beta: float = 0.0
    layers: int = 1


@dataclass
class Microbatch:
    sample_ids: List[int] = field(default_factory=list)
    token_sum: int = 0


@dataclass
class BatchingSolution:
    per_device: List[List[Microbatch]]
    mode: str
    minibatch_size_per_device: int
    step_index: int
    partial: bool


def _i64(a: Sequence[int]):
    arr = np.ascontiguousarray(np.asarray(a, np.int64))
    return arr, arr.ctypes.data_as(C.POINTER(C.c_int64))


def compute_cost(cost: CostModel, s: int) -> float:
    d = float(s)
    return cost.alpha * d * d + cost.beta * d


def token_budget(max_len: int, packing_ratio: float) -> int:
    from .errors import ParamError

    if max_len < 1:
        raise ParamError("token_budget requires max_len >= 1")
    if not packing_ratio >= 1.0:
        raise ParamError("packing ratio must be >= 1 so a single max-length sample fits")
    return int(math.floor(float(max_len) * packing_ratio))


def plan_json(strategy: str, lens: Sequence[int], devices: int, minibatch_size: int, budget: int,
              cost: CostModel = CostModel(), seed: int = 0) -> str:
    arr, p = _i64(lens)
    need = C.c_int64(0)
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        check(lib().odc_plan_json(STRATEGIES[strategy], p, len(arr), devices, minibatch_size, budget, cost.alpha,
                                  cost.beta, cost.layers, seed, buf, cap, C.byref(need)))
        if need.value <= cap:
            return buf.value.decode()
        cap = need.value


def plan(strategy: str, lens: Sequence[int], devices: int, minibatch_size: int, budget: int,
         cost: CostModel = CostModel(), seed: int = 0) -> Tuple[List[BatchingSolution], List[int]]:
    js = json.loads(plan_json(strategy, lens, devices, minibatch_size, budget, cost, seed))
    steps = []
    for st in js["steps"]:
        per_device = [[Microbatch(mb["sample_ids"], mb["token_sum"]) for mb in dev] for dev in st["per_device"]]
        steps.append(BatchingSolution(per_device, st["mode"], st["minibatch_size_per_device"], st["step"],
                                      st["partial"]))
    return steps, js["dropped_ids"]


def plan_flat(strategy: str, lens: Sequence[int], devices: int, minibatch_size: int, budget: int,
              cost: CostModel = CostModel(), seed: int = 0) -> List[List[List[List[int]]]]:
    """steps -> devices -> microbatches -> sample ids (no JSON round trip)."""
    arr, p = _i64(lens)
    need = C.c_int64(0)
    check(lib().odc_plan_flat(STRATEGIES[strategy], p, len(arr), devices, minibatch_size, budget, cost.alpha,
                              cost.beta, seed, None, 0, C.byref(need)))
    out = np.zeros(need.value, np.int64)
    check(lib().odc_plan_flat(STRATEGIES[strategy], p, len(arr), devices, minibatch_size, budget, cost.alpha,
                              cost.beta, seed, out.ctypes.data_as(C.POINTER(C.c_int64)), out.size, C.byref(need)))
    f = out.tolist()
    i = 0

    def nxt():
        nonlocal i
        i += 1
        return f[i - 1]

    steps = []
    for _ in range(nxt()):
        devs = []
        for _ in range(nxt()):
            mbs = []
            for _ in range(nxt()):
                n = nxt()
                mbs.append(f[i:i + n])
                i += n
            devs.append(mbs)
        steps.append(devs)
    return steps


def kk_partition(costs: Sequence[float], k: int, equal_size: bool) -> dict:
    arr = np.ascontiguousarray(np.asarray(costs, np.float64))
    need = C.c_int64(0)
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        check(lib().odc_kk_partition_json(arr.ctypes.data_as(C.POINTER(C.c_double)), len(arr), k, int(equal_size), buf,
                                          cap, C.byref(need)))
        if need.value <= cap:
            return json.loads(buf.value.decode())
        cap = need.value


def generate_synthetic(dist: Tuple, n: int, cap: int, seed: int, scale: float = 1.0) -> List[int]:
    kind = {"lognormal": 0, "pareto": 1, "uniform": 2}[dist[0]]
    out = np.zeros(n, np.int64)
    check(lib().odc_generate_synthetic(kind, float(dist[1]), float(dist[2]), n, cap, seed, scale,
                                       out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out.tolist()


def idle_fraction(busy: Sequence[float], total: float) -> float:
    """src/runtime.cpp:43 bubble formula: 1 - sum(busy) / (D * T)."""
    return 1.0 - sum(busy) / (len(busy) * total)
