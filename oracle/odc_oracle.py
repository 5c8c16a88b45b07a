"""CPU oracle for the ODC hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-Python/numpy restatement of the reference simulator's
algorithms for the path named in BASELINE.json's north_star (shard layout,
fetch = gather, push = scatter_accumulate, minibatch step = finalize, and the
LB-Mini / LB-Micro load balancer). Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it,
and only as the checker. The product (``paper_2601_19362_b200``) never imports
anything under ``oracle/``.

Parity pinning: ``tests/test_oracle_pinned.py`` checks every function here
against (a) the known-answer vectors of the reference's own tests
(``/root/reference/proj/tests/test_primitives.cpp``, ``test_partition.cpp``,
``acceptance_main.cpp``) restated as ``tests/golden/*.json`` fixtures and
(b) the reference library itself, compiled unmodified into ``oracle/_ref``
(see ``oracle/Makefile``) and called through ``oracle/ref_driver.cpp``.

Reference paths below: ``inc/`` = /root/reference/proj/include/odcsim/,
``src/`` = /root/reference/proj/src/.
"""
from __future__ import annotations

import heapq
import json
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

INT_MAX = 2**31 - 1
M64 = (1 << 64) - 1


# --------------------------------------------------------------------------
# error taxonomy: inc/types.hpp:14-48
# --------------------------------------------------------------------------
class ParamError(ValueError):
    pass


class FormatError(ValueError):
    pass


class InfeasibleError(RuntimeError):
    pass


class ModeError(RuntimeError):
    pass


class ProtocolError(RuntimeError):
    pass


class StateError(RuntimeError):
    pass


class InvariantError(AssertionError):
    pass


# --------------------------------------------------------------------------
# std::mt19937_64 (used by src/workload.cpp:222, src/partition.cpp:383-387,
# inc/primitives.hpp:259). Standard MT19937-64 recurrence + tempering.
# --------------------------------------------------------------------------
class MT19937_64:
    NN, MM = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UM = 0xFFFFFFFF80000000
    LM = 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        self.mt = [0] * self.NN
        self.mt[0] = seed & M64
        for i in range(1, self.NN):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & M64
        self.mti = self.NN

    def _twist(self):
        mt, NN, MM, UM, LM, A = self.mt, self.NN, self.MM, self.UM, self.LM, self.MATRIX_A
        for i in range(NN):
            x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM)
            xa = x >> 1
            if x & 1:
                xa ^= A
            mt[i] = mt[(i + MM) % NN] ^ xa
        self.mti = 0

    def __call__(self) -> int:
        if self.mti >= self.NN:
            self._twist()
        x = self.mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & M64


# --------------------------------------------------------------------------
# workload: src/workload.cpp
# --------------------------------------------------------------------------
def _unit_uniform(rng: MT19937_64) -> float:
    # src/workload.cpp:120-122 (top 53 bits * 2^-53)
    return float(rng() >> 11) * (2.0 ** -53)


def _round_half_away(x: float) -> float:
    # std::round semantics (half away from zero) without x+0.5 double rounding.
    r = math.floor(abs(x))
    if abs(x) - r >= 0.5:
        r += 1.0
    return math.copysign(r, x)


def _clamp_length(raw: float, cap: int) -> int:
    # src/workload.cpp:124-130
    if not math.isfinite(raw):
        return cap
    rounded = _round_half_away(raw)
    if rounded < 1.0:
        return 1
    if rounded >= float(cap):
        return cap
    return int(rounded)


def generate_synthetic(dist: Tuple, n: int, cap: int, seed: int) -> List[int]:
    """src/workload.cpp:218-230. dist = ('lognormal', mu, sigma) |
    ('pareto', scale, shape) | ('uniform', lo, hi). Returns lengths; sample i
    has id i."""
    if n < 1:
        raise ParamError("sample count must be >= 1")
    if cap < 1:
        raise ParamError("length cap must be >= 1")
    rng = MT19937_64(seed)
    out = []
    kind = dist[0]
    for _ in range(n):
        if kind == "lognormal":
            mu, sigma = dist[1], dist[2]
            u1 = _unit_uniform(rng)
            u2 = _unit_uniform(rng)
            z = math.sqrt(-2.0 * math.log1p(-u1)) * math.cos(2.0 * math.pi * u2)
            out.append(_clamp_length(math.exp(mu + sigma * z), cap))
        elif kind == "pareto":
            scale, shape = dist[1], dist[2]
            u = _unit_uniform(rng)
            out.append(_clamp_length(scale * math.pow(1.0 - u, -1.0 / shape), cap))
        elif kind == "uniform":
            lo, hi = int(dist[1]), int(dist[2])
            span = (hi - lo) + 1
            out.append(lo + rng() % span)
        else:
            raise FormatError(f"unknown distribution '{kind}'")
    return out


def scale_lengths(lens: Sequence[int], ratio: float) -> List[int]:
    """src/workload.cpp:263-271: max(1, llround(len * ratio))."""
    if not ratio > 0.0:
        raise ParamError("scale ratio must be > 0")
    return [max(1, int(_round_half_away(float(s) * ratio))) for s in lens]


# --------------------------------------------------------------------------
# cost model: src/cost_model.cpp
# --------------------------------------------------------------------------
@dataclass
class CostModel:
    alpha: float = 1.0
    beta: float = 0.0
    layers: int = 1

    def validate(self):
        # src/cost_model.cpp:8-12
        if not (self.alpha >= 0.0) or not (self.beta >= 0.0) or not (self.alpha + self.beta > 0.0):
            raise ParamError("cost model requires alpha >= 0, beta >= 0, alpha + beta > 0")
        if self.layers < 1:
            raise ParamError("cost model requires layers >= 1")


def compute_cost(m: CostModel, s: int) -> float:
    # src/cost_model.cpp:14-18: alpha*d*d + beta*d, evaluated left to right.
    if s < 1:
        raise ParamError("compute_cost requires length >= 1")
    d = float(s)
    return m.alpha * d * d + m.beta * d


def microbatch_cost(m: CostModel, lens: Sequence[int]) -> float:
    if len(lens) == 0:
        raise ParamError("microbatch_cost requires a non-empty microbatch")
    acc = 0.0
    for s in lens:
        acc += compute_cost(m, s)
    return acc


def token_budget(max_len: int, packing_ratio: float) -> int:
    # src/cost_model.cpp:27-32
    if max_len < 1:
        raise ParamError("token_budget requires max_len >= 1")
    if not packing_ratio >= 1.0:
        raise ParamError("packing ratio must be >= 1 so a single max-length sample fits")
    return int(math.floor(float(max_len) * packing_ratio))


def check_oom(lens: Sequence[int], budget: int) -> bool:
    return sum(lens) > budget


# --------------------------------------------------------------------------
# Karmarkar–Karp: src/partition.cpp:14-128
# --------------------------------------------------------------------------
class _Part:
    __slots__ = ("sum", "min_index", "items")

    def __init__(self, s=0.0, mi=INT_MAX, items=None):
        self.sum = s
        self.min_index = mi
        self.items = items if items is not None else []


def _part_key(p: _Part):
    # part_before (src/partition.cpp:21-24): sum desc, then min_index asc
    return (-p.sum, p.min_index)


@dataclass
class PartitionResult:
    parts: List[List[int]]
    sums: List[float]
    spread: float


def kk_partition(costs: Sequence[float], k: int, equal_size: bool) -> PartitionResult:
    """src/partition.cpp:84-128."""
    if k < 1:
        raise ParamError("kk_partition requires k >= 1")
    n = len(costs)
    if equal_size and n % k != 0:
        raise ParamError(f"equal_size requires k to divide the input size ({k} does not divide {n})")
    heap = []  # entries: (-spread, min_index, parts)

    def push(parts, mi):
        spread = parts[0].sum - parts[-1].sum
        heapq.heappush(heap, (-spread, mi, parts))

    if equal_size:
        order = sorted(range(n), key=lambda i: (-costs[i], i))
        for g in range(n // k):
            parts = []
            mi = INT_MAX
            for i in range(k):
                idx = order[g * k + i]
                parts.append(_Part(costs[idx], idx, [idx]))
                mi = min(mi, idx)
            push(parts, mi)
    else:
        for idx in range(n):
            parts = [_Part(costs[idx], idx, [idx])] + [_Part() for _ in range(k - 1)]
            push(parts, idx)
    if not heap:
        return _finish([_Part() for _ in range(k)])
    while len(heap) > 1:
        _, amin, a = heapq.heappop(heap)
        _, bmin, b = heapq.heappop(heap)
        for i in range(k):  # merge_states :41-53
            dst, src = a[i], b[k - 1 - i]
            dst.sum += src.sum
            dst.min_index = min(dst.min_index, src.min_index)
            dst.items.extend(src.items)
        a.sort(key=_part_key)
        push(a, min(amin, bmin))
    return _finish(heap[0][2])


def _finish(parts: List[_Part]) -> PartitionResult:
    # src/partition.cpp:55-70
    lo, hi = math.inf, -math.inf
    out_parts, sums = [], []
    for p in parts:
        out_parts.append(sorted(p.items))
        sums.append(p.sum)
        lo = min(lo, p.sum)
        hi = max(hi, p.sum)
    return PartitionResult(out_parts, sums, (hi - lo) if parts else 0.0)


def minibatch_partition(seqlens: Sequence[int], world_size: int, equal_size: bool,
                        cost: CostModel) -> PartitionResult:
    # src/partition.cpp:223-231
    if world_size < 1:
        raise ParamError("world_size must be >= 1")
    cost.validate()
    return kk_partition([compute_cost(cost, s) for s in seqlens], world_size, equal_size)


# samples are (id, length) tuples
def _parts_fit(parts, samples, budget) -> bool:
    for part in parts:
        lens = [samples[i][1] for i in part]
        if lens and check_oom(lens, budget):
            return False
    return True


def _require_fits_alone(samples, budget):
    for sid, length in samples:
        if length > budget:
            raise InfeasibleError(f"sample {sid} has length {length} exceeding the microbatch "
                                  f"budget of {budget} tokens")


def _kk_parts_for(samples, k, cost):
    return kk_partition([compute_cost(cost, s[1]) for s in samples], k, False).parts


def microbatch_partition(samples, budget: int, cost: CostModel) -> List[List[int]]:
    """src/partition.cpp:266-276: minimal k whose KK split fits the budget."""
    _require_fits_alone(samples, budget)
    n = len(samples)
    k = 1
    while True:
        parts = _kk_parts_for(samples, k, cost)
        if _parts_fit(parts, samples, budget):
            return parts
        if k >= n:
            raise InvariantError("microbatch partition failed at k == n")
        k += 1


def _split_to_k(parts, k, samples, cost):
    # src/partition.cpp:284-320
    parts = [list(p) for p in parts]
    while len(parts) < k:
        best, best_tokens, best_min = -1, -1, INT_MAX
        for p, part in enumerate(parts):
            if len(part) < 2:
                continue
            s = sum(samples[i][1] for i in part)
            mi = min(part)
            if s > best_tokens or (s == best_tokens and mi < best_min):
                best, best_tokens, best_min = p, s, mi
        if best < 0:
            parts.append([])
            continue
        whole = parts[best]
        halves = kk_partition([compute_cost(cost, samples[i][1]) for i in whole], 2, False).parts
        halves = [[whole[j] for j in h] for h in halves]
        parts[best] = halves[0]
        parts.append(halves[1])
    return parts


def microbatch_partition_joint(per_device, budget: int, cost: CostModel):
    # src/partition.cpp:324-348
    solo = []
    k_star = 1
    for dev in per_device:
        solo.append(microbatch_partition(dev, budget, cost))
        k_star = max(k_star, len(solo[-1]))
    out = []
    for d, dev in enumerate(per_device):
        parts = _kk_parts_for(dev, k_star, cost)
        if not _parts_fit(parts, dev, budget):
            parts = _split_to_k(solo[d], k_star, dev, cost)
        out.append(parts)
    return out


@dataclass
class Microbatch:
    sample_ids: List[int] = field(default_factory=list)
    lengths: List[int] = field(default_factory=list)
    token_sum: int = 0


@dataclass
class BatchingSolution:
    per_device: List[List[Microbatch]]
    mode: str  # "equal-micro" | "variable-micro"
    minibatch_size_per_device: int
    step_index: int
    partial: bool


STRATEGIES = ("local-sort", "lb-micro", "lb-mini", "verl-native", "verl-optimized")


def _make_mb(pool, indices) -> Microbatch:
    mb = Microbatch()
    for i in indices:
        sid, length = pool[i]
        mb.sample_ids.append(sid)
        mb.lengths.append(length)
        mb.token_sum += length
    return mb


def _seeded_shuffle(v, rng):
    for i in range(len(v), 1, -1):
        j = rng() % i
        v[i - 1], v[j] = v[j], v[i - 1]


def _from_joint(device_pools, joint, minibs, step, partial):
    per_device = [[_make_mb(device_pools[d], part) for part in joint[d]]
                  for d in range(len(device_pools))]
    return BatchingSolution(per_device, "equal-micro", minibs, step, partial)


def _plan_local_sort(pool, devices, minibs, step, partial):
    # src/partition.cpp:423-447
    srt = sorted(pool, key=lambda s: (-s[1], s[0]))
    per_device = [[] for _ in range(devices)]
    for i, (sid, length) in enumerate(srt):
        per_device[i % devices].append(Microbatch([sid], [length], length))
    mx = max(len(d) for d in per_device)
    for d in per_device:
        while len(d) < mx:
            d.append(Microbatch())
    return BatchingSolution(per_device, "equal-micro", minibs, step, partial)


def _plan_balanced_step(pool, devices, minibs, budget, cost, lb_mini, step, partial):
    # src/partition.cpp:449-486
    equal_size = (not lb_mini) and len(pool) % devices == 0
    split = minibatch_partition([s[1] for s in pool], devices, equal_size, cost)
    device_pools = [[pool[i] for i in part] for part in split.parts]
    if lb_mini:
        per_device = []
        for dev in device_pools:
            mbs = []
            if dev:
                mbs = [_make_mb(dev, part) for part in microbatch_partition(dev, budget, cost)]
            per_device.append(mbs)
        return BatchingSolution(per_device, "variable-micro", minibs, step, partial)
    joint = microbatch_partition_joint(device_pools, budget, cost)
    return _from_joint(device_pools, joint, minibs, step, partial)


def plan(strategy: str, lens: Sequence[int], devices: int, minibatch_size: int, budget: int,
         cost: CostModel, seed: int = 0) -> Tuple[List[BatchingSolution], List[int]]:
    """src/partition.cpp:490-580. Sample i of ``lens`` has id i. Returns
    (steps, dropped_ids)."""
    if devices < 1:
        raise ParamError("devices must be >= 1")
    if minibatch_size < 1:
        raise ParamError("minibatch_size must be >= 1")
    cost.validate()
    if len(lens) == 0:
        raise ParamError("workload must contain at least one sample")
    if budget < max(lens):
        raise InfeasibleError(f"microbatch budget {budget} is below the max sample length {max(lens)}")
    allv = [(i, int(l)) for i, l in enumerate(lens)]
    steps: List[BatchingSolution] = []
    dropped: List[int] = []
    span = devices * minibatch_size
    if strategy == "verl-native":
        keep = len(allv) - len(allv) % devices
        dropped = [s[0] for s in allv[keep:]]
        if keep == 0:
            raise ParamError("workload smaller than the device count")
        kept = allv[:keep]
        split = minibatch_partition([s[1] for s in kept], devices, True, cost)
        rank_pools = []
        for d in range(devices):
            pool = [kept[i] for i in split.parts[d]]
            rng = MT19937_64((seed + 0x9E3779B97F4A7C15 * (d + 1)) & M64)
            _seeded_shuffle(pool, rng)
            rank_pools.append(pool)
        per_rank = len(rank_pools[0])
        nsteps = (per_rank + minibatch_size - 1) // minibatch_size
        for m in range(nsteps):
            dmb, partial = [], False
            for d in range(devices):
                b = m * minibatch_size
                e = min(per_rank, b + minibatch_size)
                partial = partial or (e - b) < minibatch_size
                dmb.append(rank_pools[d][b:e])
            joint = microbatch_partition_joint(dmb, budget, cost)
            steps.append(_from_joint(dmb, joint, minibatch_size, m, partial))
        return steps, dropped
    ordered = list(allv)
    if strategy == "verl-optimized":
        _seeded_shuffle(ordered, MT19937_64(seed))
    step = 0
    for begin in range(0, len(ordered), span):
        pool = ordered[begin:begin + span]
        partial = len(pool) < span
        if strategy == "local-sort":
            steps.append(_plan_local_sort(pool, devices, minibatch_size, step, partial))
        elif strategy in ("lb-micro", "verl-optimized"):
            steps.append(_plan_balanced_step(pool, devices, minibatch_size, budget, cost, False, step, partial))
        elif strategy == "lb-mini":
            steps.append(_plan_balanced_step(pool, devices, minibatch_size, budget, cost, True, step, partial))
        else:
            raise ParamError(f"unknown strategy '{strategy}'")
        step += 1
    return steps, dropped


def solutions_to_json(steps: List[BatchingSolution], dropped: List[int]) -> str:
    """src/experiment.cpp:215-233, serialised like nlohmann::json::dump()
    (object keys sorted, compact separators)."""
    js = []
    for sol in steps:
        devs = [[{"sample_ids": mb.sample_ids, "token_sum": mb.token_sum} for mb in dev]
                for dev in sol.per_device]
        js.append({"step": sol.step_index, "partial": sol.partial, "mode": sol.mode,
                   "minibatch_size_per_device": sol.minibatch_size_per_device,
                   "per_device": devs})
    return json.dumps({"steps": js, "dropped_ids": dropped}, sort_keys=True, separators=(",", ":"))


# --------------------------------------------------------------------------
# analytic runtime: src/runtime.cpp:34-79 (bubble / idle-fraction formula)
# --------------------------------------------------------------------------
def busy_per_device(sol: BatchingSolution, cost: CostModel) -> List[float]:
    busy = []
    for dev in sol.per_device:
        s = 0.0
        for mb in dev:
            s += 0.0 if not mb.sample_ids else microbatch_cost(cost, mb.lengths)
        busy.append(s * float(cost.layers))
    return busy


def bubble_rate(busy: Sequence[float], total: float) -> float:
    # src/runtime.cpp:43: 1 - sum(busy) / (D * T)
    if not total > 0.0:
        raise ParamError("bubble rate undefined for zero total time")
    return 1.0 - sum(busy) / (float(len(busy)) * total)


def runtime_odc(sol: BatchingSolution, cost: CostModel) -> Tuple[float, List[float]]:
    busy = busy_per_device(sol, cost)
    return max(busy), busy


def runtime_collective(sol: BatchingSolution, cost: CostModel) -> Tuple[float, List[float]]:
    if sol.mode != "equal-micro":
        raise ModeError("per-layer collectives require a uniform microbatch count")
    m = len(sol.per_device[0])
    total = 0.0
    for i in range(m):
        worst = 0.0
        for dev in sol.per_device:
            mb = dev[i]
            worst = max(worst, 0.0 if not mb.sample_ids else microbatch_cost(cost, mb.lengths))
        total += worst
    return total * float(cost.layers), busy_per_device(sol, cost)


# --------------------------------------------------------------------------
# ODC primitives: inc/primitives.hpp:21-220
# --------------------------------------------------------------------------
def shard_range(elems: int, ranks: int, r: int) -> Tuple[int, int]:
    """inc/primitives.hpp:39, :53-56. Returns (begin, len)."""
    block = (elems + ranks - 1) // ranks
    b = min(elems, r * block)
    return b, min(elems, (r + 1) * block) - b


class ShardState:
    """inc/primitives.hpp:35-163, numpy-backed. dtype one of int64/float64/float32."""

    def __init__(self, ranks: int, elems: int, dtype=np.int64):
        if ranks < 1 or elems < 1:
            raise ParamError("need ranks >= 1 and elems >= 1")
        self.ranks, self.elems, self.dtype = ranks, elems, np.dtype(dtype)
        self.block = (elems + ranks - 1) // ranks
        self.grad = [np.zeros(self.shard_len(r), self.dtype) for r in range(ranks)]
        self.slots: List[List[Optional[tuple]]] = [[None] * ranks for _ in range(ranks)]
        self.staged = [0] * ranks
        self.max_staged = [0] * ranks
        self.params: Dict[str, List[np.ndarray]] = {}

    def slot_capacity(self):
        return self.block

    def shard_begin(self, r):
        return min(self.elems, r * self.block)

    def shard_len(self, r):
        return min(self.elems, (r + 1) * self.block) - self.shard_begin(r)

    def set_params(self, pid: str, full):
        full = np.asarray(full, self.dtype)
        if full.size != self.elems:
            raise ParamError("parameter vector length mismatch")
        self.params[pid] = [full[self.shard_begin(r):self.shard_begin(r) + self.shard_len(r)].copy()
                            for r in range(self.ranks)]

    def gather(self, client: int, pid: str) -> np.ndarray:
        # :70-77 — concatenation of owners' shards in rank order
        if pid not in self.params:
            raise StateError(f"gather of uninitialized params '{pid}'")
        return np.concatenate(self.params[pid])

    def split_gradient(self, frm: int, grad, w):
        grad = np.asarray(grad, self.dtype)
        if grad.size != self.elems:
            raise ParamError("gradient vector length mismatch")
        return [(frm, r, 0, grad[self.shard_begin(r):self.shard_begin(r) + self.shard_len(r)].copy(),
                 self.dtype.type(w)) for r in range(self.ranks)]

    def slot_free(self, server, client):
        return self.slots[server][client] is None

    def try_stage(self, msg) -> bool:
        frm, tgt, off, payload, w = msg
        if payload.size > self.block:
            raise ProtocolError(f"payload of {payload.size} elements exceeds the per-client "
                                f"buffer slot of {self.block}")
        if off < 0 or off + payload.size > self.shard_len(tgt):
            raise ProtocolError("payload does not fit the target shard")
        if self.slots[tgt][frm] is not None:
            return False
        self.staged[tgt] += payload.size
        self.max_staged[tgt] = max(self.max_staged[tgt], self.staged[tgt])
        self.slots[tgt][frm] = msg
        return True

    def consume(self, server, client) -> bool:
        # :125-136 — shard[off+i] += w * payload[i] (one multiply, one add)
        msg = self.slots[server][client]
        if msg is None:
            return False
        _, _, off, payload, w = msg
        with np.errstate(over="ignore"):
            prod = (w * payload).astype(self.dtype, copy=False)
            seg = self.grad[server][off:off + payload.size]
            seg += prod
        self.staged[server] -= payload.size
        self.slots[server][client] = None
        return True

    def any_staged(self, server):
        return any(s is not None for s in self.slots[server])

    def take_grads(self):
        out = [g.copy() for g in self.grad]
        for g in self.grad:
            g[:] = 0
        return out


class ShardFabric:
    """inc/primitives.hpp:167-207 (immediate mode)."""

    def __init__(self, ranks: int, elems: int, dtype=np.int64):
        self.st = ShardState(ranks, elems, dtype)

    def set_params(self, pid, full):
        self.st.set_params(pid, full)

    def gather(self, client, pid):
        return self.st.gather(client, pid)

    def scatter_accumulate(self, client, grad, w):
        for msg in self.st.split_gradient(client, grad, w):
            tgt = msg[1]
            while not self.st.slot_free(tgt, client):
                self.st.consume(tgt, client)
            if not self.st.try_stage(msg):
                raise InvariantError("stage into a free slot failed")

    def push_slice(self, client, target, offset, payload, w):
        while not self.st.slot_free(target, client):
            self.st.consume(target, client)
        self.st.try_stage((client, target, offset, np.asarray(payload, self.st.dtype),
                           self.st.dtype.type(w)))

    def finalize_minibatch(self):
        for s in range(self.st.ranks):
            for c in range(self.st.ranks):
                self.st.consume(s, c)
        return self.st.take_grads()


def collective_reduce_reference(grads):
    """inc/primitives.hpp:210-220: sum of w*g in input order."""
    if not grads:
        raise ParamError("collective_reduce_reference needs at least one gradient")
    g0 = np.asarray(grads[0][0])
    acc = np.zeros_like(g0)
    for g, w in grads:
        g = np.asarray(g, acc.dtype)
        if g.size != acc.size:
            raise ParamError("gradient length mismatch")
        with np.errstate(over="ignore"):
            acc += (acc.dtype.type(w) * g).astype(acc.dtype, copy=False)
    return acc


def run_schedule(ranks, elems, scripts, seed, dtype=np.int64):
    """inc/primitives.hpp:242-294: one seeded random interleaving of client
    stages and owner consumes. scripts[c] = list of (grad, weight)."""
    st = ShardState(ranks, elems, dtype)
    pending = []
    for c, sc in enumerate(scripts):
        q = []
        for g, w in sc:
            q.extend(st.split_gradient(c, g, w))
        pending.append([q, 0])
    rng = MT19937_64(seed)
    while True:
        enabled = []
        for c, (q, nxt) in enumerate(pending):
            if nxt < len(q) and st.slot_free(q[nxt][1], c):
                enabled.append((True, c, 0))
        for s in range(ranks):
            for c in range(ranks):
                if not st.slot_free(s, c):
                    enabled.append((False, s, c))
        if not enabled:
            break
        is_stage, a, b = enabled[rng() % len(enabled)]
        if is_stage:
            q, nxt = pending[a]
            if not st.try_stage(q[nxt]):
                raise InvariantError("stage of an enabled action failed")
            pending[a][1] += 1
        else:
            st.consume(a, b)
    peak = max(st.max_staged)
    return np.concatenate(st.take_grads()), peak


# --------------------------------------------------------------------------
# Deterministic push (slot mode) restated at the granularity the B200 build
# computes it: per-client sums in push order, then owner reduce in rank order
# ("Accumulation order").
# --------------------------------------------------------------------------
def slot_mode_reduce(ranks: int, elems: int, pushes, dtype=np.float32) -> np.ndarray:
    """pushes = list of (client, grad, weight) in issue order."""
    dt = np.dtype(dtype)
    slots = np.zeros((ranks, elems), dt)
    with np.errstate(over="ignore"):
        for c, g, w in pushes:
            slots[c] += (dt.type(w) * np.asarray(g, dt)).astype(dt, copy=False)
        acc = np.zeros(elems, dt)
        for c in range(ranks):
            acc += slots[c]
    return acc


def fixed_mode_reduce(elems: int, pushes, frac_bits: int = 40) -> np.ndarray:
    """FIXED push mode (no reference counterpart: the reference's
    determinism comes from integer payloads, inc/primitives.hpp:130-131 with
    T = int64, tests/test_primitives.cpp:116-130). Each push adds
    q = round_half_even(fl32(w * g) * 2^S) into an int64 accumulator; the
    result is fl32(sum) * 2^-S. Independent of push order, client and world
    size. pushes = list of (client, grad, weight)."""
    acc = np.zeros(elems, np.int64)
    scale = np.float32(2.0 ** frac_bits)
    lim = np.float32(2.0 ** 63)
    with np.errstate(over="ignore", invalid="ignore"):
        for _, g, w in pushes:
            v = (np.float32(w) * np.asarray(g, np.float32)).astype(np.float32) * scale  # exact power-of-2 scaling
            v = np.nan_to_num(v, nan=0.0)
            q = np.where(v >= lim, np.iinfo(np.int64).max,
                         np.where(v < -lim, np.iinfo(np.int64).min, np.rint(np.clip(v, -lim, lim)).astype(np.int64)))
            acc += q  # int64 wraps like the device's add.u64
    return acc.astype(np.float32) * np.float32(2.0 ** -frac_bits)


def adamw_reference(p, g, m, v, step, lr, beta1, beta2, eps, wd):
    """fp32 AdamW, torch.optim.AdamW(foreach=False) semantics (no reference
    counterpart in odcsim: parity unpinned by the reference)."""
    p = p.astype(np.float32).copy()
    p *= np.float32(1.0 - lr * wd)
    m = np.float32(beta1) * m + np.float32(1.0 - beta1) * g
    v = np.float32(beta2) * v + np.float32(1.0 - beta2) * g * g
    bc1 = 1.0 - beta1 ** step
    bc2 = 1.0 - beta2 ** step
    denom = np.sqrt(v) / np.float32(math.sqrt(bc2)) + np.float32(eps)
    p -= np.float32(lr / bc1) * m / denom
    return p, m, v
