"""Exhaustive interleaving check of the engine's device-side epoch protocol
("a host-side model checker, reused from the reference idea, for
the flag/epoch protocol"; the reference's own checker is run_schedule,
/root/reference/proj/include/odcsim/primitives.hpp:242-294).

The model restates csrc/engine.cu's ordering protocol (file header, lines
30-45, odc_ctx::gate / drain_pending, odc_minibatch_end, odc_adam_step) as one
device stream per rank; every reachable interleaving of the ranks is explored
with state hashing. Per rank and minibatch m the host issues: per microbatch
a fetch of the unit (gate: every owner's param_epoch >= adams issued here) and
a push (gate: every owner's drain_epoch >= minibatch_end calls issued here),
then minibatch_end (barrier arrive, barrier wait, then SLOT: rank-order slot
reduce + drain publish; RED: grads pending), then either AdamW (consumes the
grad shard, publishes param_epoch and drain_epoch) or the no-AdamW path
(finalize: read the shard; the next ODC call zeroes it and publishes drain).

Checked in every interleaving: no deadlock (some rank can always move until
all are done); every consumption of an owner's gradient holds exactly the
contributions of that minibatch from every client, each once; every fetch
reads the owner's parameters at exactly the version the caller expects. A
mutated protocol (the push drain gate removed) must be caught.
"""
import itertools
import random

import pytest


def programs(world, counts, adam, mode, fetch=True):
    """Per rank the op list (the host-side epochs are baked into the ops, as the host tracks them).
    fetch=False: push-only microbatches (the engine does not require a fetch before a push)."""
    progs = []
    for r in range(world):
        ops, adams, mbs, pending = [], 0, 0, False
        for m, per_rank in enumerate(counts):
            for k in range(per_rank[r]):
                if pending:  # RED without AdamW: the first ODC call of the minibatch drains
                    ops.append(("drain", mbs))
                    pending = False
                if fetch:
                    ops.append(("fetch", adams))
                ops.append(("push", mbs, (r, m, k), k == 0))
            if pending:
                ops.append(("drain", mbs))
                pending = False
            ops.append(("arrive", m + 1))
            ops.append(("wait", m + 1))
            mbs += 1
            if mode == "slot":
                ops.append(("reduce", m, mbs))
            if adam:
                ops.append(("adam", m, adams + 1, mbs))
                adams += 1
            else:
                ops.append(("consume", m))
                if mode == "red":
                    pending = True
        progs.append(ops)
    return progs


def expected(world, counts, m):
    return frozenset((c, m, k) for c in range(world) for k in range(counts[m][c]))


def check(world, counts, adam, mode, drain_gate=True, fetch=True, max_states=400_000):
    progs = programs(world, counts, adam, mode, fetch)
    N = world
    # state: pcs, param_epoch, version, drain, done, grad (per owner), slot (per owner, client)
    init = (tuple([0] * N), tuple([0] * N), tuple([0] * N), tuple([0] * N), tuple([0] * N),
            tuple(frozenset() for _ in range(N)), tuple(tuple(frozenset() for _ in range(N)) for _ in range(N)))
    seen, stack = {init}, [init]
    while stack:
        st = stack.pop()
        pcs, pe, ver, dr, done, grad, slot = st
        moved = False
        for r in range(N):
            if pcs[r] >= len(progs[r]):
                continue
            op = progs[r][pcs[r]]
            kind = op[0]
            npe, nver, ndr, ndone = list(pe), list(ver), list(dr), list(done)
            ngrad, nslot = list(grad), [list(s) for s in slot]
            if kind == "fetch":
                if not all(pe[o] >= op[1] for o in range(N)):
                    continue
                for o in range(N):  # the parameters read are the version this rank expects
                    assert ver[o] == op[1], (f"rank {r} fetched owner {o} at version {ver[o]}, expected {op[1]}", st)
            elif kind == "push":
                if drain_gate and not all(dr[o] >= op[1] for o in range(N)):
                    continue
                if mode == "red":
                    for o in range(N):
                        assert op[2] not in grad[o]
                        ngrad[o] = grad[o] | {op[2]}
                else:  # SLOT: the first push of the minibatch overwrites this client's slot at every owner
                    for o in range(N):
                        nslot[o][r] = frozenset({op[2]}) if op[3] else slot[o][r] | {op[2]}
            elif kind == "drain":  # RED, no AdamW in between: zero the shard, publish the drain epoch
                ngrad[r] = frozenset()
                ndr[r] = op[1]
            elif kind == "arrive":
                ndone[r] = op[1]
            elif kind == "wait":
                if not all(done[c] >= op[1] for c in range(N)):
                    continue
            elif kind == "reduce":  # SLOT: owner sums every client's slot (rank order), publishes drain
                m = op[1]
                got = frozenset().union(*[slot[r][c] for c in range(N) if counts[m][c] > 0])
                ngrad[r] = got
                ndr[r] = op[2]
            elif kind in ("adam", "consume"):
                m = op[1]
                want = expected(N, counts, m)
                assert grad[r] == want, (f"owner {r} consumed {sorted(grad[r])} for minibatch {m}, "
                                         f"expected {sorted(want)}", st)
                if kind == "adam":
                    ngrad[r] = frozenset()  # AdamW zeroes the shard
                    nver[r] = op[2]
                    npe[r] = op[2]
                    ndr[r] = op[3]
            npcs = list(pcs)
            npcs[r] += 1
            nst = (tuple(npcs), tuple(npe), tuple(nver), tuple(ndr), tuple(ndone), tuple(ngrad),
                   tuple(tuple(s) for s in nslot))
            moved = True
            if nst not in seen:
                seen.add(nst)
                assert len(seen) < max_states, "state space larger than the test budget"
                stack.append(nst)
        if not moved:
            assert all(pcs[r] == len(progs[r]) for r in range(N)), ("deadlock", st)
    return len(seen)


CASES = [
    (2, [(1, 1), (1, 1)]),
    (2, [(2, 0), (0, 2), (1, 1)]),  # a rank with no microbatch in a minibatch
    (3, [(1, 1, 0), (0, 1, 1)]),
    (3, [(1, 0, 1), (1, 1, 1)]),
]


@pytest.mark.parametrize("fetch", [True, False])
@pytest.mark.parametrize("mode", ["red", "slot"])
@pytest.mark.parametrize("adam", [True, False])
@pytest.mark.parametrize("world,counts", CASES)
def test_protocol_every_interleaving(world, counts, adam, mode, fetch):
    n = check(world, counts, adam, mode, fetch=fetch)
    assert n > 10


def test_random_microbatch_counts():
    rng = random.Random(7)
    for _ in range(8):
        world = rng.choice([2, 3, 4])
        counts = [tuple(rng.choice([0, 1, 1, 2]) for _ in range(world)) for _ in range(3)]
        for adam, mode, fetch in itertools.product([True, False], ["red", "slot"], [True, False]):
            check(world, counts, adam, mode, fetch=fetch)


@pytest.mark.parametrize("mode", ["red", "slot"])
@pytest.mark.parametrize("adam,fetch", [(False, True), (True, False), (False, False)])
def test_checker_catches_missing_drain_gate(mode, adam, fetch):
    """Without the push-side drain gate a fast rank pushes minibatch m+1 into a
    target the owner has not consumed yet: the checker must find that. (With
    AdamW and a fetch before every push, the fetch's parameter-epoch gate
    already orders the push after the owner's AdamW: the drain gate is what
    makes push-only callers and the no-AdamW path safe.)"""
    with pytest.raises(AssertionError):
        check(2, [(1, 1), (1, 1)], adam, mode, drain_gate=False, fetch=fetch)
