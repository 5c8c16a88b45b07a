"""Pins the CPU oracle (oracle/odc_oracle.py) before it is trusted.

(a) against the known-answer vectors of the reference's own tests
    (/root/reference/proj/tests/test_partition.cpp, test_primitives.cpp),
    restated here with their file:line;
(b) against golden fixtures produced by the reference library itself
    (tests/golden/make_golden.py -> oracle/_ref);
(c) live against oracle/_ref when it is built (here, and on the GPU box when
    the prebuilt copy travelled with the snapshot).
"""
import numpy as np
import pytest

from conftest import golden
from oracle import odc_oracle as O
from oracle import refbind as R

Q = O.CostModel(1, 0, 1)


def test_mt19937_64_first_output():
    assert O.MT19937_64(5489)() == 14514284786278117030  # first draw of std::mt19937_64 with its default seed
    g = O.MT19937_64(0)
    assert [g() for _ in range(2)] == [2947667278772165694, 18301848765998365067]


def test_kk_known_answers():
    # test_partition.cpp:67-78 — [8,7,6,5,4], k=2: sums {14,16}, spread 2
    r = O.kk_partition([8, 7, 6, 5, 4], 2, False)
    assert sorted(r.sums) == [14, 16] and r.spread == 2.0
    # :90-101 — equal_size [5,5,5,5] -> {{0,3},{1,2}}
    assert O.kk_partition([5, 5, 5, 5], 2, True).parts == [[0, 3], [1, 2]]
    # :106-112 — k > n spreads over empty parts, spread 9
    r = O.kk_partition([9, 4], 4, False)
    assert len(r.parts) == 4 and r.spread == 9.0
    # :166-172 — quadratic [8,2,2,2,2] -> sums {64,16}, spread 48
    r = O.minibatch_partition([8, 2, 2, 2, 2], 2, False, Q)
    assert sorted(r.sums) == [16, 64] and r.spread == 48.0
    with pytest.raises(O.ParamError):
        O.kk_partition([1, 2, 3], 0, False)
    with pytest.raises(O.ParamError):
        O.kk_partition([1, 2, 3], 2, True)


def test_microbatch_known_answers():
    s = list(enumerate([9, 3, 3, 3]))
    assert len(O.microbatch_partition(s, 10, Q)) == 2  # test_partition.cpp:183-196
    with pytest.raises(O.InfeasibleError, match="sample 1"):  # :198-202
        O.microbatch_partition(list(enumerate([4, 12])), 10, Q)
    joint = O.microbatch_partition_joint([[(0, 5)], [(1, 9), (2, 8), (3, 7)]], 10, Q)  # :204-214
    assert [len(j) for j in joint] == [3, 3] and sum(1 for p in joint[0] if p) == 1


def test_lb_mini_known_answers():
    # test_partition.cpp:229-241
    steps, _ = O.plan("lb-mini", [8, 2, 2, 2, 2], 2, 8, 8, Q)
    sol = steps[0]
    assert sol.mode == "variable-micro"
    assert [mb.lengths for mb in sol.per_device[0]] == [[8]]
    assert len(sol.per_device[1]) == 1 and sol.per_device[1][0].token_sum == 8
    # :243-252 — tighter budget, unequal counts
    steps, _ = O.plan("lb-mini", [7, 2, 2, 2, 2], 2, 8, 7, Q)
    assert len(steps[0].per_device[0]) != len(steps[0].per_device[1])
    # SURVEY §8(c) survey fixture
    lens = O.scale_lengths(O.generate_synthetic(("lognormal", 8.0, 1.5), 16, 32768, 0), 0.0625)
    assert lens == [451, 131, 1078, 28, 2048, 77, 27, 63, 76, 119, 89, 601, 435, 90, 712, 264]
    steps, _ = O.plan("lb-mini", lens, 2, 8, 2048, Q)
    assert [mb.sample_ids for mb in steps[0].per_device[0]] == [[4]]
    assert [mb.sample_ids for mb in steps[0].per_device[1]] == [[2], [3, 6, 12, 14], [0, 1, 5, 7, 8, 9, 10, 11, 13, 15]]


def test_fabric_known_answers():
    f = O.ShardFabric(2, 4)  # test_primitives.cpp:38-48
    f.set_params("layer0", [1, 2, 3, 4])
    assert f.gather(1, "layer0").tolist() == [1, 2, 3, 4]
    with pytest.raises(O.StateError):
        f.gather(0, "missing")
    f = O.ShardFabric(2, 4)  # :59-66
    f.scatter_accumulate(0, [1, 1, 1, 1], 1)
    f.scatter_accumulate(0, [1, 1, 1, 1], 1)
    assert [s.tolist() for s in f.finalize_minibatch()] == [[2, 2], [2, 2]]
    f = O.ShardFabric(3, 10)  # :108-114
    with pytest.raises(O.ProtocolError):
        f.push_slice(0, 1, 0, np.ones(5, np.int64), 1)
    with pytest.raises(O.ProtocolError):
        f.push_slice(0, 2, 1, np.ones(2, np.int64), 1)
    f = O.ShardFabric(2, 4)  # :90-97
    f.scatter_accumulate(0, [5, 5, 5, 5], 1)
    assert f.finalize_minibatch()[0].tolist() == [5, 5]
    assert f.finalize_minibatch()[0].tolist() == [0, 0]
    assert [O.shard_range(5, 4, r) for r in range(4)] == [(0, 2), (2, 2), (4, 1), (5, 0)]


def test_oracle_matches_golden_workloads():
    for case in golden("workloads.json"):
        d = tuple(case["dist"])
        lens = O.generate_synthetic(d, case["n"], case["cap"], case["seed"])
        if case["scale"] != 1.0:
            lens = O.scale_lengths(lens, case["scale"])
        assert lens == case["lens"], case["dist"]


def test_oracle_matches_golden_plans():
    for case in golden("plans.json"):
        if len(case["lens"]) > 200:
            continue  # large cases: product-vs-golden only (pure-Python oracle is slow there)
        cm = O.CostModel(case["alpha"], case["beta"], 1)
        if case.get("error"):
            with pytest.raises((O.ParamError, O.InfeasibleError)):
                O.plan(case["strategy"], case["lens"], case["devices"], case["minibs"], case["budget"], cm, case["seed"])
            continue
        st, dr = O.plan(case["strategy"], case["lens"], case["devices"], case["minibs"], case["budget"], cm,
                        case["seed"])
        assert O.solutions_to_json(st, dr) == case["json"]


def test_oracle_matches_golden_kk():
    for case in golden("kk.json"):
        r = O.kk_partition(case["costs"], case["k"], case["equal_size"])
        assert r.parts == case["ref"]["parts"] and r.sums == case["ref"]["sums"] and r.spread == case["ref"]["spread"]


def test_oracle_matches_golden_fabric():
    for case in golden("fabric_scripts.json"):
        dt = np.dtype(case["dtype"])
        f = O.ShardFabric(case["ranks"], case["elems"], dt)
        for c, g, w in case["pushes"]:
            f.scatter_accumulate(c, np.asarray(g, dt), w)
        got = np.concatenate(f.finalize_minibatch())
        assert np.array_equal(got, np.asarray(case["expected"], dt)), case["dtype"]


def test_oracle_matches_golden_schedules():
    for case in golden("schedules.json"):
        scripts = [[] for _ in range(case["ranks"])]
        for c, g, w in case["pushes"]:
            scripts[c].append((np.asarray(g, np.int64), w))
        out, peak = O.run_schedule(case["ranks"], case["elems"], scripts, case["seed"])
        assert out.tolist() == case["expected"] and peak == case["peak"]


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_random_plans():
    rng = np.random.default_rng(5)
    for trial in range(150):
        n = int(rng.integers(1, 60))
        D = int(rng.integers(1, 9))
        mb = int(rng.integers(1, 5))
        lens = rng.integers(1, 500, n).tolist()
        budget = max(lens) + int(rng.integers(0, 400))
        for s in ("lb-mini", "lb-micro", "local-sort"):
            st, dr = O.plan(s, lens, D, mb, budget, Q, trial)
            assert O.solutions_to_json(st, dr) == R.plan_json(s, lens, D, mb, budget, 1.0, 0.0, 1, trial)


def test_fixed_mode_oracle_is_order_independent_and_faithful():
    """FIXED push mode has no reference counterpart; its oracle
    must be order-independent bit for bit and within rel 1e-5 (norm-wise) of
    the float64 sum, like the reference's integer-payload determinism
    (tests/test_primitives.cpp:116-130)."""
    rng = np.random.default_rng(7)
    n = 4099
    pushes = [(c, (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 3, n)).astype(np.float32),
               np.float32(rng.random())) for c in range(6)]
    a = O.fixed_mode_reduce(n, pushes)
    for perm in ([5, 4, 3, 2, 1, 0], [2, 0, 5, 1, 4, 3]):
        assert np.array_equal(O.fixed_mode_reduce(n, [pushes[i] for i in perm]).view(np.int32), a.view(np.int32))
    exact = sum(np.float64(w) * g.astype(np.float64) for _, g, w in pushes)
    assert np.linalg.norm(a - exact) <= 1e-5 * np.linalg.norm(exact)
    # exactly representable values come back exactly
    g = np.array([0.5, -1.25, 3.0, 0.0], np.float32)
    assert O.fixed_mode_reduce(4, [(0, g, np.float32(1.0)), (1, g, np.float32(0.5))]).tolist() == [0.75, -1.875, 4.5, 0.0]
