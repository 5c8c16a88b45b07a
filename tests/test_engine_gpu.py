"""GPU parity of the production engine (odc_ctx_t) at world=1 on one B200:
fetch / push (RED and SLOT) / push_slice / minibatch barrier / fused AdamW,
against the CPU oracle (and torch.optim.AdamW for the optimizer, which has no
reference counterpart — parity for it is unpinned by the reference).

Tolerances: fetch and slot-mode gradients are bit-exact (integer-like data
path and a fixed-order fp32 sum); AdamW within rel 1e-5 of torch fp32."""
import numpy as np
import pytest
import torch

from oracle import odc_oracle as O
from paper_2601_19362_b200 import _lib
from paper_2601_19362_b200 import errors as E
from paper_2601_19362_b200.engine import OdcEngine

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
SIZES = [1, 3, 8, 1001, 65536 + 5, 3_000_017]


def _bf16_bits(x: torch.Tensor):
    return x.view(torch.int16).cpu().numpy()


@pytest.mark.parametrize("mode", ["red", "slot", "fixed"])
def test_set_params_fetch_roundtrip(mode):
    eng = OdcEngine(SIZES, push_mode=mode)
    g = torch.Generator(device="cpu").manual_seed(0)
    fulls = [torch.randn(n, generator=g).to(DEV) for n in SIZES]
    for l, f in enumerate(fulls):
        eng.set_params(l, f)
    for l, f in enumerate(fulls):
        out = torch.empty(SIZES[l], dtype=torch.bfloat16, device=DEV)
        eng.fetch(l, out)
        m = torch.empty(SIZES[l], dtype=torch.float32, device=DEV)
        eng.fetch_master(l, m)
        torch.cuda.synchronize()
        assert np.array_equal(_bf16_bits(out), _bf16_bits(f.to(torch.bfloat16)))
        assert torch.equal(m, f)
    eng.check()


@pytest.mark.parametrize("mode", ["red", "slot"])
@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
def test_push_accumulates_like_oracle(mode, gdt):
    eng = OdcEngine(SIZES, push_mode=mode)
    rng = np.random.default_rng(3)
    for l, n in enumerate(SIZES):
        eng.set_params(l, torch.zeros(n, device=DEV))
    pushes = {l: [] for l in range(len(SIZES))}
    for _ in range(3):  # three microbatches
        for l, n in enumerate(SIZES):
            g = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(DEV).to(gdt)
            w = float(np.float32(rng.random()))
            eng.push(l, g, w)
            pushes[l].append((0, g.float().cpu().numpy(), np.float32(w)))
    eng.minibatch_end()
    eng.check()
    for l, n in enumerate(SIZES):
        want = O.slot_mode_reduce(1, n, pushes[l], np.float32)
        got = eng.read_grad_shard(l).cpu().numpy()
        if mode == "slot":
            assert np.array_equal(got, want)
        else:  # one client: red adds happen in push order too; FTZ is the only difference
            assert np.allclose(got, want, rtol=1e-6, atol=1e-30)
    assert eng.epoch == 1


def test_push_slice_protocol_errors_and_values():
    eng = OdcEngine([10], push_mode="red")
    with pytest.raises(E.ProtocolError):
        eng.push_slice(0, 0, 0, torch.ones(11, device=DEV), 1.0)
    with pytest.raises(E.ProtocolError):
        eng.push_slice(0, 0, 5, torch.ones(6, device=DEV), 1.0)
    eng.push_slice(0, 0, 2, torch.full((3,), 2.0, device=DEV), 0.5)
    eng.minibatch_end()
    assert eng.read_grad_shard(0).cpu().tolist() == [0, 0, 1, 1, 1, 0, 0, 0, 0, 0]


@pytest.mark.parametrize("mode", ["red", "slot", "fixed"])
def test_adam_matches_torch_adamw(mode):
    sizes = [1001, 65536 + 3, 8]
    eng = OdcEngine(sizes, push_mode=mode)
    torch.manual_seed(0)
    params = [torch.randn(n, device=DEV) for n in sizes]
    ref = [p.clone().requires_grad_(True) for p in params]
    opt = torch.optim.AdamW(ref, lr=1e-2, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1, foreach=False)
    for l, p in enumerate(params):
        eng.set_params(l, p)
    for step in range(1, 4):
        grads = [torch.randn(n, device=DEV) for n in sizes]
        for l, g in enumerate(grads):
            eng.push(l, g, 1.0)
            ref[l].grad = g.clone()
            if mode == "fixed":  # the optimizer sees the fixed-point-rounded gradient
                ref[l].grad = torch.from_numpy(O.fixed_mode_reduce(g.numel(), [(0, g.cpu().numpy(), 1.0)])).to(DEV)
        eng.minibatch_end()
        eng.adam_step(lr=1e-2, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
        opt.step()
        eng.check()
        for l, n in enumerate(sizes):
            got = eng.read_master_shard(l)
            assert torch.allclose(got, ref[l].detach(), rtol=1e-5, atol=1e-6), (step, l)
            out = torch.empty(n, dtype=torch.bfloat16, device=DEV)
            eng.fetch(l, out)  # gated on the published parameter epoch
            torch.cuda.synchronize()
            assert torch.equal(out, got.to(torch.bfloat16))
            assert not eng.read_grad_shard(l).any()  # grads zeroed for the next minibatch


@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
def test_fixed_push_is_order_independent_and_matches_oracle(gdt):
    """FIXED mode: the owner's sum is the same bits whatever the
    push order, and equals the oracle's int64 fixed-point sum exactly."""
    rng = np.random.default_rng(11)
    pushes = {l: [] for l in range(len(SIZES))}
    for k in range(4):
        for l, n in enumerate(SIZES):
            g = (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 3, n)).astype(np.float32)
            g = torch.from_numpy(g).to(gdt).float().numpy()  # what a bf16 push carries
            pushes[l].append((0, g, np.float32(rng.random())))
    results = []
    for order in (lambda p: p, lambda p: p[::-1], lambda p: [p[2], p[0], p[3], p[1]]):
        eng = OdcEngine(SIZES, push_mode="fixed")
        for l, n in enumerate(SIZES):
            eng.set_params(l, torch.zeros(n, device=DEV))
        for l in range(len(SIZES)):
            for _, g, w in order(pushes[l]):
                eng.push(l, torch.from_numpy(g).to(DEV).to(gdt), float(w))
        eng.minibatch_end()
        eng.check()
        results.append([eng.read_grad_shard(l).cpu().numpy() for l in range(len(SIZES))])
        eng.close()
    for l, n in enumerate(SIZES):
        want = O.fixed_mode_reduce(n, pushes[l])
        for r in results:
            assert np.array_equal(r[l].view(np.int32), want.view(np.int32)), l
        # and it is a faithful fp32 sum: rel 1e-5 of the float64 sum (norm-wise)
        exact = sum(np.float64(w) * g.astype(np.float64) for _, g, w in pushes[l])
        assert np.linalg.norm(want - exact) <= 1e-5 * np.linalg.norm(exact) + 1e-9


def test_fixed_push_slice_and_second_minibatch():
    eng = OdcEngine([10, 7], push_mode="fixed")
    with pytest.raises(E.ProtocolError):
        eng.push_slice(0, 0, 5, torch.ones(6, device=DEV), 1.0)
    eng.push_slice(0, 0, 3, torch.full((3,), 2.0, device=DEV), 0.5)  # odd offset: unaligned path
    eng.push(1, torch.arange(7, dtype=torch.float32, device=DEV), 0.25)
    eng.minibatch_end()
    assert eng.read_grad_shard(0).cpu().tolist() == [0, 0, 0, 1, 1, 1, 0, 0, 0, 0]
    assert eng.read_grad_shard(1).cpu().tolist() == [0, 0.25, 0.5, 0.75, 1.0, 1.25, 1.5]
    # no AdamW in between: the accumulators were drained at the barrier
    eng.push(1, torch.ones(7, device=DEV), 1.0)
    eng.minibatch_end()
    eng.check()
    assert eng.read_grad_shard(1).cpu().tolist() == [1.0] * 7
    assert eng.read_grad_shard(0).cpu().tolist() == [0.0] * 10


def test_full_size_unit_roundtrip_and_accumulate():
    M = 46_797_824  # one Qwen2.5-1.5B FSDP unit
    eng = OdcEngine([M], push_mode="red")
    x = torch.arange(M, device=DEV, dtype=torch.float32) % 251 - 125
    eng.set_params(0, x)
    out = torch.empty(M, dtype=torch.bfloat16, device=DEV)
    eng.fetch(0, out)
    assert torch.equal(out, x.to(torch.bfloat16))
    for _ in range(4):  # integer-valued fp32 grads: order-independent, exact
        eng.push(0, x, 1.0)
    eng.minibatch_end()
    assert torch.equal(eng.read_grad_shard(0), 4 * x)


def test_kernel_launch_counter_moves():
    n0 = _lib.kernel_launches()
    eng = OdcEngine([1024])
    eng.set_params(0, torch.ones(1024, device=DEV))
    eng.fetch(0, torch.empty(1024, dtype=torch.bfloat16, device=DEV))
    eng.check()
    assert _lib.kernel_launches() >= n0 + 2


@pytest.mark.parametrize("mode", ["red", "slot", "fixed"])
def test_two_minibatches_without_adam(mode):
    """finalize_minibatch returns AND zeroes (inc/primitives.hpp:144-148): a
    second minibatch with no AdamW in between must see only its own pushes
    (RED: the owner drains its grad shard at its next ODC call; SLOT: the
    first push of a unit reassigns the slot once the owner's reduce is done)."""
    sizes = [1001, 65536 + 5]
    eng = OdcEngine(sizes, push_mode=mode)
    for l, n in enumerate(sizes):
        eng.set_params(l, torch.zeros(n, device=DEV))
    rng = np.random.default_rng(11)
    for mb in range(3):
        gs = [rng.integers(-8, 8, n).astype(np.float32) for n in sizes]  # exact in every mode
        for l, g in enumerate(gs):
            eng.push(l, torch.from_numpy(g).to(DEV), 0.5)
        eng.minibatch_end()
        for l, g in enumerate(gs):
            got = eng.read_grad_shard(l).cpu().numpy()
            assert np.array_equal(got, 0.5 * g), (mode, mb, l)
        eng.check()
    # a minibatch with no push at all returns zeros
    eng.minibatch_end()
    for l in range(len(sizes)):
        assert not eng.read_grad_shard(l).cpu().numpy().any(), (mode, l)
    eng.check()
    eng.close()


def test_fixed_push_range_error_and_underflow_flag():
    """FIXED push: a contribution that saturates the int64 fixed-point range
    (or is NaN) raises RangeError at the next check; a nonzero contribution
    below the resolution only sets the underflow flag."""
    eng = OdcEngine([4096], push_mode="fixed")
    eng.set_params(0, torch.zeros(4096, device=DEV))
    g = torch.full((4096,), 1e-20, device=DEV)  # < 2^-41: rounds to 0
    eng.push(0, g, 1.0)
    eng.minibatch_end()
    assert eng.flags() == _lib.ODC_FLAG_FIXED_UNDERFLOW
    eng.check()  # underflow is not an error
    assert not eng.read_grad_shard(0).cpu().numpy().any()
    eng.close()
    for bad in (float(2 ** 16), float("nan")):  # 2^16 * 2^40 = 2^56 >= 2^55
        eng = OdcEngine([4096], push_mode="fixed")
        eng.set_params(0, torch.zeros(4096, device=DEV))
        g = torch.zeros(4096, device=DEV)
        g[1234] = bad
        eng.push(0, g, 1.0)
        eng.minibatch_end()
        assert eng.flags() & _lib.ODC_FLAG_FIXED_RANGE
        with pytest.raises(E.RangeError):
            eng.check()
        eng.close()


def test_api_calls_restore_the_callers_device():
    """Every C-ABI call makes its context's device current only for the call:
    the caller's current device is unchanged afterwards (several contexts on
    several devices can be driven from one thread without stray cudaSetDevice)."""
    n = torch.cuda.device_count()
    other = n - 1
    torch.cuda.set_device(0)
    eng = OdcEngine([1000], device=other)
    eng.set_params(0, torch.randn(1000, device=f"cuda:{other}"))
    out = torch.empty(1000, dtype=torch.bfloat16, device=f"cuda:{other}")
    eng.fetch(0, out)
    eng.check()
    assert torch.cuda.current_device() == 0
    eng.close()
    assert torch.cuda.current_device() == 0
