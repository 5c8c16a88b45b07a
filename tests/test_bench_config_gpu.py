"""Parity at the benchmarked configuration (BASELINE configs[2]-[4]).

bench.py runs Qwen2.5-1.5B on 32,768-token microbatches holding sequences up
to 32K long (configs[4]: Qwen2.5-14B up to 64K, deterministic push). These
tests run the same kernels at those shapes against fp32 torch references that
scale to them (tests/bigref.py: attention chunked over query blocks, LM head +
CE chunked and recomputed):

  * tcgen05 attention fwd + bwd on single 32,768- and 65,536-token sequences
    at H/KV = 12/2 (Qwen2.5-1.5B) and 40/8 (Qwen2.5-14B), and on a packed
    32,768-token microbatch of the bench plan;
  * every dense GEMM of the 1.5B layer at T = 32,768 (fwd, dgrad, wgrad) and
    the LM head + CE at [8,192 x 151,936];
  * one full Qwen2.5-1.5B decoder layer + embedding/LM head, forward and
    backward through the ODC engine, on one 32,768-token sequence;
  * a 2-layer Llama-3-8B-shape step with selective recompute;
  * a Qwen2.5-14B-shape layer at 64K tokens with the FIXED (deterministic)
    push and full recompute, and the FIXED push's order independence at the
    14B unit size (bitwise, against the oracle's int64 sum).

Tolerances (bf16 compute, fp32 accumulate vs fp32): attention out rel-L2
< 1e-2, lse abs < 2e-3, dq/dk/dv rel-L2 < 2e-2; GEMM bf16 outputs rel-L2
< 1e-2, fp32 wgrad rel-L2 < 2e-3; model loss rel < 1e-2 and every unit's
gradient cosine > 0.995 / rel-L2 < 5e-2 (the bar of tests/test_worker_gpu.py).
"""
import math

import pytest
import torch

from bigref import attn_bwd_ref, attn_fwd_ref, cosine, ref_loss, rel_l2
from paper_2601_19362_b200 import fused as F
from paper_2601_19362_b200 import gemm as G
from paper_2601_19362_b200 import worker as W
from paper_2601_19362_b200.engine import OdcEngine
from paper_2601_19362_b200.shapes import QWEN25_1_5B, LLAMA3_8B, QWEN25_14B, Shape

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]
DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _fp32_exact():
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32 = prev
    torch.cuda.empty_cache()


def _bench_packed_microbatch():
    """The bench plan's (N=1) first microbatch that packs several samples."""
    from paper_2601_19362_b200 import partition as P

    lens = [max(512, x) for x in P.generate_synthetic(("lognormal", 8.0, 1.5), 2048, 32768, 0)]
    plan = P.plan_flat("lb-mini", lens, 1, 8, 32768, P.CostModel(1.0, QWEN25_1_5B.beta_over_alpha_b200(), 1))
    for step in plan:
        for mb in step[0]:
            if len(mb) >= 3 and sum(lens[i] for i in mb) > 16384:
                return [lens[i] for i in mb]
    raise AssertionError("no packed microbatch in the bench plan")


@pytest.mark.parametrize("lens,H,KV", [([32768], 12, 2), ([65536], 12, 2), ([32768], 40, 8), ([65536], 40, 8),
                                       ("bench", 12, 2)])
def test_attention_long_sequences(lens, H, KV):
    if lens == "bench":
        lens = _bench_packed_microbatch()
    torch.manual_seed(7)
    T = sum(lens)
    q = torch.randn(T, H, 128, device=DEV).to(torch.bfloat16)
    k = torch.randn(T, KV, 128, device=DEV).to(torch.bfloat16)
    v = torch.randn(T, KV, 128, device=DEV).to(torch.bfloat16)
    do = torch.randn(T, H, 128, device=DEV).to(torch.bfloat16)
    scale = 128 ** -0.5
    out, lse = F.attn_fwd(q, k, v, F.attn_items(lens, H, DEV), scale)
    ro, rl = attn_fwd_ref(q, k, v, lens, scale)
    assert rel_l2(out, ro) < 1e-2, rel_l2(out, ro)
    assert (lse - rl).abs().max().item() < 2e-3, (lse - rl).abs().max().item()
    del ro
    dq, dk, dv = F.attn_bwd(q, k, v, out, do, lse, F.attn_bwd_items(lens, H, KV, DEV), scale)
    rq, rk, rv = attn_bwd_ref(q, k, v, out, do, rl, lens, scale)
    for name, got, want in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv)):
        assert rel_l2(got, want) < 2e-2, (name, rel_l2(got, want))
        assert cosine(got, want) > 0.9995, (name, cosine(got, want))


def _r(*s, scale=0.5):
    return (torch.randn(*s, device=DEV) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("name,inn,out", [("qkv", 1536, 2048), ("o", 1536, 1536), ("gate_up", 1536, 17920),
                                          ("down", 8960, 1536)])
def test_layer_gemms_at_32k_tokens(name, inn, out):
    T = 32768
    torch.manual_seed(len(name) * 7 + inn)
    x, w, dy = _r(T, inn), _r(out, inn, scale=0.02), _r(T, out)
    y = G.linear_fwd(x, w)
    assert rel_l2(y, x.float() @ w.float().t()) < 1e-2
    dx = G.linear_dgrad(dy, w)
    assert rel_l2(dx, dy.float() @ w.float()) < 1e-2
    dw = G.linear_wgrad(dy, x)
    assert rel_l2(dw, dy.float().t() @ x.float()) < 2e-3


def test_lm_head_and_ce_at_full_vocab():
    """[8,192 x 151,936] logits chunk of the bench (tied head): logits GEMM,
    CE fwd+bwd in place, dgrad and wgrad vs fp32."""
    rows, d, V = 8192, 1536, 151936
    torch.manual_seed(3)
    hf = _r(rows, d, scale=1.0)
    head = _r(V, d, scale=0.02)
    labels = torch.randint(0, V, (rows,), device=DEV)
    labels[::97] = -100
    n_valid = int((labels >= 0).sum())
    loss = torch.zeros((), device=DEV)
    logits = G.linear_fwd(hf, head)
    dl = F.ce_fwd_bwd_(logits, labels, 1.0 / n_valid, loss)
    dh = G.linear_dgrad(dl, head)
    dw = G.linear_wgrad(dl, hf)
    hf32 = hf.float().requires_grad_(True)
    head32 = head.float().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(hf32 @ head32.t(), labels, ignore_index=-100, reduction="sum") / n_valid
    ref.backward()
    assert abs(loss.item() / n_valid - ref.item()) < 1e-3 * ref.item(), (loss.item() / n_valid, ref.item())
    assert rel_l2(dh, hf32.grad) < 2e-2 and cosine(dh, hf32.grad) > 0.9995
    assert rel_l2(dw, head32.grad) < 2e-2 and cosine(dw, head32.grad) > 0.9995


def _model_step(shape, lens, push_mode="slot", recompute="none", seed=0, perturb=True):
    sizes = W.unit_sizes(shape)
    gen = torch.Generator(device=DEV).manual_seed(seed)
    units32 = [W.init_unit(shape, u, gen, DEV) for u in range(len(sizes))]
    if perturb:  # norms / biases away from their init so their gradients are exercised
        for u in units32:
            u += 0.01 * torch.randn(u.shape, device=DEV, generator=gen)
    eng = OdcEngine(sizes, push_mode=push_mode)
    for u, t in enumerate(units32):
        eng.set_params(u, t)
    batch = W.make_batch(lens, list(range(len(lens))), shape.vocab, DEV, heads=shape.heads, kv_heads=shape.kv_heads)
    wk = W.Worker(shape, W.OdcComm(eng), DEV, recompute=recompute)
    loss = wk.microbatch(batch, 1.0).item()
    eng.minibatch_end()
    eng.check()
    grads = [eng.read_grad_shard(u).clone() for u in range(len(sizes))]
    eng.close()
    del wk
    torch.cuda.empty_cache()
    return units32, batch, loss, grads


def _check_against_fp32(shape, units32, batch, loss, grads):
    ref_units = [t.to(torch.bfloat16).float().requires_grad_(True) for t in units32]
    rl = ref_loss(shape, ref_units, batch)
    rl.backward()
    assert abs(loss - rl.item()) <= 1e-2 * abs(rl.item()), (loss, rl.item())
    for u, got in enumerate(grads):
        want = ref_units[u].grad
        c, r = cosine(got, want), rel_l2(got, want)
        assert c > 0.995 and r < 5e-2, (shape.name, u, c, r)


def _layers(shape, n):
    return Shape(f"{shape.name}-L{n}", shape.d, shape.ffn, n, shape.heads, shape.kv_heads, shape.vocab,
                 shape.qkv_bias, shape.tied)


def test_qwen15b_layer_one_32k_sequence():
    """One full Qwen2.5-1.5B decoder layer + tied embedding / LM head (V =
    151,936), forward and backward through the ODC engine, on the bench's
    largest microbatch: a single 32,768-token sequence."""
    s = _layers(QWEN25_1_5B, 1)
    units32, batch, loss, grads = _model_step(s, [32768])
    assert abs(loss - math.log(s.vocab)) < 0.5
    _check_against_fp32(s, units32, batch, loss, grads)


def test_llama8b_two_layers_selective_recompute():
    """Llama-3-8B shape (d 4096, GQA 32/8, untied V = 128,256), 2 layers,
    selective recompute, a 16K-token packed microbatch."""
    s = _layers(LLAMA3_8B, 2)
    units32, batch, loss, grads = _model_step(s, [9000, 4096, 2500, 788], recompute="selective", seed=1)
    _check_against_fp32(s, units32, batch, loss, grads)


def test_qwen14b_layer_64k_fixed_push():
    """Qwen2.5-14B shape (d 5120, GQA 40/8, untied V = 152,064), one layer,
    one 65,536-token sequence, full recompute, FIXED (deterministic) push,
    against fp32."""
    s = _layers(QWEN25_14B, 1)
    units32, batch, loss, grads = _model_step(s, [65536], push_mode="fixed", recompute="full", seed=2)
    torch.cuda.empty_cache()
    _check_against_fp32(s, units32, batch, loss, grads)


def test_fixed_push_order_independent_at_14b_unit():
    """The deterministic push at the 14B layer unit (275,268,608 elements):
    three microbatch gradients pushed in two different orders give bitwise
    identical shards, equal to the oracle's int64 fixed-point sum."""
    import numpy as np

    from oracle import odc_oracle as O

    M = QWEN25_14B.layer_elems
    gen = torch.Generator(device=DEV).manual_seed(4)
    gs = [torch.randn(M, device=DEV, generator=gen) * 1e-3 for _ in range(3)]
    ws = [0.5, 0.25, 0.125]
    outs = []
    for order in ((0, 1, 2), (2, 0, 1)):
        eng = OdcEngine([M], push_mode="fixed")
        eng.set_params(0, torch.zeros(M, device=DEV))
        for i in order:
            eng.push(0, gs[i], ws[i])
        eng.minibatch_end()
        eng.check()
        outs.append(eng.read_grad_shard(0).cpu().numpy())
        eng.close()
    assert np.array_equal(outs[0], outs[1])
    want = O.fixed_mode_reduce(M, [(0, g.cpu().numpy(), np.float32(w)) for g, w in zip(gs, ws)])
    assert np.array_equal(outs[0], want)
