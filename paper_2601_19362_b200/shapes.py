"""Model shapes of the BASELINE configs (public HF configs)
and the FSDP-unit element counts the ODC shard store is sized from."""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shape:
    name: str
    d: int
    ffn: int
    layers: int
    heads: int
    kv_heads: int
    vocab: int
    qkv_bias: bool
    tied: bool

    @property
    def head_dim(self) -> int:
        return self.d // self.heads

    @property
    def layer_elems(self) -> int:
        """Elements of one transformer layer = one FSDP unit:
        q, k, v (+bias), o, gate/up/down, 2 RMSNorm weights."""
        hd = self.head_dim
        q = self.d * self.d + (self.d if self.qkv_bias else 0)
        kv = 2 * (self.kv_heads * hd * self.d + (self.kv_heads * hd if self.qkv_bias else 0))
        o = self.d * self.d
        mlp = 3 * self.d * self.ffn
        return q + kv + o + mlp + 2 * self.d

    def unit_sizes(self):
        """FSDP units: 0 = embedding (+ final norm, + untied LM head), 1..L =
        decoder layers (worker.unit_sizes computes the same from the layouts)."""
        emb = self.vocab * self.d * (1 if self.tied else 2) + self.d
        return [emb] + [self.layer_elems] * self.layers

    @property
    def nonembed_params(self) -> int:
        return self.layers * self.layer_elems + self.d  # + final norm

    def beta_over_alpha(self) -> float:
        """Cost-model beta/alpha = P_nonembed / (n_layer * d):
        FLOP-proportional costs, 6*P*s (dense) vs 6*L*d*s^2 (causal attention)."""
        return self.nonembed_params / (self.layers * self.d)

    def beta_over_alpha_b200(self) -> float:
        """beta/alpha measured on B200: tools/calibrate_cost.py times one SFT
        microbatch (fwd + bwd, this repo's kernels) for 15 length mixes and fits
        t = alpha*sum(s^2) + beta*sum(s) + c (the reference's per-sample cost,
        src/cost_model.cpp:14-18): beta/alpha = 26,685 for Qwen2.5-1.5B (max
        residual 1.7%, profiles/r01/cost_calibration_qwen1.5b.jsonl). Expressed
        as the FLOP ratio (linear work incl. the LM head, per layer-width) times
        the measured attention-vs-linear cost factor, so other shapes scale by
        their own FLOP ratio. The cost model's absolute scale is a free knob
        (inc/cost_model.hpp:10-12); only beta/alpha shapes the plan, identically
        for ODC and FSDP."""
        linear = (self.nonembed_params + self.vocab * self.d) / (self.layers * self.d)
        return linear * B200_ATTN_VS_LINEAR


# measured: 26,685 / ((P_nonembed + V*d) / (L*d)) for Qwen2.5-1.5B on B200
B200_ATTN_VS_LINEAR = 0.7433

QWEN25_1_5B = Shape("qwen2.5-1.5b", 1536, 8960, 28, 12, 2, 151936, True, True)
LLAMA3_8B = Shape("llama-3-8b", 4096, 14336, 32, 32, 8, 128256, False, False)
QWEN25_14B = Shape("qwen2.5-14b", 5120, 13824, 48, 40, 8, 152064, True, False)
SHAPES = {s.name: s for s in (QWEN25_1_5B, LLAMA3_8B, QWEN25_14B)}

assert QWEN25_1_5B.layer_elems == 46_797_824
assert LLAMA3_8B.layer_elems == 218_112_000
assert QWEN25_14B.layer_elems == 275_268_608
