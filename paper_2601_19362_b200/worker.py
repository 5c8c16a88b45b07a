"""SFT worker: the caller of the ODC path (SURVEY §3 target call stack).

One rank = one GPU. For every microbatch of this rank's queue (LB-Mini plan for
ODC, LB-Micro for the FSDP comparison), a Qwen2.5/Llama-shaped decoder runs a
packed-varlen forward and a hand-written backward:

  forward   fetch unit l+1 on the comm stream while layer l computes
  backward  fetch unit l-1 while layer l computes; push unit l's fp32
            gradient as soon as its wgrads are done
  minibatch end: comm.minibatch_end() then comm.adam()

Dense layers are tcgen05 GEMMs (csrc/gemm.cu, operands used in place);
attention is the tcgen05 causal varlen forward/backward (csrc/attention.cu,
head_dim 128 only: any other shape raises, there is no library fallback);
the elementwise glue (RMSNorm, bias+RoPE+split, SwiGLU, CE) is fused sm_100a
kernels (csrc/worker_kernels.cu) and residual adds ride in the GEMM epilogue.
Activations are kept for the backward by default (they fit 180 GB for the
1.5B shape at 32K tokens). The 8B/14B shapes at 32K/64K tokens do not fit, so
`recompute` keeps only each layer's input (+ the attention output and lse in
"selective" mode) and re-runs the layer's forward in the backward, right
after the backward's own re-fetch of the unit (no extra communication).

Comm backends share one interface:
  OdcComm   odc fetch / push / device barrier / fused AdamW (libodc.so)
  FsdpComm  NCCL all_gather_into_tensor / reduce_scatter_tensor per unit
            per microbatch (the comparison path), same AdamW kernel
"""
from __future__ import annotations

import contextlib
import math
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from . import fused as F
from . import gemm as G
from .shapes import Shape

ROPE_THETA = 1_000_000.0
EPS = 1e-6


# ----------------------------------------------------------------- layouts
def layer_layout(s: Shape) -> List[Tuple[str, Tuple[int, ...]]]:
    """Flat FSDP-unit layout of one decoder layer (element order in the unit)."""
    qkv = s.d + 2 * s.kv_heads * s.head_dim
    lay = [("qkv_w", (qkv, s.d))]
    if s.qkv_bias:
        lay.append(("qkv_b", (qkv,)))
    lay += [("o_w", (s.d, s.d)), ("gu_w", (2 * s.ffn, s.d)), ("down_w", (s.d, s.ffn)), ("ln1", (s.d,)),
            ("ln2", (s.d,))]
    return lay


def embed_layout(s: Shape) -> List[Tuple[str, Tuple[int, ...]]]:
    lay = [("emb", (s.vocab, s.d)), ("norm", (s.d,))]
    if not s.tied:
        lay.append(("head", (s.vocab, s.d)))
    return lay


def numel(lay) -> int:
    return sum(math.prod(sh) for _, sh in lay)


def views(flat: torch.Tensor, lay) -> Dict[str, torch.Tensor]:
    out, off = {}, 0
    for name, sh in lay:
        n = math.prod(sh)
        out[name] = flat[off:off + n].view(*sh)
        off += n
    return out


def unit_sizes(s: Shape) -> List[int]:
    """FSDP units: 0 = embedding (+ final norm, + untied head), 1..L = layers."""
    return [numel(embed_layout(s))] + [numel(layer_layout(s))] * s.layers


def init_unit(s: Shape, unit: int, gen: torch.Generator, device) -> torch.Tensor:
    lay = embed_layout(s) if unit == 0 else layer_layout(s)
    flat = torch.empty(numel(lay), device=device)
    v = views(flat, lay)
    for name, t in v.items():
        if name in ("ln1", "ln2", "norm"):
            t.fill_(1.0)
        elif name.endswith("_b"):
            t.zero_()
        else:
            t.normal_(0.0, 0.02, generator=gen)
    return flat


# ------------------------------------------------------------ rope (test reference)
def rope_tables(positions: torch.Tensor, head_dim: int):
    inv = 1.0 / (ROPE_THETA ** (torch.arange(0, head_dim, 2, device=positions.device, dtype=torch.float32) / head_dim))
    ang = positions.float()[:, None] * inv[None, :]
    return torch.cos(ang), torch.sin(ang)  # [T, hd/2]


# NVTX ranges per fetch / layer forward / LM head / layer backward / push / barrier+AdamW,
# for ncu/nsys (`ncu --nvtx --nvtx-include "bwd l3/"`); off unless ODC_NVTX=1
_NVTX = os.environ.get("ODC_NVTX") == "1"


@contextlib.contextmanager
def nvtx(name: str):
    if not _NVTX:
        yield
        return
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()


# ------------------------------------------------------------------ comm
class OdcComm:
    """ODC: point-to-point fetch/push over CUDA-IPC-mapped peer HBM."""

    name = "odc"

    def __init__(self, engine):
        self.eng = engine

    def fetch(self, unit, out, stream):
        self.eng.fetch(unit, out, stream=stream)

    def push(self, unit, grad, weight, stream):
        self.eng.push(unit, grad, weight, stream=stream)

    def minibatch_end(self, stream):
        self.eng.minibatch_end(stream=stream)

    def adam(self, stream, **kw):
        self.eng.adam_step(stream=stream, **kw)


class FsdpComm:
    """FSDP comparison path: per-unit NCCL collectives every microbatch.
    Owned shards live in the same engine arena (world=1 engine per rank
    holding this rank's 1/N slice of every unit), AdamW is the same kernel."""

    name = "fsdp"

    def __init__(self, sizes: Sequence[int], rank: int, world: int, device, group=None):
        import torch.distributed as dist

        from .engine import OdcEngine

        self.dist, self.group, self.rank, self.world = dist, group, rank, world
        for n in sizes:
            if n % world:
                raise ValueError("FSDP path needs unit sizes divisible by the world size")
        self.shard = [n // world for n in sizes]
        self.local = OdcEngine(self.shard, rank=0, world=1, device=device)  # owned shards + AdamW state
        self.bf = [torch.empty(n, dtype=torch.bfloat16, device=device) for n in self.shard]
        self.rs = [torch.empty(n, dtype=torch.float32, device=device) for n in self.shard]
        self.dirty = True

    def set_params(self, unit, full_fp32):
        sh = self.shard[unit]
        self.local.set_params(unit, full_fp32[self.rank * sh:(self.rank + 1) * sh].contiguous())

    def _refresh(self, stream):
        if self.dirty:
            for u in range(len(self.shard)):
                self.local.fetch(u, self.bf[u], stream=stream)
            self.dirty = False

    def fetch(self, unit, out, stream):
        with torch.cuda.stream(stream):
            self._refresh(stream)
            self.dist.all_gather_into_tensor(out, self.bf[unit], group=self.group)

    def push(self, unit, grad, weight, stream):
        with torch.cuda.stream(stream):
            if weight != 1.0:  # per-rank token weight applied before the sum
                grad.mul_(weight)
            self.dist.reduce_scatter_tensor(self.rs[unit], grad, group=self.group)
            self.local.push(unit, self.rs[unit], 1.0, stream=stream)

    def minibatch_end(self, stream):
        self.local.minibatch_end(stream=stream)

    def adam(self, stream, **kw):
        self.local.adam_step(stream=stream, **kw)
        self.dirty = True


# ---------------------------------------------------------------- trace
class Tracer:
    """Measured timeline in the reference's Chrome-trace schema
    (src/commsim.cpp:240-258: name "<kind> m<mb> l<layer>", cat compute|comm,
    ph X, pid = rank, tid 0 compute / 1 comm, ts/dur in microseconds,
    args.volume_elems for comm). Spans are CUDA events on the stream that ran
    the work, so they show real overlap of fetch/push with compute."""

    def __init__(self, rank: int):
        self.rank, self.rows, self.t0 = rank, [], None
        self.mb = 0

    def start(self, stream):
        self.t0 = torch.cuda.Event(enable_timing=True)
        self.t0.record(stream)

    def span(self, kind, layer, stream, is_comm, volume=0):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        row = [kind, self.mb, layer, is_comm, volume, e0, None]
        self.rows.append(row)
        return row

    @staticmethod
    def end(row, stream):
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(stream)
        row[6] = e1

    def events(self):
        out = []
        for kind, mb, layer, is_comm, vol, e0, e1 in self.rows:
            if e1 is None:
                continue
            ts = self.t0.elapsed_time(e0) * 1e3
            ev = {"name": f"{kind} m{mb} l{layer}", "cat": "comm" if is_comm else "compute", "ph": "X",
                  "pid": self.rank, "tid": 1 if is_comm else 0, "ts": ts, "dur": e0.elapsed_time(e1) * 1e3}
            if is_comm:
                ev["args"] = {"volume_elems": vol}
            out.append(ev)
        return out

    def busy_ms(self):
        return sum(e0.elapsed_time(e1) for k, _, _, c, _, e0, e1 in self.rows if not c and e1 is not None)


def chrome_trace(events_per_rank) -> dict:
    evs = [e for evs in events_per_rank for e in evs]
    return {"traceEvents": evs, "displayTimeUnit": "ms"}


def trace_busy_total(trace: dict, world: int):
    """Per-rank busy time and step span from a measured trace: busy = summed
    durations of the rank's compute spans ("fwd"/"bwd": the reference's
    per_device_busy, src/commsim.cpp:119-121 — the "barrier" span is the wait
    at the minibatch end, i.e. idle), total = the span from the earliest event
    start to the latest event end over all ranks (us)."""
    evs = trace["traceEvents"]
    busy = [0.0] * world
    for e in evs:
        if e["cat"] == "compute" and not e["name"].startswith("barrier"):
            busy[e["pid"]] += e["dur"]
    t0 = min(e["ts"] for e in evs)
    t1 = max(e["ts"] + e["dur"] for e in evs)
    return busy, t1 - t0


def trace_idle_fraction(trace: dict, world: int) -> float:
    """The reference's bubble rate (src/runtime.cpp:43, src/commsim.cpp:232),
    1 - sum(busy) / (D * T), applied to a measured trace."""
    busy, total = trace_busy_total(trace, world)
    return 1.0 - sum(busy) / (world * total)


# --------------------------------------------------------------- worker
@dataclass
class Batch:
    ids: torch.Tensor        # [T] int64
    labels: torch.Tensor     # [T] int64, -100 = ignore
    positions: torch.Tensor  # [T]
    cu_seqlens: torch.Tensor  # [n+1] int32
    max_len: int
    tokens: int
    attn_items: Optional[torch.Tensor] = None  # tcgen05 attention work lists (built per microbatch)
    attn_bwd_items: Optional[torch.Tensor] = None


def make_batch(lens: Sequence[int], sample_ids: Sequence[int], vocab: int, device, heads: int = 0,
               kv_heads: int = 0) -> Batch:
    """Synthetic packed microbatch: token ids seeded by the global sample id, so
    every implementation sees identical data."""
    ids, labels, pos, cu = [], [], [], [0]
    for sid in sample_ids:
        n = int(lens[sid])
        g = torch.Generator().manual_seed(1_000_003 * (sid + 1))
        t = torch.randint(0, vocab, (n,), generator=g)
        ids.append(t)
        lab = torch.full((n,), -100, dtype=torch.int64)
        lab[:-1] = t[1:]
        labels.append(lab)
        pos.append(torch.arange(n))
        cu.append(cu[-1] + n)
    T = cu[-1]
    # pinned staging: the H2D copies are asynchronous (a pageable copy would
    # drain the stream while the host builds the next tensor)
    pin = torch.device(device).type == "cuda"

    def h2d(t):
        return (t.pin_memory() if pin else t).to(device, non_blocking=True)

    b = Batch(h2d(torch.cat(ids)), h2d(torch.cat(labels)), h2d(torch.cat(pos)),
              h2d(torch.tensor(cu, dtype=torch.int32)), max(int(lens[s]) for s in sample_ids), T)
    if heads:
        attach_attn_items(b, [int(lens[s]) for s in sample_ids], heads, device, kv_heads)
    return b


def attach_attn_items(b: Batch, seq_lens: Sequence[int], heads: int, device, kv_heads: int = 0) -> Batch:
    b.attn_items = F.attn_items(list(seq_lens), heads, device)
    if kv_heads:
        b.attn_bwd_items = F.attn_bwd_items(list(seq_lens), heads, kv_heads, device)
    return b


class Worker:
    def __init__(self, shape: Shape, comm, device, ce_chunk: int = 8192, max_positions: int = 65536,
                 cache_params: bool = False, recompute: str = "none"):
        if shape.head_dim != 128:
            raise ValueError(f"the tcgen05 attention kernels need head_dim 128, {shape.name} has {shape.head_dim}")
        self.s, self.comm, self.dev = shape, comm, torch.device(device)
        self.max_positions = max_positions
        if recompute not in ("none", "selective", "full"):
            raise ValueError(f"recompute must be none|selective|full, got {recompute!r}")
        self.recompute = recompute
        self.sizes = unit_sizes(shape)
        self.L = shape.layers
        self.ce_chunk = ce_chunk
        self.comm_stream = torch.cuda.Stream(device=self.dev)
        lsz = self.sizes[1]
        self.pbuf = [torch.empty(lsz, dtype=torch.bfloat16, device=self.dev) for _ in range(2)]
        self.gbuf = [torch.empty(lsz, dtype=torch.float32, device=self.dev) for _ in range(2)]
        self.ebuf = torch.empty(self.sizes[0], dtype=torch.bfloat16, device=self.dev)
        self.egrad = torch.empty(self.sizes[0], dtype=torch.float32, device=self.dev)
        self.rope = F.rope_table(max_positions, shape.head_dim, ROPE_THETA, self.dev)
        self.tracer: Optional[Tracer] = None
        # parameters cannot change inside a minibatch, so with
        # HBM to spare every unit is fetched once per minibatch and reused by
        # the backward and by later microbatches (ODC only: FSDP reshards)
        self.cache = None
        if cache_params:
            self.cache = [self.ebuf] + [torch.empty(lsz, dtype=torch.bfloat16, device=self.dev) for _ in range(self.L)]
            self.cache_ev = [None] * (self.L + 1)

    # --- stream helpers
    def _ubuf(self, unit):
        if self.cache is not None:
            return self.cache[unit]
        return self.ebuf if unit == 0 else self.pbuf[unit % 2]

    def _fetch_unit(self, unit, after: Optional[torch.cuda.Event] = None):
        if self.cache is not None and self.cache_ev[unit] is not None:
            return self.cache_ev[unit]  # already resident for this minibatch
        # a cached unit has its own buffer: no need to wait for compute to release one
        ev = self._fetch(unit, self._ubuf(unit), None if self.cache is not None else after)
        if self.cache is not None:
            self.cache_ev[unit] = ev
        return ev

    def _fetch(self, unit, buf, after: Optional[torch.cuda.Event] = None):
        if after is not None:
            self.comm_stream.wait_event(after)
        tr = self.tracer.span("gather", unit, self.comm_stream, True, buf.numel()) if self.tracer else None
        with nvtx(f"fetch u{unit}"):
            self.comm.fetch(unit, buf, self.comm_stream)
        if tr:
            Tracer.end(tr, self.comm_stream)
        ev = torch.cuda.Event()
        ev.record(self.comm_stream)
        return ev

    # --- one decoder layer forward (also the recompute of the backward)
    def _layer_fwd(self, P, x, b: Batch, o_lse=None, out: bool = True):
        """Returns the activations the backward needs and the layer output.
        With `o_lse` (selective recompute) the attention forward is skipped;
        without `out` (any recompute) so is the down projection."""
        s = self.s
        hd, H, KV = s.head_dim, s.heads, s.kv_heads
        T = b.tokens
        a, r1 = F.rmsnorm_fwd(x, P["ln1"])
        qkv = G.linear_fwd(a, P["qkv_w"])
        q, k, v = F.qkv_rope_fwd(qkv, P.get("qkv_b"), self.rope, b.positions, H, KV, hd)
        del qkv
        if o_lse is not None:
            o, lse = o_lse
        else:
            o, lse = F.attn_fwd(q, k, v, b.attn_items, 1.0 / math.sqrt(hd))
        hm = G.linear_fwd(o.view(T, H * hd), P["o_w"], residual=x)
        bn, r2 = F.rmsnorm_fwd(hm, P["ln2"])
        gu, m = G.gate_up_swiglu(bn, P["gu_w"], s.ffn)  # SwiGLU fused into the GEMM epilogue
        h = G.linear_fwd(m, P["down_w"], residual=hm) if out else None
        return (x, a, r1, q, k, v, o, lse, hm, bn, r2, gu, m), h

    def _keep(self, act):
        """What the forward keeps per layer: everything (none), the layer input
        plus the attention output and lse (selective: the backward recomputes
        the GEMMs and glue but not the attention), or the layer input (full)."""
        if self.recompute == "none":
            return act
        if self.recompute == "selective":
            return (act[0], act[6], act[7])
        return (act[0],)

    def _restore(self, P, kept, b: Batch):
        if self.recompute == "none":
            return kept
        o_lse = (kept[1], kept[2]) if self.recompute == "selective" else None
        return self._layer_fwd(P, kept[0], b, o_lse, out=False)[0]

    def microbatch(self, b: Batch, weight: float) -> torch.Tensor:
        s, L = self.s, self.L
        cur = torch.cuda.current_stream(self.dev)
        hd, H, KV = s.head_dim, s.heads, s.kv_heads
        T = b.tokens
        scale = 1.0 / math.sqrt(hd)
        lay = layer_layout(s)
        tab = self.rope
        if b.max_len > self.max_positions:  # the RoPE table has max_positions rows (positions restart per sample)
            raise ValueError(f"sample of {b.max_len} tokens exceeds the RoPE table ({self.max_positions} positions)")
        if b.attn_items is None or b.attn_bwd_items is None:
            cu = b.cu_seqlens.tolist()
            attach_attn_items(b, [cu[i + 1] - cu[i] for i in range(len(cu) - 1)], H, self.dev, KV)

        # ---------------- forward
        ev_e = self._fetch_unit(0, after=_record(cur))
        ev = self._fetch_unit(1, after=_record(cur))
        cur.wait_event(ev_e)
        E = views(self._ubuf(0), embed_layout(s))
        h = E["emb"].index_select(0, b.ids)
        saved = []
        for l in range(1, L + 1):
            cur.wait_event(ev)
            P = views(self._ubuf(l), lay)
            if l < L:  # prefetch the next unit into the other buffer once layer l-1 released it
                ev = self._fetch_unit(l + 1, after=_record(cur))
            tr = self.tracer.span("fwd", l, cur, False) if self.tracer else None
            with nvtx(f"fwd l{l}"):
                act, h = self._layer_fwd(P, h, b)
            saved.append(self._keep(act))
            if tr:
                Tracer.end(tr, cur)

        # ---------------- final norm, LM head + CE (chunked); head backward in place
        hf, rf = F.rmsnorm_fwd(h, E["norm"])
        head = E["emb"] if s.tied else E["head"]
        self.egrad.zero_()
        EG = views(self.egrad, embed_layout(s))
        headg = EG["emb"] if s.tied else EG["head"]
        dhf = torch.empty_like(hf)
        n_valid = max(1, T - (b.cu_seqlens.numel() - 1))
        loss = torch.zeros((), device=self.dev, dtype=torch.float32)
        for c0 in range(0, T, self.ce_chunk):
            c1 = min(T, c0 + self.ce_chunk)
            with nvtx(f"lm_head+ce {c0}"):
                logits = G.linear_fwd(hf[c0:c1], head)
                dl = F.ce_fwd_bwd_(logits, b.labels[c0:c1], 1.0 / n_valid, loss)  # logits -> dlogits in place
                G.linear_dgrad(dl, head, out=dhf[c0:c1])
                G.linear_wgrad(dl, hf[c0:c1], out=headg, accumulate=True)
            del logits, dl
        loss /= n_valid
        dh = F.rmsnorm_bwd(dhf, h, E["norm"], rf, EG["norm"])
        del dhf, hf

        # ---------------- backward through the layers
        if self.cache is None:  # the forward's buffers were recycled: re-fetch (FSDP semantics)
            ev = self._fetch(L, self.pbuf[L % 2], after=_record(cur))
        else:
            ev = self._fetch_unit(L)
        push_ev = [None, None]
        for l in range(L, 0, -1):
            cur.wait_event(ev)
            P = views(self._ubuf(l), lay)
            if l > 1:
                ev = (self._fetch(l - 1, self.pbuf[(l - 1) % 2], after=_record(cur)) if self.cache is None
                      else self._fetch_unit(l - 1))
            gi = l % 2
            if push_ev[gi] is not None:  # grad buffer free once its previous push finished
                cur.wait_event(push_ev[gi])
            Gv = views(self.gbuf[gi], lay)
            for name in ("ln1", "ln2", "qkv_b"):  # atomically accumulated parts
                if name in Gv:
                    Gv[name].zero_()
            tr = self.tracer.span("bwd", l, cur, False) if self.tracer else None
            rng = nvtx(f"bwd l{l}")
            rng.__enter__()
            x, a, r1, q, k, v, o, lse, hm, bn, r2, gu, m = self._restore(P, saved[l - 1], b)
            # MLP block
            dm = G.linear_dgrad(dh, P["down_w"])
            G.linear_wgrad(dh, m, out=Gv["down_w"])
            dgu = F.swiglu_bwd(dm, gu, s.ffn)
            del dm
            dbn = G.linear_dgrad(dgu, P["gu_w"])
            G.linear_wgrad(dgu, bn, out=Gv["gu_w"])
            del dgu
            dhm = F.rmsnorm_bwd(dbn, hm, P["ln2"], r2, Gv["ln2"], resid=dh)
            # attention block
            do = G.linear_dgrad(dhm, P["o_w"])
            G.linear_wgrad(dhm, o.view(T, -1), out=Gv["o_w"])
            # attention backward straight to the packed qkv gradient (inverse RoPE fused)
            dqkv = F.attn_bwd_qkv(q, k, v, o, do.view(T, H, hd), lse, b.attn_bwd_items, scale, tab, b.positions)
            del do
            if "qkv_b" in Gv:
                F.col_sum_(dqkv, Gv["qkv_b"])
            da = G.linear_dgrad(dqkv, P["qkv_w"])
            G.linear_wgrad(dqkv, a, out=Gv["qkv_w"])
            dh = F.rmsnorm_bwd(da, x, P["ln1"], r1, Gv["ln1"], resid=dhm)
            rng.__exit__(None, None, None)
            if tr:
                Tracer.end(tr, cur)
            # push this unit's gradient as soon as it is complete
            self.comm_stream.wait_event(_record(cur))
            trp = self.tracer.span("reduce", l, self.comm_stream, True, self.gbuf[gi].numel()) if self.tracer else None
            with nvtx(f"push u{l}"):
                self.comm.push(l, self.gbuf[gi], weight, self.comm_stream)
            if trp:
                Tracer.end(trp, self.comm_stream)
            push_ev[gi] = _record(self.comm_stream)
            saved[l - 1] = None
        # embedding: scatter-add of dh into the looked-up rows (+ tied head grad above)
        EG["emb"].index_add_(0, b.ids, dh.float())
        self.comm_stream.wait_event(_record(cur))
        self.comm.push(0, self.egrad, weight, self.comm_stream)
        cur.wait_event(_record(self.comm_stream))
        if self.tracer:
            self.tracer.mb += 1
        return loss

    def empty_microbatch(self):
        """FSDP padding microbatch (src/partition.cpp:305-307, :339): joins every
        collective in exactly the order microbatch() issues them, computes nothing."""
        cur = torch.cuda.current_stream(self.dev)
        L = self.L
        self._fetch(0, self.ebuf, after=_record(cur))
        for u in range(1, L + 1):
            self._fetch(u, self.pbuf[u % 2])
        self._fetch(L, self.pbuf[L % 2])
        self.egrad.zero_()
        for g in self.gbuf:
            g.zero_()
        self.comm_stream.wait_event(_record(cur))
        for l in range(L, 0, -1):
            if l > 1:
                self._fetch(l - 1, self.pbuf[(l - 1) % 2])
            self.comm.push(l, self.gbuf[l % 2], 0.0, self.comm_stream)
        self.comm.push(0, self.egrad, 0.0, self.comm_stream)
        cur.wait_event(_record(self.comm_stream))

    def minibatch_end(self, lr=1e-5):
        if self.cache is not None:  # new parameter epoch: every unit must be fetched again
            self.cache_ev = [None] * (self.L + 1)
        cur = torch.cuda.current_stream(self.dev)
        self.comm_stream.wait_event(_record(cur))
        with nvtx("barrier+adamw"):
            self.comm.minibatch_end(self.comm_stream)
            self.comm.adam(self.comm_stream, lr=lr)
        cur.wait_event(_record(self.comm_stream))


def _record(stream) -> torch.cuda.Event:
    e = torch.cuda.Event()
    e.record(stream)
    return e
