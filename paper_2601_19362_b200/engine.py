"""OdcEngine — Python host side of the production ODC engine (odc_ctx_t).

One instance per rank (one process per GPU). Construction allocates this
rank's HBM arena (owned bf16/fp32 shards + AdamW state of every FSDP unit),
exchanges CUDA IPC handles with the other ranks over torch.distributed (the
only collective on the ODC path, at init) and maps every peer arena.

After that every operation is a stream-ordered sm_100a kernel launch on
device memory; cross-rank ordering is device-side (sys-scope flags), there is
no NCCL call and no host synchronisation on the hot path:

    fetch(layer, out)            ShardState::gather         inc/primitives.hpp:70-77
    push(layer, grad, w)         ShardFabric::scatter_accumulate   :181-188
    push_slice(...)              ShardFabric::push_slice    :191-195
    minibatch_end()              ShardFabric::finalize_minibatch   :199-203
    read_grad_shard(layer)       ShardState::take_grads     :144-148 (one shard)
    adam_step(...)               fused AdamW on owned shards (no reference counterpart)
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import check, lib

PUSH_MODES = {"red": _lib.ODC_PUSH_RED, "slot": _lib.ODC_PUSH_SLOT, "fixed": _lib.ODC_PUSH_FIXED}
FETCH_ENGINES = {"tma": _lib.ODC_FETCH_TMA, "ldg": _lib.ODC_FETCH_LDG, "ce": _lib.ODC_FETCH_CE}


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor):
    if not t.is_cuda:
        raise ValueError("ODC engine operands must be CUDA tensors")
    if not t.is_contiguous():
        raise ValueError("ODC engine operands must be contiguous")
    return C.c_void_p(t.data_ptr())


class OdcEngine:
    def __init__(self, layer_elems: Sequence[int], rank: int = 0, world: int = 1, device: Optional[int] = None,
                 push_mode: str = "red", fetch_ctas: int = 0, push_ctas: int = 0, timeout_s: float = 60.0,
                 group=None, fetch_engine: str = "tma", fixed_frac_bits: int = 0, _defer_ready: bool = False):
        self.layer_elems = [int(x) for x in layer_elems]
        self.rank, self.world = rank, world
        if device is None:
            device = torch.cuda.current_device()
        self.device = device.index if isinstance(device, torch.device) else int(device)
        self.push_mode = push_mode
        arr = (C.c_int64 * len(self.layer_elems))(*self.layer_elems)
        cfg = _lib.OdcConfig(rank, world, self.device, len(self.layer_elems), arr, PUSH_MODES[push_mode], fetch_ctas,
                             push_ctas, timeout_s, FETCH_ENGINES[fetch_engine], fixed_frac_bits)
        self.fixed_frac_bits = fixed_frac_bits or _lib.ODC_FIXED_FRAC_BITS_DEFAULT
        h = C.c_void_p()
        check(lib().odc_ctx_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.adam_steps = 0
        if _defer_ready:  # local_group wires the peers itself
            return
        if world > 1:
            self._exchange(group)
        check(lib().odc_ctx_ready(self.h))

    @classmethod
    def local_group(cls, layer_elems: Sequence[int], world: int, devices: Sequence[int], **kw):
        """Single-process mode: `world` ranks in THIS process, rank r on
        devices[r % len(devices)], every peer arena mapped directly
        (odc_ctx_import_ctx) — several ranks per GPU for protocol tests on a
        one-GPU box, or one process driving several GPUs over NVLink. The
        ranks' operations are stream-ordered per rank; the device-side flag
        protocol is the same as across processes."""
        engs = [cls(layer_elems, rank=r, world=world, device=devices[r % len(devices)], _defer_ready=True, **kw)
                for r in range(world)]
        for e in engs:
            for p in engs:
                if p.rank != e.rank:
                    check(lib().odc_ctx_import_ctx(e.h, p.rank, p.h))
        for e in engs:
            check(lib().odc_ctx_ready(e.h))
        return engs

    def _exchange(self, group):
        from .dist import exchange_blobs

        n = C.c_size_t(0)
        buf = C.create_string_buffer(256)
        check(lib().odc_ctx_export(self.h, buf, 256, C.byref(n)))
        for peer, blob in enumerate(exchange_blobs(buf.raw[:n.value], group)):
            b = C.create_string_buffer(blob, len(blob))
            check(lib().odc_ctx_import(self.h, peer, b, len(blob)))

    def close(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                lib().odc_ctx_destroy(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self.h = C.c_void_p()

    __del__ = close

    # ---------------------------------------------------------------- layout
    def shard_range(self, layer: int, rank: Optional[int] = None):
        from .primitives import shard_range

        return shard_range(self.layer_elems[layer], self.world, self.rank if rank is None else rank)

    def arena_bytes(self) -> int:
        v = C.c_int64()
        check(lib().odc_ctx_arena_bytes(self.h, C.byref(v)))
        return v.value

    # ------------------------------------------------------------- hot path
    def set_params(self, layer: int, full_fp32: torch.Tensor, stream=None):
        assert full_fp32.dtype == torch.float32 and full_fp32.numel() == self.layer_elems[layer]
        check(lib().odc_set_params(self.h, layer, _ptr(full_fp32), _stream(stream)))

    def fetch(self, layer: int, out_bf16: torch.Tensor, stream=None):
        assert out_bf16.dtype == torch.bfloat16 and out_bf16.numel() == self.layer_elems[layer]
        check(lib().odc_fetch(self.h, layer, _ptr(out_bf16), _stream(stream)))
        return out_bf16

    def fetch_master(self, layer: int, out_fp32: torch.Tensor, stream=None):
        assert out_fp32.dtype == torch.float32 and out_fp32.numel() == self.layer_elems[layer]
        check(lib().odc_fetch_master(self.h, layer, _ptr(out_fp32), _stream(stream)))
        return out_fp32

    def push(self, layer: int, grad: torch.Tensor, weight: float, stream=None):
        assert grad.numel() == self.layer_elems[layer]
        dt = {torch.float32: _lib.ODC_F32, torch.bfloat16: _lib.ODC_BF16}[grad.dtype]
        check(lib().odc_push(self.h, layer, _ptr(grad), dt, float(weight), _stream(stream)))

    def push_slice(self, layer: int, target: int, offset: int, payload: torch.Tensor, weight: float, stream=None):
        assert payload.dtype == torch.float32
        check(lib().odc_push_slice(self.h, layer, target, offset, _ptr(payload), payload.numel(), float(weight),
                                   _stream(stream)))

    def minibatch_end(self, stream=None):
        check(lib().odc_minibatch_end(self.h, _stream(stream)))

    def adam_step(self, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0, stream=None):
        self.adam_steps += 1
        cfg = _lib.OdcAdamCfg(lr, betas[0], betas[1], eps, weight_decay, self.adam_steps)
        check(lib().odc_adam_step(self.h, C.byref(cfg), _stream(stream)))

    def _read_shard(self, fn, layer: int, stream=None) -> torch.Tensor:
        """The copy runs on `stream`; the current stream is made to wait for it, so
        the returned tensor is safe to use (e.g. .cpu()) on the current stream."""
        _, n = self.shard_range(layer)
        out = torch.empty(max(n, 1), dtype=torch.float32, device=f"cuda:{self.device}")[:n]
        if n:
            check(fn(self.h, layer, _ptr(out), _stream(stream)))
            if stream is not None:
                cur = torch.cuda.current_stream(self.device)
                if cur != stream:
                    cur.wait_stream(stream)
                    out.record_stream(stream)
        return out

    def read_grad_shard(self, layer: int, stream=None) -> torch.Tensor:
        return self._read_shard(lib().odc_read_grad_shard, layer, stream)

    def read_master_shard(self, layer: int, stream=None) -> torch.Tensor:
        return self._read_shard(lib().odc_read_master_shard, layer, stream)

    def check(self, stream=None):
        """Synchronise `stream`; raise BarrierTimeout if the watchdog fired,
        RangeError if a FIXED-mode push saturated the fixed-point range."""
        check(lib().odc_ctx_check(self.h, _stream(stream)))

    def flags(self, stream=None) -> int:
        """Sticky device flags (synchronises `stream`): _lib.ODC_FLAG_TIMEOUT,
        ODC_FLAG_FIXED_RANGE, ODC_FLAG_FIXED_UNDERFLOW (a nonzero w*g that the
        FIXED push rounded to 0: resolution loss, not an error)."""
        v = C.c_uint64(0)
        check(lib().odc_ctx_flags(self.h, C.byref(v), _stream(stream)))
        return int(v.value)

    @property
    def epoch(self) -> int:
        return int(lib().odc_ctx_epoch(self.h))
