"""Python host mirror of the reference ODC primitives over libodc.so.

Same names, argument meaning and error behaviour as the reference C++ API
(inc/ = /root/reference/proj/include/odcsim/):

    shard_range(elems, ranks, r)          ShardState::shard_begin/len   inc/primitives.hpp:53-56
    ShardFabric(ranks, elems, dtype)      ShardFabric<T>                :167-207
      .set_params(id, full)               :174-176 -> ShardState::set_params :58-67
      .gather(client, id)                 :177-179 -> ShardState::gather :70-77
      .scatter_accumulate(client, g, w)   :181-188
      .push_slice(client, tgt, off, p, w) :191-195
      .finalize_minibatch()               :199-203
      .state()                            ShardState<T> protocol steps :99-150

Every call runs on the GPU (fetch / stage / consume kernels of
csrc/odc_kernels.cu); host numpy arrays are only the by-value I/O the
reference API has.
"""
from __future__ import annotations

import ctypes as C
from typing import List

import numpy as np

from . import _lib
from ._lib import check, lib

_DT = {np.dtype(np.int64): _lib.ODC_I64, np.dtype(np.float64): _lib.ODC_F64, np.dtype(np.float32): _lib.ODC_F32}


def shard_range(elems: int, ranks: int, rank: int):
    """(begin, len) of rank's block shard: block = ceil(elems/ranks)."""
    b, n = C.c_int64(), C.c_int64()
    check(lib().odc_shard_range(elems, ranks, rank, C.byref(b), C.byref(n)))
    return b.value, n.value


def _buf(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class ShardState:
    """ShardState<T> protocol steps on a GPU-resident fabric."""

    def __init__(self, fabric: "ShardFabric"):
        self._f = fabric

    def ranks(self):
        return self._f.ranks

    def elems(self):
        return self._f.elems

    def slot_capacity(self):
        return self._f.block

    def shard_begin(self, r):
        return shard_range(self._f.elems, self._f.ranks, r)[0]

    def shard_len(self, r):
        return shard_range(self._f.elems, self._f.ranks, r)[1]

    def split_gradient(self, frm: int, grad, weight):
        """:80-97 — one (from, target, offset=0, payload, weight) per owner."""
        g = np.ascontiguousarray(np.asarray(grad, self._f.dtype))
        if g.size != self._f.elems:
            from .errors import ParamError

            raise ParamError("gradient vector length mismatch")
        out = []
        for r in range(self._f.ranks):
            b, n = shard_range(self._f.elems, self._f.ranks, r)
            out.append((frm, r, 0, g[b:b + n].copy(), weight))
        return out

    def try_stage(self, msg) -> bool:
        frm, tgt, off, payload, w = msg
        p = np.ascontiguousarray(np.asarray(payload, self._f.dtype))
        wv = np.asarray([w], self._f.dtype)
        staged = C.c_int()
        check(lib().odc_fabric_split_stage(self._f.h, frm, tgt, off, _buf(p), p.size, _buf(wv), C.byref(staged)))
        return bool(staged.value)

    def slot_free(self, server, client) -> bool:
        v = C.c_int()
        check(lib().odc_fabric_slot_free(self._f.h, server, client, C.byref(v)))
        return bool(v.value)

    def consume(self, server, client) -> bool:
        v = C.c_int()
        check(lib().odc_fabric_consume(self._f.h, server, client, C.byref(v)))
        return bool(v.value)

    def any_staged(self, server) -> bool:
        v = C.c_int()
        check(lib().odc_fabric_any_staged(self._f.h, server, C.byref(v)))
        return bool(v.value)

    def take_grads(self) -> List[np.ndarray]:
        out = np.zeros(self._f.elems, self._f.dtype)
        check(lib().odc_fabric_take_grads(self._f.h, _buf(out)))
        return self._f._split(out)

    def max_staged_elems(self, server) -> int:
        v = C.c_int64()
        check(lib().odc_fabric_max_staged(self._f.h, server, C.byref(v)))
        return v.value


class ShardFabric:
    """ShardFabric<T> for T in {int64, float64, float32}, shards in HBM.

    push_mode: "slot" (default) = the reference's staged protocol, bit-exact
    in every dtype; "red" = remote red.add straight into owner shards."""

    def __init__(self, ranks: int, elems: int, dtype=np.int64, device: int = 0, push_mode: str = "slot",
                 devices=None):
        """devices: single-process multi-GPU mode — simulated rank r's shards
        and slots on devices[r % len(devices)], kernels on devices[0]."""
        self.dtype = np.dtype(dtype)
        if self.dtype not in _DT:
            from .errors import ParamError

            raise ParamError("ShardFabric dtype must be int64, float64 or float32")
        h = C.c_void_p()
        devs = list(devices) if devices else [device]
        arr = (C.c_int * len(devs))(*devs)
        check(lib().odc_fabric_create_multi(ranks, elems, _DT[self.dtype], arr, len(devs), C.byref(h)))
        self.h = h
        self.ranks, self.elems = ranks, elems
        self.block = (elems + ranks - 1) // ranks
        mode = {"slot": _lib.ODC_PUSH_SLOT, "red": _lib.ODC_PUSH_RED}[push_mode]
        check(lib().odc_fabric_set_push_mode(self.h, mode))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                lib().odc_fabric_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.h = C.c_void_p()

    def state(self) -> ShardState:
        return ShardState(self)

    def _split(self, full: np.ndarray) -> List[np.ndarray]:
        out = []
        for r in range(self.ranks):
            b, n = shard_range(self.elems, self.ranks, r)
            out.append(full[b:b + n].copy())
        return out

    def _arr(self, x):
        return np.ascontiguousarray(np.asarray(x, self.dtype))

    def set_params(self, pid: str, full):
        a = self._arr(full)
        check(lib().odc_fabric_set_params(self.h, pid.encode(), _buf(a), a.size))

    def gather(self, client: int, pid: str) -> np.ndarray:
        out = np.zeros(self.elems, self.dtype)
        check(lib().odc_fabric_gather(self.h, client, pid.encode(), _buf(out)))
        return out

    def scatter_accumulate(self, client: int, grad, weight):
        g = self._arr(grad)
        w = np.asarray([weight], self.dtype)
        check(lib().odc_fabric_scatter_accumulate(self.h, client, _buf(g), g.size, _buf(w)))

    def push_slice(self, client: int, target: int, offset: int, payload, weight):
        p = self._arr(payload)
        w = np.asarray([weight], self.dtype)
        check(lib().odc_fabric_push_slice(self.h, client, target, offset, _buf(p), p.size, _buf(w)))

    def finalize_minibatch(self) -> List[np.ndarray]:
        out = np.zeros(self.elems, self.dtype)
        check(lib().odc_fabric_finalize(self.h, _buf(out)))
        return self._split(out)
