"""ctypes binding to oracle/_ref/libodcref.so — TEST INFRASTRUCTURE ONLY.

The library is the unmodified reference simulator (built by oracle/Makefile
from /root/reference/proj/src) plus our extern "C" shim oracle/ref_driver.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline legs
use it. ``available()`` is False when _ref was not built (e.g. no
/root/reference in this container and no prebuilt copy shipped).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libodcref.so")
STRATEGY_CODE = {"local-sort": 0, "lb-micro": 1, "lb-mini": 2, "verl-native": 3, "verl-optimized": 4}
_lib: Optional[C.CDLL] = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        i64p = C.POINTER(C.c_int64)
        L.ref_plan_json.argtypes = [C.c_int, i64p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_double,
                                    C.c_double, C.c_int, C.c_uint64, C.c_char_p, C.c_int64, i64p]
        L.ref_plan_seconds.argtypes = [C.c_int, i64p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_double,
                                       C.c_double, C.c_int]
        L.ref_plan_seconds.restype = C.c_double
        L.ref_kk_partition_json.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_char_p, C.c_int64, i64p]
        L.ref_generate_synthetic.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int64, C.c_int64,
                                             C.c_uint64, C.c_double, i64p]
        for suf, ct in (("i64", C.c_int64), ("f64", C.c_double), ("f32", C.c_float)):
            fn = getattr(L, f"ref_fabric_script_{suf}")
            fn.argtypes = [C.c_int, C.c_int64, C.c_int, C.POINTER(C.c_int), C.POINTER(ct), C.POINTER(ct),
                           C.POINTER(ct)]
        L.ref_push_slice_status.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int64]
        L.ref_run_schedule_i64.argtypes = [C.c_int, C.c_int64, C.c_int, C.POINTER(C.c_int), i64p, i64p,
                                           C.c_uint64, i64p]
        L.ref_run_schedule_i64.restype = C.c_int64
        L.ref_fabric_seconds_f32.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int]
        L.ref_fabric_seconds_f32.restype = C.c_double
        L.ref_fabric_seconds_f32_mt.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_fabric_seconds_f32_mt.restype = C.c_double
        L.ref_step_new.argtypes = [C.c_int, C.c_int, i64p]
        L.ref_step_new.restype = C.c_void_p
        L.ref_step_free.argtypes = [C.c_void_p]
        L.ref_step_run.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_int]
        L.ref_step_run.restype = C.c_double
        L.ref_runtime.argtypes = [C.c_int, i64p, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_double,
                                  C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _i64(a: Sequence[int]):
    arr = np.ascontiguousarray(np.asarray(a, np.int64))
    return arr, arr.ctypes.data_as(C.POINTER(C.c_int64))


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def plan_json(strategy: str, lens: Sequence[int], devices: int, minibs: int, budget: int,
              alpha: float = 1.0, beta: float = 0.0, layers: int = 1, seed: int = 0) -> str:
    arr, p = _i64(lens)
    need = C.c_int64(0)
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        rc = lib().ref_plan_json(STRATEGY_CODE[strategy], p, len(arr), devices, minibs, budget, alpha, beta,
                                 layers, seed, buf, cap, C.byref(need))
        if rc != 0:
            raise RefError(rc, buf.value.decode())
        if need.value < cap:
            return buf.value.decode()
        cap = need.value + 1


def plan_seconds(strategy: str, lens, devices, minibs, budget, alpha=1.0, beta=0.0, iters=1) -> float:
    arr, p = _i64(lens)
    return lib().ref_plan_seconds(STRATEGY_CODE[strategy], p, len(arr), devices, minibs, budget, alpha, beta,
                                  iters)


def kk_partition(costs: Sequence[float], k: int, equal_size: bool, brute: bool = False) -> dict:
    arr = np.ascontiguousarray(np.asarray(costs, np.float64))
    cap = 1 << 16
    buf = C.create_string_buffer(cap)
    need = C.c_int64(0)
    rc = lib().ref_kk_partition_json(arr.ctypes.data_as(C.POINTER(C.c_double)), len(arr), k, int(equal_size),
                                     int(brute), buf, cap, C.byref(need))
    if rc != 0:
        raise RefError(rc, buf.value.decode())
    return json.loads(buf.value.decode())


def generate_synthetic(dist, n, cap, seed, scale=1.0) -> List[int]:
    kind = {"lognormal": 0, "pareto": 1, "uniform": 2}[dist[0]]
    out = np.zeros(n, np.int64)
    rc = lib().ref_generate_synthetic(kind, float(dist[1]), float(dist[2]), n, cap, seed, scale,
                                      out.ctypes.data_as(C.POINTER(C.c_int64)))
    if rc != 0:
        raise RefError(rc, "generate_synthetic failed")
    return out.tolist()


def fabric_script(ranks: int, elems: int, pushes, dtype) -> np.ndarray:
    """pushes = [(client, grad, weight)]: ShardFabric<T>::scatter_accumulate
    for each, then finalize_minibatch(); returns the concatenated shards."""
    dt = np.dtype(dtype)
    suf, ct = {np.dtype(np.int64): ("i64", C.c_int64), np.dtype(np.float64): ("f64", C.c_double),
               np.dtype(np.float32): ("f32", C.c_float)}[dt]
    n = len(pushes)
    clients = np.asarray([p[0] for p in pushes] or [0], np.int32)
    grads = np.ascontiguousarray(np.stack([np.asarray(p[1], dt) for p in pushes]) if n else np.zeros((1, elems), dt))
    weights = np.asarray([p[2] for p in pushes] or [0], dt)
    out = np.zeros(elems, dt)
    rc = getattr(lib(), f"ref_fabric_script_{suf}")(
        ranks, elems, n, clients.ctypes.data_as(C.POINTER(C.c_int)), grads.ctypes.data_as(C.POINTER(ct)),
        weights.ctypes.data_as(C.POINTER(ct)), out.ctypes.data_as(C.POINTER(ct)))
    if rc != 0:
        raise RefError(rc, "fabric script failed")
    return out


def push_slice_status(ranks, elems, client, target, offset, length) -> int:
    return lib().ref_push_slice_status(ranks, elems, client, target, offset, length)


def run_schedule_i64(ranks, elems, pushes, seed):
    n = len(pushes)
    clients = np.asarray([p[0] for p in pushes] or [0], np.int32)
    grads = np.ascontiguousarray(np.stack([np.asarray(p[1], np.int64) for p in pushes]) if n
                                 else np.zeros((1, elems), np.int64))
    weights = np.asarray([p[2] for p in pushes] or [0], np.int64)
    out = np.zeros(elems, np.int64)
    peak = lib().ref_run_schedule_i64(ranks, elems, n, clients.ctypes.data_as(C.POINTER(C.c_int)),
                                      grads.ctypes.data_as(C.POINTER(C.c_int64)),
                                      weights.ctypes.data_as(C.POINTER(C.c_int64)), seed,
                                      out.ctypes.data_as(C.POINTER(C.c_int64)))
    return out, peak


def fabric_seconds_f32(ranks, elems, gathers_per_client, pushes_per_client, iters) -> float:
    return lib().ref_fabric_seconds_f32(ranks, elems, gathers_per_client, pushes_per_client, iters)


def fabric_seconds_f32_mt(ranks, elems, gathers_per_client, pushes_per_client, iters, threads) -> float:
    """Wall seconds for `threads` independent units on `threads` host threads."""
    return lib().ref_fabric_seconds_f32_mt(ranks, elems, gathers_per_client, pushes_per_client, iters, threads)


def runtime(strategy, lens, devices, minibs, budget, alpha=1.0, beta=0.0, layers=1):
    arr, p = _i64(lens)
    tot, bub = C.c_double(0), C.c_double(0)
    rc = lib().ref_runtime(STRATEGY_CODE[strategy], p, len(arr), devices, minibs, budget, alpha, beta, layers,
                           C.byref(tot), C.byref(bub))
    if rc != 0:
        raise RefError(rc, "runtime failed")
    return tot.value, bub.value


class RefStep:
    """The reference CPU path of one ODC minibatch step (ref_driver.cpp
    ref_step_*): one ShardFabric<float> per FSDP unit at its true size; per
    step, every client gathers each unit twice and scatter_accumulates once per
    microbatch, then finalize_minibatch. run() returns measured wall seconds."""

    def __init__(self, ranks: int, unit_elems: Sequence[int]):
        arr, p = _i64(unit_elems)
        self.ranks = ranks
        self.h = lib().ref_step_new(ranks, len(arr), p)
        if not self.h:
            raise RefError(9, "ref_step_new failed (host memory?)")

    def run(self, micro_per_client: Sequence[int], threads: int) -> float:
        m = (C.c_int * self.ranks)(*[int(x) for x in micro_per_client])
        t = lib().ref_step_run(self.h, m, int(threads))
        if t < 0:
            raise RefError(9, "ref_step_run failed")
        return t

    def close(self):
        if self.h:
            lib().ref_step_free(self.h)
            self.h = None

    __del__ = close
