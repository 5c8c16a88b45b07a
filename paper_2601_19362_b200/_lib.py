"""ctypes binding of libodc.so (include/odc/odc.h).

The product path has no fallback: if the in-tree library is missing this
module raises on first use, so a GPU box without the built extension fails
loudly instead of silently computing on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ODC_LIB_PATH") or os.path.join(PKG, "lib", "libodc.so")  # override: A/B variant builds

ODC_OK, ODC_ERR_PARAM, ODC_ERR_INFEASIBLE, ODC_ERR_INVARIANT = 0, 2, 3, 4
ODC_ERR_PROTOCOL, ODC_ERR_STATE, ODC_ERR_MODE, ODC_ERR_CUDA, ODC_ERR_TIMEOUT, ODC_ERR_RANGE = 5, 6, 7, 8, 9, 10
ODC_FLAG_TIMEOUT, ODC_FLAG_FIXED_RANGE, ODC_FLAG_FIXED_UNDERFLOW = 1, 2, 4
ODC_I64, ODC_F64, ODC_F32, ODC_BF16 = 0, 1, 2, 3
ODC_PUSH_RED, ODC_PUSH_SLOT, ODC_PUSH_FIXED = 0, 1, 2
ODC_FIXED_FRAC_BITS_DEFAULT = 40
ODC_FETCH_TMA, ODC_FETCH_LDG, ODC_FETCH_CE = 0, 1, 2

i64, i64p, vp = C.c_int64, C.POINTER(C.c_int64), C.c_void_p


class OdcConfig(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("device", C.c_int), ("n_layers", C.c_int),
                ("layer_elems", i64p), ("push_mode", C.c_int), ("fetch_ctas", C.c_int), ("push_ctas", C.c_int),
                ("timeout_s", C.c_double), ("fetch_engine", C.c_int), ("fixed_frac_bits", C.c_int)]


class OdcAdamCfg(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("step", C.c_int)]


# symbol -> (restype, argtypes); this table doubles as the export list the
# CPU test checks against include/odc/odc.h
SIGNATURES = {
    "odc_abi_version": (C.c_int, []),
    "odc_last_error": (C.c_char_p, []),
    "odc_kernel_launches": (C.c_uint64, []),
    "odc_shard_range": (C.c_int, [i64, C.c_int, C.c_int, i64p, i64p]),
    "odc_fabric_create": (C.c_int, [C.c_int, i64, C.c_int, C.c_int, C.POINTER(vp)]),
    "odc_fabric_create_multi": (C.c_int, [C.c_int, i64, C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]),
    "odc_fabric_destroy": (C.c_int, [vp]),
    "odc_fabric_set_push_mode": (C.c_int, [vp, C.c_int]),
    "odc_fabric_set_params": (C.c_int, [vp, C.c_char_p, vp, i64]),
    "odc_fabric_gather": (C.c_int, [vp, C.c_int, C.c_char_p, vp]),
    "odc_fabric_scatter_accumulate": (C.c_int, [vp, C.c_int, vp, i64, vp]),
    "odc_fabric_push_slice": (C.c_int, [vp, C.c_int, C.c_int, i64, vp, i64, vp]),
    "odc_fabric_finalize": (C.c_int, [vp, vp]),
    "odc_fabric_split_stage": (C.c_int, [vp, C.c_int, C.c_int, i64, vp, i64, vp, C.POINTER(C.c_int)]),
    "odc_fabric_slot_free": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "odc_fabric_consume": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "odc_fabric_any_staged": (C.c_int, [vp, C.c_int, C.POINTER(C.c_int)]),
    "odc_fabric_take_grads": (C.c_int, [vp, vp]),
    "odc_fabric_max_staged": (C.c_int, [vp, C.c_int, i64p]),
    "odc_ctx_create": (C.c_int, [C.POINTER(OdcConfig), C.POINTER(vp)]),
    "odc_ctx_destroy": (C.c_int, [vp]),
    "odc_ctx_export": (C.c_int, [vp, vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "odc_ctx_import": (C.c_int, [vp, C.c_int, vp, C.c_size_t]),
    "odc_ctx_import_ctx": (C.c_int, [vp, C.c_int, vp]),
    "odc_ctx_ready": (C.c_int, [vp]),
    "odc_ctx_arena_bytes": (C.c_int, [vp, i64p]),
    "odc_set_params": (C.c_int, [vp, C.c_int, vp, vp]),
    "odc_fetch": (C.c_int, [vp, C.c_int, vp, vp]),
    "odc_fetch_master": (C.c_int, [vp, C.c_int, vp, vp]),
    "odc_push": (C.c_int, [vp, C.c_int, vp, C.c_int, C.c_float, vp]),
    "odc_push_slice": (C.c_int, [vp, C.c_int, C.c_int, i64, vp, i64, C.c_float, vp]),
    "odc_minibatch_end": (C.c_int, [vp, vp]),
    "odc_read_grad_shard": (C.c_int, [vp, C.c_int, vp, vp]),
    "odc_read_master_shard": (C.c_int, [vp, C.c_int, vp, vp]),
    "odc_adam_step": (C.c_int, [vp, C.POINTER(OdcAdamCfg), vp]),
    "odc_ctx_check": (C.c_int, [vp, vp]),
    "odc_ctx_flags": (C.c_int, [vp, C.POINTER(C.c_uint64), vp]),
    "odc_ctx_epoch": (C.c_int64, [vp]),
    "odc_copy_segments": (C.c_int, [C.c_int, C.POINTER(vp), C.POINTER(vp), i64p, C.c_int, vp]),
    "odc_l2_flush": (C.c_int, [vp, i64, vp]),
    "odc_gemm_set_raster": (C.c_int, [C.c_int, C.c_int]),
    "odc_gemm_gate_up_swiglu": (C.c_int, [vp, vp, vp, vp, i64, i64, i64, vp]),
    "odc_gemm_bf16": (C.c_int, [vp, vp, vp, vp, i64, i64, i64, i64, i64, i64, C.c_int, C.c_int, C.c_int, C.c_int,
                                vp]),
    "odc_attn_fwd": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, i64, C.c_int, C.c_int, C.c_int, C.c_float, vp]),
    "odc_attn_bwd": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, i64, C.c_int, C.c_int, C.c_int,
                               C.c_float, vp]),
    "odc_attn_bwd_qkv": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, i64, C.c_int, C.c_int, C.c_int,
                                   C.c_float, vp]),
    "odc_w_rmsnorm_fwd": (C.c_int, [vp, vp, vp, vp, i64, C.c_int, C.c_float, vp]),
    "odc_w_rmsnorm_bwd": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, i64, C.c_int, vp]),
    "odc_w_qkv_rope_fwd": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, i64, C.c_int, C.c_int, C.c_int, vp]),
    "odc_w_qkv_rope_bwd": (C.c_int, [vp, vp, vp, vp, vp, vp, i64, C.c_int, C.c_int, C.c_int, vp]),
    "odc_w_col_sum": (C.c_int, [vp, vp, i64, C.c_int, vp]),
    "odc_w_swiglu_fwd": (C.c_int, [vp, vp, i64, C.c_int, vp]),
    "odc_w_swiglu_bwd": (C.c_int, [vp, vp, vp, i64, C.c_int, vp]),
    "odc_w_ce_fwd_bwd": (C.c_int, [vp, vp, i64, i64, C.c_float, vp, vp]),
    "odc_plan_json": (C.c_int, [C.c_int, i64p, i64, C.c_int, C.c_int, i64, C.c_double, C.c_double, C.c_int,
                                C.c_uint64, C.c_char_p, i64, i64p]),
    "odc_plan_flat": (C.c_int, [C.c_int, i64p, i64, C.c_int, C.c_int, i64, C.c_double, C.c_double, C.c_uint64,
                                i64p, i64, i64p]),
    "odc_kk_partition_json": (C.c_int, [C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, C.c_char_p, i64,
                                        i64p]),
    "odc_generate_synthetic": (C.c_int, [C.c_int, C.c_double, C.c_double, i64, i64, C.c_uint64, C.c_double,
                                         i64p]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libodc.so not built at {LIB_PATH}: run `python -m paper_2601_19362_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.odc_abi_version() != 5:
            raise ImportError("libodc.so ABI version mismatch")
        _lib = L
    return _lib


def check(code: int):
    """Raise the Python counterpart of the reference exception for `code`."""
    if code == ODC_OK:
        return
    msg = lib().odc_last_error().decode(errors="replace")
    from . import errors

    raise errors.from_status(code, msg)


def kernel_launches() -> int:
    return int(lib().odc_kernel_launches())
