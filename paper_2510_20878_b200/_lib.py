"""ctypes binding of libharag.so (include/harag.h) — marshalling only.

Every function here has the C name and signature of include/harag.h.  The
library is loaded eagerly; if it is missing the import fails loudly: there is
no CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HARAG_LIB") or os.path.join(_HERE, "libharag.so")  # HARAG_LIB: tuning variants only

HR_OK, HR_EINVAL, HR_ENOMEM, HR_ECUDA, HR_ENOTFOUND, HR_ECORRUPT, HR_ESTATE = range(7)
STATUS_NAMES = {0: "HR_OK", 1: "HR_EINVAL", 2: "HR_ENOMEM", 3: "HR_ECUDA", 4: "HR_ENOTFOUND",
                5: "HR_ECORRUPT", 6: "HR_ESTATE"}
HR_BF16, HR_FP16 = 0, 1
PASS16, INT8, FP8E4M3, FP8E5M2, GSE8, INT4, MXFP8 = range(7)
SCHEMES = {"PASS16": PASS16, "INT8": INT8, "FP8E4M3": FP8E4M3, "FP8E5M2": FP8E5M2, "GSE8": GSE8, "INT4": INT4,
           "MXFP8": MXFP8}
T_HBM, T_PIN, T_PAGE, T_DISK = 0, 1, 2, 3
R_HBM, R_PIN, R_PAGE, R_BACKING, R_FILE = 1, 2, 4, 8, 16


class Config(C.Structure):
    _fields_ = [
        ("L", C.c_uint32), ("H", C.c_uint32), ("D", C.c_uint32), ("T", C.c_uint32),
        ("dtype", C.c_uint32), ("group", C.c_uint32), ("gse_ebits", C.c_uint32), ("gse_mbits", C.c_uint32),
        ("n_ladder", C.c_uint32), ("ladder", C.c_uint32 * 6), ("tau", C.c_double * 6),
        ("hbm_budget", C.c_uint64), ("pin_budget", C.c_uint64),
        ("backing_pinned", C.c_int32), ("keep_backing", C.c_int32), ("demand_mode", C.c_int32),
        ("decay_shift", C.c_uint32), ("bench_alias_R", C.c_uint32),
        ("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("staging_slots", C.c_uint32),
        ("disk_backing", C.c_int32), ("page_budget", C.c_uint64), ("numa_bind", C.c_int32),
        ("guard", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("requests", C.c_uint64), ("hits", C.c_uint64 * 3), ("bytes_out", C.c_uint64),
        ("bytes_hbm_alg", C.c_uint64), ("bytes_h2d", C.c_uint64), ("kernel_launches", C.c_uint64),
        ("migrations_in", C.c_uint64), ("migrations_out", C.c_uint64), ("failed_promotions", C.c_uint64),
        ("kernel_ms", C.c_double), ("timed_launches", C.c_uint64), ("hbm_used", C.c_uint64),
        ("pin_used", C.c_uint64), ("h2d_ms", C.c_double), ("h2d_items", C.c_uint64),
        ("bytes_migrated", C.c_uint64), ("hits_disk", C.c_uint64), ("host_ms", C.c_double),
        ("quant_ms", C.c_double), ("quant_launches", C.c_uint64),
    ]


SRC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                      "(there is no fallback path)")
lib = C.CDLL(LIB_PATH)

P, U32, U64, I32, DBL, SZ = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double, C.c_size_t
PU32, PU64, PI64 = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_int64)
PP = C.POINTER(C.c_void_p)

_SIGS = {
    "hr_last_error": (C.c_char_p, []),
    "hr_abi_version": (U32, []),
    "hr_config_default": (None, [C.POINTER(Config)]),
    "hr_store_create": (I32, [C.POINTER(Config), C.POINTER(P)]),
    "hr_store_destroy": (None, [P]),
    "hr_build_store": (I32, [P, U32, PU64, SRC_FN, P, P]),
    "hr_build_begin": (I32, [P, U32, PU64]),
    "hr_build_begin_schemes": (I32, [P, U32, PU64, PU32]),
    "hr_build_put": (I32, [P, U32, P, P, P]),
    "hr_build_put_batch": (I32, [P, U32, PU32, PP, PP, P]),
    "hr_build_end": (I32, [P, P]),
    "hr_kv_bytes": (SZ, [P, U32]),
    "hr_assemble_kv": (I32, [P, U32, U32, PU32, C.POINTER(P), C.POINTER(P), P]),
    "hr_hotness_delta": (I32, [P, C.POINTER(PI64), PU32]),
    "hr_replace": (I32, [P, P]),
    "hr_attend": (I32, [P, U32, U32, PU32, P, U32, U32, P, P, C.c_float, P, P]),
    "hr_attend_layers": (I32, [P, U32, U32, PU32, U32, U32, P, U32, U32, P, P, C.c_float, P, P]),
    "hr_attend_prefill": (I32, [P, U32, U32, PU32, U32, U32, P, P, P, U32, U32, P, P, C.c_float, P]),
    "hr_store_save": (I32, [P, C.c_char_p]),
    "hr_build_from_file": (I32, [P, C.c_char_p, P]),
    "hr_item_info": (I32, [P, U32, PU32, PU32, PU64]),
    "hr_item_rank": (I32, [P, U32, PU32]),
    "hr_item_residency": (I32, [P, U32, PU32]),
    "hr_store_local_cpus": (I32, [P, C.POINTER(C.c_int32), U32, PU32]),
    "hr_placement_hash": (I32, [P, PU64]),
    "hr_export_item": (I32, [P, U32, P, SZ, C.POINTER(SZ)]),
    "hr_store_stats": (I32, [P, C.POINTER(Stats)]),
    "hr_set_timing": (I32, [P, I32]),
    "hr_last_call_ms": (I32, [P, C.POINTER(C.c_double)]),
    "hr_reset_stats": (I32, [P]),
    "hr_policy_rank": (I32, [U32, PU64, PU32]),
    "hr_policy_assign": (I32, [U32, PU64, U32, PU32, C.POINTER(C.c_double), PU32]),
    "hr_policy_lists_bytes": (I32, [U32, PU32, PU64, U64, U64, PU32]),
    "hr_policy_lists_fraction": (I32, [U32, PU32, DBL, DBL, DBL, PU32]),
    "hr_policy_lists_bytes4": (I32, [U32, PU32, PU64, U64, U64, U64, PU32]),
    "hr_policy_count": (I32, [U32, U32, PU32, U32, U64, U32, U32, PI64]),
    "hr_policy_epoch": (I32, [U32, PU64, PI64, U32]),
    "hr_item_bytes": (I32, [C.POINTER(Config), U32, PU64]),
    "hr_exponent_histogram": (I32, [U32, P, U64, P, P]),
    "hr_scheme_error": (I32, [C.POINTER(Config), U32, P, C.POINTER(C.c_double), P]),
    "hr_guard_stats": (I32, [C.POINTER(Config), P, P, P]),
    "hr_policy_guard": (I32, [U32, PU32, PU64, U32, PU32, PU32]),
    "hr_alg2_create": (I32, [U32, PU32, PU64, U64, U64, U64, C.POINTER(P)]),
    "hr_alg2_access": (I32, [P, U32, PU32, PU32, PU32, U32, PU32]),
    "hr_alg2_set_lists": (I32, [P, PU32]),
    "hr_alg2_resident": (I32, [P, U32, PU32, U32, PU32]),
    "hr_alg2_destroy": (None, [P]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


class HaragError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def check(status: int) -> None:
    if status != HR_OK:
        raise HaragError(status, lib.hr_last_error().decode(errors="replace"))


def default_config() -> Config:
    c = Config()
    lib.hr_config_default(C.byref(c))
    return c
