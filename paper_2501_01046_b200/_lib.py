"""ctypes binding of libneardup_b200.so (the C-ABI in include/neardup_b200.h).

The shared library is the product: every device entry point below runs the
hand-written sm_100a kernels.  There is no fallback -- if the library is
missing or fails to load, importing the device API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ND_LIB_PATH") or os.path.join(PKG, "libneardup_b200.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p

ND_OK = 0
ND_ERR_INTERNAL = 1
ND_ERR_CONFIG = 2
ND_ERR_IO = 3
ND_ERR_PREREQ = 4
ND_ERR_DEVICE = 5
ND_ERR_SHORT = 6


class NdHashFn(C.Structure):
    """nd_hash_fn == HashFunctionParams (minhash.hpp:17-25)."""

    _fields_ = [("modulus", C.c_uint32), ("base", C.c_uint32), ("base_inverse", C.c_uint32),
                ("base_power", C.c_uint32), ("reduce_factor", C.c_uint64)]


class NdParams(C.Structure):
    _fields_ = [("hash_count", C.c_uint32), ("bands", C.c_uint32), ("rows", C.c_uint32),
                ("shingle_len", C.c_uint32), ("unit", C.c_uint32), ("bucket_count", C.c_uint32),
                ("threshold_num", C.c_uint64), ("threshold_den", C.c_uint64),
                ("scale_num", C.c_uint64), ("scale_den", C.c_uint64), ("seed", C.c_uint64)]


class NdSynthSpec(C.Structure):
    _fields_ = [("doc_count", C.c_uint64), ("group_count", C.c_uint64),
                ("group_size_min", C.c_uint32), ("group_size_max", C.c_uint32),
                ("edit_num", C.c_uint64), ("edit_den", C.c_uint64), ("len_min", C.c_uint32),
                ("len_max", C.c_uint32), ("seed", C.c_uint64), ("mode", C.c_uint32),
                ("len_law", C.c_uint32), ("sigma_milli", C.c_uint32), ("threads", C.c_uint32)]


class NdDedupStats(C.Structure):
    _fields_ = [("documents", C.c_uint64), ("bucket_count", C.c_uint32),
                ("nonsingleton_cells", C.c_uint64), ("candidate_pairs", C.c_uint64),
                ("emitted_pairs", C.c_uint64), ("distinct_pairs", C.c_uint64),
                ("duplicate_groups", C.c_uint64), ("near_duplicates", C.c_uint64),
                ("removals", C.c_uint64), ("seconds", C.c_double * 6),
                ("cell_records", C.c_uint64), ("intervals", C.c_uint32)]


class NdFedsHeader(C.Structure):
    """nd_feds_header == SignatureFileHeader (sigstore.hpp:24-42)."""

    _fields_ = [("hash_count", C.c_uint32), ("bands", C.c_uint32), ("rows", C.c_uint32),
                ("bucket_count", C.c_uint32), ("shingle_len", C.c_uint32), ("unit", C.c_uint32),
                ("family_seed", C.c_uint64), ("scale_num", C.c_uint64), ("scale_den", C.c_uint64),
                ("record_count", C.c_uint64), ("source_ordinal", C.c_uint64)]


class NdCompareStageStats(C.Structure):
    """nd_compare_stage_stats == CompareStageOutput (pipeline.hpp:74-81) + extras."""

    _fields_ = [("buckets_per_pass", C.c_uint32), ("pass_count", C.c_uint32),
                ("candidate_pairs", C.c_uint64), ("emitted_pairs", C.c_uint64),
                ("gather_peak_bytes", C.c_uint64), ("records", C.c_uint64),
                ("distinct_pairs", C.c_uint64), ("seconds", C.c_double * 3),
                ("intervals", C.c_uint32)]


cpp = C.POINTER(C.c_char_p)

# name -> (restype, argtypes); every symbol include/neardup_b200.h declares
SIGNATURES = {
    "nd_version": (C.c_char_p, []),
    "nd_launch_count": (C.c_uint64, []),
    "nd_last_error_global": (C.c_char_p, []),
    "nd_derive_family": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.POINTER(NdHashFn)]),
    "nd_mod_pow": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
    "nd_is_prime_u32": (C.c_int, [C.c_uint32]),
    "nd_hash_window_direct": (C.c_int, [u32p, C.c_uint32, C.POINTER(NdHashFn), u32p]),
    "nd_roll_next": (C.c_uint32, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(NdHashFn)]),
    "nd_choose_bucket_count": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, u32p]),
    "nd_min_matches": (C.c_uint32, [C.c_uint32, C.c_uint64, C.c_uint64]),
    "nd_band_partition": (C.c_int, [C.c_uint32, C.c_uint32, u32p]),
    "nd_cell_partition": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, u64p]),
    "nd_synth_generate": (C.c_int, [C.POINTER(NdSynthSpec), u8p, u64p, u64p]),
    "nd_synth_text_device": (C.c_int, [vp, C.POINTER(NdSynthSpec), vp, vp]),
    "nd_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "nd_ctx_create_multi": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]),
    "nd_stage_records_packed": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, vp, u64p]),
    "nd_stage_compare_peer_packed": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64,
                                               C.c_uint64, u64p, u64p]),
    "nd_ctx_shard_count": (C.c_int, [vp]),
    "nd_ctx_destroy": (None, [vp]),
    "nd_last_error": (C.c_char_p, [vp]),
    "nd_ctx_set_stream": (C.c_int, [vp, vp]),
    "nd_family_upload": (C.c_int, [vp, C.POINTER(NdHashFn), C.c_uint32, C.c_uint32, C.c_uint32]),
    "nd_k1_kernel": (C.c_char_p, [vp]),
    "nd_dedup_compare_kind": (C.c_char_p, [vp]),
    "nd_k1j_source": (C.c_int64, [C.POINTER(NdHashFn), C.c_uint32, C.c_uint32, C.c_char_p,
                                  C.c_uint64]),
    "nd_k1j_source_units": (C.c_int64, [C.POINTER(NdHashFn), C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_char_p, C.c_uint64]),
    "nd_k1j_plan": (C.c_int64, [C.POINTER(NdHashFn), C.c_uint32, C.c_uint32,
                                C.POINTER(C.c_uint32), C.c_uint64]),
    "nd_signatures": (C.c_int, [vp, u8p, u64p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                u32p, u32p]),
    "nd_signatures_h2d": (C.c_int, [vp, u8p, u64p, C.c_uint64, C.c_uint32, C.c_uint32,
                                    C.c_uint32, vp, vp]),
    "nd_signatures_device": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.c_uint32, vp, vp]),
    "nd_text_units": (C.c_int, [vp, u8p, u64p, C.c_uint64, C.c_uint32, u64p, u32p]),
    "nd_band_keys": (C.c_int, [vp, u32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                               C.c_uint32, u32p]),
    "nd_compare_cells": (C.c_int, [vp, u32p, C.c_uint64, C.c_uint32, u64p, u32p, C.c_uint64,
                                   C.c_uint64, C.c_uint64, u64p]),
    "nd_pairs_fetch": (C.c_int, [vp, u32p, u32p, u32p]),
    "nd_union": (C.c_int, [vp, u32p, u32p, C.c_uint64, C.c_uint32, u64p, u64p]),
    "nd_groups_fetch": (C.c_int, [vp, u32p, u64p]),
    "nd_dedup": (C.c_int, [vp, u8p, u64p, u64p, C.c_uint64, C.POINTER(NdParams),
                           C.POINTER(NdDedupStats)]),
    "nd_dedup_device": (C.c_int, [vp, vp, vp, u64p, C.c_uint64, C.POINTER(NdParams),
                                  C.POINTER(NdDedupStats)]),
    "nd_dedup_signatures": (C.c_int, [vp, u32p, u32p, u64p, C.c_uint64, C.POINTER(NdParams),
                                      C.POINTER(NdDedupStats)]),
    "nd_dedup_fetch_pairs": (C.c_int, [vp, u64p, u64p, u32p]),
    "nd_dedup_fetch_signatures": (C.c_int, [vp, u32p, u32p]),
    "nd_dedup_fetch_groups": (C.c_int, [vp, u64p, u64p]),
    "nd_dedup_write_report": (C.c_int, [vp, C.c_char_p, C.c_uint64]),
    "nd_dedup_write_report_ex": (C.c_int, [vp, C.c_char_p, C.c_uint64, C.c_int]),
    "nd_ingest_last_error": (C.c_char_p, []),
    "nd_jsonl_load": (C.c_int, [C.c_char_p, C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                C.c_uint32, C.c_int, C.POINTER(vp)]),
    "nd_jsonl_counts": (None, [vp, u64p, u64p, u64p, u64p]),
    "nd_jsonl_rejects": (C.c_int, [vp, u64p, u32p]),
    "nd_jsonl_documents": (C.c_int, [vp, C.c_uint64, u8p, u64p, u64p, u64p]),
    "nd_jsonl_free": (None, [vp]),
    "nd_nfc_normalize": (C.c_int, [u8p, C.c_uint64, u8p, C.c_uint64, u64p]),
    "nd_codepoint_count": (C.c_uint64, [u8p, C.c_uint64]),
    "nd_parse_jsonl_line": (C.c_int, [C.c_char_p, C.c_uint64, C.c_char_p, u32p, u8p, C.c_uint64,
                                      u64p]),
    "nd_parse_jsonl_line_mode": (C.c_int, [C.c_char_p, C.c_uint64, C.c_char_p, C.c_int, u32p,
                                           u8p, C.c_uint64, u64p]),
    "nd_feds_write": (C.c_int, [C.c_char_p, C.POINTER(NdFedsHeader), u64p, u32p, u32p,
                                C.c_uint64, C.c_int]),
    "nd_feds_read_header": (C.c_int, [C.c_char_p, C.POINTER(NdFedsHeader)]),
    "nd_feds_read": (C.c_int, [C.c_char_p, u64p, u32p, u32p]),
    "nd_pairs_write": (C.c_int, [C.c_char_p, u64p, u64p, u32p, C.c_uint64, C.c_int]),
    "nd_pairs_read": (C.c_int, [C.c_char_p, u64p, u64p, u32p, u64p]),
    "nd_plan_gather": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                 C.c_uint32, u32p, u32p]),
    "nd_hash_file": (C.c_int, [vp, u8p, u64p, u64p, C.c_uint64, C.POINTER(NdFedsHeader),
                               C.c_char_p, C.c_int]),
    "nd_compare_stage": (C.c_int, [vp, cpp, C.c_uint32, C.POINTER(NdFedsHeader), C.c_uint64,
                                   C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                   C.c_char_p, C.c_int, C.POINTER(NdCompareStageStats)]),
    "nd_set_hbm_budget": (C.c_int, [vp, C.c_uint64]),
    "nd_union_stage": (C.c_int, [vp, cpp, C.c_uint32, C.c_uint64, C.c_uint64, C.c_char_p,
                                 C.c_int, C.POINTER(NdDedupStats)]),
    "nd_stage_cell_records": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                        vp, vp]),
    "nd_stage_compare": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, vp, vp, C.c_uint64,
                                   C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p]),
    "nd_peer_export": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, u8p]),
    "nd_peer_open": (C.c_int, [vp, u8p, u64p, C.c_uint32, C.c_uint32]),
    "nd_stage_compare_peer": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.c_uint64, u64p, u64p]),
    "nd_peer_close": (C.c_int, [vp]),
    "nd_peer_export_gjoin": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.c_uint64, C.c_uint64, u8p]),
    "nd_stage_gjoin_peer": (C.c_int, [vp, C.c_uint32, u64p, u64p]),
    "nd_stage_cell_hist": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, vp]),
    "nd_stage_pairs_copy": (C.c_int, [vp, vp, vp, vp]),
    "nd_stage_union": (C.c_int, [vp, vp, vp, vp, C.c_uint64, C.c_uint64,
                                 C.POINTER(NdDedupStats)]),
}

_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Loads the in-tree library (building it first if absent and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            from . import build as _build

            _build.build()
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class NdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ConfigError(NdError):
    pass


class IoError(NdError):
    pass


class PrerequisiteError(NdError):
    pass


class DeviceError(NdError):
    pass


class ShortDocumentError(NdError):
    pass


_CODE_TO_EXC = {ND_ERR_CONFIG: ConfigError, ND_ERR_IO: IoError, ND_ERR_PREREQ: PrerequisiteError,
                ND_ERR_DEVICE: DeviceError, ND_ERR_SHORT: ShortDocumentError}
ERRORS = _CODE_TO_EXC


def check(rc: int, ctx=None) -> None:
    if rc == ND_OK:
        return
    lib = load()
    msg = (lib.nd_last_error(ctx) if ctx else lib.nd_last_error_global()) or b""
    raise _CODE_TO_EXC.get(rc, NdError)(rc, msg.decode(errors="replace"))
