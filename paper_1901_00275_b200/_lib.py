"""ctypes binding of libvlqgpu.so (include/vlq_gpu.h).

The shared library is the product: every compute call below goes to hand-
written sm_100a kernels.  There is no fallback -- if the library is missing
or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvlqgpu.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "vlq_gpu.h")

c_u32, c_u64, c_i32, c_f32, c_vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_float, ctypes.c_void_p


class VlqConfig(ctypes.Structure):
    _fields_ = [("device", c_i32), ("shard_rank", c_i32), ("shard_count", c_i32),
                ("workspace_bytes", c_u64), ("max_tile", c_u32), ("force_exact", c_i32)]


class VlqStats(ctypes.Structure):
    _fields_ = [("launches", c_u64), ("tiles", c_u64), ("flagged", c_u64), ("tc_fallbacks", c_u64),
                ("phase_ms", ctypes.c_double * 8)]


PHASES = ["coarse", "first_level", "second_level", "term5", "scan", "rescore", "fallback", "output"]


class VlqInfo(ctypes.Structure):
    _fields_ = [("dim", c_u32), ("k", c_u32), ("n", c_u32), ("m", c_u32), ("clamp_lambda", c_i32),
                ("lambda_lo", c_f32), ("lambda_hi", c_f32), ("ntotal", c_u64), ("local_entries", c_u64)]


_SIGS = {
    "vlq_last_error": (ctypes.c_char_p, []),
    "vlq_engine_create": (c_i32, [ctypes.POINTER(VlqConfig), ctypes.POINTER(c_vp)]),
    "vlq_engine_destroy": (None, [c_vp]),
    "vlq_engine_load_vlq1": (c_i32, [c_vp, ctypes.c_char_p]),
    "vlq_engine_save_vlq1": (c_i32, [c_vp, ctypes.c_char_p, c_i32]),
    "vlq_engine_set_model": (c_i32, [c_vp, c_u32, c_u32, c_u32, c_u32, c_i32, c_f32, c_f32, c_vp, c_vp, c_vp, c_vp,
                                     c_vp]),
    "vlq_engine_add": (c_i32, [c_vp, c_vp, c_u64, c_u32]),
    "vlq_engine_add_vecs": (c_i32, [c_vp, ctypes.c_char_p, c_u64]),
    "vlq_engine_train": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_u32, c_u32, c_u32, c_u32, c_u64, c_i32]),
    "vlq_train_kmeans": (c_i32, [c_i32, c_vp, c_u64, c_u32, c_u32, c_u32, c_u64, c_vp, c_vp]),
    "vlq_engine_search": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_u32, c_f32, c_u32, c_vp, c_vp, c_vp]),
    "vlq_engine_search_device": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_f32, c_u32, c_vp, c_vp, c_vp, c_vp]),
    "vlq_engine_set_tuning": (c_i32, [c_vp, ctypes.c_char_p, ctypes.c_int64]),
    "vlq_engine_ivf_build": (c_i32, [c_vp, c_vp, c_u64, c_u32]),
    "vlq_engine_ivf_build_synthetic": (c_i32, [c_vp, c_u64, c_u32, c_f32, c_u64]),
    "vlq_engine_ivf_search": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_u32, c_u32, c_vp, c_vp, c_vp]),
    "vlq_engine_ivf_search_device": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_u32, c_vp, c_vp, c_vp, c_vp]),
    "vlq_engine_ivf_get_lists": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "vlq_engine_search_coarse_device": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_vp, c_vp]),
    "vlq_engine_search_fine_device": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_f32, c_u32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "vlq_engine_search_select_device": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_f32, c_vp, c_vp, c_vp]),
    "vlq_engine_search_fine_sel_device": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_f32, c_u32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                                  c_vp]),
    "vlq_w2": (c_u32, [c_u32, c_f32, c_u32]),
    "vlq_shard_of_cell": (c_u32, [c_u32, c_u32]),
    "vlq_code_banks": (c_i32, [c_vp, c_u32, c_vp]),
    "vlq_engine_sync": (c_i32, [c_vp, c_vp]),
    "vlq_engine_info": (c_i32, [c_vp, ctypes.POINTER(VlqInfo)]),
    "vlq_engine_add_synthetic": (c_i32, [c_vp, c_u64, c_u32, c_f32, c_u64]),
    "vlq_gen_synthetic_device": (c_i32, [c_i32, c_u64, c_u64, c_u32, c_u32, c_f32, c_u64, c_vp, c_vp]),
    "vlq_brute_force_gt_synthetic": (c_i32, [c_i32, c_u64, c_u32, c_u32, c_f32, c_u64, c_vp, c_u64, c_u32, c_vp]),
    "vlq_engine_set_profiling": (c_i32, [c_vp, c_i32]),
    "vlq_engine_get_stats": (c_i32, [c_vp, ctypes.POINTER(VlqStats)]),
    "vlq_engine_reset_stats": (c_i32, [c_vp]),
    "vlq_engine_get_lists": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "vlq_engine_get_cells": (c_i32, [c_vp, c_vp, c_u32, c_vp, c_vp, c_vp, c_vp]),
    "vlq_group_create": (c_i32, [c_vp, c_u32, c_u32, c_vp, ctypes.POINTER(c_vp)]),
    "vlq_group_destroy": (None, [c_vp]),
    "vlq_group_size": (c_u32, [c_vp]),
    "vlq_group_load_vlq1": (c_i32, [c_vp, ctypes.c_char_p]),
    "vlq_group_set_model": (c_i32, [c_vp, c_u32, c_u32, c_u32, c_u32, c_i32, c_f32, c_f32, c_vp, c_vp, c_vp, c_vp,
                                    c_vp]),
    "vlq_group_add": (c_i32, [c_vp, c_vp, c_u64, c_u32]),
    "vlq_group_add_synthetic": (c_i32, [c_vp, c_u64, c_u32, c_f32, c_u64]),
    "vlq_group_search": (c_i32, [c_vp, c_vp, c_u64, c_u32, c_u32, c_f32, c_u32, c_vp, c_vp, c_vp]),
    "vlq_group_set_queries": (c_i32, [c_vp, c_vp, c_u64, c_u32]),
    "vlq_group_search_resident": (c_i32, [c_vp, c_u32, c_f32, c_u32, ctypes.POINTER(c_f32)]),
    "vlq_group_results": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "vlq_group_info": (c_i32, [c_vp, c_u32, ctypes.POINTER(VlqInfo)]),
    "vlq_group_set_profiling": (c_i32, [c_vp, c_i32]),
    "vlq_group_get_stats": (c_i32, [c_vp, c_u32, ctypes.POINTER(VlqStats), c_i32]),
    "vlq_engine_get_model": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "vlq_engine_encode": (c_i32, [c_vp, c_vp, c_u64, c_vp, c_vp, c_vp, c_vp]),
    "vlq_merge_topk_device": (c_i32, [c_i32, c_vp, c_vp, c_u32, c_u64, c_u32, c_vp, c_vp, c_vp]),
    "vlq_brute_force_gt": (c_i32, [c_i32, c_vp, c_u64, c_vp, c_u64, c_u32, c_u32, c_vp]),
    "vlq_gen_synthetic": (c_i32, [c_u64, c_u32, c_u32, c_f32, c_u64, c_vp]),
}

_LIB = None


def header_functions() -> list[str]:
    """Names of every function include/vlq_gpu.h declares."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vlq_[a-z0-9_]+)\s*\(", text)))


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA engine library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(lib().vlq_last_error().decode())
